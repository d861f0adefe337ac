#!/usr/bin/env python
"""Cost of the search precision modes on one frame (fsk_deform, device-resident inputs).

mixed (default: fp32 pass + exact-replay fp64 escalation), mixed-fast (fused fp64 escalation), fp32 (ablation), fp64 (every solve in float64,
transform-grid J0, fused arithmetic) and exact64 (every solve in float64 replaying the
reference's operation order, weight-grid J0 — bit-identical to the oracle). Prints one JSON
line per mode: solves/s, ms per frame, and (exact64 against fp64/mixed) the converged-mask
agreement on this workload.

  python scripts/precision_modes.py [--grid 32,32,32 --points 200000 --steps 20]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_15601_b200 import synthetic as S  # noqa: E402
from paper_2211_15601_b200.deformer import Deformer, SearchOptions  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", default="32,32,32")
    ap.add_argument("--points", type=int, default=200_000)
    ap.add_argument("--max-iters", type=int, default=50)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--seed", type=int, default=0)
    a = ap.parse_args()
    dims = tuple(int(v) for v in a.grid.split(","))
    sc = S.make_scene(dims, a.points, seed=a.seed)
    D = Deformer(0)
    dev = torch.device("cuda", 0)
    w, B, x = (torch.from_numpy(v).to(dev) for v in (sc.weights, sc.bones, sc.points))
    n, nb = a.points, sc.n_bones
    buf = D.alloc_roots(n, nb)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    dense = {}
    for mode in ("mixed", "mixed-fast", "fp32", "fp64", "exact64"):
        o = SearchOptions(a.max_iters, **{k: v for k, v in sc.search_options(a.max_iters).items() if k != "max_iters"})
        o.precision = mode
        for _ in range(3):
            D.deform(w, sc.dims, sc.bbox, B, x, o, out=buf)
        torch.cuda.synchronize()
        ms = []
        for i in range(a.steps):
            flush.fill_(float(i))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            D.deform(w, sc.dims, sc.bbox, B, x, o, out=buf)
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        tg64 = torch.empty((w.shape[0], 12), dtype=torch.float64, device=dev)
        tg = D.precompute_transform_grid(w, sc.dims, sc.bbox, B, out64=tg64)
        out = D.batch_search(tg, sc.dims, sc.bbox, B, x, o, tgrid64=tg64, weights=w)
        dense[mode] = {k: v.cpu().numpy() for k, v in out.items() if v is not None}
        med = float(np.median(ms))
        line = {"mode": mode, "ms_per_frame_median": med, "solves_per_s": n * nb / (med * 1e-3),
                "workload": f"{a.points} points x {nb} inits, {a.grid} grid, max_iters {a.max_iters}",
                "converged_frac": float(dense[mode]["converged"].mean())}
        print(json.dumps(line), flush=True)
    ex = dense["exact64"]
    for mode in ("mixed", "mixed-fast", "fp32", "fp64"):
        d = dense[mode]
        both = (d["converged"] == 1) & (ex["converged"] == 1)
        print(json.dumps({"vs_exact64": mode, "mask_agreement": float((d["converged"] == ex["converged"]).mean()),
                          "mask_disagreements": int((d["converged"] != ex["converged"]).sum()),
                          "max_abs_dx_both_converged": float(np.abs(d["x_c"] - ex["x_c"])[both].max()),
                          "keep_disagreements": int((d["keep"] != ex["keep"]).sum())}), flush=True)
    D.close()


if __name__ == "__main__":
    main()
