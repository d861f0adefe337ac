"""How much does "the reference's answer" depend on its unpinned operation order?

The reference is Eigen3 (version unpinned) built with -march=native (proj/CMakeLists.txt:10-16); it
cannot be built here. oracle/Makefile builds the same f64 restatement in four plausible operation
orders (default "fma", "unfused", "invrow0", "pairsum", "gccfma"). This script runs each on the BASELINE
configurations' scenes and reports, against the default: converged-mask flips, keep-mask flips,
iteration-count changes and root moves (max |dx|, count beyond 1e-4) — the spread any
implementation of the reference must be judged against. Usage:
    python scripts/oracle_variants.py [--points N] [--scenes c1,c2,c4grid,c5grid]
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2211_15601_b200 import synthetic as S  # noqa: E402

SCENES = {
    "c1": ((32, 32, 32), 10_000, 1, "uniform", 10),
    "c2": ((32, 32, 32), 200_000, 1, "uniform", 50),
    "c2train": ((32, 32, 32), 200_000, 4, "training", 50),
    "c4grid": ((64, 64, 64), 200_000, 61, "training", 50),
    "c5grid": ((128, 128, 32), 200_000, 61, "uniform", 50),
}


def compare(a, b):
    both = (a["converged"] == 1) & (b["converged"] == 1)
    dx = np.abs(a["x_c"] - b["x_c"]).max(-1)[both]
    return dict(mask=int((a["converged"] != b["converged"]).sum()), keep=int((a["keep"] != b["keep"]).sum()),
                iters=int((a["iters"][both] != b["iters"][both]).sum()), dx_max=float(dx.max() if dx.size else 0.0),
                dx_gt_1e4=int((dx > 1e-4).sum()), bitwise=float((dx == 0).mean() if dx.size else 1.0))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scenes", default="c1,c2,c2train,c4grid,c5grid")
    ap.add_argument("--workers", type=int, default=os.cpu_count())
    args = ap.parse_args()
    for name in args.scenes.split(","):
        dims, n, seed, pts, mi = SCENES[name]
        sc = S.make_scene(dims, n, seed=seed, points=pts)
        res = {}
        for v in oracle.VARIANTS:
            t = time.time()
            res[v] = oracle.batch_search(sc.weights, sc.dims, sc.bbox, sc.bones, sc.points, workers=args.workers,
                                         variant=v, **sc.search_options(mi))
            print(f"# {name} {v}: {time.time() - t:.1f} s", flush=True)
        d0 = oracle.VARIANTS[0]
        total = res[d0]["converged"].size
        print(f"{name}: {dims} x {n} points x {sc.n_bones} inits = {total} solves, max_iters {mi}")
        for v in oracle.VARIANTS[1:]:
            c = compare(res[v], res[d0])
            print(f"  {v:8s} vs {d0}: mask flips {c['mask']} ({c['mask'] / total:.2e}), keep flips {c['keep']}, "
                  f"iteration changes {c['iters']}, max|dx| {c['dx_max']:.2e}, roots beyond 1e-4 {c['dx_gt_1e4']}, "
                  f"bit-equal roots {c['bitwise']:.4f}", flush=True)
        worst = {k: max(compare(res[a], res[b])[k] for a in oracle.VARIANTS for b in oracle.VARIANTS if a < b)
                 for k in ("mask", "keep", "dx_max", "dx_gt_1e4")}
        print(f"  pairwise worst: {worst}", flush=True)


if __name__ == "__main__":
    main()
