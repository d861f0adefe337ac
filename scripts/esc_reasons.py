"""Escalation-rule breakdown on the GPU (study tooling; needs a build with -DFSK_ESC_REASONS, e.g.
`python scripts/build_variants.py reasons=-DFSK_ESC_REASONS`, run with FSK_LIB=build/variants/reasons.so).
For each rule of the float32 pass: how many solves it flags, and how many it
flags alone (the solves that relaxing only that rule would keep in float32)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_15601_b200 import synthetic as S  # noqa: E402
from paper_2211_15601_b200.deformer import Deformer, SearchOptions  # noqa: E402

RULES = ["det0", "conv band@start", "cos (degenerate update)", "conv band@iter", "den", "capped", "unconverged>=3",
         "max|J~| (conditioning)", "step rule: next step", "step rule: last step", "div band@start", "div band@iter",
         "converged at the cap"]
D = Deformer(0)
f = D.L.fsk_ctx_esc_reasons
f.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint64), ctypes.c_int]
for dims, pts, seed in [((32, 32, 32), "uniform", 1), ((64, 64, 64), "training", 11), ((128, 128, 32), "uniform", 2)]:
    sc = S.make_scene(dims, 200_000, seed=seed, points=pts)
    o = sc.search_options(50)
    w, B, x = (torch.from_numpy(a).cuda() for a in (sc.weights, sc.bones, sc.points))
    buf = (ctypes.c_uint64 * 40)()  # fired: slots 8+bit (buf[bit]), alone: 24+bit (buf[16+bit])
    f(D._ctx, buf, 1)
    D.search_stats(reset=True)
    D.deform(w, sc.dims, sc.bbox, B, x, SearchOptions(50, o["conv_eps"], o["div_eps"], o["dedup_dist"]))
    torch.cuda.synchronize()
    st = D.search_stats(reset=True)
    f(D._ctx, buf, 1)
    tot = sc.points.shape[0] * sc.n_bones
    print(f"{dims} {pts} seed {seed}: escalated {st[3]} of {tot} ({100 * st[3] / tot:.2f} %)")
    for i, name in enumerate(RULES):
        print(f"   {name:26s} fired {buf[i]:8d} ({100 * buf[i] / tot:.3f} %)   alone {buf[16 + i]:8d} ({100 * buf[16 + i] / tot:.3f} %)")
