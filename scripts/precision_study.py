"""Escalation-rule study on the CPU (oracle-side tooling, never the product): the float32
pass is emulated with oracle/precision_emul.cpp (orc_emul_hybrid) and compared against
the f64 oracle's batch_search; a flip is a non-escalated solve whose converged flag
differs from the oracle's. Usage: python scripts/precision_study.py [cap ...]"""
import ctypes
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_2211_15601_b200 import synthetic as S  # noqa: E402

L = oracle.lib()
_d, _u8, _i32 = ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_uint8), ctypes.POINTER(ctypes.c_int32)
L.orc_emul_hybrid.argtypes = [_d, ctypes.c_int, ctypes.c_int, ctypes.c_int, _d, _d, ctypes.c_int, _d, ctypes.c_int64,
                              ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                              ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double, _d, _u8, _i32, _u8,
                              _d, ctypes.c_int]
P = lambda a, t=_d: a.ctypes.data_as(t)  # noqa: E731


def hybrid(sc, tg, o, cap, min_div=3, mixed=0, workers=8):
    n, nb = sc.points.shape[0], sc.n_bones
    x = np.ascontiguousarray(sc.points, np.float64)
    B = np.ascontiguousarray(sc.bones, np.float64)
    bb = np.ascontiguousarray(sc.bbox, np.float64)
    xo, cv = np.zeros((n, nb, 3)), np.zeros((n, nb), np.uint8)
    it, esc, jn = np.zeros((n, nb), np.int32), np.zeros((n, nb), np.uint8), np.zeros((n, nb, 16))
    L.orc_emul_hybrid(P(tg), *sc.dims, P(bb), P(B), nb, P(x), n, o["max_iters"], o["conv_eps"], o["div_eps"], workers,
                      cap, min_div, 0.02, 2e-4, 1e-5, 1e-12, P(xo), P(cv, _u8), P(it, _i32), P(esc, _u8), P(jn), mixed)
    return xo, cv, it, esc, jn


SCENES = [
    dict(dims=(32, 32, 32), n=8000, seed=1, points="uniform", mi=50),
    dict(dims=(32, 32, 32), n=8000, seed=2, points="training", mi=50),
    dict(dims=(64, 64, 64), n=8000, seed=3, points="uniform", mi=50),
    dict(dims=(128, 128, 32), n=8000, seed=4, points="uniform", mi=50),
    dict(dims=(16, 16, 16), n=8000, seed=5, points="uniform", mi=50),
    dict(dims=(32, 32, 32), n=8000, seed=6, points="uniform", mi=10),
]

if __name__ == "__main__":
    caps = [int(a) for a in sys.argv[1:]] or [8, 10, 12]
    tot = {c: [0, 0, 0] for c in caps}
    for cfg in SCENES:
        sc = S.make_scene(cfg["dims"], cfg["n"], seed=cfg["seed"], points=cfg["points"])
        o = sc.search_options(cfg["mi"])
        t = time.time()
        tg = oracle.precompute_transform_grid(sc.weights, sc.dims, sc.bbox, sc.bones, 8)
        ref = oracle.batch_search(sc.weights, sc.dims, sc.bbox, sc.bones, sc.points, workers=8, tgrid=tg, **o)
        for cap in caps:
            xo, cv, it, esc, _ = hybrid(sc, tg, o, cap)
            ok = esc == 0
            flips = int(((cv != ref["converged"]) & ok).sum())
            both = ok & (cv == 1) & (ref["converged"] == 1)
            dx = float(np.abs(xo - ref["x_c"])[both].max()) if both.any() else 0.0
            tot[cap][0] += flips
            tot[cap][1] += int(esc.sum())
            tot[cap][2] += esc.size
            print(f"{cfg['dims']} {cfg['points']:8s} mi={cfg['mi']} cap={cap:2d}: esc {esc.mean()*100:5.2f}%  "
                  f"flips {flips}  max|dx| {dx:.1e}  f64 iters of flips "
                  f"{sorted(ref['iters'][(cv != ref['converged']) & ok].tolist())[:8]}", flush=True)
        print(f"  ({time.time()-t:.1f}s)")
    for cap, (f, e, n) in tot.items():
        print(f"TOTAL cap={cap}: flips {f} / {n} solves, escalated {e/n*100:.2f}%")
