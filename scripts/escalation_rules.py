"""Escalation-rule study (oracle-side tooling). Emulates the float32
pass (oracle/precision_emul.cpp) on many seeded scenes, compares every non-escalated solve
with the f64 oracle, and evaluates extra escalation criteria computed from the float32
solve alone: final max|J~| (conditioning of the root), and the smallest |cos(dx, J~dg)|
over the Broyden updates (near-degenerate rank-one updates amplify rounding).
Usage: python scripts/escalation_rules.py [--cap 8] [--seeds 10-16] [--n 30000]"""
import argparse
import itertools
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from precision_study import S, hybrid, oracle  # noqa: E402

GRIDS = [(32, 32, 32), (64, 64, 64), (128, 128, 32), (16, 16, 16), (64, 64, 16)]


def collect(cap, seeds, n):
    rows = []
    for seed in seeds:
        for dims in GRIDS:
            pts = ["uniform", "training"][seed % 2]
            sc = S.make_scene(dims, n, seed=seed, points=pts)
            o = sc.search_options(50)
            tg = oracle.precompute_transform_grid(sc.weights, sc.dims, sc.bbox, sc.bones, 8)
            ref = oracle.batch_search(sc.weights, sc.dims, sc.bbox, sc.bones, sc.points, workers=8, tgrid=tg, **o)
            xo, cv, it, esc, jn = hybrid(sc, tg, o, cap)
            nb = sc.n_bones
            dx = np.abs(xo - ref["x_c"]).max(-1).ravel()
            dj = np.abs(jn[..., 3:12] - ref["jinv"].reshape(n, nb, 9)).max(-1).ravel()
            rows.append(dict(dims=dims, pts=pts, seed=seed, esc=esc.ravel() != 0, cv=cv.ravel(),
                             rc=ref["converged"].ravel(), dx=dx, dj=dj, jmax=jn[..., 0].ravel(),
                             cos=jn[..., 2].ravel(), e=jn[..., 12].ravel(), s_next=jn[..., 13].ravel(),
                             e_prev=jn[..., 14].ravel(), s_last=jn[..., 15].ravel()))
            r = rows[-1]
            both = ~r["esc"] & (r["cv"] == 1) & (r["rc"] == 1)
            print(f"{dims} {pts:8s} seed {seed}: esc {r['esc'].mean()*100:.2f}%  flips "
                  f"{int((~r['esc'] & (r['cv'] != r['rc'])).sum())}  max dx {(r['dx']*both).max():.1e}  "
                  f"max dJ {(r['dj']*both).max():.1e}", flush=True)
    return rows


def evaluate(rows, jt, ct):
    mx = mj = 0.0
    extra = flips = tot = 0
    for r in rows:
        conv = r["cv"] == 1
        e2 = (conv & (r["jmax"] > jt)) | (r["cos"] < ct)
        ok = ~r["esc"] & ~e2
        both = ok & conv & (r["rc"] == 1)
        mx, mj = max(mx, (r["dx"] * both).max()), max(mj, (r["dj"] * both).max())
        flips += int((ok & (r["cv"] != r["rc"])).sum())
        extra += int((e2 & ~r["esc"]).sum())
        tot += r["esc"].size
    return mx, mj, flips, extra / tot


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--cap", type=int, default=8)
    ap.add_argument("--seeds", default="10-16")
    ap.add_argument("--n", type=int, default=30000)
    a = ap.parse_args()
    s0, s1 = map(int, a.seeds.split("-"))
    rows = collect(a.cap, range(s0, s1), a.n)
    print(f"cap {a.cap}: base escalation {np.mean([r['esc'].mean() for r in rows])*100:.2f}%")
    for jt, ct in itertools.product([1e9, 20, 10, 6, 4], [0, 0.1, 0.2, 0.3]):
        mx, mj, fl, ex = evaluate(rows, jt, ct)
        print(f"  max|J~|>{jt:g} or cos<{ct}: max dx {mx:.2e}  max dJ {mj:.2e}  flips {fl}  extra esc {ex*100:.3f}%")
