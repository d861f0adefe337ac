"""Convergence-band study on the GPU (tooling): across seeded scenes on every grid shape,
compare the GPU's converged solves with the f64 oracle and report, for solves whose
iteration counts differ (one side stopped one Broyden step earlier), the GPU's final
residual relative to conv_eps, plus how many converged solves sit in a band below conv."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.join(os.path.dirname(HERE), "tests"))
from precision_study import S, oracle  # noqa: E402
from test_gpu_parity import run_gpu  # noqa: E402
from paper_2211_15601_b200.deformer import Deformer  # noqa: E402

GRIDS = [(32, 32, 32), (64, 64, 64), (128, 128, 32), (16, 16, 16), (64, 64, 16)]
seeds = range(int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else range(10, 16)
n = 30000
D = Deformer(0)
ratios, mism = [], []
for seed in seeds:
    for dims in GRIDS:
        kinds = os.environ.get("BAND_POINTS", "uniform,training").split(",")
        pts = kinds[seed % len(kinds)]
        sc = S.make_scene(dims, n, seed=seed, points=pts)
        MI = int(os.environ.get("BAND_MAX_ITERS", "50"))
        o = sc.search_options(MI)
        _, g = run_gpu(D, sc, MI, precision=os.environ.get("BAND_PRECISION", "mixed"))
        r = oracle.batch_search(sc.weights, sc.dims, sc.bbox, sc.bones, sc.points, workers=os.cpu_count(), **o)
        both = (g["converged"] == 1) & (r["converged"] == 1)
        rg = g["resid"] / o["conv_eps"]
        dx = np.abs(g["x_c"] - r["x_c"]).max(-1)
        ratios.append(rg[both])
        mm = both & (g["iters"] != r["iters"])
        for p, b in zip(*np.nonzero(mm)):
            mism.append((rg[p, b], r["resid"][p, b] / o["conv_eps"], int(g["iters"][p, b]), int(r["iters"][p, b]),
                         dx[p, b]))
        flips = int((g["converged"] != r["converged"]).sum())
        print(f"{dims} {pts} seed {seed}: flips {flips} max dx {(dx * both).max():.2e} mismatched iters {int(mm.sum())}",
              flush=True)
ratios = np.concatenate(ratios)
print("mismatched-iteration converged solves (gpu resid/conv, ref resid/conv, gpu it, ref it, dx):")
for m in sorted(mism, key=lambda t: -t[4])[:40]:
    print("   %.4f %.4f %d %d %.2e" % m)
for b in (0.02, 0.05, 0.1, 0.2, 0.3):
    print(f"band {b:.2f}: {((ratios >= 1 - b) & (ratios < 1)).mean()*100:.3f}% of converged solves")
