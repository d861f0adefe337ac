"""Diagnose the largest non-escalated root deviation of one band-study scene (tooling)."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.join(os.path.dirname(HERE), "tests"))
from precision_study import S, oracle  # noqa: E402
from test_gpu_parity import run_gpu  # noqa: E402
from paper_2211_15601_b200.deformer import Deformer  # noqa: E402

dims = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "32,32,32").split(","))
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 75
D = Deformer(0)
sc = S.make_scene(dims, 30000, seed=seed, points=["uniform", "training"][seed % 2])
o = sc.search_options(50)
_, g = run_gpu(D, sc, 50)
_, f = run_gpu(D, sc, 50, precision="fp32")
_, e = run_gpu(D, sc, 50, precision="exact64")
r = oracle.batch_search(sc.weights, sc.dims, sc.bbox, sc.bones, sc.points, workers=os.cpu_count(), **o)
both = (g["converged"] == 1) & (r["converged"] == 1)
dx = np.abs(g["x_c"] - r["x_c"]).max(-1) * both
print("conv_eps", o["conv_eps"], "max dx", dx.max())
for idx in np.argsort(dx.ravel())[::-1][:3]:
    q, b = divmod(int(idx), sc.n_bones)
    print(f"q {q} bone {b}: dx {dx[q, b]:.2e}")
    for name, z in (("mixed", g), ("fp32-only", f), ("exact64", e), ("oracle", r)):
        print(f"   {name:9s} conv {int(z['converged'][q, b])} iters {int(z['iters'][q, b]):2d} resid/conv "
              f"{float(z['resid'][q, b]) / o['conv_eps']:.3f} x {np.asarray(z['x_c'][q, b])} "
              f"max|J~| {float(np.abs(np.asarray(z['jinv'][q, b])).max()):.2f}")
