"""GPU-vs-oracle outlier diagnosis (tooling): for one scene, list the converged solves with
the largest |x_gpu - x_oracle| together with the emulated float32 solve's escalation
features (final max|J~|, min |cos(dx, J~dg)|). Usage: python scripts/diag_outliers.py D0 D1 D2 seed points"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from precision_study import S, hybrid, oracle  # noqa: E402
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_gpu_parity import run_gpu  # noqa: E402
from paper_2211_15601_b200.deformer import Deformer  # noqa: E402

dims = tuple(int(a) for a in sys.argv[1:4])
seed, pts = int(sys.argv[4]), sys.argv[5]
n = int(sys.argv[6]) if len(sys.argv) > 6 else 30000
sc = S.make_scene(dims, n, seed=seed, points=pts)
o = sc.search_options(50)
D = Deformer(0)
_, g = run_gpu(D, sc, 50)
tg = oracle.precompute_transform_grid(sc.weights, sc.dims, sc.bbox, sc.bones, 8)
r = oracle.batch_search(sc.weights, sc.dims, sc.bbox, sc.bones, sc.points, workers=8, tgrid=tg, **o)
xo, cv, it, esc, jn = hybrid(sc, tg, o, 8)
nb = sc.n_bones
both = (g["converged"] == 1) & (r["converged"] == 1)
dx = np.abs(g["x_c"] - r["x_c"]).max(-1) * both
gJ = np.abs(g["jinv"].reshape(n, nb, 9)).max(-1)
rJ = np.abs(r["jinv"].reshape(n, nb, 9)).max(-1)
for i in np.argsort(-dx.ravel())[:8]:
    p, b = divmod(i, nb)
    print(f"p {p} b {b}: dx {dx[p, b]:.2e}  iters gpu {g['iters'][p, b]} ref {r['iters'][p, b]} emu {it[p, b]}  "
          f"resid gpu {g['resid'][p, b]:.2e} ref {r['resid'][p, b]:.2e} (conv {o['conv_eps']:.2e})  "
          f"max|J~| gpu {gJ[p, b]:.2f} ref {rJ[p, b]:.2f}  emu: esc {esc[p, b]} jmax {jn[p, b, 0]:.2f} "
          f"amp {jn[p, b, 1]:.2f} cos {jn[p, b, 2]:.3f} dx_emu {np.abs(xo[p, b] - r['x_c'][p, b]).max():.1e}")
