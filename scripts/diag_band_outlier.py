"""One band-study scene's converged roots that differ from the oracle by > 1e-4 (tooling): the float32
and float64 trajectories iteration by iteration. Usage: diag_band_outlier.py D0 D1 D2 seed points"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
from paper_2211_15601_b200 import synthetic as S  # noqa: E402
from paper_2211_15601_b200.deformer import Deformer, SearchOptions  # noqa: E402
from test_gpu_parity import run_gpu  # noqa: E402

dims = tuple(int(a) for a in sys.argv[1:4])
seed, pts = int(sys.argv[4]), sys.argv[5]
sc = S.make_scene(dims, 30000, seed=seed, points=pts)
o = sc.search_options(50)
D = Deformer(0)
_, g = run_gpu(D, sc, 50)
r = oracle.batch_search(sc.weights, sc.dims, sc.bbox, sc.bones, sc.points, workers=os.cpu_count() or 8, **o)
both = (g["converged"] == 1) & (r["converged"] == 1)
dx = np.abs(g["x_c"] - r["x_c"]).max(-1) * both
w, B = torch.from_numpy(sc.weights).cuda(), torch.from_numpy(sc.bones).cuda()
tg64 = torch.empty((w.shape[0], 12), dtype=torch.float64, device="cuda")
tg = D.precompute_transform_grid(w, sc.dims, sc.bbox, B, out64=tg64)
for p, b in zip(*np.nonzero(dx > 1e-4)):
    print(f"query {p} bone {b}: |dx| {dx[p, b]:.2e} gpu it {g['iters'][p, b]} resid {g['resid'][p, b]:.3e} | "
          f"oracle it {r['iters'][p, b]} resid {r['resid'][p, b]:.3e} (conv {o['conv_eps']:.3e}); "
          f"gpu max|J~| {np.abs(g['jinv'][p, b]).max():.2f}")
    x1 = torch.from_numpy(sc.points[p:p + 1].copy()).cuda()
    for k in range(0, 12):
        s1 = SearchOptions(max(k, 1), o["conv_eps"], o["div_eps"], o["dedup_dist"])
        s1.precision = "fp32"
        g1 = D.batch_search(tg, sc.dims, sc.bbox, B, x1, s1, tgrid64=tg64, weights=w)
        rk = oracle.batch_search(sc.weights, sc.dims, sc.bbox, sc.bones, sc.points[p:p + 1], workers=1,
                                 **dict(o, max_iters=max(k, 1)))
        J = g1["jinv"][0, b].cpu().numpy()
        print(f"  k={max(k, 1)}: f32 x {g1['x_c'][0, b].cpu().numpy()} err {float(g1['resid'][0, b]):.3e} "
              f"conv {int(g1['converged'][0, b])} |J~| {np.nanmax(np.abs(J)):.2f} | f64 x {rk['x_c'][0, b]} "
              f"err {rk['resid'][0, b]:.3e} conv {int(rk['converged'][0, b])} |J~| {np.abs(rk['jinv'][0, b]).max():.2f}")
