"""Find the kept roots of the C5 workload (8 M points, 128x128x32) that differ from the reference's own
code by more than 1e-4, and print what the float32 pass saw for them (tooling)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_2211_15601_b200 import synthetic as S  # noqa: E402
from paper_2211_15601_b200.deformer import Deformer, SearchOptions  # noqa: E402

D = Deformer(0)
sc = S.make_scene((128, 128, 32), 8_000_000, seed=1, points=os.environ.get("DIAG_POINTS", "uniform"))
o = sc.search_options(50)
so = SearchOptions(50, o["conv_eps"], o["div_eps"], o["dedup_dist"])
w = torch.from_numpy(sc.weights).cuda()
B = torch.from_numpy(sc.bones).cuda()
bad = []
for c in range(0, 8_000_000, 2_000_000):
    pts = sc.points[c:c + 2_000_000]
    offs, roots = D.deform(w, sc.dims, sc.bbox, B, torch.from_numpy(pts).cuda(), so)
    go = offs.cpu().numpy()
    gr = roots[: int(go[-1])].cpu().numpy()
    rr = oracle.ref_batch_search(sc.weights, sc.dims, sc.bbox, sc.bones, pts, workers=os.cpu_count() or 8, **o)
    ro = rr["offsets"]
    cg, cr = np.diff(go), np.diff(ro)
    for p in np.nonzero((cg == cr) & (cg > 0))[0]:
        a, b = go[p], ro[p]
        k = cg[p]
        if not np.array_equal(gr[a:a + k, 13].view(np.int32), rr["bone"][b:b + k]):
            continue
        d = np.abs(gr[a:a + k, :3] - rr["x"][b:b + k]).max(1)
        for t in np.nonzero(d > 1e-4)[0]:
            bad.append((c + p, int(rr["bone"][b + t]), float(d[t]), int(gr[a + t, 14].view(np.int32)),
                        int(rr["iters"][b + t]), float(gr[a + t, 3]), float(rr["resid"][b + t])))
print("roots beyond 1e-4:", len(bad))
for q, bone, d, gi, ri, gres, rres in bad:
    print(f"query {q} bone {bone}: |dx| {d:.2e}  iters gpu {gi} ref {ri}  resid gpu {gres:.3e} ref {rres:.3e} "
          f"(conv {o['conv_eps']:.3e})")
    x1 = torch.from_numpy(sc.points[q:q + 1].copy()).cuda()
    tg64 = torch.empty((w.shape[0], 12), dtype=torch.float64, device="cuda")
    tg = D.precompute_transform_grid(w, sc.dims, sc.bbox, B, out64=tg64)
    for prec in ("mixed", "fp32"):
        s1 = SearchOptions(50, o["conv_eps"], o["div_eps"], o["dedup_dist"])
        s1.precision = prec
        D.search_stats(reset=True)
        out = D.batch_search(tg, sc.dims, sc.bbox, B, x1, s1, tgrid64=tg64, weights=w)
        st = D.search_stats(reset=True)
        J = out["jinv"][0, bone].cpu().numpy().reshape(3, 3)
        print(f"   {prec}: conv {int(out['converged'][0, bone])} iters {int(out['iters'][0, bone])} "
              f"resid {float(out['resid'][0, bone]):.3e} x {out['x_c'][0, bone].cpu().numpy()} max|J~| "
              f"{np.abs(J).max():.2f}  escalated solves in the query: {st[3]}")
    r1 = oracle.batch_search(sc.weights, sc.dims, sc.bbox, sc.bones, sc.points[q:q + 1], workers=1, **o)
    print(f"   oracle: conv {int(r1['converged'][0, bone])} iters {int(r1['iters'][0, bone])} x {r1['x_c'][0, bone]} "
          f"resid {r1['resid'][0, bone]:.3e} max|J~| {np.abs(r1['jinv'][0, bone]).max():.2f}")
    # the float32 trajectory, iteration by iteration (max_iters = k), against the oracle's
    for k in range(1, 12):
        s1 = SearchOptions(k, o["conv_eps"], o["div_eps"], o["dedup_dist"])
        s1.precision = "fp32"
        g1 = D.batch_search(tg, sc.dims, sc.bbox, B, x1, s1, tgrid64=tg64, weights=w)
        ok = dict(o, max_iters=k)
        rk = oracle.batch_search(sc.weights, sc.dims, sc.bbox, sc.bones, sc.points[q:q + 1], workers=1, **ok)
        print(f"     k={k}: f32 x {g1['x_c'][0, bone].cpu().numpy()} resid {float(g1['resid'][0, bone]):.3e} conv "
              f"{int(g1['converged'][0, bone])} | f64 x {rk['x_c'][0, bone]} resid {rk['resid'][0, bone]:.3e} conv "
              f"{int(rk['converged'][0, bone])}")
