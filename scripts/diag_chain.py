import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import oracle
from paper_2211_15601_b200 import synthetic as S
from paper_2211_15601_b200.deformer import Deformer, SearchOptions
D = Deformer(0)
for nb, seed in ((80, 3), (80, 4), (80, 5), (40, 3), (48, 3)):
    sc = S.make_scene((32, 32, 32), 4000, seed=seed, skeleton=S.chain_skeleton(nb))
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    w, B, x = dev(sc.weights), dev(sc.bones), dev(sc.points)
    tg64 = torch.empty((w.shape[0], 12), dtype=torch.float64, device="cuda")
    tg = D.precompute_transform_grid(w, sc.dims, sc.bbox, B, out64=tg64)
    o = sc.search_options(50)
    so = SearchOptions(50, o["conv_eps"], o["div_eps"], o["dedup_dist"])
    out = D.batch_search(tg, sc.dims, sc.bbox, B, x, so, tgrid64=tg64, weights=w)
    g = {k: (v.cpu().numpy() if v is not None else None) for k, v in out.items()}
    r = oracle.batch_search(sc.weights, sc.dims, sc.bbox, sc.bones, sc.points, workers=8, **o)
    both = (g["converged"] == 1) & (r["converged"] == 1)
    dx = np.abs(g["x_c"] - r["x_c"]).max(-1) * both
    flips = int((g["converged"] != r["converged"]).sum())
    print(f"nb {nb} seed {seed}: flips {flips} max dx {dx.max():.2e}  n>1e-4 {(dx>1e-4).sum()}  conv {o['conv_eps']:.2e}")
    for idx in np.argsort(dx.ravel())[::-1][:4]:
        q, b = divmod(idx, nb)
        jm = np.abs(g["jinv"][q, b]).max()
        print(f"   q {q} b {b}: dx {dx[q,b]:.2e} it gpu {g['iters'][q,b]} ora {r['iters'][q,b]} res gpu {g['resid'][q,b]:.2e} ora {r['resid'][q,b]:.2e} max|J~| {jm:.2f}")
