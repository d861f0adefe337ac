"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck / synccheck): C1-sized deform
(spatial sort with its grid-barrier scan, float32 pass, escalation queue + refill kernels, dedup,
compaction), the dense search, every backward mode, the host-buffer pipeline with chunk items and a
forced slot overflow, and the exact implicit gradient."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_15601_b200 import synthetic as S  # noqa: E402
from paper_2211_15601_b200.deformer import Deformer, SearchOptions  # noqa: E402

D = Deformer(0)
sc = S.make_scene((32, 32, 32), 10_000, seed=1, points="training")
w, B, x = (torch.from_numpy(a).cuda() for a in (sc.weights, sc.bones, sc.points))
for mi in (10, 50):
    o = SearchOptions(mi, **{k: v for k, v in sc.search_options(mi).items() if k != "max_iters"})
    offs, roots = D.deform(w, sc.dims, sc.bbox, B, x, o)
    tg64 = torch.empty((w.shape[0], 12), dtype=torch.float64, device="cuda")
    tg = D.precompute_transform_grid(w, sc.dims, sc.bbox, B, out64=tg64)
    dense = D.batch_search(tg, sc.dims, sc.bbox, B, x, o, tgrid64=tg64, weights=w)
n = sc.points.shape[0]
ridx = torch.where(offs[1:] > offs[:-1], offs[:-1], torch.full_like(offs[:-1], -1))
gx = torch.randn((n, 3), device="cuda") / n
order = D.query_order(n)
for det in (False, True):
    D.search_bwd_roots(sc.dims, sc.bbox, sc.n_bones, roots, ridx, gx, deterministic=det, order=order)
    D.search_bwd_exact_roots(w, sc.dims, sc.bbox, B, roots, ridx, gx, deterministic=det)
hw, hb, hx = (torch.from_numpy(a).pin_memory() for a in (sc.weights, sc.bones, sc.points))
os.environ["FSK_HOST_CHUNKS"] = "3"
os.environ["FSK_SLOT_ROOTS_PER_QUERY"] = "1"
ho = torch.empty(n + 1, dtype=torch.int64).pin_memory()
hr = torch.empty((n * 2, 16), dtype=torch.float32).pin_memory()
D.deform_host_frames(hw, sc.dims, sc.bbox, [hb, hb], [hx, hx[:5000]], o, [ho, ho], [hr, hr])
torch.cuda.synchronize()
print("sanitize workload done", int(offs[-1].item()))
