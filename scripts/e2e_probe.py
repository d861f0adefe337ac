"""e2e probe: fsk_deform_host_frames (20 frames, C2) and fsk_deform_host, ms per frame, repeated."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_15601_b200 import synthetic as S  # noqa: E402
from paper_2211_15601_b200.deformer import Deformer, SearchOptions  # noqa: E402

D = Deformer(0)
sc = S.make_scene((32, 32, 32), 200_000, seed=1)
o = SearchOptions(50, **{k: v for k, v in sc.search_options(50).items() if k != "max_iters"})
n, nb = sc.points.shape[0], sc.n_bones
hw, hb, hx = (torch.from_numpy(a).pin_memory() for a in (sc.weights, sc.bones, sc.points))
F = 20
hoffs = [torch.empty(n + 1, dtype=torch.int64).pin_memory() for _ in range(2)]
hroots = [torch.empty((n * nb, 16), dtype=torch.float32).pin_memory() for _ in range(2)]
for rep in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    D.deform_host_frames(hw, sc.dims, sc.bbox, [hb] * F, [hx] * F, o, [hoffs[f % 2] for f in range(F)],
                         [hroots[f % 2] for f in range(F)])
    t1 = time.perf_counter()
    for _ in range(5):
        D.deform_host(hw, sc.dims, sc.bbox, hb, hx, o, hoffs[0], hroots[0])
    t2 = time.perf_counter()
    print(f"frames {1e3 * (t1 - t0) / F:.3f} ms/frame   single {1e3 * (t2 - t1) / 5:.3f} ms", flush=True)
