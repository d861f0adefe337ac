"""Hash of the deterministic implicit-diff backward (dL/dT, dL/dw) on the C3 scene (GPU tooling): tuning
variants (FSK_LIB=...) of the backward must reproduce it bit for bit."""
import hashlib
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_15601_b200 import synthetic as S  # noqa: E402
from paper_2211_15601_b200.deformer import Deformer, SearchOptions  # noqa: E402

D = Deformer(0)
for dims, n, seed in (((32, 32, 32), 200_000, 1), ((64, 64, 16), 50_000, 7)):
    sc = S.make_scene(dims, n, seed=seed)
    o = sc.search_options(50)
    w, B, x = (torch.from_numpy(a).cuda() for a in (sc.weights, sc.bones, sc.points))
    offs, roots = D.deform(w, sc.dims, sc.bbox, B, x, SearchOptions(50, o["conv_eps"], o["div_eps"], o["dedup_dist"]))
    gx = torch.randn((n, 3), generator=torch.Generator(device="cuda").manual_seed(1), device="cuda") / n
    ridx = torch.where(offs[1:] > offs[:-1], offs[:-1], torch.full_like(offs[:-1], -1))
    order = D.query_order(n)  # used by the spatial-order deterministic kernel (FSK_DET_ORDERED builds)
    gT = D.search_bwd_roots(sc.dims, sc.bbox, sc.n_bones, roots, ridx, gx, deterministic=True, order=order)
    gW = D.grad_weights(sc.dims, sc.bbox, gT, B)
    torch.cuda.synchronize()
    h = hashlib.sha256(gT.cpu().numpy().tobytes() + gW.cpu().numpy().tobytes()).hexdigest()[:16]
    print("BWDHASH", dims, os.environ.get("FSK_LIB", "default"), h, float(gT.abs().max()))
