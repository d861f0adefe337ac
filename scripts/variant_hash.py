"""Print a hash of the dense forward-search outputs on the C2 scene (GPU), so tuning
variants (FSK_LIB=...) can be checked for bitwise identity with the production build."""
import hashlib
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_15601_b200 import synthetic as S  # noqa: E402
from paper_2211_15601_b200.deformer import Deformer, SearchOptions  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
D = Deformer(0)
sc = S.make_scene((32, 32, 32), n, seed=1)
o = sc.search_options(50)
w, B, x = (torch.from_numpy(a).cuda() for a in (sc.weights, sc.bones, sc.points))
tg = D.precompute_transform_grid(w, sc.dims, sc.bbox, B)
so = SearchOptions(50, o["conv_eps"], o["div_eps"], o["dedup_dist"])
# without the weight grid: fused float64 escalation; with it (the default of fsk_deform*): exact replay
for tag, wt in (("fused", None), ("exact", w)):
    out = D.batch_search(tg, sc.dims, sc.bbox, B, x, so, weights=wt)
    h = hashlib.sha256()
    for k in sorted(out):
        h.update(k.encode())
        h.update(out[k].cpu().numpy().tobytes())
    print("HASH", tag, os.environ.get("FSK_LIB", "default"), h.hexdigest()[:16])
