"""Standalone MLP-stage timing (tooling): the occupancy query over a C2 step's roots, and distill."""
import sys, os, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
from paper_2211_15601_b200 import synthetic as S
from paper_2211_15601_b200.deformer import Deformer, SearchOptions
D = Deformer(0)
sc = S.make_scene((32, 32, 32), 200_000, seed=1)
o = sc.search_options(50)
w, B, x = (torch.from_numpy(a).cuda() for a in (sc.weights, sc.bones, sc.points))
offs, roots = D.deform(w, sc.dims, sc.bbox, B, x, SearchOptions(50, o["conv_eps"], o["div_eps"], o["dedup_dist"]))
th = torch.from_numpy(oracle.mlp_init([3, 128, 128, 128, 1], 2).astype(np.float32)).cuda()
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
for _ in range(3):
    D.posed_occupancy(th, [3, 128, 128, 128, 1], None, offs, roots)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(reps):
    D.posed_occupancy(th, [3, 128, 128, 128, 1], None, offs, roots)
b.record()
torch.cuda.synchronize()
print("occupancy ms", a.elapsed_time(b) / reps, "roots", int(offs[-1].item()))
