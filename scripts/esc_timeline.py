"""Timeline of the escalation refill kernel (probe build -DFSK_ESC_TIMELINE -DFSK_ESC_REASONS for the
debug-counter reader): kernel start, first/last warp to find the queue dry, last warp exit."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_15601_b200 import synthetic as S  # noqa: E402
from paper_2211_15601_b200.deformer import Deformer, SearchOptions  # noqa: E402

D = Deformer(0)
f = D.L.fsk_ctx_esc_reasons
f.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint64), ctypes.c_int]
sc = S.make_scene((32, 32, 32), 200_000, seed=1)
o = sc.search_options(50)
w, B, x = (torch.from_numpy(a).cuda() for a in (sc.weights, sc.bones, sc.points))
so = SearchOptions(50, o["conv_eps"], o["div_eps"], o["dedup_dist"])
for rep in range(3):
    buf = (ctypes.c_uint64 * 40)()
    f(D._ctx, buf, 1)
    D.deform(w, sc.dims, sc.bbox, B, x, so)
    torch.cuda.synchronize()
    f(D._ctx, buf, 1)
    t0, dry0, dry1, tend = (buf[32 + i] for i in range(4))
    t0, dry0 = (~t0) & (2**64 - 1), (~dry0) & (2**64 - 1)
    print(f"rep {rep}: queue dry after {(dry0 - t0) / 1e3:.1f} us (last warp to notice +{(dry1 - t0) / 1e3:.1f}), "
          f"last warp exit +{(tend - t0) / 1e3:.1f} us")
