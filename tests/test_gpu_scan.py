"""The single-pass root-count scan (k_scan_lookback, decoupled look-back with a per-launch epoch):
CorrespondenceSet offsets equal the exclusive prefix sum of the per-query kept counts of the
dense search, across many tiles, repeated launches (the epoch retires the previous launch's
status words) and CUDA-graph replays (no host-side state per launch)."""
import numpy as np
import pytest
import torch

from paper_2211_15601_b200 import synthetic as S
from paper_2211_15601_b200.deformer import SearchOptions

pytestmark = pytest.mark.gpu


def _inputs(n, seed):
    sc = S.make_scene((16, 16, 16), n, seed=seed)
    o = SearchOptions(10, **{k: v for k, v in sc.search_options(10).items() if k != "max_iters"})
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    return sc, o, dev(sc.weights), dev(sc.bones), dev(sc.points)


def _expected(deformer, sc, o, w, B, x):
    tg64 = torch.empty((w.shape[0], 12), dtype=torch.float64, device="cuda")
    tg = deformer.precompute_transform_grid(w, sc.dims, sc.bbox, B, out64=tg64)
    out = deformer.batch_search(tg, sc.dims, sc.bbox, B, x, o, tgrid64=tg64, weights=w)
    k = out["keep"].to(torch.int64).sum(1)
    return torch.cat([torch.zeros(1, dtype=torch.int64, device="cuda"), torch.cumsum(k, 0)])


@pytest.mark.parametrize("n", [1, 4095, 4097, 300_000, 2_000_000])
def test_offsets_are_the_prefix_sum_of_kept_counts(deformer, n):
    sc, o, w, B, x = _inputs(n, seed=61)
    ref = _expected(deformer, sc, o, w, B, x)
    for _ in range(3):  # repeated launches: each advances the epoch
        offs, roots = deformer.deform(w, sc.dims, sc.bbox, B, x, o)
        torch.cuda.synchronize()
        assert torch.equal(offs, ref)


def test_offsets_under_graph_replay(deformer):
    sc, o, w, B, x = _inputs(200_000, seed=62)
    ref = _expected(deformer, sc, o, w, B, x)
    offs, roots = deformer.deform(w, sc.dims, sc.bbox, B, x, o)  # warm-up sizes the scratch
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            deformer.deform(w, sc.dims, sc.bbox, B, x, o, out=(offs, roots))
    for _ in range(4):
        offs.fill_(-1)
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(offs, ref)
