"""fsk_deform_host_frames (one subject, a sequence of poses, double-buffered host copies):
every frame's CorrespondenceSets equal a separate fsk_deform_host call bit for bit, whatever
the frame sizes (including empty frames), and a too-small root buffer fails loudly."""
import numpy as np
import pytest
import torch

from paper_2211_15601_b200 import synthetic as S
from paper_2211_15601_b200.deformer import FskInvalidArgument, SearchOptions

pytestmark = pytest.mark.gpu


def _opts(sc):
    return SearchOptions(50, **{k: v for k, v in sc.search_options(50).items() if k != "max_iters"})


def _frames(sizes, dims=(32, 32, 32)):
    """One subject (weight grid of seed 0) in len(sizes) poses with their own point sets."""
    base = S.make_scene(dims, 10, seed=0)
    out = []
    for i, n in enumerate(sizes):
        sc = S.make_scene(dims, max(n, 1), seed=100 + i)
        out.append((torch.from_numpy(sc.bones).pin_memory(), torch.from_numpy(sc.points[:n].copy()).pin_memory()))
    return base, out


@pytest.mark.parametrize("sizes", [[5000], [4000, 7000, 0, 3000, 6000], [20000, 20000, 20000, 20000]])
def test_frames_equal_single_frame_calls(deformer, sizes):
    base, frames = _frames(sizes)
    hw = torch.from_numpy(base.weights).pin_memory()
    nb = base.n_bones
    o = _opts(base)
    offs = [torch.empty(p.shape[0] + 1, dtype=torch.int64).pin_memory() for _, p in frames]
    roots = [torch.zeros((max(p.shape[0] * nb, 1), 16), dtype=torch.float32).pin_memory() for _, p in frames]
    totals = deformer.deform_host_frames(hw, base.dims, base.bbox, [b for b, _ in frames], [p for _, p in frames], o,
                                         offs, roots)
    for f, (b, p) in enumerate(frames):
        o1 = torch.empty(p.shape[0] + 1, dtype=torch.int64).pin_memory()
        r1 = torch.zeros((max(p.shape[0] * nb, 1), 16), dtype=torch.float32).pin_memory()
        t1 = deformer.deform_host(hw, base.dims, base.bbox, b, p, o, o1, r1)
        assert totals[f] == t1
        np.testing.assert_array_equal(offs[f].numpy(), o1.numpy())
        np.testing.assert_array_equal(roots[f][:t1].numpy().view(np.uint32), r1[:t1].numpy().view(np.uint32))


def test_frames_root_buffer_too_small(deformer):
    base, frames = _frames([3000, 3000])
    hw = torch.from_numpy(base.weights).pin_memory()
    offs = [torch.empty(p.shape[0] + 1, dtype=torch.int64).pin_memory() for _, p in frames]
    roots = [torch.zeros((p.shape[0] * base.n_bones, 16)).pin_memory() for _, p in frames]
    roots[1] = torch.zeros((10, 16)).pin_memory()
    with pytest.raises(FskInvalidArgument, match="root buffer too small"):
        deformer.deform_host_frames(hw, base.dims, base.bbox, [b for b, _ in frames], [p for _, p in frames],
                                    _opts(base), offs, roots)
    # the context stays usable
    totals = deformer.deform_host_frames(hw, base.dims, base.bbox, [frames[0][0]], [frames[0][1]], _opts(base),
                                         offs[:1], roots[:1])
    assert totals[0] > 0


@pytest.mark.parametrize("chunks,per_q", [(3, 4), (3, 0), (1, 1)])
def test_chunked_items_and_slot_overflow_redo(deformer, monkeypatch, chunks, per_q):
    """The host pipeline splits frames into chunk items over two bounded device slots; an item whose
    kept roots overflow its slot (FSK_SLOT_ROOTS_PER_QUERY, here forced down to 0-1 roots per query)
    is re-run into an exact-size buffer. Results equal the whole-frame call bit for bit."""
    base, frames = _frames([20000, 0, 9000, 20000])
    hw = torch.from_numpy(base.weights).pin_memory()
    nb, o = base.n_bones, _opts(base)

    def run():
        offs = [torch.empty(p.shape[0] + 1, dtype=torch.int64).pin_memory() for _, p in frames]
        roots = [torch.zeros((max(p.shape[0] * 2, 1), 16), dtype=torch.float32).pin_memory() for _, p in frames]
        t = deformer.deform_host_frames(hw, base.dims, base.bbox, [b for b, _ in frames], [p for _, p in frames], o,
                                        offs, roots)
        return t, offs, roots

    ref_t, ref_o, ref_r = run()
    monkeypatch.setenv("FSK_HOST_CHUNKS", str(chunks))
    monkeypatch.setenv("FSK_SLOT_ROOTS_PER_QUERY", str(per_q))
    t, offs, roots = run()
    assert t == ref_t
    for f in range(len(frames)):
        np.testing.assert_array_equal(offs[f].numpy(), ref_o[f].numpy())
        np.testing.assert_array_equal(roots[f][:t[f]].numpy().view(np.uint32), ref_r[f][:t[f]].numpy().view(np.uint32))


def test_host_call_reports_total_when_buffer_too_small(deformer):
    """Count-then-allocate from the caller's side: a too-small root buffer fails with FSK_EINVAL
    after the whole frame ran, and the reported total is exactly the capacity the retry needs."""
    import ctypes

    from paper_2211_15601_b200.deformer import _ptr, _stream, grid_desc
    base, frames = _frames([12000])
    b, p = frames[0]
    hw = torch.from_numpy(base.weights).pin_memory()
    o = _opts(base)
    n = p.shape[0]
    offs = torch.empty(n + 1, dtype=torch.int64).pin_memory()
    small = torch.zeros((100, 16), dtype=torch.float32).pin_memory()
    total = ctypes.c_int64()
    desc = grid_desc(base.dims, base.bbox, base.n_bones)
    rc = deformer.L.fsk_deform_host(deformer._ctx, _ptr(hw), ctypes.byref(desc), _ptr(b), base.n_bones, _ptr(p), n,
                                    ctypes.byref(o.c()), _ptr(offs), _ptr(small), 100, ctypes.byref(total),
                                    _stream(deformer.device))
    assert rc == 1 and total.value > 100
    exact = torch.zeros((total.value, 16), dtype=torch.float32).pin_memory()
    assert deformer.deform_host(hw, base.dims, base.bbox, b, p, o, offs, exact) == total.value


@pytest.mark.parametrize("chunks", [1, 3])
def test_graph_replayed_items_equal_eager(deformer, monkeypatch, chunks):
    """The host pipeline stages each item's sort + K1 on a second stream ahead of its search and replays
    an item's device work from CUDA graphs once it has seen the same launch set (slot buffers, chunk
    size, options, scratch generation) before. Ten frames of distinct poses — staged eagerly, then
    twice from graphs (the second call replays the first call's) — equal the unstaged eager pipeline
    (FSK_PIPE_STAGE=0, FSK_PIPE_GRAPH=0) bit for bit; so does a call after a scratch regrow."""
    base, frames = _frames([6000 + 100 * (i % 2) for i in range(10)])
    hw = torch.from_numpy(base.weights).pin_memory()
    o = _opts(base)
    monkeypatch.setenv("FSK_HOST_CHUNKS", str(chunks))

    def run():
        offs = [torch.empty(p.shape[0] + 1, dtype=torch.int64).pin_memory() for _, p in frames]
        roots = [torch.zeros((p.shape[0] * 3, 16), dtype=torch.float32).pin_memory() for _, p in frames]
        t = deformer.deform_host_frames(hw, base.dims, base.bbox, [b for b, _ in frames], [p for _, p in frames], o,
                                        offs, roots)
        return t, [x.numpy().copy() for x in offs], [r[:n].numpy().view(np.uint32).copy() for r, n in zip(roots, t)]

    monkeypatch.setenv("FSK_PIPE_GRAPH", "0")
    monkeypatch.setenv("FSK_PIPE_STAGE", "0")  # reference: every item whole on one stream, eagerly
    ref = run()
    monkeypatch.setenv("FSK_PIPE_STAGE", "1")  # items staged (sort + K1) on a second stream ahead of their search
    got = [run()]
    monkeypatch.setenv("FSK_PIPE_GRAPH", "1")
    got += [run(), run()]
    # a bigger search in between regrows the scratch (new generation: the cached graphs are not reused)
    big = S.make_scene(base.dims, 60000, seed=7)
    x = torch.from_numpy(big.points).cuda()
    w, B = torch.from_numpy(base.weights).cuda(), torch.from_numpy(big.bones).cuda()
    deformer.deform(w, base.dims, base.bbox, B, x, o)
    torch.cuda.synchronize()
    got.append(run())
    for t, offs, roots in got:
        assert t == ref[0]
        for f in range(len(frames)):
            np.testing.assert_array_equal(offs[f], ref[1][f])
            np.testing.assert_array_equal(roots[f], ref[2][f])


def test_graph_cache_eviction_keeps_results(deformer, monkeypatch):
    """More distinct chunk shapes than the context caches graphs for (8): every shape is seen twice per
    call sequence, so graphs are captured, evicted (least recently used) and re-captured; results stay
    equal to the eager pipeline."""
    sizes = [3000 + 500 * i for i in range(10)]
    base, frames = _frames(sizes)
    hw = torch.from_numpy(base.weights).pin_memory()
    o = _opts(base)

    def run(f):
        b, p = frames[f]
        offs = torch.empty(p.shape[0] + 1, dtype=torch.int64).pin_memory()
        roots = torch.zeros((p.shape[0] * 3, 16), dtype=torch.float32).pin_memory()
        t = deformer.deform_host(hw, base.dims, base.bbox, b, p, o, offs, roots)
        return offs.numpy().copy(), roots[:t].numpy().view(np.uint32).copy()

    monkeypatch.setenv("FSK_PIPE_GRAPH", "0")
    ref = [run(f) for f in range(len(frames))]
    monkeypatch.setenv("FSK_PIPE_GRAPH", "1")
    for _ in range(3):
        for f in list(range(len(frames))) + list(range(len(frames)))[::-1]:
            offs, roots = run(f)
            np.testing.assert_array_equal(offs, ref[f][0])
            np.testing.assert_array_equal(roots, ref[f][1])


@pytest.mark.parametrize("sort", [True, False])
def test_device_frames_equal_per_frame_deform(deformer, sort):
    """fsk_deform_frames (device buffers, frame f+1's sort + K1 staged beside frame f's search) equals one
    fsk_deform per frame bit for bit, with ragged and empty frames, eagerly and replayed from a CUDA graph
    (and without the spatial sort: the staged slot then holds the identity order)."""
    base, frames = _frames([5000, 0, 7000, 3000, 6000])
    w = torch.from_numpy(base.weights).cuda()
    o = _opts(base)
    o.sort = sort
    B = [b.cuda() for b, _ in frames]
    X = [p.cuda() for _, p in frames]
    ref = []
    for b, x in zip(B, X):
        offs, roots = deformer.deform(w, base.dims, base.bbox, b, x, o)
        torch.cuda.synchronize()
        ref.append((offs.cpu().numpy(), roots[: int(offs[-1])].cpu().numpy().view(np.uint32)))

    def check(outs):
        torch.cuda.synchronize()
        for (offs, roots), (ro, rr) in zip(outs, ref):
            o_h = offs.cpu().numpy()
            np.testing.assert_array_equal(o_h, ro)
            np.testing.assert_array_equal(roots[: int(o_h[-1])].cpu().numpy().view(np.uint32), rr)

    outs = deformer.deform_frames(w, base.dims, base.bbox, B, X, o)
    check(outs)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            deformer.deform_frames(w, base.dims, base.bbox, B, X, o, outs=outs)
    for _ in range(2):
        for offs, roots in outs:
            offs.fill_(-1)
            roots.zero_()
        g.replay()
        check(outs)


def test_device_frames_validation_and_capacity(deformer):
    """fsk_deform_frames: one bones/points entry per frame, zero frames is a no-op, and a roots buffer
    smaller than a frame's kept roots keeps the first `cap` records with the full offsets (the caller
    checks offsets[N] <= cap, as for fsk_deform)."""
    base, frames = _frames([4000, 4000])
    w = torch.from_numpy(base.weights).cuda()
    o = _opts(base)
    B = [b.cuda() for b, _ in frames]
    X = [p.cuda() for _, p in frames]
    with pytest.raises(FskInvalidArgument):
        deformer.deform_frames(w, base.dims, base.bbox, B[:1], X, o)
    assert deformer.deform_frames(w, base.dims, base.bbox, [], [], o) == []
    full = deformer.deform_frames(w, base.dims, base.bbox, B, X, o)
    small = [(torch.empty(4001, dtype=torch.int64, device="cuda"), torch.zeros((100, 16), device="cuda"))
             for _ in range(2)]
    deformer.deform_frames(w, base.dims, base.bbox, B, X, o, outs=small)
    torch.cuda.synchronize()
    for (fo, fr), (so, sr) in zip(full, small):
        assert torch.equal(fo, so) and int(so[-1]) > 100
        assert torch.equal(fr[:100].view(torch.int32), sr.view(torch.int32))
