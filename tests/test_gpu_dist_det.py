"""Deterministic backward across ranks (dist.py, one process per shard): the int64 fixed-point gradient
under a shared scale (max term all-reduced with MAX, n = all points) summed exactly over the ranks is
bitwise the single-process deterministic gradient. Two ranks share cuda:0 over gloo (a one-GPU box
cannot run NCCL ranks side by side; the protocol is the same)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _scene():
    from paper_2211_15601_b200 import synthetic as S
    return S.make_scene((32, 32, 32), 6000, seed=8, points="training")


def _worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from paper_2211_15601_b200.deformer import Deformer, SearchOptions
    from paper_2211_15601_b200.dist import MultiGPUDeformer, shard_range
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    D = Deformer(0)
    sc = _scene()
    n = sc.points.shape[0]
    a, b = shard_range(n, rank, world)
    w, B = torch.from_numpy(sc.weights).cuda(), torch.from_numpy(sc.bones).cuda()
    o = sc.search_options(50)
    tg = D.precompute_transform_grid(w, sc.dims, sc.bbox, B)
    dense = D.batch_search(tg, sc.dims, sc.bbox, B, torch.from_numpy(sc.points[a:b]).cuda(),
                           SearchOptions(50, o["conv_eps"], o["div_eps"], o["dedup_dist"]))
    keep = dense["keep"].cpu().numpy()
    sel = torch.from_numpy(np.where(keep.any(1), np.argmax(keep, 1), -1).astype(np.int32)).cuda()
    v = torch.from_numpy((np.random.default_rng(9).normal(size=(n, 3)) / n).astype(np.float32)[a:b]).cuda()
    gT, gW = MultiGPUDeformer(D).backward(sc.dims, sc.bbox, B, dense, v, sel, deterministic=True)
    np.save(os.path.join(out_dir, f"gT{rank}.npy"), gT.cpu().numpy())
    # the sharded forward through dist.py (broadcast pose inputs from rank 0, per-rank search with the
    # GPU kernels, all-gather of the dense results): equal to the single-process search
    wb = w.clone() if rank == 0 else torch.zeros_like(w)
    Bb = B.clone() if rank == 0 else torch.zeros_like(B)
    _, res, _ = MultiGPUDeformer(D).forward(wb, sc.dims, sc.bbox, Bb, torch.from_numpy(sc.points).cuda(),
                                            SearchOptions(50, o["conv_eps"], o["div_eps"], o["dedup_dist"]))
    if rank == 0:
        np.savez(os.path.join(out_dir, "fwd.npz"), **{k: t.cpu().numpy() for k, t in res.items() if t is not None})
    dist.destroy_process_group()


def test_deterministic_backward_is_bitwise_across_rank_counts(deformer, tmp_path):
    from paper_2211_15601_b200.deformer import SearchOptions
    sc = _scene()
    n = sc.points.shape[0]
    w, B = torch.from_numpy(sc.weights).cuda(), torch.from_numpy(sc.bones).cuda()
    o = sc.search_options(50)
    tg = deformer.precompute_transform_grid(w, sc.dims, sc.bbox, B)
    dense = deformer.batch_search(tg, sc.dims, sc.bbox, B, torch.from_numpy(sc.points).cuda(),
                                  SearchOptions(50, o["conv_eps"], o["div_eps"], o["dedup_dist"]))
    keep = dense["keep"].cpu().numpy()
    sel = torch.from_numpy(np.where(keep.any(1), np.argmax(keep, 1), -1).astype(np.int32)).cuda()
    v = torch.from_numpy((np.random.default_rng(9).normal(size=(n, 3)) / n).astype(np.float32)).cuda()
    ref = deformer.search_bwd(sc.dims, sc.bbox, sc.n_bones, dense, v, sel, deterministic=True).cpu().numpy()
    tg64 = torch.empty((w.shape[0], 12), dtype=torch.float64, device="cuda")
    tg = deformer.precompute_transform_grid(w, sc.dims, sc.bbox, B, out64=tg64)
    full = deformer.batch_search(tg, sc.dims, sc.bbox, B, torch.from_numpy(sc.points).cuda(),
                                 SearchOptions(50, o["conv_eps"], o["div_eps"], o["dedup_dist"]), tgrid64=tg64, weights=w)
    for world in (2, 3):
        mp.spawn(_worker, args=(world, _port(), str(tmp_path)), nprocs=world, join=True)
        for r in range(world):
            np.testing.assert_array_equal(np.load(tmp_path / f"gT{r}.npy").view(np.uint32), ref.view(np.uint32))
        fwd = np.load(tmp_path / "fwd.npz")
        for k in ("x_c", "converged", "keep", "iters", "n_roots"):
            np.testing.assert_array_equal(fwd[k], full[k].cpu().numpy())
