"""Multi-GPU plumbing: posed points shard across ranks (one process per GPU, NCCL).

The correspondence search has no data-path exchange — every (point, init) solve reads
only the immutable transform grid and bones — so the forward is pure
data parallelism over contiguous point ranges, the partition of ``parallel_for``
(``proj/include/fskin/parallel.hpp:28-29``). Collectives appear only at the edges:

* before K1: ``broadcast`` of the weight grid and bones from the rank that owns the pose
  (each rank then runs K1 locally — cheaper than broadcasting per-pose T grids);
* after K2 (optional): ``all_gather`` of the per-rank dense results (unequal shard sizes
  are padded to the largest shard);
* backward: ``all_reduce(SUM)`` of dL/dT [V,12] before the local dL/dw contraction.

The compute functions are injected so the same plumbing is exercised on CPU with the
``gloo`` backend in tests (tests/test_dist_gloo.py) and on GPUs with NCCL.
"""
from __future__ import annotations

from typing import Callable, Dict, Optional

import torch
import torch.distributed as dist


def shard_range(n: int, rank: int, world: int):
    """``parallel_for``'s static contiguous partition (parallel.hpp:28-29)."""
    return n * rank // world, n * (rank + 1) // world


def broadcast_inputs(tensors, src: int = 0, group=None):
    """Broadcast the pose inputs (weight grid, bones) from ``src`` to every rank, in place."""
    for t in tensors:
        dist.broadcast(t, src, group=group)
    return tensors


def gather_dense(local: Dict[str, Optional[torch.Tensor]], n_total: int, group=None) -> Dict[str, torch.Tensor]:
    """All-gather per-rank dense search results (leading dim = local points) into the
    full [n_total, ...] arrays in global point order."""
    world = dist.get_world_size(group)
    sizes = [shard_range(n_total, r, world) for r in range(world)]
    maxn = max(b - a for a, b in sizes)
    out = {}
    for k, t in local.items():
        if t is None:
            out[k] = None
            continue
        pad = torch.zeros((maxn, *t.shape[1:]), dtype=t.dtype, device=t.device)
        pad[: t.shape[0]] = t
        bufs = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(bufs, pad, group=group)
        out[k] = torch.cat([bufs[r][: b - a] for r, (a, b) in enumerate(sizes)], 0)
    return out


def allreduce_grad(grad: torch.Tensor, group=None) -> torch.Tensor:
    dist.all_reduce(grad, op=dist.ReduceOp.SUM, group=group)
    return grad


def sharded_forward(points_full: torch.Tensor, search_fn: Callable[[torch.Tensor], Dict[str, torch.Tensor]],
                    gather: bool = True, group=None):
    """Run ``search_fn`` on this rank's contiguous shard of ``points_full``; optionally
    all-gather the dense results. Returns (results, (begin, end))."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    a, b = shard_range(points_full.shape[0], rank, world)
    local = search_fn(points_full[a:b].contiguous())
    if gather:
        return gather_dense(local, points_full.shape[0], group=group), (a, b)
    return local, (a, b)


def sharded_backward(local_grad_fn: Callable[[], torch.Tensor],
                     contract_fn: Optional[Callable[[torch.Tensor], torch.Tensor]] = None, group=None):
    """Per-rank dL/dT from the local roots, summed over ranks, then (optionally) the local
    dL/dw contraction — identical on every rank."""
    g = allreduce_grad(local_grad_fn(), group=group)
    return (g, contract_fn(g)) if contract_fn else (g, None)


class MultiGPUDeformer:
    """One rank of the sharded deformer over ``paper_2211_15601_b200.deformer.Deformer``."""

    def __init__(self, deformer, group=None):
        self.D, self.group = deformer, group

    def forward(self, weights, dims, bbox, bones, points_full, opts, src=0, gather=True):
        broadcast_inputs([weights, bones], src=src, group=self.group)
        tg64 = torch.empty((weights.shape[0], 12), dtype=torch.float64, device=weights.device)
        tg = self.D.precompute_transform_grid(weights, dims, bbox, bones, out64=tg64)
        # the weight grid goes along (J~0 and the float64 re-solves in the oracle's operation order)
        res, rng = sharded_forward(points_full,
                                   lambda x: self.D.batch_search(tg, dims, bbox, bones, x, opts, tgrid64=tg64,
                                                                 weights=weights),
                                   gather=gather, group=self.group)
        return tg, res, rng

    def backward(self, dims, bbox, bones, local_dense, grad_xc_local, root_sel_local, deterministic=False,
                 n_total=None):
        """dL/dT (and dL/dw) of the whole batch on every rank. ``deterministic``: every rank rounds its
        terms to int64 fixed point with the SAME scale (the max term all-reduced with MAX, n = the total
        point count) and the int64 sums are all-reduced exactly, so the result is bitwise the
        single-process deterministic gradient for any world size."""
        nb = bones.numel() // 12
        if not deterministic:
            return sharded_backward(
                lambda: self.D.search_bwd(dims, bbox, nb, local_dense, grad_xc_local, root_sel_local, False),
                lambda g: self.D.grad_weights(dims, bbox, g, bones), group=self.group)
        src = dict(dense=local_dense, root_sel=root_sel_local)
        if n_total is None:
            t = torch.tensor([grad_xc_local.shape[0]], dtype=torch.int64, device=grad_xc_local.device)
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
            n_total = int(t.item())
        mt = self.D.search_bwd_max_term(dims, bbox, nb, grad_xc_local, **src)
        dist.all_reduce(mt, op=dist.ReduceOp.MAX, group=self.group)
        V = dims[0] * dims[1] * dims[2]
        acc = torch.zeros((V, 12), dtype=torch.int64, device=grad_xc_local.device)
        self.D.search_bwd_fixed(dims, bbox, nb, grad_xc_local, n_total, mt, acc, **src)
        dist.all_reduce(acc, op=dist.ReduceOp.SUM, group=self.group)
        g = self.D.fixed_to_float(acc, n_total, mt)
        return g, self.D.grad_weights(dims, bbox, g, bones)
