"""Single-process multi-GPU C-ABI (fsk_multi_*) on the devices this box has. With one device
the sharding is trivial, so the test pins the API contract: results bitwise equal to the
one-context entry points (fsk_deform_host; fsk_search_bwd_roots + fsk_grad_weights), NCCL
communicator creation and the all-reduce path included."""
import numpy as np
import pytest
import torch

from paper_2211_15601_b200 import synthetic as S
from paper_2211_15601_b200.deformer import Deformer, FskInvalidArgument, MultiDeformer, SearchOptions

pytestmark = pytest.mark.gpu


def _opts(sc):
    o = sc.search_options(50)
    return SearchOptions(50, o["conv_eps"], o["div_eps"], o["dedup_dist"])


def test_multi_deform_equals_single(deformer):
    sc = S.make_scene((32, 32, 32), 20_000, seed=8, points="training")
    n, nb = sc.points.shape[0], sc.n_bones
    hw, hb, hx = (torch.from_numpy(a) for a in (sc.weights, sc.bones, sc.points))
    o1, r1 = torch.empty(n + 1, dtype=torch.int64), torch.empty((n * nb, 16), dtype=torch.float32)
    t1 = deformer.deform_host(hw, sc.dims, sc.bbox, hb, hx, _opts(sc), o1, r1)
    M = MultiDeformer(list(range(torch.cuda.device_count())))
    o2, r2 = torch.empty(n + 1, dtype=torch.int64), torch.empty((n * nb, 16), dtype=torch.float32)
    t2 = M.deform_host(hw, sc.dims, sc.bbox, hb, hx, _opts(sc), o2, r2)
    print(f"\n{M.device_count} device(s): {t2} roots")
    assert t1 == t2 and torch.equal(o1, o2) and torch.equal(r1[:t1], r2[:t2])
    # the backward over the devices
    ridx = torch.where(o2[1:] > o2[:-1], o2[:-1], torch.full_like(o2[:-1], -1))
    gx = (torch.randn((n, 3), generator=torch.Generator().manual_seed(5)) / n).float()
    gw = M.grad_weights_host(sc.dims, sc.bbox, hb, r2, ridx, gx)
    gT = deformer.search_bwd_roots(sc.dims, sc.bbox, nb, r2[: max(t2, 1)].cuda(), ridx.cuda(), gx.cuda())
    gw1 = deformer.grad_weights(sc.dims, sc.bbox, gT, hb.cuda()).cpu()
    err = (gw - gw1).abs().max().item()
    print(f"multi grad_w vs single: max|d| {err:.2e}")
    assert err <= 1e-6 * gw1.abs().max().item()
    M.close()


def test_multi_validation():
    with pytest.raises(FskInvalidArgument, match="duplicate device"):
        MultiDeformer([0, 0])
    with pytest.raises(FskInvalidArgument, match="at least one device"):
        MultiDeformer([])
