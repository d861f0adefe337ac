"""GPU parity of the MLP stages next to the search, tcgen05 path
through the C-ABI, against the f64 oracle (oracle/mlp_oracle.cpp) on identical float32
parameters and inputs.

Tolerance: the tensor-core path is FP32-faithful (3xTF32 split), so softmax weights and
occupancies must agree with the float64 network to 1e-5 abs (measured ~1e-7)."""
import numpy as np
import pytest
import torch

import oracle
from paper_2211_15601_b200 import synthetic as S
from paper_2211_15601_b200.deformer import FskInvalidArgument, SearchOptions

pytestmark = pytest.mark.gpu

TOL = 1e-5
SKIN = [3, 64, 64, 64, 24]       # SkinningMlp (skinning.cpp:10-17)
OCC = [3, 128, 128, 128, 1]      # OccupancyMlp (shape.cpp:181-184), no pose conditioning


def theta32(widths, seed, head_scale=1.0):
    """float32 parameters; the oracle runs on the same (float32-exact) values."""
    return oracle.mlp_init(widths, seed, head_scale).astype(np.float32)


@pytest.mark.parametrize("dims,head_scale", [((32, 32, 32), 1.0), ((32, 32, 8), 0.05), ((17, 9, 5), 1.0)])
def test_distill_matches_oracle(deformer, dims, head_scale):
    sc = S.make_scene((4, 4, 4), 10, seed=1)
    th = theta32(SKIN, 3, head_scale)
    w = deformer.distill(torch.from_numpy(th).cuda(), SKIN, dims, sc.bbox).cpu().numpy()
    r = oracle.distill(th, SKIN, dims, sc.bbox)
    err = np.abs(w - r).max()
    print(f"\ndistill {dims}: max|dw| {err:.2e}, row sums within {np.abs(w.sum(1) - 1).max():.1e} of 1")
    assert err <= TOL
    assert np.abs(w.sum(1) - 1).max() <= 1e-5


def test_distill_other_widths(deformer):
    """n_b = 7 (head padded to N = 32) and one hidden layer; H = 128 (weights streamed)."""
    sc = S.make_scene((4, 4, 4), 10, seed=1)
    for widths in ([3, 64, 64, 7], [3, 128, 128, 128, 40], [3, 64, 64, 64, 64, 64, 33]):
        th = theta32(widths, 5)
        w = deformer.distill(torch.from_numpy(th).cuda(), widths, (9, 8, 7), sc.bbox).cpu().numpy()
        r = oracle.distill(th, widths, (9, 8, 7), sc.bbox)
        print(f"\n{widths}: max|dw| {np.abs(w - r).max():.2e}")
        assert np.abs(w - r).max() <= TOL


def _roots_from_search(deformer, sc):
    opts = sc.search_options(50)
    w, B, x = (torch.from_numpy(a).cuda() for a in (sc.weights, sc.bones, sc.points))
    offs, roots = deformer.deform(w, sc.dims, sc.bbox, B, x, SearchOptions(50, opts["conv_eps"], opts["div_eps"],
                                                                            opts["dedup_dist"]))
    torch.cuda.synchronize()
    return offs, roots


@pytest.mark.parametrize("n_pose", [0, 24])
def test_posed_occupancy_matches_oracle(deformer, n_pose):
    sc = S.make_scene((32, 32, 32), 6000, seed=7, points="training")
    offs, roots = _roots_from_search(deformer, sc)
    widths = [3 + n_pose] + OCC[1:]
    th = theta32(widths, 11)
    pose = np.random.default_rng(2).uniform(-0.5, 0.5, n_pose).astype(np.float32)
    pred, am = deformer.posed_occupancy(torch.from_numpy(th).cuda(), widths, pose, offs, roots)
    pred, am = pred.cpu().numpy(), am.cpu().numpy()
    o = offs.cpu().numpy()
    rx = roots[: o[-1], :3].cpu().numpy()
    rp, ra = oracle.posed_occupancy(th, widths, pose, o, rx)
    err = np.abs(pred - rp).max()
    print(f"\nposed occupancy (n_pose {n_pose}): {o[-1]} roots over {len(pred)} queries, max|d occ| {err:.2e}, "
          f"argmax agreement {(am == ra).mean():.6f}, empty sets {(ra < 0).sum()}")
    assert err <= TOL
    # argmax may differ only where two roots' occupancies tie within the tolerance
    diff = np.nonzero(am != ra)[0]
    occ_all = oracle.mlp_forward(th, widths, np.concatenate([rx, np.broadcast_to(pose, (len(rx), n_pose))], 1))
    occ_all = 1.0 / (1.0 + np.exp(-occ_all[:, 0]))
    for q in diff:
        assert am[q] >= 0 and ra[q] >= 0
        assert abs(occ_all[o[q] + am[q]] - occ_all[o[q] + ra[q]]) <= 2 * TOL


def test_posed_occupancy_empty_and_validation(deformer):
    th = torch.from_numpy(theta32(OCC, 1)).cuda()
    offs = torch.zeros(4, dtype=torch.int64, device="cuda")  # three empty sets
    roots = torch.zeros((1, 16), dtype=torch.float32, device="cuda")
    pred, am = deformer.posed_occupancy(th, OCC, None, offs, roots)
    assert (pred.cpu().numpy() == 0).all() and (am.cpu().numpy() == -1).all()
    with pytest.raises(FskInvalidArgument, match="pose vector length 2, field conditioned on 0"):
        deformer.posed_occupancy(th, OCC, np.zeros(2, np.float32), offs, roots)
    with pytest.raises(FskInvalidArgument, match="expected input >= 3, scalar output"):
        deformer.posed_occupancy(th, [3, 128, 128, 2], None, offs, roots)
    sc = S.make_scene((4, 4, 4), 10, seed=1)
    with pytest.raises(FskInvalidArgument, match="hidden width must be 64 or 128"):
        deformer.distill(torch.zeros(10000, device="cuda"), [3, 32, 32, 24], (4, 4, 4), sc.bbox)
    import ctypes
    from paper_2211_15601_b200.deformer import check, grid_desc
    desc = grid_desc((4, 4, 4), sc.bbox, 23)  # grid built for 23 bones, network has 24 outputs
    out = torch.empty((64, 24), device="cuda")
    th24 = torch.from_numpy(theta32(SKIN, 1)).cuda()
    with pytest.raises(FskInvalidArgument, match="distill: bone count mismatch"):
        check(deformer.L.fsk_distill(deformer._ctx, ctypes.c_void_p(th24.data_ptr()), deformer._widths(SKIN),
                                     len(SKIN), ctypes.byref(desc), ctypes.c_void_p(out.data_ptr()), None))


def test_distill_feeds_the_search(deformer):
    """distill -> precompute -> search: the distilled float32 grid drives the deformer like an
    analytic one (skinning weights are a partition of unity, search is sound)."""
    sc = S.make_scene((32, 32, 32), 4000, seed=3)
    th = theta32(SKIN, 9, 0.05)
    w = deformer.distill(torch.from_numpy(th).cuda(), SKIN, sc.dims, sc.bbox)
    B, x = torch.from_numpy(sc.bones).cuda(), torch.from_numpy(sc.points).cuda()
    o = sc.search_options(50)
    offs, roots = deformer.deform(w, sc.dims, sc.bbox, B, x, SearchOptions(50, o["conv_eps"], o["div_eps"],
                                                                          o["dedup_dist"]))
    torch.cuda.synchronize()
    n_roots = int(offs[-1].item())
    assert n_roots > 0
    assert (roots[:n_roots, 3] < o["conv_eps"]).all()  # every emitted root converged


@pytest.mark.parametrize("dims,widths", [((32, 32, 8), SKIN), ((16, 16, 16), [3, 64, 64, 7]),
                                         ((9, 8, 7), [3, 128, 128, 128, 30])])
def test_distill_backward_matches_oracle_vjp(deformer, dims, widths):
    """dL/dtheta of distill (Mlp::backward through the softmax head) vs the f64 oracle VJP."""
    sc = S.make_scene((4, 4, 4), 10, seed=1)
    th = theta32(widths, 13, 0.05)
    V = dims[0] * dims[1] * dims[2]
    dw = (np.random.default_rng(4).normal(size=(V, widths[-1])) / V).astype(np.float32)
    g = deformer.distill_bwd(torch.from_numpy(th).cuda(), widths, dims, sc.bbox, torch.from_numpy(dw).cuda())
    g = g.cpu().numpy()
    r = oracle.distill_vjp(th, widths, dims, sc.bbox, dw)
    err = np.abs(g - r).max()
    print(f"\ndistill bwd {dims} {widths}: max|dg| {err:.2e} (max|g| {np.abs(r).max():.2e})")
    assert err <= 1e-4 * np.abs(r).max() + 1e-7


def test_training_chain_grid_to_skinning_params(deformer):
    """K3 (implicit-diff backward to the transform grid) -> dL/dw -> dL/dtheta: the GPU chain
    against the oracle chain on the same roots (diff.cpp:336-359 with the grid in the loop)."""
    sc = S.make_scene((32, 32, 8), 3000, seed=12, points="training")
    th = theta32(SKIN, 21, 0.05)
    tht = torch.from_numpy(th).cuda()
    w = deformer.distill(tht, SKIN, sc.dims, sc.bbox)
    B, x = torch.from_numpy(sc.bones).cuda(), torch.from_numpy(sc.points).cuda()
    o = sc.search_options(50)
    offs, roots = deformer.deform(w, sc.dims, sc.bbox, B, x, SearchOptions(50, o["conv_eps"], o["div_eps"],
                                                                          o["dedup_dist"]))
    n = x.shape[0]
    ridx = torch.where(offs[1:] > offs[:-1], offs[:-1], torch.full_like(offs[:-1], -1))
    gx = torch.randn((n, 3), generator=torch.Generator(device="cuda").manual_seed(3), device="cuda") / n
    gT = deformer.search_bwd_roots(sc.dims, sc.bbox, 24, roots, ridx, gx)
    gW = deformer.grad_weights(sc.dims, sc.bbox, gT, B)
    gth = deformer.distill_bwd(tht, SKIN, sc.dims, sc.bbox, gW).cpu().numpy()
    # oracle chain from the same roots (x*, J~) and cotangents
    ri = ridx.cpu().numpy()
    sel = ri >= 0
    R = roots.cpu().numpy()
    _, rw = oracle.grid_vjp(sc.dims, sc.bbox, sc.bones, R[ri[sel], :3], R[ri[sel], 4:13], gx.cpu().numpy()[sel])
    rth = oracle.distill_vjp(th, SKIN, sc.dims, sc.bbox, rw)
    err = np.abs(gth - rth).max()
    print(f"\nchain dL/dtheta: max|d| {err:.2e} (max|g| {np.abs(rth).max():.2e})")
    assert err <= 1e-4 * np.abs(rth).max() + 1e-7
