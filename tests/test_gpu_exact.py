"""GPU exact-replay mode (FSK_SEARCH_EXACT64, SearchOptions.precision="exact64") against the oracle.

The replay runs every solve in float64 with the reference's own operation order (unfused
multiply/add, the oracle's locate/trilerp/apply order, J~0 from the n_b-wide weight grid), so
its results are the oracle's BIT FOR BIT — no tolerance: masks, iteration counts, keep masks
equal; x_c, J~ and the residual equal the oracle's float64 values rounded to float32. This
closes the rare long-trajectory outliers of the default mixed path.
"""
import numpy as np
import pytest
import torch

import oracle
from paper_2211_15601_b200 import synthetic as S
from paper_2211_15601_b200.deformer import FskInvalidArgument, SearchOptions

pytestmark = pytest.mark.gpu


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def opts_of(sc, max_iters, precision="exact64"):
    o = SearchOptions(max_iters=max_iters,
                      **{k: v for k, v in sc.search_options(max_iters).items() if k != "max_iters"})
    o.precision = precision
    return o


def exact_search(deformer, sc, max_iters, tg64=None):
    w, B, x = dev(sc.weights), dev(sc.bones), dev(sc.points)
    if tg64 is None:
        tg64 = torch.empty((w.shape[0], 12), dtype=torch.float64, device="cuda")
        deformer.precompute_transform_grid(w, sc.dims, sc.bbox, B, out64=tg64)
    out = deformer.batch_search(None, sc.dims, sc.bbox, B, x, opts_of(sc, max_iters), tgrid64=tg64, weights=w,
                                out=deformer.alloc_search_out(x.shape[0], sc.n_bones, x64=True))
    torch.cuda.synchronize()
    return {k: (v.cpu().numpy() if v is not None else None) for k, v in out.items()}


def assert_bitwise(g, r):
    n, nb = r["converged"].shape
    np.testing.assert_array_equal(g["converged"], r["converged"])
    np.testing.assert_array_equal(g["iters"].astype(np.int32), r["iters"])
    np.testing.assert_array_equal(g["x_c"], r["x_c"].astype(np.float32))
    if g.get("x_c64") is not None:  # the replay's float64 roots themselves (Root::x), not just their rounding
        np.testing.assert_array_equal(g["x_c64"], r["x_c"])
    np.testing.assert_array_equal(g["jinv"], r["jinv"].astype(np.float32).reshape(g["jinv"].shape))
    np.testing.assert_array_equal(g["resid"], r["resid"].astype(np.float32))
    np.testing.assert_array_equal(g["keep"], r["keep"])


def test_precompute_f64_grid_is_lbs_blend_bitwise(deformer):
    """K1's float64 grid accumulates unfused in bone order: the oracle's lbs_blend exactly."""
    sc = S.make_scene((32, 32, 32), 10, seed=3)
    w, B = dev(sc.weights), dev(sc.bones)
    tg64 = torch.empty((w.shape[0], 12), dtype=torch.float64, device="cuda")
    deformer.precompute_transform_grid(w, sc.dims, sc.bbox, B, out64=tg64)
    ref = oracle.precompute_transform_grid(sc.weights, sc.dims, sc.bbox, sc.bones)
    np.testing.assert_array_equal(tg64.cpu().numpy(), ref)


@pytest.mark.parametrize("dims,seed,points,max_iters", [
    ((32, 32, 32), 1, "uniform", 10),     # BASELINE config 1
    ((32, 32, 32), 1, "uniform", 50),
    ((64, 64, 64), 10, "uniform", 50),
    ((16, 16, 16), 11, "training", 50),
    ((64, 64, 16), 11, "training", 50),
    ((64, 64, 64), 25, "training", 50),
])
def test_exact64_search_is_the_oracle_bitwise(deformer, dims, seed, points, max_iters):
    sc = S.make_scene(dims, 10_000, seed=seed, points=points)
    g = exact_search(deformer, sc, max_iters)
    r = oracle.batch_search(sc.weights, sc.dims, sc.bbox, sc.bones, sc.points, workers=8,
                            **sc.search_options(max_iters))
    assert_bitwise(g, r)


def test_exact64_with_the_oracle_grid(deformer):
    """A caller-provided float64 TransformGrid (the oracle's) gives the same bits."""
    sc = S.make_scene((32, 32, 32), 5_000, seed=4, points="training")
    tg = oracle.precompute_transform_grid(sc.weights, sc.dims, sc.bbox, sc.bones)
    g = exact_search(deformer, sc, 50, tg64=dev(tg))
    r = oracle.batch_search(sc.weights, sc.dims, sc.bbox, sc.bones, sc.points, workers=8, tgrid=tg,
                            **sc.search_options(50))
    assert_bitwise(g, r)


def test_exact64_deform_roots_equal_oracle(deformer):
    """fsk_deform (K1 + exact search + dedup + compaction) emits the oracle's kept roots."""
    sc = S.make_scene((32, 32, 32), 8_000, seed=5, points="training")
    w, B, x = dev(sc.weights), dev(sc.bones), dev(sc.points)
    offs, roots = deformer.deform(w, sc.dims, sc.bbox, B, x, opts_of(sc, 50))
    torch.cuda.synchronize()
    offs, roots = offs.cpu().numpy(), roots.cpu().numpy()
    r = oracle.batch_search(sc.weights, sc.dims, sc.bbox, sc.bones, sc.points, workers=8, **sc.search_options(50))
    n, nb = r["keep"].shape
    np.testing.assert_array_equal(np.diff(offs), r["keep"].sum(1))
    q, b = np.nonzero(r["keep"])  # row-major: per query, bone order
    np.testing.assert_array_equal(roots[: offs[-1], :3], r["x_c"][q, b].astype(np.float32))
    np.testing.assert_array_equal(roots[: offs[-1], 3], r["resid"][q, b].astype(np.float32))


def test_exact64_needs_weights(deformer):
    sc = S.make_scene((16, 16, 16), 100, seed=1)
    w, B, x = dev(sc.weights), dev(sc.bones), dev(sc.points)
    tg64 = torch.empty((w.shape[0], 12), dtype=torch.float64, device="cuda")
    deformer.precompute_transform_grid(w, sc.dims, sc.bbox, B, out64=tg64)
    with pytest.raises(FskInvalidArgument, match="needs the weight grid"):
        deformer.batch_search(None, sc.dims, sc.bbox, B, x, opts_of(sc, 10), tgrid64=tg64)
    o = opts_of(sc, 10)
    o.precision = "exact64"
    o.sort = False  # order-independent like every mode
    a = deformer.batch_search(None, sc.dims, sc.bbox, B, x, o, tgrid64=tg64, weights=w)
    b = deformer.batch_search(None, sc.dims, sc.bbox, B, x, opts_of(sc, 10), tgrid64=tg64, weights=w)
    for k in a:
        if a[k] is not None:
            torch.testing.assert_close(a[k], b[k], rtol=0, atol=0)


@pytest.mark.parametrize("dims,seed,points", [((32, 32, 32), 1, "uniform"), ((64, 64, 16), 11, "training"),
                                              ((64, 64, 64), 25, "training")])
def test_mixed_escalations_are_the_oracle_bitwise(deformer, dims, seed, points):
    """Default mixed mode with the weight grid: the float64 escalation pass runs the exact replay, so every
    escalated solve equals the oracle bit for bit (at least as many bit-equal solves as were
    escalated), and the whole result keeps the north-star bar."""
    sc = S.make_scene(dims, 20_000, seed=seed, points=points)
    w, B, x = dev(sc.weights), dev(sc.bones), dev(sc.points)
    tg64 = torch.empty((w.shape[0], 12), dtype=torch.float64, device="cuda")
    tg = deformer.precompute_transform_grid(w, sc.dims, sc.bbox, B, out64=tg64)
    deformer.search_stats(reset=True)
    out = deformer.batch_search(tg, sc.dims, sc.bbox, B, x, opts_of(sc, 50, "mixed"), tgrid64=tg64, weights=w,
                                out=deformer.alloc_search_out(x.shape[0], sc.n_bones, x64=True))
    torch.cuda.synchronize()
    n_esc = deformer.search_stats(reset=True)[3]
    g = {k: (v.cpu().numpy() if v is not None else None) for k, v in out.items()}
    r = oracle.batch_search(sc.weights, sc.dims, sc.bbox, sc.bones, sc.points, workers=8, **sc.search_options(50))
    same = ((g["converged"] == r["converged"]) & (g["iters"].astype(np.int32) == r["iters"])
            & (g["resid"] == r["resid"].astype(np.float32))
            & (g["x_c64"] == r["x_c"]).all(-1))  # the float64 root itself (Root::x)
    print(f"\n{dims} {points}: escalated {n_esc}, bit-equal to the oracle in float64 {int(same.sum())} of {same.size}, "
          f"mask agreement {(g['converged'] == r['converged']).mean():.7f}")
    assert n_esc > 0
    assert same.sum() >= n_esc
    assert (g["converged"] == r["converged"]).mean() >= 0.9999
    both = (g["converged"] == 1) & (r["converged"] == 1)
    assert np.abs(g["x_c"] - r["x_c"])[both].max() <= 1e-4


@pytest.mark.parametrize("n_bones", [21, 80])
def test_mixed_escalations_bitwise_other_bone_counts(deformer, n_bones, monkeypatch):
    """The escalation start kernel's one-pass J~0 (weight gradients parked in shared memory) has a
    scalar-weight path for n_b % 4 != 0 (21 bones) and falls back to the two-pass form when the
    stash does not fit in shared memory (80 bones: 80·3 doubles × 128 threads > 227 KB). Both must
    still replay the oracle bit for bit.

    Position tolerance: the north star's 1e-4 abs. These chains are long (80 bones: diag ≈ 99,
    conv_eps ≈ 1e-3), so the float32 pass escalates every converged solve (conv_eps > 5e-5,
    SearchP::esc_conv_all) and the converged roots are the exact replay's."""
    # 80 bones: the start states k_esc_start precomputes are capped below the escalation count
    # (FSK_ESC_START_CAP, a testing override), so the refill kernel's own start path runs too
    n = 8_000 if n_bones == 80 else 4_000
    if n_bones == 80:
        monkeypatch.setenv("FSK_ESC_START_CAP", "20000")
    sc = S.make_scene((32, 32, 32), n, seed=3, skeleton=S.chain_skeleton(n_bones))
    w, B, x = dev(sc.weights), dev(sc.bones), dev(sc.points)
    tg64 = torch.empty((w.shape[0], 12), dtype=torch.float64, device="cuda")
    tg = deformer.precompute_transform_grid(w, sc.dims, sc.bbox, B, out64=tg64)
    deformer.search_stats(reset=True)
    out = deformer.batch_search(tg, sc.dims, sc.bbox, B, x, opts_of(sc, 50, "mixed"), tgrid64=tg64, weights=w)
    torch.cuda.synchronize()
    n_esc = deformer.search_stats(reset=True)[3]
    g = {k: (v.cpu().numpy() if v is not None else None) for k, v in out.items()}
    r = oracle.batch_search(sc.weights, sc.dims, sc.bbox, sc.bones, sc.points, workers=8, **sc.search_options(50))
    same = ((g["converged"] == r["converged"]) & (g["iters"].astype(np.int32) == r["iters"])
            & (g["resid"] == r["resid"].astype(np.float32))
            & (g["x_c"] == r["x_c"].astype(np.float32)).all(-1))
    both = (g["converged"] == 1) & (r["converged"] == 1)
    dx = np.abs(g["x_c"] - r["x_c"])[both].max()
    conv = sc.search_options(50)["conv_eps"]
    print(f"\n{n_bones} bones: escalated {n_esc}, bit-equal to the oracle {int(same.sum())} of {same.size}, "
          f"max|dx| {dx:.2e} (conv_eps {conv:.2e})")
    assert n_esc > 0
    if n_bones == 80:
        assert n_esc > 20000  # the in-kernel start path ran
    assert same.sum() >= n_esc
    assert (g["converged"] == r["converged"]).mean() >= 0.9999
    assert dx <= 1e-4
