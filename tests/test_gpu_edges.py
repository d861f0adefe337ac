"""Edge cases of the search against the f64 oracle (through the C-ABI): short iteration caps
(below the float32 pass's escalation cap), no dedup, minimal / thin grids, ragged point counts
around the warp and CTA sizes, points far outside the grid, duplicated queries, a 40-bone chain
skeleton, and non-finite queries (no oracle: the reference's cell lookup of a NaN is undefined;
the contract kept here is "never converged, never a crash")."""
import numpy as np
import pytest
import torch

import oracle
from paper_2211_15601_b200 import synthetic as S

from test_gpu_parity import MASK_AGREE, TOL_X, _parity, run_gpu

pytestmark = pytest.mark.gpu


def _check(deformer, sc, max_iters, dedup=None, tol=TOL_X):
    o = sc.search_options(max_iters)
    if dedup is not None:
        o["dedup_dist"] = dedup
    from test_gpu_parity import dev
    from paper_2211_15601_b200.deformer import SearchOptions
    w, B, x = dev(sc.weights), dev(sc.bones), dev(sc.points)
    tg64 = torch.empty((w.shape[0], 12), dtype=torch.float64, device="cuda")
    tg = deformer.precompute_transform_grid(w, sc.dims, sc.bbox, B, out64=tg64)
    out = deformer.batch_search(tg, sc.dims, sc.bbox, B, x, SearchOptions(max_iters, o["conv_eps"], o["div_eps"],
                                                                         o["dedup_dist"]), tgrid64=tg64, weights=w)
    g = {k: (v.cpu().numpy() if v is not None else None) for k, v in out.items()}
    r = oracle.batch_search(sc.weights, sc.dims, sc.bbox, sc.bones, sc.points, workers=8, **o)
    agree, dx, _, keep_agree, _ = _parity(g, r, o["conv_eps"])
    assert agree >= MASK_AGREE and keep_agree >= MASK_AGREE and dx <= tol, (agree, keep_agree, dx)
    return g, r


@pytest.mark.parametrize("max_iters", [1, 2, 5, 8, 9])
def test_short_iteration_caps(deformer, max_iters):
    """max_iters at and around the float32 pass's cap of 8 (the cap-escalation boundary)."""
    _check(deformer, S.make_scene((32, 32, 32), 3000, seed=20 + max_iters), max_iters)


def test_no_dedup_keeps_every_converged_root(deformer):
    g, r = _check(deformer, S.make_scene((32, 32, 32), 2000, seed=31), 50, dedup=0.0)
    assert (g["keep"] == g["converged"]).all()


@pytest.mark.parametrize("dims", [(2, 2, 2), (2, 17, 3), (33, 5, 2)])
def test_minimal_and_thin_grids(deformer, dims):
    _check(deformer, S.make_scene(dims, 2000, seed=32), 50)


@pytest.mark.parametrize("n", [1, 31, 33, 127, 129, 1000])
def test_ragged_point_counts(deformer, n):
    g, _ = _check(deformer, S.make_scene((16, 16, 16), n, seed=33), 50)
    assert g["converged"].shape == (n, 24)


def test_points_far_outside_the_grid(deformer):
    sc = S.make_scene((16, 16, 16), 1500, seed=34)
    far = np.random.default_rng(1).normal(size=(500, 3)) * 10 * sc.diag
    sc.points = np.concatenate([sc.points[:1000], far.astype(np.float32)], 0).astype(np.float32)
    _check(deformer, sc, 50)


def test_duplicated_queries_get_identical_results(deformer):
    sc = S.make_scene((32, 32, 32), 64, seed=35)
    sc.points = np.repeat(sc.points[:8], 8, axis=0).astype(np.float32)
    g, _ = _check(deformer, sc, 50)
    for k in ("x_c", "converged", "keep", "iters"):
        v = g[k].reshape(8, 8, *g[k].shape[1:])
        assert (v == v[:, :1]).all(), k


def test_forty_bone_chain(deformer):
    """A 40 m chain (conv_eps = 1e-5·diag = 5e-4): the search's own stopping tolerance is coarser
    than the north star's 1e-4, so the float32 pass hands every converged solve to the float64
    pass (SearchP::esc_conv_all) and positions meet 1e-4 abs like the SMPL-scale scenes."""
    skel = S.chain_skeleton(40, radius=0.2)
    sc = S.make_scene((48, 12, 12), 2000, seed=36, skeleton=skel)
    g, _ = _check(deformer, sc, 50)
    assert g["converged"].shape == (2000, 40)


def test_non_finite_queries_never_converge(deformer):
    sc = S.make_scene((16, 16, 16), 100, seed=37)
    bad = np.array([[np.nan, 0, 0], [np.inf, 0, 0], [0, -np.inf, 0], [np.nan] * 3], np.float32)
    sc.points = np.concatenate([sc.points, bad], 0).astype(np.float32)
    _, g = run_gpu(deformer, sc, 50)
    assert (g["converged"][-4:] == 0).all() and (g["n_roots"][-4:] == 0).all()
    assert g["converged"][:-4].any()


def test_max_iters_beyond_255(deformer):
    """The reference accepts any max_iters >= 1 (correspondence.cpp:20); iteration counts are
    int32 end to end (the long float64 re-solves run to the cap)."""
    g, r = _check(deformer, S.make_scene((32, 32, 32), 3000, seed=38), 300)
    both = (g["converged"] == 1) & (r["converged"] == 1)
    assert (g["iters"][both] == r["iters"][both]).mean() > 0.999


def test_float64_bbox_not_representable_in_float32(deformer):
    """The reference's Aabb is float64 (geometry.hpp:14-39): a box that float32 cannot represent
    reaches the search as given (the float32 pass rounds it, the float64 re-solves do not)."""
    sc = S.make_scene((32, 32, 32), 3000, seed=39)
    sc.bbox = sc.bbox.astype(np.float64) + np.array([1e-9, -3e-9, 2e-9, 5e-9, 1e-9, -7e-9])
    assert (sc.bbox.astype(np.float32).astype(np.float64) != sc.bbox).all()
    _check(deformer, sc, 50)
