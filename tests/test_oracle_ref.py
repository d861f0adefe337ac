"""The oracle against the REFERENCE'S OWN hot-path sources: oracle/_ref/libfskin_ref.so is
/root/reference/proj/src/{geometry,skinning,deformer,correspondence}.cpp compiled unmodified with the
reference's build flags against a minimal restatement of the Eigen3 subset they use
(oracle/eigen_shim; Eigen3 is the path's only third-party dependency and is absent from this image).
Everything but Eigen's internals — cell lookup, trilinear loops, lbs_blend, the analytic Jacobian,
init_states, iterate, dedup_roots, batch_search, parallel_for — is the reference's code. CPU tests:
the oracle (every operation-order variant) gives the reference's CorrespondenceSets."""
import numpy as np
import pytest

import oracle
from paper_2211_15601_b200 import synthetic as S

pytestmark = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built (needs /root/reference)")


def _sets(r):
    q, b = np.nonzero(r["keep"])
    return np.concatenate([[0], np.cumsum(r["keep"].sum(1))]), q, b


@pytest.mark.parametrize("dims,n,seed,points,max_iters", [((32, 32, 32), 10_000, 1, "uniform", 10),
                                                         ((32, 32, 32), 4_000, 4, "training", 50),
                                                         ((64, 64, 16), 3_000, 11, "training", 50),
                                                         ((16, 16, 16), 3_000, 7, "uniform", 50)])
def test_oracle_equals_reference_sources(dims, n, seed, points, max_iters):
    sc = S.make_scene(dims, n, seed=seed, points=points)
    o = sc.search_options(max_iters)
    rr = oracle.ref_batch_search(sc.weights, sc.dims, sc.bbox, sc.bones, sc.points, workers=8, **o)
    for v in oracle.VARIANTS:
        r = oracle.batch_search(sc.weights, sc.dims, sc.bbox, sc.bones, sc.points, workers=8, variant=v, **o)
        offs, q, b = _sets(r)
        np.testing.assert_array_equal(offs, rr["offsets"])  # identical CorrespondenceSets
        np.testing.assert_array_equal(b, rr["bone"])
        np.testing.assert_array_equal(r["iters"][q, b], rr["iters"])
        # roots within the spread of float64 operation orders (identical at the oracle configuration)
        assert np.abs(r["x_c"][q, b] - rr["x"]).max() <= (1e-12 if max_iters == 10 else 1e-6)
        assert np.abs(r["resid"][q, b] - rr["resid"]).max() <= (1e-12 if max_iters == 10 else 1e-9)


def test_precompute_and_init_states_equal_reference_sources():
    sc = S.make_scene((32, 32, 32), 200, seed=3)
    tg = oracle.precompute_transform_grid(sc.weights, sc.dims, sc.bbox, sc.bones)
    rt = oracle.ref_precompute_transform_grid(sc.weights, sc.dims, sc.bbox, sc.bones)
    assert np.abs(tg - rt).max() <= 1e-15
    x0, j0 = oracle.init_states(sc.weights, sc.dims, sc.bbox, sc.bones, sc.points)
    rx0, rj0 = oracle.ref_init_states(sc.weights, sc.dims, sc.bbox, sc.bones, sc.points)
    np.testing.assert_array_equal(x0, rx0)
    assert np.abs(j0 - rj0).max() <= 1e-11 * max(1.0, np.abs(rj0).max())


def test_reference_sources_error_messages():
    sc = S.make_scene((16, 16, 16), 10, seed=3)
    o = sc.search_options(10)
    for bad, msg in [(dict(max_iters=0), "search: max_iters must be >= 1"),
                     (dict(div_eps=o["conv_eps"]), "search: div_eps must exceed conv_eps"),
                     (dict(dedup_dist=-1.0), "search: dedup_dist must be >= 0")]:
        with pytest.raises(oracle.OracleInvalidArgument, match=msg):
            oracle.ref_batch_search(sc.weights, sc.dims, sc.bbox, sc.bones, sc.points, **{**o, **bad})
        with pytest.raises(oracle.OracleInvalidArgument, match=msg):
            oracle.batch_search(sc.weights, sc.dims, sc.bbox, sc.bones, sc.points, **{**o, **bad})
