"""Pins the CPU oracle (oracle/fskin_oracle.cpp) to the reference's only executable
specification: the SPEC.md known-answer examples and acceptance criteria (the reference
ships no tests or golden vectors and cannot be built here — SURVEY §4, §8(c)).
Each test cites the SPEC line it transcribes."""
import numpy as np
import pytest

import oracle
from paper_2211_15601_b200 import synthetic as S

BBOX = np.array([0.0, 0.0, 0.0, 1.0, 2.0, 0.5])
DIMS = (5, 6, 4)
V = DIMS[0] * DIMS[1] * DIMS[2]


def rand_bones(rng, nb):
    out = []
    for _ in range(nb):
        T = S.about_axis(rng.normal(size=3), rng.normal(size=3), rng.uniform(-1, 1))
        T[:, 3] += rng.normal(size=3) * 0.1
        out.append(T.reshape(12))
    return np.stack(out)


def rand_weights(rng, nb, v=V):
    w = rng.random((v, nb)) + 0.05
    return w / w.sum(1, keepdims=True)


def identity_bones(nb):
    return np.tile(np.eye(3, 4).reshape(12), (nb, 1))


def translation(t):
    T = np.eye(3, 4)
    T[:, 3] = t
    return T.reshape(12)


def vertex(i, j, k, dims=DIMS, bbox=BBOX):
    h = (bbox[3:] - bbox[:3]) / (np.array(dims) - 1)
    return bbox[:3] + np.array([i, j, k]) * h


def vidx(i, j, k, dims=DIMS):
    return (k * dims[1] + j) * dims[0] + i


# ------------------------------------------------------------------ lbs_blend
def test_lbs_blend_one_hot_is_bone():
    rng = np.random.default_rng(0)
    B = rand_bones(rng, 4)
    w = np.array([0, 0, 1.0, 0])
    np.testing.assert_allclose(oracle.lbs_blend(w, B), B[2], atol=0, rtol=0)


def test_lbs_blend_identity_bones():
    w = np.array([0.2, 0.3, 0.5])
    np.testing.assert_allclose(oracle.lbs_blend(w, identity_bones(3)), np.eye(3, 4).reshape(12), atol=1e-15)


def test_lbs_blend_linearity_translation_example():
    B = np.stack([translation([1, 0, 0]), translation([0, 1, 0])])
    out = oracle.lbs_blend([0.5, 0.5], B).reshape(3, 4)
    np.testing.assert_allclose(out[:, 3], [0.5, 0.5, 0.0])
    np.testing.assert_allclose(out[:, :3], np.eye(3))


def test_lbs_blend_mismatch_raises_reference_message():
    with pytest.raises(oracle.OracleInvalidArgument, match="lbs_blend: weight/bone count mismatch"):
        oracle.lbs_blend([1.0, 0.0], identity_bones(3))


# ------------------------------------------------------------------ precompute
def test_precompute_identity_bones_gives_identity_grid():
    rng = np.random.default_rng(1)
    tg = oracle.precompute_transform_grid(rand_weights(rng, 3), DIMS, BBOX, identity_bones(3))
    np.testing.assert_allclose(tg, np.tile(np.eye(3, 4).reshape(12), (V, 1)), atol=1e-15)


def test_precompute_one_hot_grid_holds_bone_verbatim():
    rng = np.random.default_rng(2)
    B = rand_bones(rng, 3)
    lab = rng.integers(0, 3, V)
    w = np.eye(3)[lab]
    tg = oracle.precompute_transform_grid(w, DIMS, BBOX, B)
    np.testing.assert_array_equal(tg, B[lab])


def test_precompute_vertex_recompute_oracle_and_workers():
    rng = np.random.default_rng(3)
    w, B = rand_weights(rng, 5), rand_bones(rng, 5)
    tg1 = oracle.precompute_transform_grid(w, DIMS, BBOX, B, workers=1)
    tg4 = oracle.precompute_transform_grid(w, DIMS, BBOX, B, workers=4)
    np.testing.assert_array_equal(tg1, tg4)  # SPEC.md:573 determinism
    for (i, j, k) in [(0, 0, 0), (2, 3, 1), (4, 5, 3)]:
        x = vertex(i, j, k)
        ev = oracle.eval_points(w, DIMS, BBOX, B, tg1, x[None])
        np.testing.assert_allclose(ev["t12"][0], oracle.lbs_blend(w[vidx(i, j, k)], B), atol=1e-12)


def test_precompute_bone_count_mismatch():
    rng = np.random.default_rng(4)
    with pytest.raises(oracle.OracleInvalidArgument, match="precompute_transform_grid: bone count mismatch"):
        oracle.precompute_transform_grid(rand_weights(rng, 3), DIMS, BBOX, identity_bones(2))


# ------------------------------------------------------------------ trilerp
def test_trilerp_weights_vertex_center_edge():
    rng = np.random.default_rng(5)
    w, B = rand_weights(rng, 4), identity_bones(4)
    pts = np.stack([vertex(1, 2, 1), vertex(1.5, 2.5, 1.5), vertex(1.5, 2, 1)])
    ev = oracle.eval_points(w, DIMS, BBOX, B, None, pts)
    np.testing.assert_allclose(ev["weights"][0], w[vidx(1, 2, 1)], atol=1e-14)
    corners = [w[vidx(1 + a, 2 + b, 1 + c)] for a in (0, 1) for b in (0, 1) for c in (0, 1)]
    np.testing.assert_allclose(ev["weights"][1], np.mean(corners, 0), atol=1e-14)
    np.testing.assert_allclose(ev["weights"][2], 0.5 * (w[vidx(1, 2, 1)] + w[vidx(2, 2, 1)]), atol=1e-14)


def test_trilerp_weights_convex_and_clamped():
    rng = np.random.default_rng(6)
    w = rand_weights(rng, 4)
    x = rng.uniform(-1, 3, (200, 3))
    ev = oracle.eval_points(w, DIMS, BBOX, identity_bones(4), None, x)
    np.testing.assert_allclose(ev["weights"].sum(1), 1.0, atol=1e-12)
    assert (ev["weights"] >= w.min(0) - 1e-12).all() and (ev["weights"] <= w.max(0) + 1e-12).all()
    xc = np.clip(x, BBOX[:3], BBOX[3:])  # out-of-box queries clamp to the bbox
    ev2 = oracle.eval_points(w, DIMS, BBOX, identity_bones(4), None, xc)
    np.testing.assert_array_equal(ev["weights"], ev2["weights"])


def test_trilerp_transform_vertex_and_uniform():
    rng = np.random.default_rng(7)
    w, B = rand_weights(rng, 3), rand_bones(rng, 3)
    tg = oracle.precompute_transform_grid(w, DIMS, BBOX, B)
    ev = oracle.eval_points(w, DIMS, BBOX, B, tg, vertex(3, 1, 2)[None])
    np.testing.assert_allclose(ev["t12"][0], tg[vidx(3, 1, 2)], atol=1e-14)
    uni = np.tile(B[1], (V, 1))
    ev = oracle.eval_points(w, DIMS, BBOX, B, uni, rng.uniform(0, 1, (20, 3)))
    np.testing.assert_allclose(ev["t12"], np.tile(B[1], (20, 1)), atol=1e-14)


# ------------------------------------------------------------------ weight gradient
def test_weight_gradient_constant_and_linear():
    w = np.full((V, 2), 0.5)
    ev = oracle.eval_points(w, DIMS, BBOX, identity_bones(2), None, np.array([[0.3, 0.7, 0.2]]))
    np.testing.assert_allclose(ev["wgrad"], 0.0, atol=1e-14)
    x = S.vertex_positions(DIMS, BBOX[:3], BBOX[3:])
    w0 = (x[:, 0] - BBOX[0]) / (BBOX[3] - BBOX[0])
    w = np.stack([w0, 1 - w0], 1)
    ev = oracle.eval_points(w, DIMS, BBOX, identity_bones(2), None, np.array([[0.33, 0.71, 0.21]]))
    np.testing.assert_allclose(ev["wgrad"][0, 0], [1.0, 0, 0], atol=1e-12)
    np.testing.assert_allclose(ev["wgrad"][0, 1], [-1.0, 0, 0], atol=1e-12)


def test_weight_gradient_matches_central_fd():
    rng = np.random.default_rng(8)
    w = rand_weights(rng, 3)
    h = (BBOX[3:] - BBOX[:3]) / (np.array(DIMS) - 1)
    x = BBOX[:3] + rng.uniform(0.05, 0.95, (50, 3)) * (BBOX[3:] - BBOX[:3])
    g = oracle.eval_points(w, DIMS, BBOX, identity_bones(3), None, x)["wgrad"]
    for a in range(3):
        e = np.zeros(3)
        e[a] = 1e-4 * h[a]
        wp = oracle.eval_points(w, DIMS, BBOX, identity_bones(3), None, x + e)["weights"]
        wm = oracle.eval_points(w, DIMS, BBOX, identity_bones(3), None, x - e)["weights"]
        fd = (wp - wm) / (2 * e[a])
        np.testing.assert_allclose(g[:, :, a], fd, rtol=1e-4, atol=1e-6)


def test_weight_gradient_face_tiebreak_uses_lower_cell():
    # skinning.cpp:122-139: a point exactly on an interior face uses the lower-index cell.
    x = S.vertex_positions(DIMS, BBOX[:3], BBOX[3:])
    w0 = np.where(x[:, 0] <= vertex(2, 0, 0)[0] + 1e-12, 0.0, (x[:, 0] - vertex(2, 0, 0)[0]) * 4)
    w = np.stack([w0, 1 - w0], 1)
    face = vertex(2, 1.3, 1.4)
    g = oracle.eval_points(w, DIMS, BBOX, identity_bones(2), None, face[None])["wgrad"]
    np.testing.assert_allclose(g[0, 0, 0], 0.0, atol=1e-12)  # lower cell is flat


# ------------------------------------------------------------------ lossless precompute
def test_lossless_precomputation_1e10():
    sc = S.make_scene((16, 16, 16), 0, seed=3)
    rng = np.random.default_rng(9)
    lo, hi = sc.bbox[:3].astype(float), sc.bbox[3:].astype(float)
    x = lo + rng.random((10_000, 3)) * (hi - lo)
    ev = oracle.eval_points(sc.weights, sc.dims, sc.bbox, sc.bones, None, x)
    np.testing.assert_allclose(ev["d_tgrid"], ev["d_grid"], atol=1e-10, rtol=0)


# ------------------------------------------------------------------ init_states
def test_init_states_identity_bones():
    rng = np.random.default_rng(10)
    x = rng.uniform(0, 0.5, (10, 3))
    x0, j0 = oracle.init_states(rand_weights(rng, 3), DIMS, BBOX, identity_bones(3), x)
    np.testing.assert_allclose(x0, np.repeat(x[:, None], 3, 1), atol=1e-15)
    np.testing.assert_allclose(j0, np.broadcast_to(np.eye(3), j0.shape), atol=1e-12)


def test_init_states_two_bone_translation():
    B = np.stack([translation([1, 0, 0]), identity_bones(1)[0]])
    w = np.full((V, 2), 0.5)
    x0, _ = oracle.init_states(w, DIMS, BBOX, B, np.array([[1.5, 0.0, 0.0]]))
    np.testing.assert_allclose(x0[0], [[0.5, 0, 0], [1.5, 0, 0]], atol=1e-15)


def test_init_states_one_hot_region_is_rotation_transpose():
    rng = np.random.default_rng(11)
    B = rand_bones(rng, 2)
    w = np.tile([1.0, 0.0], (V, 1))  # bone 0 everywhere: locally rigid
    xp = S.apply(B[0].reshape(3, 4), np.array([0.4, 0.9, 0.2]))
    _, j0 = oracle.init_states(w, DIMS, BBOX, B, xp[None])
    np.testing.assert_allclose(j0[0, 0], B[0].reshape(3, 4)[:, :3].T, atol=1e-12)


# ------------------------------------------------------------------ broyden_search
def _search(sc_w, dims, bbox, B, x, max_iters=50, workers=1, **kw):
    diag = float(np.linalg.norm(np.asarray(bbox[3:], float) - np.asarray(bbox[:3], float)))
    o = dict(conv_eps=1e-5 * diag, div_eps=0.5 * diag, dedup_dist=1e-2 * diag)
    o.update(kw)
    return oracle.batch_search(sc_w, dims, bbox, B, x, max_iters, workers=workers, **o)


def test_identity_pose_single_root_equals_query():
    sc = S.make_scene((8, 8, 8), 1000, seed=5, pose="rest")
    lo, hi = sc.bbox[:3].astype(float), sc.bbox[3:].astype(float)
    x = lo + np.random.default_rng(0).random((1000, 3)) * (hi - lo)
    r = _search(sc.weights, sc.dims, sc.bbox, sc.bones, x)
    assert (r["keep"].sum(1) == 1).all()
    kept = r["x_c"][r["keep"] == 1]
    np.testing.assert_allclose(kept, x, atol=1e-5 * sc.diag)
    assert r["iters"][r["keep"] == 1].max() <= 1


def test_single_rigid_bone_exact_inverse():
    rng = np.random.default_rng(12)
    B = rand_bones(rng, 1)
    w = np.ones((V, 1))
    y = BBOX[:3] + rng.random((100, 3)) * (BBOX[3:] - BBOX[:3])
    xp = S.apply(B[0].reshape(3, 4), y)
    r = _search(w, DIMS, BBOX, B, xp)
    assert r["keep"].all()
    np.testing.assert_allclose(r["x_c"][:, 0], y, atol=1e-5 * np.linalg.norm(BBOX[3:] - BBOX[:3]))


def test_empty_query_list():
    sc = S.make_scene((8, 8, 8), 10, seed=5)
    r = _search(sc.weights, sc.dims, sc.bbox, sc.bones, np.zeros((0, 3)))
    assert r["x_c"].shape == (0, sc.n_bones, 3)


def test_soundness_and_worker_determinism():
    # SPEC.md:566 (criterion 1) and :573 (criterion 8)
    sc = S.make_scene((32, 32, 32), 1500, seed=7)
    opts = sc.search_options(50)
    r1 = oracle.batch_search(sc.weights, sc.dims, sc.bbox, sc.bones, sc.points, workers=1, **opts)
    r4 = oracle.batch_search(sc.weights, sc.dims, sc.bbox, sc.bones, sc.points, workers=4, **opts)
    for k in r1:
        np.testing.assert_array_equal(r1[k], r4[k])
    tg = oracle.precompute_transform_grid(sc.weights, sc.dims, sc.bbox, sc.bones)
    keep = r1["keep"] == 1
    roots = r1["x_c"][keep]
    queries = np.repeat(sc.points.astype(float)[:, None], sc.n_bones, 1)[keep]
    d = oracle.eval_points(sc.weights, sc.dims, sc.bbox, sc.bones, tg, roots)["d_tgrid"]
    assert (np.linalg.norm(d - queries, axis=1) < opts["conv_eps"]).all()
    assert (r1["keep"] <= r1["converged"]).all()


def test_search_option_validation_messages():
    sc = S.make_scene((8, 8, 8), 4, seed=5)
    args = (sc.weights, sc.dims, sc.bbox, sc.bones, sc.points)
    with pytest.raises(ValueError, match="search: max_iters must be >= 1"):
        oracle.batch_search(*args, 0, 1e-5, 0.5, 0.01)
    with pytest.raises(ValueError, match="search: conv_eps must be > 0"):
        oracle.batch_search(*args, 5, 0.0, 0.5, 0.01)
    with pytest.raises(ValueError, match="search: div_eps must exceed conv_eps"):
        oracle.batch_search(*args, 5, 1e-3, 1e-3, 0.01)
    with pytest.raises(ValueError, match="search: dedup_dist must be >= 0"):
        oracle.batch_search(*args, 5, 1e-5, 0.5, -1.0)


# ------------------------------------------------------------------ dedup
def test_dedup_examples():
    d = 0.1
    assert oracle.dedup_roots([[0, 0, 0], [0, 0, 0]], d).tolist() == [1, 0]
    assert oracle.dedup_roots([[0, 0, 0], [0.2, 0, 0]], d).tolist() == [1, 1]
    rng = np.random.default_rng(13)
    cluster = rng.normal(size=(5, 3))
    cluster = 0.5 * d / 2 * cluster / np.linalg.norm(cluster, axis=1, keepdims=True)
    pts = np.vstack([cluster, [[5.0, 5.0, 5.0]]])
    assert oracle.dedup_roots(pts, d).sum() == 2
    # strict '<': a root exactly dedup_dist away survives (correspondence.cpp:168)
    assert oracle.dedup_roots([[0, 0, 0], [0.5, 0, 0]], 0.5).tolist() == [1, 1]


# ------------------------------------------------------------------ implicit gradients
def test_implicit_grad_rest_pose_is_zero():
    # rest pose → d(x)=x for any normalized w, so dL/dw = 0 (grad_w columns equal:
    # a uniform shift of w_{c,·} is invisible because Σ_i w_i = 1 is maintained by the softmax
    # head in the reference; on the grid, all bones contribute the same u·x̃).
    sc = S.make_scene((8, 8, 8), 50, seed=5, pose="rest")
    r = _search(sc.weights, sc.dims, sc.bbox, sc.bones, sc.points)
    sel = np.argmax(r["keep"], 1)
    n = sc.points.shape[0]
    v = np.random.default_rng(1).normal(size=(n, 3))
    gT, gw = oracle.grid_vjp(sc.dims, sc.bbox, sc.bones, r["x_c"][np.arange(n), sel], r["jinv"][np.arange(n), sel], v)
    # every bone's weight-gradient is identical (B_i = I), so the softmax VJP of the reference is 0
    np.testing.assert_allclose(gw - gw.mean(1, keepdims=True), 0.0, atol=1e-12)


def _fd_setup():
    sc = S.make_scene((8, 8, 8), 60, seed=11)
    tg = oracle.precompute_transform_grid(sc.weights, sc.dims, sc.bbox, sc.bones)
    tight = dict(conv_eps=1e-12 * sc.diag, div_eps=0.5 * sc.diag, dedup_dist=1e-2 * sc.diag)
    r = oracle.batch_search(sc.weights, sc.dims, sc.bbox, sc.bones, sc.points, 100, tgrid=tg, **tight)
    return sc, tg, tight, r


def test_grid_vjp_exact_matches_finite_differences():
    # implicit gradient vs central FD (h = 1e-4) rel < 1e-3.
    sc, tg, tight, r = _fd_setup()
    rng = np.random.default_rng(2)
    # roots strictly inside the bbox: outside it the clamped lookup makes d(x) affine in the
    # clamped axis while weight_spatial_gradient still reports the in-box stencil
    lo, hi = sc.bbox[:3].astype(float), sc.bbox[3:].astype(float)
    inside = ((r["x_c"] > lo + 1e-3) & (r["x_c"] < hi - 1e-3)).all(-1)
    ok_pts = np.where((r["keep"].sum(1) == 1) & (inside & (r["keep"] == 1)).any(1))[0][:20]
    assert len(ok_pts) >= 10
    checked = 0
    for p in ok_pts:
        i = int(np.argmax(r["keep"][p]))
        xs = r["x_c"][p, i]
        v = rng.normal(size=3)
        u, ok = oracle.implicit_u_exact(sc.weights, sc.dims, sc.bbox, sc.bones, xs[None], v[None])
        if not ok[0]:
            continue
        # grad_T from the exact u: φ_c u x̃ᵀ (u already carries the minus sign)
        J_exact_inv_T = np.eye(3)  # dummy jinv so that grid_vjp's −J̃ᵀv equals u
        gT, _ = oracle.grid_vjp(sc.dims, sc.bbox, sc.bones, xs[None], J_exact_inv_T[None], -u[None])
        c = int(np.argmax(np.abs(gT).sum(1)))
        e = int(np.argmax(np.abs(gT[c])))
        h = 1e-4
        vals = []
        for s in (+1, -1):
            tp = tg.copy()
            tp[c, e] += s * h
            rr = oracle.batch_search(sc.weights, sc.dims, sc.bbox, sc.bones, sc.points[p:p + 1], 100, tgrid=tp, **tight)
            vals.append(rr["x_c"][0, i] @ v)
        fd = (vals[0] - vals[1]) / (2 * h)
        assert abs(fd - gT[c, e]) <= 1e-3 * abs(gT[c, e]) + 1e-9, (fd, gT[c, e])
        checked += 1
    assert checked >= 10


def test_implicit_grad_approx_cosine_and_one_hot_exact():
    sc, tg, tight, r = _fd_setup()
    keep = np.argwhere(r["keep"] == 1)
    xs = r["x_c"][keep[:, 0], keep[:, 1]]
    J = r["jinv"][keep[:, 0], keep[:, 1]]
    v = np.random.default_rng(3).normal(size=(len(xs), 3))
    u_ex, ok = oracle.implicit_u_exact(sc.weights, sc.dims, sc.bbox, sc.bones, xs, v)
    u_ap = -np.einsum("nij,ni->nj", J, v)
    cos = (u_ex * u_ap).sum(1) / (np.linalg.norm(u_ex, axis=1) * np.linalg.norm(u_ap, axis=1))
    assert cos[ok == 1].mean() > 0.9
    # locally rigid (one-hot) region → J̃ = Rᵀ exactly, approx == exact
    rng = np.random.default_rng(4)
    B = rand_bones(rng, 1)
    w = np.ones((V, 1))
    y = BBOX[:3] + rng.random((20, 3)) * (BBOX[3:] - BBOX[:3])
    rr = _search(w, DIMS, BBOX, B, S.apply(B[0].reshape(3, 4), y))
    vv = rng.normal(size=(20, 3))
    ue, _ = oracle.implicit_u_exact(w, DIMS, BBOX, B, rr["x_c"][:, 0], vv)
    ua = -np.einsum("nij,ni->nj", rr["jinv"][:, 0], vv)
    np.testing.assert_allclose(ua, ue, atol=1e-10)


# ---------------------------------------------------------------- MLP stages
def _np_mlp(theta, widths, X):
    """numpy f64 Mlp::forward (mlp.cpp:115-138) on Mlp::parameters() order (mlp.cpp:207-219)."""
    off, h = 0, np.asarray(X, np.float64)
    for l in range(len(widths) - 1):
        n_in, n_out = widths[l], widths[l + 1]
        W = theta[off:off + n_in * n_out].reshape(n_in, n_out).T  # column-major storage
        off += n_in * n_out
        b = theta[off:off + n_out]
        off += n_out
        z = h @ W.T + b
        h = (np.maximum(z, 0) + np.log1p(np.exp(-np.abs(z)))) if l + 2 < len(widths) else z
    return h


def test_oracle_mlp_forward_and_distill_match_numpy():
    widths = [3, 64, 64, 64, 24]
    th = oracle.mlp_init(widths, 4, 0.05)
    X = np.random.default_rng(0).uniform(-1, 1, (50, 3))
    assert np.allclose(oracle.mlp_forward(th, widths, X), _np_mlp(th, widths, X), rtol=0, atol=1e-12)
    bbox = np.array([-1.0, -0.5, -0.25, 1.0, 2.0, 0.25])
    dims = (5, 4, 3)
    W = oracle.distill(th, widths, dims, bbox)
    g = np.stack(np.meshgrid(*[np.linspace(bbox[a], bbox[3 + a], dims[a]) for a in range(3)], indexing="ij"), -1)
    V = g.transpose(2, 1, 0, 3).reshape(-1, 3)  # x fastest (skinning.cpp:72-80 vertex order)
    z = _np_mlp(th, widths, V)
    e = np.exp(z - z.max(1, keepdims=True))
    assert np.allclose(W, e / e.sum(1, keepdims=True), rtol=0, atol=1e-12)


def test_oracle_distill_vjp_matches_finite_differences():
    widths = [3, 8, 8, 5]
    th = oracle.mlp_init(widths, 2)
    dims, bbox = (3, 3, 2), np.array([0.0, 0.0, 0.0, 1.0, 1.0, 1.0])
    dw = np.random.default_rng(1).normal(size=(18, 5))
    g = oracle.distill_vjp(th, widths, dims, bbox, dw)
    rng = np.random.default_rng(3)
    for i in rng.choice(len(th), 12, replace=False):
        e = np.zeros_like(th)
        e[i] = 1e-6
        fd = ((oracle.distill(th + e, widths, dims, bbox) - oracle.distill(th - e, widths, dims, bbox)) * dw).sum() / 2e-6
        assert abs(fd - g[i]) <= 1e-6 * max(1.0, abs(fd))


def test_oracle_posed_occupancy_semantics():
    """max over each set's roots, first root wins ties, empty set -> (0, -1) (shape.cpp:242-269)."""
    widths = [3, 16, 16, 1]
    th = oracle.mlp_init(widths, 7)
    x = np.random.default_rng(5).uniform(-1, 1, (6, 3))
    x[4] = x[3]  # a tie inside set 2
    offs = np.array([0, 2, 2, 5, 6])
    pred, am = oracle.posed_occupancy(th, widths, None, offs, x)
    occ = 1 / (1 + np.exp(-_np_mlp(th, widths, x)[:, 0]))
    assert am[1] == -1 and pred[1] == 0.0
    for q, (a, b) in enumerate(zip(offs[:-1], offs[1:])):
        if b > a:
            assert pred[q] == pytest.approx(occ[a:b].max(), abs=1e-14)
            assert am[q] == int(np.argmax(occ[a:b]))  # numpy argmax = first maximum
    with pytest.raises(oracle.OracleInvalidArgument, match="pose vector length 1, field conditioned on 0"):
        oracle.posed_occupancy(th, widths, np.zeros(1), offs, x)


def test_oracle_mlp_weight_jacobian_matches_finite_differences():
    widths = [3, 64, 64, 64, 24]
    th = oracle.mlp_init(widths, 6, 0.5)
    x = np.random.default_rng(2).uniform(-1, 1, (20, 3))
    w, dw = oracle.mlp_weights_jacobian(th, widths, x)
    sm = lambda z: np.exp(z - z.max(1, keepdims=True)) / np.exp(z - z.max(1, keepdims=True)).sum(1, keepdims=True)  # noqa: E731
    assert np.allclose(w, sm(oracle.mlp_forward(th, widths, x)), atol=1e-14)
    for c in range(3):
        e = np.zeros(3)
        e[c] = 1e-6
        fd = (sm(oracle.mlp_forward(th, widths, x + e)) - sm(oracle.mlp_forward(th, widths, x - e))) / 2e-6
        assert np.abs(fd - dw[:, :, c]).max() <= 1e-7


def test_oracle_mlp_variant_known_answers():
    """SPEC.md:273-274 for the MLP variant: identity pose -> one root = the query; a single
    rigid bone -> the exact inverse (w = 1 whatever the network)."""
    widths = [3, 16, 16, 3]
    th = oracle.mlp_init(widths, 1)
    rng = np.random.default_rng(3)
    x = rng.uniform(-1, 1, (50, 3))
    ident = np.tile(np.array([1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0.0]), (3, 1))
    r = oracle.batch_search_mlp(th, widths, ident, x, 50, 1e-5, 1.0, 1e-2)
    assert (r["keep"].sum(1) == 1).all() and r["converged"].all()
    np.testing.assert_allclose(r["x_c"][:, 0], x, atol=1e-12)
    T = S.about_axis(np.array([0.1, 0.2, 0.3]), np.array([0.3, 1.0, 0.2]), 0.7)
    r = oracle.batch_search_mlp(oracle.mlp_init([3, 8, 8, 1], 2), [3, 8, 8, 1], T.reshape(1, 12), S.apply(T, x),
                                50, 1e-9, 10.0, 1e-2)
    np.testing.assert_allclose(r["x_c"][:, 0], x, atol=1e-9)


def test_oracle_operation_order_variants_agree_at_c1():
    """The four plausible operation orders of the reference (oracle/Makefile) give the same masks
    and roots to ~1e-14 on the oracle configuration (C1 shape, max_iters 10); at max_iters 50 they
    differ by a few mask flips per 4.8M solves (profiles/r02_oracle_variants.log)."""
    from paper_2211_15601_b200 import synthetic as S
    sc = S.make_scene((32, 32, 32), 2000, seed=1)
    res = [oracle.batch_search(sc.weights, sc.dims, sc.bbox, sc.bones, sc.points, workers=4, variant=v,
                               **sc.search_options(10)) for v in oracle.VARIANTS]
    for r in res[1:]:
        np.testing.assert_array_equal(r["converged"], res[0]["converged"])
        np.testing.assert_array_equal(r["keep"], res[0]["keep"])
        conv = r["converged"] == 1  # (unconverged iterates of diverging solves may go anywhere)
        np.testing.assert_allclose(r["x_c"][conv], res[0]["x_c"][conv], rtol=0, atol=1e-12)
