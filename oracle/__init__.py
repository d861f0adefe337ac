"""ctypes wrapper of the CPU oracle (``oracle/liboracle.so``).

TEST INFRASTRUCTURE ONLY: imported by ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s CPU-baseline / ``--impl reference`` leg — never by the product package.
See ``fskin_oracle.cpp`` for the reference lines each function restates and for the
parity status ("parity unpinned" against reference outputs: the reference cannot be
built here; pinned by SPEC.md known answers).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "liboracle.so")
# operation-order variants of the same restatement (oracle/Makefile): the reference's
# Eigen version and build flags are not pinned, so its exact float64 operation order is not either
VARIANTS = ("fma", "unfused", "invrow0", "pairsum", "gccfma")
_libs = {}
_variant = None  # module-wide default for every call below (None = "fma", the default build); see use_variant()

_d = ctypes.POINTER(ctypes.c_double)
_u8 = ctypes.POINTER(ctypes.c_uint8)
_i32 = ctypes.POINTER(ctypes.c_int32)
_i64 = ctypes.c_int64
_int = ctypes.c_int


def _path(variant):
    return _LIB if variant in (None, "fma") else os.path.join(_HERE, f"liboracle_{variant}.so")


def build(force: bool = False) -> str:
    srcs = [os.path.join(_HERE, f) for f in ("fskin_oracle.cpp", "precision_emul.cpp", "mlp_oracle.cpp", "Makefile")]
    newest = max(os.path.getmtime(s) for s in srcs)
    if force or any(not os.path.exists(_path(v)) or os.path.getmtime(_path(v)) < newest for v in VARIANTS):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB


def use_variant(variant):
    """Route every oracle call of this process to an operation-order variant (None = default)."""
    global _variant
    if variant not in (None,) + VARIANTS:
        raise ValueError(variant)
    _variant = None if variant == "fma" else variant


def lib(variant=None):
    variant = variant if variant is not None else _variant
    key = variant or "fma"
    if key not in _libs:
        build()
        L = ctypes.CDLL(_path(variant))
        L.orc_variant.restype = ctypes.c_char_p
        L.orc_last_error.restype = ctypes.c_char_p
        L.orc_precompute_tgrid.argtypes = [_d, _int, _int, _int, _int, _d, _d, _int, _d, _int]
        L.orc_lbs_blend.argtypes = [_d, _d, _int, _int, _d]
        L.orc_eval_points.argtypes = [_d, _int, _int, _int, _int, _d, _d, _d, _d, _i64, _d, _d, _d, _d, _d, _d]
        L.orc_init_states.argtypes = [_d, _int, _int, _int, _int, _d, _d, _int, _d, _i64, _d, _d]
        L.orc_batch_search.argtypes = [_d, _int, _int, _int, _int, _d, _d, _d, _int, _d, _i64, _int,
                                       ctypes.c_double, ctypes.c_double, ctypes.c_double, _int,
                                       _d, _d, _d, _i32, _u8, _u8]
        L.orc_dedup_roots.argtypes = [_d, _int, ctypes.c_double, _u8]
        L.orc_grid_vjp.argtypes = [_int, _int, _int, _int, _d, _d, _d, _d, _d, _i32, _i64, _d, _d]
        L.orc_implicit_u_exact.argtypes = [_d, _int, _int, _int, _int, _d, _d, _d, _d, _i64, _d, _u8]
        L.orc_mlp_last_error.restype = ctypes.c_char_p
        _pi = ctypes.POINTER(ctypes.c_int)
        _pi64 = ctypes.POINTER(ctypes.c_int64)
        L.orc_mlp_forward.argtypes = [_d, _pi, _int, _d, _i64, _d, _int]
        L.orc_distill.argtypes = [_d, _pi, _int, _int, _int, _int, _d, _d, _int]
        L.orc_distill_vjp.argtypes = [_d, _pi, _int, _int, _int, _int, _d, _d, _d, _int]
        L.orc_posed_occupancy.argtypes = [_d, _pi, _int, _d, _int, _pi64, _d, _i64, _d, _i32, _int]
        L.orc_mlp_weights_jacobian.argtypes = [_d, _pi, _int, _d, _i64, _d, _d, _int]
        L.orc_batch_search_mlp.argtypes = [_d, _pi, _int, _d, _int, _d, _i64, _int, ctypes.c_double,
                                           ctypes.c_double, ctypes.c_double, _int, _d, _d, _d, _i32, _u8, _u8]
        _libs[key] = L
    return _libs[key]


class OracleError(Exception):
    pass


class OracleInvalidArgument(OracleError, ValueError):
    pass


def _check(rc):
    if rc != 0:
        msg = lib().orc_last_error().decode()  # errors are raised by the validation shared by all variants
        raise (OracleInvalidArgument if rc == 1 else OracleError)(msg)


def _p(a, t=_d):
    return None if a is None else a.ctypes.data_as(t)


def _f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def precompute_transform_grid(weights, dims, bbox, bones, workers=1, variant=None):
    """deformer.cpp:61-77 → tgrid [V,12] float64."""
    w, bb, B = _f64(weights), _f64(bbox), _f64(bones).reshape(-1, 12)
    nx, ny, nz = dims
    nb = w.shape[1] if w.ndim == 2 else B.shape[0]
    out = np.zeros((nx * ny * nz, 12))
    _check(lib(variant).orc_precompute_tgrid(_p(w), nx, ny, nz, nb, _p(bb), _p(B), B.shape[0], _p(out), workers))
    return out


def lbs_blend(weights, bones):
    w, B = _f64(weights), _f64(bones).reshape(-1, 12)
    out = np.zeros(12)
    _check(lib().orc_lbs_blend(_p(w), _p(B), B.shape[0], w.shape[0], _p(out)))
    return out


def eval_points(weights, dims, bbox, bones, tgrid, x):
    """Batched trilerp_weights, weight_spatial_gradient, trilerp_transform,
    forward_deform (tgrid and weight-grid forms) and deform_jacobian at points x."""
    w, bb, B, x = _f64(weights), _f64(bbox), _f64(bones).reshape(-1, 12), _f64(x).reshape(-1, 3)
    tg = _f64(tgrid) if tgrid is not None else precompute_transform_grid(w, dims, bb, B)
    n, nb = x.shape[0], B.shape[0]
    out = dict(weights=np.zeros((n, nb)), wgrad=np.zeros((n, nb, 3)), t12=np.zeros((n, 12)),
               d_tgrid=np.zeros((n, 3)), d_grid=np.zeros((n, 3)), jac=np.zeros((n, 3, 3)))
    _check(lib().orc_eval_points(_p(w), *dims, nb, _p(bb), _p(B), _p(tg), _p(x), n,
                                 *[_p(out[k]) for k in ("weights", "wgrad", "t12", "d_tgrid", "d_grid", "jac")]))
    return out


def init_states(weights, dims, bbox, bones, x_prime, variant=None):
    w, bb, B, x = _f64(weights), _f64(bbox), _f64(bones).reshape(-1, 12), _f64(x_prime).reshape(-1, 3)
    n, nb = x.shape[0], B.shape[0]
    x0, j0 = np.zeros((n, nb, 3)), np.zeros((n, nb, 3, 3))
    _check(lib(variant).orc_init_states(_p(w), *dims, w.shape[1], _p(bb), _p(B), nb, _p(x), n, _p(x0), _p(j0)))
    return x0, j0


def batch_search(weights, dims, bbox, bones, x_prime, max_iters, conv_eps, div_eps, dedup_dist,
                 workers=1, tgrid=None, variant=None):
    """correspondence.cpp:178-192 with per-(point, init) dense outputs."""
    w, bb, B, x = _f64(weights), _f64(bbox), _f64(bones).reshape(-1, 12), _f64(x_prime).reshape(-1, 3)
    tg = _f64(tgrid) if tgrid is not None else precompute_transform_grid(w, dims, bb, B, workers, variant)
    n, nb = x.shape[0], B.shape[0]
    out = dict(x_c=np.zeros((n, nb, 3)), jinv=np.zeros((n, nb, 3, 3)), resid=np.zeros((n, nb)),
               iters=np.zeros((n, nb), np.int32), converged=np.zeros((n, nb), np.uint8),
               keep=np.zeros((n, nb), np.uint8))
    _check(lib(variant).orc_batch_search(_p(w), *dims, w.shape[1], _p(bb), _p(tg), _p(B), nb, _p(x), n,
                                  int(max_iters), conv_eps, div_eps, dedup_dist, workers,
                                  _p(out["x_c"]), _p(out["jinv"]), _p(out["resid"]), _p(out["iters"], _i32),
                                  _p(out["converged"], _u8), _p(out["keep"], _u8)))
    return out


def dedup_roots(xs, dedup_dist):
    xs = _f64(xs).reshape(-1, 3)
    keep = np.zeros(xs.shape[0], np.uint8)
    _check(lib().orc_dedup_roots(_p(xs), xs.shape[0], dedup_dist, _p(keep, _u8)))
    return keep


def grid_vjp(dims, bbox, bones, x_star, jinv, v, sel=None, n_bones=None):
    bb, B = _f64(bbox), _f64(bones).reshape(-1, 12)
    xs, J, v = _f64(x_star).reshape(-1, 3), _f64(jinv).reshape(-1, 9), _f64(v).reshape(-1, 3)
    n, nb = xs.shape[0], B.shape[0]
    V = dims[0] * dims[1] * dims[2]
    gT, gw = np.zeros((V, 12)), np.zeros((V, nb))
    s = None if sel is None else np.ascontiguousarray(sel, dtype=np.int32)
    _check(lib().orc_grid_vjp(*dims, nb, _p(bb), _p(B), _p(xs), _p(J), _p(v), _p(s, _i32), n, _p(gT), _p(gw)))
    return gT, gw


def implicit_u_exact(weights, dims, bbox, bones, x_star, v):
    w, bb, B = _f64(weights), _f64(bbox), _f64(bones).reshape(-1, 12)
    xs, v = _f64(x_star).reshape(-1, 3), _f64(v).reshape(-1, 3)
    n = xs.shape[0]
    u, ok = np.zeros((n, 3)), np.zeros(n, np.uint8)
    _check(lib().orc_implicit_u_exact(_p(w), *dims, w.shape[1], _p(bb), _p(B), _p(xs), _p(v), n, _p(u), _p(ok, _u8)))
    return u, ok


# ---------------------------------------------------------------- MLP stages
def _mlp_check(rc):
    if rc != 0:
        msg = lib().orc_mlp_last_error().decode()
        raise (OracleInvalidArgument if rc == 1 else OracleError)(msg)


def _widths(widths):
    return (ctypes.c_int * len(widths))(*widths)


def mlp_param_count(widths):
    return sum(widths[l + 1] * widths[l] + widths[l + 1] for l in range(len(widths) - 1))


def mlp_init(widths, seed=0, head_scale=1.0):
    """Seeded fan-in-scaled normal init (mlp.cpp:97-110 recipe; numpy stream, not mt19937),
    flattened in Mlp::parameters() order: per layer W column-major, then b (mlp.cpp:207-219).
    Biases get a small random value so the bias path is exercised."""
    rng = np.random.default_rng(seed)
    out = []
    for l in range(len(widths) - 1):
        W = rng.normal(0.0, np.sqrt(2.0 / widths[l]), (widths[l + 1], widths[l]))
        b = rng.normal(0.0, 0.05, widths[l + 1])
        if l == len(widths) - 2:
            W, b = W * head_scale, b * head_scale
        out += [W.reshape(-1, order="F"), b]
    return np.concatenate(out)


def mlp_forward(theta, widths, X, workers=8):
    X = _f64(X).reshape(-1, widths[0])
    out = np.zeros((X.shape[0], widths[-1]))
    _mlp_check(lib().orc_mlp_forward(_p(_f64(theta)), _widths(widths), len(widths), _p(X), X.shape[0], _p(out), workers))
    return out


def distill(theta, widths, dims, bbox, workers=8):
    """distill (skinning.cpp:195-221) -> weights [V, nb] float64."""
    nx, ny, nz = dims
    out = np.zeros((nx * ny * nz, widths[-1]))
    _mlp_check(lib().orc_distill(_p(_f64(theta)), _widths(widths), len(widths), nx, ny, nz, _p(_f64(bbox)),
                                 _p(out), workers))
    return out


def distill_vjp(theta, widths, dims, bbox, dw, workers=8):
    nx, ny, nz = dims
    out = np.zeros(mlp_param_count(widths))
    _mlp_check(lib().orc_distill_vjp(_p(_f64(theta)), _widths(widths), len(widths), nx, ny, nz, _p(_f64(bbox)),
                                     _p(_f64(dw)), _p(out), workers))
    return out


def posed_occupancy(theta, widths, pose, offsets, roots_x, workers=8):
    """posed_occupancy_batch (shape.cpp:242-269) -> (pred [n], argmax [n] int32)."""
    offs = np.ascontiguousarray(offsets, dtype=np.int64)
    n = offs.shape[0] - 1
    pose = _f64(pose if pose is not None else np.zeros(0))
    pred, am = np.zeros(n), np.zeros(n, np.int32)
    _mlp_check(lib().orc_posed_occupancy(_p(_f64(theta)), _widths(widths), len(widths), _p(pose), pose.shape[0],
                                         offs.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                         _p(_f64(roots_x).reshape(-1, 3)), n, _p(pred), _p(am, _i32), workers))
    return pred, am


def mlp_weights_jacobian(theta, widths, x, workers=8):
    """SkinningMlp::weights and weight_jacobian (skinning.cpp:41-64) at x [n,3]."""
    x = _f64(x).reshape(-1, 3)
    n, nb = x.shape[0], widths[-1]
    w, dw = np.zeros((n, nb)), np.zeros((n, nb, 3))
    _mlp_check(lib().orc_mlp_weights_jacobian(_p(_f64(theta)), _widths(widths), len(widths), _p(x), n, _p(w), _p(dw),
                                              workers))
    return w, dw


def batch_search_mlp(theta, widths, bones, x_prime, max_iters, conv_eps, div_eps, dedup_dist, workers=8):
    """batch_search with SearchVariant::Mlp (correspondence.cpp:126-192), dense outputs."""
    B, x = _f64(bones).reshape(-1, 12), _f64(x_prime).reshape(-1, 3)
    n, nb = x.shape[0], B.shape[0]
    out = dict(x_c=np.zeros((n, nb, 3)), jinv=np.zeros((n, nb, 3, 3)), resid=np.zeros((n, nb)),
               iters=np.zeros((n, nb), np.int32), converged=np.zeros((n, nb), np.uint8),
               keep=np.zeros((n, nb), np.uint8))
    _mlp_check(lib().orc_batch_search_mlp(_p(_f64(theta)), _widths(widths), len(widths), _p(B), nb, _p(x), n,
                                          int(max_iters), conv_eps, div_eps, dedup_dist, workers, _p(out["x_c"]),
                                          _p(out["jinv"]), _p(out["resid"]), _p(out["iters"], _i32),
                                          _p(out["converged"], _u8), _p(out["keep"], _u8)))
    return out


# ---------------------------------------------------------------- the reference's own sources (oracle/_ref)
_REF = os.path.join(_HERE, "_ref", "libfskin_ref.so")
_ref = None


def ref_available() -> bool:
    """oracle/_ref/libfskin_ref.so: the reference's proj/src/{geometry,skinning,deformer,correspondence}.cpp
    compiled unmodified against oracle/eigen_shim (oracle/ref_build.sh; built here, travels to the box)."""
    deps = [os.path.join(_HERE, f) for f in ("ref_capi.cpp", "ref_stubs.cpp", "ref_build.sh",
                                              os.path.join("eigen_shim", "Eigen", "Dense"))]
    stale = not os.path.exists(_REF) or os.path.getmtime(_REF) < max(os.path.getmtime(d) for d in deps)
    if stale and os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["sh", os.path.join(_HERE, "ref_build.sh")], check=True, capture_output=True)
    return os.path.exists(_REF)


def ref_lib():
    global _ref
    if _ref is None:
        if not ref_available():
            raise OracleError("oracle/_ref/libfskin_ref.so not built (needs /root/reference at build time)")
        L = ctypes.CDLL(_REF)
        L.ref_last_error.restype = ctypes.c_char_p
        L.ref_precompute_tgrid.argtypes = [_d, _int, _int, _int, _int, _d, _d, _int, _d]
        L.ref_batch_search.argtypes = [_d, _int, _int, _int, _int, _d, _d, _d, _i64, _int, ctypes.c_double,
                                       ctypes.c_double, ctypes.c_double, _int, ctypes.POINTER(ctypes.c_int64), _d, _d,
                                       _d, _i32, _i32, _i64, ctypes.POINTER(ctypes.c_int64)]
        L.ref_init_states.argtypes = [_d, _int, _int, _int, _int, _d, _d, _d, _i64, _d, _d]
        _ref = L
    return _ref


def _ref_check(rc):
    if rc != 0:
        msg = ref_lib().ref_last_error().decode()
        raise (OracleInvalidArgument if rc == 1 else OracleError)(msg)


def ref_precompute_transform_grid(weights, dims, bbox, bones, workers=1):
    w, bb, B = _f64(weights), _f64(bbox), _f64(bones).reshape(-1, 12)
    out = np.zeros((dims[0] * dims[1] * dims[2], 12))
    _ref_check(ref_lib().ref_precompute_tgrid(_p(w), *dims, w.shape[1], _p(bb), _p(B), workers, _p(out)))
    return out


def ref_batch_search(weights, dims, bbox, bones, x_prime, max_iters, conv_eps, div_eps, dedup_dist, workers=1):
    """The reference's precompute_transform_grid + batch_search (its own code): CorrespondenceSets as
    dict(offsets [n+1], x [M,3], resid [M], jinv [M,3,3], bone [M], iters [M])."""
    w, bb, B, x = _f64(weights), _f64(bbox), _f64(bones).reshape(-1, 12), _f64(x_prime).reshape(-1, 3)
    n, nb = x.shape[0], B.shape[0]
    cap = max(1, min(n * nb, 4 * n + 1024))  # ~1.05 roots are kept per query; rerun with the exact count if not
    while True:
        offs = np.zeros(n + 1, np.int64)
        out = dict(x=np.empty((cap, 3)), resid=np.empty(cap), jinv=np.empty((cap, 3, 3)), bone=np.empty(cap, np.int32),
                   iters=np.empty(cap, np.int32))
        total = ctypes.c_int64()
        rc = ref_lib().ref_batch_search(_p(w), *dims, w.shape[1], _p(bb), _p(B), _p(x), n, int(max_iters), conv_eps,
                                        div_eps, dedup_dist, workers, offs.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                        _p(out["x"]), _p(out["resid"]), _p(out["jinv"]), _p(out["bone"], _i32),
                                        _p(out["iters"], _i32), cap, ctypes.byref(total))
        if rc == 1 and total.value > cap:
            cap = total.value
            continue
        _ref_check(rc)
        m = total.value
        return dict(offsets=offs, **{k: v[:m] for k, v in out.items()})


def ref_init_states(weights, dims, bbox, bones, x_prime):
    w, bb, B, x = _f64(weights), _f64(bbox), _f64(bones).reshape(-1, 12), _f64(x_prime).reshape(-1, 3)
    n, nb = x.shape[0], B.shape[0]
    x0, j0 = np.zeros((n, nb, 3)), np.zeros((n, nb, 3, 3))
    _ref_check(ref_lib().ref_init_states(_p(w), *dims, nb, _p(bb), _p(B), _p(x), n, _p(x0), _p(j0)))
    return x0, j0

