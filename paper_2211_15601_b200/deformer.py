"""Python host mirror of the reference deformer/correspondence API over the C-ABI.

Names, argument meaning and error behaviour follow
``proj/include/fskin/deformer.hpp`` and ``correspondence.hpp``; tensors are torch CUDA
tensors (float32) resident on the context's device. All compute goes through
``libfsk_b200.so`` (``include/fsk.h``) — there is no CPU path: without the library or
an sm_100 GPU every call raises.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import FskError, FskInvalidArgument, GridDesc, SearchOpts, SearchOut, check  # noqa: F401


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _stream(device):
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


@dataclass
class GridDims:
    """``GridDims`` (skinning.hpp:45-52)."""
    nx: int = 64
    ny: int = 64
    nz: int = 16

    def vertex_count(self) -> int:
        return self.nx * self.ny * self.nz


@dataclass
class SearchOptions:
    """``SearchOptions`` (correspondence.hpp:14-26)."""
    max_iters: int = 50
    conv_eps: float = 1e-5
    div_eps: float = 0.5
    dedup_dist: float = 1e-2
    sort: bool = True  # spatial ordering of queries (performance only)
    # "mixed" (fp32 pass + fp64 escalation, the escalation an exact replay of the reference when the
    # weight grid is given), "mixed-fast" (ablation: fused fp64 escalation), "fp32" (ablation),
    # "fp64" (every solve in fp64), "exact64" (every solve an exact fp64 replay; needs the weights)
    precision: str = "mixed"

    @staticmethod
    def defaults_for(bbox) -> "SearchOptions":
        """``SearchOptions::defaults_for`` (correspondence.cpp:10-17)."""
        lo, hi = [float(v) for v in bbox[:3]], [float(v) for v in bbox[3:]]
        diag = math.sqrt(sum((h - l) ** 2 for l, h in zip(lo, hi)))
        return SearchOptions(50, 1e-5 * diag, 0.5 * diag, 1e-2 * diag)

    def validate(self) -> None:
        """``SearchOptions::validate`` (correspondence.cpp:19-25)."""
        if self.max_iters < 1:
            raise FskInvalidArgument("search: max_iters must be >= 1")
        if not self.conv_eps > 0.0:
            raise FskInvalidArgument("search: conv_eps must be > 0")
        if not self.div_eps > self.conv_eps:
            raise FskInvalidArgument("search: div_eps must exceed conv_eps")
        if not self.dedup_dist >= 0.0:
            raise FskInvalidArgument("search: dedup_dist must be >= 0")

    def c(self) -> SearchOpts:
        flags = 0 if self.sort else _lib.FSK_SEARCH_NO_SORT
        flags |= {"mixed": 0, "fp32": _lib.FSK_SEARCH_FP32_ONLY, "fp64": _lib.FSK_SEARCH_FP64,
                  "exact64": _lib.FSK_SEARCH_EXACT64, "mixed-fast": _lib.FSK_SEARCH_FAST_ESC}[self.precision]
        return SearchOpts(int(self.max_iters), flags, float(self.conv_eps), float(self.div_eps),
                          float(self.dedup_dist))


def grid_desc(dims, bbox, n_bones) -> GridDesc:
    d = GridDesc()
    d.nx, d.ny, d.nz = (int(v) for v in dims)
    d.n_bones = int(n_bones)
    for a in range(3):
        d.bbox_min[a] = float(bbox[a])
        d.bbox_max[a] = float(bbox[3 + a])
    return d


def _f32(t, name, device):
    if not isinstance(t, torch.Tensor):
        raise FskInvalidArgument(f"fsk: {name} must be a torch tensor")
    if t.device != device or t.dtype != torch.float32 or not t.is_contiguous():
        raise FskInvalidArgument(f"fsk: {name} must be a contiguous float32 tensor on {device}")
    return t


def _check_roots_out(out, n, device):
    """Caller-supplied CorrespondenceSet buffers: offsets [N+1] int64 and roots [cap,16] float32, contiguous,
    on the context's device (a short or mistyped buffer would be an out-of-bounds device write)."""
    offsets, roots = out
    for t, name, dt in ((offsets, "offsets", torch.int64), (roots, "roots", torch.float32)):
        if not isinstance(t, torch.Tensor) or t.device != device or t.dtype != dt or not t.is_contiguous():
            raise FskInvalidArgument(f"fsk: {name} must be a contiguous {dt} tensor on {device}")
    if offsets.numel() < n + 1:
        raise FskInvalidArgument("fsk: offsets needs n+1 entries")
    if roots.dim() != 2 or roots.shape[1] != 16:
        raise FskInvalidArgument("fsk: roots must be [cap, 16] float32 (fsk_root records)")
    return offsets, roots


class Deformer:
    """One context (``fsk_ctx``) on one GPU. The methods mirror the reference free
    functions; results are dense per-(point, init) tensors plus dedup masks."""

    def __init__(self, device=0):
        self.L = _lib.load()
        self.device = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
        self._ctx = ctypes.c_void_p()
        check(self.L.fsk_ctx_create(self.device.index or 0, ctypes.byref(self._ctx)))

    def close(self):
        if self._ctx:
            self.L.fsk_ctx_destroy(self._ctx)
            self._ctx = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def launch_count(self) -> int:
        return int(self.L.fsk_ctx_launch_count(self._ctx))

    @property
    def sm_count(self) -> int:
        return int(self.L.fsk_device_sm_count(self._ctx))

    # ---------------------------------------------------------------- measurement hooks
    def set_profiling(self, on: bool) -> None:
        check(self.L.fsk_ctx_set_profiling(self._ctx, 1 if on else 0))

    def prof_read(self, name=None, reset=True):
        """(total device ms, launches) of this context's kernels named ``name`` (None = all)."""
        ms, cnt = ctypes.c_double(), ctypes.c_int64()
        check(self.L.fsk_ctx_prof_read(self._ctx, name.encode() if name else None, ctypes.byref(ms),
                                       ctypes.byref(cnt), 1 if reset else 0))
        return ms.value, cnt.value

    def search_stats(self, reset=True):
        """(f32 solves, f32 iterations, f32 converged-terminating iterations, f64 solves,
        f64 iterations, f64 converged-terminating iterations, f32 iteration gathers)
        accumulated by searches."""
        buf = (ctypes.c_uint64 * 7)()
        check(self.L.fsk_ctx_search_stats(self._ctx, buf, 1 if reset else 0))
        return tuple(int(v) for v in buf)

    def measure_fp32_peak(self) -> float:
        t = ctypes.c_double()
        check(self.L.fsk_measure_fp32_peak(self._ctx, ctypes.byref(t)))
        return t.value

    def measure_l1_gather_peak(self) -> float:
        t = ctypes.c_double()
        check(self.L.fsk_measure_l1_gather_peak(self._ctx, ctypes.byref(t)))
        return t.value

    def measure_fp64_peak(self) -> float:
        t = ctypes.c_double()
        check(self.L.fsk_measure_fp64_peak(self._ctx, ctypes.byref(t)))
        return t.value

    # ---------------------------------------------------------------- K1
    def precompute_transform_grid(self, weights, dims, bbox, bones, out=None, out64=None):
        """``precompute_transform_grid`` (deformer.hpp:53-55) → tgrid [V,12] float32 (and the
        float64 grid into ``out64`` [V,12] when given)."""
        weights = _f32(weights, "weights", self.device)
        bones = _f32(bones, "bones", self.device)
        nb = weights.shape[1] if weights.dim() == 2 else bones.shape[0]
        desc = grid_desc(dims, bbox, nb)
        V = desc.nx * desc.ny * desc.nz
        if out is None:
            out = torch.empty((V, 12), dtype=torch.float32, device=self.device)
        check(self.L.fsk_precompute_tgrid(self._ctx, _ptr(weights), ctypes.byref(desc), _ptr(bones),
                                          bones.numel() // 12, _ptr(out), _ptr(out64), _stream(self.device)))
        return out

    # ---------------------------------------------------------------- K2 + dedup
    def alloc_search_out(self, n, nb, jinv=True, resid=True, iters=True, keep=True, x64=False):
        dev = self.device
        extra = {"x_c64": torch.empty((n, nb, 3), dtype=torch.float64, device=dev)} if x64 else {}
        return dict(
            **extra,
            x_c=torch.empty((n, nb, 3), dtype=torch.float32, device=dev),
            jinv=torch.empty((n, nb, 3, 3), dtype=torch.float32, device=dev) if jinv else None,
            resid=torch.empty((n, nb), dtype=torch.float32, device=dev) if resid else None,
            iters=torch.empty((n, nb), dtype=torch.int32, device=dev) if iters else None,
            converged=torch.empty((n, nb), dtype=torch.uint8, device=dev),
            keep=torch.empty((n, nb), dtype=torch.uint8, device=dev) if keep else None,
            n_roots=torch.empty((n,), dtype=torch.int32, device=dev) if keep else None,
        )

    @staticmethod
    def _c_out(o) -> SearchOut:
        return SearchOut(*[o[k].data_ptr() if o.get(k) is not None else None
                           for k in ("x_c", "jinv", "resid", "iters", "converged", "keep", "n_roots", "x_c64")])

    def batch_search(self, tgrid, dims, bbox, bones, points, opts: SearchOptions, out=None, tgrid64=None,
                     weights=None):
        """``batch_search`` voxel variant (correspondence.hpp:77-80) → dense per-(point, init)
        results: x_c, jinv, resid, iters, converged, keep (dedup), n_roots. ``weights`` (the
        SearchContext's skinning grid, [V, n_b]) is needed only for precision="exact64"."""
        tgrid = None if tgrid is None and tgrid64 is not None else _f32(tgrid, "tgrid", self.device)
        weights = None if weights is None else _f32(weights, "weights", self.device)
        bones = _f32(bones, "bones", self.device)
        points = _f32(points, "points", self.device)
        nb = bones.numel() // 12
        n = points.shape[0]
        desc = grid_desc(dims, bbox, nb)
        if out is None:
            out = self.alloc_search_out(n, nb)
        co = self._c_out(out)
        check(self.L.fsk_search_fwd(self._ctx, _ptr(tgrid), _ptr(tgrid64), _ptr(weights), ctypes.byref(desc), _ptr(bones), nb,
                                    _ptr(points), n,
                                    ctypes.byref(opts.c()), ctypes.byref(co), _stream(self.device)))
        return out

    def alloc_roots(self, n, nb, cap=None):
        """Device CorrespondenceSet buffers: offsets [N+1] int64, roots [cap,16] float32
        (fsk_root records: x(3), residual, J~(9), bone, iterations, pad)."""
        cap = n * nb if cap is None else cap
        return (torch.empty((n + 1,), dtype=torch.int64, device=self.device),
                torch.empty((max(cap, 1), 16), dtype=torch.float32, device=self.device))

    def batch_search_roots(self, tgrid, dims, bbox, bones, points, opts: SearchOptions, out=None, tgrid64=None,
                           weights=None):
        """``batch_search`` straight to CorrespondenceSets on the device (fsk_batch_search):
        returns (offsets, roots); roots of query p are roots[offsets[p]:offsets[p+1]]."""
        nb, n = bones.numel() // 12, points.shape[0]
        offsets, roots = _check_roots_out(out, n, self.device) if out is not None else self.alloc_roots(n, nb)
        desc = grid_desc(dims, bbox, nb)
        weights = None if weights is None else _f32(weights, "weights", self.device)
        tgrid = None if tgrid is None and tgrid64 is not None else _f32(tgrid, "tgrid", self.device)
        check(self.L.fsk_batch_search(self._ctx, _ptr(tgrid), _ptr(tgrid64),
                                      _ptr(weights), ctypes.byref(desc),
                                      _ptr(_f32(bones, "bones", self.device)), nb,
                                      _ptr(_f32(points, "points", self.device)), n, ctypes.byref(opts.c()),
                                      _ptr(offsets), _ptr(roots), roots.shape[0], _stream(self.device)))
        return offsets, roots

    def deform(self, weights, dims, bbox, bones, points, opts: SearchOptions, tgrid=None, out=None):
        """One deformer frame on device buffers (fsk_deform): precompute_transform_grid +
        batch_search → (offsets, roots). ``tgrid`` [V,12] receives the transform grid if given.
        Kept roots beyond the capacity of ``roots`` are dropped: check offsets[N] <= roots.shape[0]."""
        nb, n = bones.numel() // 12, points.shape[0]
        offsets, roots = _check_roots_out(out, n, self.device) if out is not None else self.alloc_roots(n, nb)
        if tgrid is not None:
            tgrid = _f32(tgrid, "tgrid", self.device)
        desc = grid_desc(dims, bbox, nb)
        check(self.L.fsk_deform(self._ctx, _ptr(_f32(weights, "weights", self.device)), ctypes.byref(desc),
                                _ptr(_f32(bones, "bones", self.device)), nb, _ptr(_f32(points, "points", self.device)),
                                n, ctypes.byref(opts.c()), _ptr(tgrid), _ptr(offsets), _ptr(roots), roots.shape[0],
                                _stream(self.device)))
        return offsets, roots

    def deform_frames(self, weights, dims, bbox, bones, points, opts: SearchOptions, tgrid=None, outs=None):
        """``fsk_deform_frames``: F frames (lists of device tensors bones [n_b,12], points [N_f,3]) of one
        subject; frame f+1's sort + K1 run beside frame f's search. Returns [(offsets, roots)] per frame
        (``outs``: caller-provided pairs, checked like ``deform``'s ``out``)."""
        F = len(points)
        if len(bones) != F or (outs is not None and len(outs) != F):
            raise FskInvalidArgument("fsk: one bones/points (and out) entry per frame")
        nb = bones[0].numel() // 12 if F else 1
        if outs is None:
            outs = [self.alloc_roots(p.shape[0], nb) for p in points]
        else:
            outs = [_check_roots_out(o, p.shape[0], self.device) for o, p in zip(outs, points)]
        bones = [_f32(b, "bones", self.device) for b in bones]
        points = [_f32(p, "points", self.device) for p in points]
        if tgrid is not None:
            tgrid = _f32(tgrid, "tgrid", self.device)
        desc = grid_desc(dims, bbox, nb)
        vp = ctypes.c_void_p
        arr = lambda ts: (vp * max(F, 1))(*[t.data_ptr() for t in ts])  # noqa: E731
        n = (ctypes.c_int64 * max(F, 1))(*[p.shape[0] for p in points])
        caps = (ctypes.c_int64 * max(F, 1))(*[r.shape[0] for _, r in outs])
        check(self.L.fsk_deform_frames(self._ctx, _ptr(_f32(weights, "weights", self.device)), ctypes.byref(desc), F,
                                       arr(bones), nb, arr(points), n, ctypes.byref(opts.c()), _ptr(tgrid),
                                       arr([o for o, _ in outs]), arr([r for _, r in outs]), caps,
                                       _stream(self.device)))
        return outs

    def search_bwd_roots(self, dims, bbox, n_bones, roots, root_index, grad_xc, deterministic=False, out=None,
                         order=None):
        """Backward from compact roots: root_index [N] int64 into ``roots`` (or -1). ``order`` (int32 [N],
        e.g. ``query_order(N)`` after the forward) visits the queries in the search's spatial order, so the
        fast mode aggregates per-cell contributions within each warp."""
        desc = grid_desc(dims, bbox, n_bones)
        V = desc.nx * desc.ny * desc.nz
        if out is None:
            out = torch.empty((V, 12), dtype=torch.float32, device=self.device)
        ri = root_index.to(device=self.device, dtype=torch.int64).contiguous()
        if ri.numel() != grad_xc.shape[0]:
            raise FskInvalidArgument("fsk: root_index needs one entry per query")
        if order is not None and (order.dtype != torch.int32 or order.device != self.device or
                                  order.numel() != grad_xc.shape[0] or not order.is_contiguous()):
            raise FskInvalidArgument("fsk: order must be a contiguous int32 tensor with one entry per query")
        check(self.L.fsk_search_bwd_roots_ordered(self._ctx, ctypes.byref(desc), _ptr(roots), _ptr(ri),
                                                  _ptr(_f32(grad_xc, "grad_xc", self.device)), grad_xc.shape[0],
                                                  _ptr(order), _ptr(out), 1 if deterministic else 0,
                                                  _stream(self.device)))
        return out

    def query_order(self, n, out=None):
        """The spatial order of the queries of this context's last device search (fsk_ctx_query_order)."""
        if out is None:
            out = torch.empty((n,), dtype=torch.int32, device=self.device)
        check(self.L.fsk_ctx_query_order(self._ctx, n, _ptr(out), _stream(self.device)))
        return out

    def measure_red_peak(self) -> float:
        t = ctypes.c_double()
        check(self.L.fsk_measure_red_peak(self._ctx, ctypes.byref(t)))
        return t.value

    def compact_roots(self, dense, n, nb):
        """Kept roots in CorrespondenceSet form: (offsets [N+1] int64, roots [M,16] float32 view of
        fsk_root records: x(3), residual, J~(9), bone, iterations, pad)."""
        offsets = torch.empty((n + 1,), dtype=torch.int64, device=self.device)
        cap = int(dense["n_roots"].sum().item()) if n else 0
        roots = torch.empty((max(cap, 1), 16), dtype=torch.float32, device=self.device)
        total = ctypes.c_int64()
        co = self._c_out(dense)
        check(self.L.fsk_compact_roots(self._ctx, ctypes.byref(co), n, nb, _ptr(offsets), _ptr(roots), cap,
                                       ctypes.byref(total), _stream(self.device)))
        return offsets, roots[: total.value]

    def init_states(self, tgrid, dims, bbox, bones, points):
        """``init_states`` (correspondence.hpp:62-63) → x0 [N,nb,3], J~0 [N,nb,3,3]."""
        nb = bones.numel() // 12
        n = points.shape[0]
        desc = grid_desc(dims, bbox, nb)
        x0 = torch.empty((n, nb, 3), dtype=torch.float32, device=self.device)
        j0 = torch.empty((n, nb, 3, 3), dtype=torch.float32, device=self.device)
        check(self.L.fsk_init_states(self._ctx, _ptr(_f32(tgrid, "tgrid", self.device)), ctypes.byref(desc),
                                     _ptr(_f32(bones, "bones", self.device)), nb,
                                     _ptr(_f32(points, "points", self.device)), n, _ptr(x0), _ptr(j0),
                                     _stream(self.device)))
        return x0, j0

    def eval_points(self, tgrid, dims, bbox, n_bones, x):
        """Batched ``trilerp_transform`` / ``forward_deform`` / ``deform_jacobian``
        (deformer.hpp:59-68): (T [N,12], d [N,3], J [N,3,3])."""
        n = x.shape[0]
        desc = grid_desc(dims, bbox, n_bones)
        t12 = torch.empty((n, 12), dtype=torch.float32, device=self.device)
        d = torch.empty((n, 3), dtype=torch.float32, device=self.device)
        J = torch.empty((n, 3, 3), dtype=torch.float32, device=self.device)
        check(self.L.fsk_eval_points(self._ctx, _ptr(_f32(tgrid, "tgrid", self.device)), ctypes.byref(desc),
                                     _ptr(_f32(x, "x", self.device)), n, _ptr(t12), _ptr(d), _ptr(J),
                                     _stream(self.device)))
        return t12, d, J

    # ---------------------------------------------------------------- K3 + GW
    def search_bwd(self, dims, bbox, n_bones, dense, grad_xc, root_sel, deterministic=False, out=None):
        """Implicit-differentiation backward (diff.cpp:43-51, :336-359), grid-routed:
        dL/dT [V,12] from per-point cotangents dL/dx* and the selected root per point."""
        desc = grid_desc(dims, bbox, n_bones)
        V = desc.nx * desc.ny * desc.nz
        n = grad_xc.shape[0]
        if out is None:
            out = torch.empty((V, 12), dtype=torch.float32, device=self.device)
        rs = root_sel.to(device=self.device, dtype=torch.int32).contiguous()
        check(self.L.fsk_search_bwd(self._ctx, ctypes.byref(desc), _ptr(dense["x_c"]), _ptr(dense["jinv"]),
                                    dense["x_c"].shape[1], _ptr(_f32(grad_xc, "grad_xc", self.device)), _ptr(rs), n,
                                    _ptr(out), 1 if deterministic else 0, _stream(self.device)))
        return out

    def implicit_u_exact(self, weights, dims, bbox, bones, x_star, grad_xc):
        """``implicit_grad_exact``'s cotangent (diff.cpp:31-41), grid-routed: u = −(∂d/∂x*)⁻ᵀ v in
        float64 from the weight-grid Jacobian at x* → (u [N,3] float64, ok [N] uint8, det [N] float64);
        ok = 0 marks a singular root (|det| < 1e-10, the reference's SingularRootError)."""
        nb = bones.numel() // 12
        desc = grid_desc(dims, bbox, nb)
        n = x_star.shape[0]
        u = torch.empty((n, 3), dtype=torch.float64, device=self.device)
        ok = torch.empty((n,), dtype=torch.uint8, device=self.device)
        det = torch.empty((n,), dtype=torch.float64, device=self.device)
        check(self.L.fsk_implicit_u_exact(self._ctx, _ptr(_f32(weights, "weights", self.device)), ctypes.byref(desc),
                                          _ptr(_f32(bones, "bones", self.device)), nb,
                                          _ptr(_f32(x_star, "x_star", self.device)),
                                          _ptr(_f32(grad_xc, "grad_xc", self.device)), n, _ptr(u), _ptr(ok), _ptr(det),
                                          _stream(self.device)))
        return u, ok, det

    def search_bwd_exact_roots(self, weights, dims, bbox, bones, roots, root_index, grad_xc, deterministic=False,
                               out=None):
        """Backward from compact roots with the exact cotangent (implicit_grad_exact) → (dL/dT [V,12],
        ok [N] uint8: 0 = singular root, skipped)."""
        nb = bones.numel() // 12
        desc = grid_desc(dims, bbox, nb)
        V = desc.nx * desc.ny * desc.nz
        n = grad_xc.shape[0]
        if out is None:
            out = torch.empty((V, 12), dtype=torch.float32, device=self.device)
        ok = torch.empty((n,), dtype=torch.uint8, device=self.device)
        ri = root_index.to(device=self.device, dtype=torch.int64).contiguous()
        check(self.L.fsk_search_bwd_exact_roots(self._ctx, _ptr(_f32(weights, "weights", self.device)),
                                                ctypes.byref(desc), _ptr(_f32(bones, "bones", self.device)), nb,
                                                _ptr(roots), _ptr(ri), _ptr(_f32(grad_xc, "grad_xc", self.device)), n,
                                                _ptr(out), _ptr(ok), 1 if deterministic else 0, _stream(self.device)))
        return out, ok

    # ---------------------------------------------------------------- deterministic backward across ranks
    def _bwd_src(self, dense=None, root_sel=None, roots=None, root_index=None):
        if roots is not None:
            ri = root_index.to(device=self.device, dtype=torch.int64).contiguous()
            return _lib.BwdSrc(None, None, None, 0, roots.data_ptr(), ri.data_ptr()), ri
        rs = root_sel.to(device=self.device, dtype=torch.int32).contiguous()
        return _lib.BwdSrc(dense["x_c"].data_ptr(), dense["jinv"].data_ptr(), rs.data_ptr(), dense["x_c"].shape[1],
                           None, None), rs

    def search_bwd_max_term(self, dims, bbox, n_bones, grad_xc, **src):
        """Max term of the deterministic backward's fixed-point scale over this shard's roots → [1] float32
        (dense=..., root_sel=... or roots=..., root_index=...)."""
        desc = grid_desc(dims, bbox, n_bones)
        c, keep = self._bwd_src(**src)
        m = torch.empty((1,), dtype=torch.float32, device=self.device)
        check(self.L.fsk_search_bwd_max_term(self._ctx, ctypes.byref(desc), ctypes.byref(c),
                                             _ptr(_f32(grad_xc, "grad_xc", self.device)), grad_xc.shape[0], _ptr(m),
                                             _stream(self.device)))
        return m

    def search_bwd_fixed(self, dims, bbox, n_bones, grad_xc, n_scale, max_term, acc, **src):
        """Accumulate this shard's int64 fixed-point dL/dT into ``acc`` [V,12] int64 with the scale of
        (max_term, n_scale) — the max over all shards and the total point count."""
        desc = grid_desc(dims, bbox, n_bones)
        c, keep = self._bwd_src(**src)
        check(self.L.fsk_search_bwd_fixed(self._ctx, ctypes.byref(desc), ctypes.byref(c),
                                          _ptr(_f32(grad_xc, "grad_xc", self.device)), grad_xc.shape[0], int(n_scale),
                                          _ptr(max_term), _ptr(acc), _stream(self.device)))
        return acc

    def fixed_to_float(self, acc, n_scale, max_term, out=None):
        if out is None:
            out = torch.empty(acc.shape, dtype=torch.float32, device=self.device)
        check(self.L.fsk_fixed_to_float(self._ctx, _ptr(acc), acc.numel(), int(n_scale), _ptr(max_term), _ptr(out),
                                        _stream(self.device)))
        return out

    def grad_weights(self, dims, bbox, grad_tgrid, bones, out=None):
        """dL/dw [V, n_b] = <dL/dT_v, B_i>_F."""
        nb = bones.numel() // 12
        desc = grid_desc(dims, bbox, nb)
        V = desc.nx * desc.ny * desc.nz
        if out is None:
            out = torch.empty((V, nb), dtype=torch.float32, device=self.device)
        check(self.L.fsk_grad_weights(self._ctx, ctypes.byref(desc), _ptr(_f32(grad_tgrid, "grad_tgrid", self.device)),
                                      _ptr(_f32(bones, "bones", self.device)), nb, _ptr(out), _stream(self.device)))
        return out

    # ---------------------------------------------------------------- MLP stages
    @staticmethod
    def _widths(widths):
        return (ctypes.c_int32 * len(widths))(*[int(w) for w in widths])

    def distill(self, theta, widths, dims, bbox, out=None):
        """``distill`` (skinning.cpp:195-221): skinning-network softmax weights [V, n_b] at the
        grid vertices. ``theta``: the flat Mlp::parameters() vector (mlp.cpp:207-219)."""
        nb = int(widths[-1])
        desc = grid_desc(dims, bbox, nb)
        V = desc.nx * desc.ny * desc.nz
        if out is None:
            out = torch.empty((V, nb), dtype=torch.float32, device=self.device)
        check(self.L.fsk_distill(self._ctx, _ptr(_f32(theta, "theta", self.device)), self._widths(widths), len(widths),
                                 ctypes.byref(desc), _ptr(out), _stream(self.device)))
        return out

    def batch_search_mlp(self, theta, widths, bones, points, opts: SearchOptions, out=None):
        """``batch_search`` with ``SearchVariant::Mlp`` (correspondence.cpp:77-79): the skinning
        network evaluated at every Broyden iterate (tensor cores) instead of the grid."""
        bones = _f32(bones, "bones", self.device)
        points = _f32(points, "points", self.device)
        nb, n = bones.numel() // 12, points.shape[0]
        if out is None:
            out = self.alloc_search_out(n, nb)
        co = self._c_out(out)
        check(self.L.fsk_search_fwd_mlp(self._ctx, _ptr(_f32(theta, "theta", self.device)), self._widths(widths),
                                        len(widths), _ptr(bones), nb, _ptr(points), n, ctypes.byref(opts.c()),
                                        ctypes.byref(co), _stream(self.device)))
        return out

    def distill_bwd(self, theta, widths, dims, bbox, grad_w, out=None):
        """VJP of ``distill``: dL/dtheta [P] from dL/dw [V, n_b] (Mlp::backward through the
        softmax head, mlp.cpp:38-41,140-163)."""
        nb = int(widths[-1])
        desc = grid_desc(dims, bbox, nb)
        if out is None:
            P = sum(int(widths[i + 1]) * int(widths[i]) + int(widths[i + 1]) for i in range(len(widths) - 1))
            out = torch.empty((P,), dtype=torch.float32, device=self.device)
        check(self.L.fsk_distill_bwd(self._ctx, _ptr(_f32(theta, "theta", self.device)), self._widths(widths),
                                     len(widths), ctypes.byref(desc), _ptr(_f32(grad_w, "grad_w", self.device)),
                                     _ptr(out), _stream(self.device)))
        return out

    def posed_occupancy(self, theta, widths, pose, offsets, roots, occ_per_root=None):
        """``posed_occupancy_batch`` (shape.cpp:242-269) over device CorrespondenceSets
        (offsets [N+1] int64, roots [M,16] fsk_root records): returns (pred [N], argmax [N])."""
        n = offsets.shape[0] - 1
        n_roots = int(offsets[-1].item()) if n >= 0 else 0
        pose_t = None
        if pose is not None and len(pose) > 0:
            pose_t = torch.as_tensor(pose, dtype=torch.float32).to(self.device).contiguous()
        n_pose = 0 if pose_t is None else pose_t.numel()
        pred = torch.empty((max(n, 0),), dtype=torch.float32, device=self.device)
        am = torch.empty((max(n, 0),), dtype=torch.int32, device=self.device)
        check(self.L.fsk_posed_occupancy(self._ctx, _ptr(_f32(theta, "theta", self.device)), self._widths(widths),
                                         len(widths), _ptr(pose_t), n_pose, _ptr(offsets), _ptr(roots), n, n_roots,
                                         _ptr(pred), _ptr(am), _ptr(occ_per_root), _stream(self.device)))
        return pred, am

    # ---------------------------------------------------------------- end to end (host buffers)
    def deform_host(self, weights, dims, bbox, bones, points, opts: SearchOptions, offsets, roots):
        """``fsk_deform_host``: host (pinned) buffers in, CorrespondenceSets out. Returns the
        number of kept roots written into ``roots`` (a [cap,16] float32 pinned tensor)."""
        nb = bones.numel() // 12
        desc = grid_desc(dims, bbox, nb)
        total = ctypes.c_int64()
        check(self.L.fsk_deform_host(self._ctx, _ptr(weights), ctypes.byref(desc), _ptr(bones), nb, _ptr(points),
                                     points.shape[0], ctypes.byref(opts.c()), _ptr(offsets), _ptr(roots),
                                     roots.shape[0], ctypes.byref(total), _stream(self.device)))
        return total.value

    def deform_host_frames(self, weights, dims, bbox, bones, points, opts: SearchOptions, offsets, roots):
        """``fsk_deform_host_frames``: one subject, F frames (lists of host tensors: bones [n_b,12],
        points [N_f,3], offsets [N_f+1] int64, roots [cap_f,16] float32), double-buffered so frame
        f+1's upload and search overlap frame f's download. Returns the kept-root count per frame."""
        F = len(points)
        if not (len(bones) == len(offsets) == len(roots) == F):
            raise FskInvalidArgument("fsk: one bones/points/offsets/roots entry per frame")
        nb = bones[0].numel() // 12 if F else 1
        desc = grid_desc(dims, bbox, nb)
        vp = ctypes.c_void_p
        arr = lambda ts: (vp * max(F, 1))(*[t.data_ptr() for t in ts])  # noqa: E731
        n = (ctypes.c_int64 * max(F, 1))(*[p.shape[0] for p in points])
        caps = (ctypes.c_int64 * max(F, 1))(*[r.shape[0] for r in roots])
        totals = (ctypes.c_int64 * max(F, 1))()
        check(self.L.fsk_deform_host_frames(self._ctx, _ptr(weights), ctypes.byref(desc), F, arr(bones), nb,
                                            arr(points), n, ctypes.byref(opts.c()), arr(offsets), arr(roots), caps,
                                            totals, _stream(self.device)))
        return [int(totals[i]) for i in range(F)]


class MultiDeformer:
    """Single-process multi-GPU C-ABI (``fsk_multi_*``): one context, stream and host thread
    per device, points sharded in contiguous ranges (parallel.hpp:28-29), NCCL all-reduce of
    dL/dT in the backward. Host (pinned or pageable) buffers in and out."""

    def __init__(self, devices):
        self.L = _lib.load()
        self._m = ctypes.c_void_p()
        devs = (ctypes.c_int32 * len(devices))(*devices)
        check(self.L.fsk_multi_create(len(devices), devs, ctypes.byref(self._m)))

    @property
    def device_count(self) -> int:
        return int(self.L.fsk_multi_device_count(self._m))

    def close(self):
        if self._m:
            self.L.fsk_multi_destroy(self._m)
            self._m = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def deform_host(self, weights, dims, bbox, bones, points, opts: SearchOptions, offsets, roots):
        nb = bones.numel() // 12
        desc = grid_desc(dims, bbox, nb)
        total = ctypes.c_int64()
        check(self.L.fsk_multi_deform_host(self._m, _ptr(weights), ctypes.byref(desc), _ptr(bones), nb, _ptr(points),
                                           points.shape[0], ctypes.byref(opts.c()), _ptr(offsets), _ptr(roots),
                                           roots.shape[0], ctypes.byref(total)))
        return total.value

    def grad_weights_host(self, dims, bbox, bones, roots, root_index, grad_xc, deterministic=False):
        nb = bones.numel() // 12
        desc = grid_desc(dims, bbox, nb)
        V = desc.nx * desc.ny * desc.nz
        out = torch.empty((V, nb), dtype=torch.float32)
        check(self.L.fsk_multi_grad_weights_host(self._m, ctypes.byref(desc), _ptr(bones), nb, _ptr(roots),
                                                 _ptr(root_index), _ptr(grad_xc), grad_xc.shape[0], _ptr(out),
                                                 1 if deterministic else 0))
        return out


# ---------------------------------------------------------------- wire and disk formats
def _io_check(rc):
    if rc != _lib.FSK_OK:
        L = _lib.load()
        msg = (L.fsk_io_last_error() or L.fsk_last_error()).decode()
        raise (FskInvalidArgument if rc == _lib.FSK_EINVAL else FskError)(msg)


def read_sknv(path):
    """load_sknv (skinning.cpp:264-288) -> (dims, bbox [6] float32, weights [V, n_b] float32)."""
    L = _lib.load()
    d = GridDesc()
    _io_check(L.fsk_sknv_read(path.encode(), ctypes.byref(d), None, 0))
    w = torch.empty((d.nx * d.ny * d.nz, d.n_bones), dtype=torch.float32)
    _io_check(L.fsk_sknv_read(path.encode(), ctypes.byref(d), _ptr(w), w.numel()))
    bbox = torch.tensor(list(d.bbox_min) + list(d.bbox_max), dtype=torch.float32)
    return (d.nx, d.ny, d.nz), bbox.numpy(), w


def write_sknv(path, dims, bbox, weights):
    L = _lib.load()
    w = weights.contiguous().float().cpu()
    _io_check(L.fsk_sknv_write(path.encode(), ctypes.byref(grid_desc(dims, bbox, w.shape[1])), _ptr(w)))


def read_points_bin(path):
    L = _lib.load()
    n = ctypes.c_int64()
    _io_check(L.fsk_points_bin_read(path.encode(), None, 0, ctypes.byref(n)))
    p = torch.empty((n.value, 3), dtype=torch.float32)
    _io_check(L.fsk_points_bin_read(path.encode(), _ptr(p), n.value, ctypes.byref(n)))
    return p


def write_points_bin(path, points):
    L = _lib.load()
    p = points.contiguous().float().cpu()
    _io_check(L.fsk_points_bin_write(path.encode(), _ptr(p), p.shape[0]))


def write_correspondence_dump(path, queries, offsets, roots, threads=0):
    """save_correspondence_dump (pointio.cpp:97-117) from host CorrespondenceSets."""
    L = _lib.load()
    q, o, r = (t.contiguous().cpu() for t in (queries.float(), offsets.long(), roots.float()))
    _io_check(L.fsk_write_correspondence_dump(path.encode(), _ptr(q), q.shape[0], _ptr(o), _ptr(r), threads))


def deform_files(deformer, grid_path, bones, points_path, opts: SearchOptions, dump_path):
    """One cmd_deform frame from files to file (fskin_cli.cpp:395-429): returns (queries, roots)."""
    b = bones.contiguous().float().cpu()
    nq, nr = ctypes.c_int64(), ctypes.c_int64()
    _io_check(deformer.L.fsk_deform_files(deformer._ctx, grid_path.encode(), _ptr(b), b.numel() // 12,
                                          points_path.encode(), ctypes.byref(opts.c()), dump_path.encode(),
                                          ctypes.byref(nq), ctypes.byref(nr)))
    return nq.value, nr.value
