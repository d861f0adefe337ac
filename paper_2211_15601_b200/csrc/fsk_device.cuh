// fsk_device.cuh — device-side building blocks of the Fast-SNARF deformer kernels (sm_100a),
// templated on the arithmetic type R (float for the fast pass, double for the escalation /
// parity pass).
//
// Semantics follow SURVEY Appendix A: the cell lookup clamps x to the bbox while the
// affine map is applied to the unclamped x (deformer.cpp:79-94,107-113); the initial
// Jacobian takes its gradient stencil from the locate_cell_lower cell
// (skinning.cpp:122-139,164-193). The Jacobian is formed from the 12-wide transform
// grid instead of the n_b-wide weight grid (equal in real arithmetic).
//
// Gather layout ("x-pair planes"): the reference's [V][12] transform grid is re-laid out
// once per pose into three planes, one per matrix row r, whose element v is
//     P[r][v] = { row r of T_v , row r of T_{v+1} }      (8 values)
// so one 256-bit load (LDG.E.ENL2.256, new on sm_100) returns one row of BOTH x-corners
// of a cell edge in float32 (two loads in float64), and x-neighbouring vertices sit 32 B
// apart. A trilinear evaluation is 12 LDG.256 (4 (dj,dk) edges × 3 rows) instead of 24
// LDG.128 in [V][12].
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace fsk {

struct GridP {
    int nx, ny, nz, nb;
    float lo[3], hi[3];
    float scale[3];  // (n-1)/ext: u = (p-lo)*scale; also 1/h for the gradient stencil
    double lod[3], hid[3], scaled[3];
};

template <typename R> __device__ __forceinline__ R g_lo(const GridP& g, int a);
template <> __device__ __forceinline__ float g_lo<float>(const GridP& g, int a) { return g.lo[a]; }
template <> __device__ __forceinline__ double g_lo<double>(const GridP& g, int a) { return g.lod[a]; }
template <typename R> __device__ __forceinline__ R g_hi(const GridP& g, int a);
template <> __device__ __forceinline__ float g_hi<float>(const GridP& g, int a) { return g.hi[a]; }
template <> __device__ __forceinline__ double g_hi<double>(const GridP& g, int a) { return g.hid[a]; }
template <typename R> __device__ __forceinline__ R g_scale(const GridP& g, int a);
template <> __device__ __forceinline__ float g_scale<float>(const GridP& g, int a) { return g.scale[a]; }
template <> __device__ __forceinline__ double g_scale<double>(const GridP& g, int a) { return g.scaled[a]; }

// Search thresholds (SearchOptions, correspondence.hpp:14-26) squared, plus the
// precision-escalation rule of the float32 pass.
struct SearchP {
    int max_iters;
    int esc_cap;        // fp32 pass stops after this many iterations and escalates
    int esc_min_div;    // escalate unconverged solves with at least this many iterations
    double conv2, div2, dedup2;
    double conv_eps, div_eps;  // unsquared, for the exact replay (err = sqrt(g·g) compared as the reference does)
    float esc_conv_lo, esc_conv_hi;  // err2 within [lo,hi]·conv2 → threshold too close to call in fp32
    float esc_div_lo, esc_div_hi;
    float esc_det;      // |det J0| below this → singular-fallback decision too close to call
    float esc_den;      // |dx·J~dg| below this → Broyden-guard decision too close to call
    float esc_jmax;     // converged root with max|J~| above this → ill-conditioned, x* not settled in fp32
    float esc_cos2;     // (dx·J~dg)² < esc_cos2·|dx|²|J~dg|² → near-degenerate rank-one update
    float esc_face;     // init point within this many cells of a grid plane: the cell (and so the
                        // piecewise Jacobian J0) is chosen within float32 noise
    float esc_spike;    // max|J~| above this at any iteration (a transient spike of the Broyden matrix) on a
                        // converged solve: float32 rounding was amplified on the way
    float esc_stag2;    // a step from iteration 2 on with err² > esc_stag2·(err² before it): a stagnating,
    float esc_stag_jmax;  // path-sensitive trajectory — escalated if it converges with max|J~| > esc_stag_jmax
    float esc_rho2;     // step rule: the stop decision is "near" when err² ∈ [rho², 1/rho²]·conv² ...
    float esc_tau2;     // ... and the step it decides (taken or not) is longer than tau·conv
    bool esc_conv_band_last;  // apply the ±conv band only where a conv decision can flip the mask (the last iteration)
    int esc_capconv;    // converged exactly at the float32 cap iteration: 0 keep, 1 escalate, 2 escalate if the last step > tau·conv
    bool esc_conv_all;  // every converged float32 solve escalates (scenes whose conv_eps is too coarse for 1e-4 abs)
};

template <typename R>
struct Cell {
    int base;  // vertex index of corner (i0, j0, k0)
    R tx, ty, tz;
};

// locate_cell (skinning.cpp:104-120) / locate_cell_lower (:122-139).
template <bool kLower, typename R>
__device__ __forceinline__ Cell<R> locate(const GridP& g, R x, R y, R z) {
    const R xs[3] = {x, y, z};
    const int n[3] = {g.nx, g.ny, g.nz};
    int idx[3];
    R t[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const R p = fmin(fmax(xs[a], g_lo<R>(g, a)), g_hi<R>(g, a));  // Aabb::clamp
        const R u = (p - g_lo<R>(g, a)) * g_scale<R>(g, a);
        int i = (int)floor(u);  // NaN -> 0 (cvt.rzi of NaN)
        if (kLower && i >= 1 && u == (R)i) i -= 1;
        i = max(0, min(i, n[a] - 2));
        idx[a] = i;
        t[a] = fmin(fmax(u - (R)i, (R)0), (R)1);
    }
    Cell<R> c;
    c.base = (idx[2] * g.ny + idx[1]) * g.nx + idx[0];
    c.tx = t[0];
    c.ty = t[1];
    c.tz = t[2];
    return c;
}

template <typename R>
struct V4 {
    R x, y, z, w;
};

// x-pair planes; stride = V * 8 elements between row planes.
template <typename R>
struct Planes {
    const R* p;
    int64_t stride;
};

__device__ __forceinline__ void load_edge(const Planes<float>& P, int v, int r, V4<float>& a, V4<float>& b) {
    const float* q = P.p + r * P.stride + (int64_t)v * 8;
#ifdef FSK_LDG128  // tuning ablation: two 128-bit loads instead of one 256-bit load
    const float4 lo = __ldg(reinterpret_cast<const float4*>(q)), hi = __ldg(reinterpret_cast<const float4*>(q) + 1);
    a = V4<float>{lo.x, lo.y, lo.z, lo.w};
    b = V4<float>{hi.x, hi.y, hi.z, hi.w};
#else
    asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
        : "l"(q));
#endif
}

__device__ __forceinline__ void load_edge(const Planes<double>& P, int v, int r, V4<double>& a, V4<double>& b) {
    const double* q = P.p + r * P.stride + (int64_t)v * 8;
    asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a.x), "=d"(a.y), "=d"(a.z), "=d"(a.w) : "l"(q));
    asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(b.x), "=d"(b.y), "=d"(b.z), "=d"(b.w) : "l"(q + 4));
}

template <typename R>
__device__ __forceinline__ void fma4(R* T, R w, const V4<R>& a) {
    T[0] = fma(w, a.x, T[0]);
    T[1] = fma(w, a.y, T[1]);
    T[2] = fma(w, a.z, T[2]);
    T[3] = fma(w, a.w, T[3]);
}

#ifndef FSK_NO_FFMA2
// Blackwell's packed FP32 FMA (FFMA2): two independent fma.rn.f32 per issue slot — the same
// two roundings as the scalar form, so results are bitwise unchanged. The trilinear accumulate
// (96 FMAs per evaluation) is the bulk of the float32 pass's FP instructions.
__device__ __forceinline__ void ffma2(float& c0, float& c1, float a0, float a1, float b0, float b1) {
    // c0 = fma(a0, b0, c0), c1 = fma(a1, b1, c1)
    asm("{\n\t.reg .b64 pa, pb, pc;\n\t"
        "mov.b64 pa, {%2, %3};\n\t"
        "mov.b64 pb, {%4, %5};\n\t"
        "mov.b64 pc, {%0, %1};\n\t"
        "fma.rn.f32x2 pc, pa, pb, pc;\n\t"
        "mov.b64 {%0, %1}, pc;\n\t}"
        : "+f"(c0), "+f"(c1)
        : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}

template <>
__device__ __forceinline__ void fma4<float>(float* T, float w, const V4<float>& a) {
    ffma2(T[0], T[1], w, w, a.x, a.y);
    ffma2(T[2], T[3], w, w, a.z, a.w);
}
#endif

// r0 = a·b0, r1 = a·b1 (the two x-corner weights of a cell edge); float: one packed FMUL2
template <typename R>
__device__ __forceinline__ void mul_pair(R a, R b0, R b1, R& r0, R& r1) {
    r0 = a * b0;
    r1 = a * b1;
}
#if !defined(FSK_NO_FFMA2) && defined(FSK_FMUL2)  // ablation: measured slower (C2 0.9700 -> 0.9716 ms, hashes equal)
template <>
__device__ __forceinline__ void mul_pair<float>(float a, float b0, float b1, float& r0, float& r1) {
    asm("{\n\t.reg .b64 pa, pb, pr;\n\t"
        "mov.b64 pa, {%2, %2};\n\t"
        "mov.b64 pb, {%3, %4};\n\t"
        "mul.rn.f32x2 pr, pa, pb;\n\t"
        "mov.b64 {%0, %1}, pr;\n\t}"
        : "=f"(r0), "=f"(r1)
        : "f"(a), "f"(b0), "f"(b1));
}
#endif

template <typename R>
__device__ __forceinline__ R row_dot(const V4<R>& a, R x, R y, R z) {
    return a.x * x + a.y * y + a.z * z + a.w;
}

// trilerp_transform_into (deformer.cpp:79-94) on the x-pair planes. Corner weights are
// formed as (wz*wy)*wx like the reference; accumulation is per (dk, dj) edge.
template <typename R>
__device__ __forceinline__ void trilerp_T(const Planes<R>& P, const GridP& g, const Cell<R>& c, R T[12]) {
#pragma unroll
    for (int e = 0; e < 12; ++e) T[e] = 0;
    const int nxy = g.nx * g.ny;
#pragma unroll
    for (int dk = 0; dk < 2; ++dk) {
        const R wz = dk ? c.tz : (R)1 - c.tz;
#pragma unroll
        for (int dj = 0; dj < 2; ++dj) {
            const R wyz = wz * (dj ? c.ty : (R)1 - c.ty);
            R w0, w1;
            mul_pair(wyz, (R)1 - c.tx, c.tx, w0, w1);
            const int v = c.base + dk * nxy + dj * g.nx;
#pragma unroll
            for (int r = 0; r < 3; ++r) {
                V4<R> a, b;
                load_edge(P, v, r, a, b);
                fma4(T + 4 * r, w0, a);
                fma4(T + 4 * r, w1, b);
            }
        }
    }
}

// Register cache of the 8 corners of one cell (4 x-pair edges × 3 rows = 96 values) for the
// float32 pass: about half of all Broyden re-evaluations land in the cell of the previous
// evaluation (late iterations take short steps), and those then issue no gather at all.
// The arithmetic is the same as trilerp_T's, so results are bitwise identical.
#ifndef FSK_CACHE_ROWS
#define FSK_CACHE_ROWS 3  // matrix rows of the current cell held in registers (the rest re-read from L1)
#endif
constexpr int kCacheRows = FSK_CACHE_ROWS;

template <typename R>
struct CellCache {
    int base;
    V4<R> a[4][3], b[4][3];  // [edge (dj + 2·dk)][row]: corner di = 0 / 1 (rows < kCacheRows used)
};

template <typename R>
__device__ __forceinline__ void cache_fill(const Planes<R>& P, const GridP& g, int base, CellCache<R>& C) {
    const int nxy = g.nx * g.ny;
    C.base = base;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const int v = base + (e >> 1) * nxy + (e & 1) * g.nx;
#pragma unroll
        for (int r = 0; r < kCacheRows; ++r) load_edge(P, v, r, C.a[e][r], C.b[e][r]);
    }
}

template <typename R>
__device__ __forceinline__ void trilerp_cached(const Planes<R>& P, const GridP& g, const CellCache<R>& C,
                                               const Cell<R>& c, R T[12]) {
#pragma unroll
    for (int e = 0; e < 12; ++e) T[e] = 0;
    const int nxy = g.nx * g.ny;
#pragma unroll
    for (int dk = 0; dk < 2; ++dk) {
        const R wz = dk ? c.tz : (R)1 - c.tz;
#pragma unroll
        for (int dj = 0; dj < 2; ++dj) {
            const R wyz = wz * (dj ? c.ty : (R)1 - c.ty);
            R w0, w1;
            mul_pair(wyz, (R)1 - c.tx, c.tx, w0, w1);
#pragma unroll
            for (int r = 0; r < 3; ++r) {
                V4<R> a, b;
                if (r < kCacheRows) {
                    a = C.a[2 * dk + dj][r];
                    b = C.b[2 * dk + dj][r];
                } else {
                    load_edge(P, c.base + dk * nxy + dj * g.nx, r, a, b);
                }
                fma4(T + 4 * r, w0, a);
                fma4(T + 4 * r, w1, b);
            }
        }
    }
}

// d = T·[x;1] on the unclamped x (deformer.cpp:107-113).
template <typename R>
__device__ __forceinline__ void apply_T(const R T[12], R x, R y, R z, R d[3]) {
    d[0] = T[0] * x + T[1] * y + T[2] * z + T[3];
    d[1] = T[4] * x + T[5] * y + T[6] * z + T[7];
    d[2] = T[8] * x + T[9] * y + T[10] * z + T[11];
}

template <typename R>
__device__ __forceinline__ void grad_term(R G[9], R y0, R y1, R y2, R gx, R gy, R gz) {
    G[0] = fma(y0, gx, G[0]); G[1] = fma(y0, gy, G[1]); G[2] = fma(y0, gz, G[2]);
    G[3] = fma(y1, gx, G[3]); G[4] = fma(y1, gy, G[4]); G[5] = fma(y1, gz, G[5]);
    G[6] = fma(y2, gx, G[6]); G[7] = fma(y2, gy, G[7]); G[8] = fma(y2, gz, G[8]);
}
#if !defined(FSK_NO_FFMA2) && defined(FSK_FFMA2_GRAD)  // ablation: spills 16 B in k_search_fast (pair constraints)
template <>
__device__ __forceinline__ void grad_term<float>(float G[9], float y0, float y1, float y2, float gx, float gy,
                                                 float gz) {
    ffma2(G[0], G[1], y0, y0, gx, gy);
    ffma2(G[2], G[3], y0, y1, gz, gx);
    ffma2(G[4], G[5], y1, y1, gy, gz);
    ffma2(G[6], G[7], y2, y2, gx, gy);
    G[8] = fmaf(y2, gz, G[8]);
}
#endif

// Analytic Jacobian and T(p) at x:
//   J = T_lin(p) + Σ_c (T_c x̃) ∇φ_c(p)ᵀ
// T from the locate_cell cell, ∇φ from the locate_cell_lower cell (±1/h stencils); both
// from one gather unless x lies exactly on an interior face (then the lower cell is
// gathered again).
template <typename R, bool kCache = false>
__device__ __forceinline__ void jacobian_and_T(const Planes<R>& P, const GridP& g, R x, R y, R z, R T[12], R J[9],
                                               bool grad = true, CellCache<R>* C = nullptr) {
    const Cell<R> c = locate<false, R>(g, x, y, z);
    if constexpr (kCache) cache_fill(P, g, c.base, *C);
    const Cell<R> cl = locate<true, R>(g, x, y, z);
    const int nxy = g.nx * g.ny;
    const bool same = (c.base == cl.base);
#pragma unroll
    for (int e = 0; e < 12; ++e) T[e] = 0;
    R G[9];
#pragma unroll
    for (int e = 0; e < 9; ++e) G[e] = 0;
    const R sx = g_scale<R>(g, 0), sy = g_scale<R>(g, 1), sz = g_scale<R>(g, 2);
#pragma unroll
    for (int dk = 0; dk < 2; ++dk) {
        const R wz = dk ? c.tz : (R)1 - c.tz;
        const R fz = dk ? cl.tz : (R)1 - cl.tz, gz_s = dk ? sz : -sz;
#pragma unroll
        for (int dj = 0; dj < 2; ++dj) {
            const R wyz = wz * (dj ? c.ty : (R)1 - c.ty);
            R w0, w1;
            mul_pair(wyz, (R)1 - c.tx, c.tx, w0, w1);
            const R fy = dj ? cl.ty : (R)1 - cl.ty, gy_s = dj ? sy : -sy;
            const R fx0 = (R)1 - cl.tx, fx1 = cl.tx;
            const int v = c.base + dk * nxy + dj * g.nx;
            R y0[3], y1[3];
#pragma unroll
            for (int r = 0; r < 3; ++r) {
                V4<R> a, b;
                if (kCache && r < kCacheRows) {
                    a = C->a[2 * dk + dj][r];
                    b = C->b[2 * dk + dj][r];
                } else {
                    load_edge(P, v, r, a, b);
                }
                fma4(T + 4 * r, w0, a);
                fma4(T + 4 * r, w1, b);
                y0[r] = row_dot(a, x, y, z);
                y1[r] = row_dot(b, x, y, z);
            }
            if (grad && same) {
                grad_term(G, y0[0], y0[1], y0[2], -sx * fy * fz, fx0 * gy_s * fz, fx0 * fy * gz_s);
                grad_term(G, y1[0], y1[1], y1[2], sx * fy * fz, fx1 * gy_s * fz, fx1 * fy * gz_s);
            }
        }
    }
    if (grad && !same) {  // x on an interior cell face: gradient from the lower-index cell
#pragma unroll 1
        for (int q = 0; q < 4; ++q) {
            const int dj = q & 1, dk = q >> 1;
            const R fz = dk ? cl.tz : (R)1 - cl.tz, gz_s = dk ? sz : -sz;
            const R fy = dj ? cl.ty : (R)1 - cl.ty, gy_s = dj ? sy : -sy;
            const R fx0 = (R)1 - cl.tx, fx1 = cl.tx;
            const int v = cl.base + dk * nxy + dj * g.nx;
            R y0[3], y1[3];
#pragma unroll
            for (int r = 0; r < 3; ++r) {
                V4<R> a, b;
                load_edge(P, v, r, a, b);
                y0[r] = row_dot(a, x, y, z);
                y1[r] = row_dot(b, x, y, z);
            }
            grad_term(G, y0[0], y0[1], y0[2], -sx * fy * fz, fx0 * gy_s * fz, fx0 * fy * gz_s);
            grad_term(G, y1[0], y1[1], y1[2], sx * fy * fz, fx1 * gy_s * fz, fx1 * fy * gz_s);
        }
    }
    J[0] = T[0] + G[0]; J[1] = T[1] + G[1]; J[2] = T[2] + G[2];
    J[3] = T[4] + G[3]; J[4] = T[5] + G[4]; J[5] = T[6] + G[5];
    J[6] = T[8] + G[6]; J[7] = T[9] + G[7]; J[8] = T[10] + G[8];
}

// initial_inverse_jacobian (correspondence.cpp:43-54): cofactor inverse, identity if
// |det| < 1e-8. Returns det (for the escalation rule).
template <typename R>
__device__ __forceinline__ R inverse_or_identity(const R J[9], R Ji[9]) {
    const R c00 = J[4] * J[8] - J[5] * J[7];
    const R c01 = J[2] * J[7] - J[1] * J[8];
    const R c02 = J[1] * J[5] - J[2] * J[4];
    const R c10 = J[5] * J[6] - J[3] * J[8];
    const R c11 = J[0] * J[8] - J[2] * J[6];
    const R c12 = J[2] * J[3] - J[0] * J[5];
    const R c20 = J[3] * J[7] - J[4] * J[6];
    const R c21 = J[1] * J[6] - J[0] * J[7];
    const R c22 = J[0] * J[4] - J[1] * J[3];
    const R det = J[0] * c00 + J[1] * c10 + J[2] * c20;
    if (fabs(det) < (R)1e-8) {  // NaN det fails the test and propagates, as in the reference
        Ji[0] = 1; Ji[1] = 0; Ji[2] = 0;
        Ji[3] = 0; Ji[4] = 1; Ji[5] = 0;
        Ji[6] = 0; Ji[7] = 0; Ji[8] = 1;
        return det;
    }
    const R inv = (R)1 / det;
    Ji[0] = c00 * inv; Ji[1] = c01 * inv; Ji[2] = c02 * inv;
    Ji[3] = c10 * inv; Ji[4] = c11 * inv; Ji[5] = c12 * inv;
    Ji[6] = c20 * inv; Ji[7] = c21 * inv; Ji[8] = c22 * inv;
    return det;
}

// Per-init start of search_one (correspondence.cpp:135-137): x0 = B_i^-1 x' as
// Rᵀx' + (−Rᵀt) (geometry.hpp:58-61), J~0 = J(x0)^-1 or I (:43-54), and T(x0) for g0.
// Returns det J(x0).
template <typename R, bool kCache = false>
__device__ __forceinline__ R solve_init(const Planes<R>& P, const GridP& g, const float* __restrict__ B, R xp0, R xp1,
                                        R xp2, R& x0, R& x1, R& x2, R Ji[9], R T[12], CellCache<R>* C = nullptr) {
    const R r00 = __ldg(B + 0), r01 = __ldg(B + 1), r02 = __ldg(B + 2), t0 = __ldg(B + 3);
    const R r10 = __ldg(B + 4), r11 = __ldg(B + 5), r12 = __ldg(B + 6), t1 = __ldg(B + 7);
    const R r20 = __ldg(B + 8), r21 = __ldg(B + 9), r22 = __ldg(B + 10), t2 = __ldg(B + 11);
    const R it0 = -(r00 * t0 + r10 * t1 + r20 * t2);
    const R it1 = -(r01 * t0 + r11 * t1 + r21 * t2);
    const R it2 = -(r02 * t0 + r12 * t1 + r22 * t2);
    x0 = r00 * xp0 + r10 * xp1 + r20 * xp2 + it0;
    x1 = r01 * xp0 + r11 * xp1 + r21 * xp2 + it1;
    x2 = r02 * xp0 + r12 * xp1 + r22 * xp2 + it2;
    R Jm[9];
    jacobian_and_T<R, kCache>(P, g, x0, x1, x2, T, Jm, true, C);
    return inverse_or_identity(Jm, Ji);
}

// One Broyden solve: search_one's per-init body (correspondence.cpp:132-146) with iterate
// (:97-124). With kFast (the float32 pass) the solve stops after p.esc_cap iterations and
// raises `esc` whenever its outcome could differ from a float64 solve: a long trajectory
// (iters >= esc_cap), an unconverged run of >= esc_min_div iterations, or a threshold
// decision (conv, div, |det|<1e-8, |den|>1e-18) taken within float32 noise of the threshold.
struct SolveOut {
    int iters;
    bool conv;
    bool esc;
    bool capped;  // escalated because the float32 pass hit its iteration cap (a long trajectory)
    int fills = 0;  // iteration gathers (cell-cache misses) of the float32 pass
    unsigned reasons = 0;  // FSK_ESC_REASONS study builds: which escalation rules fired (bit per rule)
};
#ifdef FSK_ESC_REASONS
#define FSK_REASON(bit) (reasons |= (1u << (bit)))
#else
#define FSK_REASON(bit) ((void)0)
#endif

// J~ += q wᵀ (the good-Broyden rank-one update, correspondence.cpp:120-121), one FMA per entry
template <typename R>
__device__ __forceinline__ void rank1_update(R Ji[9], R q0, R q1, R q2, R w0, R w1, R w2) {
    Ji[0] = fma(q0, w0, Ji[0]); Ji[1] = fma(q0, w1, Ji[1]); Ji[2] = fma(q0, w2, Ji[2]);
    Ji[3] = fma(q1, w0, Ji[3]); Ji[4] = fma(q1, w1, Ji[4]); Ji[5] = fma(q1, w2, Ji[5]);
    Ji[6] = fma(q2, w0, Ji[6]); Ji[7] = fma(q2, w1, Ji[7]); Ji[8] = fma(q2, w2, Ji[8]);
}
#if !defined(FSK_NO_FFMA2) && defined(FSK_FFMA2_RANK1)  // ablation: no fewer SASS instructions (pair moves)
template <>
__device__ __forceinline__ void rank1_update<float>(float Ji[9], float q0, float q1, float q2, float w0, float w1,
                                                    float w2) {
    ffma2(Ji[0], Ji[1], q0, q0, w0, w1);
    ffma2(Ji[2], Ji[3], q0, q1, w2, w0);
    ffma2(Ji[4], Ji[5], q1, q1, w1, w2);
    ffma2(Ji[6], Ji[7], q2, q2, w0, w1);
    Ji[8] = fmaf(q2, w2, Ji[8]);
}
#endif

#ifndef FSK_ESC_SPIKE
#define FSK_ESC_SPIKE 7.0f  // max|J~| of a transient Broyden-matrix spike that escalates a converged float32 solve
#endif
// One Broyden iteration after the divergence check (correspondence.cpp:106-122): step,
// re-evaluate, and — unless the new residual converged — the good-Broyden rank-one update.
// Returns true iff converged; `den` receives dx·J~dg (0 when converged).
template <typename R, bool kCache = false>
__device__ __forceinline__ bool broyden_step(const Planes<R>& P, const GridP& g, R xp0, R xp1, R xp2, R conv2, R& x0,
                                             R& x1, R& x2, R Ji[9], R& g0, R& g1, R& g2, R& err2, R& den,
                                             CellCache<R>* C = nullptr, R cos2 = 0, bool* degenerate = nullptr,
                                             int* fills = nullptr, R spike_at = 0) {
    // dx = −J~ g; x += dx (:106-107)
    const R dx0 = -(Ji[0] * g0 + Ji[1] * g1 + Ji[2] * g2);
    const R dx1 = -(Ji[3] * g0 + Ji[4] * g1 + Ji[5] * g2);
    const R dx2 = -(Ji[6] * g0 + Ji[7] * g1 + Ji[8] * g2);
    x0 += dx0;
    x1 += dx1;
    x2 += dx2;
    // g' = d(x) − x'; dg = g' − g (:108-112)
    R T[12], d[3];
    const Cell<R> c = locate<false, R>(g, x0, x1, x2);
    if constexpr (kCache) {
        if (c.base != C->base) {
            cache_fill(P, g, c.base, *C);
            if (fills) ++*fills;
        }
        trilerp_cached(P, g, *C, c, T);
    } else {
        trilerp_T(P, g, c, T);
    }
    apply_T(T, x0, x1, x2, d);
    const R n0 = d[0] - xp0, n1 = d[1] - xp1, n2 = d[2] - xp2;
    const R dg0 = n0 - g0, dg1 = n1 - g1, dg2 = n2 - g2;
    g0 = n0;
    g1 = n1;
    g2 = n2;
    err2 = g0 * g0 + g1 * g1 + g2 * g2;
    den = 0;
    if (err2 < conv2) return true;  // (:113-116)
    // good Broyden: J~ += ((dx − J~dg)/(dx·J~dg)) (dxᵀJ~) if |den| > 1e-18 (:118-122)
    const R j0 = Ji[0] * dg0 + Ji[1] * dg1 + Ji[2] * dg2;
    const R j1 = Ji[3] * dg0 + Ji[4] * dg1 + Ji[5] * dg2;
    const R j2 = Ji[6] * dg0 + Ji[7] * dg1 + Ji[8] * dg2;
    den = dx0 * j0 + dx1 * j1 + dx2 * j2;
    if (degenerate) {  // float32 pass: |cos(dx, J~dg)| < sqrt(cos2)
        const R nd = dx0 * dx0 + dx1 * dx1 + dx2 * dx2, nj = j0 * j0 + j1 * j1 + j2 * j2;
        if (den * den < cos2 * (nd * nj)) *degenerate = true;
    }
    if (fabs(den) > (R)1e-18) {
        const R inv = (R)1 / den;
        const R q0 = (dx0 - j0) * inv, q1 = (dx1 - j1) * inv, q2 = (dx2 - j2) * inv;
        const R w0 = dx0 * Ji[0] + dx1 * Ji[3] + dx2 * Ji[6];
        const R w1 = dx0 * Ji[1] + dx1 * Ji[4] + dx2 * Ji[7];
        const R w2 = dx0 * Ji[2] + dx1 * Ji[5] + dx2 * Ji[8];
        rank1_update(Ji, q0, q1, q2, w0, w1, w2);
        if (fills && spike_at > (R)0) {  // float32 pass: a transient spike of the updated matrix
            R m = 0;
#pragma unroll
            for (int e = 0; e < 9; ++e) m = fmax(m, fabs(Ji[e]));
            if (m > spike_at) *fills |= 1 << 29;
        }
    }
    return false;
}

// Start of a solve (correspondence.cpp:135-137): x0, J~0 and g0 = d(x0) − x' from one
// gather. Returns det J(x0).
template <typename R, bool kCache = false>
__device__ __forceinline__ R solve_start(const Planes<R>& P, const GridP& g, const float* __restrict__ B, R xp0, R xp1,
                                         R xp2, R& x0, R& x1, R& x2, R Ji[9], R& g0, R& g1, R& g2, R& err2,
                                         CellCache<R>* C = nullptr) {
    R T[12], d[3];
    const R det = solve_init<R, kCache>(P, g, B, xp0, xp1, xp2, x0, x1, x2, Ji, T, C);
    apply_T(T, x0, x1, x2, d);
    g0 = d[0] - xp0;
    g1 = d[1] - xp1;
    g2 = d[2] - xp2;
    err2 = g0 * g0 + g1 * g1 + g2 * g2;
    return det;
}

template <typename R, bool kFast>
__device__ __forceinline__ SolveOut solve_one(const Planes<R>& P, const GridP& g, const float* __restrict__ B, R xp0,
                                              R xp1, R xp2, const SearchP& o, R& x0, R& x1, R& x2, R Ji[9], R& err2) {
    R g0, g1, g2;
#ifdef FSK_NO_REGCACHE
    constexpr bool kCache = false;
#else
    constexpr bool kCache = kFast;  // float32 pass: per-thread register cache of the current cell
#endif
    CellCache<R> cache;
    const R det = solve_start<R, kCache>(P, g, B, xp0, xp1, xp2, x0, x1, x2, Ji, g0, g1, g2, err2, &cache);
    const R conv2 = (R)o.conv2, div2 = (R)o.div2;
    bool esc = false, capped = false;
    int fills = 0;
    unsigned reasons = 0;
    auto near_conv = [&](R e2) { return e2 >= (R)o.esc_conv_lo * conv2 && e2 <= (R)o.esc_conv_hi * conv2; };
    auto near_div = [&](R e2) { return e2 >= (R)o.esc_div_lo * div2 && e2 <= (R)o.esc_div_hi * div2; };
    if (kFast) {
        if (fabs(det) < (R)o.esc_det) esc = true, FSK_REASON(0);
        // J0 is piecewise (the trilinear gradient jumps across cell faces): an init point within float32
        // noise of a grid plane may take the other cell's Jacobian than float64 does
        {
            const R xi[3] = {x0, x1, x2};
            const int nn[3] = {g.nx, g.ny, g.nz};
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                const R u = (xi[a] - g_lo<R>(g, a)) * g_scale<R>(g, a);
                const R r = rint(u);
                if (r >= (R)0 && r <= (R)(nn[a] - 1) && fabs(u - r) < (R)o.esc_face) esc = true, FSK_REASON(14);
            }
        }
        if (near_conv(err2) && (!o.esc_conv_band_last || o.max_iters == 0)) esc = true, FSK_REASON(1);
        if (near_div(err2)) esc = true, FSK_REASON(10);
    }
    int iters = 0;
    R xl0 = x0, xl1 = x1, xl2 = x2, e2l = 0;  // float32 pass: position and err² before the last step
    // float32 pass: a stagnating step from iteration 2 on is flagged in bit 30 of `fills` (no extra register)
    constexpr int kStagBit = 1 << 30;
    constexpr int kSpikeBit = 1 << 29;  // a J~ spike above esc_spike on the way (also carried in `fills`)
    bool conv = err2 < conv2;  // (:100-103)
    if (!conv) {
        const int limit = kFast ? min(o.max_iters, o.esc_cap) : o.max_iters;
        int k = 0;
        for (; k < limit; ++k) {
            if (err2 > div2) break;  // divergence check at the top (:105)
            if (kFast) {
                xl0 = x0;
                xl1 = x1;
                xl2 = x2;
                e2l = err2;
            }
            R den;
            bool degen = false;
            const bool c = broyden_step<R, kCache>(P, g, xp0, xp1, xp2, conv2, x0, x1, x2, Ji, g0, g1, g2, err2, den,
                                                   &cache, (R)o.esc_cos2, kFast ? &degen : nullptr, &fills,
#if defined(FSK_NO_SPIKE)
                                                   (R)0);
#else
                                                   // a compile-time threshold (an immediate operand: the
                                                   // parameter held in a register spilled the loop)
                                                   kFast ? (R)FSK_ESC_SPIKE : (R)0);
#endif
            if (degen) esc = true, FSK_REASON(2);
            iters = k + 1;
            if (kFast && iters >= 2 && err2 > (R)o.esc_stag2 * e2l) fills |= kStagBit;

            if (kFast && near_conv(err2) && (!o.esc_conv_band_last || iters == o.max_iters)) esc = true, FSK_REASON(3);
            if (kFast && near_div(err2)) esc = true, FSK_REASON(11);
            if (c) {
                conv = true;
                break;
            }
            if (kFast && fabs(den) < (R)o.esc_den) esc = true, FSK_REASON(4);
        }
        // the float32 pass hit its iteration cap before max_iters: the f64 pass decides
        if (kFast && !conv && k == limit && limit < o.max_iters && !(err2 > div2)) esc = capped = true, FSK_REASON(5);
        if (kFast && !conv && iters >= o.esc_min_div) esc = true, FSK_REASON(6);
    }
    if (kFast && conv && o.esc_conv_all) esc = true, FSK_REASON(7);
    if (kFast && conv) {  // ill-conditioned root: float32 rounding is amplified into x*
        R m = 0;
#pragma unroll
        for (int e = 0; e < 9; ++e) m = fmax(m, fabs(Ji[e]));
        if (m > (R)o.esc_jmax) esc = true, FSK_REASON(7);
        if ((fills & kStagBit) && m > (R)o.esc_stag_jmax) esc = true, FSK_REASON(13);
        if (fills & kSpikeBit) esc = true, FSK_REASON(15);
        // Step rule: a float64 solve may stop one Broyden step earlier or later than this one
        // when a stop decision sat near conv; the roots then differ by that step. Escalate if
        // the step in question is long: |J~g| (the next step) when err ≥ rho·conv, or the last
        // step when the previous err ≤ conv/rho.
        const R tau2 = (R)o.esc_tau2 * conv2;
        if (err2 >= (R)o.esc_rho2 * conv2) {
            const R s0 = Ji[0] * g0 + Ji[1] * g1 + Ji[2] * g2;
            const R s1 = Ji[3] * g0 + Ji[4] * g1 + Ji[5] * g2;
            const R s2 = Ji[6] * g0 + Ji[7] * g1 + Ji[8] * g2;
            if (s0 * s0 + s1 * s1 + s2 * s2 > tau2) esc = true, FSK_REASON(8);
        }
        if (iters > 0 && e2l * (R)o.esc_rho2 <= conv2) {
            const R d0 = x0 - xl0, d1 = x1 - xl1, d2 = x2 - xl2;
            if (d0 * d0 + d1 * d1 + d2 * d2 > tau2) esc = true, FSK_REASON(9);
        }
        if (o.esc_capconv && iters >= o.esc_cap && o.esc_cap < o.max_iters) {
            // converged on the cap iteration: as long as a capped trajectory
            const R d0 = x0 - xl0, d1 = x1 - xl1, d2 = x2 - xl2;
            if (o.esc_capconv == 1 || d0 * d0 + d1 * d1 + d2 * d2 > tau2) esc = true, FSK_REASON(12);
        }
    }
    return SolveOut{iters, conv, esc, capped, fills & ~(kStagBit | kSpikeBit), reasons};
}

}  // namespace fsk
