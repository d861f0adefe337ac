// fsk_exact.cuh — float64 replay of the reference's operation order (opt-in: FSK_SEARCH_EXACT64).
//
// Broyden trajectories of 25-50 iterations are chaotic even in float64: two implementations
// that round one operation differently (an FMA contraction, (p−lo)·scale instead of
// (p−lo)/ext·(n−1), the transform-grid form of J0 instead of the weight-grid form) part ways
// and may stop at a different root. This path removes every such difference for the solves it
// runs: each operation is an explicit round-to-nearest intrinsic (__dmul_rn / __dadd_rn /
// __dsub_rn / __ddiv_rn, never contracted) in the order of the reference as restated by the
// oracle —
//   locate_cell / locate_cell_lower        skinning.cpp:104-139
//   trilerp_weights_into                   skinning.cpp:141-156
//   weight_spatial_gradient                skinning.cpp:164-193
//   trilerp_transform_into, forward_deform deformer.cpp:79-94, :107-113
//   deform_jacobian (weight-grid form)     deformer.cpp:117-136
//   initial_inverse_jacobian (det, inv)    correspondence.cpp:43-54 (Eigen closed forms)
//   RigidTransform::inverse / apply        geometry.hpp:51-61
//   iterate                                correspondence.cpp:97-124
// so a solve's float64 state is bit-identical to the oracle's (given the same float64 transform
// grid, which k_precompute builds in lbs_blend's order). It needs the weight grid ([V][n_b]
// float32, exactly representable in float64) for J0, like the reference's SearchContext.
#pragma once

#include "fsk_device.cuh"

namespace fsk {
#ifndef FSK_EXACT_PREFETCH
#define FSK_EXACT_PREFETCH 0  // measured slower: refill 0.269 -> 0.297 ms (the L1 data pipe, not latency, binds)
#endif

namespace exact {

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
#ifdef FSK_EXACT_TIMING_NODIV  // timing probe only (not bit-exact): division as a*(1/b)
__device__ __forceinline__ double div(double a, double b) { return a * __drcp_rn(b); }
#else
__device__ __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }
#endif
// The oracle's contraction rule (oracle/fskin_oracle.cpp): every addition whose right operand is a
// product is one fused multiply-add, the reference's -march=native/gnu++20 build contracting its
// scalar code and Eigen accumulating with pmadd:
//   acc + a·b -> fma(a, b, acc);  a0b0 + a1b1 + a2b2 -> fma(a2, b2, fma(a1, b1, a0·b0));  a·b − c·d -> fma(−c, d, a·b)
__device__ __forceinline__ double madd(double acc, double a, double b) { return __fma_rn(a, b, acc); }
__device__ __forceinline__ double msub(double a, double b, double c, double d) { return __fma_rn(-c, d, mul(a, b)); }
// a0*b0 + a1*b1 + a2*b2 (argument order as the round-1 replay: a0 a1 a2 then b0 b1 b2)
__device__ __forceinline__ double dot3(double a0, double a1, double a2, double b0, double b1, double b2) {
    return madd(madd(mul(a0, b0), a1, b1), a2, b2);
}

struct XCell {
    int i, j, k;
    double tx, ty, tz;
};

// locate_cell (skinning.cpp:104-120) / locate_cell_lower (:122-139)
__device__ __forceinline__ XCell locate(const GridP& g, double x0, double x1, double x2, bool lower) {
    const double xs[3] = {x0, x1, x2};
    const int n[3] = {g.nx, g.ny, g.nz};
    int idx[3];
    double t[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        double p = xs[a];
        p = (p < g.lod[a]) ? g.lod[a] : p;  // Aabb::clamp (cwiseMax then cwiseMin)
        p = (p > g.hid[a]) ? g.hid[a] : p;
        const double ext = sub(g.hid[a], g.lod[a]);
        const double u = mul(div(sub(p, g.lod[a]), ext), (double)(n[a] - 1));
        int i = (u == u) ? (int)floor(u) : 0;
        if (lower && i >= 1 && u == (double)i) i -= 1;
        i = i < 0 ? 0 : (i > n[a] - 2 ? n[a] - 2 : i);
        idx[a] = i;
        const double tt = sub(u, (double)i);
        t[a] = tt < 0.0 ? 0.0 : (tt > 1.0 ? 1.0 : tt);
    }
    return XCell{idx[0], idx[1], idx[2], t[0], t[1], t[2]};
}

__device__ __forceinline__ int vidx(const GridP& g, int i, int j, int k) { return (k * g.ny + j) * g.nx + i; }

// Register cache of the first FSK_EXACT_CACHE_ROWS matrix rows of the 4 x-pair edges of one cell
// (the float64 planes' values themselves, so results are unchanged): a Broyden step that stays in
// the cell of the previous evaluation skips those loads. The refill kernel is L1-bound on its
// 768-B gathers; its registers beyond the replay's own ~168 hold the cache.
#ifndef FSK_EXACT_CACHE_ROWS
#define FSK_EXACT_CACHE_ROWS 0
#endif
struct XCache {
    int base = -1;  // vertex index of the cached cell's corner (i, j, k); -1: empty
    V4<double> a[4][FSK_EXACT_CACHE_ROWS > 0 ? FSK_EXACT_CACHE_ROWS : 1], b[4][FSK_EXACT_CACHE_ROWS > 0 ? FSK_EXACT_CACHE_ROWS : 1];
};

// forward_deform(x, tgrid) (deformer.cpp:79-94, :107-113) from the float64 x-pair planes
__device__ __forceinline__ void deform(const Planes<double>& P, const GridP& g, double x0, double x1, double x2,
                                       double d[3], XCache* C = nullptr) {
    const XCell c = locate(g, x0, x1, x2, false);
    const int cbase = vidx(g, c.i, c.j, c.k);
    const bool hit = FSK_EXACT_CACHE_ROWS > 0 && C && C->base == cbase;
#if FSK_EXACT_PREFETCH
    // all 12 corner rows (4 x-pair edges x 3 matrix rows, 64 B each) requested up front, so their L2
    // latencies overlap instead of stalling the accumulate chain edge by edge (no effect on the values)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const int v = vidx(g, c.i, c.j + (e & 1), c.k + (e >> 1));
#pragma unroll
        for (int r = 0; r < 3; ++r)
            asm volatile("prefetch.global.L1 [%0];" ::"l"(P.p + r * P.stride + (int64_t)v * 8));
    }
#endif
    double m[12];
#pragma unroll
    for (int e = 0; e < 12; ++e) m[e] = 0.0;
#ifdef FSK_EXACT_ROW_OUTER
    // row-outer: the entries of row r only read row r of the corners, so processing one row's
    // 4 edges at a time keeps fewer float64 loads in flight (same operations, same bits)
    const double w1x = c.tx, w0x = sub(1.0, c.tx);
    double wyz[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) wyz[e] = mul((e >> 1) ? c.tz : sub(1.0, c.tz), (e & 1) ? c.ty : sub(1.0, c.ty));
#pragma unroll
    for (int r = 0; r < 3; ++r) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            V4<double> a, b;
            load_edge(P, vidx(g, c.i, c.j + (e & 1), c.k + (e >> 1)), r, a, b);
            const double w0 = mul(wyz[e], w0x), w1 = mul(wyz[e], w1x);
            m[4 * r + 0] = madd(m[4 * r + 0], w0, a.x);
            m[4 * r + 1] = madd(m[4 * r + 1], w0, a.y);
            m[4 * r + 2] = madd(m[4 * r + 2], w0, a.z);
            m[4 * r + 3] = madd(m[4 * r + 3], w0, a.w);
            m[4 * r + 0] = madd(m[4 * r + 0], w1, b.x);
            m[4 * r + 1] = madd(m[4 * r + 1], w1, b.y);
            m[4 * r + 2] = madd(m[4 * r + 2], w1, b.z);
            m[4 * r + 3] = madd(m[4 * r + 3], w1, b.w);
        }
    }
#else
#pragma unroll
    for (int dk = 0; dk < 2; ++dk) {
        const double wz = dk ? c.tz : sub(1.0, c.tz);
#pragma unroll
        for (int dj = 0; dj < 2; ++dj) {
            const double wyz = mul(wz, dj ? c.ty : sub(1.0, c.ty));
            const int v = vidx(g, c.i, c.j + dj, c.k + dk);
#pragma unroll
            for (int r = 0; r < 3; ++r) {
                V4<double> a, b;
                if (r < FSK_EXACT_CACHE_ROWS && hit) {
                    a = C->a[2 * dk + dj][r < FSK_EXACT_CACHE_ROWS ? r : 0];
                    b = C->b[2 * dk + dj][r < FSK_EXACT_CACHE_ROWS ? r : 0];
                } else {
                    load_edge(P, v, r, a, b);
                    if (r < FSK_EXACT_CACHE_ROWS && C) {
                        C->a[2 * dk + dj][r < FSK_EXACT_CACHE_ROWS ? r : 0] = a;
                        C->b[2 * dk + dj][r < FSK_EXACT_CACHE_ROWS ? r : 0] = b;
                    }
                }
                const double w0 = mul(wyz, sub(1.0, c.tx)), w1 = mul(wyz, c.tx);
                // corner di = 0 then di = 1, entries in row order (the oracle's e loop per corner;
                // each entry's sum runs over corners in the same (dk, dj, di) order)
                m[4 * r + 0] = madd(m[4 * r + 0], w0, a.x);
                m[4 * r + 1] = madd(m[4 * r + 1], w0, a.y);
                m[4 * r + 2] = madd(m[4 * r + 2], w0, a.z);
                m[4 * r + 3] = madd(m[4 * r + 3], w0, a.w);
                m[4 * r + 0] = madd(m[4 * r + 0], w1, b.x);
                m[4 * r + 1] = madd(m[4 * r + 1], w1, b.y);
                m[4 * r + 2] = madd(m[4 * r + 2], w1, b.z);
                m[4 * r + 3] = madd(m[4 * r + 3], w1, b.w);
            }
        }
    }
#endif
    if (FSK_EXACT_CACHE_ROWS > 0 && C) C->base = cbase;
#pragma unroll
    for (int r = 0; r < 3; ++r) d[r] = add(dot3(m[4 * r], m[4 * r + 1], m[4 * r + 2], x0, x1, x2), m[4 * r + 3]);
}

// x0 = B^-1 x' = Rᵀx' + (−Rᵀt) (geometry.hpp:51-61)
__device__ __forceinline__ void inverse_apply(const double* B, double xp0, double xp1, double xp2, double& x0,
                                              double& x1, double& x2) {
    double R[9], t[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
#pragma unroll
        for (int c = 0; c < 3; ++c) R[3 * r + c] = B[4 * r + c];
        t[r] = B[4 * r + 3];
    }
    double xo[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const double rt = dot3(R[i], R[3 + i], R[6 + i], t[0], t[1], t[2]);  // (Rᵀ t)_i
        xo[i] = add(dot3(R[i], R[3 + i], R[6 + i], xp0, xp1, xp2), -rt);
    }
    x0 = xo[0];
    x1 = xo[1];
    x2 = xo[2];
}

// deform_jacobian(x, grid, bones) via jacobian_from_weights (deformer.cpp:117-136): weights from
// locate_cell (trilerp_weights_into), gradient from locate_cell_lower with ±1/h stencils
// (weight_spatial_gradient), J = Σ_i w_i R_i then + Σ_i (B_i x)(∇w_i)ᵀ, bone order. The
// per-corner factors are bone-independent and computed once (same operations, same bits);
// the weights of 4 consecutive bones come in one 16-byte load when n_b % 4 == 0 (a float64 copy
// of the grid measured slower: the J~0 gathers are L1-bound); the bone transforms are float64
// copies in shared memory.
template <int kVec>
__device__ __forceinline__ void corner_weights(const float* __restrict__ W, int v, int nb, int b, double out[kVec]) {
    const float* q = W + (int64_t)v * nb + b;
    if constexpr (kVec == 4) {
        const float4 w = __ldg(reinterpret_cast<const float4*>(q));
        out[0] = w.x;
        out[1] = w.y;
        out[2] = w.z;
        out[3] = w.w;
    } else {
        out[0] = __ldg(q);
    }
}

template <int kVec>
__device__ __forceinline__ void jacobian_vec(const GridP& g, const float* __restrict__ W, const double* bones,
                                             double x0, double x1, double x2, double J[9]) {
    const int nb = g.nb;
    const XCell c = locate(g, x0, x1, x2, false), cl = locate(g, x0, x1, x2, true);
    const int n[3] = {g.nx, g.ny, g.nz};
    double h[3], dmin[3], dplus[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        h[a] = div(sub(g.hid[a], g.lod[a]), (double)(n[a] - 1));  // cell_size (skinning.cpp:72-75)
        dmin[a] = div(-1.0, h[a]);
        dplus[a] = div(1.0, h[a]);
    }
    int vc[8], vl[8];  // vertex indices (< 2^30)
    double w8[8];
#pragma unroll
    for (int dk = 0; dk < 2; ++dk) {
        const double wz = dk ? c.tz : sub(1.0, c.tz);
#pragma unroll
        for (int dj = 0; dj < 2; ++dj) {
            const double wyz = mul(wz, dj ? c.ty : sub(1.0, c.ty));
#pragma unroll
            for (int di = 0; di < 2; ++di) {
                const int k8 = 4 * dk + 2 * dj + di;
                w8[k8] = mul(wyz, di ? c.tx : sub(1.0, c.tx));
                vc[k8] = vidx(g, c.i + di, c.j + dj, c.k + dk);
                vl[k8] = vidx(g, cl.i + di, cl.j + dj, cl.k + dk);
            }
        }
    }
#pragma unroll
    for (int e = 0; e < 9; ++e) J[e] = 0.0;
    for (int b0 = 0; b0 < nb; b0 += kVec) {  // Σ_i w_i R_i
        double wb[kVec];
#pragma unroll
        for (int u = 0; u < kVec; ++u) wb[u] = 0.0;
#pragma unroll
        for (int k8 = 0; k8 < 8; ++k8) {
            double q[kVec];
            corner_weights<kVec>(W, vc[k8], nb, b0, q);
#pragma unroll
            for (int u = 0; u < kVec; ++u) wb[u] = madd(wb[u], w8[k8], q[u]);
        }
#pragma unroll
        for (int u = 0; u < kVec; ++u) {
            const double* B = bones + 12 * (b0 + u);
#pragma unroll
            for (int r = 0; r < 3; ++r)
#pragma unroll
                for (int cc = 0; cc < 3; ++cc) J[3 * r + cc] = madd(J[3 * r + cc], wb[u], B[4 * r + cc]);
        }
    }
    const double fx[2] = {sub(1.0, cl.tx), cl.tx}, fy[2] = {sub(1.0, cl.ty), cl.ty}, fz[2] = {sub(1.0, cl.tz), cl.tz};
    for (int b0 = 0; b0 < nb; b0 += kVec) {  // + Σ_i (B_i x) ∇w_iᵀ
        double gg[kVec][3];
#pragma unroll
        for (int u = 0; u < kVec; ++u) gg[u][0] = gg[u][1] = gg[u][2] = 0.0;
#pragma unroll
        for (int k8 = 0; k8 < 8; ++k8) {
            const int di = k8 & 1, dj = (k8 >> 1) & 1, dk = k8 >> 2;
            // stencil factors recomputed per bone group (the same operations, fewer live registers)
            const double gx = mul(mul(di ? dplus[0] : dmin[0], fy[dj]), fz[dk]);
            const double gy = mul(mul(fx[di], dj ? dplus[1] : dmin[1]), fz[dk]);
            const double gz = mul(mul(fx[di], fy[dj]), dk ? dplus[2] : dmin[2]);
            double q[kVec];
            corner_weights<kVec>(W, vl[k8], nb, b0, q);
#pragma unroll
            for (int u = 0; u < kVec; ++u) {
                const double v = q[u];
                gg[u][0] = madd(gg[u][0], gx, v);
                gg[u][1] = madd(gg[u][1], gy, v);
                gg[u][2] = madd(gg[u][2], gz, v);
            }
        }
#pragma unroll
        for (int u = 0; u < kVec; ++u) {
            const double* B = bones + 12 * (b0 + u);
            double bx[3];
#pragma unroll
            for (int r = 0; r < 3; ++r)
                bx[r] = add(dot3(B[4 * r], B[4 * r + 1], B[4 * r + 2], x0, x1, x2), B[4 * r + 3]);
#pragma unroll
            for (int r = 0; r < 3; ++r)
#pragma unroll
                for (int cc = 0; cc < 3; ++cc) J[3 * r + cc] = madd(J[3 * r + cc], bx[r], gg[u][cc]);
        }
    }
}

__device__ __forceinline__ void jacobian(const GridP& g, const float* __restrict__ W, const double* bones,
                                         double x0, double x1, double x2, double J[9]) {
    if (g.nb % 4 == 0) jacobian_vec<4>(g, W, bones, x0, x1, x2, J);
    else jacobian_vec<1>(g, W, bones, x0, x1, x2, J);
}

// jacobian() with one pass over the weight grid when both lookups pick the same cell (always,
// unless x lies exactly on an interior cell face): each corner's weights are loaded and widened
// once, feeding both Σ_i w_i R_i (accumulated into J in bone order) and ∇w_i, which is parked in
// shared memory (stash: n_b·3 doubles per thread, strided by blockDim) until the second sum,
// so J is added up in exactly jacobian_vec's order (same operations, same bits).
template <int kVec>
__device__ __noinline__ void jacobian_cold(const GridP& g, const float* __restrict__ W, const double* bones, double x0,
                                           double x1, double x2, double J[9]) {
    jacobian_vec<kVec>(g, W, bones, x0, x1, x2, J);
}

template <int kVec>
__device__ __forceinline__ void jacobian_stash_vec(const GridP& g, const float* __restrict__ W, const double* bones,
                                                   double x0, double x1, double x2, double J[9], double* stash) {
    const int nb = g.nb;
    const XCell c = locate(g, x0, x1, x2, false), cl = locate(g, x0, x1, x2, true);
    if (c.i != cl.i || c.j != cl.j || c.k != cl.k) {
        jacobian_cold<kVec>(g, W, bones, x0, x1, x2, J);  // x on an interior cell face (rare)
        return;
    }
    const int n[3] = {g.nx, g.ny, g.nz};
    double dmin[3], dplus[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double h = div(sub(g.hid[a], g.lod[a]), (double)(n[a] - 1));  // cell_size (skinning.cpp:72-75)
        dmin[a] = div(-1.0, h);
        dplus[a] = div(1.0, h);
    }
    const double fx[2] = {sub(1.0, cl.tx), cl.tx}, fy[2] = {sub(1.0, cl.ty), cl.ty}, fz[2] = {sub(1.0, cl.tz), cl.tz};
    int vc[8];
    double w8[8];
#pragma unroll
    for (int dk = 0; dk < 2; ++dk) {
        const double wz = dk ? c.tz : sub(1.0, c.tz);
#pragma unroll
        for (int dj = 0; dj < 2; ++dj) {
            const double wyz = mul(wz, dj ? c.ty : sub(1.0, c.ty));
#pragma unroll
            for (int di = 0; di < 2; ++di) {
                const int k8 = 4 * dk + 2 * dj + di;
                w8[k8] = mul(wyz, di ? c.tx : sub(1.0, c.tx));
                vc[k8] = vidx(g, c.i + di, c.j + dj, c.k + dk);
            }
        }
    }
    const int ld = blockDim.x;
#pragma unroll
    for (int e = 0; e < 9; ++e) J[e] = 0.0;
    for (int b0 = 0; b0 < nb; b0 += kVec) {
        double wb[kVec], gg[kVec][3];
#pragma unroll
        for (int u = 0; u < kVec; ++u) wb[u] = gg[u][0] = gg[u][1] = gg[u][2] = 0.0;
#pragma unroll
        for (int k8 = 0; k8 < 8; ++k8) {
            const int di = k8 & 1, dj = (k8 >> 1) & 1, dk = k8 >> 2;
            // stencil factors recomputed per bone group (the same operations, fewer live registers)
            const double gx = mul(mul(di ? dplus[0] : dmin[0], fy[dj]), fz[dk]);
            const double gy = mul(mul(fx[di], dj ? dplus[1] : dmin[1]), fz[dk]);
            const double gz = mul(mul(fx[di], fy[dj]), dk ? dplus[2] : dmin[2]);
            double q[kVec];
            corner_weights<kVec>(W, vc[k8], nb, b0, q);
#pragma unroll
            for (int u = 0; u < kVec; ++u) {
                wb[u] = madd(wb[u], w8[k8], q[u]);
                gg[u][0] = madd(gg[u][0], gx, q[u]);
                gg[u][1] = madd(gg[u][1], gy, q[u]);
                gg[u][2] = madd(gg[u][2], gz, q[u]);
            }
        }
#pragma unroll
        for (int u = 0; u < kVec; ++u) {
            const double* B = bones + 12 * (b0 + u);
#pragma unroll
            for (int r = 0; r < 3; ++r)
#pragma unroll
                for (int cc = 0; cc < 3; ++cc) J[3 * r + cc] = madd(J[3 * r + cc], wb[u], B[4 * r + cc]);
#pragma unroll
            for (int cc = 0; cc < 3; ++cc) stash[(3 * (b0 + u) + cc) * ld] = gg[u][cc];
        }
    }
    for (int b = 0; b < nb; ++b) {  // + Σ_i (B_i x) ∇w_iᵀ
        const double* B = bones + 12 * b;
        const double gg0 = stash[(3 * b) * ld], gg1 = stash[(3 * b + 1) * ld], gg2 = stash[(3 * b + 2) * ld];
        double bx[3];
#pragma unroll
        for (int r = 0; r < 3; ++r) bx[r] = add(dot3(B[4 * r], B[4 * r + 1], B[4 * r + 2], x0, x1, x2), B[4 * r + 3]);
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            J[3 * r + 0] = madd(J[3 * r + 0], bx[r], gg0);
            J[3 * r + 1] = madd(J[3 * r + 1], bx[r], gg1);
            J[3 * r + 2] = madd(J[3 * r + 2], bx[r], gg2);
        }
    }
}

// initial_inverse_jacobian (correspondence.cpp:43-54): Eigen's determinant() (expansion along row 0)
// against 1e-8, then Eigen's cofactor inverse with its own det (column-0 cofactors; adjugate · 1/det)
__device__ __forceinline__ void inverse_or_identity(const double a[9], double Ji[9]) {
    auto X = [&](int c1, int c2) { return msub(a[3 + c1], a[6 + c2], a[3 + c2], a[6 + c1]); };
    const double det = madd(madd(mul(a[0], X(1, 2)), -a[1], X(0, 2)), a[2], X(0, 1));  // oracle det3
    if (fabs(det) < 1e-8) {
#pragma unroll
        for (int e = 0; e < 9; ++e) Ji[e] = (e % 4 == 0) ? 1.0 : 0.0;
        return;
    }
    double c[9];
    c[0] = msub(a[4], a[8], a[5], a[7]);
    c[1] = msub(a[2], a[7], a[1], a[8]);
    c[2] = msub(a[1], a[5], a[2], a[4]);
    c[3] = msub(a[5], a[6], a[3], a[8]);
    c[4] = msub(a[0], a[8], a[2], a[6]);
    c[5] = msub(a[2], a[3], a[0], a[5]);
    c[6] = msub(a[3], a[7], a[4], a[6]);
    c[7] = msub(a[1], a[6], a[0], a[7]);
    c[8] = msub(a[0], a[4], a[1], a[3]);
    // Eigen's inverse() takes its own determinant from the column-0 cofactors (InverseImpl.h
    // compute_inverse<.., 3>: cofactors_col0 · col(0))
    const double d2 = madd(madd(mul(c[0], a[0]), c[1], a[3]), c[2], a[6]);
    const double inv = div(1.0, d2);
#pragma unroll
    for (int e = 0; e < 9; ++e) Ji[e] = mul(c[e], inv);
}

__device__ __forceinline__ double norm3(double g0, double g1, double g2) {
    return __dsqrt_rn(dot3(g0, g1, g2, g0, g1, g2));
}

// Solve state of the replay (search_one's per-init body, correspondence.cpp:132-146)
struct XState {
    double x0, x1, x2, g0, g1, g2, err;
    double Ji[9];
    double dx0, dx1, dx2;
    int k;
};

// start: x0, J~0, g0 and err (the converged / diverged decisions are the caller's)
// W: the weight grid; bones: float64 copies of the transforms (shared memory)
__device__ __forceinline__ void start(const Planes<double>& P, const GridP& g, const float* __restrict__ W,
                                      const double* bones, int bone, double xp0, double xp1, double xp2, XState& s,
                                      double* stash = nullptr) {
    inverse_apply(bones + 12 * bone, xp0, xp1, xp2, s.x0, s.x1, s.x2);
    double J[9];
    if (stash) {
        if (g.nb % 4 == 0) jacobian_stash_vec<4>(g, W, bones, s.x0, s.x1, s.x2, J, stash);
        else jacobian_stash_vec<1>(g, W, bones, s.x0, s.x1, s.x2, J, stash);
    } else {
        jacobian(g, W, bones, s.x0, s.x1, s.x2, J);
    }
    inverse_or_identity(J, s.Ji);
    double d[3];
    deform(P, g, s.x0, s.x1, s.x2, d);
    s.g0 = sub(d[0], xp0);
    s.g1 = sub(d[1], xp1);
    s.g2 = sub(d[2], xp2);
    s.err = norm3(s.g0, s.g1, s.g2);
    s.k = 0;
}

// one pass of iterate's loop body after the divergence check (correspondence.cpp:106-122);
// returns true iff converged
__device__ __forceinline__ bool step(const Planes<double>& P, const GridP& g, double xp0, double xp1, double xp2,
                                     double conv_eps, XState& s, XCache* C = nullptr) {
    const double* J = s.Ji;
    const double dx0 = -dot3(J[0], J[1], J[2], s.g0, s.g1, s.g2);
    const double dx1 = -dot3(J[3], J[4], J[5], s.g0, s.g1, s.g2);
    const double dx2 = -dot3(J[6], J[7], J[8], s.g0, s.g1, s.g2);
    s.x0 = add(s.x0, dx0);
    s.x1 = add(s.x1, dx1);
    s.x2 = add(s.x2, dx2);
    double d[3];
    deform(P, g, s.x0, s.x1, s.x2, d, C);
    const double n0 = sub(d[0], xp0), n1 = sub(d[1], xp1), n2 = sub(d[2], xp2);
    const double dg0 = sub(n0, s.g0), dg1 = sub(n1, s.g1), dg2 = sub(n2, s.g2);
    s.g0 = n0;
    s.g1 = n1;
    s.g2 = n2;
    s.k += 1;
    s.err = norm3(n0, n1, n2);
    if (s.err < conv_eps) return true;
    const double j0 = dot3(J[0], J[1], J[2], dg0, dg1, dg2);
    const double j1 = dot3(J[3], J[4], J[5], dg0, dg1, dg2);
    const double j2 = dot3(J[6], J[7], J[8], dg0, dg1, dg2);
    const double den = dot3(dx0, dx1, dx2, j0, j1, j2);
    if (fabs(den) > 1e-18) {
        const double r0 = div(sub(dx0, j0), den), r1 = div(sub(dx1, j1), den), r2 = div(sub(dx2, j2), den);
        const double w0 = dot3(dx0, dx1, dx2, J[0], J[3], J[6]);
        const double w1 = dot3(dx0, dx1, dx2, J[1], J[4], J[7]);
        const double w2 = dot3(dx0, dx1, dx2, J[2], J[5], J[8]);
        const double r[3] = {r0, r1, r2}, w[3] = {w0, w1, w2};
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int c = 0; c < 3; ++c) s.Ji[3 * i + c] = madd(s.Ji[3 * i + c], r[i], w[c]);
    }
    return false;
}

}  // namespace exact
}  // namespace fsk
