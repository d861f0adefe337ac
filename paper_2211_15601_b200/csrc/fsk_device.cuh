// fsk_device.cuh — device-side building blocks of the Fast-SNARF deformer kernels (sm_100a).
//
// Semantics follow SURVEY Appendix A: the cell lookup clamps x to the bbox while the
// affine map is applied to the unclamped x (deformer.cpp:79-94,107-113); the initial
// Jacobian takes its gradient stencil from the locate_cell_lower cell
// (skinning.cpp:122-139,164-193). The Jacobian is formed from the 12-wide transform
// grid instead of the n_b-wide weight grid (equal in real arithmetic).
//
// Gather layout ("x-pair planes"): the reference's [V][12] transform grid is re-laid out
// once per pose into three planes, one per matrix row r, whose element v is 32 bytes:
//     P[r][v] = { row r of T_v , row r of T_{v+1} }      (8 floats)
// so one 256-bit load (LDG.E.ENL2.256, new on sm_100) returns one row of BOTH x-corners of
// a cell edge, and x-neighbouring vertices sit 32 B apart (4 per 128-B line). A trilinear
// evaluation is 12 LDG.256 (4 (dj,dk) edges × 3 rows) instead of 24 LDG.128 in [V][12].
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace fsk {

struct GridP {
    int nx, ny, nz, nb;
    float lo[3], hi[3];
    float scale[3];  // (n-1)/ext: u = (p-lo)*scale; also 1/h for the gradient stencil
};

struct SearchP {
    int max_iters;
    float conv2;  // conv_eps^2
    float div2;   // div_eps^2
    float dedup2;
};

struct Cell {
    int base;  // vertex index of corner (i0, j0, k0)
    float tx, ty, tz;
};

// locate_cell (skinning.cpp:104-120) / locate_cell_lower (:122-139) in float32.
template <bool kLower>
__device__ __forceinline__ Cell locate(const GridP& g, float x, float y, float z) {
    const float xs[3] = {x, y, z};
    const int n[3] = {g.nx, g.ny, g.nz};
    int idx[3];
    float t[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const float p = fminf(fmaxf(xs[a], g.lo[a]), g.hi[a]);  // Aabb::clamp
        const float u = (p - g.lo[a]) * g.scale[a];
        int i = __float2int_rd(u);  // floor; NaN -> 0
        if (kLower && i >= 1 && u == (float)i) i -= 1;
        i = max(0, min(i, n[a] - 2));
        idx[a] = i;
        t[a] = fminf(fmaxf(u - (float)i, 0.f), 1.f);
    }
    Cell c;
    c.base = (idx[2] * g.ny + idx[1]) * g.nx + idx[0];
    c.tx = t[0];
    c.ty = t[1];
    c.tz = t[2];
    return c;
}

// 256-bit read-only load (sm_100: LDG.E.ENL2.256.CONSTANT).
__device__ __forceinline__ void ldg256(const float* p, float4& a, float4& b) {
    asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
        : "l"(p));
}

struct Planes {
    const float* p;   // [3][V][8]
    int64_t stride;   // V*8 floats between row planes
};

__device__ __forceinline__ void load_edge(const Planes& P, int v, int r, float4& a, float4& b) {
    ldg256(P.p + r * P.stride + (int64_t)v * 8, a, b);
}

__device__ __forceinline__ void fma4(float* T, float w, const float4& a) {
    T[0] = fmaf(w, a.x, T[0]);
    T[1] = fmaf(w, a.y, T[1]);
    T[2] = fmaf(w, a.z, T[2]);
    T[3] = fmaf(w, a.w, T[3]);
}

__device__ __forceinline__ float row_dot(const float4& a, float x, float y, float z) {
    return a.x * x + a.y * y + a.z * z + a.w;
}

// trilerp_transform_into (deformer.cpp:79-94) on the x-pair planes. Corner weights are
// formed as (wz*wy)*wx like the reference; accumulation is per (dk, dj) edge.
__device__ __forceinline__ void trilerp_T(const Planes& P, const GridP& g, const Cell& c, float T[12]) {
#pragma unroll
    for (int e = 0; e < 12; ++e) T[e] = 0.f;
    const int nxy = g.nx * g.ny;
#pragma unroll
    for (int dk = 0; dk < 2; ++dk) {
        const float wz = dk ? c.tz : 1.f - c.tz;
#pragma unroll
        for (int dj = 0; dj < 2; ++dj) {
            const float wyz = wz * (dj ? c.ty : 1.f - c.ty);
            const float w0 = wyz * (1.f - c.tx), w1 = wyz * c.tx;
            const int v = c.base + dk * nxy + dj * g.nx;
#pragma unroll
            for (int r = 0; r < 3; ++r) {
                float4 a, b;
                load_edge(P, v, r, a, b);
                fma4(T + 4 * r, w0, a);
                fma4(T + 4 * r, w1, b);
            }
        }
    }
}

// d = T·[x;1] on the unclamped x (deformer.cpp:107-113).
__device__ __forceinline__ void apply_T(const float T[12], float x, float y, float z, float d[3]) {
    d[0] = T[0] * x + T[1] * y + T[2] * z + T[3];
    d[1] = T[4] * x + T[5] * y + T[6] * z + T[7];
    d[2] = T[8] * x + T[9] * y + T[10] * z + T[11];
}

// Gradient-stencil term of one corner: G += (T_c x̃) ∇φ_cᵀ, ∇φ from fractions (fx,fy,fz)
// of the lower cell with ±1/h (skinning.cpp:164-193).
__device__ __forceinline__ void grad_term(float G[9], float y0, float y1, float y2, float gx, float gy, float gz) {
    G[0] = fmaf(y0, gx, G[0]); G[1] = fmaf(y0, gy, G[1]); G[2] = fmaf(y0, gz, G[2]);
    G[3] = fmaf(y1, gx, G[3]); G[4] = fmaf(y1, gy, G[4]); G[5] = fmaf(y1, gz, G[5]);
    G[6] = fmaf(y2, gx, G[6]); G[7] = fmaf(y2, gy, G[7]); G[8] = fmaf(y2, gz, G[8]);
}

// Analytic Jacobian and T(p) at x:
//   J = T_lin(p) + Σ_c (T_c x̃) ∇φ_c(p)ᵀ
// T from the locate_cell cell, ∇φ from the locate_cell_lower cell; both from one gather
// unless x lies exactly on an interior face (then the lower cell is gathered again).
__device__ __forceinline__ void jacobian_and_T(const Planes& P, const GridP& g, float x, float y, float z,
                                               float T[12], float J[9]) {
    const Cell c = locate<false>(g, x, y, z);
    const Cell cl = locate<true>(g, x, y, z);
    const int nxy = g.nx * g.ny;
    const bool same = (c.base == cl.base);
#pragma unroll
    for (int e = 0; e < 12; ++e) T[e] = 0.f;
    float G[9];
#pragma unroll
    for (int e = 0; e < 9; ++e) G[e] = 0.f;
    const float sx = g.scale[0], sy = g.scale[1], sz = g.scale[2];
#pragma unroll
    for (int dk = 0; dk < 2; ++dk) {
        const float wz = dk ? c.tz : 1.f - c.tz;
        const float fz = dk ? cl.tz : 1.f - cl.tz, gz_s = dk ? sz : -sz;
#pragma unroll
        for (int dj = 0; dj < 2; ++dj) {
            const float wyz = wz * (dj ? c.ty : 1.f - c.ty);
            const float w0 = wyz * (1.f - c.tx), w1 = wyz * c.tx;
            const float fy = dj ? cl.ty : 1.f - cl.ty, gy_s = dj ? sy : -sy;
            // ∇φ of the two x-corners of this edge
            const float fx0 = 1.f - cl.tx, fx1 = cl.tx;
            const float g0x = -sx * fy * fz, g0y = fx0 * gy_s * fz, g0z = fx0 * fy * gz_s;
            const float g1x = sx * fy * fz, g1y = fx1 * gy_s * fz, g1z = fx1 * fy * gz_s;
            const int v = c.base + dk * nxy + dj * g.nx;
            float y0[3], y1[3];
#pragma unroll
            for (int r = 0; r < 3; ++r) {
                float4 a, b;
                load_edge(P, v, r, a, b);
                fma4(T + 4 * r, w0, a);
                fma4(T + 4 * r, w1, b);
                y0[r] = row_dot(a, x, y, z);
                y1[r] = row_dot(b, x, y, z);
            }
            if (same) {
                grad_term(G, y0[0], y0[1], y0[2], g0x, g0y, g0z);
                grad_term(G, y1[0], y1[1], y1[2], g1x, g1y, g1z);
            }
        }
    }
    if (!same) {  // x on an interior cell face: gradient from the lower-index cell
#pragma unroll 1
        for (int q = 0; q < 4; ++q) {
            const int dj = q & 1, dk = q >> 1;
            const float fz = dk ? cl.tz : 1.f - cl.tz, gz_s = dk ? sz : -sz;
            const float fy = dj ? cl.ty : 1.f - cl.ty, gy_s = dj ? sy : -sy;
            const float fx0 = 1.f - cl.tx, fx1 = cl.tx;
            const int v = cl.base + dk * nxy + dj * g.nx;
            float y0[3], y1[3];
#pragma unroll
            for (int r = 0; r < 3; ++r) {
                float4 a, b;
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

// initial_inverse_jacobian (correspondence.cpp:43-54): cofactor inverse, identity if |det|<1e-8.
__device__ __forceinline__ void inverse_or_identity(const float J[9], float Ji[9]) {
    const float c00 = J[4] * J[8] - J[5] * J[7];
    const float c01 = J[2] * J[7] - J[1] * J[8];
    const float c02 = J[1] * J[5] - J[2] * J[4];
    const float c10 = J[5] * J[6] - J[3] * J[8];
    const float c11 = J[0] * J[8] - J[2] * J[6];
    const float c12 = J[2] * J[3] - J[0] * J[5];
    const float c20 = J[3] * J[7] - J[4] * J[6];
    const float c21 = J[1] * J[6] - J[0] * J[7];
    const float c22 = J[0] * J[4] - J[1] * J[3];
    const float det = J[0] * c00 + J[1] * c10 + J[2] * c20;
    if (fabsf(det) < 1e-8f) {  // NaN det fails the test and propagates, as in the reference
        Ji[0] = 1.f; Ji[1] = 0.f; Ji[2] = 0.f;
        Ji[3] = 0.f; Ji[4] = 1.f; Ji[5] = 0.f;
        Ji[6] = 0.f; Ji[7] = 0.f; Ji[8] = 1.f;
        return;
    }
    const float inv = 1.f / det;
    Ji[0] = c00 * inv; Ji[1] = c01 * inv; Ji[2] = c02 * inv;
    Ji[3] = c10 * inv; Ji[4] = c11 * inv; Ji[5] = c12 * inv;
    Ji[6] = c20 * inv; Ji[7] = c21 * inv; Ji[8] = c22 * inv;
}

// Per-init start of search_one (correspondence.cpp:135-137): x0 = B_i^-1 x' as
// Rᵀx' + (−Rᵀt) (geometry.hpp:58-61), J~0 = J(x0)^-1 or I (:43-54), and T(x0) for g0.
__device__ __forceinline__ void solve_init(const Planes& P, const GridP& g, const float* __restrict__ B,
                                           float xp0, float xp1, float xp2, float& x0, float& x1, float& x2,
                                           float Ji[9], float T[12]) {
    const float r00 = __ldg(B + 0), r01 = __ldg(B + 1), r02 = __ldg(B + 2), t0 = __ldg(B + 3);
    const float r10 = __ldg(B + 4), r11 = __ldg(B + 5), r12 = __ldg(B + 6), t1 = __ldg(B + 7);
    const float r20 = __ldg(B + 8), r21 = __ldg(B + 9), r22 = __ldg(B + 10), t2 = __ldg(B + 11);
    const float it0 = -(r00 * t0 + r10 * t1 + r20 * t2);
    const float it1 = -(r01 * t0 + r11 * t1 + r21 * t2);
    const float it2 = -(r02 * t0 + r12 * t1 + r22 * t2);
    x0 = r00 * xp0 + r10 * xp1 + r20 * xp2 + it0;
    x1 = r01 * xp0 + r11 * xp1 + r21 * xp2 + it1;
    x2 = r02 * xp0 + r12 * xp1 + r22 * xp2 + it2;
    float Jm[9];
    jacobian_and_T(P, g, x0, x1, x2, T, Jm);
    inverse_or_identity(Jm, Ji);
}

}  // namespace fsk
