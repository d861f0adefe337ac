// fsk_kernels.cuh — sm_100a kernels of the Fast-SNARF deformer hot path.
//
// K1  k_precompute_tgrid   deformer.cpp:61-77 (+ lbs_blend :9-19)          HBM stream
// S*  k_sort_*             spatial (Morton) ordering of the queries         (new; perf only)
// K2  k_search             correspondence.cpp:126-150 + iterate :97-124     FP32 + L1/L2 gather
// D   k_dedup              dedup_roots correspondence.cpp:162-176
// C*  k_scan_* / k_emit    compaction to CorrespondenceSet (correspondence.hpp:29-42)
// K3  k_bwd_*              implicit_grad_approx diff.cpp:43-51, :336-359 (grid-routed)
// GW  k_grad_weights       chain rule through deformer.cpp:70-74
// E   k_eval_points        trilerp_transform / forward_deform / deform_jacobian
//
// Semantics follow SURVEY Appendix A exactly: the cell lookup clamps x to the bbox
// while the affine map is applied to the unclamped x (deformer.cpp:79-94,107-113); the
// initial Jacobian uses the locate_cell_lower cell for the gradient stencil
// (skinning.cpp:122-139,164-193); the divergence test is at the top of each iteration
// (correspondence.cpp:105). The initial Jacobian is formed from the 12-wide transform
// grid instead of the n_b-wide weight grid (equal in real arithmetic).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace fsk {

constexpr int kSortBitsPerAxis = 5;                       // 32^3 Morton buckets
constexpr int kSortBuckets = 1 << (3 * kSortBitsPerAxis);  // 32768

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

struct DenseOut {
    float* x_c;
    float* jinv;
    float* resid;
    uint8_t* iters;
    uint8_t* converged;
    uint8_t* keep;
    int32_t* n_roots;
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

__device__ __forceinline__ void load_T(const float4* __restrict__ tg, int v, float4& r0, float4& r1, float4& r2) {
    const float4* p = tg + 3 * (int64_t)v;
    r0 = __ldg(p);
    r1 = __ldg(p + 1);
    r2 = __ldg(p + 2);
}

// trilerp_transform_into (deformer.cpp:79-94): corner weight = (wz*wy)*wx, k-j-i order.
__device__ __forceinline__ void trilerp_T(const float4* __restrict__ tg, const GridP& g, const Cell& c,
                                          float T[12]) {
#pragma unroll
    for (int e = 0; e < 12; ++e) T[e] = 0.f;
    const int nxy = g.nx * g.ny;
#pragma unroll
    for (int dk = 0; dk < 2; ++dk) {
        const float wz = dk ? c.tz : 1.f - c.tz;
#pragma unroll
        for (int dj = 0; dj < 2; ++dj) {
            const float wyz = wz * (dj ? c.ty : 1.f - c.ty);
#pragma unroll
            for (int di = 0; di < 2; ++di) {
                const float w = wyz * (di ? c.tx : 1.f - c.tx);
                float4 r0, r1, r2;
                load_T(tg, c.base + dk * nxy + dj * g.nx + di, r0, r1, r2);
                T[0] = fmaf(w, r0.x, T[0]); T[1] = fmaf(w, r0.y, T[1]); T[2] = fmaf(w, r0.z, T[2]); T[3] = fmaf(w, r0.w, T[3]);
                T[4] = fmaf(w, r1.x, T[4]); T[5] = fmaf(w, r1.y, T[5]); T[6] = fmaf(w, r1.z, T[6]); T[7] = fmaf(w, r1.w, T[7]);
                T[8] = fmaf(w, r2.x, T[8]); T[9] = fmaf(w, r2.y, T[9]); T[10] = fmaf(w, r2.z, T[10]); T[11] = fmaf(w, r2.w, T[11]);
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

// Analytic Jacobian at x from the transform grid:
//   J = T_lin(p) + Σ_c (T_c x̃) ∇φ_c(p)ᵀ,
// T_lin from the locate_cell cell, ∇φ from the locate_cell_lower cell with ±1/h stencils
// (skinning.cpp:164-193). Also returns T(p) (for d(x)) from the same gathers.
__device__ __forceinline__ void jacobian_and_T(const float4* __restrict__ tg, const GridP& g, float x, float y,
                                               float z, float T[12], float J[9]) {
    const Cell c = locate<false>(g, x, y, z);
    const Cell cl = locate<true>(g, x, y, z);
    const int nxy = g.nx * g.ny;
    const bool same = (c.base == cl.base);
#pragma unroll
    for (int e = 0; e < 12; ++e) T[e] = 0.f;
    float G[9];
#pragma unroll
    for (int e = 0; e < 9; ++e) G[e] = 0.f;
    const float fx[2] = {1.f - cl.tx, cl.tx}, fy[2] = {1.f - cl.ty, cl.ty}, fz[2] = {1.f - cl.tz, cl.tz};
    const float sx[2] = {-g.scale[0], g.scale[0]}, sy[2] = {-g.scale[1], g.scale[1]}, sz[2] = {-g.scale[2], g.scale[2]};
#pragma unroll
    for (int dk = 0; dk < 2; ++dk) {
        const float wz = dk ? c.tz : 1.f - c.tz;
#pragma unroll
        for (int dj = 0; dj < 2; ++dj) {
            const float wyz = wz * (dj ? c.ty : 1.f - c.ty);
#pragma unroll
            for (int di = 0; di < 2; ++di) {
                const float w = wyz * (di ? c.tx : 1.f - c.tx);
                float4 r0, r1, r2;
                load_T(tg, c.base + dk * nxy + dj * g.nx + di, r0, r1, r2);
                T[0] = fmaf(w, r0.x, T[0]); T[1] = fmaf(w, r0.y, T[1]); T[2] = fmaf(w, r0.z, T[2]); T[3] = fmaf(w, r0.w, T[3]);
                T[4] = fmaf(w, r1.x, T[4]); T[5] = fmaf(w, r1.y, T[5]); T[6] = fmaf(w, r1.z, T[6]); T[7] = fmaf(w, r1.w, T[7]);
                T[8] = fmaf(w, r2.x, T[8]); T[9] = fmaf(w, r2.y, T[9]); T[10] = fmaf(w, r2.z, T[10]); T[11] = fmaf(w, r2.w, T[11]);
                if (same) {
                    const float gx = sx[di] * fy[dj] * fz[dk];
                    const float gy = fx[di] * sy[dj] * fz[dk];
                    const float gz = fx[di] * fy[dj] * sz[dk];
                    const float y0 = r0.x * x + r0.y * y + r0.z * z + r0.w;
                    const float y1 = r1.x * x + r1.y * y + r1.z * z + r1.w;
                    const float y2 = r2.x * x + r2.y * y + r2.z * z + r2.w;
                    G[0] = fmaf(y0, gx, G[0]); G[1] = fmaf(y0, gy, G[1]); G[2] = fmaf(y0, gz, G[2]);
                    G[3] = fmaf(y1, gx, G[3]); G[4] = fmaf(y1, gy, G[4]); G[5] = fmaf(y1, gz, G[5]);
                    G[6] = fmaf(y2, gx, G[6]); G[7] = fmaf(y2, gy, G[7]); G[8] = fmaf(y2, gz, G[8]);
                }
            }
        }
    }
    if (!same) {  // x on an interior cell face: gradient from the lower-index cell
#pragma unroll 1
        for (int q = 0; q < 8; ++q) {
            const int di = q & 1, dj = (q >> 1) & 1, dk = q >> 2;
            float4 r0, r1, r2;
            load_T(tg, cl.base + dk * nxy + dj * g.nx + di, r0, r1, r2);
            const float fxi = di ? cl.tx : 1.f - cl.tx, fyj = dj ? cl.ty : 1.f - cl.ty, fzk = dk ? cl.tz : 1.f - cl.tz;
            const float gx = (di ? g.scale[0] : -g.scale[0]) * fyj * fzk;
            const float gy = fxi * (dj ? g.scale[1] : -g.scale[1]) * fzk;
            const float gz = fxi * fyj * (dk ? g.scale[2] : -g.scale[2]);
            const float y0 = r0.x * x + r0.y * y + r0.z * z + r0.w;
            const float y1 = r1.x * x + r1.y * y + r1.z * z + r1.w;
            const float y2 = r2.x * x + r2.y * y + r2.z * z + r2.w;
            G[0] = fmaf(y0, gx, G[0]); G[1] = fmaf(y0, gy, G[1]); G[2] = fmaf(y0, gz, G[2]);
            G[3] = fmaf(y1, gx, G[3]); G[4] = fmaf(y1, gy, G[4]); G[5] = fmaf(y1, gz, G[5]);
            G[6] = fmaf(y2, gx, G[6]); G[7] = fmaf(y2, gy, G[7]); G[8] = fmaf(y2, gz, G[8]);
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

}  // namespace fsk
