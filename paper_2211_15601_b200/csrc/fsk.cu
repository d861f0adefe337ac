// fsk.cu — kernels and C-ABI (include/fsk.h) of the B200-native Fast-SNARF deformer.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 (see build.py).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "fsk.h"
#include "fsk_kernels.cuh"

namespace fsk {

// ============================================================================ K1
// precompute_transform_grid (deformer.cpp:61-77): T_v = Σ_i w_{v,i}·B_i, accumulated in
// bone order like lbs_blend (deformer.cpp:9-19). One thread per vertex; bones staged in
// shared memory; output written as 3 float4 (48 B, coalesced across the warp).
__global__ void __launch_bounds__(256) k_precompute_tgrid(const float* __restrict__ w, const float* __restrict__ bones,
                                                          int nb, int64_t V, float4* __restrict__ tg) {
    extern __shared__ float sB[];
    for (int e = threadIdx.x; e < nb * 12; e += blockDim.x) sB[e] = bones[e];
    __syncthreads();
    const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v >= V) return;
    const float* wv = w + v * nb;
    float T[12];
#pragma unroll
    for (int e = 0; e < 12; ++e) T[e] = 0.f;
    for (int i = 0; i < nb; ++i) {
        const float wi = __ldg(wv + i);
#pragma unroll
        for (int e = 0; e < 12; ++e) T[e] = fmaf(wi, sB[i * 12 + e], T[e]);
    }
    float4* o = tg + 3 * v;
    o[0] = make_float4(T[0], T[1], T[2], T[3]);
    o[1] = make_float4(T[4], T[5], T[6], T[7]);
    o[2] = make_float4(T[8], T[9], T[10], T[11]);
}

// ============================================================================ sort
// Spatial ordering of the queries (performance only; every solve is computed by the
// same instruction sequence wherever it lands, so results are order-independent and
// bitwise deterministic). Counting sort on a 15-bit Morton key of the posed position
// within the points' bounding box: neighbouring lanes then gather neighbouring cells.
__device__ __forceinline__ int f2ord(float f) {
    const int i = __float_as_int(f);
    return i >= 0 ? i : i ^ 0x7fffffff;
}
__device__ __forceinline__ float ord2f(int i) { return __int_as_float(i >= 0 ? i : i ^ 0x7fffffff); }

__global__ void k_sort_init(int* __restrict__ hist, int* __restrict__ bbox) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    for (int i = t; i < kSortBuckets; i += gridDim.x * blockDim.x) hist[i] = 0;
    if (t < 3) {
        bbox[t] = f2ord(INFINITY);
        bbox[3 + t] = f2ord(-INFINITY);
    }
}

__global__ void __launch_bounds__(256) k_sort_bbox(const float* __restrict__ x, int64_t n, int* __restrict__ bbox) {
    float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const float v = x[3 * p + a];
            if (isfinite(v)) {
                lo[a] = fminf(lo[a], v);
                hi[a] = fmaxf(hi[a], v);
            }
        }
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        for (int o = 16; o > 0; o >>= 1) {
            lo[a] = fminf(lo[a], __shfl_xor_sync(0xffffffff, lo[a], o));
            hi[a] = fmaxf(hi[a], __shfl_xor_sync(0xffffffff, hi[a], o));
        }
    }
    if ((threadIdx.x & 31) == 0) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            atomicMin(bbox + a, f2ord(lo[a]));
            atomicMax(bbox + 3 + a, f2ord(hi[a]));
        }
    }
}

__device__ __forceinline__ uint32_t spread3(uint32_t v) {  // 5 bits -> every third bit
    v &= 0x1f;
    v = (v | (v << 8)) & 0x100f;
    v = (v | (v << 4)) & 0x10c3;
    v = (v | (v << 2)) & 0x1249;
    return v;
}

__device__ __forceinline__ uint32_t morton_key(const float* __restrict__ x, int64_t p, const int* __restrict__ bbox) {
    uint32_t q[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const float lo = ord2f(bbox[a]), hi = ord2f(bbox[3 + a]);
        const float s = (float)(1 << kSortBitsPerAxis) / fmaxf(hi - lo, 1e-30f);
        const float u = (x[3 * p + a] - lo) * s;
        const int qi = isfinite(u) ? __float2int_rd(u) : 0;
        q[a] = (uint32_t)max(0, min(qi, (1 << kSortBitsPerAxis) - 1));
    }
    return spread3(q[0]) | (spread3(q[1]) << 1) | (spread3(q[2]) << 2);
}

__global__ void __launch_bounds__(256) k_sort_hist(const float* __restrict__ x, int64_t n, const int* __restrict__ bbox,
                                                   uint16_t* __restrict__ keys, int* __restrict__ hist) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n) return;
    const uint32_t k = morton_key(x, p, bbox);
    keys[p] = (uint16_t)k;
    atomicAdd(hist + k, 1);
}

// Single-block exclusive scan of the 32768 bucket counts (1024 threads × 32).
__global__ void __launch_bounds__(1024) k_sort_scan(int* __restrict__ hist) {
    __shared__ int warp_tot[32];
    constexpr int kPer = kSortBuckets / 1024;
    const int t = threadIdx.x;
    int v[kPer];
    int s = 0;
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
        v[i] = hist[t * kPer + i];
        s += v[i];
    }
    int incl = s;
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffff, incl, o);
        if ((t & 31) >= o) incl += y;
    }
    if ((t & 31) == 31) warp_tot[t >> 5] = incl;
    __syncthreads();
    if (t < 32) {
        int w = warp_tot[t];
        int wi = w;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffff, wi, o);
            if (t >= o) wi += y;
        }
        warp_tot[t] = wi - w;
    }
    __syncthreads();
    int run = warp_tot[t >> 5] + incl - s;
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
        hist[t * kPer + i] = run;
        run += v[i];
    }
}

__global__ void __launch_bounds__(256) k_sort_scatter(const uint16_t* __restrict__ keys, int64_t n, int* __restrict__ offs,
                                                      int* __restrict__ perm) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n) return;
    const int pos = atomicAdd(offs + keys[p], 1);
    perm[pos] = (int)p;
}

// ============================================================================ K2
// One thread per (posed point, bone-init) solve: search_one's per-init body
// (correspondence.cpp:132-146) with iterate (:97-124) in registers. Blocks are
// bone-major (the bone is block-uniform, so B_i^-1 is a broadcast load) over
// spatially sorted points (neighbouring lanes gather neighbouring grid cells).
constexpr int kSearchBlock = 256;

// Per-init start of search_one (correspondence.cpp:135-136): x0 = B_i^-1 x' computed as
// Rᵀx' + (−Rᵀt) (geometry.hpp:58-61), J~0 = J(x0)^-1 or I if |det| < 1e-8 (:43-54).
__device__ __forceinline__ void solve_init(const float4* __restrict__ tg, const GridP& g, const float* __restrict__ B,
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
    jacobian_and_T(tg, g, x0, x1, x2, T, Jm);
    inverse_or_identity(Jm, Ji);
}

// init_states (correspondence.cpp:58-70): one thread per (point, bone), point-major output.
__global__ void __launch_bounds__(256) k_init_states(const float4* __restrict__ tg, GridP g,
                                                     const float* __restrict__ bones, const float* __restrict__ pts,
                                                     int64_t n, float* __restrict__ x0o, float* __restrict__ jo) {
    const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (s >= n * g.nb) return;
    const int64_t p = s / g.nb;
    const int bone = (int)(s - p * g.nb);
    float x0, x1, x2, Ji[9], T[12];
    solve_init(tg, g, bones + 12 * bone, pts[3 * p], pts[3 * p + 1], pts[3 * p + 2], x0, x1, x2, Ji, T);
    if (x0o) {
        x0o[3 * s] = x0;
        x0o[3 * s + 1] = x1;
        x0o[3 * s + 2] = x2;
    }
    if (jo)
        for (int e = 0; e < 9; ++e) jo[9 * s + e] = Ji[e];
}

__global__ void __launch_bounds__(kSearchBlock) k_search(const float4* __restrict__ tg, GridP g,
                                                         const float* __restrict__ bones, const float* __restrict__ pts,
                                                         const int* __restrict__ perm, int64_t n, int blocks_per_bone,
                                                         SearchP o, DenseOut out) {
    const int bone = blockIdx.x / blocks_per_bone;
    const int64_t j = (int64_t)(blockIdx.x - bone * blocks_per_bone) * kSearchBlock + threadIdx.x;
    if (j >= n) return;
    const int64_t p = perm ? (int64_t)__ldg(perm + j) : j;
    const float xp0 = __ldg(pts + 3 * p), xp1 = __ldg(pts + 3 * p + 1), xp2 = __ldg(pts + 3 * p + 2);

    float x0, x1, x2, Ji[9], T[12], d[3];
    solve_init(tg, g, bones + 12 * bone, xp0, xp1, xp2, x0, x1, x2, Ji, T);
    // g0 = d(x0) − x' from the same gather (correspondence.cpp:137)
    apply_T(T, x0, x1, x2, d);
    float g0 = d[0] - xp0, g1 = d[1] - xp1, g2 = d[2] - xp2;
    float err2 = g0 * g0 + g1 * g1 + g2 * g2;

    int iters = 0;
    bool conv = err2 < o.conv2;
    if (!conv) {
        for (int k = 0; k < o.max_iters; ++k) {
            if (err2 > o.div2) break;  // divergence check at the top (:105)
            // dx = −J~ g; x += dx (:106-107)
            const float dx0 = -(Ji[0] * g0 + Ji[1] * g1 + Ji[2] * g2);
            const float dx1 = -(Ji[3] * g0 + Ji[4] * g1 + Ji[5] * g2);
            const float dx2 = -(Ji[6] * g0 + Ji[7] * g1 + Ji[8] * g2);
            x0 += dx0;
            x1 += dx1;
            x2 += dx2;
            // g' = d(x) − x'; dg = g' − g (:108-112)
            const Cell c = locate<false>(g, x0, x1, x2);
            trilerp_T(tg, g, c, T);
            apply_T(T, x0, x1, x2, d);
            const float n0 = d[0] - xp0, n1 = d[1] - xp1, n2 = d[2] - xp2;
            const float dg0 = n0 - g0, dg1 = n1 - g1, dg2 = n2 - g2;
            g0 = n0;
            g1 = n1;
            g2 = n2;
            iters = k + 1;
            err2 = g0 * g0 + g1 * g1 + g2 * g2;
            if (err2 < o.conv2) {
                conv = true;
                break;
            }
            // Good Broyden: J~ += ((dx − J~dg)/(dx·J~dg)) (dxᵀJ~) if |den| > 1e-18 (:118-122)
            const float j0 = Ji[0] * dg0 + Ji[1] * dg1 + Ji[2] * dg2;
            const float j1 = Ji[3] * dg0 + Ji[4] * dg1 + Ji[5] * dg2;
            const float j2 = Ji[6] * dg0 + Ji[7] * dg1 + Ji[8] * dg2;
            const float den = dx0 * j0 + dx1 * j1 + dx2 * j2;
            if (fabsf(den) > 1e-18f) {
                const float inv = 1.f / den;
                const float q0 = (dx0 - j0) * inv, q1 = (dx1 - j1) * inv, q2 = (dx2 - j2) * inv;
                const float w0 = dx0 * Ji[0] + dx1 * Ji[3] + dx2 * Ji[6];
                const float w1 = dx0 * Ji[1] + dx1 * Ji[4] + dx2 * Ji[7];
                const float w2 = dx0 * Ji[2] + dx1 * Ji[5] + dx2 * Ji[8];
                Ji[0] = fmaf(q0, w0, Ji[0]); Ji[1] = fmaf(q0, w1, Ji[1]); Ji[2] = fmaf(q0, w2, Ji[2]);
                Ji[3] = fmaf(q1, w0, Ji[3]); Ji[4] = fmaf(q1, w1, Ji[4]); Ji[5] = fmaf(q1, w2, Ji[5]);
                Ji[6] = fmaf(q2, w0, Ji[6]); Ji[7] = fmaf(q2, w1, Ji[7]); Ji[8] = fmaf(q2, w2, Ji[8]);
            }
        }
    }

    const int64_t s = p * g.nb + bone;
    if (out.x_c) {
        out.x_c[3 * s] = x0;
        out.x_c[3 * s + 1] = x1;
        out.x_c[3 * s + 2] = x2;
    }
    if (out.jinv) {
#pragma unroll
        for (int e = 0; e < 9; ++e) out.jinv[9 * s + e] = Ji[e];
    }
    if (out.resid) out.resid[s] = sqrtf(err2);
    if (out.iters) out.iters[s] = (uint8_t)iters;
    out.converged[s] = conv ? 1 : 0;
}

// ============================================================================ dedup
// dedup_roots (correspondence.cpp:162-176) over each point's converged inits in bone
// order: kept iff ||x − k|| >= dedup_dist for every already-kept k (strict '<' drops).
__global__ void __launch_bounds__(256) k_dedup(int64_t n, int nb, float dedup2, const float* __restrict__ x_c,
                                               const uint8_t* __restrict__ conv, uint8_t* __restrict__ keep,
                                               int32_t* __restrict__ n_roots) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n) return;
    const float* xp = x_c + p * nb * 3;
    const uint8_t* cp = conv + p * nb;
    uint8_t* kp = keep + p * nb;
    int count = 0;
    for (int i = 0; i < nb; ++i) {
        int k = 0;
        if (cp[i]) {
            const float a0 = xp[3 * i], a1 = xp[3 * i + 1], a2 = xp[3 * i + 2];
            k = 1;
            for (int q = 0; q < i; ++q) {
                if (!kp[q]) continue;
                const float e0 = a0 - xp[3 * q], e1 = a1 - xp[3 * q + 1], e2 = a2 - xp[3 * q + 2];
                if (e0 * e0 + e1 * e1 + e2 * e2 < dedup2) {
                    k = 0;
                    break;
                }
            }
        }
        kp[i] = (uint8_t)k;
        count += k;
    }
    if (n_roots) n_roots[p] = count;
}

// ============================================================================ scan (int32 -> int64 exclusive)
constexpr int kScanThreads = 1024, kScanPer = 4, kScanTile = kScanThreads * kScanPer;

__device__ __forceinline__ int64_t block_excl_scan(int64_t v, int64_t* warp_tot, int64_t* total) {
    const int t = threadIdx.x;
    int64_t incl = v;
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffff, incl, o);
        if ((t & 31) >= o) incl += y;
    }
    if ((t & 31) == 31) warp_tot[t >> 5] = incl;
    __syncthreads();
    if (t < 32) {
        const int64_t w = warp_tot[t];
        int64_t wi = w;
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t y = __shfl_up_sync(0xffffffff, wi, o);
            if (t >= o) wi += y;
        }
        warp_tot[t] = wi - w;
        if (t == 31) *total = wi;
    }
    __syncthreads();
    const int64_t r = warp_tot[t >> 5] + incl - v;
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_partial(const int32_t* __restrict__ in, int64_t n,
                                                               int64_t* __restrict__ part) {
    __shared__ int64_t wt[32];
    __shared__ int64_t tot;
    const int64_t base = blockIdx.x * (int64_t)kScanTile + threadIdx.x * kScanPer;
    int64_t s = 0;
#pragma unroll
    for (int i = 0; i < kScanPer; ++i)
        if (base + i < n) s += in[base + i];
    block_excl_scan(s, wt, &tot);
    if (threadIdx.x == 0) part[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_top(int64_t* __restrict__ part, int64_t nparts) {
    __shared__ int64_t wt[32];
    __shared__ int64_t tot;
    int64_t carry = 0;
    for (int64_t b0 = 0; b0 < nparts; b0 += kScanThreads) {
        const int64_t i = b0 + threadIdx.x;
        const int64_t v = i < nparts ? part[i] : 0;
        const int64_t e = block_excl_scan(v, wt, &tot);
        if (i < nparts) part[i] = carry + e;
        carry += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) part[nparts] = carry;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_apply(const int32_t* __restrict__ in, int64_t n,
                                                             const int64_t* __restrict__ part,
                                                             int64_t* __restrict__ out) {
    __shared__ int64_t wt[32];
    __shared__ int64_t tot;
    const int64_t base = blockIdx.x * (int64_t)kScanTile + threadIdx.x * kScanPer;
    int64_t v[kScanPer];
    int64_t s = 0;
#pragma unroll
    for (int i = 0; i < kScanPer; ++i) {
        v[i] = (base + i < n) ? in[base + i] : 0;
        s += v[i];
    }
    int64_t run = part[blockIdx.x] + block_excl_scan(s, wt, &tot);
#pragma unroll
    for (int i = 0; i < kScanPer; ++i) {
        if (base + i < n) out[base + i] = run;
        run += v[i];
    }
    const int64_t nblocks = n > 0 ? (n + kScanTile - 1) / kScanTile : 1;
    if (blockIdx.x == nblocks - 1 && threadIdx.x == 0) out[n] = part[nblocks];
}

// Emit the kept roots of each point in bone order (CorrespondenceSet::roots).
__global__ void __launch_bounds__(256) k_emit(int64_t n, int nb, DenseOut d, const int64_t* __restrict__ offs,
                                              fsk_root* __restrict__ roots) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n) return;
    int64_t o = offs[p];
    for (int i = 0; i < nb; ++i) {
        const int64_t s = p * nb + i;
        if (!d.keep[s]) continue;
        fsk_root r;
        r.x[0] = d.x_c[3 * s];
        r.x[1] = d.x_c[3 * s + 1];
        r.x[2] = d.x_c[3 * s + 2];
        r.residual = d.resid ? d.resid[s] : 0.f;
#pragma unroll
        for (int e = 0; e < 9; ++e) r.inv_jacobian[e] = d.jinv ? d.jinv[9 * s + e] : 0.f;
        r.source_bone = i;
        r.iterations = d.iters ? d.iters[s] : 0;
        r._pad = 0;
        float4* dst = reinterpret_cast<float4*>(roots + o);
        const float4* src = reinterpret_cast<const float4*>(&r);
#pragma unroll
        for (int q = 0; q < 4; ++q) dst[q] = src[q];
        ++o;
    }
}

// ============================================================================ K3
// implicit_grad_approx (diff.cpp:43-51) routed to the grid: u = −J~ᵀ v (diff.cpp:351),
// dL/dT_c += φ_c(x*) · u (x*,1)ᵀ for the 8 corners of locate_cell(x*).
__device__ __forceinline__ bool bwd_load(int64_t p, int n_init, const float* __restrict__ x_c,
                                         const float* __restrict__ jinv, const float* __restrict__ gx,
                                         const int32_t* __restrict__ sel, float xs[3], float u[3]) {
    const int sidx = sel[p];
    if (sidx < 0 || sidx >= n_init) return false;
    const int64_t s = p * n_init + sidx;
    const float* J = jinv + 9 * s;
    const float v0 = gx[3 * p], v1 = gx[3 * p + 1], v2 = gx[3 * p + 2];
    u[0] = -(J[0] * v0 + J[3] * v1 + J[6] * v2);
    u[1] = -(J[1] * v0 + J[4] * v1 + J[7] * v2);
    u[2] = -(J[2] * v0 + J[5] * v1 + J[8] * v2);
    xs[0] = x_c[3 * s];
    xs[1] = x_c[3 * s + 1];
    xs[2] = x_c[3 * s + 2];
    return true;
}

__global__ void k_zero(float4* __restrict__ p, int64_t n4) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = make_float4(0.f, 0.f, 0.f, 0.f);
}

__global__ void __launch_bounds__(256) k_bwd_scatter(GridP g, int n_init, const float* __restrict__ x_c,
                                                     const float* __restrict__ jinv, const float* __restrict__ gx,
                                                     const int32_t* __restrict__ sel, int64_t n,
                                                     float4* __restrict__ gT) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n) return;
    float xs[3], u[3];
    if (!bwd_load(p, n_init, x_c, jinv, gx, sel, xs, u)) return;
    const Cell c = locate<false>(g, xs[0], xs[1], xs[2]);
    const int nxy = g.nx * g.ny;
#pragma unroll
    for (int dk = 0; dk < 2; ++dk) {
        const float wz = dk ? c.tz : 1.f - c.tz;
#pragma unroll
        for (int dj = 0; dj < 2; ++dj) {
            const float wyz = wz * (dj ? c.ty : 1.f - c.ty);
#pragma unroll
            for (int di = 0; di < 2; ++di) {
                const float phi = wyz * (di ? c.tx : 1.f - c.tx);
                float4* dst = gT + 3 * (int64_t)(c.base + dk * nxy + dj * g.nx + di);
#pragma unroll
                for (int r = 0; r < 3; ++r) {
                    const float a = phi * u[r];
                    atomicAdd(dst + r, make_float4(a * xs[0], a * xs[1], a * xs[2], a));
                }
            }
        }
    }
}

// Deterministic mode: every term is rounded to int64 fixed point with a data-derived
// power-of-two scale and accumulated with integer atomics (associative ⇒ bitwise
// reproducible for any launch order / GPU count).
__global__ void __launch_bounds__(256) k_bwd_maxterm(int n_init, const float* __restrict__ x_c,
                                                     const float* __restrict__ jinv, const float* __restrict__ gx,
                                                     const int32_t* __restrict__ sel, int64_t n,
                                                     unsigned int* __restrict__ maxbits) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    float m = 0.f;
    if (p < n) {
        float xs[3], u[3];
        if (bwd_load(p, n_init, x_c, jinv, gx, sel, xs, u)) {
            const float mu = fmaxf(fabsf(u[0]), fmaxf(fabsf(u[1]), fabsf(u[2])));
            const float mx = fmaxf(1.f, fmaxf(fabsf(xs[0]), fmaxf(fabsf(xs[1]), fabsf(xs[2]))));
            m = mu * mx;
            if (!isfinite(m)) m = 3.0e38f;
        }
    }
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffff, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(maxbits, __float_as_uint(m));  // m >= 0: bit order == value order
}

__device__ __forceinline__ double fixed_scale(unsigned int maxbits, int64_t n) {
    const double m = (double)__uint_as_float(maxbits) * (double)(n > 0 ? n : 1);
    if (!(m > 0.0)) return 1.0;
    const int e = (int)floor(log2(m));
    return ldexp(1.0, 61 - e);  // n·max|term|·scale < 2^62
}

__global__ void __launch_bounds__(256) k_bwd_scatter_fixed(GridP g, int n_init, const float* __restrict__ x_c,
                                                           const float* __restrict__ jinv, const float* __restrict__ gx,
                                                           const int32_t* __restrict__ sel, int64_t n,
                                                           const unsigned int* __restrict__ maxbits,
                                                           unsigned long long* __restrict__ acc) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n) return;
    float xs[3], u[3];
    if (!bwd_load(p, n_init, x_c, jinv, gx, sel, xs, u)) return;
    const double scale = fixed_scale(*maxbits, n);
    const Cell c = locate<false>(g, xs[0], xs[1], xs[2]);
    const int nxy = g.nx * g.ny;
    const double xt[4] = {xs[0], xs[1], xs[2], 1.0};
    for (int q = 0; q < 8; ++q) {
        const int di = q & 1, dj = (q >> 1) & 1, dk = q >> 2;
        const float phi = ((dk ? c.tz : 1.f - c.tz) * (dj ? c.ty : 1.f - c.ty)) * (di ? c.tx : 1.f - c.tx);
        unsigned long long* dst = acc + 12 * (int64_t)(c.base + dk * nxy + dj * g.nx + di);
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            const double a = (double)phi * (double)u[r] * scale;
#pragma unroll
            for (int col = 0; col < 4; ++col)
                atomicAdd(dst + 4 * r + col, (unsigned long long)__double2ll_rn(a * xt[col]));
        }
    }
}

__global__ void k_bwd_fixed_to_float(const long long* __restrict__ acc, int64_t m, const unsigned int* __restrict__ maxbits,
                                     int64_t n, float* __restrict__ out) {
    const double inv = 1.0 / fixed_scale(*maxbits, n);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (float)((double)acc[i] * inv);
}

// ============================================================================ GW
// dL/dw[v][i] = Σ_e dL/dT[v][e] · B_i[e]  (T_v = Σ_i w_{v,i} B_i, deformer.cpp:70-74).
// Tile of 128 vertices staged in shared memory so the [V][n_b] store is coalesced.
constexpr int kGwTile = 128;
__global__ void __launch_bounds__(kGwTile) k_grad_weights(const float* __restrict__ gT, const float* __restrict__ bones,
                                                          int nb, int64_t V, float* __restrict__ gw) {
    extern __shared__ float sm[];
    float* sB = sm;                 // nb*12
    float* sO = sm + nb * 12;       // kGwTile*nb
    for (int e = threadIdx.x; e < nb * 12; e += blockDim.x) sB[e] = bones[e];
    __syncthreads();
    const int64_t v0 = blockIdx.x * (int64_t)kGwTile;
    const int64_t v = v0 + threadIdx.x;
    if (v < V) {
        float G[12];
        const float4* src = reinterpret_cast<const float4*>(gT) + 3 * v;
        const float4 a = src[0], b = src[1], c = src[2];
        G[0] = a.x; G[1] = a.y; G[2] = a.z; G[3] = a.w; G[4] = b.x; G[5] = b.y;
        G[6] = b.z; G[7] = b.w; G[8] = c.x; G[9] = c.y; G[10] = c.z; G[11] = c.w;
        for (int i = 0; i < nb; ++i) {
            float s = 0.f;
#pragma unroll
            for (int e = 0; e < 12; ++e) s = fmaf(G[e], sB[i * 12 + e], s);
            sO[threadIdx.x * nb + i] = s;
        }
    }
    __syncthreads();
    const int64_t cnt = min((int64_t)kGwTile, V - v0) * nb;
    for (int64_t e = threadIdx.x; e < cnt; e += blockDim.x) gw[v0 * nb + e] = sO[e];
}

// ============================================================================ E
__global__ void __launch_bounds__(256) k_eval_points(const float4* __restrict__ tg, GridP g, const float* __restrict__ x,
                                                     int64_t n, float* __restrict__ t12, float* __restrict__ dout,
                                                     float* __restrict__ jac) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n) return;
    const float x0 = x[3 * p], x1 = x[3 * p + 1], x2 = x[3 * p + 2];
    float T[12], J[9], d[3];
    jacobian_and_T(tg, g, x0, x1, x2, T, J);
    apply_T(T, x0, x1, x2, d);
    if (t12)
        for (int e = 0; e < 12; ++e) t12[12 * p + e] = T[e];
    if (dout)
        for (int e = 0; e < 3; ++e) dout[3 * p + e] = d[e];
    if (jac)
        for (int e = 0; e < 9; ++e) jac[9 * p + e] = J[e];
}

}  // namespace fsk

// ################################################################################ C-ABI
using namespace fsk;

struct fsk_ctx {
    int device = 0;
    int sm_count = 0;
    int64_t launches = 0;
    // optional per-launch CUDA-event profiling (bench.py reads per-kernel device time)
    bool prof_on = false;
    cudaEvent_t pending = nullptr;
    struct Rec {
        const char* name;
        cudaEvent_t a, b;
    };
    std::vector<Rec> prof;
    std::vector<cudaEvent_t> pool;
    // growable device scratch
    void* buf[16] = {};
    size_t cap[16] = {};
};

namespace {

thread_local std::string g_err;

enum Slot {
    kHist, kBbox, kKeys, kPerm, kScanPart, kBwdAcc, kBwdMax,
    kHW, kHB, kHP, kHT, kHDense, kHOffs, kHRoots, kHNroots, kSlots
};

struct Error {
    int code;
    std::string msg;
};

[[noreturn]] void fail(int code, const std::string& m) { throw Error{code, m}; }

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(FSK_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename Fn>
int guard(Fn&& fn) {
    try {
        fn();
        return FSK_OK;
    } catch (const Error& e) {
        g_err = e.msg;
        return e.code;
    } catch (const std::exception& e) {
        g_err = e.what();
        return FSK_ECUDA;
    }
}

void* scratch(fsk_ctx* ctx, int slot, size_t bytes) {
    if (bytes == 0) bytes = 16;
    if (ctx->cap[slot] < bytes) {
        if (ctx->buf[slot]) cuda_check(cudaFree(ctx->buf[slot]), "cudaFree");
        ctx->buf[slot] = nullptr;
        ctx->cap[slot] = 0;
        const size_t b = bytes + bytes / 8;
        cuda_check(cudaMalloc(&ctx->buf[slot], b), "cudaMalloc");
        ctx->cap[slot] = b;
    }
    return ctx->buf[slot];
}

void set_device(fsk_ctx* ctx) {
    if (!ctx) fail(FSK_EINVAL, "fsk: null context");
    cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
}

cudaEvent_t pooled_event(fsk_ctx* ctx) {
    if (!ctx->pool.empty()) {
        cudaEvent_t e = ctx->pool.back();
        ctx->pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cuda_check(cudaEventCreate(&e), "cudaEventCreate");
    return e;
}

cudaStream_t g_prof_stream = nullptr;

void prof_begin(fsk_ctx* ctx, cudaStream_t st) {
    if (!ctx->prof_on) return;
    ctx->pending = pooled_event(ctx);
    g_prof_stream = st;
    cuda_check(cudaEventRecord(ctx->pending, st), "cudaEventRecord");
}

void after_launch(fsk_ctx* ctx, const char* name) {
    ctx->launches++;
    cuda_check(cudaGetLastError(), name);
    if (ctx->prof_on && ctx->pending) {
        cudaEvent_t b = pooled_event(ctx);
        cuda_check(cudaEventRecord(b, g_prof_stream), "cudaEventRecord");
        ctx->prof.push_back({name, ctx->pending, b});
        ctx->pending = nullptr;
    }
}

GridP make_grid(const fsk_grid_desc* d) {
    if (!d) fail(FSK_EINVAL, "fsk: null grid descriptor");
    if (d->nx < 2 || d->ny < 2 || d->nz < 2) fail(FSK_EINVAL, "SkinningVoxelGrid: dims must be >= 2 per axis");
    if (d->n_bones < 1) fail(FSK_EINVAL, "SkinningVoxelGrid: n_bones must be >= 1");
    GridP g;
    g.nx = d->nx;
    g.ny = d->ny;
    g.nz = d->nz;
    g.nb = d->n_bones;
    const int n[3] = {d->nx, d->ny, d->nz};
    for (int a = 0; a < 3; ++a) {
        g.lo[a] = d->bbox_min[a];
        g.hi[a] = d->bbox_max[a];
        const float ext = g.hi[a] - g.lo[a];
        if (!(ext > 0.f)) fail(FSK_EINVAL, "SkinningVoxelGrid: bbox must have positive extent");
        g.scale[a] = (float)((double)(n[a] - 1) / (double)ext);
    }
    if ((int64_t)d->nx * d->ny * d->nz >= (int64_t(1) << 31)) fail(FSK_EINVAL, "fsk: grid too large (>= 2^31 vertices)");
    return g;
}

SearchP make_search(const fsk_search_opts* o) {
    if (!o) fail(FSK_EINVAL, "fsk: null search options");
    // SearchOptions::validate (correspondence.cpp:19-25)
    if (o->max_iters < 1) fail(FSK_EINVAL, "search: max_iters must be >= 1");
    if (!(o->conv_eps > 0.f)) fail(FSK_EINVAL, "search: conv_eps must be > 0");
    if (!(o->div_eps > o->conv_eps)) fail(FSK_EINVAL, "search: div_eps must exceed conv_eps");
    if (!(o->dedup_dist >= 0.f)) fail(FSK_EINVAL, "search: dedup_dist must be >= 0");
    if (o->max_iters > 255) fail(FSK_EINVAL, "fsk: max_iters must be <= 255 (uint8 iteration counts)");
    SearchP s;
    s.max_iters = o->max_iters;
    s.conv2 = (float)((double)o->conv_eps * (double)o->conv_eps);
    s.div2 = (float)((double)o->div_eps * (double)o->div_eps);
    s.dedup2 = (float)((double)o->dedup_dist * (double)o->dedup_dist);
    return s;
}

inline unsigned blocks_for(int64_t n, int t) { return (unsigned)std::max<int64_t>(1, (n + t - 1) / t); }

void run_precompute(fsk_ctx* ctx, const float* w, const GridP& g, const float* bones, float* tg, cudaStream_t st) {
    const int64_t V = (int64_t)g.nx * g.ny * g.nz;
    prof_begin(ctx, st);
    k_precompute_tgrid<<<blocks_for(V, 256), 256, g.nb * 12 * sizeof(float), st>>>(w, bones, g.nb, V,
                                                                                  reinterpret_cast<float4*>(tg));
    after_launch(ctx, "k_precompute_tgrid");
}

void run_search(fsk_ctx* ctx, const float* tg, const GridP& g, const float* bones, const float* pts, int64_t n,
                const SearchP& sp, int flags, const DenseOut& d, cudaStream_t st) {
    if (n == 0) return;
    if (n >= (int64_t(1) << 31) / std::max(1, g.nb)) fail(FSK_EINVAL, "fsk: too many points for one call (split the batch)");
    const int* perm = nullptr;
    if (!(flags & FSK_SEARCH_NO_SORT)) {
        int* hist = (int*)scratch(ctx, kHist, kSortBuckets * sizeof(int));
        int* bbox = (int*)scratch(ctx, kBbox, 6 * sizeof(int));
        uint16_t* keys = (uint16_t*)scratch(ctx, kKeys, n * sizeof(uint16_t));
        int* pm = (int*)scratch(ctx, kPerm, n * sizeof(int));
        prof_begin(ctx, st);
        k_sort_init<<<32, 1024, 0, st>>>(hist, bbox);
        after_launch(ctx, "k_sort_init");
        const unsigned gb = (unsigned)std::min<int64_t>(blocks_for(n, 256), (int64_t)ctx->sm_count * 8);
        prof_begin(ctx, st);
        k_sort_bbox<<<gb, 256, 0, st>>>(pts, n, bbox);
        after_launch(ctx, "k_sort_bbox");
        prof_begin(ctx, st);
        k_sort_hist<<<blocks_for(n, 256), 256, 0, st>>>(pts, n, bbox, keys, hist);
        after_launch(ctx, "k_sort_hist");
        prof_begin(ctx, st);
        k_sort_scan<<<1, 1024, 0, st>>>(hist);
        after_launch(ctx, "k_sort_scan");
        prof_begin(ctx, st);
        k_sort_scatter<<<blocks_for(n, 256), 256, 0, st>>>(keys, n, hist, pm);
        after_launch(ctx, "k_sort_scatter");
        perm = pm;
    }
    const int bpb = (int)blocks_for(n, kSearchBlock);
    const int64_t nblocks = (int64_t)bpb * g.nb;
    if (nblocks >= (int64_t(1) << 31)) fail(FSK_EINVAL, "fsk: search grid too large");
    prof_begin(ctx, st);
    k_search<<<(unsigned)nblocks, kSearchBlock, 0, st>>>(reinterpret_cast<const float4*>(tg), g, bones, pts, perm, n,
                                                         bpb, sp, d);
    after_launch(ctx, "k_search");
    if (d.keep) {
        prof_begin(ctx, st);
        k_dedup<<<blocks_for(n, 256), 256, 0, st>>>(n, g.nb, sp.dedup2, d.x_c, d.converged, d.keep, d.n_roots);
        after_launch(ctx, "k_dedup");
    }
}

void run_scan(fsk_ctx* ctx, const int32_t* in, int64_t n, int64_t* out, cudaStream_t st) {
    const int64_t nb = std::max<int64_t>(1, (n + kScanTile - 1) / kScanTile);
    int64_t* part = (int64_t*)scratch(ctx, kScanPart, (nb + 1) * sizeof(int64_t));
    prof_begin(ctx, st);
    k_scan_partial<<<(unsigned)nb, kScanThreads, 0, st>>>(in, n, part);
    after_launch(ctx, "k_scan_partial");
    prof_begin(ctx, st);
    k_scan_top<<<1, kScanThreads, 0, st>>>(part, nb);
    after_launch(ctx, "k_scan_top");
    prof_begin(ctx, st);
    k_scan_apply<<<(unsigned)nb, kScanThreads, 0, st>>>(in, n, part, out);
    after_launch(ctx, "k_scan_apply");
}

void check_dense(const fsk_search_out* o, bool need_keep) {
    if (!o) fail(FSK_EINVAL, "fsk: null search output");
    if (!o->converged) fail(FSK_EINVAL, "fsk: search output needs a converged mask");
    if (need_keep && (!o->keep || !o->x_c || !o->n_roots))
        fail(FSK_EINVAL, "fsk: compaction needs x_c, keep and n_roots");
}

DenseOut to_dense(const fsk_search_out* o) {
    return DenseOut{o->x_c, o->jinv, o->resid, o->iters, o->converged, o->keep, o->n_roots};
}

}  // namespace

extern "C" {

const char* fsk_last_error(void) { return g_err.c_str(); }

int fsk_ctx_create(int device, fsk_ctx** out) {
    return guard([&] {
        if (!out) fail(FSK_EINVAL, "fsk: null output pointer");
        *out = nullptr;
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
            cudaGetLastError();
            fail(FSK_ENODEV, "fsk: no CUDA device available (this library has no CPU fallback)");
        }
        if (device < 0 || device >= n) fail(FSK_EINVAL, "fsk: device ordinal out of range");
        cudaDeviceProp prop;
        cuda_check(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
        if (prop.major != 10) fail(FSK_ENODEV, std::string("fsk: built for sm_100a, device is ") + prop.name);
        auto* c = new fsk_ctx();
        c->device = device;
        c->sm_count = prop.multiProcessorCount;
        *out = c;
    });
}

int fsk_ctx_destroy(fsk_ctx* ctx) {
    return guard([&] {
        if (!ctx) return;
        cudaSetDevice(ctx->device);
        for (auto& b : ctx->buf)
            if (b) cudaFree(b);
        for (auto& r : ctx->prof) {
            cudaEventDestroy(r.a);
            cudaEventDestroy(r.b);
        }
        for (auto& e : ctx->pool) cudaEventDestroy(e);
        delete ctx;
    });
}

int64_t fsk_ctx_launch_count(const fsk_ctx* ctx) { return ctx ? ctx->launches : -1; }

int fsk_ctx_set_profiling(fsk_ctx* ctx, int on) {
    return guard([&] {
        set_device(ctx);
        ctx->prof_on = on != 0;
    });
}

int fsk_ctx_prof_read(fsk_ctx* ctx, const char* name, double* total_ms, int64_t* count, int reset) {
    return guard([&] {
        set_device(ctx);
        if (!total_ms || !count) fail(FSK_EINVAL, "fsk: null output pointer");
        double t = 0.0;
        int64_t c = 0;
        for (auto& r : ctx->prof) {
            if (name && std::strcmp(name, r.name) != 0) continue;
            cuda_check(cudaEventSynchronize(r.b), "cudaEventSynchronize");
            float ms = 0.f;
            cuda_check(cudaEventElapsedTime(&ms, r.a, r.b), "cudaEventElapsedTime");
            t += ms;
            ++c;
        }
        *total_ms = t;
        *count = c;
        if (reset) {
            for (auto& r : ctx->prof) {
                cuda_check(cudaEventSynchronize(r.b), "cudaEventSynchronize");
                ctx->pool.push_back(r.a);
                ctx->pool.push_back(r.b);
            }
            ctx->prof.clear();
        }
    });
}

// FFMA throughput microbenchmark: the FP32 roofline denominator, measured live on the box.
namespace {
__global__ void __launch_bounds__(256) k_peak_fp32(float* out, int iters, float a, float b) {
    float x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3f + i;
    for (int k = 0; k < iters; ++k) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], a, b);
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.678f) out[0] = s;  // keep the chains alive
}
}  // namespace

int fsk_measure_fp32_peak(fsk_ctx* ctx, double* tflops) {
    return guard([&] {
        set_device(ctx);
        if (!tflops) fail(FSK_EINVAL, "fsk: null output pointer");
        float* o = (float*)scratch(ctx, kBwdMax, 16);
        const int blocks = ctx->sm_count * 8, iters = 1 << 14;
        cudaEvent_t a = pooled_event(ctx), b = pooled_event(ctx);
        k_peak_fp32<<<blocks, 256>>>(o, 256, 0.999f, 1e-3f);  // warm-up
        cuda_check(cudaEventRecord(a, 0), "cudaEventRecord");
        k_peak_fp32<<<blocks, 256>>>(o, iters, 0.999f, 1e-3f);
        cuda_check(cudaEventRecord(b, 0), "cudaEventRecord");
        cuda_check(cudaEventSynchronize(b), "cudaEventSynchronize");
        float ms = 0.f;
        cuda_check(cudaEventElapsedTime(&ms, a, b), "cudaEventElapsedTime");
        ctx->pool.push_back(a);
        ctx->pool.push_back(b);
        *tflops = 2.0 * 8.0 * iters * (double)blocks * 256.0 / (ms * 1e-3) / 1e12;
    });
}
int fsk_device_sm_count(const fsk_ctx* ctx) { return ctx ? ctx->sm_count : -1; }

fsk_search_opts fsk_search_opts_defaults(const fsk_grid_desc* d) {
    fsk_search_opts o{50, 1e-5f, 0.5f, 1e-2f, 0};
    if (!d) return o;
    double s = 0.0;
    for (int a = 0; a < 3; ++a) {
        const double e = (double)d->bbox_max[a] - (double)d->bbox_min[a];
        s += e * e;
    }
    const double diag = std::sqrt(s);
    o.conv_eps = (float)(1e-5 * diag);
    o.div_eps = (float)(0.5 * diag);
    o.dedup_dist = (float)(1e-2 * diag);
    return o;
}

int fsk_precompute_tgrid(fsk_ctx* ctx, const float* weights, const fsk_grid_desc* desc, const float* bones,
                         int32_t n_bones_pose, float* tgrid, void* stream) {
    return guard([&] {
        set_device(ctx);
        const GridP g = make_grid(desc);
        if (n_bones_pose != g.nb) fail(FSK_EINVAL, "precompute_transform_grid: bone count mismatch");
        if (!weights || !bones || !tgrid) fail(FSK_EINVAL, "fsk: null buffer");
        run_precompute(ctx, weights, g, bones, tgrid, (cudaStream_t)stream);
    });
}

int fsk_search_fwd(fsk_ctx* ctx, const float* tgrid, const fsk_grid_desc* desc, const float* bones,
                   int32_t n_bones_pose, const float* points, int64_t n, const fsk_search_opts* opts,
                   fsk_search_out* out, void* stream) {
    return guard([&] {
        set_device(ctx);
        // check_context (correspondence.cpp:29-41), then validate (:19-25)
        if (n_bones_pose < 1) fail(FSK_EINVAL, "search: no bone transforms");
        if (!tgrid) fail(FSK_EINVAL, "search: voxel variant needs skinning and transform grids");
        const GridP g = make_grid(desc);
        if (n_bones_pose != g.nb) fail(FSK_EINVAL, "search: grid bone count mismatch");
        const SearchP sp = make_search(opts);
        check_dense(out, false);
        if (n < 0) fail(FSK_EINVAL, "fsk: negative point count");
        if (n > 0 && (!points || !bones)) fail(FSK_EINVAL, "fsk: null buffer");
        run_search(ctx, tgrid, g, bones, points, n, sp, opts->flags, to_dense(out), (cudaStream_t)stream);
    });
}

int fsk_compact_roots(fsk_ctx* ctx, const fsk_search_out* dense, int64_t n, int32_t n_init, int64_t* offsets,
                      fsk_root* roots, int64_t cap, int64_t* total_out, void* stream) {
    return guard([&] {
        set_device(ctx);
        check_dense(dense, true);
        if (!offsets || !total_out) fail(FSK_EINVAL, "fsk: null buffer");
        cudaStream_t st = (cudaStream_t)stream;
        run_scan(ctx, dense->n_roots, n, offsets, st);
        int64_t total = 0;
        cuda_check(cudaMemcpyAsync(&total, offsets + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st), "cudaMemcpyAsync");
        cuda_check(cudaStreamSynchronize(st), "cudaStreamSynchronize");
        *total_out = total;
        if (total > cap) fail(FSK_EINVAL, "fsk: root buffer too small");
        if (n > 0 && total > 0) {
            if (!roots) fail(FSK_EINVAL, "fsk: null buffer");
            prof_begin(ctx, st);
            k_emit<<<blocks_for(n, 256), 256, 0, st>>>(n, n_init, to_dense(dense), offsets, roots);
            after_launch(ctx, "k_emit");
        }
    });
}

int fsk_deform_host(fsk_ctx* ctx, const float* weights, const fsk_grid_desc* desc, const float* bones,
                    int32_t n_bones_pose, const float* points, int64_t n, const fsk_search_opts* opts,
                    int64_t* offsets, fsk_root* roots, int64_t cap, int64_t* total_out, void* stream) {
    return guard([&] {
        set_device(ctx);
        if (n_bones_pose < 1) fail(FSK_EINVAL, "search: no bone transforms");
        const GridP g = make_grid(desc);
        if (n_bones_pose != g.nb) fail(FSK_EINVAL, "precompute_transform_grid: bone count mismatch");
        const SearchP sp = make_search(opts);
        if (!weights || !bones || !offsets || !total_out || (n > 0 && !points)) fail(FSK_EINVAL, "fsk: null buffer");
        if (n < 0) fail(FSK_EINVAL, "fsk: negative point count");
        cudaStream_t st = (cudaStream_t)stream;
        const int64_t V = (int64_t)g.nx * g.ny * g.nz;
        const int nb = g.nb;
        float* dW = (float*)scratch(ctx, kHW, V * nb * sizeof(float));
        float* dB = (float*)scratch(ctx, kHB, nb * 12 * sizeof(float));
        float* dP = (float*)scratch(ctx, kHP, std::max<int64_t>(1, n) * 3 * sizeof(float));
        float* dT = (float*)scratch(ctx, kHT, V * 12 * sizeof(float));
        const int64_t S = std::max<int64_t>(1, n) * nb;
        char* dense = (char*)scratch(ctx, kHDense, S * (12 + 36 + 4 + 3));
        DenseOut d;
        d.x_c = (float*)dense;
        d.jinv = d.x_c + 3 * S;
        d.resid = d.jinv + 9 * S;
        d.iters = (uint8_t*)(d.resid + S);
        d.converged = d.iters + S;
        d.keep = d.converged + S;
        d.n_roots = (int32_t*)scratch(ctx, kHNroots, std::max<int64_t>(1, n) * sizeof(int32_t));
        int64_t* dOff = (int64_t*)scratch(ctx, kHOffs, (n + 1) * sizeof(int64_t));
        cuda_check(cudaMemcpyAsync(dW, weights, V * nb * sizeof(float), cudaMemcpyHostToDevice, st), "H2D weights");
        cuda_check(cudaMemcpyAsync(dB, bones, nb * 12 * sizeof(float), cudaMemcpyHostToDevice, st), "H2D bones");
        if (n > 0)
            cuda_check(cudaMemcpyAsync(dP, points, n * 3 * sizeof(float), cudaMemcpyHostToDevice, st), "H2D points");
        run_precompute(ctx, dW, g, dB, dT, st);
        run_search(ctx, dT, g, dB, dP, n, sp, opts->flags, d, st);
        run_scan(ctx, d.n_roots, n, dOff, st);
        cuda_check(cudaMemcpyAsync(offsets, dOff, (n + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st), "D2H offsets");
        cuda_check(cudaStreamSynchronize(st), "cudaStreamSynchronize");
        const int64_t total = offsets[n];
        *total_out = total;
        if (total > cap) fail(FSK_EINVAL, "fsk: root buffer too small");
        if (total > 0) {
            if (!roots) fail(FSK_EINVAL, "fsk: null buffer");
            fsk_root* dR = (fsk_root*)scratch(ctx, kHRoots, total * sizeof(fsk_root));
            prof_begin(ctx, st);
            k_emit<<<blocks_for(n, 256), 256, 0, st>>>(n, nb, d, dOff, dR);
            after_launch(ctx, "k_emit");
            cuda_check(cudaMemcpyAsync(roots, dR, total * sizeof(fsk_root), cudaMemcpyDeviceToHost, st), "D2H roots");
            cuda_check(cudaStreamSynchronize(st), "cudaStreamSynchronize");
        }
    });
}

int fsk_init_states(fsk_ctx* ctx, const float* tgrid, const fsk_grid_desc* desc, const float* bones,
                    int32_t n_bones_pose, const float* points, int64_t n, float* x0, float* jinv0, void* stream) {
    return guard([&] {
        set_device(ctx);
        cudaStream_t st = (cudaStream_t)stream;
        if (n_bones_pose < 1) fail(FSK_EINVAL, "search: no bone transforms");
        if (!tgrid) fail(FSK_EINVAL, "search: voxel variant needs skinning and transform grids");
        const GridP g = make_grid(desc);
        if (n_bones_pose != g.nb) fail(FSK_EINVAL, "search: grid bone count mismatch");
        if (n < 0) fail(FSK_EINVAL, "fsk: negative point count");
        if (n == 0) return;
        if (!points || !bones) fail(FSK_EINVAL, "fsk: null buffer");
        prof_begin(ctx, st);
        k_init_states<<<blocks_for(n * g.nb, 256), 256, 0, st>>>(
            reinterpret_cast<const float4*>(tgrid), g, bones, points, n, x0, jinv0);
        after_launch(ctx, "k_init_states");
    });
}

int fsk_eval_points(fsk_ctx* ctx, const float* tgrid, const fsk_grid_desc* desc, const float* x, int64_t n,
                    float* t12, float* d, float* jac, void* stream) {
    return guard([&] {
        set_device(ctx);
        cudaStream_t st = (cudaStream_t)stream;
        const GridP g = make_grid(desc);
        if (n < 0) fail(FSK_EINVAL, "fsk: negative point count");
        if (n == 0) return;
        if (!tgrid || !x) fail(FSK_EINVAL, "fsk: null buffer");
        prof_begin(ctx, st);
        k_eval_points<<<blocks_for(n, 256), 256, 0, st>>>(reinterpret_cast<const float4*>(tgrid), g, x,
                                                                            n, t12, d, jac);
        after_launch(ctx, "k_eval_points");
    });
}

int fsk_search_bwd(fsk_ctx* ctx, const fsk_grid_desc* desc, const float* x_c, const float* jinv, int32_t n_init,
                   const float* grad_xc, const int32_t* root_sel, int64_t n, float* grad_tgrid, int deterministic,
                   void* stream) {
    return guard([&] {
        set_device(ctx);
        const GridP g = make_grid(desc);
        if (n < 0) fail(FSK_EINVAL, "fsk: negative point count");
        if (n_init < 1) fail(FSK_EINVAL, "fsk: n_init must be >= 1");
        if (!grad_tgrid || (n > 0 && (!x_c || !jinv || !grad_xc || !root_sel))) fail(FSK_EINVAL, "fsk: null buffer");
        cudaStream_t st = (cudaStream_t)stream;
        const int64_t V = (int64_t)g.nx * g.ny * g.nz;
        if (!deterministic) {
            const unsigned zb = (unsigned)std::min<int64_t>(blocks_for(V * 3, 256), (int64_t)ctx->sm_count * 8);
            prof_begin(ctx, st);
            k_zero<<<zb, 256, 0, st>>>(reinterpret_cast<float4*>(grad_tgrid), V * 3);
            after_launch(ctx, "k_zero");
            if (n > 0) {
                prof_begin(ctx, st);
                k_bwd_scatter<<<blocks_for(n, 256), 256, 0, st>>>(g, n_init, x_c, jinv, grad_xc, root_sel, n,
                                                                  reinterpret_cast<float4*>(grad_tgrid));
                after_launch(ctx, "k_bwd_scatter");
            }
            return;
        }
        unsigned long long* acc = (unsigned long long*)scratch(ctx, kBwdAcc, V * 12 * sizeof(unsigned long long));
        unsigned int* mx = (unsigned int*)scratch(ctx, kBwdMax, 16);
        const unsigned zb = (unsigned)std::min<int64_t>(blocks_for(V * 6, 256), (int64_t)ctx->sm_count * 8);
        prof_begin(ctx, st);
        k_zero<<<zb, 256, 0, st>>>(reinterpret_cast<float4*>(acc), V * 6);
        after_launch(ctx, "k_zero");
        prof_begin(ctx, st);
        k_zero<<<1, 32, 0, st>>>(reinterpret_cast<float4*>(mx), 1);
        after_launch(ctx, "k_zero");
        if (n > 0) {
            prof_begin(ctx, st);
            k_bwd_maxterm<<<blocks_for(n, 256), 256, 0, st>>>(n_init, x_c, jinv, grad_xc, root_sel, n, mx);
            after_launch(ctx, "k_bwd_maxterm");
            prof_begin(ctx, st);
            k_bwd_scatter_fixed<<<blocks_for(n, 256), 256, 0, st>>>(g, n_init, x_c, jinv, grad_xc, root_sel, n, mx, acc);
            after_launch(ctx, "k_bwd_scatter_fixed");
        }
        const unsigned cb = (unsigned)std::min<int64_t>(blocks_for(V * 12, 256), (int64_t)ctx->sm_count * 8);
        prof_begin(ctx, st);
        k_bwd_fixed_to_float<<<cb, 256, 0, st>>>(reinterpret_cast<const long long*>(acc), V * 12, mx, n, grad_tgrid);
        after_launch(ctx, "k_bwd_fixed_to_float");
    });
}

int fsk_grad_weights(fsk_ctx* ctx, const fsk_grid_desc* desc, const float* grad_tgrid, const float* bones,
                     int32_t n_bones_pose, float* grad_w, void* stream) {
    return guard([&] {
        set_device(ctx);
        cudaStream_t st = (cudaStream_t)stream;
        const GridP g = make_grid(desc);
        if (n_bones_pose != g.nb) fail(FSK_EINVAL, "precompute_transform_grid: bone count mismatch");
        if (!grad_tgrid || !bones || !grad_w) fail(FSK_EINVAL, "fsk: null buffer");
        const int64_t V = (int64_t)g.nx * g.ny * g.nz;
        const size_t smem = (size_t)(g.nb * 12 + kGwTile * g.nb) * sizeof(float);
        if (smem > 200 * 1024) fail(FSK_EINVAL, "fsk: too many bones for grad_weights");
        if (smem > 48 * 1024)
            cuda_check(cudaFuncSetAttribute(k_grad_weights, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                       "cudaFuncSetAttribute");
        prof_begin(ctx, st);
        k_grad_weights<<<blocks_for(V, kGwTile), kGwTile, smem, st>>>(grad_tgrid, bones, g.nb, V,
                                                                                       grad_w);
        after_launch(ctx, "k_grad_weights");
    });
}

}  // extern "C"
