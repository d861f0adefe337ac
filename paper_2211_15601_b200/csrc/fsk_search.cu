// fsk_search.cu — forward hot path of the deformer on sm_100a and its C-ABI entry points.
//
//   K1  k_precompute_v      precompute_transform_grid (deformer.cpp:61-77, lbs_blend :9-19), one
//                           thread per vertex, fused with the x-pair gather-plane relayout
//                           (fsk_device.cuh), in float32 and (for the escalation pass) float64
//   S*  k_sort_*            spatial (Morton) ordering of the queries — performance only
//   K2  k_search_fast       search_one per (point, bone-init) (correspondence.cpp:126-150)
//                           with iterate (:97-124) in registers, float32, iteration-capped,
//                           flags solves whose float32 outcome is not trustworthy
//   K2b k_esc_start,        the flagged solves re-run from scratch in float64, replaying the
//       k_search_escalated  oracle's operation order (fsk_exact.cuh)
//   D   k_dedup             dedup_roots (correspondence.cpp:162-176)
//   C*  k_scan_lookback,    compaction into CorrespondenceSets (correspondence.hpp:29-42)
//       k_emit
//   k_scatter_dense         the dense per-(point, init) form (fsk_search_out)
//   E   k_eval_points, k_init_states
//
// K2 writes its per-solve state bone-major in sorted-query order ("search planes") so
// every store of a warp is one contiguous, coalesced segment; dedup then reads the n_b
// inits of a query with coalesced loads, and only kept roots are scattered to the
// caller's query order (≈1 root per query instead of n_b dense records).
//
// Precision: long Broyden trajectories are chaotic — a float32
// rounding of the transform grid alone flips ~0.03 % of converged masks against the
// float64 reference. The float32 pass therefore stops at esc_cap iterations and flags
// every solve whose outcome float32 cannot settle (long or late-diverging trajectories,
// threshold decisions within float32 noise); those (~5 %) are solved again in float64,
// which B200 runs at half the float32 rate.
#include <cooperative_groups.h>
#include <cstdlib>
#include <cstring>
#include <functional>

#include "fsk_ctx.h"
#include "fsk_exact.cuh"

namespace cg = cooperative_groups;

// FSK_CHECKED builds (scripts: the GPU suite under FSK_LIB=build/variants/checked.so) trap on any
// out-of-range index at the places a logic error would write out of bounds: the sort's scatter, the
// escalation queue's two ends, its start states and the refill buffer, the CorrespondenceSet emission.
// compute-sanitizer is not available on the GPU pool.
#ifdef FSK_CHECKED
#define FSK_CHECK(c)                                                                          \
    do {                                                                                      \
        if (!(c)) {                                                                           \
            printf("FSK_CHECK failed %s:%d block %d thread %d: %s\n", __FILE__, __LINE__,      \
                   (int)blockIdx.x, (int)threadIdx.x, #c);                                     \
            __trap();                                                                         \
        }                                                                                     \
    } while (0)
#else
#define FSK_CHECK(c) ((void)0)
#endif

namespace fsk {

// ============================================================================ K1
// T_v = Σ_i w_{v,i}·B_i, accumulated in bone order like lbs_blend. One thread per vertex,
// bones staged in shared memory. Writes the reference-layout [V][12] grid (if tg != null)
// and the gather planes: P[r][v].lo = row r of T_v, P[r][v-1].hi = row r of T_v — in
// float32 (p32) and, when p64 != null, float64 from the same float32 inputs.
template <typename R>
__device__ __forceinline__ void put_planes(R* planes, int64_t V, int64_t v, bool has_left, const R* T) {
    const int64_t stride = 8 * V;
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        R* lo = planes + r * stride + 8 * v;
#pragma unroll
        for (int e = 0; e < 4; ++e) lo[e] = T[4 * r + e];
        if (has_left) {
            R* hi = planes + r * stride + 8 * (v - 1) + 4;
#pragma unroll
            for (int e = 0; e < 4; ++e) hi[e] = T[4 * r + e];
        }
    }
}

__global__ void __launch_bounds__(256) k_precompute(const float* __restrict__ w, const float* __restrict__ bones,
                                                    int nb, int nx, int64_t V, float4* __restrict__ tg,
                                                    float* __restrict__ p32, double* __restrict__ p64,
                                                    double* __restrict__ tg64) {
    // one thread per (vertex, matrix row r): three threads share a vertex's weights (L1 broadcast)
    extern __shared__ float sB[];
    for (int e = threadIdx.x; e < nb * 12; e += blockDim.x) sB[e] = bones[e];
    __syncthreads();
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= 3 * V) return;
    const int64_t v = t / 3;
    const int r = (int)(t - 3 * v);
    const float* wv = w + v * nb;
    float T[4] = {0.f, 0.f, 0.f, 0.f};
    double D[4] = {0.0, 0.0, 0.0, 0.0};
    const bool f64 = p64 || tg64;
    for (int i = 0; i < nb; ++i) {
        const float wi = __ldg(wv + i);
        const float* Bi = sB + i * 12 + 4 * r;
#pragma unroll
        for (int e = 0; e < 4; ++e) T[e] = fmaf(wi, Bi[e], T[e]);  // lbs_blend bone order (deformer.cpp:9-19)
        if (f64)
#pragma unroll
            for (int e = 0; e < 4; ++e) D[e] = __fma_rn((double)wi, (double)Bi[e], D[e]);  // lbs_blend as the oracle contracts it
    }
    const bool has_left = (v % nx) != 0;
    if (tg) tg[3 * v + r] = make_float4(T[0], T[1], T[2], T[3]);
    const int64_t stride = 8 * V;
    if (p32) {
        float* lo = p32 + r * stride + 8 * v;
        *reinterpret_cast<float4*>(lo) = make_float4(T[0], T[1], T[2], T[3]);
        if (has_left) *reinterpret_cast<float4*>(lo - 4) = make_float4(T[0], T[1], T[2], T[3]);
    }
    if (p64) {
        double* lo = p64 + r * stride + 8 * v;
#pragma unroll
        for (int e = 0; e < 4; ++e) lo[e] = D[e];
        if (has_left)
#pragma unroll
            for (int e = 0; e < 4; ++e) lo[e - 4] = D[e];
    }
    if (tg64)
#pragma unroll
        for (int e = 0; e < 4; ++e) tg64[12 * v + 4 * r + e] = D[e];
}

// K1, one thread per vertex (FSK_K1_V1 keeps the thread-per-(vertex, row) kernel above): the vertex's
// n_b weights in 16-B loads (a warp reads 32 consecutive weight rows, one contiguous span), all 12
// entries in float32 and float64 accumulated in bone order exactly as k_precompute (same bits), then
// per matrix row one 16-B (float32) / 32-B (float64) store to record v and one to record v-1 of the
// x-pair planes — a warp's stores to a row plane cover one contiguous span. Bones staged in shared
// memory (float32 and float64 copies).
#ifndef FSK_K1_WIDE
#define FSK_K1_WIDE 1
#endif
__device__ __forceinline__ void st_v8f32(float* p, const float4& a, const float4& b) {
    asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(a.x), "f"(a.y), "f"(a.z),
                 "f"(a.w), "f"(b.x), "f"(b.y), "f"(b.z), "f"(b.w)
                 : "memory");
}
__device__ __forceinline__ void st_v4f64(double* p, double a, double b, double c, double d) {
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}

__global__ void __launch_bounds__(128) k_precompute_v(const float* __restrict__ w, const float* __restrict__ bones,
                                                     int nb, int nx, int64_t V, float4* __restrict__ tg,
                                                     float* __restrict__ p32, double* __restrict__ p64,
                                                     double* __restrict__ tg64) {
    extern __shared__ float sB[];
    for (int e = threadIdx.x; e < nb * 12; e += blockDim.x) sB[e] = bones[e];
    __syncthreads();
    const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
#if FSK_K1_WIDE
    if (v - (threadIdx.x & 31) >= V) return;  // whole warp past the end (the stores below shuffle)
    const bool valid = v < V;
#else
    if (v >= V) return;
    const bool valid = true;
#endif
    const float* wv = w + v * nb;
    float T[12];
    double D[12];
#pragma unroll
    for (int e = 0; e < 12; ++e) {
        T[e] = 0.f;
        D[e] = 0.0;
    }
    const bool f64 = p64 || tg64;
    auto bone = [&](int i, float wi) {
        const float* Bi = sB + 12 * i;
#pragma unroll
        for (int e = 0; e < 12; ++e) T[e] = fmaf(wi, Bi[e], T[e]);  // lbs_blend bone order (deformer.cpp:9-19)
        if (f64)
#pragma unroll
            for (int e = 0; e < 12; ++e) D[e] = __fma_rn((double)wi, (double)Bi[e], D[e]);
    };
    if (valid) {
        if ((nb & 3) == 0) {
            for (int i = 0; i < nb; i += 4) {
                const float4 q = __ldg(reinterpret_cast<const float4*>(wv + i));
                bone(i, q.x);
                bone(i + 1, q.y);
                bone(i + 2, q.z);
                bone(i + 3, q.w);
            }
        } else {
            for (int i = 0; i < nb; ++i) bone(i, __ldg(wv + i));
        }
    }
    const bool has_left = (v % nx) != 0;
    const int64_t stride = 8 * V;
    if (tg && valid)  // (staging these rows through shared memory for full-line stores measured no faster)
#pragma unroll
        for (int r = 0; r < 3; ++r) tg[3 * v + r] = make_float4(T[4 * r], T[4 * r + 1], T[4 * r + 2], T[4 * r + 3]);
#if FSK_K1_WIDE
    // x-pair rows written whole by their owner: pair v = {row r of T_v, row r of T_{v+1}} in one
    // 32-B (float32) / 2 × 32-B (float64) store per row, T_{v+1} from the next lane; lane 31 writes
    // the first half only and lane 0 of the next warp the second half (its own row) — the same
    // bytes as the per-half stores, in full sectors.
    const int lane = threadIdx.x & 31;
    const bool has_right = v + 1 < V && ((v + 1) % nx) != 0;
    const bool whole = lane < 31 && has_right;
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        if (p32) {
            const float4 own = make_float4(T[4 * r], T[4 * r + 1], T[4 * r + 2], T[4 * r + 3]);
            float4 nxt;
            nxt.x = __shfl_down_sync(0xffffffffu, own.x, 1);
            nxt.y = __shfl_down_sync(0xffffffffu, own.y, 1);
            nxt.z = __shfl_down_sync(0xffffffffu, own.z, 1);
            nxt.w = __shfl_down_sync(0xffffffffu, own.w, 1);
            float* row = p32 + r * stride + 8 * v;
            if (valid) {
                if (whole) st_v8f32(row, own, nxt);
                else *reinterpret_cast<float4*>(row) = own;
                if (lane == 0 && has_left) *reinterpret_cast<float4*>(row - 4) = own;
            }
        }
        if (p64) {
            double nxt[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) nxt[e] = __shfl_down_sync(0xffffffffu, D[4 * r + e], 1);
            double* row = p64 + r * stride + 8 * v;
            if (valid) {
                st_v4f64(row, D[4 * r], D[4 * r + 1], D[4 * r + 2], D[4 * r + 3]);
                if (whole) st_v4f64(row + 4, nxt[0], nxt[1], nxt[2], nxt[3]);
                if (lane == 0 && has_left) st_v4f64(row - 4, D[4 * r], D[4 * r + 1], D[4 * r + 2], D[4 * r + 3]);
            }
        }
        if (tg64 && valid)
#pragma unroll
            for (int e = 0; e < 4; ++e) tg64[12 * v + 4 * r + e] = D[4 * r + e];
    }
#else
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        if (p32) {
            float4* lo = reinterpret_cast<float4*>(p32 + r * stride + 8 * v);
            const float4 t4 = make_float4(T[4 * r], T[4 * r + 1], T[4 * r + 2], T[4 * r + 3]);
            lo[0] = t4;
            if (has_left) lo[-1] = t4;
        }
        if (p64) {
            double2* lo = reinterpret_cast<double2*>(p64 + r * stride + 8 * v);
            const double2 a = make_double2(D[4 * r], D[4 * r + 1]), b = make_double2(D[4 * r + 2], D[4 * r + 3]);
            lo[0] = a;
            lo[1] = b;
            if (has_left) {
                lo[-2] = a;
                lo[-1] = b;
            }
        }
        if (tg64)
#pragma unroll
            for (int e = 0; e < 4; ++e) tg64[12 * v + 4 * r + e] = D[4 * r + e];
    }
#endif
}

// Relayout of a caller-provided [V][12] grid (float32, or float64 when tg64 != null) into
// the gather planes of both precisions.
__global__ void __launch_bounds__(256) k_relayout(const float* __restrict__ tg, const double* __restrict__ tg64, int nx,
                                                  int64_t V, float* __restrict__ p32, double* __restrict__ p64) {
    const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v >= V) return;
    const bool has_left = (v % nx) != 0;
    float T[12];
    double D[12];
#pragma unroll
    for (int e = 0; e < 12; ++e) {
        D[e] = tg64 ? tg64[12 * v + e] : (double)tg[12 * v + e];
        T[e] = tg ? tg[12 * v + e] : (float)D[e];
    }
    if (p32) put_planes(p32, V, v, has_left, T);
    if (p64) put_planes(p64, V, v, has_left, D);
}

// ============================================================================ sort
// Counting sort of the queries on a 15-bit Morton key of their posed position within
// the queries' bounding box. Performance only: every solve runs the same instruction
// sequence wherever it lands, so results are order-independent (and bitwise
// deterministic); neighbouring lanes then gather neighbouring grid cells.
constexpr int kSortBitsPerAxis = 5;
constexpr int kSortBuckets = 1 << (3 * kSortBitsPerAxis);

__device__ __forceinline__ int f2ord(float f) {
    const int i = __float_as_int(f);
    return i >= 0 ? i : i ^ 0x7fffffff;
}
__device__ __forceinline__ float ord2f(int i) { return __int_as_float(i >= 0 ? i : i ^ 0x7fffffff); }

// Sort state, one contiguous int block zeroed by a single memset per call:
//   [0, kSortBuckets) histogram, then bbox (6 words), escalation counters (4), scan barrier (2).
// The bbox is kept in a zero-identity encoding: u = f2ord(f) ^ 0x80000000 (unsigned order);
// max stored as u, min stored as ~u, both reduced with atomicMax.
constexpr int kSortMaxBlocks = 1024;  // block sums of the fused sort's bucket scan
constexpr int kSortStateInts = kSortBuckets + 64 + kSortMaxBlocks;  // + bbox, counters, barrier + 32 block sums, fused-sort sums
constexpr int kBboxOff = kSortBuckets, kEscOff = kSortBuckets + 8, kScanBarOff = kSortBuckets + 16,
              kSortSumsOff = kSortBuckets + 64;
__device__ __forceinline__ unsigned bb_enc(float f) { return (unsigned)f2ord(f) ^ 0x80000000u; }
__device__ __forceinline__ float bb_dec(unsigned u) { return ord2f((int)(u ^ 0x80000000u)); }

__global__ void __launch_bounds__(256) k_sort_bbox(const float* __restrict__ x, int64_t n, unsigned* __restrict__ bbox) {
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
    // warp, then block reduction: 6 atomics per block (per-warp atomics on 6 addresses
    // serialized in the L2 atomic unit)
    __shared__ float s_lo[3][8], s_hi[3][8];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        for (int o = 16; o > 0; o >>= 1) {
            lo[a] = fminf(lo[a], __shfl_xor_sync(0xffffffff, lo[a], o));
            hi[a] = fmaxf(hi[a], __shfl_xor_sync(0xffffffff, hi[a], o));
        }
        if (lane == 0) {
            s_lo[a][warp] = lo[a];
            s_hi[a][warp] = hi[a];
        }
    }
    __syncthreads();
    if (threadIdx.x < 3) {
        const int a = threadIdx.x;
        float l = s_lo[a][0], h = s_hi[a][0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
            l = fminf(l, s_lo[a][w]);
            h = fmaxf(h, s_hi[a][w]);
        }
        atomicMax(bbox + a, ~bb_enc(l));
        atomicMax(bbox + 3 + a, bb_enc(h));
    }
}

__device__ __forceinline__ uint32_t spread3(uint32_t v) {  // 5 bits -> every third bit
    v &= 0x1f;
    v = (v | (v << 8)) & 0x100f;
    v = (v | (v << 4)) & 0x10c3;
    v = (v | (v << 2)) & 0x1249;
    return v;
}

__global__ void __launch_bounds__(256) k_sort_hist(const float* __restrict__ x, int64_t n, const unsigned* __restrict__ bbox,
                                                   uint16_t* __restrict__ keys, int* __restrict__ hist) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n) return;
    uint32_t q[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const float lo = bb_dec(~bbox[a]), hi = bb_dec(bbox[3 + a]);
        const float s = (float)(1 << kSortBitsPerAxis) / fmaxf(hi - lo, 1e-30f);
        const float u = (x[3 * p + a] - lo) * s;
        const int qi = isfinite(u) ? __float2int_rd(u) : 0;
        q[a] = (uint32_t)max(0, min(qi, (1 << kSortBitsPerAxis) - 1));
    }
    const uint32_t k = spread3(q[0]) | (spread3(q[1]) << 1) | (spread3(q[2]) << 2);
    keys[p] = (uint16_t)k;
    atomicAdd(hist + k, 1);
}

// Exclusive scan of the 32768 bucket counts by 32 co-resident blocks of 1024 (one bucket per
// thread): block sums, a grid barrier on a counter, then each block adds the sums before it.
constexpr int kScanBlocks = kSortBuckets / 1024;
__global__ void __launch_bounds__(1024) k_sort_scan(int* __restrict__ hist, int* __restrict__ bar) {
    __shared__ int warp_tot[32];
    __shared__ int prefix;
    const int t = threadIdx.x, b = blockIdx.x;
    const int v = hist[b * 1024 + t];
    int incl = v;
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffff, incl, o);
        if ((t & 31) >= o) incl += y;
    }
    if ((t & 31) == 31) warp_tot[t >> 5] = incl;
    __syncthreads();
    if (t < 32) {
        const int w = warp_tot[t];
        int wi = w;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffff, wi, o);
            if (t >= o) wi += y;
        }
        warp_tot[t] = wi - w;
        if (t == 31) {
            volatile int* sums = bar + 2;
            sums[b] = wi;  // block total
            __threadfence();
            atomicAdd(bar, 1);
            while (*(volatile int*)bar < (int)gridDim.x) {
            }
            __threadfence();
            int p = 0;
            for (int i = 0; i < b; ++i) p += sums[i];
            prefix = p;
        }
    }
    __syncthreads();
    hist[b * 1024 + t] = prefix + warp_tot[t >> 5] + incl - v;
}

// The same scan by one block of 1024 threads, 32 consecutive buckets per thread (no grid barrier).
// Ablation (off by default).
#ifndef FSK_SORT_SCAN1
#define FSK_SORT_SCAN1 0  // measured slower: 14.6 us vs 9.7 for the 32-block scan (C2 step 0.9695 -> 0.9756 ms)
#endif
#ifndef FSK_SORT_BBOX_BLOCKS_PER_SM
#define FSK_SORT_BBOX_BLOCKS_PER_SM 8  // 2 measured the same (11.5 us)
#endif
__global__ void __launch_bounds__(1024) k_sort_scan1(int* __restrict__ hist) {
    __shared__ int warp_tot[32];
    constexpr int kPer = kSortBuckets / 1024;
    const int t = threadIdx.x;
    int4 v[kPer / 4];
    int sum = 0;
#pragma unroll
    for (int i = 0; i < kPer / 4; ++i) {
        v[i] = reinterpret_cast<const int4*>(hist)[t * (kPer / 4) + i];
        sum += v[i].x + v[i].y + v[i].z + v[i].w;
    }
    int incl = sum;
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffff, incl, o);
        if ((t & 31) >= o) incl += y;
    }
    if ((t & 31) == 31) warp_tot[t >> 5] = incl;
    __syncthreads();
    if (t < 32) {
        const int w = warp_tot[t];
        int wi = w;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffff, wi, o);
            if (t >= o) wi += y;
        }
        warp_tot[t] = wi - w;
    }
    __syncthreads();
    int run = warp_tot[t >> 5] + incl - sum;
#pragma unroll
    for (int i = 0; i < kPer / 4; ++i) {
        int4 o;
        o.x = run; run += v[i].x;
        o.y = run; run += v[i].y;
        o.z = run; run += v[i].z;
        o.w = run; run += v[i].w;
        reinterpret_cast<int4*>(hist)[t * (kPer / 4) + i] = o;
    }
}

// Scatter into sorted order: perm[pos] = p, xs[pos] = (x_p, 0) as float4 (16-B loads in K2).
__global__ void __launch_bounds__(256) k_sort_scatter(const float* __restrict__ x, const uint16_t* __restrict__ keys,
                                                      int64_t n, int* __restrict__ offs, int* __restrict__ perm,
                                                      float4* __restrict__ xs) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n) return;
    const int pos = atomicAdd(offs + keys[p], 1);
    FSK_CHECK(pos >= 0 && pos < n);
    perm[pos] = (int)p;
    xs[pos] = make_float4(x[3 * p], x[3 * p + 1], x[3 * p + 2], 0.f);
}

__global__ void __launch_bounds__(256) k_identity_order(const float* __restrict__ x, int64_t n, int* __restrict__ perm,
                                                        float4* __restrict__ xs, int* __restrict__ esc_count) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p == 0) esc_count[0] = esc_count[1] = esc_count[2] = esc_count[3] = 0;
    if (p >= n) return;
    perm[p] = (int)p;
    xs[p] = make_float4(x[3 * p], x[3 * p + 1], x[3 * p + 2], 0.f);
}


// ============================================================================ K2
// Per-solve state, bone-major in sorted order: q = bone*n + j.
struct SearchPlanes {
    float4* xr;      // {x, y, z, residual}
    float4* ja;      // J~[0..3]
    float4* jb;      // J~[4..7]
    float* jc;       // J~[8]
    uint32_t* meta;  // iterations (30 bits; any max_iters >= 1, correspondence.cpp:20) | J~ stored << 30 | converged << 31
    uint8_t* keep;   // dedup survivors
    uint32_t* kmask = nullptr;  // per sorted query: bit b = bone b's root kept (n_b <= 32), for k_emit
    double* xd = nullptr;       // optional [S][3] float64 root (fsk_search_out::x_c64): the float64 state of
                                // the float64-solved solves, the float32 root widened otherwise
};

#ifndef FSK_SEARCH_BLOCK
#define FSK_SEARCH_BLOCK 128
#endif
constexpr int kSearchBlock = FSK_SEARCH_BLOCK;
#ifndef FSK_SEARCH_MINB
#define FSK_SEARCH_MINB 3  // 128-thread CTAs: 168 registers hold the 96-float cell cache without spills (measured best: 128x3 0.598 ms, 256x1 0.802, 128x4 0.722 with spills, no cache 256x3 0.691)
#endif

template <typename R>
__device__ __forceinline__ void store_solve(const SearchPlanes& out, int64_t q, R x0, R x1, R x2, const R Ji[9], R err2,
                                            const SolveOut& s, bool store_jt = true) {
    // the residual's sign bit carries the converged flag (dedup reads one float4 per solve)
    const float4 xr = make_float4((float)x0, (float)x1, (float)x2, copysignf((float)sqrt(err2), s.conv ? 1.f : -1.f));
    if (out.xd) {
        out.xd[3 * q] = (double)x0;
        out.xd[3 * q + 1] = (double)x1;
        out.xd[3 * q + 2] = (double)x2;
    }
#ifdef FSK_NO_STORE_HINTS
    out.xr[q] = xr;
    out.ja[q] = make_float4((float)Ji[0], (float)Ji[1], (float)Ji[2], (float)Ji[3]);
    out.jb[q] = make_float4((float)Ji[4], (float)Ji[5], (float)Ji[6], (float)Ji[7]);
    out.jc[q] = (float)Ji[8];
    out.meta[q] = (uint32_t)s.iters | (s.conv ? 0x80000000u : 0u) | (store_jt ? 0x40000000u : 0u);
#else
    // x / residual stay in L2 for dedup (read right after the search); J~ and meta are read only
    // for the ~1 kept root per query (emit), so they stream out (evict-first). Measured on C2:
    // k_dedup 37.6 -> 34.6 us, step 1.0140 -> 1.0096 ms.
#ifndef FSK_NO_XR_EVICT_LAST
    asm volatile("{ .reg .b64 pol; createpolicy.fractional.L2::evict_last.b64 pol, 1.0;\n"
                 "  st.global.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, pol; }"
                 :: "l"(out.xr + q), "f"(xr.x), "f"(xr.y), "f"(xr.z), "f"(xr.w) : "memory");
#else
    out.xr[q] = xr;
#endif
    if (store_jt) {  // J~ is read only for roots (converged solves); the float32 pass skips it otherwise
        __stcs(out.ja + q, make_float4((float)Ji[0], (float)Ji[1], (float)Ji[2], (float)Ji[3]));
        __stcs(out.jb + q, make_float4((float)Ji[4], (float)Ji[5], (float)Ji[6], (float)Ji[7]));
        __stcs(out.jc + q, (float)Ji[8]);
    }
    __stcs(reinterpret_cast<unsigned int*>(out.meta) + q,
           (unsigned int)s.iters | (s.conv ? 0x80000000u : 0u) | (store_jt ? 0x40000000u : 0u));
#endif
}

// Final state of an exact-replay solve (fsk_exact.cuh): the residual is the replay's own norm.
__device__ __forceinline__ void store_exact(const SearchPlanes& out, int64_t q, const exact::XState& s, bool conv) {
    if (out.xd) {
        out.xd[3 * q] = s.x0;
        out.xd[3 * q + 1] = s.x1;
        out.xd[3 * q + 2] = s.x2;
    }
    out.xr[q] = make_float4((float)s.x0, (float)s.x1, (float)s.x2, copysignf((float)s.err, conv ? 1.f : -1.f));
    out.ja[q] = make_float4((float)s.Ji[0], (float)s.Ji[1], (float)s.Ji[2], (float)s.Ji[3]);
    out.jb[q] = make_float4((float)s.Ji[4], (float)s.Ji[5], (float)s.Ji[6], (float)s.Ji[7]);
    out.jc[q] = (float)s.Ji[8];
    out.meta[q] = (uint32_t)s.k | (conv ? 0x80000000u : 0u) | 0x40000000u;
}

// Work counters for the roofline (bench.py): per pass, solves / Broyden iterations /
// converged-terminating iterations, one warp-aggregated atomic per warp.
__device__ __forceinline__ void count_work(unsigned long long* stats, const SolveOut& s) {
    if (!stats) return;
    const unsigned act = __activemask();
    const unsigned it = __reduce_add_sync(act, (unsigned)s.iters);
    const unsigned fin = __reduce_add_sync(act, (unsigned)(s.conv && s.iters > 0));
    const unsigned fl = __reduce_add_sync(act, (unsigned)s.fills);
    if ((threadIdx.x & 31) == __ffs(act) - 1) {
        atomicAdd(stats + 0, (unsigned long long)__popc(act));
        atomicAdd(stats + 1, (unsigned long long)it);
        atomicAdd(stats + 2, (unsigned long long)fin);
        if (fl) atomicAdd(stats + 6, (unsigned long long)fl);
    }
}

// Fast pass: one thread per posed point, looping over a group of `bpg` bone inits (one float32
// solve each) over spatially sorted queries. Blocks are tile-major: block = (query tile, bone
// group), so one SM solves several inits of the same queries back to back — they converge to the
// same few canonical roots, and the iterations' gathers hit the cells the previous init left in
// L1. B_i^-1 stays a block-uniform broadcast load. Solves flagged for escalation are appended
// (warp-aggregated) to esc_q.
#ifndef FSK_FAST_MAP
#define FSK_FAST_MAP 1  // C2 fast pass: 0.556 -> 0.551 ms (bone groups of a tile on one SM in the first wave)
#endif
#ifndef FSK_FAST_BPG
#define FSK_FAST_BPG 8  // bone inits per block (0: all). C2 fast pass: 1 0.638 ms, 2 0.594, 4 0.575, 8 0.572, 12 0.581, 24 0.601 (bone-major blocks: 0.633)
#endif
#ifndef FSK_INIT_PREFETCH
#define FSK_INIT_PREFETCH 0  // measured slower: C2 fast pass 0.544 -> 0.583 ms, C4-grid 2.905 -> 3.121 ms (hashes equal)
#endif
// (ablation) L1 prefetch of the next init's cell: x0 = B^-1 x' of the next bone (an address hint only — the
// solve recomputes it exactly), its 4 x-pair edges × 3 rows. The init gathers are the pass's
// L1 misses (the cell is new for every bone); issued one solve ahead, they land during it.
__device__ __forceinline__ void prefetch_init(const Planes<float>& P, const GridP& g, const float* __restrict__ B,
                                              const float4& xq) {
    const float t0 = __ldg(B + 3), t1 = __ldg(B + 7), t2 = __ldg(B + 11);
    const float d0 = xq.x - t0, d1 = xq.y - t1, d2 = xq.z - t2;
    const float x0 = __ldg(B + 0) * d0 + __ldg(B + 4) * d1 + __ldg(B + 8) * d2;
    const float x1 = __ldg(B + 1) * d0 + __ldg(B + 5) * d1 + __ldg(B + 9) * d2;
    const float x2 = __ldg(B + 2) * d0 + __ldg(B + 6) * d1 + __ldg(B + 10) * d2;
    const Cell<float> c = locate<false, float>(g, x0, x1, x2);
    const int nxy = g.nx * g.ny;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const int v = c.base + (e >> 1) * nxy + (e & 1) * g.nx;
#pragma unroll
        for (int r = 0; r < 3; ++r)
            asm volatile("prefetch.global.L1 [%0];" ::"l"(P.p + r * P.stride + (int64_t)v * 8));
    }
}

__global__ void __launch_bounds__(kSearchBlock, FSK_SEARCH_MINB)
    k_search_fast(Planes<float> P, GridP g, const float* __restrict__ bones, const float4* __restrict__ xs, int64_t n,
                  int bpg, SearchP o, SearchPlanes out, int4* __restrict__ esc_q, int64_t esc_cap,
                  int* __restrict__ esc_count, unsigned long long* __restrict__ stats, int wave_sms) {
    const int ngroups = (g.nb + bpg - 1) / bpg;
#if FSK_FAST_MAP == 1
    // wave-aligned: blocks b, b + W, b + 2W, ... (W = SM count) land on one SM in the first wave under the
    // breadth-first block dispatch — they take the bone groups of the same tile, so an SM's resident
    // CTAs share that tile's cells in L1
    const int W = wave_sms;
    const int chunk = blockIdx.x / (W * ngroups), r = blockIdx.x - chunk * (W * ngroups);
    const int grp = r / W, tile = chunk * W + (r - grp * W);
#else
    const int tile = blockIdx.x / ngroups, grp = blockIdx.x - tile * ngroups;
#endif
    const int64_t j = (int64_t)tile * kSearchBlock + threadIdx.x;
    if (j >= n) return;
    const float4 xq = __ldg(xs + j);
    const int b_end = min(g.nb, (grp + 1) * bpg);
#ifndef FSK_PER_SOLVE_STATS
    unsigned w_solves = 0, w_iters = 0, w_fin = 0, w_fills = 0;  // work counters, flushed once per thread
#endif
#if FSK_INIT_PREFETCH
    prefetch_init(P, g, bones + 12 * (grp * bpg), xq);
#endif
    for (int bone = grp * bpg; bone < b_end; ++bone) {
#if FSK_INIT_PREFETCH
        if (bone + 1 < b_end) prefetch_init(P, g, bones + 12 * (bone + 1), xq);
#endif
        float x0, x1, x2, Ji[9], err2;
        const SolveOut s = solve_one<float, true>(P, g, bones + 12 * bone, xq.x, xq.y, xq.z, o, x0, x1, x2, Ji, err2);
        const int64_t q = (int64_t)bone * n + j;
        // J~ only for a root the float32 pass settles (an escalated solve is stored again by the float64
        // pass; an unconverged one has no root): C2 DRAM writes of the pass fall by ~half of 36 B per solve
        store_solve(out, q, x0, x1, x2, Ji, err2, s, s.conv && !s.esc);
#ifdef FSK_PER_SOLVE_STATS
        count_work(stats, s);
#else
        w_solves += 1;
        w_iters += s.iters;
        w_fin += (s.conv && s.iters > 0);
        w_fills += s.fills;
#endif
#ifdef FSK_ESC_REASONS  // study builds: per-rule escalation counts (slot 8+bit: fired; 24+bit: fired alone)
        if (stats && s.reasons) {
            for (int bit = 0; bit < 16; ++bit)
                if (s.reasons >> bit & 1u) {
                    atomicAdd(stats + 8 + bit, 1ull);
                    if (__popc(s.reasons) == 1) atomicAdd(stats + 24 + bit, 1ull);
                }
        }
#endif
        if (esc_q) {
            // Capped (long) trajectories are queued from the front, the rest from the back, so
            // the escalation pass starts the long float64 solves first and the short ones fill
            // its tail (the pass reads front entries [0, A) then back entries [S-B, S)).
            const unsigned act = __activemask();
            const unsigned ml = __ballot_sync(act, s.esc && s.capped), ms = __ballot_sync(act, s.esc && !s.capped);
            const int lane = threadIdx.x & 31, leader = __ffs(act) - 1;
            const unsigned lt = (1u << lane) - 1;
            unsigned long long b = 0;  // one atomic for both counters: {short (low word), long (high word)}
            if (lane == leader && (ml | ms))
                b = atomicAdd(reinterpret_cast<unsigned long long*>(esc_count + 2),
                              ((unsigned long long)__popc(ml) << 32) | (unsigned long long)__popc(ms));
            b = __shfl_sync(act, b, leader);
            const int bl = (int)(b >> 32), bs = (int)(b & 0xffffffffu);
            const int4 rec = make_int4((int)q, __float_as_int(xq.x), __float_as_int(xq.y), __float_as_int(xq.z));
            FSK_CHECK(!(s.esc && s.capped) || bl + __popc(ml & lt) < esc_cap - (bs + __popc(ms)));
            FSK_CHECK(!(s.esc && !s.capped) || esc_cap - 1 - (bs + __popc(ms & lt)) >= bl + __popc(ml));
            if (s.esc && s.capped) esc_q[bl + __popc(ml & lt)] = rec;
            else if (s.esc) esc_q[esc_cap - 1 - (bs + __popc(ms & lt))] = rec;
        }
    }
#ifndef FSK_PER_SOLVE_STATS
    // one warp-aggregated flush of the thread's counters (per solve, 4 same-address atomics per warp
    // were ~600 k L2 atomics per C2 launch)
    if (stats) {
        const unsigned act = __activemask();
        w_solves = __reduce_add_sync(act, w_solves);
        w_iters = __reduce_add_sync(act, w_iters);
        w_fin = __reduce_add_sync(act, w_fin);
        w_fills = __reduce_add_sync(act, w_fills);
        if ((threadIdx.x & 31) == __ffs(act) - 1) {
            atomicAdd(stats + 0, (unsigned long long)w_solves);
            atomicAdd(stats + 1, (unsigned long long)w_iters);
            atomicAdd(stats + 2, (unsigned long long)w_fin);
            if (w_fills) atomicAdd(stats + 6, (unsigned long long)w_fills);
        }
    }
#endif
}

// Escalation pass: the flagged solves from scratch in float64 (persistent warps over the
// device-side queue), overwriting their float32 results. The queue holds {q, x'} records,
// long (capped) trajectories first, so long float64 solves start early and short ones fill
// the tail (measured on C2: 0.286 -> 0.203 ms against an unordered queue of indices).
#ifndef FSK_ESC_MINB
#define FSK_ESC_MINB 2  // measured: 254 regs / 8 warps per SM beats 168 regs / 12 warps (0.263 vs 0.277 ms)
#endif
#ifndef FSK_ESC_EXACT_MINB
#define FSK_ESC_EXACT_MINB 2  // 254 regs, no spills: 0.271 ms vs 0.302 at 3 (168 regs, loop-carried spills); refill threshold 16 vs 1/4/8 measured best too
#endif
constexpr int kEscBlock = 128;
#ifndef FSK_REFILL_IDLE
#define FSK_REFILL_IDLE 16  // measured 16 (0.253 ms) vs 12 (0.260) vs 8 (0.265) vs 20 (0.255)
#endif
#ifndef FSK_REFILL_IDLE_EXACT  // exact replay: starts come precomputed from k_esc_start, so a refill is one 128-B load
#define FSK_REFILL_IDLE_EXACT 16
#endif
// float64 copies of the bone transforms in shared memory for the exact replay (dynamic smem of
// n_b·12 doubles; widening is exact)
__device__ __forceinline__ const double* stage_bones64(const float* __restrict__ bones, int nb) {
    extern __shared__ double s_bones64[];
    for (int e = threadIdx.x; e < 12 * nb; e += blockDim.x) s_bones64[e] = (double)__ldg(bones + e);
    __syncthreads();
    return s_bones64;
}

// Start states of the escalated solves, one thread per queue entry (no refill divergence):
// x0 = B^-1 x', J~0, g0 and the residual e (err for the exact replay, err² otherwise), packed
// as 8 double2 [x0 x1 | x2 g0 | g1 g2 | e J0 | J1 J2 | J3 J4 | J5 J6 | J7 J8]. A solve that stops
// at its start (converged or diverged, correspondence.cpp:100-105) is stored here and marked
// e = -1. Entries at or beyond st_cap are started by the refill kernel itself.
template <bool kExact>
__device__ __forceinline__ void esc_start_one(const Planes<double>& P, const GridP& g, const float* __restrict__ W,
                                              const float* __restrict__ bones, const double* bones64, int64_t n,
                                              const SearchP& o, const int4& rec, double s[16], bool& stop,
                                              bool& conv, double* stash = nullptr) {
    const int64_t q = rec.x;
    const int bone = (int)(q / n);
    const float xp0 = __int_as_float(rec.y), xp1 = __int_as_float(rec.z), xp2 = __int_as_float(rec.w);
    if constexpr (kExact) {
        exact::XState xs;
        exact::start(P, g, W, bones64, bone, xp0, xp1, xp2, xs, stash);
        conv = xs.err < o.conv_eps;
        stop = conv || xs.err > o.div_eps;
        s[0] = xs.x0, s[1] = xs.x1, s[2] = xs.x2, s[3] = xs.g0, s[4] = xs.g1, s[5] = xs.g2, s[6] = xs.err;
#pragma unroll
        for (int e = 0; e < 9; ++e) s[7 + e] = xs.Ji[e];
    } else {
        solve_start<double>(P, g, bones + 12 * bone, xp0, xp1, xp2, s[0], s[1], s[2], s + 7, s[3], s[4], s[5], s[6]);
        conv = s[6] < o.conv2;                // (:100-103)
        stop = conv || s[6] > o.div2;         // divergence check at the top (:105)
    }
    stop = stop || o.max_iters <= 0;
}

#ifndef FSK_ESC_START_MINB
#define FSK_ESC_START_MINB 2  // with the ∇w stash (72 KB per CTA at 24 bones): 0.099 ms vs 0.124 at 3 (spills) and 0.106 without the stash
#endif
template <bool kExact>
__global__ void __launch_bounds__(128, FSK_ESC_START_MINB)
    k_esc_start(Planes<double> P, GridP g, const float* __restrict__ W, const float* __restrict__ bones, int64_t n,
                SearchP o, SearchPlanes out, const int4* __restrict__ esc_q, int64_t esc_cap,
                const int* __restrict__ esc_count, double2* __restrict__ st, int st_cap,
                unsigned long long* __restrict__ stats, bool stash_on) {
    const int cnt_long = esc_count[3], cnt = min(esc_count[3] + esc_count[2], st_cap);
    const double* bones64 = kExact ? stage_bones64(bones, g.nb) : nullptr;
    // exact replay: per-thread stash of ∇w (n_b·3 doubles, strided) behind the bone copies, when sized in
    double* stash = (kExact && stash_on) ? const_cast<double*>(bones64) + 12 * g.nb + threadIdx.x : nullptr;
    unsigned n_solves = 0;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < cnt; idx += gridDim.x * blockDim.x) {
        FSK_CHECK(idx < cnt && idx < st_cap && cnt <= esc_cap);
        const int4 rec = esc_q[idx < cnt_long ? idx : esc_cap - 1 - (idx - cnt_long)];
        FSK_CHECK(rec.x >= 0 && rec.x < n * g.nb);
        double s[16];
        bool stop, conv;
        esc_start_one<kExact>(P, g, W, bones, bones64, n, o, rec, s, stop, conv, stash);
        if (stop) {
            if constexpr (kExact) {
                exact::XState xs;
                xs.x0 = s[0], xs.x1 = s[1], xs.x2 = s[2], xs.err = s[6], xs.k = 0;
#pragma unroll
                for (int e = 0; e < 9; ++e) xs.Ji[e] = s[7 + e];
                store_exact(out, rec.x, xs, conv);
            } else {
                store_solve(out, rec.x, s[0], s[1], s[2], s + 7, s[6], SolveOut{0, conv, false});
            }
            s[6] = -1.0;
            n_solves += 1;
        }
        double2* d = st + 8 * (int64_t)idx;
#pragma unroll
        for (int h = 0; h < 8; ++h) d[h] = make_double2(s[2 * h], s[2 * h + 1]);
    }
    if (stats) {
        const unsigned full = __activemask();
        n_solves = __reduce_add_sync(full, n_solves);
        if ((threadIdx.x & 31) == __ffs(full) - 1 && n_solves) atomicAdd(stats + 3, (unsigned long long)n_solves);
    }
}

template <bool kExact>  // kExact: the solves replay the reference's operation order (fsk_exact.cuh)
__global__ void __launch_bounds__(kEscBlock, kExact ? FSK_ESC_EXACT_MINB : FSK_ESC_MINB)
    k_search_escalated(Planes<double> P, GridP g, const float* __restrict__ W, const float* __restrict__ bones,
                       int64_t n, SearchP o,
                       SearchPlanes out, const int4* __restrict__ esc_q, int64_t esc_cap,
                       const int* __restrict__ esc_count, const double2* __restrict__ st, int st_cap,
                       unsigned long long* __restrict__ stats) {
    // Persistent lanes with refill: a lane whose solve finished takes the next queue entry
    // (one warp-aggregated atomic per refill round), so long float64 trajectories do not hold
    // a whole warp idle. Each solve runs exactly solve_one<double>'s arithmetic (solve_start +
    // broyden_step), so results are identical to the one-thread-per-solve kernel.
    const int cnt_long = esc_count[3], cnt = esc_count[3] + esc_count[2];
    const double* bones64 = kExact ? stage_bones64(bones, g.nb) : nullptr;
    int* work = const_cast<int*>(esc_count) + 1;
#ifdef FSK_ESC_TIMELINE  // probe builds: kernel start, queue-dry and exit times (globaltimer, ns)
    if (threadIdx.x == 0 && stats) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        atomicMax(stats + 40, ~t);  // kernel start (min as max of ~t)
    }
#endif
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const double conv2 = o.conv2, div2 = o.div2;
    bool active = false;
    unsigned n_solves = 0, n_iters = 0, n_final = 0;
    int64_t q = 0;
    int k = 0;
    float4 xq = make_float4(0.f, 0.f, 0.f, 0.f);
    double x0 = 0, x1 = 0, x2 = 0, Ji[9], g0 = 0, g1 = 0, g2 = 0, err2 = 0;
#pragma unroll
    for (int e = 0; e < 9; ++e) Ji[e] = 0;
    exact::XState xs{};
    exact::XCache xcache;  // grid values of the last evaluated cell (valid for any solve)
    // Warp-local buffer of 32 queue slots (lane i holds slot base+i): one atomic per 32 solves.
    // Idle lanes are refilled in batches (>= kRefillIdle idle, or the whole warp), so the
    // divergent init path (x0, Jacobian stencil, inverse) runs for many lanes at once and the
    // iteration trips — the bulk of the work — run with most lanes active.
    constexpr int kRefillIdle = kExact ? FSK_REFILL_IDLE_EXACT : FSK_REFILL_IDLE;
    int buf_idx = 0, bused = 32;
    bool dry = false;
    while (true) {
        const unsigned idle = __ballot_sync(full, !active);
        if (!dry && (__popc(idle) >= kRefillIdle || idle == full)) {
            if (bused == 32) {
                int base = 0;
                if (lane == 0) base = atomicAdd(work, 32);
                base = __shfl_sync(full, base, 0);
                buf_idx = base + lane;
                bused = 0;
                dry = base >= cnt;
            }
            const int rank = __popc(idle & ((1u << lane) - 1));
            const bool take = !dry && ((idle >> lane) & 1u) && rank < 32 - bused;
            const int idx = __shfl_sync(full, buf_idx, min(bused + rank, 31));
            const bool got = take && idx < cnt;
            bused += __popc(__ballot_sync(full, take));
            if (__any_sync(full, take && !got)) {  // queue exhausted
#ifdef FSK_ESC_TIMELINE
                if (!dry && lane == 0 && stats) {
                    unsigned long long t;
                    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
                    atomicMax(stats + 41, ~t);  // first warp to find the queue dry (min as max of ~t)
                    atomicMax(stats + 42, t);  // last warp to find it dry
                }
#endif
                dry = true;
            }
            if (got) {  // start of the solve (correspondence.cpp:135-137, :43-54)
                FSK_CHECK(idx >= 0 && idx < cnt && cnt <= esc_cap);
                const int4 rec = esc_q[idx < cnt_long ? idx : esc_cap - 1 - (idx - cnt_long)];
                q = rec.x;
                FSK_CHECK(q >= 0 && q < n * g.nb);
                xq = make_float4(__int_as_float(rec.y), __int_as_float(rec.z), __int_as_float(rec.w), 0.f);
                k = 0;
                double s[16];
                bool conv = false, stop;
                if (idx < st_cap) {  // started by k_esc_start (stopped ones are already stored)
                    const double2* d = st + 8 * (int64_t)idx;
#pragma unroll
                    for (int h = 0; h < 8; ++h) {
                        const double2 v = d[h];
                        s[2 * h] = v.x;
                        s[2 * h + 1] = v.y;
                    }
                    stop = s[6] < 0.0;
                    active = !stop;
                } else {
                    esc_start_one<kExact>(P, g, W, bones, bones64, n, o, rec, s, stop, conv);
                    active = true;
                }
                if constexpr (kExact) {
                    xs.x0 = s[0], xs.x1 = s[1], xs.x2 = s[2], xs.g0 = s[3], xs.g1 = s[4], xs.g2 = s[5];
                    xs.err = s[6], xs.k = 0;
#pragma unroll
                    for (int e = 0; e < 9; ++e) xs.Ji[e] = s[7 + e];
                } else {
                    x0 = s[0], x1 = s[1], x2 = s[2], g0 = s[3], g1 = s[4], g2 = s[5], err2 = s[6];
#pragma unroll
                    for (int e = 0; e < 9; ++e) Ji[e] = s[7 + e];
                }
                if (active && stop) {
                    if constexpr (kExact) store_exact(out, q, xs, conv);
                    else store_solve(out, q, x0, x1, x2, Ji, err2, SolveOut{0, conv, false});
                    n_solves += 1;
                    active = false;
                }
            }
        }
        if (!__any_sync(full, active)) {
            if (dry) break;
            continue;
        }
        if (active) {  // one Broyden iteration (:106-122)
            bool conv, div;
            if constexpr (kExact) {
                conv = exact::step(P, g, xq.x, xq.y, xq.z, o.conv_eps, xs, &xcache);
                div = xs.err > o.div_eps;
            } else {
                double den;
                conv = broyden_step<double>(P, g, xq.x, xq.y, xq.z, conv2, x0, x1, x2, Ji, g0, g1, g2, err2, den);
                div = err2 > div2;
            }
            ++k;
            if (conv || k >= o.max_iters || div) {
                if constexpr (kExact) store_exact(out, q, xs, conv);
                else store_solve(out, q, x0, x1, x2, Ji, err2, SolveOut{k, conv, false});
                n_solves += 1;
                n_iters += k;
                n_final += (conv && k > 0);
                active = false;
            }
        }
    }
#ifdef FSK_ESC_TIMELINE
    if (lane == 0 && stats) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        atomicMax(stats + 43, t);  // last warp exit
    }
#endif
    if (stats) {
        n_solves = __reduce_add_sync(full, n_solves);
        n_iters = __reduce_add_sync(full, n_iters);
        n_final = __reduce_add_sync(full, n_final);
        if (lane == 0 && n_solves) {
            atomicAdd(stats + 3, (unsigned long long)n_solves);
            atomicAdd(stats + 4, (unsigned long long)n_iters);
            atomicAdd(stats + 5, (unsigned long long)n_final);
        }
    }
}

// Exact-replay refill with prefetched work (ablation, off by default): every lane keeps
// its NEXT queue entry — the {q, x'} record and its precomputed start state, 144 B — in a shared-
// memory slot, fetched with cp.async while it iterates. A lane whose solve ends swaps the slot in
// (nine LDS.128, no global latency on the warp) and issues the fetch for the entry after, so lanes
// are refilled as soon as FSK_REFILL_IDLE_PF of them are idle instead of waiting for half the warp
// to idle behind one batched global load. Arithmetic per solve is k_search_escalated<true>'s.
#ifndef FSK_ESC_PREFETCH
#define FSK_ESC_PREFETCH 0  // measured slower on C2: refill 0.268 -> ~0.32-0.36 ms (idle threshold 1/4/8/16), hashes equal
#endif
#ifndef FSK_REFILL_IDLE_PF
#define FSK_REFILL_IDLE_PF 4
#endif
constexpr int kEscSlotF4 = 9;  // float4 words per prefetch slot: record + 8 double2 of start state
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

__global__ void __launch_bounds__(kEscBlock, FSK_ESC_EXACT_MINB)
    k_search_escalated_pf(Planes<double> P, GridP g, const float* __restrict__ W, const float* __restrict__ bones,
                          int64_t n, SearchP o, SearchPlanes out, const int4* __restrict__ esc_q, int64_t esc_cap,
                          const int* __restrict__ esc_count, const double2* __restrict__ st, int st_cap,
                          unsigned long long* __restrict__ stats) {
    const int cnt_long = esc_count[3], cnt = esc_count[3] + esc_count[2];
    const double* bones64 = stage_bones64(bones, g.nb);
    float4* slot = reinterpret_cast<float4*>(const_cast<double*>(bones64) + 12 * g.nb + ((12 * g.nb) & 1)) +
                   kEscSlotF4 * threadIdx.x;
    int* work = const_cast<int*>(esc_count) + 1;
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1;
    unsigned n_solves = 0, n_iters = 0, n_final = 0;
    exact::XState xs{};
    exact::XCache xcache;
    int64_t q = 0;
    float4 xq = make_float4(0.f, 0.f, 0.f, 0.f);
    bool active = false;
    int pend = -1;  // queue index of the entry in this lane's slot (-1: none)
    // warp-local buffer of 32 claimed queue indices (lane i holds base + i): one atomic per 32 claims
    int buf_idx = 0, bused = 32;
    // claim one queue index for every lane with `want` (warp-collective), prefetch it into the slot
    auto claim_and_fetch = [&](bool want) {
        unsigned m = __ballot_sync(full, want);
        int got = -1;
        while (m) {
            if (bused == 32) {
                int base = 0;
                if (lane == 0) base = atomicAdd(work, 32);
                base = __shfl_sync(full, base, 0);
                buf_idx = base + lane;
                bused = 0;
            }
            const int rank = __popc(m & lt);
            const bool take = ((m >> lane) & 1u) && rank < 32 - bused;
            const int idx = __shfl_sync(full, buf_idx, min(bused + rank, 31));
            if (take) got = idx;
            const unsigned tk = __ballot_sync(full, take);
            bused += __popc(tk);
            m &= ~tk;
        }
        if (want) {
            pend = got < cnt ? got : -1;
            if (pend >= 0) {
                FSK_CHECK(pend < cnt && cnt <= esc_cap);
                cp_async16(slot, esc_q + (pend < cnt_long ? pend : esc_cap - 1 - (pend - cnt_long)));
                if (pend < st_cap) {
                    const double2* d = st + 8 * (int64_t)pend;
#pragma unroll
                    for (int h = 0; h < 8; ++h) cp_async16(slot + 1 + h, d + h);
                }
                cp_async_commit();
            }
        }
    };
    claim_and_fetch(true);
    while (true) {
        const bool ready = !active && pend >= 0;
        const unsigned rdy = __ballot_sync(full, ready);
        const unsigned act = __ballot_sync(full, active);
        if (!rdy && !act) break;  // nothing running, nothing fetched: the queue is drained for this warp
        if (rdy && (__popc(rdy) >= FSK_REFILL_IDLE_PF || !act || __popc(~act) == 32)) {
            bool refetch = false;
            if (ready) {  // start of the solve (correspondence.cpp:135-137, :43-54): the prefetched slot
                cp_async_wait_all();
                const int idx = pend;
                const float4 r0 = slot[0];
                const int4 rec = make_int4(__float_as_int(r0.x), __float_as_int(r0.y), __float_as_int(r0.z),
                                           __float_as_int(r0.w));
                q = rec.x;
                FSK_CHECK(q >= 0 && q < n * g.nb);
                xq = make_float4(__int_as_float(rec.y), __int_as_float(rec.z), __int_as_float(rec.w), 0.f);
                double sv[16];
                bool conv = false, stop;
                if (idx < st_cap) {  // started by k_esc_start (stopped ones are already stored)
#pragma unroll
                    for (int h = 0; h < 8; ++h) {
                        const float4 v = slot[1 + h];
                        sv[2 * h] = __hiloint2double(__float_as_int(v.y), __float_as_int(v.x));
                        sv[2 * h + 1] = __hiloint2double(__float_as_int(v.w), __float_as_int(v.z));
                    }
                    stop = sv[6] < 0.0;
                    active = !stop;
                } else {
                    esc_start_one<true>(P, g, W, bones, bones64, n, o, rec, sv, stop, conv);
                    active = true;
                }
                xs.x0 = sv[0], xs.x1 = sv[1], xs.x2 = sv[2], xs.g0 = sv[3], xs.g1 = sv[4], xs.g2 = sv[5];
                xs.err = sv[6], xs.k = 0;
#pragma unroll
                for (int e = 0; e < 9; ++e) xs.Ji[e] = sv[7 + e];
                if (active && stop) {
                    store_exact(out, q, xs, conv);
                    n_solves += 1;
                    active = false;
                }
                refetch = true;
            }
            claim_and_fetch(refetch);
        }
        if (active) {  // one Broyden iteration (:106-122)
            const bool conv = exact::step(P, g, xq.x, xq.y, xq.z, o.conv_eps, xs, &xcache);
            const bool div = xs.err > o.div_eps;
            if (conv || xs.k >= o.max_iters || div) {
                store_exact(out, q, xs, conv);
                n_solves += 1;
                n_iters += xs.k;
                n_final += (conv && xs.k > 0);
                active = false;
            }
        }
    }
    cp_async_wait_all();
    if (stats) {
        n_solves = __reduce_add_sync(full, n_solves);
        n_iters = __reduce_add_sync(full, n_iters);
        n_final = __reduce_add_sync(full, n_final);
        if (lane == 0 && n_solves) {
            atomicAdd(stats + 3, (unsigned long long)n_solves);
            atomicAdd(stats + 4, (unsigned long long)n_iters);
            atomicAdd(stats + 5, (unsigned long long)n_final);
        }
    }
}

// Parity mode: every solve in float64.
__global__ void __launch_bounds__(128) k_search_f64(Planes<double> P, GridP g, const float* __restrict__ bones,
                                                    const float4* __restrict__ xs, int64_t n, int blocks_per_bone,
                                                    SearchP o, SearchPlanes out, unsigned long long* __restrict__ stats) {
    const int bone = blockIdx.x / blocks_per_bone;
    const int64_t j = (int64_t)(blockIdx.x - bone * blocks_per_bone) * 128 + threadIdx.x;
    if (j >= n) return;
    const float4 xq = __ldg(xs + j);
    double x0, x1, x2, Ji[9], err2;
    const SolveOut s = solve_one<double, false>(P, g, bones + 12 * bone, xq.x, xq.y, xq.z, o, x0, x1, x2, Ji, err2);
    store_solve(out, (int64_t)bone * n + j, x0, x1, x2, Ji, err2, s);
    count_work(stats ? stats + 3 : nullptr, s);
}

// Exact replay mode (FSK_SEARCH_EXACT64): every solve in float64 with the oracle's restatement of the
// reference's operation order (fsk_exact.cuh), J~0 from the n_b-wide weight grid — bit-identical to the
// oracle's search_one (correspondence.cpp:126-150) given the same float64 transform grid.
__global__ void __launch_bounds__(128) k_search_exact(Planes<double> P, GridP g, const float* __restrict__ W,
                                                      const float* __restrict__ bones, const float4* __restrict__ xs,
                                                      int64_t n, int blocks_per_bone, SearchP o, SearchPlanes out,
                                                      unsigned long long* __restrict__ stats) {
    const int bone = blockIdx.x / blocks_per_bone;
    const int64_t j = (int64_t)(blockIdx.x - bone * blocks_per_bone) * 128 + threadIdx.x;
    const double* bones64 = stage_bones64(bones, g.nb);
    if (j >= n) return;
    const float4 xq = __ldg(xs + j);
    const double xp0 = xq.x, xp1 = xq.y, xp2 = xq.z;
    exact::XState s;
    exact::start(P, g, W, bones64, bone, xp0, xp1, xp2, s);
    bool conv = s.err < o.conv_eps;  // iterate (correspondence.cpp:97-124)
    if (!conv)
        for (int k = 0; k < o.max_iters; ++k) {
            if (s.err > o.div_eps) break;
            if (exact::step(P, g, xp0, xp1, xp2, o.conv_eps, s)) {
                conv = true;
                break;
            }
        }
    store_exact(out, (int64_t)bone * n + j, s, conv);
    count_work(stats ? stats + 3 : nullptr, SolveOut{s.k, conv, false, false});
}

// ============================================================================ dedup
#ifndef FSK_DEDUP_BATCH
#define FSK_DEDUP_BATCH 6  // plane rows in flight per batch: 24 35 us, 12 30, 8 28, 6 26, 4 26 (C2; fewer registers, more warps)
#endif
// One query's dedup. kStaged: the query's n_b plane rows were bulk-copied to shared memory
// (row b at srow[b * kDedupTile]); else they are loaded from the planes kBatch bones at a time.
template <bool kStaged>
__device__ __forceinline__ void dedup_query(int64_t j, int64_t n, int nb, float dedup2, const SearchPlanes& sp,
                                            const int* __restrict__ perm, int32_t* __restrict__ n_roots_p,
                                            const float4* srow = nullptr) {
    // The first kRegKept kept roots stay in registers (a query has ~1 root); later kept roots
    // are re-read from the planes. Converged = sign bit of the residual clear.
    constexpr int kRegKept = 4, kBatch = kStaged ? 1 : FSK_DEDUP_BATCH;
    constexpr int kStride = 128;  // kDedupTile
    float kx[kRegKept], ky[kRegKept], kz[kRegKept];
#pragma unroll
    for (int c = 0; c < kRegKept; ++c) kx[c] = ky[c] = kz[c] = 0.f;
    int count = 0;
    uint32_t kept = 0;  // bit b: bone b's root kept (used when n_b <= 32)
    for (int b0 = 0; b0 < nb; b0 += kBatch) {
        float4 xv[kBatch];
#pragma unroll
        for (int i = 0; i < kBatch; ++i)
            if (b0 + i < nb) xv[i] = kStaged ? srow[(b0 + i) * kStride] : __ldcs(sp.xr + (int64_t)(b0 + i) * n + j);
#pragma unroll
        for (int i = 0; i < kBatch; ++i) {
            const int b = b0 + i;
            if (b >= nb) continue;
            int k = 0;
            if (!signbit(xv[i].w)) {
                k = 1;
#pragma unroll
                for (int c = 0; c < kRegKept; ++c) {
                    const float e0 = xv[i].x - kx[c], e1 = xv[i].y - ky[c], e2 = xv[i].z - kz[c];
                    if (c < count && e0 * e0 + e1 * e1 + e2 * e2 < dedup2) k = 0;
                }
                if (k && count > kRegKept) {  // rare: compare with the kept roots beyond the registers
                    int seen = 0;
                    for (int c = 0; c < b && k; ++c) {
                        const int64_t qc = (int64_t)c * n + j;
                        if (!sp.keep[qc]) continue;
                        if (seen++ < kRegKept) continue;
                        const float4 e = sp.xr[qc];
                        const float e0 = xv[i].x - e.x, e1 = xv[i].y - e.y, e2 = xv[i].z - e.z;
                        if (e0 * e0 + e1 * e1 + e2 * e2 < dedup2) k = 0;
                    }
                }
                if (k) {
#pragma unroll
                    for (int c = 0; c < kRegKept; ++c)
                        if (c == count) {
                            kx[c] = xv[i].x;
                            ky[c] = xv[i].y;
                            kz[c] = xv[i].z;
                        }
                }
            }
            sp.keep[(int64_t)b * n + j] = (uint8_t)k;
            kept |= (uint32_t)k << (b & 31);
            count += k;
        }
    }
    if (sp.kmask) sp.kmask[j] = kept;
    n_roots_p[perm[j]] = count;
}

// dedup_roots over each query's converged inits in bone order: a root is kept iff
// ||x − k|| >= dedup_dist for every already-kept k (strict '<' drops; :162-176).
// One thread per sorted query; all loads of a warp are coalesced rows of the planes.
__global__ void __launch_bounds__(256) k_dedup(int64_t n, int nb, float dedup2, SearchPlanes sp,
                                               const int* __restrict__ perm, int32_t* __restrict__ n_roots_p) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= n) return;
    dedup_query<false>(j, n, nb, dedup2, sp, perm, n_roots_p);
}

// The same with the block's n_b plane rows (128 queries × 16 B each) brought into shared memory by
// n_b TMA bulk copies (cp.async.bulk, one mbarrier): long DRAM bursts instead of 24 interleaved
// 512-B streams per warp. Ablation (off by default).
#ifndef FSK_DEDUP_BULK
#define FSK_DEDUP_BULK 0  // measured slower on C2: 36.0 us vs 26.3 for k_dedup (outputs bitwise equal)
#endif
constexpr int kDedupTile = 128;
__device__ __forceinline__ uint32_t sm_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void __launch_bounds__(kDedupTile) k_dedup_bulk(int64_t n, int nb, float dedup2, SearchPlanes sp,
                                                          const int* __restrict__ perm,
                                                          int32_t* __restrict__ n_roots_p) {
    extern __shared__ __align__(16) float4 s_rows[];  // [nb][kDedupTile]
    __shared__ __align__(8) uint64_t bar;
    const int64_t j0 = blockIdx.x * (int64_t)kDedupTile;
    const int cnt = (int)min((int64_t)kDedupTile, n - j0);
    const uint32_t b = sm_u32(&bar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t bytes = (uint32_t)cnt * 16u;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes * (uint32_t)nb)
                     : "memory");
        for (int r = 0; r < nb; ++r)
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    sm_u32(s_rows + r * kDedupTile)),
                "l"(sp.xr + (int64_t)r * n + j0), "r"(bytes), "r"(b)
                : "memory");
    }
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t"
        "@!P1 bra WAIT_%=;\n\t}" ::"r"(b)
        : "memory");
    if ((int)threadIdx.x < cnt) dedup_query<true>(j0 + threadIdx.x, n, nb, dedup2, sp, perm, n_roots_p, s_rows + threadIdx.x);
}

void launch_dedup(fsk_ctx* ctx, cudaStream_t st, int64_t n, int nb, float dedup2, const SearchPlanes& sp,
                  const int* perm, int32_t* n_roots) {
    const size_t smem = (size_t)nb * kDedupTile * sizeof(float4);
    if (FSK_DEDUP_BULK && n > 0 && smem <= 96 * 1024) {
        // (the static mbarrier counts against the 48 KB default too: always raise the limit)
        cuda_check(cudaFuncSetAttribute(k_dedup_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024),
                   "cudaFuncSetAttribute");
        FSK_LAUNCH(ctx, st, k_dedup_bulk, blocks_for(n, kDedupTile), kDedupTile, smem, n, nb, dedup2, sp, perm, n_roots);
    } else {
        FSK_LAUNCH(ctx, st, k_dedup, blocks_for(n, 256), 256, 0, n, nb, dedup2, sp, perm, n_roots);
    }
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

// The spatial sort in one cooperative launch (grid = one 1024-thread block per SM, all
// co-resident): bbox → grid sync → Morton keys + histogram → grid sync → bucket scan (block
// sums, grid sync, prefix) → grid sync → scatter. Same keys, buckets and within-bucket
// atomics as the four-kernel form (k_sort_bbox/_hist/_scan/_scatter). Ablation (off by default).
#ifndef FSK_SORT_FUSED
#define FSK_SORT_FUSED 0  // measured slower: C2 step 0.967 -> 0.988 ms (38.9 us alone vs 41.6 for the four kernels, and it no longer overlaps K1); C5 sort 365 -> 379 us
#endif
__global__ void __launch_bounds__(1024) k_sort_fused(const float* __restrict__ x, int64_t n, int* __restrict__ state,
                                                     uint16_t* __restrict__ keys, int* __restrict__ perm,
                                                     float4* __restrict__ xs) {
    cg::grid_group grid = cg::this_grid();
    unsigned* bbox = (unsigned*)(state + kBboxOff);
    int* hist = state;
    int* sums = state + kSortSumsOff;
    const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, stride = (int64_t)gridDim.x * blockDim.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __shared__ float s_lo[3][32], s_hi[3][32];
    __shared__ int64_t wt[32];
    __shared__ int64_t tot;
    __shared__ int s_prefix;
    {  // 1. bbox of the finite coordinates (k_sort_bbox)
        float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
        for (int64_t p = t0; p < n; p += stride) {
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
            if (lane == 0) {
                s_lo[a][warp] = lo[a];
                s_hi[a][warp] = hi[a];
            }
        }
        __syncthreads();
        if (threadIdx.x < 3) {
            const int a = threadIdx.x;
            float l = s_lo[a][0], h = s_hi[a][0];
            for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
                l = fminf(l, s_lo[a][w]);
                h = fmaxf(h, s_hi[a][w]);
            }
            atomicMax(bbox + a, ~bb_enc(l));
            atomicMax(bbox + 3 + a, bb_enc(h));
        }
    }
    grid.sync();
    {  // 2. Morton keys + bucket histogram (k_sort_hist)
        float lo[3], sc[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            lo[a] = bb_dec(~__ldcg(bbox + a));
            const float hi = bb_dec(__ldcg(bbox + 3 + a));
            sc[a] = (float)(1 << kSortBitsPerAxis) / fmaxf(hi - lo[a], 1e-30f);
        }
        for (int64_t p = t0; p < n; p += stride) {
            uint32_t q[3];
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                const float u = (x[3 * p + a] - lo[a]) * sc[a];
                const int qi = isfinite(u) ? __float2int_rd(u) : 0;
                q[a] = (uint32_t)max(0, min(qi, (1 << kSortBitsPerAxis) - 1));
            }
            const uint32_t k = spread3(q[0]) | (spread3(q[1]) << 1) | (spread3(q[2]) << 2);
            keys[p] = (uint16_t)k;
            atomicAdd(hist + k, 1);
        }
    }
    grid.sync();
    // 3. exclusive scan of the buckets: block b owns a contiguous chunk (at most one bucket per thread)
    const int chunk = (kSortBuckets + gridDim.x - 1) / gridDim.x;
    const int bk = blockIdx.x * chunk + threadIdx.x;
    const bool mine = threadIdx.x < chunk && bk < kSortBuckets;
    const int v = mine ? __ldcg(hist + bk) : 0;
    const int64_t ex = block_excl_scan(v, wt, &tot);
    if (threadIdx.x == 0) sums[blockIdx.x] = (int)tot;
    grid.sync();
    {
        int64_t pre = 0;
        for (int i = threadIdx.x; i < (int)blockIdx.x; i += blockDim.x) pre += __ldcg(sums + i);
        for (int o = 16; o > 0; o >>= 1) pre += __shfl_xor_sync(0xffffffff, pre, o);
        if (lane == 0) wt[warp] = pre;
        __syncthreads();
        if (threadIdx.x == 0) {
            int64_t p = 0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) p += wt[w];
            s_prefix = (int)p;
        }
        __syncthreads();
    }
    if (mine) hist[bk] = s_prefix + (int)ex;
    grid.sync();
    // 4. scatter into sorted order (k_sort_scatter)
    for (int64_t p = t0; p < n; p += stride) {
        const int pos = atomicAdd(hist + keys[p], 1);
        FSK_CHECK(pos >= 0 && pos < n);
        perm[pos] = (int)p;
        xs[pos] = make_float4(x[3 * p], x[3 * p + 1], x[3 * p + 2], 0.f);
    }
}

// Single-pass form of the scan for the search's root counts (decoupled look-back): each block
// takes a tile by ticket (so every tile it waits on has started), publishes its aggregate, then
// walks back over its predecessors' published aggregates / inclusive prefixes. Status word per
// tile: flag (bits 62-63: 1 aggregate, 2 inclusive prefix) | epoch (bits 32-61) | value (bits
// 0-31; the counts total at most n·n_b < 2^31). The epoch (advanced by the last tile) retires
// the previous launch's words without a memset, so the launch is graph-replayable.
// ctl[0] = ticket, ctl[1] = epoch; the buffer is zeroed when allocated.
#ifndef FSK_SCAN_LOOKBACK
#define FSK_SCAN_LOOKBACK 1
#endif
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__global__ void __launch_bounds__(kScanThreads) k_scan_lookback(const int32_t* __restrict__ in, int64_t n,
                                                                unsigned* __restrict__ ctl,
                                                                unsigned long long* __restrict__ status,
                                                                int64_t* __restrict__ out) {
    __shared__ int64_t wt[32];
    __shared__ int64_t tot;
    __shared__ unsigned s_tile, s_epoch;
    __shared__ int64_t s_prefix;
    const unsigned ntiles = (unsigned)((n + kScanTile - 1) / kScanTile);
    if (threadIdx.x == 0) {
        s_epoch = *(volatile unsigned*)(ctl + 1);
        s_tile = atomicAdd(ctl, 1u);
    }
    __syncthreads();
    const unsigned tile = s_tile;
    const unsigned long long ep = (unsigned long long)(s_epoch & 0x3fffffffu) << 32;
    const int64_t base = tile * (int64_t)kScanTile + threadIdx.x * kScanPer;
    int64_t v[kScanPer];
    int64_t sum = 0;
#pragma unroll
    for (int i = 0; i < kScanPer; ++i) {
        v[i] = (base + i < n) ? in[base + i] : 0;
        sum += v[i];
    }
    const int64_t excl = block_excl_scan(sum, wt, &tot);
    if (threadIdx.x == 0) {
        const unsigned long long agg = (unsigned long long)(uint32_t)tot;
        int64_t pre = 0;
        if (tile == 0) {
            st_relaxed_u64(status, (2ull << 62) | ep | agg);
        } else {
            st_relaxed_u64(status + tile, (1ull << 62) | ep | agg);
            for (int64_t t = (int64_t)tile - 1;; --t) {
                unsigned long long w;
                do {
                    w = ld_relaxed_u64(status + t);
                } while ((w & 0x3fffffff00000000ull) != ep || (w >> 62) == 0);
                pre += (int64_t)(w & 0xffffffffull);
                if ((w >> 62) == 2) break;
            }
            st_relaxed_u64(status + tile, (2ull << 62) | ep | (unsigned long long)(uint32_t)(pre + tot));
        }
        s_prefix = pre;
        if (tile == ntiles - 1) {  // the last ticket: every block has read the epoch and taken its ticket
            out[n] = pre + tot;
            ctl[0] = 0;
            ctl[1] = (s_epoch + 1) & 0x3fffffffu;
        }
    }
    __syncthreads();
    int64_t run = s_prefix + excl;
#pragma unroll
    for (int i = 0; i < kScanPer; ++i) {
        if (base + i < n) out[base + i] = run;
        run += v[i];
    }
}

// ============================================================================ compaction
__device__ __forceinline__ void store_root(fsk_root* dst, float4 xr, float4 ja, float4 jb, float jc, int bone,
                                           int iters) {
    float4* d = reinterpret_cast<float4*>(dst);
    d[0] = xr;  // x[3], residual
    d[1] = ja;  // J~[0..3]
    d[2] = jb;  // J~[4..7]
    d[3] = make_float4(jc, __int_as_float(bone), __int_as_float(iters), 0.f);
}

// Kept roots of each query, in bone order, at offsets[p] (CorrespondenceSet::roots).
// Records at index >= cap are dropped (the caller checks offsets[N] <= cap).
__global__ void __launch_bounds__(256) k_emit(int64_t n, int nb, SearchPlanes sp, const int* __restrict__ perm,
                                              const int64_t* __restrict__ offs, fsk_root* __restrict__ roots,
                                              int64_t cap) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= n) return;
    int64_t o = offs[perm[j]];
    if (sp.kmask) {  // the kept bones straight from dedup's mask (≈ 1 per query) instead of n_b keep bytes
        for (uint32_t m = sp.kmask[j]; m; m &= m - 1) {
            const int b = __ffs(m) - 1;
            const int64_t q = (int64_t)b * n + j;
            FSK_CHECK(b < nb && o >= offs[perm[j]] && o < offs[perm[j]] + nb);
            if (o < cap) {
                float4 xr = sp.xr[q];
                xr.w = fabsf(xr.w);
                store_root(roots + o, xr, sp.ja[q], sp.jb[q], sp.jc[q], b, (int)(sp.meta[q] & 0x3fffffffu));
            }
            ++o;
        }
        return;
    }
    for (int b = 0; b < nb; ++b) {
        const int64_t q = (int64_t)b * n + j;
        if (!sp.keep[q]) continue;
        if (o < cap) {
            float4 xr = sp.xr[q];
            xr.w = fabsf(xr.w);
            store_root(roots + o, xr, sp.ja[q], sp.jb[q], sp.jc[q], b, (int)(sp.meta[q] & 0x3fffffffu));
        }
        ++o;
    }
}

// Dense per-(point, init) form, point-major (fsk_search_out). One thread per solve.
struct DenseOut {
    double* x_c64;
    float* x_c;
    float* jinv;
    float* resid;
    int32_t* iters;
    uint8_t* converged;
    uint8_t* keep;
    int32_t* n_roots;
};

__global__ void __launch_bounds__(256) k_scatter_dense(int64_t n, int nb, SearchPlanes sp, const int* __restrict__ perm,
                                                       DenseOut d) {
    const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= n * nb) return;
    const int b = (int)(q / n);
    const int64_t j = q - (int64_t)b * n;
    const int64_t s = (int64_t)perm[j] * nb + b;
    const float4 xr = sp.xr[q];
    if (d.x_c64) {
        d.x_c64[3 * s] = sp.xd ? sp.xd[3 * q] : (double)xr.x;
        d.x_c64[3 * s + 1] = sp.xd ? sp.xd[3 * q + 1] : (double)xr.y;
        d.x_c64[3 * s + 2] = sp.xd ? sp.xd[3 * q + 2] : (double)xr.z;
    }
    if (d.x_c) {
        d.x_c[3 * s] = xr.x;
        d.x_c[3 * s + 1] = xr.y;
        d.x_c[3 * s + 2] = xr.z;
    }
    if (d.resid) d.resid[s] = fabsf(xr.w);
    const uint32_t mq = sp.meta[q];
    if (d.jinv && !(mq & 0x40000000u)) {  // J~ not stored (an unconverged float32 solve: no Root): NaN
        for (int e = 0; e < 9; ++e) d.jinv[9 * s + e] = __int_as_float(0x7fc00000);
    } else if (d.jinv) {
        const float4 a = sp.ja[q], c = sp.jb[q];
        float* J = d.jinv + 9 * s;
        J[0] = a.x; J[1] = a.y; J[2] = a.z; J[3] = a.w;
        J[4] = c.x; J[5] = c.y; J[6] = c.z; J[7] = c.w;
        J[8] = sp.jc[q];
    }
    const uint32_t m = sp.meta[q];
    if (d.iters) d.iters[s] = (int32_t)(m & 0x3fffffffu);
    d.converged[s] = (uint8_t)(m >> 31);
    if (d.keep) d.keep[s] = sp.keep[q];
}

// Compaction of a caller-held dense result (fsk_compact_roots).
__global__ void __launch_bounds__(256) k_emit_dense(int64_t n, int nb, DenseOut d, const int64_t* __restrict__ offs,
                                                    fsk_root* __restrict__ roots) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n) return;
    int64_t o = offs[p];
    for (int i = 0; i < nb; ++i) {
        const int64_t s = p * nb + i;
        if (!d.keep[s]) continue;
        const float* J = d.jinv ? d.jinv + 9 * s : nullptr;
        store_root(roots + o, make_float4(d.x_c[3 * s], d.x_c[3 * s + 1], d.x_c[3 * s + 2], d.resid ? d.resid[s] : 0.f),
                   J ? make_float4(J[0], J[1], J[2], J[3]) : make_float4(0.f, 0.f, 0.f, 0.f),
                   J ? make_float4(J[4], J[5], J[6], J[7]) : make_float4(0.f, 0.f, 0.f, 0.f), J ? J[8] : 0.f, i,
                   d.iters ? d.iters[s] : 0);
        ++o;
    }
}


// ============================================================================ E
__global__ void __launch_bounds__(256) k_eval_points(Planes<float> P, GridP g, const float* __restrict__ x, int64_t n,
                                                     float* __restrict__ t12, float* __restrict__ dout,
                                                     float* __restrict__ jac) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n) return;
    const float x0 = x[3 * p], x1 = x[3 * p + 1], x2 = x[3 * p + 2];
    float T[12], J[9], d[3];
    jacobian_and_T<float>(P, g, x0, x1, x2, T, J);
    apply_T<float>(T, x0, x1, x2, d);
    if (t12)
        for (int e = 0; e < 12; ++e) t12[12 * p + e] = T[e];
    if (dout)
        for (int e = 0; e < 3; ++e) dout[3 * p + e] = d[e];
    if (jac)
        for (int e = 0; e < 9; ++e) jac[9 * p + e] = J[e];
}

// init_states (correspondence.cpp:58-70): one thread per (point, bone), point-major output.
__global__ void __launch_bounds__(256) k_init_states(Planes<float> P, GridP g, const float* __restrict__ bones,
                                                     const float* __restrict__ pts, int64_t n, float* __restrict__ x0o,
                                                     float* __restrict__ jo) {
    const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (s >= n * g.nb) return;
    const int64_t p = s / g.nb;
    const int bone = (int)(s - p * g.nb);
    float x0, x1, x2, Ji[9], T[12];
    solve_init<float>(P, g, bones + 12 * bone, pts[3 * p], pts[3 * p + 1], pts[3 * p + 2], x0, x1, x2, Ji, T);
    if (x0o) {
        x0o[3 * s] = x0;
        x0o[3 * s + 1] = x1;
        x0o[3 * s + 2] = x2;
    }
    if (jo)
        for (int e = 0; e < 9; ++e) jo[9 * s + e] = Ji[e];
}

// init_states in float64 with the reference's operation order (fsk_exact.cuh): x0 = B_i^-1 x' and
// J~0 = J(x0)^-1 from the n_b-wide weight grid (correspondence.cpp:43-70), one thread per (point,
// bone), point-major output — what the drop-in's init_states returns.
__global__ void __launch_bounds__(128) k_init_states64(GridP g, const float* __restrict__ W, const float* __restrict__ bones,
                                                       const double* __restrict__ pts, int64_t n,
                                                       double* __restrict__ x0o, double* __restrict__ jo) {
    const double* bones64 = stage_bones64(bones, g.nb);
    const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (s >= n * g.nb) return;
    const int64_t p = s / g.nb;
    const int bone = (int)(s - p * g.nb);
    double x0, x1, x2, J[9], Ji[9];
    exact::inverse_apply(bones64 + 12 * bone, pts[3 * p], pts[3 * p + 1], pts[3 * p + 2], x0, x1, x2);
    exact::jacobian(g, W, bones64, x0, x1, x2, J);
    exact::inverse_or_identity(J, Ji);
    if (x0o) {
        x0o[3 * s] = x0;
        x0o[3 * s + 1] = x1;
        x0o[3 * s + 2] = x2;
    }
    if (jo)
        for (int e = 0; e < 9; ++e) jo[9 * s + e] = Ji[e];
}

// ============================================================================ host pipeline
namespace {

int64_t vertex_count(const GridP& g) { return (int64_t)g.nx * g.ny * g.nz; }

struct GridPlanes {
    Planes<float> p32;
    Planes<double> p64;
};

// scratch of the sort / K1 stage: slot 1 is the second copy the host pipeline stages into
int sslot(int base, int slot) {
    if (!slot) return base;
    switch (base) {
        case kHist: return kHistB;
        case kKeys: return kKeysB;
        case kPerm: return kPermB;
        case kXs: return kXsB;
        case kEscN: return kEscNB;
        case kPlanes: return kPlanesB;
        case kPlanes64: return kPlanes64B;
        default: return base;
    }
}

GridPlanes planes_scratch(fsk_ctx* ctx, const GridP& g, int slot = 0) {
    const int64_t V = vertex_count(g);
    GridPlanes P;
    P.p32.p = (const float*)scratch(ctx, sslot(kPlanes, slot), 3 * V * 8 * sizeof(float));
    P.p32.stride = V * 8;
    P.p64.p = (const double*)scratch(ctx, sslot(kPlanes64, slot), 3 * V * 8 * sizeof(double));
    P.p64.stride = V * 8;
    return P;
}

bool needs_f64(int flags) { return !(flags & FSK_SEARCH_FP32_ONLY); }

// K1: tg / tg64 outputs optional; planes in both precisions when `planes`.
GridPlanes run_precompute(fsk_ctx* ctx, const float* w, const GridP& g, const float* bones, float* tg, double* tg64,
                          bool planes, bool f64, cudaStream_t st, int slot = 0) {
    const int64_t V = vertex_count(g);
    GridPlanes P = planes_scratch(ctx, g, slot);
#ifdef FSK_K1_V1
    FSK_LAUNCH(ctx, st, k_precompute, blocks_for(3 * V, 256), 256, g.nb * 12 * sizeof(float), w, bones, g.nb, g.nx, V,
               reinterpret_cast<float4*>(tg), planes ? (float*)P.p32.p : nullptr,
               planes && f64 ? (double*)P.p64.p : nullptr, tg64);
#else
    FSK_LAUNCH(ctx, st, k_precompute_v, blocks_for(V, 128), 128, g.nb * 12 * sizeof(float), w, bones, g.nb, g.nx, V,
               reinterpret_cast<float4*>(tg), planes ? (float*)P.p32.p : nullptr,
               planes && f64 ? (double*)P.p64.p : nullptr, tg64);
#endif
    return P;
}

GridPlanes run_relayout(fsk_ctx* ctx, const float* tg, const double* tg64, const GridP& g, bool f64, cudaStream_t st) {
    const int64_t V = vertex_count(g);
    GridPlanes P = planes_scratch(ctx, g);
    FSK_LAUNCH(ctx, st, k_relayout, blocks_for(V, 256), 256, 0, tg, tg64, g.nx, V, (float*)P.p32.p,
               f64 ? (double*)P.p64.p : nullptr);
    return P;
}

struct SearchState {
    SearchPlanes sp;
    int* perm;
    int32_t* n_roots_p;
};

// K1 issued by run_search itself, concurrently with the spatial sort (which only reads the points)
struct PrecomputeReq {
    const float* w;
    const float* bones;
    float* tg;
    bool f64;
};

// sort + K2 (+ K2b escalation) + dedup into the ctx's search planes. With `pre`, K1 runs on `st`
// while the sort runs on the ctx's side stream (fork/join by events, capturable in a graph), and
// P is filled in here.
// cooperative launch of k_sort_fused: one block per SM (all co-resident; capturable in graphs)
void sort_fused(fsk_ctx* ctx, cudaStream_t st, const float* pts, int64_t n, int* state, uint16_t* keys, int* perm,
                float4* xs) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)ctx->sm_count);
    cfg.blockDim = dim3(1024);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    prof_begin(ctx, st);
    cuda_check(cudaLaunchKernelEx(&cfg, k_sort_fused, pts, n, state, keys, perm, xs), "k_sort_fused");
    after_launch(ctx, "k_sort_fused");
}

// mode: the whole search (kRunFull), only its sort + K1 stage into the given scratch slot (kRunStage),
// or everything after a stage already done into that slot (kRunAfterStage: P = the slot's planes)
enum { kRunFull = 0, kRunStage = 1, kRunAfterStage = 2 };
SearchState run_search(fsk_ctx* ctx, GridPlanes& P, const GridP& g, const float* weights, const float* bones,
                       const float* pts, int64_t n, const SearchP& sp, int flags, cudaStream_t st,
                       const PrecomputeReq* pre = nullptr, bool want_x64 = false, int mode = kRunFull, int slot = 0) {
    if ((flags & FSK_SEARCH_EXACT64) && !weights)
        fail(FSK_EINVAL, "fsk: FSK_SEARCH_EXACT64 needs the weight grid (J~0 from the skinning weights)");
    // the exact replay reads the weight grid and float64 copies of the bones (shared memory)
    const bool exact_any = weights && ((flags & FSK_SEARCH_EXACT64) ||
                                       !(flags & (FSK_SEARCH_FAST_ESC | FSK_SEARCH_FP32_ONLY | FSK_SEARCH_FP64)));
    const size_t smem64 = (size_t)g.nb * 12 * sizeof(double);
    const float* Wx = exact_any ? weights : nullptr;
    if (n >= (int64_t(1) << 31) / std::max(1, g.nb)) fail(FSK_EINVAL, "fsk: too many points for one call (split the batch)");
    const int64_t S = std::max<int64_t>(1, n * g.nb);
    SearchState s;
    auto precompute = [&] {
        if (pre && mode != kRunAfterStage)
            P = run_precompute(ctx, pre->w, g, pre->bones, pre->tg, nullptr, true, pre->f64, st, slot);
    };
    if (mode == kRunStage) {  // sort + K1 only (the search scratch belongs to the item searching meanwhile)
        s.perm = (int*)scratch(ctx, sslot(kPerm, slot), std::max<int64_t>(1, n) * sizeof(int));
        s.n_roots_p = nullptr;
    } else {
    s.sp.xr = (float4*)scratch(ctx, kOXr, S * sizeof(float4));
    s.sp.ja = (float4*)scratch(ctx, kOJa, S * sizeof(float4));
    s.sp.jb = (float4*)scratch(ctx, kOJb, S * sizeof(float4));
    s.sp.jc = (float*)scratch(ctx, kOJc, S * sizeof(float));
    s.sp.meta = (uint32_t*)scratch(ctx, kOMeta, S * sizeof(uint32_t));
    s.sp.keep = (uint8_t*)scratch(ctx, kOKeep, S);
    s.sp.kmask = g.nb <= 32 ? (uint32_t*)scratch(ctx, kOKeepMask, std::max<int64_t>(1, n) * sizeof(uint32_t)) : nullptr;
    s.sp.xd = want_x64 ? (double*)scratch(ctx, kOXd, S * 3 * sizeof(double)) : nullptr;
    s.perm = (int*)scratch(ctx, sslot(kPerm, slot), std::max<int64_t>(1, n) * sizeof(int));
    if (slot == 0) ctx->last_search_n = n;  // fsk_ctx_query_order reads slot 0
    s.n_roots_p = (int32_t*)scratch(ctx, kNRoots, std::max<int64_t>(1, n) * sizeof(int32_t));
    }
    if (n == 0) {
        precompute();
        return s;
    }
    float4* xs = (float4*)scratch(ctx, sslot(kXs, slot), n * sizeof(float4));
    int* esc_n = (int*)scratch(ctx, sslot(kEscN, slot), 4 * sizeof(int));  // {-, work cursor, short count, long count}
    // (with the spatial sort, the counters live in the sort state and are zeroed with it)
    if (mode == kRunAfterStage) {
        if (!(flags & FSK_SEARCH_NO_SORT))
            esc_n = (int*)scratch(ctx, sslot(kHist, slot), kSortStateInts * sizeof(int)) + kEscOff;
    } else if (!(flags & FSK_SEARCH_NO_SORT)) {
        int* hist = (int*)scratch(ctx, sslot(kHist, slot), kSortStateInts * sizeof(int));
        unsigned* bbox = (unsigned*)(hist + kBboxOff);
        esc_n = hist + kEscOff;  // zeroed with the histogram
        uint16_t* keys = (uint16_t*)scratch(ctx, sslot(kKeys, slot), n * sizeof(uint16_t));
        cudaStream_t ss = st;
        if (pre) {  // fork: the sort on the side stream, K1 on st
            cuda_check(cudaEventRecord(ctx->ev_fork, st), "cudaEventRecord");
            cuda_check(cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0), "cudaStreamWaitEvent");
            ss = ctx->side;
        }
        cuda_check(cudaMemsetAsync(hist, 0, kSortStateInts * sizeof(int), ss), "cudaMemsetAsync");
        if (FSK_SORT_FUSED && ctx->sm_count <= kSortMaxBlocks) {
            sort_fused(ctx, ss, pts, n, hist, keys, s.perm, xs);
        } else {
            const unsigned gb = (unsigned)std::min<int64_t>(blocks_for(n, 256), (int64_t)ctx->sm_count * FSK_SORT_BBOX_BLOCKS_PER_SM);
            FSK_LAUNCH(ctx, ss, k_sort_bbox, gb, 256, 0, pts, n, bbox);
            FSK_LAUNCH(ctx, ss, k_sort_hist, blocks_for(n, 256), 256, 0, pts, n, bbox, keys, hist);
            if (FSK_SORT_SCAN1)
                FSK_LAUNCH(ctx, ss, k_sort_scan1, 1, 1024, 0, hist);
            else
                FSK_LAUNCH(ctx, ss, k_sort_scan, kScanBlocks, 1024, 0, hist, hist + kScanBarOff);
            FSK_LAUNCH(ctx, ss, k_sort_scatter, blocks_for(n, 256), 256, 0, pts, keys, n, hist, s.perm, xs);
        }
        if (pre) {  // join
            cuda_check(cudaEventRecord(ctx->ev_join, ss), "cudaEventRecord");
            precompute();
            cuda_check(cudaStreamWaitEvent(st, ctx->ev_join, 0), "cudaStreamWaitEvent");
        }
    } else {
        precompute();
        FSK_LAUNCH(ctx, st, k_identity_order, blocks_for(n, 256), 256, 0, pts, n, s.perm, xs, esc_n);
    }
    if (mode == kRunStage) return s;
    if (flags & FSK_SEARCH_EXACT64) {
        const int bpb = (int)blocks_for(n, 128);
        const int64_t nblocks = (int64_t)bpb * g.nb;
        if (nblocks >= (int64_t(1) << 31)) fail(FSK_EINVAL, "fsk: search grid too large");
        FSK_LAUNCH(ctx, st, k_search_exact, (unsigned)nblocks, 128, smem64, P.p64, g, Wx, bones, xs, n, bpb, sp, s.sp,
                   ctx->stats);
    } else if (flags & FSK_SEARCH_FP64) {
        const int bpb = (int)blocks_for(n, 128);
        const int64_t nblocks = (int64_t)bpb * g.nb;
        if (nblocks >= (int64_t(1) << 31)) fail(FSK_EINVAL, "fsk: search grid too large");
        FSK_LAUNCH(ctx, st, k_search_f64, (unsigned)nblocks, 128, 0, P.p64, g, bones, xs, n, bpb, sp, s.sp, ctx->stats);
    } else {
        const bool esc = needs_f64(flags);
        int4* esc_q = esc ? (int4*)scratch(ctx, kEscQ, S * sizeof(int4)) : nullptr;
        const int bpg = (FSK_FAST_BPG > 0) ? std::min(FSK_FAST_BPG, g.nb) : g.nb;
        const int ngrp = (g.nb + bpg - 1) / bpg;
#if FSK_FAST_MAP == 1
        const int64_t ntiles = blocks_for(n, kSearchBlock);
        const int64_t nblocks = (ntiles + ctx->sm_count - 1) / ctx->sm_count * ctx->sm_count * ngrp;
#else
        const int64_t nblocks = (int64_t)blocks_for(n, kSearchBlock) * ngrp;
#endif
        if (nblocks >= (int64_t(1) << 31)) fail(FSK_EINVAL, "fsk: search grid too large");
        SearchP spf = sp;
        if (!esc) {  // float32 only (ablation): no cap, no flags
            spf.esc_cap = sp.max_iters;
        }
        FSK_LAUNCH(ctx, st, k_search_fast, (unsigned)nblocks, kSearchBlock, 0, P.p32, g, bones, xs, n, bpg, spf, s.sp,
                   esc_q, S, esc_n, ctx->stats, ctx->sm_count);
        int per_sm = 0;  // persistent kernel: exactly the resident capacity
        // exact replay of the reference whenever the weight grid is at hand
        const bool exact_esc = weights && !(flags & FSK_SEARCH_FAST_ESC);
        // exact refill with prefetch slots: bones + 144 B per thread of shared memory
        const size_t smem_pf = smem64 + (size_t)kEscBlock * kEscSlotF4 * sizeof(float4);
        const bool pf = FSK_ESC_PREFETCH && exact_esc && smem_pf <= 227 * 1024;
        if (pf && smem_pf > 48 * 1024)
            cuda_check(cudaFuncSetAttribute(k_search_escalated_pf, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)smem_pf), "cudaFuncSetAttribute");
        cuda_check(pf ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_search_escalated_pf, kEscBlock, smem_pf)
                   : exact_esc ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_search_escalated<true>,
                                                                               kEscBlock, smem64)
                               : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_search_escalated<false>,
                                                                               kEscBlock, 0),
                   "occupancy");
        const unsigned egrid = (unsigned)(ctx->sm_count * std::max(per_sm, 1));
        // start states of up to st_cap escalated solves (~5 % escalate; the rest start in-kernel)
        int st_cap = (int)std::min<int64_t>(S, std::max<int64_t>(1 << 16, S / 8));
        if (const char* e = getenv("FSK_ESC_START_CAP"))  // testing override (exercises the in-kernel starts)
            st_cap = std::max(1, std::min(st_cap, atoi(e)));
        double2* est = esc && exact_esc ? (double2*)scratch(ctx, kEscState, (size_t)st_cap * 8 * sizeof(double2))
                                        : nullptr;
        if (esc && exact_esc) {
            // ∇w stash for the one-pass initial Jacobian: n_b·3 doubles per thread, if it fits
            // (up to 73 bones at 128 threads; larger skeletons take the two-pass form)
            const size_t stash_b = (size_t)g.nb * 3 * sizeof(double) * 128;
#ifdef FSK_NO_STASH
            const bool stash_on = false;
#else
            const bool stash_on = smem64 + stash_b <= 227 * 1024;
#endif
            const size_t smem_s = smem64 + (stash_on ? stash_b : 0);
            int per_sm_s = 0;
            if (smem_s > 48 * 1024)
                cuda_check(cudaFuncSetAttribute(k_esc_start<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                (int)smem_s), "cudaFuncSetAttribute");
            cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_s, k_esc_start<true>, 128, smem_s),
                       "occupancy");
            const unsigned sgrid = (unsigned)(ctx->sm_count * std::max(1, std::min(per_sm_s, FSK_ESC_START_MINB)));
            FSK_LAUNCH(ctx, st, k_esc_start<true>, sgrid, 128, smem_s, P.p64, g, Wx, bones, n, sp, s.sp, esc_q, S,
                       esc_n, est, st_cap, ctx->stats, stash_on);
            if (pf)
                FSK_LAUNCH(ctx, st, k_search_escalated_pf, egrid, kEscBlock, smem_pf, P.p64, g, Wx, bones, n, sp, s.sp,
                           esc_q, S, esc_n, est, st_cap, ctx->stats);
            else
                FSK_LAUNCH(ctx, st, k_search_escalated<true>, egrid, kEscBlock, smem64, P.p64, g, Wx, bones, n, sp,
                           s.sp, esc_q, S, esc_n, est, st_cap, ctx->stats);
        } else if (esc) {  // cheap starts (transform-grid J~0): measured faster inside the refill kernel
            FSK_LAUNCH(ctx, st, k_search_escalated<false>, egrid, kEscBlock, 0, P.p64, g, nullptr, bones, n, sp, s.sp,
                       esc_q, S, esc_n, nullptr, 0, ctx->stats);
        }
    }
    launch_dedup(ctx, st, n, g.nb, (float)sp.dedup2, s.sp, s.perm, s.n_roots_p);
    return s;
}

void run_scan(fsk_ctx* ctx, const int32_t* in, int64_t n, int64_t* out, cudaStream_t st) {
    const int64_t nb = std::max<int64_t>(1, (n + kScanTile - 1) / kScanTile);
    int64_t* part = (int64_t*)scratch(ctx, kScanPart, (nb + 1) * sizeof(int64_t));
    FSK_LAUNCH(ctx, st, k_scan_partial, (unsigned)nb, kScanThreads, 0, in, n, part);
    FSK_LAUNCH(ctx, st, k_scan_top, 1, kScanThreads, 0, part, nb);
    FSK_LAUNCH(ctx, st, k_scan_apply, (unsigned)nb, kScanThreads, 0, in, n, part, out);
}

// exclusive scan of the search's per-query root counts (each <= n_b, total < 2^31)
void scan_root_counts(fsk_ctx* ctx, const int32_t* in, int64_t n, int64_t* out, cudaStream_t st) {
#if FSK_SCAN_LOOKBACK
    if (n > 0) {
        const int64_t ntiles = (n + kScanTile - 1) / kScanTile;
        const uint64_t gen0 = ctx->scratch_gen;
        auto* buf = (unsigned long long*)scratch(ctx, kScanLB, (ntiles + 1) * sizeof(unsigned long long));
        if (ctx->scratch_gen != gen0)  // fresh allocation: zero ticket, epoch and status words
            cuda_check(cudaMemsetAsync(buf, 0, ctx->cap[kScanLB], st), "cudaMemsetAsync");
        FSK_LAUNCH(ctx, st, k_scan_lookback, (unsigned)ntiles, kScanThreads, 0, in, n, (unsigned*)buf, buf + 1, out);
        return;
    }
#endif
    run_scan(ctx, in, n, out, st);
}

void compact(fsk_ctx* ctx, const SearchState& s, int64_t n, int nb, int64_t* offsets, fsk_root* roots, int64_t cap,
             cudaStream_t st) {
    scan_root_counts(ctx, s.n_roots_p, n, offsets, st);
    if (n > 0 && roots && cap > 0)
        FSK_LAUNCH(ctx, st, k_emit, blocks_for(n, 256), 256, 0, n, nb, s.sp, s.perm, offsets, roots, cap);
}

void check_search_args(const GridP& g, int32_t n_bones_pose, const void* grid_ptr, const char* mismatch) {
    if (n_bones_pose < 1) fail(FSK_EINVAL, "search: no bone transforms");
    if (!grid_ptr) fail(FSK_EINVAL, "search: voxel variant needs skinning and transform grids");
    if (n_bones_pose != g.nb) fail(FSK_EINVAL, mismatch);
}

// ============================================================================ MLP-variant search
// SearchVariant::Mlp (correspondence.cpp:77-79, deformer.cpp:22-26,
// :117-141): d(x) = lbs_blend(softmax(net(x)), B)·x, the initial Jacobian from the network's
// input tangents. Batched in rounds: every round evaluates the skinning network on the tensor
// cores (fsk_mlp.cu, 3xTF32) at the positions of all still-active solves, then one thread per
// solve takes the Broyden step (the same iterate() arithmetic as K2, float32). Solves are
// bone-major (q = bone·n + j) so dedup and compaction are K2's.
struct MvState {
    float4* x;   // x, -
    float4* g;   // g, err2
    float* ji;   // J~ [9]
    float4* dx;  // last step
    int* k;
};

__device__ __forceinline__ void mv_deform(const float* sB, int nb, const float* w, float x0, float x1, float x2,
                                          float d[3]) {
    float M[12];
#pragma unroll
    for (int e = 0; e < 12; ++e) M[e] = 0.f;
    for (int i = 0; i < nb; ++i) {  // lbs_blend (deformer.cpp:9-19), bone order
        const float wi = w[i];
#pragma unroll
        for (int e = 0; e < 12; ++e) M[e] = fmaf(wi, sB[12 * i + e], M[e]);
    }
    d[0] = M[0] * x0 + M[1] * x1 + M[2] * x2 + M[3];
    d[1] = M[4] * x0 + M[5] * x1 + M[6] * x2 + M[7];
    d[2] = M[8] * x0 + M[9] * x1 + M[10] * x2 + M[11];
}

__device__ __forceinline__ void mv_append(int* cnt, int* act, float4* pos, int s, float x0, float x1, float x2,
                                          bool on) {
    const unsigned m = __ballot_sync(__activemask(), on);
    if (!on) return;
    const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(cnt, __popc(m));
    base = __shfl_sync(m, base, leader);
    const int slot = base + __popc(m & ((1u << lane) - 1));
    act[slot] = s;
    pos[slot] = make_float4(x0, x1, x2, 0.f);
}

__global__ void __launch_bounds__(256) k_mv_init(const float* __restrict__ bones, const float* __restrict__ pts,
                                                 int64_t n, int nb, float4* __restrict__ pos) {
    const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (s >= n * nb) return;
    const int b = (int)(s / n);
    const int64_t j = s - (int64_t)b * n;
    const float* B = bones + 12 * b;
    const float xp0 = pts[3 * j], xp1 = pts[3 * j + 1], xp2 = pts[3 * j + 2];
    const float it0 = -(B[0] * B[3] + B[4] * B[7] + B[8] * B[11]);
    const float it1 = -(B[1] * B[3] + B[5] * B[7] + B[9] * B[11]);
    const float it2 = -(B[2] * B[3] + B[6] * B[7] + B[10] * B[11]);
    pos[s] = make_float4(B[0] * xp0 + B[4] * xp1 + B[8] * xp2 + it0, B[1] * xp0 + B[5] * xp1 + B[9] * xp2 + it1,
                         B[2] * xp0 + B[6] * xp1 + B[10] * xp2 + it2, 0.f);  // x0 = B_i^-1 x' (geometry.hpp:58-61)
}

// solve start (correspondence.cpp:135-137): J = Σ w_i R_i + Σ (B_i x)(∇w_i)ᵀ (deformer.cpp:117-128)
// from the tangent rows, J~0 = J^-1 or I, g0; then the divergence check and the first step.
__global__ void __launch_bounds__(256) k_mv_start(const float* __restrict__ bones, const float* __restrict__ pts,
                                                  int64_t n, int nb, SearchP o, const float4* __restrict__ pos,
                                                  const float* __restrict__ wt, SearchPlanes out, MvState st,
                                                  int* __restrict__ cnt_next, int* __restrict__ act_next,
                                                  float4* __restrict__ pos_next) {
    extern __shared__ float sB[];
    for (int e = threadIdx.x; e < nb * 12; e += blockDim.x) sB[e] = bones[e];
    __syncthreads();
    const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const bool live = s < n * nb;
    bool go = false;
    float x0 = 0, x1 = 0, x2 = 0;
    if (live) {
        const int64_t j = s - (s / n) * n;
        const float4 xv = pos[s];
        x0 = xv.x;
        x1 = xv.y;
        x2 = xv.z;
        const float* w = wt + (4 * s) * nb;
        float J[9];
#pragma unroll
        for (int e = 0; e < 9; ++e) J[e] = 0.f;
        for (int i = 0; i < nb; ++i) {
            const float* B = sB + 12 * i;
            const float wi = w[i];
            J[0] = fmaf(wi, B[0], J[0]); J[1] = fmaf(wi, B[1], J[1]); J[2] = fmaf(wi, B[2], J[2]);
            J[3] = fmaf(wi, B[4], J[3]); J[4] = fmaf(wi, B[5], J[4]); J[5] = fmaf(wi, B[6], J[5]);
            J[6] = fmaf(wi, B[8], J[6]); J[7] = fmaf(wi, B[9], J[7]); J[8] = fmaf(wi, B[10], J[8]);
        }
        for (int i = 0; i < nb; ++i) {
            const float* B = sB + 12 * i;
            const float bx[3] = {B[0] * x0 + B[1] * x1 + B[2] * x2 + B[3], B[4] * x0 + B[5] * x1 + B[6] * x2 + B[7],
                                 B[8] * x0 + B[9] * x1 + B[10] * x2 + B[11]};
            const float gw[3] = {w[nb + i], w[2 * nb + i], w[3 * nb + i]};  // ∂w_i/∂x_c from tangent row c
#pragma unroll
            for (int r = 0; r < 3; ++r)
#pragma unroll
                for (int c = 0; c < 3; ++c) J[3 * r + c] = fmaf(bx[r], gw[c], J[3 * r + c]);
        }
        float Ji[9];
        inverse_or_identity(J, Ji);
        float d[3];
        mv_deform(sB, nb, w, x0, x1, x2, d);
        const float g0 = d[0] - pts[3 * j], g1 = d[1] - pts[3 * j + 1], g2 = d[2] - pts[3 * j + 2];
        const float err2 = g0 * g0 + g1 * g1 + g2 * g2;
        const bool conv = err2 < (float)o.conv2;  // (:100-103)
        if (conv || err2 > (float)o.div2 || o.max_iters <= 0) {
            store_solve(out, s, x0, x1, x2, Ji, err2, SolveOut{0, conv, false, false});
        } else {
            const float dx0 = -(Ji[0] * g0 + Ji[1] * g1 + Ji[2] * g2);
            const float dx1 = -(Ji[3] * g0 + Ji[4] * g1 + Ji[5] * g2);
            const float dx2 = -(Ji[6] * g0 + Ji[7] * g1 + Ji[8] * g2);
            st.g[s] = make_float4(g0, g1, g2, err2);
            for (int e = 0; e < 9; ++e) st.ji[9 * s + e] = Ji[e];
            st.dx[s] = make_float4(dx0, dx1, dx2, 0.f);
            st.k[s] = 0;
            x0 += dx0;
            x1 += dx1;
            x2 += dx2;
            st.x[s] = make_float4(x0, x1, x2, 0.f);
            go = true;
        }
    }
    mv_append(cnt_next, act_next, pos_next, (int)s, x0, x1, x2, go);
}

// one Broyden iteration after the network evaluation at x (correspondence.cpp:108-122)
__global__ void __launch_bounds__(256) k_mv_step(const float* __restrict__ bones, const float* __restrict__ pts,
                                                 int64_t n, int nb, SearchP o, const int* __restrict__ cnt,
                                                 const int* __restrict__ act, const float* __restrict__ wv,
                                                 SearchPlanes out, MvState st, int* __restrict__ cnt_next,
                                                 int* __restrict__ act_next, float4* __restrict__ pos_next) {
    extern __shared__ float sB[];
    for (int e = threadIdx.x; e < nb * 12; e += blockDim.x) sB[e] = bones[e];
    __syncthreads();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int c = *cnt;
    bool go = false;
    int s = 0;
    float x0 = 0, x1 = 0, x2 = 0;
    if (i < c) {
        s = act[i];
        const int64_t j = (int64_t)s - ((int64_t)s / n) * n;
        const float4 xv = st.x[s], gv = st.g[s], dv = st.dx[s];
        x0 = xv.x;
        x1 = xv.y;
        x2 = xv.z;
        float Ji[9];
        for (int e = 0; e < 9; ++e) Ji[e] = st.ji[9 * s + e];
        float d[3];
        mv_deform(sB, nb, wv + (int64_t)i * nb, x0, x1, x2, d);
        const float n0 = d[0] - pts[3 * j], n1 = d[1] - pts[3 * j + 1], n2 = d[2] - pts[3 * j + 2];
        const float dg0 = n0 - gv.x, dg1 = n1 - gv.y, dg2 = n2 - gv.z;
        const float err2 = n0 * n0 + n1 * n1 + n2 * n2;
        const int k = st.k[s] + 1;
        const bool conv = err2 < (float)o.conv2;  // (:113-116)
        if (!conv) {
            const float dx0 = dv.x, dx1 = dv.y, dx2 = dv.z;
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
        if (conv || k >= o.max_iters || err2 > (float)o.div2) {
            store_solve(out, s, x0, x1, x2, Ji, err2, SolveOut{k, conv, false, false});
        } else {  // divergence check passed: the next step (:105-107)
            const float dx0 = -(Ji[0] * n0 + Ji[1] * n1 + Ji[2] * n2);
            const float dx1 = -(Ji[3] * n0 + Ji[4] * n1 + Ji[5] * n2);
            const float dx2 = -(Ji[6] * n0 + Ji[7] * n1 + Ji[8] * n2);
            st.g[s] = make_float4(n0, n1, n2, err2);
            for (int e = 0; e < 9; ++e) st.ji[9 * s + e] = Ji[e];
            st.dx[s] = make_float4(dx0, dx1, dx2, 0.f);
            st.k[s] = k;
            x0 += dx0;
            x1 += dx1;
            x2 += dx2;
            st.x[s] = make_float4(x0, x1, x2, 0.f);
            go = true;
        }
    }
    mv_append(cnt_next, act_next, pos_next, s, x0, x1, x2, go);
}

}  // namespace

// Exclusive int32 → int64 scan for other translation units (fsk_ctx.h).
void scan_i32_to_i64(fsk_ctx* ctx, const int32_t* in, int64_t n, int64_t* out, cudaStream_t st) {
    run_scan(ctx, in, n, out, st);
}

}  // namespace fsk

// Host-buffer pipeline shared by fsk_deform_host (one frame) and fsk_deform_host_frames (the pose
// loop of cmd_bench, fskin_cli.cpp:663-678, with cmd_deform's host copies, :395-429). Every frame is
// split into chunks of at most kHostChunkMax points (one work item each); items alternate between
// two device slots {bones, points, offsets, roots}, so device memory is bounded by the chunk size,
// not by N·n_b: item i+1 uploads and searches while item i's CorrespondenceSets download. The roots
// slot holds kSlotRootsPerQuery records per query (≈ 1.05 are kept on average); an item with more
// kept roots than that (counted by the compaction's scan) is re-run into a buffer of exactly its
// count (count-then-allocate, synchronous, rare). Host buffers are the caller's; a frame whose kept
// roots exceed its capacity still reports its total and the call returns FSK_EINVAL ("root buffer
// too small") after all frames ran — call again with cap >= total.
namespace fsk {
namespace {
#ifndef FSK_HOST_CHUNK_MAX
#define FSK_HOST_CHUNK_MAX (int64_t(1) << 22)  // 4M points per work item
#endif

int64_t host_chunks(int64_t n) {
    // whole below 2M points (each chunk pays its own launches and float64 tail; C2 200k: 1 chunk
    // 1.63 ms vs 4 chunks 1.99 ms), then ~2M-point chunks, at most FSK_HOST_CHUNK_MAX each
    int64_t k = std::max<int64_t>(1, std::min<int64_t>(8, n / (1 << 21)));
    if (const char* e = getenv("FSK_HOST_CHUNKS")) k = std::max<int64_t>(1, std::min<int64_t>(64, atoll(e)));
    k = std::max<int64_t>(k, (n + FSK_HOST_CHUNK_MAX - 1) / FSK_HOST_CHUNK_MAX);
    return std::max<int64_t>(1, std::min(k, std::max<int64_t>(1, n)));
}

void deform_host_pipeline(fsk_ctx* ctx, const float* weights, const GridP& g, int n_frames, const float* const* bones,
                          const float* const* points, const int64_t* n_points, const SearchP& sp, int flags,
                          int64_t* const* offsets, fsk_root* const* roots, const int64_t* caps, int64_t* totals,
                          cudaStream_t st) {
    struct Item {
        int f;
        int64_t p0, m;
        bool first, last;
    };
    std::vector<Item> items;
    int64_t cmax = 1;
    for (int f = 0; f < n_frames; ++f) {
        const int64_t n = n_points[f], k = host_chunks(n), csz = (n + k - 1) / k;
        for (int64_t c = 0; c < k; ++c) {
            const int64_t p0 = std::min(n, c * csz), m = std::max<int64_t>(0, std::min(csz, n - p0));
            items.push_back({f, p0, m, c == 0, c == k - 1});
            cmax = std::max(cmax, m);
        }
    }
    const int nb = g.nb;
    const int64_t V = vertex_count(g);
    int64_t per_q = 4;  // kSlotRootsPerQuery
    if (const char* e = getenv("FSK_SLOT_ROOTS_PER_QUERY")) per_q = std::max<int64_t>(0, atoll(e));  // testing override
    const int64_t slotcap = std::max<int64_t>(1, std::min<int64_t>(cmax * nb, cmax * per_q));
    float* dW = (float*)scratch(ctx, kHW, V * nb * sizeof(float));
    float* dB = (float*)scratch(ctx, kFB, 2 * nb * 12 * sizeof(float));
    float* dP = (float*)scratch(ctx, kFP, 2 * cmax * 3 * sizeof(float));
    int64_t* dOff = (int64_t*)scratch(ctx, kFOffs, 2 * (cmax + 1) * sizeof(int64_t));
    fsk_root* dR = (fsk_root*)scratch(ctx, kFRoots, 2 * slotcap * sizeof(fsk_root));
    if (!ctx->copy) cuda_check(cudaStreamCreateWithFlags(&ctx->copy, cudaStreamNonBlocking), "cudaStreamCreate");
    if (!ctx->upload) cuda_check(cudaStreamCreateWithFlags(&ctx->upload, cudaStreamNonBlocking), "cudaStreamCreate");
    if (!ctx->hcount) cuda_check(cudaMallocHost(&ctx->hcount, 64 * sizeof(int64_t)), "cudaMallocHost");
    const int N = (int)items.size();
    // per item: uploaded, searched, offsets downloaded, roots downloaded
    std::vector<cudaEvent_t> ev(4 * (size_t)N + 1, nullptr);
    struct Cleanup {  // on every exit (errors included): drain the three streams, then free the events
        fsk_ctx* ctx;
        cudaStream_t st;
        std::vector<cudaEvent_t>* ev;
        ~Cleanup() {
            cudaStreamSynchronize(ctx->upload);
            if (ctx->pre) cudaStreamSynchronize(ctx->pre);
            cudaStreamSynchronize(st);
            cudaStreamSynchronize(ctx->copy);
            for (auto e : *ev)
                if (e) cudaEventDestroy(e);
        }
    } cleanup{ctx, st, &ev};
    for (auto& e : ev) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    cudaEvent_t* up = ev.data();
    cudaEvent_t* done = up + N;
    cudaEvent_t* offs_ready = done + N;
    cudaEvent_t* fetched = offs_ready + N;
    cudaEvent_t start = ev.back();
    cuda_check(cudaEventRecord(start, st), "cudaEventRecord");  // order after prior use of the buffers
    cuda_check(cudaStreamWaitEvent(ctx->upload, start, 0), "cudaStreamWaitEvent");
    cuda_check(cudaStreamWaitEvent(ctx->copy, start, 0), "cudaStreamWaitEvent");
    cuda_check(cudaMemcpyAsync(dW, weights, V * nb * sizeof(float), cudaMemcpyHostToDevice, st), "H2D weights");
    auto slot_b = [&](int i) { return dB + (i & 1) * nb * 12; };
    auto slot_p = [&](int i) { return dP + (i & 1) * cmax * 3; };
    auto slot_o = [&](int i) { return dOff + (i & 1) * (cmax + 1); };
    auto slot_r = [&](int i) { return dR + (i & 1) * slotcap; };
    GridPlanes P;  // the current frame's gather planes (K1 runs with the frame's first chunk)
    // Staged pipeline (default with the spatial sort): item i's sort + K1 (its "stage") run on ctx->pre into
    // scratch slot i & 1 while item i-1 is still searching on st, and item i's search starts from the staged
    // slot — the sort and K1 leave the critical path. FSK_PIPE_STAGE=0 (or FSK_SEARCH_NO_SORT): each item
    // whole on st, K1 once per frame (the fsk_deform order).
    const bool staged = !(flags & FSK_SEARCH_NO_SORT) && [] {
        const char* e = getenv("FSK_PIPE_STAGE");
        return !(e && e[0] == '0');
    }();
    if (staged && !ctx->pre) cuda_check(cudaStreamCreateWithFlags(&ctx->pre, cudaStreamNonBlocking), "cudaStreamCreate");
    GridPlanes Ps[2];  // the staged slots' gather planes
    auto body_full = [&](int i, fsk_root* out, int64_t cap, cudaStream_t s_) {
        const Item& it = items[i];
        const PrecomputeReq pre{dW, slot_b(i), nullptr, needs_f64(flags)};
        const SearchState s =
            run_search(ctx, P, g, dW, slot_b(i), slot_p(i), it.m, sp, flags, s_, it.first ? &pre : nullptr);
        compact(ctx, s, it.m, nb, slot_o(i), out, cap, s_);
    };
    auto body_stage = [&](int i, cudaStream_t s_) {
        const PrecomputeReq pre{dW, slot_b(i), nullptr, needs_f64(flags)};
        run_search(ctx, Ps[i & 1], g, dW, slot_b(i), slot_p(i), items[i].m, sp, flags, s_, &pre, false, kRunStage,
                   i & 1);
    };
    auto body_search = [&](int i, fsk_root* out, int64_t cap, cudaStream_t s_) {
        const SearchState s = run_search(ctx, Ps[i & 1], g, dW, slot_b(i), slot_p(i), items[i].m, sp, flags, s_,
                                         nullptr, false, kRunAfterStage, i & 1);
        compact(ctx, s, items[i].m, nb, slot_o(i), out, cap, s_);
    };
    // Each item's device work is replayed from a CUDA graph once the same launch set has been seen before —
    // same slot buffers, chunk size, options and scratch generation (a scratch regrow frees buffers a graph
    // points into, so it changes the key). First sight runs eagerly (warms the scratch sizes), the second
    // captures. FSK_PIPE_GRAPH=0 turns it off.
    const bool graphs_on = [] {
        const char* e = getenv("FSK_PIPE_GRAPH");
        return !(e && e[0] == '0');
    }();
    static_assert(sizeof(GridPlanes) <= sizeof(fsk_ctx::PipeGraph::planes), "planes record");
    // key: everything the body's launches bake in besides the scratch generation; p_out: planes the body
    // produces (restored on replay)
    auto cached = [&](std::vector<unsigned char> key, GridPlanes* p_out, const std::function<void(cudaStream_t)>& body,
                      cudaStream_t launch, int64_t search_n) {
        auto note_search = [&] {
            if (search_n >= 0) ctx->last_search_n = search_n;
        };
        if (!graphs_on || ctx->prof_on) return body(launch);
        const uint64_t gen = ctx->scratch_gen;
        key.insert(key.begin(), (const unsigned char*)&gen, (const unsigned char*)&gen + sizeof gen);
        auto& cache = ctx->pipe_graphs;
        fsk_ctx::PipeGraph* hit = nullptr;
        for (auto& pg : cache)
            if (pg.key == key) hit = &pg;
        if (hit && hit->exec) {
            hit->last_use = ++ctx->pipe_clock;
            if (p_out) memcpy(p_out, hit->planes, sizeof *p_out);
            ctx->launches += hit->launches;
            note_search();
            cuda_check(cudaGraphLaunch(hit->exec, launch), "cudaGraphLaunch");
            return;
        }
        if (!hit) {  // first sight: run eagerly, remember the key
            body(launch);
            if (ctx->scratch_gen != gen) return;  // grew while running: the key is stale
            if (cache.size() >= 8) {
                auto lru = std::min_element(cache.begin(), cache.end(), [](const auto& a, const auto& b) {
                    return a.last_use < b.last_use;
                });
                if (lru->exec) cudaGraphExecDestroy(lru->exec);
                cache.erase(lru);
            }
            cache.push_back({});
            cache.back().key = std::move(key);
            cache.back().last_use = ++ctx->pipe_clock;
            return;
        }
        // second sight: capture on the private stream, instantiate, launch on the caller's
        if (!ctx->cap_stream)
            cuda_check(cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking), "cudaStreamCreate");
        const int64_t l0 = ctx->launches;
        cudaGraph_t graph = nullptr;
        cuda_check(cudaStreamBeginCapture(ctx->cap_stream, cudaStreamCaptureModeRelaxed), "cudaStreamBeginCapture");
        try {
            body(ctx->cap_stream);
        } catch (...) {
            cudaStreamEndCapture(ctx->cap_stream, &graph);
            if (graph) cudaGraphDestroy(graph);
            cudaGetLastError();
            throw;
        }
        cuda_check(cudaStreamEndCapture(ctx->cap_stream, &graph), "cudaStreamEndCapture");
        cudaGraphExec_t exec = nullptr;
        const cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
        cudaGraphDestroy(graph);
        cuda_check(ie, "cudaGraphInstantiate");
        if (ctx->scratch_gen != gen) {  // buffers moved under the capture: do not keep it
            cudaGraphExecDestroy(exec);
            ctx->launches = l0;
            return body(launch);
        }
        hit->exec = exec;
        hit->launches = ctx->launches - l0;
        hit->last_use = ++ctx->pipe_clock;
        if (p_out) memcpy(hit->planes, p_out, sizeof *p_out);
        note_search();
        cuda_check(cudaGraphLaunch(exec, launch), "cudaGraphLaunch");
    };
    auto key_of = [&](int kind, int i, const fsk_root* out, int64_t cap, const GridPlanes* p_in) {
        std::vector<unsigned char> key;
        auto put = [&](const void* p, size_t b) {
            key.insert(key.end(), (const unsigned char*)p, (const unsigned char*)p + b);
        };
        const Item& it = items[i];
        const void* ptrs[6] = {dW, slot_b(i), slot_p(i), slot_o(i), out, nullptr};
        const int64_t ints[4] = {(int64_t)kind, it.m, cap, (int64_t)it.first};
        put(ptrs, sizeof ptrs);
        put(ints, sizeof ints);
        put(&flags, sizeof flags);
        put(&sp, sizeof sp);
        put(&g, sizeof g);
        if (p_in) put(p_in, sizeof *p_in);
        return key;
    };
    auto stage_item = [&](int i) {
        cached(key_of(1, i, nullptr, 0, nullptr), &Ps[i & 1], [&](cudaStream_t s_) { body_stage(i, s_); }, ctx->pre, -1);
    };
    auto search_item = [&](int i, fsk_root* out, int64_t cap) {
        if (staged) {
            cached(key_of(2, i, out, cap, &Ps[i & 1]), nullptr, [&](cudaStream_t s_) { body_search(i, out, cap, s_); },
                   st, -1);
        } else {
            const Item& it = items[i];
            cached(key_of(0, i, out, cap, it.first ? nullptr : &P), it.first ? &P : nullptr,
                   [&](cudaStream_t s_) { body_full(i, out, cap, s_); }, st, it.m);
        }
    };
    cudaEvent_t w_up = nullptr;  // the weights are on the device (the stages read them on ctx->pre)
    std::vector<cudaEvent_t> staged_ev(staged ? (size_t)N : 0, nullptr);
    struct EvFree {
        std::vector<cudaEvent_t>* v;
        cudaEvent_t* w;
        ~EvFree() {
            for (auto e : *v)
                if (e) cudaEventDestroy(e);
            if (*w) cudaEventDestroy(*w);
        }
    } ev_free{&staged_ev, &w_up};
    if (staged) {
        for (auto& e : staged_ev) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
        cuda_check(cudaEventCreateWithFlags(&w_up, cudaEventDisableTiming), "cudaEventCreate");
        cuda_check(cudaEventRecord(w_up, st), "cudaEventRecord");
        cuda_check(cudaStreamWaitEvent(ctx->pre, w_up, 0), "cudaStreamWaitEvent");
    }
    auto enqueue = [&](int i) {
        const Item& it = items[i];
        if (i >= 2) cuda_check(cudaStreamWaitEvent(ctx->upload, done[i - 2], 0), "cudaStreamWaitEvent");
        cuda_check(cudaMemcpyAsync(slot_b(i), bones[it.f], nb * 12 * sizeof(float), cudaMemcpyHostToDevice, ctx->upload),
                   "H2D bones");
        if (it.m > 0)
            cuda_check(cudaMemcpyAsync(slot_p(i), points[it.f] + 3 * it.p0, it.m * 3 * sizeof(float),
                                       cudaMemcpyHostToDevice, ctx->upload),
                       "H2D points");
        cuda_check(cudaEventRecord(up[i], ctx->upload), "cudaEventRecord");
        if (staged) {  // stage on ctx->pre once the inputs landed and slot i & 1 is free (item i-2 searched)
            cuda_check(cudaStreamWaitEvent(ctx->pre, up[i], 0), "cudaStreamWaitEvent");
            if (i >= 2) cuda_check(cudaStreamWaitEvent(ctx->pre, done[i - 2], 0), "cudaStreamWaitEvent");
            stage_item(i);
            cuda_check(cudaEventRecord(staged_ev[i], ctx->pre), "cudaEventRecord");
            cuda_check(cudaStreamWaitEvent(st, staged_ev[i], 0), "cudaStreamWaitEvent");
        } else {
            cuda_check(cudaStreamWaitEvent(st, up[i], 0), "cudaStreamWaitEvent");
        }
        if (i >= 2) cuda_check(cudaStreamWaitEvent(st, fetched[i - 2], 0), "cudaStreamWaitEvent");
        search_item(i, slot_r(i), slotcap);
        cuda_check(cudaEventRecord(done[i], st), "cudaEventRecord");
    };
    // the offsets download of item i is queued on the (in-order) copy stream only after item i-1's roots
    // download, so that one never waits behind item i's search
    auto enqueue_offsets = [&](int i) {
        const Item& it = items[i];
        cuda_check(cudaStreamWaitEvent(ctx->copy, done[i], 0), "cudaStreamWaitEvent");
        if (it.m > 0)
            cuda_check(cudaMemcpyAsync(offsets[it.f] + it.p0, slot_o(i), it.m * sizeof(int64_t), cudaMemcpyDeviceToHost,
                                       ctx->copy),
                       "D2H offsets");
        cuda_check(cudaMemcpyAsync(ctx->hcount + (i % 64), slot_o(i) + it.m, sizeof(int64_t), cudaMemcpyDeviceToHost,
                                   ctx->copy),
                   "D2H count");
        cuda_check(cudaEventRecord(offs_ready[i], ctx->copy), "cudaEventRecord");
    };
    bool overflow = false;
    int64_t base = 0;
    if (N > 0) {
        enqueue(0);
        enqueue_offsets(0);
    }
    for (int i = 0; i < N; ++i) {
        const Item& it = items[i];
        if (i + 1 < N) enqueue(i + 1);  // the device runs ahead while we wait
        cuda_check(cudaEventSynchronize(offs_ready[i]), "cudaEventSynchronize");
        const int64_t cnt = ctx->hcount[i % 64];  // the item's kept roots
        if (it.first) base = 0;
        const fsk_root* src = slot_r(i);
        if (cnt > slotcap) {
            // more kept roots than the slot holds (k_emit dropped the rest): re-run the item into a
            // buffer of exactly `cnt` records. Its inputs are still in slot i&1 (item i+2 is not
            // enqueued yet); the device is drained first (item i+1 shares the search scratch).
            cuda_check(cudaStreamSynchronize(ctx->upload), "cudaStreamSynchronize");
            if (ctx->pre) cuda_check(cudaStreamSynchronize(ctx->pre), "cudaStreamSynchronize");
            cuda_check(cudaStreamSynchronize(st), "cudaStreamSynchronize");
            cuda_check(cudaStreamSynchronize(ctx->copy), "cudaStreamSynchronize");
            fsk_root* big = (fsk_root*)scratch(ctx, kHRoots, cnt * sizeof(fsk_root));
            if (staged) {  // re-stage into slot i & 1 (zeroes its escalation counters; item i+1 owns the other slot)
                body_stage(i, st);
                body_search(i, big, cnt, st);
            } else {
                const PrecomputeReq pre{dW, slot_b(i), nullptr, needs_f64(flags)};
                GridPlanes Pr;
                const SearchState s = run_search(ctx, Pr, g, dW, slot_b(i), slot_p(i), it.m, sp, flags, st, &pre);
                compact(ctx, s, it.m, nb, slot_o(i), big, cnt, st);
                if (i + 1 < N) {  // restore the planes of the frame of the last enqueued item (its later chunks read them)
                    const PrecomputeReq pre1{dW, slot_b(i + 1), nullptr, needs_f64(flags)};
                    P = run_precompute(ctx, pre1.w, g, pre1.bones, nullptr, nullptr, true, pre1.f64, st);
                }
            }
            cuda_check(cudaEventRecord(done[i], st), "cudaEventRecord");
            cuda_check(cudaStreamWaitEvent(ctx->copy, done[i], 0), "cudaStreamWaitEvent");
            src = big;
        }
        if (base + cnt > caps[it.f] || (cnt > 0 && !roots[it.f])) {
            overflow = true;
        } else if (cnt > 0) {
            cuda_check(cudaMemcpyAsync(roots[it.f] + base, src, cnt * sizeof(fsk_root), cudaMemcpyDeviceToHost, ctx->copy),
                       "D2H roots");
        }
        if (base)
            for (int64_t q = 0; q < it.m; ++q) offsets[it.f][it.p0 + q] += base;
        base += cnt;
        cuda_check(cudaEventRecord(fetched[i], ctx->copy), "cudaEventRecord");
        if (cnt > slotcap) cuda_check(cudaStreamSynchronize(ctx->copy), "cudaStreamSynchronize");  // `big` is reused
        if (it.last) {
            offsets[it.f][n_points[it.f]] = base;
            totals[it.f] = base;
        }
        if (i + 1 < N) enqueue_offsets(i + 1);
    }
    cuda_check(cudaStreamSynchronize(ctx->copy), "cudaStreamSynchronize");
    cuda_check(cudaStreamSynchronize(st), "cudaStreamSynchronize");
    if (overflow) fail(FSK_EINVAL, "fsk: root buffer too small");
}
}  // namespace
}  // namespace fsk

using namespace fsk;

extern "C" {

int fsk_precompute_tgrid(fsk_ctx* ctx, const float* weights, const fsk_grid_desc* desc, const float* bones,
                         int32_t n_bones_pose, float* tgrid, double* tgrid64, void* stream) {
    return guard([&] {
        set_device(ctx);
        const GridP g = make_grid(desc);
        if (n_bones_pose != g.nb) fail(FSK_EINVAL, "precompute_transform_grid: bone count mismatch");
        if (!weights || !bones || (!tgrid && !tgrid64)) fail(FSK_EINVAL, "fsk: null buffer");
        run_precompute(ctx, weights, g, bones, tgrid, tgrid64, false, false, (cudaStream_t)stream);
    });
}

int fsk_search_fwd(fsk_ctx* ctx, const float* tgrid, const double* tgrid64, const float* weights,
                   const fsk_grid_desc* desc,
                   const float* bones, int32_t n_bones_pose, const float* points, int64_t n,
                   const fsk_search_opts* opts, fsk_search_out* out, void* stream) {
    return guard([&] {
        set_device(ctx);
        // check_context (correspondence.cpp:29-41), then validate (:19-25)
        const GridP g = make_grid(desc);
        check_search_args(g, n_bones_pose, tgrid ? (const void*)tgrid : (const void*)tgrid64,
                          "search: grid bone count mismatch");
        const SearchP sp = make_search(opts);
        if (!out || (n > 0 && !out->converged)) fail(FSK_EINVAL, "fsk: search output needs a converged mask");
        if (n < 0) fail(FSK_EINVAL, "fsk: negative point count");
        if (n > 0 && (!points || !bones)) fail(FSK_EINVAL, "fsk: null buffer");
        if (n == 0) return;
        cudaStream_t st = (cudaStream_t)stream;
        GridPlanes P = run_relayout(ctx, tgrid, tgrid64, g, needs_f64(opts->flags), st);
        const SearchState s = run_search(ctx, P, g, weights, bones, points, n, sp, opts->flags, st, nullptr,
                                         out->x_c64 != nullptr);
        DenseOut d{out->x_c64, out->x_c, out->jinv, out->resid, out->iters, out->converged, out->keep, out->n_roots};
        FSK_LAUNCH(ctx, st, k_scatter_dense, blocks_for(n * g.nb, 256), 256, 0, n, g.nb, s.sp, s.perm, d);
        if (out->n_roots)
            cuda_check(cudaMemcpyAsync(out->n_roots, s.n_roots_p, n * sizeof(int32_t), cudaMemcpyDeviceToDevice, st),
                       "cudaMemcpyAsync");
    });
}

int fsk_search_fwd_mlp(fsk_ctx* ctx, const float* theta, const int32_t* widths, int32_t n_widths,
                       const float* bones, int32_t n_bones_pose, const float* points, int64_t n,
                       const fsk_search_opts* opts, fsk_search_out* out, void* stream) {
    return guard([&] {
        set_device(ctx);
        if (n_bones_pose < 1) fail(FSK_EINVAL, "search: no bone transforms");
        if (!theta || !widths) fail(FSK_EINVAL, "search: mlp variant needs a skinning network");
        if (n_widths < 2 || widths[0] != 3) fail(FSK_EINVAL, "SkinningMlp: network input width must be 3");
        if (widths[n_widths - 1] != n_bones_pose) fail(FSK_EINVAL, "search: mlp bone count mismatch");
        const SearchP sp = make_search(opts);
        if (!out || (n > 0 && !out->converged)) fail(FSK_EINVAL, "fsk: search output needs a converged mask");
        if (n < 0) fail(FSK_EINVAL, "fsk: negative point count");
        if (n > 0 && (!points || !bones)) fail(FSK_EINVAL, "fsk: null buffer");
        if (n == 0) return;
        const int nb = n_bones_pose;
        const int64_t S = n * nb;
        if (4 * S >= (int64_t(1) << 31)) fail(FSK_EINVAL, "fsk: too many points for one call (split the batch)");
        cudaStream_t st = (cudaStream_t)stream;
        // search planes, identity order (dedup + dense scatter are K2's)
        SearchState ss;
        ss.sp.xr = (float4*)scratch(ctx, kOXr, S * sizeof(float4));
        ss.sp.ja = (float4*)scratch(ctx, kOJa, S * sizeof(float4));
        ss.sp.jb = (float4*)scratch(ctx, kOJb, S * sizeof(float4));
        ss.sp.jc = (float*)scratch(ctx, kOJc, S * sizeof(float));
        ss.sp.meta = (uint32_t*)scratch(ctx, kOMeta, S * sizeof(uint32_t));
        ss.sp.keep = (uint8_t*)scratch(ctx, kOKeep, S);
        ss.perm = (int*)scratch(ctx, kPerm, n * sizeof(int));
        ss.n_roots_p = (int32_t*)scratch(ctx, kNRoots, n * sizeof(int32_t));
        float4* xs = (float4*)scratch(ctx, kXs, n * sizeof(float4));
        int* esc_n = (int*)scratch(ctx, kEscN, 4 * sizeof(int));
        FSK_LAUNCH(ctx, st, k_identity_order, blocks_for(n, 256), 256, 0, points, n, ss.perm, xs, esc_n);
        MvState mv;
        mv.x = (float4*)scratch(ctx, kMvX, S * sizeof(float4));
        mv.g = (float4*)scratch(ctx, kMvG, S * sizeof(float4));
        mv.ji = (float*)scratch(ctx, kMvJ, S * 9 * sizeof(float));
        mv.dx = (float4*)scratch(ctx, kMvDx, S * sizeof(float4));
        mv.k = (int*)scratch(ctx, kMvK, S * sizeof(int));
        float4* pos[2] = {(float4*)scratch(ctx, kMvPos, S * sizeof(float4)),
                          (float4*)scratch(ctx, kMvPosNext, S * sizeof(float4))};
        int* act[2] = {(int*)scratch(ctx, kMvAct, S * sizeof(int)), (int*)scratch(ctx, kMvActNext, S * sizeof(int))};
        int* cnt = (int*)scratch(ctx, kMvCnt, 2 * sizeof(int));
        float* w = (float*)scratch(ctx, kMvW, 4 * S * nb * sizeof(float));
        if (!ctx->hcount) cuda_check(cudaMallocHost(&ctx->hcount, 64 * sizeof(int64_t)), "cudaMallocHost");
        const size_t smb = nb * 12 * sizeof(float);
        const float* pk = mlp_skinning_pack(ctx, theta, widths, n_widths, st);
        // starts: x0 for every solve, the network with input tangents (4 rows per solve)
        FSK_LAUNCH(ctx, st, k_mv_init, blocks_for(S, 256), 256, 0, bones, points, n, nb, pos[0]);
        mlp_skinning_eval(ctx, pk, widths, n_widths, pos[0], 4 * S, true, w, st);
        cuda_check(cudaMemsetAsync(cnt, 0, 2 * sizeof(int), st), "cudaMemsetAsync");
        FSK_LAUNCH(ctx, st, k_mv_start, blocks_for(S, 256), 256, smb, bones, points, n, nb, sp, pos[0], w, ss.sp, mv,
                   cnt + 1, act[1], pos[1]);
        int cur = 1;
        for (int it = 0; it < sp.max_iters; ++it) {
            int32_t* hc = reinterpret_cast<int32_t*>(ctx->hcount);
            cuda_check(cudaMemcpyAsync(hc, cnt + cur, sizeof(int), cudaMemcpyDeviceToHost, st), "D2H count");
            cuda_check(cudaStreamSynchronize(st), "cudaStreamSynchronize");
            const int c = hc[0];
            if (c == 0) break;
            const int nxt = cur ^ 1;
            cuda_check(cudaMemsetAsync(cnt + nxt, 0, sizeof(int), st), "cudaMemsetAsync");
            mlp_skinning_eval(ctx, pk, widths, n_widths, pos[cur], c, false, w, st);
            FSK_LAUNCH(ctx, st, k_mv_step, blocks_for(c, 256), 256, smb, bones, points, n, nb, sp, cnt + cur, act[cur],
                       w, ss.sp, mv, cnt + nxt, act[nxt], pos[nxt]);
            cur = nxt;
        }
        launch_dedup(ctx, st, n, nb, (float)sp.dedup2, ss.sp, ss.perm, ss.n_roots_p);
        DenseOut d{out->x_c64, out->x_c, out->jinv, out->resid, out->iters, out->converged, out->keep, out->n_roots};
        FSK_LAUNCH(ctx, st, k_scatter_dense, blocks_for(S, 256), 256, 0, n, nb, ss.sp, ss.perm, d);
        if (out->n_roots)
            cuda_check(cudaMemcpyAsync(out->n_roots, ss.n_roots_p, n * sizeof(int32_t), cudaMemcpyDeviceToDevice, st),
                       "cudaMemcpyAsync");
    });
}

int fsk_batch_search(fsk_ctx* ctx, const float* tgrid, const double* tgrid64, const float* weights,
                     const fsk_grid_desc* desc,
                     const float* bones, int32_t n_bones_pose, const float* points, int64_t n,
                     const fsk_search_opts* opts, int64_t* offsets, fsk_root* roots, int64_t cap, void* stream) {
    return guard([&] {
        set_device(ctx);
        const GridP g = make_grid(desc);
        check_search_args(g, n_bones_pose, tgrid ? (const void*)tgrid : (const void*)tgrid64,
                          "search: grid bone count mismatch");
        const SearchP sp = make_search(opts);
        if (n < 0) fail(FSK_EINVAL, "fsk: negative point count");
        if (!offsets || (n > 0 && (!points || !bones))) fail(FSK_EINVAL, "fsk: null buffer");
        cudaStream_t st = (cudaStream_t)stream;
        GridPlanes P = run_relayout(ctx, tgrid, tgrid64, g, needs_f64(opts->flags), st);
        const SearchState s = run_search(ctx, P, g, weights, bones, points, n, sp, opts->flags, st);
        compact(ctx, s, n, g.nb, offsets, roots, cap, st);
    });
}

int fsk_deform(fsk_ctx* ctx, const float* weights, const fsk_grid_desc* desc, const float* bones,
               int32_t n_bones_pose, const float* points, int64_t n, const fsk_search_opts* opts, float* tgrid,
               int64_t* offsets, fsk_root* roots, int64_t cap, void* stream) {
    return guard([&] {
        set_device(ctx);
        const GridP g = make_grid(desc);
        check_search_args(g, n_bones_pose, weights, "precompute_transform_grid: bone count mismatch");
        const SearchP sp = make_search(opts);
        if (n < 0) fail(FSK_EINVAL, "fsk: negative point count");
        if (!offsets || !bones || (n > 0 && !points)) fail(FSK_EINVAL, "fsk: null buffer");
        cudaStream_t st = (cudaStream_t)stream;
        GridPlanes P;  // K1 runs inside run_search, beside the spatial sort
        const PrecomputeReq pre{weights, bones, tgrid, needs_f64(opts->flags)};
        const SearchState s = run_search(ctx, P, g, weights, bones, points, n, sp, opts->flags, st, &pre);
        compact(ctx, s, n, g.nb, offsets, roots, cap, st);
    });
}

int fsk_deform_frames(fsk_ctx* ctx, const float* weights, const fsk_grid_desc* desc, int32_t n_frames,
                      const float* const* bones, int32_t n_bones_pose, const float* const* points,
                      const int64_t* n_points, const fsk_search_opts* opts, float* tgrid, int64_t* const* offsets,
                      fsk_root* const* roots, const int64_t* caps, void* stream) {
    return guard([&] {
        set_device(ctx);
        const GridP g = make_grid(desc);
        check_search_args(g, n_bones_pose, weights, "precompute_transform_grid: bone count mismatch");
        const SearchP sp = make_search(opts);
        if (n_frames < 0) fail(FSK_EINVAL, "fsk: negative frame count");
        if (n_frames > 0 && (!bones || !points || !n_points || !offsets || !roots || !caps))
            fail(FSK_EINVAL, "fsk: null buffer");
        for (int f = 0; f < n_frames; ++f) {
            if (n_points[f] < 0) fail(FSK_EINVAL, "fsk: negative point count");
            if (!offsets[f] || !bones[f] || (n_points[f] > 0 && !points[f])) fail(FSK_EINVAL, "fsk: null buffer");
        }
        cudaStream_t st = (cudaStream_t)stream;
        if (!ctx->pre) cuda_check(cudaStreamCreateWithFlags(&ctx->pre, cudaStreamNonBlocking), "cudaStreamCreate");
        // events: start, then per frame {staged, searched}; pooled on the context (graph-capturable)
        const size_t need = 1 + 2 * (size_t)n_frames;
        while (ctx->frame_ev.size() < need) {
            cudaEvent_t e;
            cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
            ctx->frame_ev.push_back(e);
        }
        cudaEvent_t* ev = ctx->frame_ev.data();
        cuda_check(cudaEventRecord(ev[0], st), "cudaEventRecord");  // after prior work on the caller's stream
        cuda_check(cudaStreamWaitEvent(ctx->pre, ev[0], 0), "cudaStreamWaitEvent");
        GridPlanes Ps[2];
        for (int f = 0; f < n_frames; ++f) {
            const int slot = f & 1;
            cudaEvent_t staged = ev[1 + 2 * f], searched = ev[2 + 2 * f];
            // frame f's sort + K1 on ctx->pre into slot f & 1, once frame f-2 (the slot's last user) searched
            if (f >= 2) cuda_check(cudaStreamWaitEvent(ctx->pre, ev[2 + 2 * (f - 2)], 0), "cudaStreamWaitEvent");
            const PrecomputeReq pre{weights, bones[f], tgrid, needs_f64(opts->flags)};
            run_search(ctx, Ps[slot], g, weights, bones[f], points[f], n_points[f], sp, opts->flags, ctx->pre, &pre,
                       false, kRunStage, slot);
            cuda_check(cudaEventRecord(staged, ctx->pre), "cudaEventRecord");
            cuda_check(cudaStreamWaitEvent(st, staged, 0), "cudaStreamWaitEvent");
            const SearchState s = run_search(ctx, Ps[slot], g, weights, bones[f], points[f], n_points[f], sp,
                                             opts->flags, st, nullptr, false, kRunAfterStage, slot);
            compact(ctx, s, n_points[f], g.nb, offsets[f], roots[f], caps[f], st);
            cuda_check(cudaEventRecord(searched, st), "cudaEventRecord");
        }
    });
}

int fsk_compact_roots(fsk_ctx* ctx, const fsk_search_out* dense, int64_t n, int32_t n_init, int64_t* offsets,
                      fsk_root* roots, int64_t cap, int64_t* total_out, void* stream) {
    return guard([&] {
        set_device(ctx);
        if (!dense || !dense->keep || !dense->x_c || !dense->n_roots)
            fail(FSK_EINVAL, "fsk: compaction needs x_c, keep and n_roots");
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
            DenseOut d{nullptr, dense->x_c, dense->jinv, dense->resid, dense->iters, dense->converged, dense->keep,
                       dense->n_roots};
            FSK_LAUNCH(ctx, st, k_emit_dense, blocks_for(n, 256), 256, 0, n, n_init, d, offsets, roots);
        }
    });
}

int fsk_deform_host(fsk_ctx* ctx, const float* weights, const fsk_grid_desc* desc, const float* bones,
                    int32_t n_bones_pose, const float* points, int64_t n, const fsk_search_opts* opts,
                    int64_t* offsets, fsk_root* roots, int64_t cap, int64_t* total_out, void* stream) {
    return guard([&] {
        set_device(ctx);
        const GridP g = make_grid(desc);
        check_search_args(g, n_bones_pose, weights, "precompute_transform_grid: bone count mismatch");
        const SearchP sp = make_search(opts);
        if (n < 0) fail(FSK_EINVAL, "fsk: negative point count");
        if (!bones || !offsets || !total_out || (n > 0 && !points)) fail(FSK_EINVAL, "fsk: null buffer");
        *total_out = 0;
        deform_host_pipeline(ctx, weights, g, 1, &bones, &points, &n, sp, opts->flags, &offsets, &roots, &cap, total_out,
                             (cudaStream_t)stream);
    });
}

// A sequence of frames of one subject: the weights are uploaded once, then every frame is
// fsk_deform_host's H2D → K1 + search + compaction → D2H, pipelined over two device slots so item
// i+1's upload and search run while item i's CorrespondenceSets download. Per frame the results are
// identical to a fsk_deform_host call.
int fsk_deform_host_frames(fsk_ctx* ctx, const float* weights, const fsk_grid_desc* desc, int32_t n_frames,
                           const float* const* bones, int32_t n_bones_pose, const float* const* points,
                           const int64_t* n_points, const fsk_search_opts* opts, int64_t* const* offsets,
                           fsk_root* const* roots, const int64_t* caps, int64_t* totals, void* stream) {
    return guard([&] {
        set_device(ctx);
        const GridP g = make_grid(desc);
        check_search_args(g, n_bones_pose, weights, "precompute_transform_grid: bone count mismatch");
        const SearchP sp = make_search(opts);
        if (n_frames < 0) fail(FSK_EINVAL, "fsk: negative frame count");
        if (n_frames == 0) return;
        if (!bones || !points || !n_points || !offsets || !roots || !caps || !totals)
            fail(FSK_EINVAL, "fsk: null buffer");
        for (int f = 0; f < n_frames; ++f) {
            if (n_points[f] < 0) fail(FSK_EINVAL, "fsk: negative point count");
            if (!bones[f] || !offsets[f] || (n_points[f] > 0 && !points[f])) fail(FSK_EINVAL, "fsk: null buffer");
            totals[f] = 0;
        }
        deform_host_pipeline(ctx, weights, g, n_frames, bones, points, n_points, sp, opts->flags, offsets, roots, caps,
                             totals, (cudaStream_t)stream);
    });
}

int fsk_ctx_query_order(fsk_ctx* ctx, int64_t n, int32_t* order, void* stream) {
    return guard([&] {
        set_device(ctx);
        if (!order && n > 0) fail(FSK_EINVAL, "fsk: null buffer");
        if (n != ctx->last_search_n) fail(FSK_EINVAL, "fsk: no device search of that many points to take the order of");
        if (n > 0)
            cuda_check(cudaMemcpyAsync(order, ctx->buf[kPerm], n * sizeof(int32_t), cudaMemcpyDeviceToDevice,
                                       (cudaStream_t)stream),
                       "cudaMemcpyAsync");
    });
}

int fsk_init_states(fsk_ctx* ctx, const float* tgrid, const fsk_grid_desc* desc, const float* bones,
                    int32_t n_bones_pose, const float* points, int64_t n, float* x0, float* jinv0, void* stream) {
    return guard([&] {
        set_device(ctx);
        const GridP g = make_grid(desc);
        check_search_args(g, n_bones_pose, tgrid, "search: grid bone count mismatch");
        if (n < 0) fail(FSK_EINVAL, "fsk: negative point count");
        if (n == 0) return;
        if (!points || !bones) fail(FSK_EINVAL, "fsk: null buffer");
        cudaStream_t st = (cudaStream_t)stream;
        const GridPlanes P = run_relayout(ctx, tgrid, nullptr, g, false, st);
        FSK_LAUNCH(ctx, st, k_init_states, blocks_for(n * g.nb, 256), 256, 0, P.p32, g, bones, points, n, x0, jinv0);
    });
}

int fsk_init_states64(fsk_ctx* ctx, const float* weights, const fsk_grid_desc* desc, const float* bones,
                      int32_t n_bones_pose, const double* points, int64_t n, double* x0, double* jinv0, void* stream) {
    return guard([&] {
        set_device(ctx);
        const GridP g = make_grid(desc);
        check_search_args(g, n_bones_pose, weights, "search: grid bone count mismatch");
        if (n < 0) fail(FSK_EINVAL, "fsk: negative point count");
        if (n == 0) return;
        if (!points || !bones) fail(FSK_EINVAL, "fsk: null buffer");
        FSK_LAUNCH(ctx, (cudaStream_t)stream, k_init_states64, blocks_for(n * g.nb, 128), 128,
                   (size_t)g.nb * 12 * sizeof(double), g, weights, bones, points, n, x0, jinv0);
    });
}

int fsk_eval_points(fsk_ctx* ctx, const float* tgrid, const fsk_grid_desc* desc, const float* x, int64_t n,
                    float* t12, float* d, float* jac, void* stream) {
    return guard([&] {
        set_device(ctx);
        const GridP g = make_grid(desc);
        if (n < 0) fail(FSK_EINVAL, "fsk: negative point count");
        if (n == 0) return;
        if (!tgrid || !x) fail(FSK_EINVAL, "fsk: null buffer");
        cudaStream_t st = (cudaStream_t)stream;
        const GridPlanes P = run_relayout(ctx, tgrid, nullptr, g, false, st);
        FSK_LAUNCH(ctx, st, k_eval_points, blocks_for(n, 256), 256, 0, P.p32, g, x, n, t12, d, jac);
    });
}

}  // extern "C"
