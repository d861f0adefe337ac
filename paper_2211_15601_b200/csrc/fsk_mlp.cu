// fsk_mlp.cu — the MLP stages on either side of the deformer search, on the 5th-generation
// tensor cores:
//
//   fsk_distill            distill(SkinningMlp, dims, bbox) (skinning.cpp:195-221): softmax of
//                          the skinning network 3→64→64→64→n_b at every grid vertex
//   fsk_posed_occupancy    posed_occupancy_batch (shape.cpp:242-269): the occupancy network
//                          (3+n_p)→128→128→128→1 with sigmoid at every kept root, max and argmax
//                          over each query's CorrespondenceSet
//
// Both are Mlp::forward (mlp.cpp:115-138): softplus hidden units, linear head. One fused,
// persistent kernel per network runs a 128-row tile through every layer without leaving the
// SM: the input layer (K = 3 + n_p) on the FP32 pipe, the H×H hidden layers and the n_b-wide
// softmax head as tcgen05.mma (kind::tf32) with the activations in TMEM (A operand, written
// by the epilogue with tcgen05.st) and the weights in shared memory (B operand, K-major
// core-matrix layout, bulk-copied by TMA), accumulators in TMEM, softplus / bias / head in
// the epilogue registers.
//
// Precision: FP32-faithful "3xTF32": every operand is split x = hi + lo with hi = tf32(x)
// and A·B ≈ Ah·Bh + Ah·Bl + Al·Bh, accumulated in FP32 — max error vs a float64 network
// ≈ 2e-7 on the softmax weights (numpy emulation of this scheme; plain TF32 would be ~1e-3).
//
// Parameters are the reference's flat vector (Mlp::parameters(), mlp.cpp:207-219: per layer
// W column-major then b), in float32 on the device; k_mlp_pack re-lays them out once per call.
#include <cstring>

#include "fsk_ctx.h"

namespace fsk {
namespace {

// ------------------------------------------------------------------ tcgen05 / mbarrier PTX
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}" ::"r"(bar),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
// 1-D TMA bulk copy global → shared, completion counted on an mbarrier (tx bytes)
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
// D[tmem] (+)= A[tmem] · B[smem desc], kind::tf32, M = 128
__device__ __forceinline__ void mma_tf32_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
        "r"(a), "l"(bdesc), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float* v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
        "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15])
        : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]), "=f"(v[8]),
          "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]), "=f"(v[14]), "=f"(v[15])
        : "r"(taddr)
        : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ float tf32_hi(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

// sigmoid (mlp.cpp:15-21) in FP32 (softplus: act_fwd below)
__device__ __forceinline__ float sigmoid_f(float x) {
    if (x >= 0.f) return 1.f / (1.f + __expf(-x));
    const float e = __expf(x);
    return e / (1.f + e);
}

// Shared-memory matrix descriptor (tcgen05 "SmemDescriptor"): K-major, no swizzle, 8-row ×
// 16-byte core matrices; LBO = byte stride between the two K-adjacent core matrices of one
// MMA (K = 8 tf32), SBO = byte stride between 8-row groups; version 1 (sm_100).
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
// Instruction descriptor: D f32, A/B tf32, both K-major, M = 128, N.
__host__ __device__ constexpr uint32_t idesc_tf32(int n) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

// ------------------------------------------------------------------ packed parameters
// Packed layout (floats):
//   W0 [H][K0] row-major, b0 [H]
//   per hidden layer l (H×H): Bh [H·H] image, Bl [H·H] image, b [H]
//   head: softmax (kOutTC): Bh [NP·H], Bl [NP·H], b [NP] (rows >= n_out zero)
//         sigmoid scalar:  w [H], b [1] (+3 pad)
// Image of an N×K K-major operand: element (n, k) at float offset
//   ((n/8)·(K/4) + k/4)·32 + (n%8)·4 + k%4      (core matrix = 8 rows × 4 tf32 = 128 B)
__host__ __device__ inline int64_t img_off(int n, int k, int K) {
    return ((int64_t)(n >> 3) * (K >> 2) + (k >> 2)) * 32 + (n & 7) * 4 + (k & 3);
}

struct MlpShape {
    int n_layers;  // weight layers
    int K0, H, n_out, NP;
    int n_hidden;  // H×H layers
    bool softmax_head;
    int64_t off_W0, off_b0, off_hidden, off_head, total;
    int64_t hidden_stride() const { return 2 * (int64_t)H * H + H; }
};

MlpShape mlp_shape(const int32_t* widths, int nw, bool softmax_head) {
    if (nw < 3) fail(FSK_EINVAL, "Mlp: need at least input and output widths");
    MlpShape s{};
    s.n_layers = nw - 1;
    s.K0 = widths[0];
    s.H = widths[1];
    s.n_out = widths[nw - 1];
    s.n_hidden = nw - 3;
    s.softmax_head = softmax_head;
    for (int l = 1; l < nw - 1; ++l)
        if (widths[l] != s.H) fail(FSK_EINVAL, "fsk mlp: hidden layers must share one width");
    if (s.H != 64 && s.H != 128) fail(FSK_EINVAL, "fsk mlp: hidden width must be 64 or 128");
    if (s.K0 < 1 || s.K0 > 64) fail(FSK_EINVAL, "fsk mlp: input width must be in [1, 64]");
    if (softmax_head) {
        if (s.n_out < 1 || s.n_out > 64) fail(FSK_EINVAL, "fsk mlp: softmax head width must be in [1, 64]");
        s.NP = s.n_out <= 32 ? 32 : 64;
    } else {
        if (s.n_out != 1) fail(FSK_EINVAL, "occupancy mlp: expected input >= 3, scalar output");
        s.NP = 0;
    }
    s.off_W0 = 0;
    s.off_b0 = (int64_t)s.H * s.K0;
    s.off_hidden = (s.off_b0 + s.H + 31) / 32 * 32;  // 128-B aligned images
    s.off_head = s.off_hidden + s.n_hidden * ((s.hidden_stride() + 31) / 32 * 32);
    s.total = s.off_head + (softmax_head ? 2 * (int64_t)s.NP * s.H + s.NP : s.H + 4);
    return s;
}

constexpr int kMaxWidths = 32;

struct MlpDev {
    int K0, H, n_out, NP, n_hidden, softmax;
    int64_t off_W0, off_b0, off_hidden, off_head, hidden_stride_al;
    int nw;
    int widths[kMaxWidths];  // by value: no host→device copy per call
};

MlpDev to_dev(const MlpShape& s, const int32_t* widths, int nw) {
    MlpDev d{s.K0, s.H, s.n_out, s.NP, s.n_hidden, s.softmax_head ? 1 : 0, s.off_W0, s.off_b0, s.off_hidden,
             s.off_head, (s.hidden_stride() + 31) / 32 * 32, nw, {}};
    for (int i = 0; i < nw; ++i) d.widths[i] = widths[i];
    return d;
}

// theta offsets of layer l in Mlp::parameters() order
__device__ inline int64_t theta_off(const int* w, int l) {
    int64_t o = 0;
    for (int i = 0; i < l; ++i) o += (int64_t)w[i + 1] * w[i] + w[i + 1];
    return o;
}

__global__ void k_mlp_pack(const float* __restrict__ theta, MlpDev m, float* __restrict__ pk) {
    const int* widths = m.widths;
    const int nw = m.nw;
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int H = m.H;
    // input layer, row-major [H][K0]
    {
        const float* W = theta;  // layer 0 starts at 0
        for (int64_t i = t; i < (int64_t)H * m.K0; i += stride) {
            const int r = (int)(i / m.K0), c = (int)(i % m.K0);
            pk[m.off_W0 + i] = W[(int64_t)c * H + r];
        }
        for (int64_t i = t; i < H; i += stride) pk[m.off_b0 + i] = W[(int64_t)H * m.K0 + i];
    }
    for (int l = 0; l < m.n_hidden; ++l) {
        const float* W = theta + theta_off(widths, l + 1);
        float* dst = pk + m.off_hidden + l * m.hidden_stride_al;
        for (int64_t i = t; i < (int64_t)H * H; i += stride) {
            const int n = (int)(i % H), k = (int)(i / H);  // column-major source: (n, k) at k*H + n
            const float w = W[i];
            uint32_t r;
            asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(w));
            const float wh = __uint_as_float(r);
            dst[img_off(n, k, H)] = wh;
            dst[(int64_t)H * H + img_off(n, k, H)] = w - wh;
        }
        for (int64_t i = t; i < H; i += stride) dst[2 * (int64_t)H * H + i] = W[(int64_t)H * H + i];
    }
    const float* W = theta + theta_off(widths, nw - 2);
    float* dst = pk + m.off_head;
    if (m.softmax) {
        for (int64_t i = t; i < (int64_t)m.NP * H; i += stride) {
            const int n = (int)(i % m.NP), k = (int)(i / m.NP);
            const float w = n < m.n_out ? W[(int64_t)k * m.n_out + n] : 0.f;
            uint32_t r;
            asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(w));
            const float wh = __uint_as_float(r);
            dst[img_off(n, k, H)] = wh;
            dst[(int64_t)m.NP * H + img_off(n, k, H)] = w - wh;
        }
        for (int64_t i = t; i < m.NP; i += stride)
            dst[2 * (int64_t)m.NP * H + i] = i < m.n_out ? W[(int64_t)H * m.n_out + i] : 0.f;
    } else {
        for (int64_t i = t; i < H; i += stride) dst[i] = W[i];  // 1×H: column-major == row
        if (t == 0) dst[H] = W[H];
    }
}

// ------------------------------------------------------------------ fused MLP kernel
enum RowSource { kRowsGrid = 0, kRowsRoots = 1, kRowsPositions = 2 };

struct MlpRows {
    int source;
    int64_t n;
    // grid vertices (distill): vertex_position (skinning.cpp:77-80)
    int nx, ny;
    float lo[3], h[3];
    // roots (occupancy): fsk_root records (x at offset 0), pose broadcast
    const fsk_root* roots;
    const float* pose;
    int n_pose;
    // positions (MLP-variant search): float4 {x, y, z, -} per point; with `tangent` every point
    // owns 4 consecutive rows {value, d/dx, d/dy, d/dz} (forward-mode input tangents,
    // Mlp::input_tangent mlp.cpp:142-155) and n counts rows
    const float4* pos;
    int tangent;
};

constexpr int kTile = 128;
#ifndef FSK_MLP_THREADS
#define FSK_MLP_THREADS 512  // kSplit warps per TMEM lane quarter, each owning H / kSplit columns of every layer (512 vs 256 measured: occupancy query 189 -> 182 us, distill 64^3 153 -> 150 us, MLP-variant search 28.1 -> 23.1 ms)
#endif
constexpr int kThreads = FSK_MLP_THREADS;
constexpr int kSplit = kThreads / kTile;
static_assert(kSplit == 2 || kSplit == 4, "MLP CTA: 256 or 512 threads");

__device__ __forceinline__ void row_input(const MlpRows& R, int64_t r, float* x) {
    if (R.source == kRowsGrid) {
        const int64_t i = r % R.nx, j = (r / R.nx) % R.ny, k = r / ((int64_t)R.nx * R.ny);
        x[0] = R.lo[0] + (float)i * R.h[0];
        x[1] = R.lo[1] + (float)j * R.h[1];
        x[2] = R.lo[2] + (float)k * R.h[2];
    } else if (R.source == kRowsRoots) {
        const float4 a = __ldg(reinterpret_cast<const float4*>(R.roots + r));
        x[0] = a.x;
        x[1] = a.y;
        x[2] = a.z;
    } else {
        const float4 a = __ldg(R.pos + (R.tangent ? r >> 2 : r));
        x[0] = a.x;
        x[1] = a.y;
        x[2] = a.z;
    }
}

// softplus and its slope in one: e = exp(−|z|), softplus = max(z, 0) + log(1 + e), sigmoid
// from the same e. With input tangents the value row of a 4-row group gives the slope to its
// tangent rows (lanes 4m..4m+3 of one warp): h = softplus(z) for the value row, σ(z_value)·ż
// for a tangent row (the chain rule of Mlp::input_tangent, mlp.cpp:148-152).
__device__ __forceinline__ float act_fwd(float z, bool tangent, int role) {
    const float e = __expf(-fabsf(z));
    const float sp = fmaxf(z, 0.f) + __logf(1.f + e);
    if (!tangent) return sp;
    const float sig = z >= 0.f ? 1.f / (1.f + e) : e / (1.f + e);
    const float sv = __shfl_sync(0xffffffffu, sig, (threadIdx.x & 31) & ~3);
    return role == 0 ? sp : sv * z;
}

// One 128-row tile per iteration of a persistent CTA (kThreads threads: lane l of warp w owns TMEM
// lane 32·(w % 4) + l = tile row, and column part w / 4 of every layer). TMEM columns: D [0, H),
// A_hi [H, 2H), A_lo [2H, 3H).
// act (optional, for the backward): x [n][4] then the softplus outputs h_l [(n_hidden+1)][n][H].
template <int H, bool kStream, bool kTangent>
__global__ void __launch_bounds__(kThreads, H == 64 ? 2 : 1)  // H = 64: two CTAs per SM (256 TMEM columns each)
    k_mlp_fwd(MlpDev m, const float* __restrict__ pk, MlpRows R, float* __restrict__ out, float* __restrict__ act) {
    extern __shared__ __align__(128) float smem[];
    // smem: [weights (hidden layers resident, or one streamed layer) | head image | W0, b0 | pose]
    constexpr int kHidImg = 2 * H * H;  // floats (hi + lo)
    const int n_res = kStream ? (m.n_hidden > 0 ? 1 : 0) : m.n_hidden;
    float* s_hid = smem;
    float* s_head = s_hid + (int64_t)n_res * kHidImg;
    const int head_floats = m.softmax ? 2 * m.NP * H : 0;
    float* s_w0 = s_head + head_floats;
    float* s_b0 = s_w0 + H * m.K0;
    float* s_bias = s_b0 + H;  // hidden biases [n_hidden][H], then head bias [NP] / scalar head w [H], b
    float* s_headv = s_bias + m.n_hidden * H;
    float* s_pose = s_headv + (m.softmax ? m.NP : H + 1);
    __shared__ __align__(8) uint64_t bar_mma, bar_w;
    __shared__ uint32_t s_tmem;

    const int tid = threadIdx.x, warp = tid >> 5;
    // warp w reads/writes TMEM lanes [32 (w % 4), +32) (tcgen05 lane-quarter rule) and the
    // column half w / 4 of every layer; tile row = its TMEM lane
    const int quarter = warp & 3, half = warp >> 2;  // half: the warp's column part (0 .. kSplit-1)
    const int trow = quarter * 32 + (tid & 31);
    constexpr int HC = H / kSplit;  // columns per thread
    __shared__ float s_logit[kSplit - 1][kTile];
    const uint32_t b_mma = smem_u32(&bar_mma), b_w = smem_u32(&bar_w);

    for (int i = tid; i < H * m.K0; i += kThreads) s_w0[i] = pk[m.off_W0 + i];
    for (int i = tid; i < H; i += kThreads) s_b0[i] = pk[m.off_b0 + i];
    for (int l = 0; l < m.n_hidden; ++l)
        for (int i = tid; i < H; i += kThreads)
            s_bias[l * H + i] = pk[m.off_hidden + l * m.hidden_stride_al + kHidImg + i];
    if (m.softmax) {
        for (int i = tid; i < m.NP; i += kThreads) s_headv[i] = pk[m.off_head + 2 * m.NP * H + i];
    } else {
        for (int i = tid; i <= H; i += kThreads) s_headv[i] = pk[m.off_head + i];
    }
    if (R.source == kRowsRoots)
        for (int i = tid; i < R.n_pose; i += kThreads) s_pose[i] = R.pose[i];
    __syncthreads();
    // the pose inputs are the same for every row: fold W0[:, 3:]·pose into the input bias
    if (m.K0 > 3)
        for (int j = tid; j < H; j += kThreads) {
            float z = s_b0[j];
            for (int p = 3; p < m.K0; ++p) z = fmaf(s_w0[j * m.K0 + p], s_pose[p - 3], z);
            s_b0[j] = z;
        }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                     "r"(H == 64 ? 256 : 512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        mbar_init(b_mma, 1);
        mbar_init(b_w, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s_tmem;
    const uint32_t t_row = tmem + ((uint32_t)(quarter * 32) << 16);  // this warp's lane quarter
    const uint32_t tD = 0, tAh = H, tAl = 2 * H;

    // weights: bulk copies (TMA) of the pre-laid-out images
    uint32_t ph_w = 0, ph_mma = 0;
    bool w_ready = true;  // streamed weights: slot 0 holds the layer the next MMA needs
    auto load_hidden = [&](int l, int slot) {
        mbar_expect_tx(b_w, kHidImg * 4);
        bulk_g2s(smem_u32(s_hid + (int64_t)slot * kHidImg), pk + m.off_hidden + l * m.hidden_stride_al,
                 kHidImg * 4, b_w);
    };
    if (tid == 0) {
        const uint32_t bytes = (uint32_t)((kStream ? (m.n_hidden > 0 ? 1 : 0) : m.n_hidden) * kHidImg + head_floats) * 4;
        mbar_expect_tx(b_w, bytes);
        for (int l = 0; l < n_res; ++l)
            bulk_g2s(smem_u32(s_hid + (int64_t)l * kHidImg), pk + m.off_hidden + l * m.hidden_stride_al, kHidImg * 4,
                     b_w);
        if (head_floats) bulk_g2s(smem_u32(s_head), pk + m.off_head, head_floats * 4, b_w);
    }
    __syncthreads();
    mbar_wait(b_w, ph_w);
    ph_w ^= 1;

    const int64_t n_tiles = (R.n + kTile - 1) / kTile;
    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const int64_t row = tile * kTile + trow;
        const int64_t rr = row < R.n ? row : R.n - 1;
        // ---- layer 0 (K0 inputs) on the FP32 pipe → A (hi/lo) in TMEM
        float x[3];
        row_input(R, rr, x);
        constexpr bool tan = kTangent;  // 4-row groups {value, d/dx, d/dy, d/dz} (MLP-variant starts)
        const int role = tan ? (int)(row & 3) : 0;  // 0: value row, 1..3: d/dx_{role-1}
        float* act_h = act ? act + 4 * R.n : nullptr;
        if (act && half == 0 && row < R.n)
            reinterpret_cast<float4*>(act)[row] = make_float4(x[0], x[1], x[2], 0.f);
#pragma unroll 1
        for (int c0 = half * HC; c0 < (half + 1) * HC; c0 += 16) {
            float hv[16], lv[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const float* w = s_w0 + (c0 + j) * m.K0;
                float z;
                if (role == 0) {
                    z = s_b0[c0 + j];
                    z = fmaf(w[0], x[0], z);
                    z = fmaf(w[1], x[1], z);
                    z = fmaf(w[2], x[2], z);
                } else {
                    z = w[role - 1];  // W0 · e_k
                }
                const float h = act_fwd(z, tan, role);
                hv[j] = tf32_hi(h);
                lv[j] = h - hv[j];
            }
            if (act_h && row < R.n)
#pragma unroll
                for (int j = 0; j < 16; ++j) act_h[row * H + c0 + j] = hv[j] + lv[j];
            tmem_st16(t_row + tAh + c0, hv);
            tmem_st16(t_row + tAl + c0, lv);
        }
        float logit = 0.f;  // scalar head (occupancy)
        for (int l = 0; l <= m.n_hidden; ++l) {
            const bool head = l == m.n_hidden;
            if (head && !m.softmax) break;
            const int N = head ? m.NP : H;
            tmem_wait_st();
            tc_fence_before();
            __syncthreads();
            const bool wait_w = !head && kStream && !w_ready;
            if (tid == 0) {
                tc_fence_after();
                if (wait_w) mbar_wait(b_w, ph_w);  // this layer's streamed weights landed
                const float* img = head ? s_head : s_hid + (int64_t)(kStream ? 0 : l) * kHidImg;
                const uint32_t bh = smem_u32(img), bl = smem_u32(img + N * H);
                const uint32_t sbo = H * 32;  // (K/4) core matrices × 128 B per 8-row group
                const uint32_t id = head ? idesc_tf32(m.NP) : idesc_tf32(H);
#pragma unroll 1
                for (int s = 0; s < H / 8; ++s) {
                    const uint64_t dh = smem_desc(bh + s * 256, 128, sbo), dl = smem_desc(bl + s * 256, 128, sbo);
                    mma_tf32_ts(tmem + tD, tmem + tAh + 8 * s, dh, id, s > 0);
                    mma_tf32_ts(tmem + tD, tmem + tAh + 8 * s, dl, id, 1);
                    mma_tf32_ts(tmem + tD, tmem + tAl + 8 * s, dh, id, 1);
                }
                tc_commit(b_mma);
            }
            if (wait_w) ph_w ^= 1;  // every thread tracks the weight-barrier phase
            mbar_wait(b_mma, ph_mma);
            ph_mma ^= 1;
            tc_fence_after();
#ifndef FSK_MLP_PROBE_NO_STREAM  // timing probe only (wrong results): every layer reuses the first layer's weights
            if (!head && kStream) {
                // the MMAs have read this layer's weights: stream the next hidden layer's
                // (the first hidden layer again after the last), overlapping this epilogue
                if (tid == 0) load_hidden(l + 1 < m.n_hidden ? l + 1 : 0, 0);
                w_ready = false;
            }
#endif
            if (head && half == 0) {  // softmax head (SkinningMlp::weights_batch, skinning.cpp:47-51)
                float z[64];
#pragma unroll
                for (int c0 = 0; c0 < 64; c0 += 16)
                    if (c0 < m.NP) tmem_ld16(t_row + tD + c0, z + c0);
                tmem_wait_ld();
                float mx = -INFINITY;
                for (int i = 0; i < m.n_out; ++i) {
                    if (role == 0) z[i] += s_headv[i];
                    mx = fmaxf(mx, z[i]);
                }
                float sum = 0.f, zt[kTangent ? 64 : 1];
                for (int i = 0; i < m.n_out; ++i) {
                    if constexpr (kTangent) zt[i] = z[i];
                    z[i] = __expf(z[i] - mx);
                    sum += z[i];
                }
                const float inv = 1.f / sum;
                for (int i = 0; i < m.n_out; ++i) z[i] *= inv;
                if constexpr (kTangent) {  // softmax Jacobian on the tangent rows: ẇ = w ⊙ (ż − <w, ż>) (skinning.cpp:57-63)
                    float dot = 0.f;
                    for (int i = 0; i < m.n_out; ++i) {
                        const float wv = __shfl_sync(0xffffffffu, z[i], (threadIdx.x & 31) & ~3);
                        z[i] = wv;
                        dot = fmaf(wv, zt[i], dot);
                    }
                    if (role != 0)
                        for (int i = 0; i < m.n_out; ++i) z[i] = z[i] * (zt[i] - dot);
                }
                if (row < R.n)
                    for (int i = 0; i < m.n_out; ++i) out[row * m.n_out + i] = z[i];
            } else if (!head) {  // hidden epilogue: bias, softplus, split → next layer's A (and scalar head)
                const float* b = s_bias + l * H;
                const bool last_hidden = l + 1 == m.n_hidden;
                // all of the row's accumulators in flight at once, one wait (64 or 128 registers)
                float acc[HC];
                const int cb = half * HC;
#pragma unroll
                for (int c0 = 0; c0 < HC; c0 += 16) tmem_ld16(t_row + tD + cb + c0, acc + c0);
                tmem_wait_ld();
#pragma unroll
                for (int c0 = 0; c0 < HC; c0 += 16) {
                    float v[16], lv[16];
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const float h = act_fwd(role == 0 ? acc[c0 + j] + b[cb + c0 + j] : acc[c0 + j], tan, role);
                        if (!m.softmax && last_hidden) logit = fmaf(s_headv[cb + c0 + j], h, logit);
                        v[j] = tf32_hi(h);
                        lv[j] = h - v[j];
                    }
                    if (act_h && row < R.n)
#pragma unroll
                        for (int j = 0; j < 16; ++j)
                            act_h[((int64_t)(l + 1) * R.n + row) * H + cb + c0 + j] = v[j] + lv[j];
                    if (!(last_hidden && !m.softmax)) {
                        tmem_st16(t_row + tAh + cb + c0, v);
                        tmem_st16(t_row + tAl + cb + c0, lv);
                    }
                }
            }
        }
        if (!m.softmax && half > 0) s_logit[half - 1][trow] = logit;  // partials over the upper column parts
        tmem_wait_st();
        tc_fence_before();
        __syncthreads();  // TMEM A/D reuse by the next tile
        tc_fence_after();
        if (!m.softmax && half == 0 && row < R.n) {  // OccupancyMlp (shape.cpp:208-228)
            float z = logit;
#pragma unroll
            for (int p = 0; p < kSplit - 1; ++p) z += s_logit[p][trow];
            out[row] = sigmoid_f(z + s_headv[H]);
        }
    }
    if (kStream && tid == 0 && !w_ready) mbar_wait(b_w, ph_w);  // drain the last prefetch
    tc_fence_before();
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(H == 64 ? 256 : 512));
}

// posed_occupancy_batch aggregation (shape.cpp:256-267): max over each query's roots, the
// first root wins ties; empty sets give 0 and argmax -1.
__global__ void k_occ_reduce(const float* __restrict__ occ, const int64_t* __restrict__ offs, int64_t n,
                             float* __restrict__ pred, int32_t* __restrict__ argmax) {
    const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= n) return;
    float best = 0.f;
    int32_t am = -1;
    for (int64_t r = offs[q]; r < offs[q + 1]; ++r) {
        const float o = occ[r];
        if (am < 0 || o > best) {
            best = o;
            am = (int32_t)(r - offs[q]);
        }
    }
    pred[q] = best;
    if (argmax) argmax[q] = am;
}

size_t fwd_smem_bytes(const MlpShape& s, bool stream) {
    const int64_t hid = 2 * (int64_t)s.H * s.H;
    const int n_res = stream ? (s.n_hidden > 0 ? 1 : 0) : s.n_hidden;
    int64_t f = n_res * hid + (s.softmax_head ? 2 * (int64_t)s.NP * s.H : 0) + (int64_t)s.H * s.K0 + s.H +
                (int64_t)s.n_hidden * s.H + (s.softmax_head ? s.NP : s.H + 1) + 64;
    return (size_t)f * 4;
}

template <int H, bool kStream, bool kTangent>
void launch_fwd(fsk_ctx* ctx, const MlpShape& s, const int32_t* widths, int nw, const float* pk, const MlpRows& R,
                float* out, float* act, cudaStream_t st) {
    const size_t sm = fwd_smem_bytes(s, kStream);
    // the dynamic-smem opt-in and the residency query once per (instantiation, size)
    static thread_local size_t set_for = 0;
    static thread_local int per_sm = 1;
    if (set_for != sm) {
        cuda_check(cudaFuncSetAttribute(k_mlp_fwd<H, kStream, kTangent>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm),
                   "cudaFuncSetAttribute");
        // persistent grid = resident capacity (two CTAs per SM for H = 64: one's MMAs overlap the other's epilogue)
        cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_mlp_fwd<H, kStream, kTangent>, kThreads, sm),
                   "occupancy");
        set_for = sm;
    }
    const int64_t tiles = (R.n + kTile - 1) / kTile;
    const unsigned grid =
        (unsigned)std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)ctx->sm_count * std::max(per_sm, 1)));
    FSK_LAUNCH(ctx, st, (k_mlp_fwd<H, kStream, kTangent>), grid, kThreads, sm, to_dev(s, widths, nw), pk, R, out, act);
}

void run_fwd(fsk_ctx* ctx, const MlpShape& s, const int32_t* widths, int nw, const float* pk, const MlpRows& R,
             float* out, cudaStream_t st, float* act = nullptr) {
    if (R.n == 0) return;
    // weights resident when they fit next to the head image (227 KB per CTA), else streamed per layer
    const bool stream = fwd_smem_bytes(s, false) > 200 * 1024;
    if (fwd_smem_bytes(s, stream) > 227 * 1024) fail(FSK_EINVAL, "fsk mlp: network too large for one CTA");
    const bool tan = R.source == kRowsPositions && R.tangent;
    if (s.H == 64) {
        if (tan && stream) launch_fwd<64, true, true>(ctx, s, widths, nw, pk, R, out, act, st);
        else if (tan) launch_fwd<64, false, true>(ctx, s, widths, nw, pk, R, out, act, st);
        else if (stream) launch_fwd<64, true, false>(ctx, s, widths, nw, pk, R, out, act, st);
        else launch_fwd<64, false, false>(ctx, s, widths, nw, pk, R, out, act, st);
    } else {
        if (tan && stream) launch_fwd<128, true, true>(ctx, s, widths, nw, pk, R, out, act, st);
        else if (tan) launch_fwd<128, false, true>(ctx, s, widths, nw, pk, R, out, act, st);
        else if (stream) launch_fwd<128, true, false>(ctx, s, widths, nw, pk, R, out, act, st);
        else launch_fwd<128, false, false>(ctx, s, widths, nw, pk, R, out, act, st);
    }
}

const float* pack(fsk_ctx* ctx, const MlpShape& s, const float* theta, const int32_t* widths, int nw,
                  cudaStream_t st) {
    if (nw > kMaxWidths) fail(FSK_EINVAL, "fsk mlp: too many layers");
    float* pk = (float*)scratch(ctx, kMlpPack, (size_t)s.total * sizeof(float));
    FSK_LAUNCH(ctx, st, k_mlp_pack, (unsigned)ctx->sm_count, 256, 0, theta, to_dev(s, widths, nw), pk);
    return pk;
}

// ------------------------------------------------------------------ distill backward
// Fused Mlp::backward over tiles of 64 rows (mlp.cpp:140-163), FP32 on the CUDA cores: per
// tile the softmax VJP, then per layer (last to first) dW_l += δ_lᵀ·in_l, db_l += Σ δ_l and
// δ_{l-1} = (δ_l·W_l) ⊙ softplus'(z_{l-1}) with softplus' = 1 − e^{−h} from the stored
// activation. 4×4 register blocks over shared-memory tiles; each CTA accumulates into its own
// slot of `part` ([grid][P], no atomics) and k_bwd_reduce sums the slots in a fixed order.
constexpr int kBT = 64;  // rows per tile
struct BwdNet {
    int L, nw;
    int w[kMaxWidths];
    int64_t off[kMaxWidths];  // layer offsets in theta
    int64_t P;
    int maxw;
};

__device__ __forceinline__ void bwd_outer(const float* D, int ldd, const float* IN, int ldi, int n_out, int n_in,
                                          float* dst_W, float* dst_b, int tid, int nthreads) {
    // dW[o][i] += Σ_r D[r][o] IN[r][i] (column-major dst: i*n_out + o); db[o] += Σ_r D[r][o]
    const int bo = (n_out + 3) / 4, bi = (n_in + 3) / 4;
    for (int blk = tid; blk < bo * bi; blk += nthreads) {
        const int o0 = (blk / bi) * 4, i0 = (blk % bi) * 4;
        float acc[4][4] = {};
        for (int r = 0; r < kBT; ++r) {
            float d[4], v[4];
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                d[a] = o0 + a < n_out ? D[r * ldd + o0 + a] : 0.f;
                v[a] = i0 + a < n_in ? IN[r * ldi + i0 + a] : 0.f;
            }
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) acc[a][b] = fmaf(d[a], v[b], acc[a][b]);
        }
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b)
                if (o0 + a < n_out && i0 + b < n_in) dst_W[(int64_t)(i0 + b) * n_out + o0 + a] += acc[a][b];
    }
    for (int o = tid; o < n_out; o += nthreads) {
        float sacc = 0.f;
        for (int r = 0; r < kBT; ++r) sacc += D[r * ldd + o];
        dst_b[o] += sacc;
    }
}

__global__ void __launch_bounds__(256) k_mlp_bwd(BwdNet net, const float* __restrict__ theta,
                                                 const float* __restrict__ act, const float* __restrict__ w,
                                                 const float* __restrict__ gw, int64_t n, int H,
                                                 float* __restrict__ part) {
    extern __shared__ float sm[];
    const int M = net.maxw;
    float* D0 = sm;                 // [kBT][M]
    float* D1 = D0 + kBT * M;       // [kBT][M]
    float* IN = D1 + kBT * M;       // [kBT][M]
    float* Wl = IN + kBT * M;       // [M][M] row-major (n_out x n_in)
    const int tid = threadIdx.x, nt = blockDim.x;
    float* my = part + (int64_t)blockIdx.x * net.P;
    for (int64_t i = tid; i < net.P; i += nt) my[i] = 0.f;
    const int nb = net.w[net.nw - 1];
    const int64_t n_tiles = (n + kBT - 1) / kBT;
    const float* act_h = act + 4 * n;
    for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const int64_t r0 = t * kBT;
        // δ_L = softmax_vjp(w, dw) (mlp.cpp:38-41); rows beyond n contribute 0
        for (int r = tid; r < kBT; r += nt) {
            const int64_t v = r0 + r;
            float dot = 0.f;
            if (v < n)
                for (int i = 0; i < nb; ++i) dot = fmaf(w[v * nb + i], gw[v * nb + i], dot);
            for (int i = 0; i < nb; ++i) D0[r * M + i] = v < n ? w[v * nb + i] * (gw[v * nb + i] - dot) : 0.f;
        }
        float *Dc = D0, *Dn = D1;
        for (int l = net.L - 1; l >= 0; --l) {
            const int n_out = net.w[l + 1], n_in = net.w[l];
            __syncthreads();
            // this layer's input rows: x (layer 0) or h_{l-1}
            for (int e = tid; e < kBT * n_in; e += nt) {
                const int r = e / n_in, c = e - r * n_in;
                const int64_t v = r0 + r;
                IN[r * M + c] = v < n ? (l == 0 ? act[4 * v + c] : act_h[((int64_t)(l - 1) * n + v) * H + c]) : 0.f;
            }
            if (l > 0)  // W_l row-major [n_out][n_in] from the column-major parameters
                for (int e = tid; e < n_out * n_in; e += nt) {
                    const int o = e / n_in, c = e - o * n_in;
                    Wl[o * M + c] = theta[net.off[l] + (int64_t)c * n_out + o];
                }
            __syncthreads();
            bwd_outer(Dc, M, IN, M, n_out, n_in, my + net.off[l], my + net.off[l] + (int64_t)n_out * n_in, tid, nt);
            if (l == 0) break;
            // δ_{l-1}[r][c] = (Σ_k δ_l[r][k] W_l[k][c]) · (1 − e^{−h_{l-1}[r][c]})
            const int br = kBT / 4, bc = (n_in + 3) / 4;
            for (int blk = tid; blk < br * bc; blk += nt) {
                const int rr = (blk / bc) * 4, c0 = (blk % bc) * 4;
                float acc[4][4] = {};
                for (int k = 0; k < n_out; ++k) {
                    float d[4], wv[4];
#pragma unroll
                    for (int a = 0; a < 4; ++a) {
                        d[a] = Dc[(rr + a) * M + k];
                        wv[a] = c0 + a < n_in ? Wl[k * M + c0 + a] : 0.f;
                    }
#pragma unroll
                    for (int a = 0; a < 4; ++a)
#pragma unroll
                        for (int b = 0; b < 4; ++b) acc[a][b] = fmaf(d[a], wv[b], acc[a][b]);
                }
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < 4; ++b)
                        if (c0 + b < n_in) Dn[(rr + a) * M + c0 + b] = acc[a][b] * -expm1f(-IN[(rr + a) * M + c0 + b]);
            }
            float* tmp = Dc;
            Dc = Dn;
            Dn = tmp;
        }
    }
}

__global__ void k_bwd_reduce(const float* __restrict__ part, int parts, int64_t P, float* __restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= P) return;
    float s = 0.f;
    for (int c = 0; c < parts; ++c) s += part[(int64_t)c * P + i];  // fixed order: deterministic
    out[i] = s;
}


}  // namespace

// For the MLP-variant search (fsk_search.cu): pack once, then evaluate the skinning network
// (softmax head) at float4 positions, optionally with the 3 forward-mode input tangents per
// point (rows = 4 × points).
const float* mlp_skinning_pack(fsk_ctx* ctx, const float* theta, const int32_t* widths, int nw, cudaStream_t st) {
    const MlpShape s = mlp_shape(widths, nw, true);
    return pack(ctx, s, theta, widths, nw, st);
}

void mlp_skinning_eval(fsk_ctx* ctx, const float* pk, const int32_t* widths, int nw, const float4* pos, int64_t n_rows,
                       bool tangent, float* out, cudaStream_t st) {
    const MlpShape s = mlp_shape(widths, nw, true);
    MlpRows R{};
    R.source = kRowsPositions;
    R.n = n_rows;
    R.pos = pos;
    R.tangent = tangent ? 1 : 0;
    run_fwd(ctx, s, widths, nw, pk, R, out, st);
}

}  // namespace fsk

using namespace fsk;

extern "C" {

int fsk_distill(fsk_ctx* ctx, const float* theta, const int32_t* widths, int32_t n_widths,
                const fsk_grid_desc* desc, float* weights, void* stream) {
    return guard([&] {
        set_device(ctx);
        if (!desc || !widths || !theta || !weights) fail(FSK_EINVAL, "fsk: null buffer");
        if (desc->nx < 2 || desc->ny < 2 || desc->nz < 2) fail(FSK_EINVAL, "distill: dims must be >= 2 per axis");
        if (n_widths < 2 || widths[0] != 3) fail(FSK_EINVAL, "SkinningMlp: network input width must be 3");
        if (widths[n_widths - 1] != desc->n_bones) fail(FSK_EINVAL, "distill: bone count mismatch");
        const MlpShape s = mlp_shape(widths, n_widths, true);
        cudaStream_t st = (cudaStream_t)stream;
        const float* pk = pack(ctx, s, theta, widths, n_widths, st);
        MlpRows R{};
        R.source = kRowsGrid;
        R.n = (int64_t)desc->nx * desc->ny * desc->nz;
        R.nx = desc->nx;
        R.ny = desc->ny;
        const int n3[3] = {desc->nx, desc->ny, desc->nz};
        for (int a = 0; a < 3; ++a) {
            R.lo[a] = (float)desc->bbox_min[a];
            R.h[a] = (float)(((double)desc->bbox_max[a] - (double)desc->bbox_min[a]) / (n3[a] - 1));
        }
        run_fwd(ctx, s, widths, n_widths, pk, R, weights, st);
    });
}

int fsk_posed_occupancy(fsk_ctx* ctx, const float* theta, const int32_t* widths, int32_t n_widths,
                        const float* pose, int32_t n_pose, const int64_t* offsets, const fsk_root* roots, int64_t n,
                        int64_t n_roots, float* pred, int32_t* argmax, float* occ_per_root, void* stream) {
    return guard([&] {
        set_device(ctx);
        if (!widths || !theta) fail(FSK_EINVAL, "fsk: null buffer");
        if (n_widths < 2 || widths[0] < 3 || widths[n_widths - 1] != 1)
            fail(FSK_EINVAL, "occupancy mlp: expected input >= 3, scalar output");
        if (n_pose != widths[0] - 3)
            fail(FSK_EINVAL, "occupancy mlp: pose vector length " + std::to_string(n_pose) +
                                 ", field conditioned on " + std::to_string(widths[0] - 3));
        if (n < 0 || n_roots < 0) fail(FSK_EINVAL, "fsk: negative count");
        if (n > 0 && (!offsets || !pred)) fail(FSK_EINVAL, "fsk: null buffer");
        if (n_roots > 0 && !roots) fail(FSK_EINVAL, "fsk: null buffer");
        if (n_pose > 0 && !pose) fail(FSK_EINVAL, "fsk: null buffer");
        const MlpShape s = mlp_shape(widths, n_widths, false);
        cudaStream_t st = (cudaStream_t)stream;
        const float* pk = pack(ctx, s, theta, widths, n_widths, st);
        float* occ = occ_per_root ? occ_per_root
                                  : (float*)scratch(ctx, kMlpOcc, std::max<int64_t>(1, n_roots) * sizeof(float));
        MlpRows R{};
        R.source = kRowsRoots;
        R.n = n_roots;
        R.roots = roots;
        R.pose = pose;
        R.n_pose = n_pose;
        run_fwd(ctx, s, widths, n_widths, pk, R, occ, st);
        if (n > 0) FSK_LAUNCH(ctx, st, k_occ_reduce, blocks_for(n, 256), 256, 0, occ, offsets, n, pred, argmax);
    });
}

int fsk_distill_bwd(fsk_ctx* ctx, const float* theta, const int32_t* widths, int32_t n_widths,
                    const fsk_grid_desc* desc, const float* grad_w, float* grad_theta, void* stream) {
    return guard([&] {
        set_device(ctx);
        if (!desc || !widths || !theta || !grad_w || !grad_theta) fail(FSK_EINVAL, "fsk: null buffer");
        if (desc->nx < 2 || desc->ny < 2 || desc->nz < 2) fail(FSK_EINVAL, "distill: dims must be >= 2 per axis");
        if (n_widths < 2 || widths[0] != 3) fail(FSK_EINVAL, "SkinningMlp: network input width must be 3");
        if (widths[n_widths - 1] != desc->n_bones) fail(FSK_EINVAL, "distill: bone count mismatch");
        const MlpShape s = mlp_shape(widths, n_widths, true);
        cudaStream_t st = (cudaStream_t)stream;
        const int64_t V = (int64_t)desc->nx * desc->ny * desc->nz;
        if (V >= (int64_t(1) << 31)) fail(FSK_EINVAL, "fsk: grid too large");
        const int H = s.H, nb = s.n_out, L = n_widths - 1;  // weight layers
        // forward with the activations kept: x [V][4], h_l [L-1][V][H], w [V][nb]
        const float* pk = pack(ctx, s, theta, widths, n_widths, st);
        float* act = (float*)scratch(ctx, kMlpAct, (size_t)(4 * V + (int64_t)(L - 1) * V * H) * sizeof(float));
        float* w = (float*)scratch(ctx, kMlpOcc, (size_t)V * nb * sizeof(float));
        MlpRows R{};
        R.source = kRowsGrid;
        R.n = V;
        R.nx = desc->nx;
        R.ny = desc->ny;
        const int n3[3] = {desc->nx, desc->ny, desc->nz};
        for (int a = 0; a < 3; ++a) {
            R.lo[a] = (float)desc->bbox_min[a];
            R.h[a] = (float)(((double)desc->bbox_max[a] - (double)desc->bbox_min[a]) / (n3[a] - 1));
        }
        run_fwd(ctx, s, widths, n_widths, pk, R, w, st, act);
        // backward (Mlp::backward, mlp.cpp:140-163): fused tiles on the CUDA cores, FP32
        BwdNet net{};
        net.L = L;
        net.nw = n_widths;
        int64_t o = 0;
        net.maxw = 0;
        for (int l = 0; l < n_widths; ++l) {
            net.w[l] = widths[l];
            net.maxw = std::max(net.maxw, (int)widths[l]);
        }
        net.maxw = (net.maxw + 3) / 4 * 4;
        for (int l = 0; l < L; ++l) {
            net.off[l] = o;
            o += (int64_t)widths[l + 1] * widths[l] + widths[l + 1];
        }
        net.P = o;
        const size_t smb = (size_t)(3 * kBT * net.maxw + net.maxw * net.maxw) * sizeof(float);
        cuda_check(cudaFuncSetAttribute(k_mlp_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb),
                   "cudaFuncSetAttribute");
        const int64_t tiles = (V + kBT - 1) / kBT;
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, ctx->sm_count));
        float* part = (float*)scratch(ctx, kMlpD0, (size_t)grid * net.P * sizeof(float));
        FSK_LAUNCH(ctx, st, k_mlp_bwd, grid, 256, smb, net, theta, act, w, grad_w, V, H, part);
        FSK_LAUNCH(ctx, st, k_bwd_reduce, blocks_for(net.P, 256), 256, 0, part, grid, net.P, grad_theta);
    });
}

}  // extern "C"
