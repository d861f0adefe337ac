// fsk_ctx.cu — context lifecycle, scratch, errors, validation, profiling hooks and the
// FP32 roofline microbenchmark of the C-ABI (include/fsk.h).
#include <cstdlib>
#include <cstring>
#include <stdexcept>

#include "fsk_ctx.h"

namespace fsk {

namespace {
thread_local std::string g_err;
}

void set_error(const std::string& m) { g_err = m; }

void* scratch(fsk_ctx* ctx, int slot, size_t bytes) {
    if (bytes == 0) bytes = 16;
    if (ctx->cap[slot] < bytes) {
        if (ctx->buf[slot]) cuda_check(cudaFree(ctx->buf[slot]), "cudaFree");
        ctx->buf[slot] = nullptr;
        ctx->cap[slot] = 0;
        const size_t b = bytes + bytes / 8;
        cuda_check(cudaMalloc(&ctx->buf[slot], b), "cudaMalloc");
        ctx->cap[slot] = b;
        ctx->scratch_gen++;
    }
    return ctx->buf[slot];
}

void set_device(fsk_ctx* ctx) {
    if (!ctx) fail(FSK_EINVAL, "fsk: null context");
    cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
}

namespace {
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
}  // namespace

void prof_begin(fsk_ctx* ctx, cudaStream_t st) {
    if (!ctx->prof_on) return;
    ctx->pending = pooled_event(ctx);
    ctx->pending_stream = st;
    cuda_check(cudaEventRecord(ctx->pending, st), "cudaEventRecord");
}

void after_launch(fsk_ctx* ctx, const char* name) {
    ctx->launches++;
    cuda_check(cudaGetLastError(), name);
    if (ctx->prof_on && ctx->pending) {
        cudaEvent_t b = pooled_event(ctx);
        cuda_check(cudaEventRecord(b, ctx->pending_stream), "cudaEventRecord");
        ctx->prof.push_back({name, ctx->pending, b});
        ctx->pending = nullptr;
    }
}

GridP make_grid(const fsk_grid_desc* d) {
    if (!d) fail(FSK_EINVAL, "fsk: null grid descriptor");
    // SkinningVoxelGrid ctor checks (skinning.cpp:60-70)
    if (d->nx < 2 || d->ny < 2 || d->nz < 2) fail(FSK_EINVAL, "SkinningVoxelGrid: dims must be >= 2 per axis");
    if (d->n_bones < 1) fail(FSK_EINVAL, "SkinningVoxelGrid: n_bones must be >= 1");
    if ((int64_t)d->nx * d->ny * d->nz >= (int64_t(1) << 30)) fail(FSK_EINVAL, "fsk: grid too large (>= 2^30 vertices)");
    GridP g;
    g.nx = d->nx;
    g.ny = d->ny;
    g.nz = d->nz;
    g.nb = d->n_bones;
    const int n[3] = {d->nx, d->ny, d->nz};
    for (int a = 0; a < 3; ++a) {
        // the reference's float64 Aabb as given (the exact replay and the float64 re-solves use it);
        // the float32 pass works on its rounding
        g.lod[a] = d->bbox_min[a];
        g.hid[a] = d->bbox_max[a];
        if (!(g.hid[a] - g.lod[a] > 0.0)) fail(FSK_EINVAL, "SkinningVoxelGrid: bbox must have positive extent");
        g.lo[a] = (float)g.lod[a];
        g.hi[a] = (float)g.hid[a];
        if (!(g.hi[a] - g.lo[a] > 0.f)) fail(FSK_EINVAL, "fsk: bbox extent below float32 resolution");
        g.scaled[a] = (double)(n[a] - 1) / (g.hid[a] - g.lod[a]);  // skinning.cpp:109 in f64
        g.scale[a] = (float)g.scaled[a];
    }
    return g;
}

SearchP make_search(const fsk_search_opts* o) {
    if (!o) fail(FSK_EINVAL, "fsk: null search options");
    // SearchOptions::validate (correspondence.cpp:19-25)
    if (o->max_iters < 1) fail(FSK_EINVAL, "search: max_iters must be >= 1");
    if (!(o->conv_eps > 0.0)) fail(FSK_EINVAL, "search: conv_eps must be > 0");
    if (!(o->div_eps > o->conv_eps)) fail(FSK_EINVAL, "search: div_eps must exceed conv_eps");
    if (!(o->dedup_dist >= 0.0)) fail(FSK_EINVAL, "search: dedup_dist must be >= 0");
    if ((o->flags & FSK_SEARCH_FP32_ONLY) && (o->flags & FSK_SEARCH_FP64))
        fail(FSK_EINVAL, "fsk: FSK_SEARCH_FP32_ONLY and FSK_SEARCH_FP64 are exclusive");
    SearchP s;
    s.max_iters = o->max_iters;
    if ((o->flags & FSK_SEARCH_FP32_ONLY) && (o->flags & FSK_SEARCH_EXACT64))
        fail(FSK_EINVAL, "fsk: FSK_SEARCH_FP32_ONLY and FSK_SEARCH_EXACT64 are exclusive");
    if ((o->flags & FSK_SEARCH_FAST_ESC) && (o->flags & (FSK_SEARCH_FP32_ONLY | FSK_SEARCH_FP64 | FSK_SEARCH_EXACT64)))
        fail(FSK_EINVAL, "fsk: FSK_SEARCH_FAST_ESC applies to the mixed mode only");
    s.conv_eps = o->conv_eps;
    s.div_eps = o->div_eps;
    s.conv2 = o->conv_eps * o->conv_eps;
    s.div2 = o->div_eps * o->div_eps;
    s.dedup2 = o->dedup_dist * o->dedup_dist;
    // Escalation rule of the float32 pass (validated on 1.5M solves
    // against the f64 oracle with oracle/precision_emul.cpp): cap at 8 iterations, escalate
    // unconverged runs of >= esc_min_div iterations, and any threshold decision within float32 noise:
    // err^2 within ±2% of conv^2 (f32 residuals near conv carry ~1e-7/3e-5 relative error),
    // within ±2e-4 of div^2, |det J0| < 1e-5 (vs the 1e-8 singular cut), |den| < 1e-12
    // (vs the 1e-18 Broyden guard).
    // Conditioning (scripts/escalation_rules.py, 72 scenes × 720k solves: without it
    // max|dx| reached 4.8e-4 on 64^3 / 128x128x32 grids): a converged root with max|J~| > 6 (5 since round 2)
    // (rounding amplified into x*), or any Broyden update with |cos(dx, J~dg)| < 0.1
    // (near-degenerate rank-one update). Bands are on err, like the emulator's:
    // |err/conv - 1| < 2 %, |err/div - 1| < 2e-4.
    s.esc_cap = 8;
    // unconverged (diverged) runs escalate from 5 iterations on: GPU band study over 150 scenes
    // (108 M solves, scripts/gpu_esc_study.sh) — 3: 1 mask flip, 5: 5, 6: 10, 8 (rule off): 61; roots
    // unchanged (max |dx| 8.1e-5 in all). 5 escalates 12 % fewer solves than 3 (C2: 4.85 % -> 4.25 %).
    s.esc_min_div = 5;
    s.esc_conv_lo = 0.98f * 0.98f;
    s.esc_conv_hi = 1.02f * 1.02f;
    s.esc_div_lo = (1.0f - 2e-4f) * (1.0f - 2e-4f);
    s.esc_div_hi = (1.0f + 2e-4f) * (1.0f + 2e-4f);
    s.esc_det = 1e-5f;
    s.esc_den = 1e-12f;
    // 6 until round 2; the round-2 band study (seeds 112-141, FMA oracle) found one 3-iteration root
    // 1.01e-4 from the oracle's with max|J~| 5.17 — at 5 it is escalated (+0.006 % of solves on C2)
    s.esc_jmax = 5.0f;
    s.esc_cos2 = 0.1f * 0.1f;
    // Stagnation (round 2, C5 ray workload in full against the reference's own code, 192 M solves): one
    // 6-iteration root 1.07e-4 from float64's — the two trajectories parted at iteration 2, where the
    // residual barely fell (3.544e-3 -> 3.535e-3), and both stopped within conv of the root on opposite
    // sides (|x - x*| ~ |J~|·conv with max|J~| 3.3). A converged solve with a step from iteration 2 on that
    // cut err by < 10 % and max|J~| > 2.5 is escalated: +0.04 % of the solves (oracle trajectories, 480 k
    // solves of the ray workload).
    // Init on a cell face (round 2, 150-scene ray-sample band study, seed 252): an init point whose y sat
    // on a grid plane to float32 precision took the other cell's (piecewise) Jacobian in float32 — J0
    // differed by 0.15 in one column, the first steps parted, and the solve converged to another root
    // 0.22 away. Init points within 1e-4 cells of a grid plane escalate (~0.06 % of the solves).
    s.esc_face = 1e-4f;
    // Transient J~ spike (round 2, 600-scene band study, seeds 322-441, and seed 265): converged roots
    // 1.1-1.9e-4 from float64's whose Broyden matrices reached max|J~| 7-36 on the way (ending at 1.3-1.7):
    // the spike amplified float32 rounding into the path. Converged solves whose matrix exceeded 7 at any
    // iteration escalate (~0.07 % of the solves on oracle trajectories).
    s.esc_spike = FSK_ESC_SPIKE;  // informational: the float32 pass uses the compile-time constant
    s.esc_stag2 = 0.9f * 0.9f;
    s.esc_stag_jmax = 2.5f;
    // Step rule (scripts/band_study.py on the GPU, 30 scenes × 720k solves: converged solves
    // whose iteration count differed from the oracle's by one had the float32 err/conv as low
    // as 0.84 on one side and the oracle's as high as 0.93 on the other; the roots then differ
    // by one step, up to 4·conv): rho = 0.7, tau = 2 (a one-step difference stays < 2·conv).
    s.esc_rho2 = 0.7f * 0.7f;
    s.esc_tau2 = 2.0f * 2.0f;
    // Absolute bar: the step rule bounds a one-step disagreement by tau·conv = 2·conv_eps, which is
    // within the north star's 1e-4 only while conv_eps <= 5e-5 (SMPL scale: conv 3.4e-5). On larger
    // scenes (conv_eps = 1e-5·diag, e.g. 40-80-bone chains of 50-100 m, where float32 also resolves
    // coordinates only to ~4e-6) every converged float32 solve is re-solved by the float64 pass.
    s.esc_conv_all = o->conv_eps > 5e-5;
    s.esc_conv_band_last = false;
    // Converged on the cap iteration with a last step > tau·conv: as chaotic as a capped trajectory.
    // Band study on seeds 52-81 (108 M solves): without it one root 1.6e-4 from the oracle's (float32
    // stopped at iteration 8 with err 0.52·conv, float64 needed 9); with it max |dx| 8.7e-5.
    // Escalation on C2 4.25 % -> 5.15 %.
    s.esc_capconv = 2;
#ifdef FSK_ESC_STUDY  // rule-study builds only: overrides from the environment
    if (const char* v = getenv("FSK_ESC_CONV_BAND_LAST")) s.esc_conv_band_last = atoi(v) != 0;
    if (const char* v = getenv("FSK_ESC_MIN_DIV")) s.esc_min_div = atoi(v);
    if (const char* v = getenv("FSK_ESC_COS")) s.esc_cos2 = (float)(atof(v) * atof(v));
    if (const char* v = getenv("FSK_ESC_CAPCONV")) s.esc_capconv = atoi(v);
    if (const char* v = getenv("FSK_ESC_CAP")) s.esc_cap = atoi(v);
    if (const char* v = getenv("FSK_ESC_JMAX")) s.esc_jmax = (float)atof(v);
    if (const char* v = getenv("FSK_ESC_STAG_JMAX")) s.esc_stag_jmax = (float)atof(v);
    if (const char* v = getenv("FSK_ESC_FACE")) s.esc_face = (float)atof(v);
#endif
    return s;
}

// FMA throughput microbenchmark: 8 independent dependency chains per thread over all SMs.
template <typename R>
__global__ void __launch_bounds__(256) k_peak_fma(R* out, int iters, R a, R b) {
    R x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * (R)1e-3 + i;
    for (int k = 0; k < iters; ++k) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
    }
    R s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == (R)12345.678) out[0] = s;  // keep the chains alive
}

// L1 gather microbenchmark: every lane issues independent 256-bit loads at pseudo-random
// 32-byte-aligned offsets of a 64 KiB table (L1-resident after the first touch) — the access
// pattern of the search's x-pair gathers with no reuse between lanes. Returns the bytes
// delivered to registers per second: the roofline denominator of the gather-bound kernels.
__global__ void __launch_bounds__(256) k_peak_l1_gather(const float* __restrict__ table, float* out, int iters) {
    uint32_t s = (blockIdx.x * 256u + threadIdx.x) * 2654435761u + 12345u;
    float acc = 0.f;
    for (int k = 0; k < iters; ++k) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            s = s * 1664525u + 1013904223u;
            const float* q = table + ((s >> 8) & 2047u) * 8;  // 2048 slots × 32 B
            float a0, a1, a2, a3, a4, a5, a6, a7;
            asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=f"(a0), "=f"(a1), "=f"(a2), "=f"(a3), "=f"(a4), "=f"(a5), "=f"(a6), "=f"(a7)
                         : "l"(q));
            acc += ((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7));
        }
    }
    if (acc == 12345.678f) out[0] = acc;
}

// L2 vector reductions at random float4 slots of a [32^3][12] float grid (the backward's scatter target)
__global__ void __launch_bounds__(256) k_peak_red(float4* __restrict__ grid, uint32_t slots, int iters) {
    uint32_t s = (blockIdx.x * 256u + threadIdx.x) * 2654435761u + 777u;
    for (int k = 0; k < iters; ++k) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            s = s * 1664525u + 1013904223u;
            atomicAdd(grid + (s >> 8) % slots, make_float4(1e-7f, 1e-7f, 1e-7f, 1e-7f));
        }
    }
}

template <typename R>
double measure_peak(fsk_ctx* ctx, int iters) {
    R* o = (R*)scratch(ctx, kBwdMax, 16);
    const int blocks = ctx->sm_count * 8;
    cudaEvent_t a, b;
    cuda_check(cudaEventCreate(&a), "cudaEventCreate");
    cuda_check(cudaEventCreate(&b), "cudaEventCreate");
    k_peak_fma<R><<<blocks, 256>>>(o, 256, (R)0.999, (R)1e-3);  // warm-up
    cuda_check(cudaEventRecord(a, 0), "cudaEventRecord");
    k_peak_fma<R><<<blocks, 256>>>(o, iters, (R)0.999, (R)1e-3);
    cuda_check(cudaEventRecord(b, 0), "cudaEventRecord");
    cuda_check(cudaEventSynchronize(b), "cudaEventSynchronize");
    float ms = 0.f;
    cuda_check(cudaEventElapsedTime(&ms, a, b), "cudaEventElapsedTime");
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return 2.0 * 8.0 * iters * (double)blocks * 256.0 / (ms * 1e-3) / 1e12;
}

}  // namespace fsk

using namespace fsk;

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
        cuda_check(cudaSetDevice(device), "cudaSetDevice");
        auto* c = new fsk_ctx();
        c->device = device;
        c->sm_count = prop.multiProcessorCount;
#ifdef FSK_L2_PERSIST_STUDY  // study builds: L2 set-aside for evict_last lines (FSK_L2_PERSIST_MB)
        if (const char* e = getenv("FSK_L2_PERSIST_MB"))
            cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)atoll(e) << 20);
#endif
        if (cudaMalloc(&c->stats, fsk_ctx::kStatSlots * sizeof(unsigned long long)) != cudaSuccess ||
            cudaMemset(c->stats, 0, fsk_ctx::kStatSlots * sizeof(unsigned long long)) != cudaSuccess ||
            cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming) != cudaSuccess) {
            cudaGetLastError();
            fsk_ctx_destroy(c);  // releases whatever was created
            fail(FSK_ECUDA, "fsk: cannot allocate context state");
        }
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
        if (ctx->stats) cudaFree(ctx->stats);
        if (ctx->copy) cudaStreamDestroy(ctx->copy);
        if (ctx->upload) cudaStreamDestroy(ctx->upload);
        if (ctx->side) cudaStreamDestroy(ctx->side);
        if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
        if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
        if (ctx->hcount) cudaFreeHost(ctx->hcount);
        for (auto& pg : ctx->pipe_graphs)
            if (pg.exec) cudaGraphExecDestroy(pg.exec);
        if (ctx->cap_stream) cudaStreamDestroy(ctx->cap_stream);
        if (ctx->pre) cudaStreamDestroy(ctx->pre);
        for (auto e : ctx->frame_ev) cudaEventDestroy(e);
        delete ctx;
    });
}

int64_t fsk_ctx_launch_count(const fsk_ctx* ctx) { return ctx ? ctx->launches : -1; }
int fsk_device_sm_count(const fsk_ctx* ctx) { return ctx ? ctx->sm_count : -1; }

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
            if (name) {  // a kernel template matches its base name ("k" matches "k<true>")
                const size_t L = std::strlen(name);
                if (std::strncmp(name, r.name, L) != 0 || (r.name[L] != '\0' && r.name[L] != '<')) continue;
            }
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

#ifdef FSK_ESC_REASONS
// study builds only (scripts/esc_reasons.py, esc_timeline.py): debug counters, slots 8..47
extern "C" int fsk_ctx_esc_reasons(fsk_ctx* ctx, uint64_t out[40], int reset) {
    return guard([&] {
        set_device(ctx);
        cuda_check(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
        unsigned long long h[fsk_ctx::kStatSlots];
        cuda_check(cudaMemcpy(h, ctx->stats, sizeof(h), cudaMemcpyDeviceToHost), "cudaMemcpy");
        for (int i = 0; i < 40; ++i) out[i] = h[8 + i];
        if (reset) cuda_check(cudaMemset(ctx->stats + 8, 0, 40 * sizeof(unsigned long long)), "cudaMemset");
    });
}
#endif

int fsk_ctx_search_stats(fsk_ctx* ctx, uint64_t out[7], int reset) {
    return guard([&] {
        set_device(ctx);
        if (!out) fail(FSK_EINVAL, "fsk: null output pointer");
        cuda_check(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
        unsigned long long h[8];
        cuda_check(cudaMemcpy(h, ctx->stats, sizeof(h), cudaMemcpyDeviceToHost), "cudaMemcpy");
        for (int i = 0; i < 7; ++i) out[i] = h[i];
        if (reset) cuda_check(cudaMemset(ctx->stats, 0, sizeof(h)), "cudaMemset");
    });
}

int fsk_measure_fp32_peak(fsk_ctx* ctx, double* tflops) {
    return guard([&] {
        set_device(ctx);
        if (!tflops) fail(FSK_EINVAL, "fsk: null output pointer");
        *tflops = measure_peak<float>(ctx, 1 << 14);
    });
}

int fsk_measure_l1_gather_peak(fsk_ctx* ctx, double* gbps) {
    return guard([&] {
        set_device(ctx);
        if (!gbps) fail(FSK_EINVAL, "fsk: null output pointer");
        float* table = (float*)scratch(ctx, kPeakTable, 2048 * 8 * sizeof(float) + 64);
        cuda_check(cudaMemset(table, 0, 2048 * 8 * sizeof(float) + 64), "cudaMemset");
        const int blocks = ctx->sm_count * 8, iters = 1 << 10;
        cudaEvent_t a, b;
        cuda_check(cudaEventCreate(&a), "cudaEventCreate");
        cuda_check(cudaEventCreate(&b), "cudaEventCreate");
        k_peak_l1_gather<<<blocks, 256>>>(table, table + 2048 * 8, 16);  // warm-up
        cuda_check(cudaEventRecord(a, 0), "cudaEventRecord");
        k_peak_l1_gather<<<blocks, 256>>>(table, table + 2048 * 8, iters);
        cuda_check(cudaEventRecord(b, 0), "cudaEventRecord");
        cuda_check(cudaEventSynchronize(b), "cudaEventSynchronize");
        float ms = 0.f;
        cuda_check(cudaEventElapsedTime(&ms, a, b), "cudaEventElapsedTime");
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        *gbps = 32.0 * 8.0 * iters * (double)blocks * 256.0 / (ms * 1e-3) / 1e9;
    });
}

int fsk_measure_red_peak(fsk_ctx* ctx, double* gbps) {
    return guard([&] {
        set_device(ctx);
        if (!gbps) fail(FSK_EINVAL, "fsk: null output pointer");
        const uint32_t slots = 32 * 32 * 32 * 3;
        float4* grid = (float4*)scratch(ctx, kPeakTable, slots * sizeof(float4));
        cuda_check(cudaMemset(grid, 0, slots * sizeof(float4)), "cudaMemset");
        const int blocks = ctx->sm_count * 8, iters = 64;
        cudaEvent_t a, b;
        cuda_check(cudaEventCreate(&a), "cudaEventCreate");
        cuda_check(cudaEventCreate(&b), "cudaEventCreate");
        k_peak_red<<<blocks, 256>>>(grid, slots, 4);  // warm-up
        cuda_check(cudaEventRecord(a, 0), "cudaEventRecord");
        k_peak_red<<<blocks, 256>>>(grid, slots, iters);
        cuda_check(cudaEventRecord(b, 0), "cudaEventRecord");
        cuda_check(cudaEventSynchronize(b), "cudaEventSynchronize");
        float ms = 0.f;
        cuda_check(cudaEventElapsedTime(&ms, a, b), "cudaEventElapsedTime");
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        *gbps = 16.0 * 8.0 * iters * (double)blocks * 256.0 / (ms * 1e-3) / 1e9;
    });
}

int fsk_measure_fp64_peak(fsk_ctx* ctx, double* tflops) {
    return guard([&] {
        set_device(ctx);
        if (!tflops) fail(FSK_EINVAL, "fsk: null output pointer");
        *tflops = measure_peak<double>(ctx, 1 << 12);
    });
}

fsk_search_opts fsk_search_opts_defaults(const fsk_grid_desc* d) {
    fsk_search_opts o{50, 0, 1e-5, 0.5, 1e-2};
    if (!d) return o;
    double s = 0.0;
    for (int a = 0; a < 3; ++a) {
        const double e = (double)d->bbox_max[a] - (double)d->bbox_min[a];
        s += e * e;
    }
    const double diag = std::sqrt(s);
    o.conv_eps = 1e-5 * diag;
    o.div_eps = 0.5 * diag;
    o.dedup_dist = 1e-2 * diag;
    return o;
}

}  // extern "C"
