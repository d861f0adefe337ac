// fsk_ctx.h — host-side internals shared by the C-ABI translation units: the context
// (device, growable scratch, launch counter, optional per-launch event profiling), error
// handling (no exception crosses the C-ABI), and argument validation with the
// reference's messages.
#pragma once

#include <cuda_runtime.h>


#include <algorithm>
#include <cmath>
#include <cstdint>
#include <string>
#include <vector>

#include "fsk.h"
#include "fsk_device.cuh"

struct fsk_ctx {
    int device = 0;
    int sm_count = 0;
    int64_t launches = 0;
    static constexpr int kSlots = 80;
    void* buf[kSlots] = {};
    size_t cap[kSlots] = {};
    // optional per-launch CUDA-event profiling (bench.py reads per-kernel device time)
    bool prof_on = false;
    cudaEvent_t pending = nullptr;
    cudaStream_t pending_stream = nullptr;
    struct Rec {
        const char* name;
        cudaEvent_t a, b;
    };
    std::vector<Rec> prof;
    std::vector<cudaEvent_t> pool;
    // search work counters [solves32, iters32, final32, solves64, iters64, final64, fills32, -],
    // then (FSK_ESC_REASONS study builds) per-rule escalation counters
    static constexpr int kStatSlots = 48;
    unsigned long long* stats = nullptr;
    // device→host copy stream of the host-buffer entry point (created on first use)
    cudaStream_t copy = nullptr;
    cudaStream_t upload = nullptr;  // host→device stream of the host-buffer entry point
    // side stream + fork/join events: the spatial sort of a search runs beside K1 (precompute)
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    int64_t* hcount = nullptr;  // pinned per-chunk root counts
    int64_t last_search_n = -1;  // point count of the last device search (its order is in scratch kPerm)
    // bumped on every scratch (re)allocation: the host pipeline's captured graphs key on it
    uint64_t scratch_gen = 0;
    // CUDA graphs of the host pipeline's per-chunk device work (search + dedup + compaction),
    // keyed on everything the captured launches bake in (fsk_search.cu, deform_host_pipeline)
    struct PipeGraph {
        std::vector<unsigned char> key;
        cudaGraphExec_t exec = nullptr;  // null: seen once (ran eagerly); captured on the next sight
        int64_t launches = 0;
        unsigned char planes[64];
        uint64_t last_use = 0;
    };
    std::vector<PipeGraph> pipe_graphs;
    uint64_t pipe_clock = 0;
    cudaStream_t cap_stream = nullptr;  // capture stream (the caller's may be the legacy default stream)
    cudaStream_t pre = nullptr;  // host pipeline: sort + K1 of the next item, beside the current item's search
    std::vector<cudaEvent_t> frame_ev;  // fsk_deform_frames' fork/join events
};

namespace fsk {

// Scratch slots (one growable device buffer each).
enum Slot {
    kHist, kBbox, kKeys, kPerm, kXs, kScanPart, kScanLB, kBwdAcc, kBwdMax, kPlanes, kPlanes64, kEscQ, kEscN, kEscState,
    kBwdStart, kBwdCell, kBwdRec, kPeakTable, kBwdU, kBwdOk,
    kOXr, kOJa, kOJb, kOJc, kOMeta, kOKeep, kOKeepMask, kNRoots, kOffs, kRootsTmp, kOXd,
    kHW, kHB, kHP, kHT, kHOffs, kHRoots, kFB, kFP, kFOffs, kFRoots,
    kMlpPack, kMlpWidths, kMlpOcc, kMlpAct, kMlpD0, kMlpD1, kMlpOnes,
    kMvPos, kMvPosNext, kMvW, kMvX, kMvG, kMvJ, kMvDx, kMvK, kMvAct, kMvActNext, kMvCnt,
    // second copies of the sort / K1 scratch: the host pipeline stages item i+1 while item i searches
    kHistB, kKeysB, kPermB, kXsB, kEscNB, kPlanesB, kPlanes64B,
    kSlotCount
};
static_assert(kSlotCount <= fsk_ctx::kSlots, "scratch slots");

struct Error {
    int code;
    std::string msg;
};

[[noreturn]] inline void fail(int code, const std::string& m) { throw Error{code, m}; }

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(FSK_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

void set_error(const std::string& m);  // thread-local fsk_last_error text (fsk_ctx.cu)

template <typename Fn>
int guard(Fn&& fn) {
    try {
        fn();
        return FSK_OK;
    } catch (const Error& e) {
        set_error(e.msg);
        return e.code;
    } catch (const std::exception& e) {
        set_error(e.what());
        return FSK_ECUDA;
    }
}

void* scratch(fsk_ctx* ctx, int slot, size_t bytes);
void set_device(fsk_ctx* ctx);
void prof_begin(fsk_ctx* ctx, cudaStream_t st);
void after_launch(fsk_ctx* ctx, const char* name);

GridP make_grid(const fsk_grid_desc* d);
SearchP make_search(const fsk_search_opts* o);
// exclusive scan of n int32 into n+1 int64 (out[n] = total); fsk_search.cu
void scan_i32_to_i64(fsk_ctx* ctx, const int32_t* in, int64_t n, int64_t* out, cudaStream_t st);

// fsk_mlp.cu: the skinning network for the MLP-variant search
const float* mlp_skinning_pack(fsk_ctx* ctx, const float* theta, const int32_t* widths, int nw, cudaStream_t st);
void mlp_skinning_eval(fsk_ctx* ctx, const float* pk, const int32_t* widths, int nw, const float4* pos, int64_t n_rows,
                       bool tangent, float* out, cudaStream_t st);

inline unsigned blocks_for(int64_t n, int t) { return (unsigned)std::max<int64_t>(1, (n + t - 1) / t); }

}  // namespace fsk

// Launch helper: optional profiling events around the launch, launch counting and error
// check. Usage: FSK_LAUNCH(ctx, st, kernel, grid, block, smem, args...).
#define FSK_LAUNCH(ctx, st, kern, grid, block, smem, ...)       \
    do {                                                        \
        ::fsk::prof_begin((ctx), (st));                         \
        kern<<<(grid), (block), (smem), (st)>>>(__VA_ARGS__);   \
        ::fsk::after_launch((ctx), #kern);                      \
    } while (0)
