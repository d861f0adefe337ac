/* fsk.h — C-ABI of the B200-native Fast-SNARF deformer (sm_100a).
 *
 * Drop-in boundary for the reference's deformer/correspondence hot path
 * (/root/reference/proj/include/fskin/deformer.hpp, correspondence.hpp). Every entry
 * point is `extern "C"`, takes plain pointers and sizes, never throws, and returns
 *   FSK_OK (0)            success
 *   FSK_EINVAL (1)        invalid argument — fsk_last_error() holds the reference's
 *                         std::invalid_argument message text where one exists
 *   FSK_ECUDA (2)         CUDA / allocation failure (std::runtime_error)
 *   FSK_ENODEV (3)        no usable sm_100 device (the library has no CPU fallback)
 *   FSK_EIO (4)           file I/O failure of the wire-format helpers (std::runtime_error;
 *                         text in fsk_io_last_error())
 * Device pointers ("dev") must live on the context's device. Calls are stream-ordered
 * on `stream` (a cudaStream_t; NULL = legacy default stream) and asynchronous unless
 * stated otherwise. A context is not thread-safe; distinct (ctx, stream) pairs are.
 *
 * Layouts (the reference's storage order; float32 unless noted):
 *   weights  [V][n_b]     x-fastest vertex order, bone innermost (skinning.hpp:54-77)
 *   tgrid    [V][12]      rows of the blended 3x4 [R|t], x-fastest (deformer.hpp:35-39)
 *   bones    [n_b][12]    rows of RigidTransform [R|t] (geometry.hpp:42-78)
 *   points   [N][3]
 *   per-(point, init) outputs are point-major: [N][n_init][...], init i = bone i.
 *
 * Precision: searches run a float32 pass and re-solve in float64 every (point, init)
 * whose float32 outcome could differ from a float64 solve (long or late-diverging Broyden
 * trajectories, threshold decisions within float32 noise); see DESIGN.md §precision.
 */
#ifndef FSK_H_
#define FSK_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FSK_OK 0
#define FSK_EINVAL 1
#define FSK_ECUDA 2
#define FSK_ENODEV 3
#define FSK_EIO 4

typedef struct fsk_ctx fsk_ctx;

/* GridDims + canonical Aabb of a SkinningVoxelGrid / TransformGrid
 * (skinning.hpp:45-52, :57-91; deformer.hpp:27-49). */
typedef struct fsk_grid_desc {
    int32_t nx, ny, nz;   /* >= 2 per axis (skinning.cpp:62-64) */
    int32_t n_bones;      /* n_b of the weight grid */
    double bbox_min[3];   /* the reference's float64 Aabb (geometry.hpp:14-39); the float32 pass */
    double bbox_max[3];   /* rounds it, the float64 re-solves use it as given */
} fsk_grid_desc;

/* SearchOptions (correspondence.hpp:14-26); fill from fsk_search_opts_defaults()
 * = SearchOptions::defaults_for(bbox) (correspondence.cpp:10-17). */
typedef struct fsk_search_opts {
    int32_t max_iters;    /* >= 1 (correspondence.cpp:20) */
    int32_t flags;        /* FSK_SEARCH_* */
    double conv_eps;      /* > 0 */
    double div_eps;       /* > conv_eps */
    double dedup_dist;    /* >= 0 */
} fsk_search_opts;

#define FSK_SEARCH_NO_SORT 0x1    /* ablation: skip the spatial ordering of queries */
#define FSK_SEARCH_FP32_ONLY 0x2  /* ablation: float32 only, no float64 escalation */
#define FSK_SEARCH_FP64 0x4       /* parity mode: every solve in float64 */
#define FSK_SEARCH_EXACT64 0x8    /* replay mode: every solve in float64 in the oracle's operation order
                                     (oracle/fskin_oracle.cpp: the reference's code with Eigen's closed
                                     forms, unfused, J~0 from the n_b-wide weight grid), bit-identical to
                                     the oracle given the same transform grid. The reference's own
                                     operation order is not pinned (Eigen unpinned, -march=native): its
                                     plausible builds differ from each other by ~1 mask flip per 2M solves
                                     (scripts/oracle_variants.py). Needs the weight
                                     grid (fsk_search_fwd / fsk_batch_search `weights`; always present in
                                     fsk_deform*) */
#define FSK_SEARCH_FAST_ESC 0x10  /* mixed mode, ablation: escalate to the fused float64 solver
                                     (transform-grid J~0) even when the weight grid is given. By
                                     default the escalation pass is the exact replay whenever the weight
                                     grid is available (always in fsk_deform*; fsk_search_fwd /
                                     fsk_batch_search when `weights` != NULL), so escalated solves equal
                                     the oracle's bit for bit */

/* Dense per-(point, init) search result (the GPU form of Root / CorrespondenceSet,
 * correspondence.hpp:29-42). All pointers dev, [N][n_b] point-major; any may be NULL
 * except `converged`. `keep` is the dedup_roots mask (correspondence.cpp:162-176):
 * keep=1 iff the init converged and survived greedy bone-order dedup. `n_roots`
 * [N] int32 = number of kept roots per point. */
typedef struct fsk_search_out {
    float* x_c;           /* [N][n_b][3] canonical root (Root::x) */
    float* jinv;          /* [N][n_b][9] Broyden inverse-Jacobian estimate (Root::inv_jacobian) of the
                             converged solves; NaN for the others (no Root) */
    float* resid;         /* [N][n_b] ||d(x)-x'|| at termination (Root::residual) */
    int32_t* iters;       /* [N][n_b] iterations executed (Root::iterations) */
    uint8_t* converged;   /* [N][n_b] 1 iff residual < conv_eps was reached */
    uint8_t* keep;        /* [N][n_b] dedup survivors */
    int32_t* n_roots;     /* [N] kept roots per point */
    double* x_c64;        /* [N][n_b][3] optional: Root::x in float64 — the float64 state of the solves the
                             float64 pass ran (escalated / FSK_SEARCH_FP64 / EXACT64), the float32 root
                             widened otherwise */
} fsk_search_out;

/* Compact root record — one kept Root, in bone order per query (CorrespondenceSet). */
typedef struct fsk_root {
    float x[3];
    float residual;
    float inv_jacobian[9];
    int32_t source_bone;
    int32_t iterations;
    int32_t _pad;
} fsk_root; /* 64 bytes */

/* ---- lifecycle ------------------------------------------------------------------ */
int fsk_ctx_create(int device, fsk_ctx** out);
int fsk_ctx_destroy(fsk_ctx* ctx);
const char* fsk_last_error(void);                 /* thread-local, never NULL */
int64_t fsk_ctx_launch_count(const fsk_ctx* ctx); /* kernels launched by this ctx so far */
int fsk_device_sm_count(const fsk_ctx* ctx);

/* Measurement hooks (bench.py): when profiling is on, every kernel launch of the context is
 * bracketed by CUDA events on its stream; fsk_ctx_prof_read synchronizes and returns the
 * summed device time and launch count of the kernels named `name` (NULL = all), and
 * recycles the events when `reset` != 0. fsk_measure_fp32_peak times an FFMA-chain kernel
 * over all SMs (the FP32 roofline denominator) and returns TFLOP/s. */
int fsk_ctx_set_profiling(fsk_ctx* ctx, int on);
int fsk_ctx_prof_read(fsk_ctx* ctx, const char* name, double* total_ms, int64_t* count, int reset);
int fsk_measure_fp32_peak(fsk_ctx* ctx, double* tflops);
int fsk_measure_fp64_peak(fsk_ctx* ctx, double* tflops);  /* same with DFMA chains */
/* L1 gather delivery rate (GB/s): independent 256-bit loads at random 32-B slots of an
 * L1-resident table, the access pattern of the search's gathers (roofline denominator). */
int fsk_measure_l1_gather_peak(fsk_ctx* ctx, double* gbps);
/* L2 vector-reduction rate (GB/s of red payload): RED.E.ADD.F32x4 from all SMs to random float4 slots of
 * an L2-resident [32^3][12] float grid — the access pattern of the backward's scatter (K3 roofline). */
int fsk_measure_red_peak(fsk_ctx* ctx, double* gbps);
/* Search work counters accumulated by the context's searches (synchronizes the device):
 * out = {float32 solves, float32 Broyden iterations, float32 converged-terminating
 * iterations, float64 solves, float64 iterations, float64 converged-terminating iterations,
 * float32 iteration gathers (re-evaluations that left the cell cached in registers)}. */
int fsk_ctx_search_stats(fsk_ctx* ctx, uint64_t out[7], int reset);

/* SearchOptions::defaults_for (correspondence.cpp:10-17): conv 1e-5*diag,
 * div 0.5*diag, dedup 1e-2*diag, max_iters 50. */
fsk_search_opts fsk_search_opts_defaults(const fsk_grid_desc* desc);

/* ---- K1: precompute_transform_grid (deformer.hpp:53-55; deformer.cpp:61-77) -------
 * tgrid[v] = lbs_blend(weights[v], bones) (deformer.cpp:9-19) in float32 and/or, into
 * tgrid64 (double [V][12], the reference's TransformGrid precision), in float64; either
 * output may be NULL (not both). n_bones_pose must equal desc->n_bones
 * ("precompute_transform_grid: bone count mismatch"). All dev. */
int fsk_precompute_tgrid(fsk_ctx* ctx, const float* weights, const fsk_grid_desc* desc,
                         const float* bones, int32_t n_bones_pose, float* tgrid, double* tgrid64,
                         void* stream);

/* ---- K2: batch_search, voxel variant (correspondence.hpp:77-80; correspondence.cpp:178-192)
 * One Broyden solve per (point, bone-init): x0 = B_i^-1 x' (:135), J~0 from the analytic
 * grid Jacobian (:43-54), good-Broyden iterate (:97-124), converged mask, dedup (:162-176).
 * The transform grid is given as float32 `tgrid` and/or float64 `tgrid64` (either may be
 * NULL, not both); the float64 re-solves read tgrid64 when given (exact parity with an f64
 * TransformGrid), else the float32 grid widened. `weights` [V][n_b] (dev) is the skinning
 * weight grid (SearchContext::grid); it is read only under FSK_SEARCH_EXACT64 and may be NULL
 * otherwise. points, grids, bones dev. N may be 0. */
int fsk_search_fwd(fsk_ctx* ctx, const float* tgrid, const double* tgrid64,
                   const float* weights, const fsk_grid_desc* desc, const float* bones, int32_t n_bones_pose,
                   const float* points, int64_t n, const fsk_search_opts* opts,
                   fsk_search_out* out, void* stream);

/* batch_search straight to CorrespondenceSets on the device: K2 + dedup + compaction.
 * offsets [N+1] int64 (dev): roots of query p are roots[offsets[p] .. offsets[p+1]), in bone
 * order (Root::source_bone ascending); offsets[N] = total kept roots. roots (dev) has room for
 * `cap` records; records beyond cap are dropped — check offsets[N] <= cap (N*n_b always
 * suffices). Fully asynchronous (no host synchronization). */
int fsk_batch_search(fsk_ctx* ctx, const float* tgrid, const double* tgrid64,
                     const float* weights, const fsk_grid_desc* desc, const float* bones, int32_t n_bones_pose,
                     const float* points, int64_t n, const fsk_search_opts* opts,
                     int64_t* offsets, fsk_root* roots, int64_t cap, void* stream);

/* One frame of the deformer on device buffers — precompute_transform_grid followed by
 * batch_search (what cmd_deform / cmd_bench / train do per pose: fskin_cli.cpp:395-408,
 * :663-678, diff.cpp:278-289): K1 (fused with the gather relayout, float32 + float64), K2,
 * dedup, compaction. tgrid [V][12] (dev) receives the float32 transform grid, or NULL.
 * Outputs as for fsk_batch_search. Fully asynchronous. */
int fsk_deform(fsk_ctx* ctx, const float* weights, const fsk_grid_desc* desc, const float* bones,
               int32_t n_bones_pose, const float* points, int64_t n, const fsk_search_opts* opts,
               float* tgrid, int64_t* offsets, fsk_root* roots, int64_t cap, void* stream);

/* Several frames (poses) of one subject on device buffers — fsk_deform per frame (cmd_deform over
 * a pose sequence, fskin_cli.cpp:395-429), with frame f+1's sort and K1 run on a second stream while
 * frame f searches. bones[f] [n_b][12], points[f] [n_points[f]][3], offsets[f] [n_points[f]+1],
 * roots[f] with capacity caps[f] (records beyond it are dropped: check offsets[f][n_points[f]]);
 * the arrays of device pointers are host arrays. tgrid [V][12] (dev) receives the last frame's
 * float32 transform grid, or NULL. Results equal per-frame fsk_deform calls bit for bit. Fully
 * asynchronous (capturable in a CUDA graph). */
int fsk_deform_frames(fsk_ctx* ctx, const float* weights, const fsk_grid_desc* desc, int32_t n_frames,
                      const float* const* bones, int32_t n_bones_pose, const float* const* points,
                      const int64_t* n_points, const fsk_search_opts* opts, float* tgrid,
                      int64_t* const* offsets, fsk_root* const* roots, const int64_t* caps, void* stream);

/* Stream-compaction of a dense result's kept roots into CorrespondenceSet form: offsets
 * [N+1] int64 (dev), roots [total] (dev, capacity `cap`). *total_out (host) receives the
 * number of kept roots; this call synchronizes `stream` to read it. Returns FSK_EINVAL if
 * cap is too small (roots untouched, *total_out still set). */
int fsk_compact_roots(fsk_ctx* ctx, const fsk_search_out* dense, int64_t n, int32_t n_init,
                      int64_t* offsets, fsk_root* roots, int64_t cap, int64_t* total_out,
                      void* stream);

/* End-to-end host-buffer entry point (one cmd_deform / cmd_bench frame): H2D of weights,
 * bones and points, fsk_deform, D2H of the CorrespondenceSets. All pointers are HOST memory
 * (pinned recommended). offsets [N+1]; roots capacity `cap`. Synchronous. */
int fsk_deform_host(fsk_ctx* ctx, const float* weights, const fsk_grid_desc* desc,
                    const float* bones, int32_t n_bones_pose, const float* points, int64_t n,
                    const fsk_search_opts* opts, int64_t* offsets, fsk_root* roots, int64_t cap,
                    int64_t* total_out, void* stream);

/* A sequence of frames of one subject (the pose loop of cmd_bench, fskin_cli.cpp:663-678, each
 * frame with cmd_deform's host copies, :395-429): weights [V][n_b] uploaded once; frame f has
 * its own bones[f] [n_b][12], points[f] [n_points[f]][3] and outputs offsets[f] [n_points[f]+1],
 * roots[f] (capacity caps[f]) and totals[f] — exactly what fsk_deform_host returns for that
 * frame. Double-buffered on the device: frame f+1's upload and search overlap frame f's
 * download. All pointers HOST memory (pinned for the overlap). Synchronous. */
int fsk_deform_host_frames(fsk_ctx* ctx, const float* weights, const fsk_grid_desc* desc, int32_t n_frames,
                           const float* const* bones, int32_t n_bones_pose, const float* const* points,
                           const int64_t* n_points, const fsk_search_opts* opts, int64_t* const* offsets,
                           fsk_root* const* roots, const int64_t* caps, int64_t* totals, void* stream);

/* ---- point evaluators (batch forms of trilerp_transform / forward_deform /
 * deform_jacobian, deformer.hpp:59-68): at points x [N][3] (dev) write T(x) [N][12],
 * d(x) [N][3] and the analytic Jacobian dd/dx [N][9] (transform-grid form).
 * Any output may be NULL. float32. */
int fsk_eval_points(fsk_ctx* ctx, const float* tgrid, const fsk_grid_desc* desc,
                    const float* x, int64_t n, float* t12, float* d, float* jac, void* stream);

/* init_states (correspondence.hpp:62-63; correspondence.cpp:58-70): for every (point, bone)
 * x0 [N][n_b][3] = B_i^-1 x' and jinv0 [N][n_b][9] = J(x0)^-1, or I when |det J| < 1e-8.
 * Either output may be NULL. float32. */
int fsk_init_states(fsk_ctx* ctx, const float* tgrid, const fsk_grid_desc* desc, const float* bones,
                    int32_t n_bones_pose, const float* points, int64_t n, float* x0, float* jinv0,
                    void* stream);

/* init_states in float64, in the reference's own operation order (the exact replay's start,
 * DESIGN §precision): x0 = B_i^-1 x' (geometry.hpp:51-61) and jinv0 = J(x0)^-1 or I, J from the
 * n_b-wide weight grid (deformer.cpp:117-136, correspondence.cpp:43-54) — bit-identical to the
 * oracle's init_states. weights [V][n_b] float32, bones float32, points [N][3] float64; outputs
 * float64 point-major [N][n_b][3] / [N][n_b][9], either may be NULL. All dev. */
int fsk_init_states64(fsk_ctx* ctx, const float* weights, const fsk_grid_desc* desc, const float* bones,
                      int32_t n_bones_pose, const double* points, int64_t n, double* x0, double* jinv0,
                      void* stream);

/* ---- K3: implicit-differentiation backward (diff.cpp:43-51, :336-359), grid-routed.
 * For each point p with root_sel[p] >= 0 (init index into the dense result), with
 * v = grad_xc[p] (dL/dx*), u = -J~^T v and x* = x_c[p][sel]:
 *    grad_tgrid[c] += phi_c(x*) * u (x*,1)^T        (3x4, 8 corners c of locate_cell(x*))
 * grad_tgrid [V][12] dev is OVERWRITTEN (zeroed first). deterministic != 0 selects the
 * bitwise-reproducible int64 fixed-point accumulation; 0 = float vector atomics. */
int fsk_search_bwd(fsk_ctx* ctx, const fsk_grid_desc* desc, const float* x_c, const float* jinv,
                   int32_t n_init, const float* grad_xc, const int32_t* root_sel, int64_t n,
                   float* grad_tgrid, int deterministic, void* stream);

/* Same backward from compact roots (fsk_batch_search / fsk_deform output): root_index [N]
 * int64 (dev) selects roots[root_index[p]] as x* / J~ of query p, or -1 for none. */
int fsk_search_bwd_roots(fsk_ctx* ctx, const fsk_grid_desc* desc, const fsk_root* roots,
                         const int64_t* root_index, const float* grad_xc, int64_t n,
                         float* grad_tgrid, int deterministic, void* stream);

/* ---- B2: implicit_grad_exact (diff.cpp:31-41; SingularRootError diff.hpp:20-22), grid-routed.
 * Per point p: J = deform_jacobian(x*_p, grid, bones) in float64 in the reference's operation order
 * (weight-grid form, deformer.cpp:117-136), det = Mat3::determinant; |det| < 1e-10 (or NaN) →
 * ok[p] = 0 and u = 0 (the reference throws SingularRootError; its callers skip the sample), else
 * u = −J⁻ᵀ v by partial-pivot LU of Jᵀ (:36, the sign of :39 folded in) and ok[p] = 1.
 * weights [V][n_b], bones, x_star [N][3] and grad_xc (v) [N][3] float32; u [N][3] float64; ok [N],
 * det [N] float64 (either may be NULL). All dev. */
int fsk_implicit_u_exact(fsk_ctx* ctx, const float* weights, const fsk_grid_desc* desc, const float* bones,
                         int32_t n_bones_pose, const float* x_star, const float* grad_xc, int64_t n, double* u,
                         uint8_t* ok, double* det, void* stream);

/* fsk_search_bwd_roots with the exact cotangent (fsk_implicit_u_exact) instead of −J~ᵀv: the
 * implicit_grad_exact form of the training backward. Singular roots contribute nothing (ok[p] = 0
 * when ok != NULL). grad_tgrid [V][12] overwritten. */
int fsk_search_bwd_exact_roots(fsk_ctx* ctx, const float* weights, const fsk_grid_desc* desc, const float* bones,
                               int32_t n_bones_pose, const fsk_root* roots, const int64_t* root_index,
                               const float* grad_xc, int64_t n, float* grad_tgrid, uint8_t* ok, int deterministic,
                               void* stream);

/* fsk_search_bwd_roots visiting the queries in `order` (int32 [N] dev, a permutation of [0, N), e.g. the
 * search's spatial order from fsk_ctx_query_order; NULL = query order). With a spatial order the fast
 * mode aggregates the contributions of consecutive roots that share a cell within each warp before its
 * vector reductions (k_bwd_scatter_agg); the deterministic mode is order-independent. */
int fsk_search_bwd_roots_ordered(fsk_ctx* ctx, const fsk_grid_desc* desc, const fsk_root* roots,
                                 const int64_t* root_index, const float* grad_xc, int64_t n, const int32_t* order,
                                 float* grad_tgrid, int deterministic, void* stream);

/* The spatial (Morton) order of the queries of the context's last device search (fsk_search_fwd,
 * fsk_batch_search, fsk_deform; N must be that search's point count): order[k] = index of the k-th query
 * in the order the search visited them. Stream-ordered copy into `order` (int32 [N] dev). */
int fsk_ctx_query_order(fsk_ctx* ctx, int64_t n, int32_t* order, void* stream);

/* ---- deterministic backward across devices or ranks. The deterministic mode rounds every term to int64
 * fixed point with a power-of-two scale from (max term, n): scale = 2^(61 - floor(log2(max·n))). With
 * the max over ALL shards and n = the total point count on every shard, the int64 sums of the shards add
 * up (ncclInt64 sum) to exactly the one-device sums, so the gradient is bitwise the same for any number
 * of devices. Per shard: fsk_search_bwd_max_term → all-reduce MAX of the float → fsk_search_bwd_fixed
 * (accumulates into acc, which the caller zeroes) → all-reduce SUM of acc → fsk_fixed_to_float.
 * Roots are given densely (x_c, jinv, root_sel, n_init as fsk_search_bwd) or compact (roots,
 * root_index as fsk_search_bwd_roots, when roots != NULL). */
typedef struct fsk_bwd_src {
    const float* x_c;
    const float* jinv;
    const int32_t* root_sel;
    int32_t n_init;
    const fsk_root* roots;
    const int64_t* root_index;
} fsk_bwd_src;
int fsk_search_bwd_max_term(fsk_ctx* ctx, const fsk_grid_desc* desc, const fsk_bwd_src* src, const float* grad_xc,
                            int64_t n, float* max_term /* dev, 1 float, overwritten */, void* stream);
int fsk_search_bwd_fixed(fsk_ctx* ctx, const fsk_grid_desc* desc, const fsk_bwd_src* src, const float* grad_xc,
                         int64_t n, int64_t n_scale, const float* max_term /* dev */, int64_t* acc /* dev [V][12] */,
                         void* stream);
int fsk_fixed_to_float(fsk_ctx* ctx, const int64_t* acc, int64_t m, int64_t n_scale, const float* max_term,
                       float* out, void* stream);

/* dL/dw[v][i] = <dL/dT[v], B_i>_F  (chain rule through deformer.cpp:70-74). [V][n_b] dev. */
int fsk_grad_weights(fsk_ctx* ctx, const fsk_grid_desc* desc, const float* grad_tgrid,
                     const float* bones, int32_t n_bones_pose, float* grad_w, void* stream);

/* ---- single-process multi-GPU: one context, stream and host thread per
 * device; points shard in contiguous ranges [n*r/R, n*(r+1)/R) (the parallel_for partition,
 * parallel.hpp:28-29); no collective on the forward; the backward sums dL/dT over the devices
 * with one NCCL all-reduce (ncclCommInitAll communicator, created on first use). */
typedef struct fsk_multi fsk_multi;
int fsk_multi_create(int32_t n_devices, const int32_t* devices, fsk_multi** out);
int fsk_multi_destroy(fsk_multi* m);
int32_t fsk_multi_device_count(const fsk_multi* m);

/* fsk_deform_host over all devices: HOST buffers in/out, results identical to the one-device
 * call (CorrespondenceSets in query order; offsets [N+1], roots [cap], *total_out). */
int fsk_multi_deform_host(fsk_multi* m, const float* weights, const fsk_grid_desc* desc, const float* bones,
                          int32_t n_bones_pose, const float* points, int64_t n, const fsk_search_opts* opts,
                          int64_t* offsets, fsk_root* roots, int64_t cap, int64_t* total_out);

/* Training-step backward over all devices from HOST buffers: root_index [N] selects
 * roots[root_index[p]] (or -1) as x*, J~ of query p; grad_xc [N][3] = dL/dx*. Each device runs
 * K3 on its query shard into dL/dT, NCCL sums dL/dT, device 0 contracts to grad_w [V][n_b]
 * (host). Equal to fsk_search_bwd_roots + fsk_grad_weights on one device up to the order of
 * the float sums (bitwise for one device). */
int fsk_multi_grad_weights_host(fsk_multi* m, const fsk_grid_desc* desc, const float* bones, int32_t n_bones_pose,
                                const fsk_root* roots, const int64_t* root_index, const float* grad_xc, int64_t n,
                                float* grad_w, int deterministic);

/* ---- wire and disk formats, host functions; errors in fsk_io_last_error().
 * SKNV grids (skinning.cpp:239-288), .bin points (pointio.cpp:43-62), correspondence dumps
 * (pointio.cpp:97-117, "%.17g" text, formatted by `threads` host threads, 0 = all cores). */
const char* fsk_io_last_error(void);
int fsk_sknv_read(const char* path, fsk_grid_desc* desc, float* weights /* [V][n_b] host, NULL = header */,
                  int64_t cap);
int fsk_sknv_write(const char* path, const fsk_grid_desc* desc, const float* weights);
int fsk_points_bin_read(const char* path, float* points /* [n][3] host, NULL = count */, int64_t cap,
                        int64_t* n_out);
int fsk_points_bin_write(const char* path, const float* points, int64_t n);
int fsk_write_correspondence_dump(const char* path, const float* queries, int64_t n, const int64_t* offsets,
                                  const fsk_root* roots, int32_t threads);
/* one cmd_deform frame from files to file (fskin_cli.cpp:395-429, correspondences only):
 * SKNV + .bin in, fsk_deform_host, dump out. */
int fsk_deform_files(fsk_ctx* ctx, const char* grid_path, const float* bones, int32_t n_bones,
                     const char* points_path, const fsk_search_opts* opts, const char* dump_path,
                     int64_t* n_queries, int64_t* n_roots);

/* ---- MLP-variant search (SearchVariant::Mlp): batch_search with
 * d(x) = lbs_blend(softmax(net(x)), B)·x (deformer.cpp:22-26, correspondence.cpp:77-79) and the
 * initial Jacobian from the network's input tangents (deform_jacobian(x, mlp, bones),
 * deformer.cpp:117-141). theta/widths as for fsk_distill (widths = {3, H.., n_b}); outputs as
 * fsk_search_fwd (dense per (point, init), dedup'd). Rounds of one batched network evaluation
 * (tcgen05, 3xTF32) + one Broyden step per active solve, float32 state; synchronizes `stream`
 * once per round. The ablation the paper's voxel search is measured against. */
int fsk_search_fwd_mlp(fsk_ctx* ctx, const float* theta, const int32_t* widths, int32_t n_widths,
                       const float* bones, int32_t n_bones_pose, const float* points, int64_t n,
                       const fsk_search_opts* opts, fsk_search_out* out, void* stream);

/* ---- MLP stages next to the search, tcgen05 tensor cores, 3xTF32 (FP32-faithful).
 * theta: the network's flat parameter vector in Mlp::parameters() order (mlp.cpp:207-219: per
 * layer W column-major [out x in], then b), float32, device. widths: host array {in, H, ..., out}
 * with every hidden width equal to H in {64, 128}; softplus hidden units, linear head
 * (Mlp::forward, mlp.cpp:115-138). */

/* distill (skinning.cpp:195-221): weights [V][n_b] (dev, float32) = softmax(net(vertex_position(v)))
 * over the grid of desc (vertex_position, skinning.cpp:77-80). widths = {3, H.., n_b}, n_b <= 64
 * and == desc->n_bones. Replaces fskin::distill(const SkinningMlp&, GridDims, const Aabb&). */
int fsk_distill(fsk_ctx* ctx, const float* theta, const int32_t* widths, int32_t n_widths,
                const fsk_grid_desc* desc, float* weights, void* stream);

/* VJP of distill (the chain the training step takes through the skinning network,
 * diff.cpp:348-359, with the grid vertices in place of the roots): given dL/dw [V][n_b] (dev,
 * e.g. fsk_grad_weights' output), writes dL/dtheta [P] (dev, Mlp::parameters() order) =
 * sum_v Mlp::backward(softmax_vjp(w_v, dL/dw_v)) (mlp.cpp:38-41, :140-163). FP32: the forward
 * is recomputed on the tensor cores (activations kept), the backward runs fused per 64-row
 * tile on the CUDA cores with per-CTA partial sums reduced in a fixed order (deterministic). */
int fsk_distill_bwd(fsk_ctx* ctx, const float* theta, const int32_t* widths, int32_t n_widths,
                    const fsk_grid_desc* desc, const float* grad_w, float* grad_theta, void* stream);

/* posed_occupancy_batch (shape.cpp:242-269) over CorrespondenceSets on the device: for query q,
 * pred[q] = max over roots r in [offsets[q], offsets[q+1]) of sigmoid(net(roots[r].x, pose))
 * (OccupancyMlp::occupancy_batch, shape.cpp:218-228) and argmax[q] = r - offsets[q] of the first
 * maximum, -1 (pred 0) for an empty set. widths = {3 + n_pose, H.., 1}. n_roots = offsets[n].
 * argmax and occ_per_root ([n_roots], per-root occupancy) may be NULL. All device buffers.
 * Replaces fskin::posed_occupancy_batch(std::span<const CorrespondenceSet>, const OccupancyMlp&,
 * const VectorXd&, std::vector<int>*). */
int fsk_posed_occupancy(fsk_ctx* ctx, const float* theta, const int32_t* widths, int32_t n_widths,
                        const float* pose, int32_t n_pose, const int64_t* offsets, const fsk_root* roots,
                        int64_t n, int64_t n_roots, float* pred, int32_t* argmax, float* occ_per_root,
                        void* stream);

#ifdef __cplusplus
}
#endif

#endif /* FSK_H_ */
