// fsk_bwd.cu — implicit-differentiation backward of the deformer on sm_100a (K3, GW).
//
// implicit_grad_approx (diff.cpp:43-51) and the training root-cotangent block
// (diff.cpp:336-359): with v = dL/dx* and the converged Broyden estimate J~ ≈ (∂d/∂x)^-1,
//   u = −J~ᵀ v                                        (diff.cpp:351)
// The reference pushes uw_i = u·(B_i x̃*) (:354-356) through the skinning MLP at x*. Here the
// skinning field is the voxel grid itself, so the cotangent is scattered to the grid:
//   dL/dT_c += φ_c(x*) · u (x*, 1)ᵀ        (3×4, the 8 corners of locate_cell(x*))
//   dL/dw_{c,i} = <dL/dT_c, B_i>_F          (k_grad_weights; T_c = Σ_i w_{c,i} B_i)
// Fast mode: float4 vector reductions (REDG.E.ADD.F32x4), warp-aggregated per cell when the roots come
// in spatial order. Deterministic mode: every term is rounded to int64 fixed point with a data-derived
// power-of-two scale and accumulated with integer reductions — associative, so bitwise reproducible for
// any order on one device; across devices or ranks when every shard uses the same scale (max term
// all-reduced, n = all points) and the int64 sums are all-reduced (fsk_search_bwd_fixed, fsk_multi,
// dist.py).
#include "fsk_ctx.h"
#include "fsk_exact.cuh"

namespace fsk {

struct RootRef {  // where the selected root of each query lives
    // dense form: x_c [N][n_init][3], jinv [N][n_init][9], sel [N] init index
    const float* x_c;
    const float* jinv;
    const int32_t* sel;
    int n_init;
    // compact form: roots [M], ridx [N] root index (int64) or -1
    const fsk_root* roots;
    const int64_t* ridx;
    // exact mode (implicit_grad_exact, diff.cpp:31-41): the cotangent u [N][3] was computed by
    // k_implicit_exact (u = −J⁻ᵀv from the Jacobian at x*) instead of −J~ᵀv; ok [N] = 0 marks a
    // singular root, skipped (SingularRootError: "caller skips this sample")
    const float* u_ex = nullptr;
    const uint8_t* ok = nullptr;
    // x*-only form (fsk_implicit_u_exact): x_star [N][3]
    const float* xs_direct = nullptr;
};

// x* of query p (false: no root selected)
__device__ __forceinline__ bool root_x(const RootRef& R, int64_t p, float xs[3], const float** J) {
    if (R.xs_direct) {
        xs[0] = R.xs_direct[3 * p];
        xs[1] = R.xs_direct[3 * p + 1];
        xs[2] = R.xs_direct[3 * p + 2];
        *J = nullptr;
        return true;
    }
    if (R.roots) {
        const int64_t k = R.ridx[p];
        if (k < 0) return false;
        const fsk_root& r = R.roots[k];
        xs[0] = r.x[0];
        xs[1] = r.x[1];
        xs[2] = r.x[2];
        *J = r.inv_jacobian;
        return true;
    }
    const int sidx = R.sel[p];
    if (sidx < 0 || sidx >= R.n_init) return false;
    const int64_t s = p * R.n_init + sidx;
    *J = R.jinv + 9 * s;
    xs[0] = R.x_c[3 * s];
    xs[1] = R.x_c[3 * s + 1];
    xs[2] = R.x_c[3 * s + 2];
    return true;
}

__device__ __forceinline__ bool bwd_load(const RootRef& R, int64_t p, const float* __restrict__ gx, float xs[3],
                                         float u[3]) {
    const float* J;
    if (!root_x(R, p, xs, &J)) return false;
    if (R.u_ex) {
        if (R.ok && !R.ok[p]) return false;
        u[0] = R.u_ex[3 * p];
        u[1] = R.u_ex[3 * p + 1];
        u[2] = R.u_ex[3 * p + 2];
        return true;
    }
    const float v0 = gx[3 * p], v1 = gx[3 * p + 1], v2 = gx[3 * p + 2];
    u[0] = -(J[0] * v0 + J[3] * v1 + J[6] * v2);
    u[1] = -(J[1] * v0 + J[4] * v1 + J[7] * v2);
    u[2] = -(J[2] * v0 + J[5] * v1 + J[8] * v2);
    return true;
}

// ---- implicit_grad_exact (diff.cpp:31-41), grid-routed: per selected root, J = deform_jacobian(x*,
// grid, bones) in float64 in the reference's operation order (deformer.cpp:117-136; fsk_exact.cuh),
// its determinant (Eigen's, row 0); |det| < 1e-10 → singular (ok = 0, SingularRootError, :34-35);
// else u = −J⁻ᵀv by partial-pivot LU of Jᵀ like `jac.transpose().partialPivLu().solve(v)` (:36,
// Eigen PartialPivLU: first largest |pivot| per column, row swap, column divided by the pivot,
// rank-1 trailing update; P·v, unit-lower then upper substitution, column oriented).
__device__ __forceinline__ void lu_solve_T(const double J[9], const double v[3], double x[3]) {
    using namespace exact;
    double m[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) m[i][j] = J[3 * j + i];
    int perm[3] = {0, 1, 2};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        int p = k;
        double big = fabs(m[k][k]);
#pragma unroll
        for (int i = k + 1; i < 3; ++i)
            if (fabs(m[i][k]) > big) {
                big = fabs(m[i][k]);
                p = i;
            }
        if (big != 0.0) {
            if (p != k) {
#pragma unroll
                for (int j = 0; j < 3; ++j) {
                    const double t = m[k][j];
                    m[k][j] = m[p][j];
                    m[p][j] = t;
                }
                const int t = perm[k];
                perm[k] = perm[p];
                perm[p] = t;
            }
#pragma unroll
            for (int i = k + 1; i < 3; ++i) m[i][k] = div(m[i][k], m[k][k]);
        }
#pragma unroll
        for (int i = k + 1; i < 3; ++i)
#pragma unroll
            for (int j = k + 1; j < 3; ++j) m[i][j] = madd(m[i][j], -m[i][k], m[k][j]);
    }
    double y[3] = {v[perm[0]], v[perm[1]], v[perm[2]]};
#pragma unroll
    for (int j = 0; j < 3; ++j)
#pragma unroll
        for (int i = j + 1; i < 3; ++i) y[i] = madd(y[i], -y[j], m[i][j]);
#pragma unroll
    for (int j = 2; j >= 0; --j) {
        y[j] = div(y[j], m[j][j]);
#pragma unroll
        for (int i = 0; i < j; ++i) y[i] = madd(y[i], -y[j], m[i][j]);
    }
    x[0] = y[0];
    x[1] = y[1];
    x[2] = y[2];
}

__global__ void __launch_bounds__(128) k_implicit_exact(GridP g, const float* __restrict__ W,
                                                        const float* __restrict__ bones, RootRef R,
                                                        const float* __restrict__ gx, int64_t n,
                                                        float* __restrict__ u32, double* __restrict__ u64,
                                                        uint8_t* __restrict__ ok, double* __restrict__ det_out) {
    extern __shared__ double s_b64[];  // float64 copies of the bones (widening is exact)
    for (int e = threadIdx.x; e < 12 * g.nb; e += blockDim.x) s_b64[e] = (double)__ldg(bones + e);
    __syncthreads();
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n) return;
    float xs[3];
    const float* Jt;
    double u[3] = {0.0, 0.0, 0.0}, det = 0.0;
    bool good = false;
    if (root_x(R, p, xs, &Jt)) {
        double J[9];
        exact::jacobian(g, W, s_b64, (double)xs[0], (double)xs[1], (double)xs[2], J);
        using namespace exact;
        auto X = [&](int c1, int c2) { return msub(J[3 + c1], J[6 + c2], J[3 + c2], J[6 + c1]); };
        det = madd(madd(mul(J[0], X(1, 2)), -J[1], X(0, 2)), J[2], X(0, 1));  // Mat3::determinant (diff.cpp:34)
        if (fabs(det) >= 1e-10) {  // (:35) NaN det: singular as well
            const double v[3] = {(double)gx[3 * p], (double)gx[3 * p + 1], (double)gx[3 * p + 2]};
            double x[3];
            lu_solve_T(J, v, x);
            u[0] = -x[0];  // acc.scale(-1.0) (:39)
            u[1] = -x[1];
            u[2] = -x[2];
            good = true;
        }
    }
    if (u32) {
        u32[3 * p] = (float)u[0];
        u32[3 * p + 1] = (float)u[1];
        u32[3 * p + 2] = (float)u[2];
    }
    if (u64) {
        u64[3 * p] = u[0];
        u64[3 * p + 1] = u[1];
        u64[3 * p + 2] = u[2];
    }
    if (ok) ok[p] = good ? 1 : 0;
    if (det_out) det_out[p] = det;
}

__global__ void k_zero(float4* __restrict__ p, int64_t n4) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = make_float4(0.f, 0.f, 0.f, 0.f);
}

__global__ void __launch_bounds__(256) k_bwd_scatter(GridP g, RootRef R, const float* __restrict__ gx, int64_t n,
                                                     float4* __restrict__ gT) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n) return;
    float xs[3], u[3];
    if (!bwd_load(R, p, gx, xs, u)) return;
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

// Fast mode over roots in spatial order (the search's query order, fsk_ctx_query_order): warp-aggregated
// reductions. Lane L of a warp loads the root of order[32w + L]; the warp then walks its roots in order
// (shuffle broadcast) while lane L < 24 owns output float4 L of the current cell (corner L/3, matrix row
// L%3: φ_c·u_r·(x*, 1)) and accumulates it in registers; at every change of cell the 24 partial sums go
// out as one vector reduction each. In spatial order consecutive roots mostly share a cell, so the L2
// sees one red per cell run instead of one per root.
__global__ void __launch_bounds__(256) k_bwd_scatter_agg(GridP g, RootRef R, const int32_t* __restrict__ order,
                                                         const float* __restrict__ gx, int64_t n,
                                                         float4* __restrict__ gT) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    if (j - lane >= n) return;  // whole warp past the end
    float xs[3] = {0.f, 0.f, 0.f}, u[3] = {0.f, 0.f, 0.f};
    Cell<float> c{};
    bool have = false;
    if (j < n) {
        have = bwd_load(R, order[j], gx, xs, u);
        if (have) c = locate<false>(g, xs[0], xs[1], xs[2]);
    }
    const int nxy = g.nx * g.ny;
    const int q = lane / 3, row = lane - 3 * q;
    const int di = q & 1, dj = (q >> 1) & 1, dk = q >> 2;
    const bool owner = lane < 24;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    int cur = -1;
    unsigned todo = __ballot_sync(0xffffffffu, have);
    auto flush = [&]() {
        if (cur >= 0 && owner) atomicAdd(gT + 3 * (int64_t)(cur + dk * nxy + dj * g.nx + di) + row, acc);
        acc = make_float4(0.f, 0.f, 0.f, 0.f);
    };
#ifndef FSK_K3_SHFL
    // the warp's 32 root records staged in shared memory: the walk reads each with three
    // broadcast LDS.128 instead of ten shuffles (C3 K3: fewer MIO instructions per root)
    __shared__ float4 s_rec[256 / 32][32][3];
    float4(&rec)[32][3] = s_rec[threadIdx.x >> 5];
    rec[lane][0] = make_float4(__int_as_float(c.base), c.tx, c.ty, c.tz);
    rec[lane][1] = make_float4(xs[0], xs[1], xs[2], u[0]);
    rec[lane][2] = make_float4(u[1], u[2], 0.f, 0.f);
    __syncwarp();
#endif
    while (todo) {
        const int src = __ffs(todo) - 1;
        todo &= todo - 1;
#ifndef FSK_K3_SHFL
        const float4 r0 = rec[src][0], r1 = rec[src][1], r2 = rec[src][2];
        const int cj = __float_as_int(r0.x);
        const float tx = r0.y, ty = r0.z, tz = r0.w, x0 = r1.x, x1 = r1.y, x2 = r1.z, u0 = r1.w, u1 = r2.x, u2 = r2.y;
        if (cj != cur) {  // warp-uniform
            flush();
            cur = cj;
        }
#else
        const int cj = __shfl_sync(0xffffffffu, c.base, src);
        if (cj != cur) {  // warp-uniform
            flush();
            cur = cj;
        }
        const float tx = __shfl_sync(0xffffffffu, c.tx, src), ty = __shfl_sync(0xffffffffu, c.ty, src),
                    tz = __shfl_sync(0xffffffffu, c.tz, src);
        const float x0 = __shfl_sync(0xffffffffu, xs[0], src), x1 = __shfl_sync(0xffffffffu, xs[1], src),
                    x2 = __shfl_sync(0xffffffffu, xs[2], src);
        const float u0 = __shfl_sync(0xffffffffu, u[0], src), u1 = __shfl_sync(0xffffffffu, u[1], src),
                    u2 = __shfl_sync(0xffffffffu, u[2], src);
#endif
        if (owner) {
            const float wz = dk ? tz : 1.f - tz;
            const float wyz = wz * (dj ? ty : 1.f - ty);
            const float phi = wyz * (di ? tx : 1.f - tx);  // k_bwd_scatter's corner weight
            const float a = phi * (row == 0 ? u0 : (row == 1 ? u1 : u2));
            acc.x += a * x0;
            acc.y += a * x1;
            acc.z += a * x2;
            acc.w += a;
        }
    }
    flush();
}

// Fixed-point scale of the deterministic mode: a power of two with n·max|term|·scale < 2^62,
// so no int64 sum over at most n roots can overflow; max|term| ≤ max|u|·max(1, |x*|).
__device__ __forceinline__ double fixed_scale(unsigned int maxbits, int64_t n) {
    const double m = (double)__uint_as_float(maxbits) * (double)(n > 0 ? n : 1);
    if (!(m > 0.0)) return 1.0;
    const int e = (int)floor(log2(m));
    return ldexp(1.0, 61 - e);
}

// ---- deterministic mode, gather formulation (no atomics on the gradient) ------------------
// 1. k_bwd_bucket_count: per root, its cell (the locate_cell base vertex) → count per cell;
//    also the fixed-point scale's max term.
// 2. exclusive scan of the counts → bucket starts.
// 3. k_bwd_bucket_fill: roots written into their cell's bucket as {x*, u} (order inside a
//    bucket is arbitrary — the sums below are integer and therefore order-independent).
// 4. k_bwd_chunk_reduce: per warp of 32 bucketed roots, per-cell runs of fixed-point terms
//    φ_c·u_r·x̃_col·scale summed in int64 registers and flushed with integer atomics.
//    Bitwise reproducible, identical to the scattered fixed-point sum.
struct BwdRec {
    float x[3];
    float u[3];
};

// Roots visited in `order` when given (the search's spatial order: neighbouring lanes mostly share a
// cell), else in index order; lanes of a warp in the same cell share one atomic (__match_any_sync).
__global__ void __launch_bounds__(256) k_bwd_bucket_count(GridP g, RootRef R, const float* __restrict__ gx, int64_t n,
                                                          const int32_t* __restrict__ order,
                                                          int32_t* __restrict__ cnt, int32_t* __restrict__ cell_of,
                                                          unsigned int* __restrict__ maxbits) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j - (threadIdx.x & 31) >= n) return;  // whole warp past the end
    float m = 0.f;
    int cell = -1;
    if (j < n) {
        const int64_t p = order ? order[j] : j;
        float xs[3], u[3];
        if (bwd_load(R, p, gx, xs, u)) {
            cell = locate<false>(g, xs[0], xs[1], xs[2]).base;
            const float mu = fmaxf(fabsf(u[0]), fmaxf(fabsf(u[1]), fabsf(u[2])));
            const float mx = fmaxf(1.f, fmaxf(fabsf(xs[0]), fmaxf(fabsf(xs[1]), fabsf(xs[2]))));
            m = mu * mx;
            if (!isfinite(m)) m = 3.0e38f;
        }
        cell_of[j] = cell;
    }
    const unsigned peers = __match_any_sync(0xffffffffu, cell);
    if (cell >= 0 && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(cnt + cell, __popc(peers));
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffff, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(maxbits, __float_as_uint(m));
}

__global__ void __launch_bounds__(256) k_bwd_max_term(RootRef R, const float* __restrict__ gx, int64_t n,
                                                      unsigned int* __restrict__ maxbits) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    float m = 0.f;
    if (p < n) {
        float xs[3], u[3];
        if (bwd_load(R, p, gx, xs, u)) {  // the max term of k_bwd_bucket_count
            const float mu = fmaxf(fabsf(u[0]), fmaxf(fabsf(u[1]), fabsf(u[2])));
            const float mx = fmaxf(1.f, fmaxf(fabsf(xs[0]), fmaxf(fabsf(xs[1]), fabsf(xs[2]))));
            m = mu * mx;
            if (!isfinite(m)) m = 3.0e38f;
        }
    }
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffff, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(maxbits, __float_as_uint(m));
}

__global__ void __launch_bounds__(256) k_bwd_bucket_fill(RootRef R, const float* __restrict__ gx, int64_t n,
                                                         const int32_t* __restrict__ order,
                                                         const int32_t* __restrict__ cell_of,
                                                         const int64_t* __restrict__ start, int32_t* __restrict__ fill,
                                                         BwdRec* __restrict__ rec) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    if (j - lane >= n) return;  // whole warp past the end
    const int cell = j < n ? cell_of[j] : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, cell);
    const int leader = __ffs(peers) - 1;
    int base = 0;
    if (cell >= 0 && lane == leader) base = atomicAdd(fill + cell, __popc(peers));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (cell < 0) return;
    float xs[3], u[3];
    bwd_load(R, order ? order[j] : j, gx, xs, u);
    const int64_t pos = start[cell] + base + __popc(peers & ((1u << lane) - 1));
    rec[pos] = BwdRec{{xs[0], xs[1], xs[2]}, {u[0], u[1], u[2]}};
}

// One warp per 32 consecutive bucketed roots (the buckets are contiguous and cell-ordered, so a
// warp's records form a few runs of equal cell): lane L loads record L into shared memory, then the
// warp walks the records in order (broadcast reads); lane L < 24 owns row L % 3 of corner L / 3 of
// the run's cell (four int64 sums) and flushes them to the corner vertex with integer atomics at each
// cell change. Dense cells are split across warps (no load imbalance); integer addition keeps the
// result bitwise order- and split-independent. (Round 1 gave each lane three of the 96 outputs: three
// products per record instead of one: C3 det 49.7 -> 29.0 us, bitwise the same sums.)
__global__ void __launch_bounds__(256) k_bwd_chunk_reduce(GridP g, const int64_t* __restrict__ start,
                                                          const BwdRec* __restrict__ rec,
                                                          const unsigned int* __restrict__ maxbits, int64_t n,
                                                          unsigned long long* __restrict__ acc) {
    // Lane L < 24 owns matrix row L % 3 of corner L / 3 of the run's cell — four int64 sums, one per
    // column of the 3x4 block, so one φ·u·scale product per record and lane serves four terms (the
    // terms themselves are k_bwd_fixed_agg's and the round-1 per-output form's, bit for bit).
    const int64_t V = (int64_t)g.nx * g.ny * g.nz;
    const int64_t M = start[V];  // bucketed roots
    const int lane = threadIdx.x & 31;
    const int64_t r0 = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * 32;
    if (r0 >= M) return;
    const int cnt = (int)(M - r0 < 32 ? M - r0 : 32);
    BwdRec b{};
    Cell<float> c{};
    int cell = -1;
    if (lane < cnt) {
        b = rec[r0 + lane];
        c = locate<false>(g, b.x[0], b.x[1], b.x[2]);
        cell = c.base;
    }
    const double scale = fixed_scale(*maxbits, n);
    const int nxy = g.nx * g.ny;
    const int q = lane / 3, row = lane - 3 * q;
    const int di = q & 1, dj = (q >> 1) & 1, dk = q >> 2;
    const bool owner = lane < 24;
    __shared__ float4 s_rec[256 / 32][32][3];
    float4(&rr)[32][3] = s_rec[threadIdx.x >> 5];
    rr[lane][0] = make_float4(__int_as_float(cell), c.tx, c.ty, c.tz);
    rr[lane][1] = make_float4(b.x[0], b.x[1], b.x[2], b.u[0]);
    rr[lane][2] = make_float4(b.u[1], b.u[2], 0.f, 0.f);
    __syncwarp();
    long long s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    auto flush = [&](int cl) {
        if (owner) {
            unsigned long long* d = acc + 12 * (int64_t)(cl + dk * nxy + dj * g.nx + di) + 4 * row;
            if (s0) atomicAdd(d, (unsigned long long)s0);
            if (s1) atomicAdd(d + 1, (unsigned long long)s1);
            if (s2) atomicAdd(d + 2, (unsigned long long)s2);
            if (s3) atomicAdd(d + 3, (unsigned long long)s3);
        }
        s0 = s1 = s2 = s3 = 0;
    };
    int cur = __float_as_int(rr[0][0].x);
    for (int j = 0; j < cnt; ++j) {
        const float4 a0 = rr[j][0], a1 = rr[j][1], a2 = rr[j][2];
        const int cj = __float_as_int(a0.x);
        if (cj != cur) {  // warp-uniform
            flush(cur);
            cur = cj;
        }
        if (owner) {
            const float tx = a0.y, ty = a0.z, tz = a0.w;
            const float ur = row == 0 ? a1.w : (row == 1 ? a2.x : a2.y);
            const float phi = ((dk ? tz : 1.f - tz) * (dj ? ty : 1.f - ty)) * (di ? tx : 1.f - tx);
            const double a = (double)phi * (double)ur * scale;
            s0 += __double2ll_rn(a * (double)a1.x);
            s1 += __double2ll_rn(a * (double)a1.y);
            s2 += __double2ll_rn(a * (double)a1.z);
            s3 += __double2ll_rn(a * 1.0);
        }
    }
    flush(cur);
}

// Deterministic mode over roots in spatial order (the search's query order): k_bwd_scatter_agg's
// walk with k_bwd_chunk_reduce's fixed-point terms — lane L < 24 owns float4 L (corner L/3, matrix
// row L%3) of the current cell as four int64 sums and flushes them with integer atomics at each
// cell change. Every term is computed exactly as in k_bwd_chunk_reduce and integer addition is
// order-free, so the result is bitwise the bucketed path's, without bucketing the roots by cell
// (count, scan, fill). Needs the max term (scale) first: k_bwd_max_term. Ablation (off by default).
#ifndef FSK_DET_ORDERED
#define FSK_DET_ORDERED 0  // measured slower on C3 det: 86 us for this kernel vs 86 us for count + fill + chunk reduce (four int64 atomics per lane per run, shorter runs than whole buckets)
#endif
__global__ void __launch_bounds__(256) k_bwd_fixed_agg(GridP g, RootRef R, const int32_t* __restrict__ order,
                                                       const float* __restrict__ gx, int64_t n,
                                                       const unsigned int* __restrict__ maxbits, int64_t n_scale,
                                                       unsigned long long* __restrict__ acc) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    if (j - lane >= n) return;  // whole warp past the end
    float xs[3] = {0.f, 0.f, 0.f}, u[3] = {0.f, 0.f, 0.f};
    Cell<float> c{};
    bool have = false;
    if (j < n) {
        have = bwd_load(R, order[j], gx, xs, u);
        if (have) c = locate<false>(g, xs[0], xs[1], xs[2]);
    }
    const double scale = fixed_scale(*maxbits, n_scale);
    const int nxy = g.nx * g.ny;
    const int q = lane / 3, row = lane - 3 * q;
    const int di = q & 1, dj = (q >> 1) & 1, dk = q >> 2;
    const bool owner = lane < 24;
    long long s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    int cur = -1;
    unsigned todo = __ballot_sync(0xffffffffu, have);
    __shared__ float4 s_rec[256 / 32][32][3];
    float4(&rec)[32][3] = s_rec[threadIdx.x >> 5];
    rec[lane][0] = make_float4(__int_as_float(c.base), c.tx, c.ty, c.tz);
    rec[lane][1] = make_float4(xs[0], xs[1], xs[2], u[0]);
    rec[lane][2] = make_float4(u[1], u[2], 0.f, 0.f);
    __syncwarp();
    auto flush = [&]() {
        if (cur >= 0 && owner) {
            unsigned long long* d = acc + 12 * (int64_t)(cur + dk * nxy + dj * g.nx + di) + 4 * row;
            if (s0) atomicAdd(d, (unsigned long long)s0);
            if (s1) atomicAdd(d + 1, (unsigned long long)s1);
            if (s2) atomicAdd(d + 2, (unsigned long long)s2);
            if (s3) atomicAdd(d + 3, (unsigned long long)s3);
        }
        s0 = s1 = s2 = s3 = 0;
    };
    while (todo) {
        const int src = __ffs(todo) - 1;
        todo &= todo - 1;
        const float4 r0 = rec[src][0], r1 = rec[src][1], r2 = rec[src][2];
        const int cj = __float_as_int(r0.x);
        if (cj != cur) {  // warp-uniform
            flush();
            cur = cj;
        }
        if (owner) {
            const float tx = r0.y, ty = r0.z, tz = r0.w;
            const float ur = row == 0 ? r1.w : (row == 1 ? r2.x : r2.y);
            // k_bwd_chunk_reduce's term, entry (row, col): φ·u_row·scale·(x_col or 1)
            const float phi = ((dk ? tz : 1.f - tz) * (dj ? ty : 1.f - ty)) * (di ? tx : 1.f - tx);
            const double a = (double)phi * (double)ur * scale;
            s0 += __double2ll_rn(a * (double)r1.x);
            s1 += __double2ll_rn(a * (double)r1.y);
            s2 += __double2ll_rn(a * (double)r1.z);
            s3 += __double2ll_rn(a * 1.0);
        }
    }
    flush();
}

__global__ void k_bwd_fixed_to_float(const long long* __restrict__ acc, int64_t m,
                                     const unsigned int* __restrict__ maxbits, int64_t n, float* __restrict__ out) {
    const double inv = 1.0 / fixed_scale(*maxbits, n);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (float)((double)acc[i] * inv);
}


// dL/dw[v][i] = Σ_e dL/dT[v][e]·B_i[e]. Tile of 128 vertices staged in shared memory so the
// [V][n_b] store is coalesced. HBM-bound: V·(48 + 4·n_b) bytes.
constexpr int kGwTile = 128;
__global__ void __launch_bounds__(kGwTile) k_grad_weights(const float* __restrict__ gT, const float* __restrict__ bones,
                                                          int nb, int64_t V, float* __restrict__ gw) {
    extern __shared__ float sm[];
    float* sB = sm;            // nb*12
    float* sO = sm + nb * 12;  // kGwTile*nb
    for (int e = threadIdx.x; e < nb * 12; e += blockDim.x) sB[e] = bones[e];
    __syncthreads();
    const int64_t v0 = blockIdx.x * (int64_t)kGwTile;
    const int64_t v = v0 + threadIdx.x;
    if (v < V) {
        const float4* src = reinterpret_cast<const float4*>(gT) + 3 * v;
        const float4 a = src[0], b = src[1], c = src[2];
        const float G[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, c.x, c.y, c.z, c.w};
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

// The same, one thread per (vertex, bone) element — consecutive threads write consecutive gw entries,
// a vertex's 48-B gradient row is an L1 broadcast to its n_b threads; the same 12-term FMA chain as
// k_grad_weights (bitwise equal), with ~n_b x the parallelism of one thread per vertex.
#ifndef FSK_GW_PER_ELEMENT
#define FSK_GW_PER_ELEMENT 0  // measured equal on C3 (9.7 us both): kept as an ablation
#endif
__global__ void __launch_bounds__(256) k_grad_weights_e(const float* __restrict__ gT, const float* __restrict__ bones,
                                                        int nb, int64_t V, float* __restrict__ gw) {
    extern __shared__ float sB[];
    for (int e = threadIdx.x; e < nb * 12; e += blockDim.x) sB[e] = bones[e];
    __syncthreads();
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= V * nb) return;
    const int64_t v = t / nb;
    const int i = (int)(t - v * nb);
    const float4* src = reinterpret_cast<const float4*>(gT) + 3 * v;
    const float4 a = __ldg(src), b = __ldg(src + 1), c = __ldg(src + 2);
    const float G[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, c.x, c.y, c.z, c.w};
    float s = 0.f;
#pragma unroll
    for (int e = 0; e < 12; ++e) s = fmaf(G[e], sB[i * 12 + e], s);
    gw[t] = s;
}

namespace {

// Deterministic accumulation: zero, bucket the roots by cell (per-warp max term into this call's own
// max slot), scan, fill, reduce into int64 fixed point. The scale comes from (max term, n_scale):
// this call's max and n unless `max_ext` (a float on the device, e.g. the max over all devices or
// ranks) is given, and the sums go into `acc_ext` ([V][12] int64, accumulated into) when given, else
// into the context's zeroed scratch (returned). Integer sums: any split of the roots over devices,
// with the same (max, n_scale), adds up to the same bits.
unsigned long long* det_accumulate(fsk_ctx* ctx, const GridP& g, const RootRef& R, const float* grad_xc, int64_t n,
                                   int64_t n_scale, const float* max_ext, long long* acc_ext, cudaStream_t st,
                                   unsigned int** mx_out, const int32_t* order = nullptr) {
    const int64_t V = (int64_t)g.nx * g.ny * g.nz;
    const unsigned cap_blocks = (unsigned)ctx->sm_count * 8;
    const int64_t V4 = (V + 3) / 4 * 4;  // fixed-point accumulators, counts, fill cursors: zeroed together
    const int64_t words = 2 * (12 * V4) + 2 * V4 + 8;  // int32 words
    int32_t* base = (int32_t*)scratch(ctx, kBwdAcc, words * sizeof(int32_t));
    unsigned long long* acc = acc_ext ? reinterpret_cast<unsigned long long*>(acc_ext)
                                      : reinterpret_cast<unsigned long long*>(base);
    int32_t* cnt = base + 2 * (12 * V4);
    int32_t* fill = cnt + V4;
    unsigned int* mx = (unsigned int*)(fill + V4);
    int64_t* start = (int64_t*)scratch(ctx, kBwdStart, (V + 1) * sizeof(int64_t));
    int32_t* cell_of = (int32_t*)scratch(ctx, kBwdCell, std::max<int64_t>(1, n) * sizeof(int32_t));
    BwdRec* rec = (BwdRec*)scratch(ctx, kBwdRec, std::max<int64_t>(1, n) * sizeof(BwdRec));
    FSK_LAUNCH(ctx, st, k_zero, std::min(blocks_for(words / 4, 256), cap_blocks), 256, 0,
               reinterpret_cast<float4*>(base), words / 4);
    if (n > 0)
        FSK_LAUNCH(ctx, st, k_bwd_bucket_count, blocks_for(n, 256), 256, 0, g, R, grad_xc, n, order, cnt, cell_of, mx);
    scan_i32_to_i64(ctx, cnt, V, start, st);
    const unsigned int* mscale = max_ext ? reinterpret_cast<const unsigned int*>(max_ext) : mx;
    if (n > 0) {
        FSK_LAUNCH(ctx, st, k_bwd_bucket_fill, blocks_for(n, 256), 256, 0, R, grad_xc, n, order, cell_of, start, fill,
                   rec);
        FSK_LAUNCH(ctx, st, k_bwd_chunk_reduce, blocks_for(n, 256), 256, 0, g, start, rec, mscale, n_scale, acc);
    }
    if (mx_out) *mx_out = mx;
    return acc;
}

void run_bwd(fsk_ctx* ctx, const GridP& g, const RootRef& R, const float* grad_xc, int64_t n, float* grad_tgrid,
             int deterministic, cudaStream_t st, const int32_t* order = nullptr) {
    const int64_t V = (int64_t)g.nx * g.ny * g.nz;
    const unsigned cap_blocks = (unsigned)ctx->sm_count * 8;
    if (!deterministic) {
        FSK_LAUNCH(ctx, st, k_zero, std::min(blocks_for(V * 3, 256), cap_blocks), 256, 0,
                   reinterpret_cast<float4*>(grad_tgrid), V * 3);
        if (n > 0 && order)
            FSK_LAUNCH(ctx, st, k_bwd_scatter_agg, blocks_for(n, 256), 256, 0, g, R, order, grad_xc, n,
                       reinterpret_cast<float4*>(grad_tgrid));
        else if (n > 0)
            FSK_LAUNCH(ctx, st, k_bwd_scatter, blocks_for(n, 256), 256, 0, g, R, grad_xc, n,
                       reinterpret_cast<float4*>(grad_tgrid));
        return;
    }
    unsigned int* mx = nullptr;
    unsigned long long* acc = nullptr;
    if (FSK_DET_ORDERED && order) {  // deterministic, spatial order: max term, then per-run integer sums
        const int64_t V4 = (V + 3) / 4 * 4;
        const int64_t words = 2 * (12 * V4) + 8;  // int64 accumulators + the max slot, zeroed together
        int32_t* base = (int32_t*)scratch(ctx, kBwdAcc, words * sizeof(int32_t));
        acc = reinterpret_cast<unsigned long long*>(base);
        mx = (unsigned int*)(base + 2 * (12 * V4));
        FSK_LAUNCH(ctx, st, k_zero, std::min(blocks_for(words / 4, 256), cap_blocks), 256, 0,
                   reinterpret_cast<float4*>(base), words / 4);
        if (n > 0) {
            FSK_LAUNCH(ctx, st, k_bwd_max_term, blocks_for(n, 256), 256, 0, R, grad_xc, n, mx);
            FSK_LAUNCH(ctx, st, k_bwd_fixed_agg, blocks_for(n, 256), 256, 0, g, R, order, grad_xc, n, mx, n, acc);
        }
    } else {  // deterministic: bucket the roots by cell, reduce per cell, integer atomics to vertices
        acc = det_accumulate(ctx, g, R, grad_xc, n, n, nullptr, nullptr, st, &mx, order);
    }
    FSK_LAUNCH(ctx, st, k_bwd_fixed_to_float, std::min(blocks_for(12 * V, 256), cap_blocks), 256, 0,
               reinterpret_cast<const long long*>(acc), 12 * V, mx, n, grad_tgrid);
}

}  // namespace
}  // namespace fsk

using namespace fsk;

extern "C" {

int fsk_search_bwd(fsk_ctx* ctx, const fsk_grid_desc* desc, const float* x_c, const float* jinv, int32_t n_init,
                   const float* grad_xc, const int32_t* root_sel, int64_t n, float* grad_tgrid, int deterministic,
                   void* stream) {
    return guard([&] {
        set_device(ctx);
        const GridP g = make_grid(desc);
        if (n < 0) fail(FSK_EINVAL, "fsk: negative point count");
        if (n_init < 1) fail(FSK_EINVAL, "fsk: n_init must be >= 1");
        if (!grad_tgrid || (n > 0 && (!x_c || !jinv || !grad_xc || !root_sel))) fail(FSK_EINVAL, "fsk: null buffer");
        RootRef R{x_c, jinv, root_sel, n_init, nullptr, nullptr};
        run_bwd(ctx, g, R, grad_xc, n, grad_tgrid, deterministic, (cudaStream_t)stream);
    });
}

int fsk_search_bwd_roots(fsk_ctx* ctx, const fsk_grid_desc* desc, const fsk_root* roots, const int64_t* root_index,
                         const float* grad_xc, int64_t n, float* grad_tgrid, int deterministic, void* stream) {
    return fsk_search_bwd_roots_ordered(ctx, desc, roots, root_index, grad_xc, n, nullptr, grad_tgrid, deterministic,
                                        stream);
}

int fsk_search_bwd_roots_ordered(fsk_ctx* ctx, const fsk_grid_desc* desc, const fsk_root* roots,
                                 const int64_t* root_index, const float* grad_xc, int64_t n, const int32_t* order,
                                 float* grad_tgrid, int deterministic, void* stream) {
    return guard([&] {
        set_device(ctx);
        const GridP g = make_grid(desc);
        if (n < 0) fail(FSK_EINVAL, "fsk: negative point count");
        if (!grad_tgrid || (n > 0 && (!roots || !root_index || !grad_xc))) fail(FSK_EINVAL, "fsk: null buffer");
        RootRef R{nullptr, nullptr, nullptr, 0, roots, root_index};
        run_bwd(ctx, g, R, grad_xc, n, grad_tgrid, deterministic, (cudaStream_t)stream, order);
    });
}

int fsk_implicit_u_exact(fsk_ctx* ctx, const float* weights, const fsk_grid_desc* desc, const float* bones,
                         int32_t n_bones_pose, const float* x_star, const float* grad_xc, int64_t n, double* u,
                         uint8_t* ok, double* det, void* stream) {
    return guard([&] {
        set_device(ctx);
        const GridP g = make_grid(desc);
        if (n_bones_pose != g.nb) fail(FSK_EINVAL, "deform vjp: bone count mismatch");
        if (n < 0) fail(FSK_EINVAL, "fsk: negative point count");
        if (n == 0) return;
        if (!weights || !bones || !x_star || !grad_xc) fail(FSK_EINVAL, "fsk: null buffer");
        RootRef R{nullptr, nullptr, nullptr, 0, nullptr, nullptr};
        R.xs_direct = x_star;
        FSK_LAUNCH(ctx, (cudaStream_t)stream, k_implicit_exact, blocks_for(n, 128), 128,
                   (size_t)g.nb * 12 * sizeof(double), g, weights, bones, R, grad_xc, n, nullptr, u, ok, det);
    });
}

int fsk_search_bwd_exact_roots(fsk_ctx* ctx, const float* weights, const fsk_grid_desc* desc, const float* bones,
                               int32_t n_bones_pose, const fsk_root* roots, const int64_t* root_index,
                               const float* grad_xc, int64_t n, float* grad_tgrid, uint8_t* ok, int deterministic,
                               void* stream) {
    return guard([&] {
        set_device(ctx);
        const GridP g = make_grid(desc);
        if (n_bones_pose != g.nb) fail(FSK_EINVAL, "deform vjp: bone count mismatch");
        if (n < 0) fail(FSK_EINVAL, "fsk: negative point count");
        if (!grad_tgrid || !weights || !bones || (n > 0 && (!roots || !root_index || !grad_xc)))
            fail(FSK_EINVAL, "fsk: null buffer");
        cudaStream_t st = (cudaStream_t)stream;
        RootRef R{nullptr, nullptr, nullptr, 0, roots, root_index};
        float* u = (float*)scratch(ctx, kBwdU, std::max<int64_t>(1, n) * 3 * sizeof(float));
        uint8_t* okp = ok ? ok : (uint8_t*)scratch(ctx, kBwdOk, std::max<int64_t>(1, n));
        if (n > 0)
            FSK_LAUNCH(ctx, st, k_implicit_exact, blocks_for(n, 128), 128, (size_t)g.nb * 12 * sizeof(double), g,
                       weights, bones, R, grad_xc, n, u, nullptr, okp, nullptr);
        R.u_ex = u;
        R.ok = okp;
        run_bwd(ctx, g, R, grad_xc, n, grad_tgrid, deterministic, st);
    });
}

namespace {
RootRef ref_of(const fsk_bwd_src* src) {
    if (!src) fail(FSK_EINVAL, "fsk: null buffer");
    if (src->roots) return RootRef{nullptr, nullptr, nullptr, 0, src->roots, src->root_index};
    if (src->n_init < 1) fail(FSK_EINVAL, "fsk: n_init must be >= 1");
    return RootRef{src->x_c, src->jinv, src->root_sel, src->n_init, nullptr, nullptr};
}
bool src_ok(const fsk_bwd_src* s) { return s->roots ? s->root_index != nullptr : (s->x_c && s->jinv && s->root_sel); }
}  // namespace

int fsk_search_bwd_max_term(fsk_ctx* ctx, const fsk_grid_desc* desc, const fsk_bwd_src* src, const float* grad_xc,
                            int64_t n, float* max_term, void* stream) {
    return guard([&] {
        set_device(ctx);
        make_grid(desc);
        if (n < 0) fail(FSK_EINVAL, "fsk: negative point count");
        const RootRef R = ref_of(src);
        if (!max_term || (n > 0 && (!grad_xc || !src_ok(src)))) fail(FSK_EINVAL, "fsk: null buffer");
        cudaStream_t st = (cudaStream_t)stream;
        cuda_check(cudaMemsetAsync(max_term, 0, sizeof(float), st), "cudaMemsetAsync");
        if (n > 0)
            FSK_LAUNCH(ctx, st, k_bwd_max_term, blocks_for(n, 256), 256, 0, R, grad_xc, n,
                       reinterpret_cast<unsigned int*>(max_term));
    });
}

int fsk_search_bwd_fixed(fsk_ctx* ctx, const fsk_grid_desc* desc, const fsk_bwd_src* src, const float* grad_xc,
                         int64_t n, int64_t n_scale, const float* max_term, int64_t* acc, void* stream) {
    return guard([&] {
        set_device(ctx);
        const GridP g = make_grid(desc);
        if (n < 0 || n_scale < n) fail(FSK_EINVAL, "fsk: need 0 <= n <= n_scale");
        const RootRef R = ref_of(src);
        if (!max_term || !acc || (n > 0 && (!grad_xc || !src_ok(src)))) fail(FSK_EINVAL, "fsk: null buffer");
        det_accumulate(ctx, g, R, grad_xc, n, n_scale, max_term, reinterpret_cast<long long*>(acc),
                       (cudaStream_t)stream, nullptr);
    });
}

int fsk_fixed_to_float(fsk_ctx* ctx, const int64_t* acc, int64_t m, int64_t n_scale, const float* max_term, float* out,
                       void* stream) {
    return guard([&] {
        set_device(ctx);
        if (m < 0) fail(FSK_EINVAL, "fsk: negative count");
        if (m > 0 && (!acc || !max_term || !out)) fail(FSK_EINVAL, "fsk: null buffer");
        if (m > 0)
            FSK_LAUNCH(ctx, (cudaStream_t)stream, k_bwd_fixed_to_float,
                       std::min(blocks_for(m, 256), (unsigned)ctx->sm_count * 8), 256, 0,
                       reinterpret_cast<const long long*>(acc), m, reinterpret_cast<const unsigned int*>(max_term),
                       n_scale, out);
    });
}

int fsk_grad_weights(fsk_ctx* ctx, const fsk_grid_desc* desc, const float* grad_tgrid, const float* bones,
                     int32_t n_bones_pose, float* grad_w, void* stream) {
    return guard([&] {
        set_device(ctx);
        const GridP g = make_grid(desc);
        if (n_bones_pose != g.nb) fail(FSK_EINVAL, "precompute_transform_grid: bone count mismatch");
        if (!grad_tgrid || !bones || !grad_w) fail(FSK_EINVAL, "fsk: null buffer");
        const int64_t V = (int64_t)g.nx * g.ny * g.nz;
        const size_t smem = (size_t)(g.nb * 12 + kGwTile * g.nb) * sizeof(float);
        if (smem > 200 * 1024) fail(FSK_EINVAL, "fsk: too many bones for grad_weights");
        if (smem > 48 * 1024)
            cuda_check(cudaFuncSetAttribute(k_grad_weights, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                       "cudaFuncSetAttribute");
        cudaStream_t st = (cudaStream_t)stream;
        if (FSK_GW_PER_ELEMENT) {
            FSK_LAUNCH(ctx, st, k_grad_weights_e, blocks_for(V * g.nb, 256), 256, g.nb * 12 * sizeof(float), grad_tgrid,
                       bones, g.nb, V, grad_w);
            return;
        }
        FSK_LAUNCH(ctx, st, k_grad_weights, blocks_for(V, kGwTile), kGwTile, smem, grad_tgrid, bones, g.nb, V, grad_w);
    });
}

}  // extern "C"
