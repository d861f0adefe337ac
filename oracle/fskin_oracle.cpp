// ORACLE — TEST INFRASTRUCTURE ONLY. Not part of the product.
//
// Double-precision, Eigen-free CPU restatement of the Fast-SNARF hot path of the
// reference (`/root/reference/proj`). Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / `--impl reference` leg may load this library, and
// only as the checker / CPU baseline — never as the thing measured or shipped.
//
// Parity status: the reference itself cannot be built in this container
// (`proj/CMakeLists.txt:16` requires Eigen3, absent on disk; `vendor/` json/CLI11
// are git-ignored), and the reference ships no tests or golden vectors
// (`proj/tests/CMakeLists.txt` is empty). This restatement is therefore pinned
// only by the SPEC.md known-answer examples and acceptance criteria, transcribed
// in tests/test_oracle_kat.py — "parity unpinned" against reference outputs.
//
// Every function cites the reference lines it restates. Operation order follows
// the reference where it matters numerically (cell lookup, trilerp accumulation
// order, Broyden update). The cost structure is kept: the initial Jacobian goes
// through the n_b-wide weight grid exactly like deformer.cpp:117-136, not the
// cheaper 12-wide transform-grid form the CUDA kernel uses.
//
// Eigen specifics mirrored: 3×3 determinant/inverse are closed-form cofactors,
// norm() = sqrt of the sum of squares.

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace orc {

// ---------------------------------------------------------------- tiny linear algebra
// Operation order. The reference is built with -march=native under CMake's default -std=gnu++20
// (proj/CMakeLists.txt:3-14): GCC contracts `a*b + c` into FMA (-ffp-contract=fast is the GNU-mode
// default) and Eigen's products accumulate with pmadd, so the reference binary on any FMA-capable
// host computes with fused multiply-adds. The default restatement states one such contraction
// explicitly and compiler-independently (std::fma): every addition (or subtraction) whose right
// operand is a product is one FMA —
//   acc + a·b -> fma(a, b, acc);  a0b0 + a1b1 + a2b2 -> fma(a2, b2, fma(a1, b1, a0·b0));
//   a·b − c·d -> fma(−c, d, a·b).
// Builds of other plausible operation orders (oracle/Makefile; Eigen unpinned):
//   ORC_UNFUSED — no contraction (each product rounded; the round-1 oracle), with
//     ORC_INV_ROW0 — inverse()'s determinant along row 0,  ORC_SUM_PAIR — 3-term sums as a+(b+c)
//     (Eigen's unvectorized redux unroller), or GCC's own -ffp-contract=fast on the unfused source.
#if defined(ORC_UNFUSED)
static inline double madd(double acc, double a, double b) { return acc + a * b; }
static inline double msub(double a, double b, double c, double d) { return a * b - c * d; }
#else
static inline double madd(double acc, double a, double b) { return std::fma(a, b, acc); }
static inline double msub(double a, double b, double c, double d) { return std::fma(-c, d, a * b); }
#endif
// a0·b0 + a1·b1 + a2·b2 (Eigen's 3-term redux: mat-vec coefficients, dot, squaredNorm)
static inline double dot3(double a0, double b0, double a1, double b1, double a2, double b2) {
#if defined(ORC_SUM_PAIR)
    return a0 * b0 + (a1 * b1 + a2 * b2);
#else
    return madd(madd(a0 * b0, a1, b1), a2, b2);
#endif
}
struct V3 {
    double v[3] = {0, 0, 0};
    double& operator[](int i) { return v[i]; }
    double operator[](int i) const { return v[i]; }
};
struct M3 {
    double m[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    static M3 identity() {
        M3 r;
        r.m[0][0] = r.m[1][1] = r.m[2][2] = 1.0;
        return r;
    }
};
static inline V3 mul(const M3& a, const V3& x) {
    V3 r;
    for (int i = 0; i < 3; ++i) r[i] = dot3(a.m[i][0], x[0], a.m[i][1], x[1], a.m[i][2], x[2]);
    return r;
}
static inline double dot(const V3& a, const V3& b) { return dot3(a[0], b[0], a[1], b[1], a[2], b[2]); }
static inline double norm(const V3& a) { return std::sqrt(dot(a, a)); }

// Eigen's closed-form 3×3 determinant (Determinant.h: expansion along the first row),
// h(0,1,2) − h(1,0,2) + h(2,0,1) with h(c0,c1,c2) = a0c0·(a1c1·a2c2 − a1c2·a2c1).
static inline double det3(const M3& a) {
    auto X = [&](int c1, int c2) { return msub(a.m[1][c1], a.m[2][c2], a.m[1][c2], a.m[2][c1]); };
    return madd(madd(a.m[0][0] * X(1, 2), -a.m[0][1], X(0, 2)), a.m[0][2], X(0, 1));
}
// Eigen's 3×3 inverse (InverseImpl.h compute_inverse<.., 3>): the cofactors of column 0, their
// determinant (cofactors_col0 · col(0), a 3-term redux), 1/det, then every cofactor times 1/det.
// ORC_INV_ROW0 (variant "invrow0", the round-1 oracle) takes that determinant along row 0.
static inline M3 inv3(const M3& a) {
    M3 c;
    c.m[0][0] = msub(a.m[1][1], a.m[2][2], a.m[1][2], a.m[2][1]);
    c.m[0][1] = msub(a.m[0][2], a.m[2][1], a.m[0][1], a.m[2][2]);
    c.m[0][2] = msub(a.m[0][1], a.m[1][2], a.m[0][2], a.m[1][1]);
    c.m[1][0] = msub(a.m[1][2], a.m[2][0], a.m[1][0], a.m[2][2]);
    c.m[1][1] = msub(a.m[0][0], a.m[2][2], a.m[0][2], a.m[2][0]);
    c.m[1][2] = msub(a.m[0][2], a.m[1][0], a.m[0][0], a.m[1][2]);
    c.m[2][0] = msub(a.m[1][0], a.m[2][1], a.m[1][1], a.m[2][0]);
    c.m[2][1] = msub(a.m[0][1], a.m[2][0], a.m[0][0], a.m[2][1]);
    c.m[2][2] = msub(a.m[0][0], a.m[1][1], a.m[0][1], a.m[1][0]);
#ifdef ORC_INV_ROW0
    const double det = dot3(a.m[0][0], c.m[0][0], a.m[0][1], c.m[1][0], a.m[0][2], c.m[2][0]);
#else
    const double det = dot3(c.m[0][0], a.m[0][0], c.m[0][1], a.m[1][0], c.m[0][2], a.m[2][0]);
#endif
    const double inv = 1.0 / det;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) c.m[i][j] *= inv;
    return c;
}

// Jᵀu = v by Eigen's PartialPivLU (PartialPivLU.h unblocked_lu: per column k the first largest |.|
// below the diagonal is the pivot, rows swapped, the column below divided by the pivot, rank-1
// update of the trailing block; then P·v, unit-lower forward and upper back substitution, column
// oriented) — `jac.transpose().partialPivLu().solve(cotangent)` (diff.cpp:36).
static inline V3 lu_solve_transposed(const M3& J, const V3& v) {
    double m[3][3];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) m[i][j] = J.m[j][i];
    int perm[3] = {0, 1, 2};
    for (int k = 0; k < 3; ++k) {
        int p = k;
        double big = std::abs(m[k][k]);
        for (int i = k + 1; i < 3; ++i)
            if (std::abs(m[i][k]) > big) {
                big = std::abs(m[i][k]);
                p = i;
            }
        if (big != 0.0) {
            if (p != k) {
                for (int j = 0; j < 3; ++j) std::swap(m[k][j], m[p][j]);
                std::swap(perm[k], perm[p]);
            }
            for (int i = k + 1; i < 3; ++i) m[i][k] /= m[k][k];
        }
        for (int i = k + 1; i < 3; ++i)
            for (int j = k + 1; j < 3; ++j) m[i][j] = madd(m[i][j], -m[i][k], m[k][j]);
    }
    double x[3] = {v[perm[0]], v[perm[1]], v[perm[2]]};
    for (int j = 0; j < 3; ++j)  // unit lower
        for (int i = j + 1; i < 3; ++i) x[i] = madd(x[i], -x[j], m[i][j]);
    for (int j = 2; j >= 0; --j) {  // upper
        x[j] /= m[j][j];
        for (int i = 0; i < j; ++i) x[i] = madd(x[i], -x[j], m[i][j]);
    }
    return V3{{x[0], x[1], x[2]}};
}

// Rigid transform [R | t] stored as 12 doubles row-major (geometry.hpp:42-78).
struct Rigid {
    M3 r;
    V3 t;
    V3 apply(const V3& x) const {  // geometry.hpp:51
        V3 y = mul(r, x);
        for (int i = 0; i < 3; ++i) y[i] += t[i];
        return y;
    }
    Rigid inverse() const {  // geometry.hpp:58-61: [Rᵀ | −(Rᵀt)]
        Rigid o;
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) o.r.m[i][j] = r.m[j][i];
        V3 rt = mul(o.r, t);
        for (int i = 0; i < 3; ++i) o.t[i] = -rt[i];
        return o;
    }
};
static inline Rigid rigid_from12(const double* b) {
    Rigid o;
    for (int i = 0; i < 3; ++i) {
        for (int j = 0; j < 3; ++j) o.r.m[i][j] = b[i * 4 + j];
        o.t[i] = b[i * 4 + 3];
    }
    return o;
}

// ---------------------------------------------------------------- grid description
struct Grid {
    int nx = 0, ny = 0, nz = 0, nb = 0;
    double lo[3] = {0, 0, 0}, hi[3] = {1, 1, 1};
    const double* w = nullptr;  // [V][nb], x-fastest, bone innermost (skinning.hpp:54-77)
    int64_t vertex_count() const { return int64_t(nx) * ny * nz; }
    int64_t vidx(int i, int j, int k) const { return (int64_t(k) * ny + j) * nx + i; }  // skinning.hpp:69-71
    V3 cell_size() const {  // skinning.cpp:72-75
        return V3{{(hi[0] - lo[0]) / (nx - 1), (hi[1] - lo[1]) / (ny - 1), (hi[2] - lo[2]) / (nz - 1)}};
    }
};

struct Cell {
    int i0, j0, k0;
    double tx, ty, tz;
};

// locate_cell (skinning.cpp:104-120) and locate_cell_lower (:122-139).
// The reference casts floor(NaN) to int (UB); NaN lookups are pinned to cell 0
// here, which the CUDA kernel does as well (its float→int conversion of NaN is 0).
static Cell locate(const Grid& g, const V3& x, bool lower) {
    Cell c;
    const int n[3] = {g.nx, g.ny, g.nz};
    int idx[3];
    double t[3];
    for (int a = 0; a < 3; ++a) {
        // Aabb::clamp = cwiseMax(min).cwiseMin(max) (geometry.hpp:28-30)
        double p = x[a];
        p = (p < g.lo[a]) ? g.lo[a] : p;
        p = (p > g.hi[a]) ? g.hi[a] : p;
        const double ext = g.hi[a] - g.lo[a];
        const double u = (p - g.lo[a]) / ext * (n[a] - 1);
        int i = (u == u) ? static_cast<int>(std::floor(u)) : 0;
        if (lower && i >= 1 && u == static_cast<double>(i)) i -= 1;
        if (i < 0) i = 0;
        if (i > n[a] - 2) i = n[a] - 2;
        idx[a] = i;
        t[a] = std::clamp(u - i, 0.0, 1.0);
    }
    c.i0 = idx[0]; c.j0 = idx[1]; c.k0 = idx[2];
    c.tx = t[0]; c.ty = t[1]; c.tz = t[2];
    return c;
}

// trilerp_weights_into (skinning.cpp:141-156)
static void trilerp_weights_into(const Grid& g, const V3& x, double* out) {
    const Cell c = locate(g, x, false);
    for (int b = 0; b < g.nb; ++b) out[b] = 0.0;
    for (int dk = 0; dk < 2; ++dk) {
        const double wz = dk ? c.tz : 1.0 - c.tz;
        for (int dj = 0; dj < 2; ++dj) {
            const double wyz = wz * (dj ? c.ty : 1.0 - c.ty);
            for (int di = 0; di < 2; ++di) {
                const double w = wyz * (di ? c.tx : 1.0 - c.tx);
                const double* v = g.w + g.vidx(c.i0 + di, c.j0 + dj, c.k0 + dk) * g.nb;
                for (int b = 0; b < g.nb; ++b) out[b] = madd(out[b], w, v[b]);
            }
        }
    }
}

// weight_spatial_gradient (skinning.cpp:164-193): out is nb×3 row-major.
static void weight_spatial_gradient(const Grid& g, const V3& x, double* out) {
    const Cell c = locate(g, x, true);
    const V3 h = g.cell_size();
    for (int e = 0; e < g.nb * 3; ++e) out[e] = 0.0;
    const double fx[2] = {1.0 - c.tx, c.tx};
    const double fy[2] = {1.0 - c.ty, c.ty};
    const double fz[2] = {1.0 - c.tz, c.tz};
    const double dx[2] = {-1.0 / h[0], 1.0 / h[0]};
    const double dy[2] = {-1.0 / h[1], 1.0 / h[1]};
    const double dz[2] = {-1.0 / h[2], 1.0 / h[2]};
    for (int dk = 0; dk < 2; ++dk)
        for (int dj = 0; dj < 2; ++dj)
            for (int di = 0; di < 2; ++di) {
                const double* v = g.w + g.vidx(c.i0 + di, c.j0 + dj, c.k0 + dk) * g.nb;
                const double gx = dx[di] * fy[dj] * fz[dk];
                const double gy = fx[di] * dy[dj] * fz[dk];
                const double gz = fx[di] * fy[dj] * dz[dk];
                for (int b = 0; b < g.nb; ++b) {
                    out[b * 3 + 0] = madd(out[b * 3 + 0], gx, v[b]);
                    out[b * 3 + 1] = madd(out[b * 3 + 1], gy, v[b]);
                    out[b * 3 + 2] = madd(out[b * 3 + 2], gz, v[b]);
                }
            }
}

// lbs_blend (deformer.cpp:9-19): Σᵢ wᵢ·[Rᵢ|tᵢ], 12 entries row-major.
static void lbs_blend(const double* w, const std::vector<Rigid>& bones, double* out12) {
    for (int e = 0; e < 12; ++e) out12[e] = 0.0;
    for (size_t i = 0; i < bones.size(); ++i) {
        for (int r = 0; r < 3; ++r) {
            for (int c = 0; c < 3; ++c) out12[r * 4 + c] = madd(out12[r * 4 + c], w[i], bones[i].r.m[r][c]);
            out12[r * 4 + 3] = madd(out12[r * 4 + 3], w[i], bones[i].t[r]);
        }
    }
}

// parallel_for (parallel.hpp:17-33): static contiguous partition.
template <typename Fn>
static void parallel_for(int64_t n, int workers, Fn&& fn) {
    if (n <= 0) return;
    if (workers < 1) workers = 1;
    if (workers == 1 || n < 2 * workers) {
        fn(int64_t(0), n);
        return;
    }
    std::vector<std::thread> pool;
    pool.reserve(workers);
    for (int w = 0; w < workers; ++w) {
        const int64_t begin = n * w / workers;
        const int64_t end = n * (w + 1) / workers;
        pool.emplace_back([&fn, begin, end] { fn(begin, end); });
    }
    for (auto& t : pool) t.join();
}

// trilerp_transform_into (deformer.cpp:79-94)
static void trilerp_transform_into(const Grid& g, const double* tgrid, const V3& x, double* out12) {
    const Cell c = locate(g, x, false);
    for (int e = 0; e < 12; ++e) out12[e] = 0.0;
    for (int dk = 0; dk < 2; ++dk) {
        const double wz = dk ? c.tz : 1.0 - c.tz;
        for (int dj = 0; dj < 2; ++dj) {
            const double wyz = wz * (dj ? c.ty : 1.0 - c.ty);
            for (int di = 0; di < 2; ++di) {
                const double w = wyz * (di ? c.tx : 1.0 - c.tx);
                const double* m = tgrid + g.vidx(c.i0 + di, c.j0 + dj, c.k0 + dk) * 12;
                for (int e = 0; e < 12; ++e) out12[e] = madd(out12[e], w, m[e]);
            }
        }
    }
}

// forward_deform(x, tgrid) (deformer.cpp:107-113) == eval_deform voxel branch
// (correspondence.cpp:75-85): T(clamp(x)) applied to the UNCLAMPED x.
static V3 forward_deform_tgrid(const Grid& g, const double* tgrid, const V3& x) {
    double m[12];
    trilerp_transform_into(g, tgrid, x, m);
    return V3{{dot3(m[0], x[0], m[1], x[1], m[2], x[2]) + m[3], dot3(m[4], x[0], m[5], x[1], m[6], x[2]) + m[7],
               dot3(m[8], x[0], m[9], x[1], m[10], x[2]) + m[11]}};
}

// deform_jacobian(x, grid, bones) (deformer.cpp:117-136) via jacobian_from_weights:
// J = Σᵢ wᵢ Rᵢ + Σᵢ (Bᵢ x) ∇wᵢᵀ, weights from locate_cell, gradient from locate_cell_lower.
static M3 deform_jacobian(const Grid& g, const std::vector<Rigid>& bones, const V3& x,
                          std::vector<double>& wbuf, std::vector<double>& gbuf) {
    trilerp_weights_into(g, x, wbuf.data());
    weight_spatial_gradient(g, x, gbuf.data());
    M3 jac;
    for (size_t i = 0; i < bones.size(); ++i)
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) jac.m[r][c] = madd(jac.m[r][c], wbuf[i], bones[i].r.m[r][c]);
    for (size_t i = 0; i < bones.size(); ++i) {
        const V3 bx = bones[i].apply(x);
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) jac.m[r][c] = madd(jac.m[r][c], bx[r], gbuf[i * 3 + c]);
    }
    return jac;
}

// initial_inverse_jacobian (correspondence.cpp:43-54)
static M3 initial_inverse_jacobian(const Grid& g, const std::vector<Rigid>& bones, const V3& x0,
                                   std::vector<double>& wbuf, std::vector<double>& gbuf) {
    const M3 jac = deform_jacobian(g, bones, x0, wbuf, gbuf);
    const double det = det3(jac);
    if (std::abs(det) < 1e-8) return M3::identity();
    return inv3(jac);
}

struct Opts {
    int max_iters;
    double conv_eps, div_eps, dedup_dist;
};

struct State {
    V3 x;
    M3 inv_jac;
    V3 g;
    int iterations = 0;
    bool converged = false;
};

// iterate (correspondence.cpp:97-124): good-Broyden with divergence check at the top.
static void iterate(State& st, const V3& xp, const Grid& g, const double* tgrid, const Opts& o) {
    double err = norm(st.g);
    if (err < o.conv_eps) {
        st.converged = true;
        return;
    }
    for (int k = 0; k < o.max_iters; ++k) {
        if (err > o.div_eps) return;
        V3 dx = mul(st.inv_jac, st.g);
        for (int i = 0; i < 3; ++i) dx[i] = -dx[i];
        for (int i = 0; i < 3; ++i) st.x[i] += dx[i];
        V3 gn = forward_deform_tgrid(g, tgrid, st.x);
        for (int i = 0; i < 3; ++i) gn[i] -= xp[i];
        V3 dg;
        for (int i = 0; i < 3; ++i) dg[i] = gn[i] - st.g[i];
        st.g = gn;
        st.iterations = k + 1;
        err = norm(st.g);
        if (err < o.conv_eps) {
            st.converged = true;
            return;
        }
        const V3 jdg = mul(st.inv_jac, dg);
        const double denom = dot(dx, jdg);
        if (std::abs(denom) > 1e-18) {
            V3 r;
            for (int i = 0; i < 3; ++i) r[i] = (dx[i] - jdg[i]) / denom;
            V3 wrow;  // dxᵀ J̃
            for (int c = 0; c < 3; ++c)
                wrow[c] = dot3(dx[0], st.inv_jac.m[0][c], dx[1], st.inv_jac.m[1][c], dx[2], st.inv_jac.m[2][c]);
            for (int i = 0; i < 3; ++i)
                for (int c = 0; c < 3; ++c) st.inv_jac.m[i][c] = madd(st.inv_jac.m[i][c], r[i], wrow[c]);
        }
    }
}

// dedup_roots (correspondence.cpp:162-176): greedy in input order, strict '<'.
static void dedup(const double* xs, const uint8_t* valid, int m, double dist, uint8_t* keep) {
    std::vector<int> kept;
    kept.reserve(m);
    for (int r = 0; r < m; ++r) {
        keep[r] = 0;
        if (valid && !valid[r]) continue;
        bool dup = false;
        for (int k : kept) {
            V3 d{{xs[r * 3 + 0] - xs[k * 3 + 0], xs[r * 3 + 1] - xs[k * 3 + 1], xs[r * 3 + 2] - xs[k * 3 + 2]}};
            if (norm(d) < dist) {
                dup = true;
                break;
            }
        }
        if (!dup) {
            kept.push_back(r);
            keep[r] = 1;
        }
    }
}

thread_local std::string g_err;

static Grid make_grid(const double* w, int nx, int ny, int nz, int nb, const double* bbox6) {
    // SkinningVoxelGrid ctor checks (skinning.cpp:60-70)
    if (nx < 2 || ny < 2 || nz < 2) throw std::invalid_argument("SkinningVoxelGrid: dims must be >= 2 per axis");
    if (nb < 1) throw std::invalid_argument("SkinningVoxelGrid: n_bones must be >= 1");
    Grid g;
    g.nx = nx; g.ny = ny; g.nz = nz; g.nb = nb; g.w = w;
    for (int a = 0; a < 3; ++a) {
        g.lo[a] = bbox6[a];
        g.hi[a] = bbox6[3 + a];
        if (!(g.hi[a] - g.lo[a] > 0.0)) throw std::invalid_argument("SkinningVoxelGrid: bbox must have positive extent");
    }
    return g;
}

static std::vector<Rigid> make_bones(const double* b, int n) {
    std::vector<Rigid> out(n);
    for (int i = 0; i < n; ++i) out[i] = rigid_from12(b + 12 * i);
    return out;
}

static void validate_opts(const Opts& o) {  // correspondence.cpp:19-25
    if (o.max_iters < 1) throw std::invalid_argument("search: max_iters must be >= 1");
    if (!(o.conv_eps > 0.0)) throw std::invalid_argument("search: conv_eps must be > 0");
    if (!(o.div_eps > o.conv_eps)) throw std::invalid_argument("search: div_eps must exceed conv_eps");
    if (!(o.dedup_dist >= 0.0)) throw std::invalid_argument("search: dedup_dist must be >= 0");
}

template <typename Fn>
static int guard(Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

}  // namespace orc

using namespace orc;

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }

// precompute_transform_grid (deformer.cpp:61-77)
int orc_precompute_tgrid(const double* w, int nx, int ny, int nz, int nb, const double* bbox6,
                         const double* bones, int n_bones, double* tgrid, int workers) {
    return guard([&] {
        Grid g = make_grid(w, nx, ny, nz, nb, bbox6);
        if (n_bones != nb) throw std::invalid_argument("precompute_transform_grid: bone count mismatch");
        const auto B = make_bones(bones, n_bones);
        parallel_for(g.vertex_count(), workers, [&](int64_t b0, int64_t b1) {
            for (int64_t v = b0; v < b1; ++v) lbs_blend(w + v * nb, B, tgrid + v * 12);
        });
    });
}

int orc_lbs_blend(const double* w, const double* bones, int n_bones, int n_weights, double* out12) {
    return guard([&] {
        if (n_weights != n_bones) throw std::invalid_argument("lbs_blend: weight/bone count mismatch");
        lbs_blend(w, make_bones(bones, n_bones), out12);
    });
}

// Batched point evaluators (skinning.cpp:141-193, deformer.cpp:79-136). Any output may be null.
int orc_eval_points(const double* w, int nx, int ny, int nz, int nb, const double* bbox6, const double* bones,
                    const double* tgrid, const double* x, int64_t n, double* weights_out, double* wgrad_out,
                    double* t12_out, double* d_tgrid_out, double* d_grid_out, double* jac_out) {
    return guard([&] {
        Grid g = make_grid(w, nx, ny, nz, nb, bbox6);
        const auto B = make_bones(bones, nb);
        std::vector<double> wb(nb), gb(nb * 3);
        for (int64_t p = 0; p < n; ++p) {
            const V3 xp{{x[3 * p], x[3 * p + 1], x[3 * p + 2]}};
            if (weights_out) trilerp_weights_into(g, xp, weights_out + p * nb);
            if (wgrad_out) weight_spatial_gradient(g, xp, wgrad_out + p * nb * 3);
            if (t12_out) trilerp_transform_into(g, tgrid, xp, t12_out + p * 12);
            if (d_tgrid_out) {
                const V3 d = forward_deform_tgrid(g, tgrid, xp);
                for (int i = 0; i < 3; ++i) d_tgrid_out[3 * p + i] = d[i];
            }
            if (d_grid_out) {  // forward_deform(x, grid, bones) (deformer.cpp:27-31)
                trilerp_weights_into(g, xp, wb.data());
                double m[12];
                lbs_blend(wb.data(), B, m);
                for (int r = 0; r < 3; ++r)
                    d_grid_out[3 * p + r] = dot3(m[r * 4], xp[0], m[r * 4 + 1], xp[1], m[r * 4 + 2], xp[2]) + m[r * 4 + 3];
            }
            if (jac_out) {
                const M3 j = deform_jacobian(g, B, xp, wb, gb);
                for (int r = 0; r < 3; ++r)
                    for (int c = 0; c < 3; ++c) jac_out[9 * p + 3 * r + c] = j.m[r][c];
            }
        }
    });
}

// init_states (correspondence.cpp:58-70): x0 [n][nb][3], jinv0 [n][nb][9].
int orc_init_states(const double* w, int nx, int ny, int nz, int nb, const double* bbox6, const double* bones,
                    int n_bones, const double* x_prime, int64_t n, double* x0, double* jinv0) {
    return guard([&] {
        if (n_bones < 1) throw std::invalid_argument("search: no bone transforms");
        if (n_bones != nb) throw std::invalid_argument("search: grid bone count mismatch");
        Grid g = make_grid(w, nx, ny, nz, nb, bbox6);
        const auto B = make_bones(bones, n_bones);
        std::vector<double> wb(nb), gb(nb * 3);
        for (int64_t p = 0; p < n; ++p) {
            const V3 xp{{x_prime[3 * p], x_prime[3 * p + 1], x_prime[3 * p + 2]}};
            for (int i = 0; i < nb; ++i) {
                const V3 x = B[i].inverse().apply(xp);
                const M3 J = initial_inverse_jacobian(g, B, x, wb, gb);
                for (int a = 0; a < 3; ++a) x0[(p * nb + i) * 3 + a] = x[a];
                for (int r = 0; r < 3; ++r)
                    for (int c = 0; c < 3; ++c) jinv0[(p * nb + i) * 9 + 3 * r + c] = J.m[r][c];
            }
        }
    });
}

// batch_search (correspondence.cpp:178-192) → search_one (:126-150) per query, with the
// per-(point, init) state exposed BEFORE filtering: x_c [n][nb][3], jinv [n][nb][9],
// resid [n][nb], iters [n][nb], converged [n][nb]; keep [n][nb] = dedup_roots result
// over the converged inits in bone order. Output pointers other than x_c/converged may be null.
int orc_batch_search(const double* w, int nx, int ny, int nz, int nb, const double* bbox6, const double* tgrid,
                     const double* bones, int n_bones, const double* x_prime, int64_t n, int max_iters,
                     double conv_eps, double div_eps, double dedup_dist, int workers, double* x_c, double* jinv,
                     double* resid, int32_t* iters, uint8_t* converged, uint8_t* keep) {
    return guard([&] {
        if (n_bones < 1) throw std::invalid_argument("search: no bone transforms");
        if (w == nullptr || tgrid == nullptr)
            throw std::invalid_argument("search: voxel variant needs skinning and transform grids");
        if (n_bones != nb) throw std::invalid_argument("search: grid bone count mismatch");
        const Opts o{max_iters, conv_eps, div_eps, dedup_dist};
        validate_opts(o);
        Grid g = make_grid(w, nx, ny, nz, nb, bbox6);
        const auto B = make_bones(bones, n_bones);
        parallel_for(n, workers, [&](int64_t b0, int64_t b1) {
            std::vector<double> wb(nb), gb(nb * 3), xs(nb * 3);
            std::vector<uint8_t> conv(nb), kp(nb);
            for (int64_t p = b0; p < b1; ++p) {
                const V3 xp{{x_prime[3 * p], x_prime[3 * p + 1], x_prime[3 * p + 2]}};
                for (int i = 0; i < nb; ++i) {
                    State st;
                    st.x = B[i].inverse().apply(xp);  // :135, recomputed per init as the reference does
                    st.inv_jac = initial_inverse_jacobian(g, B, st.x, wb, gb);
                    st.g = forward_deform_tgrid(g, tgrid, st.x);
                    for (int a = 0; a < 3; ++a) st.g[a] -= xp[a];
                    iterate(st, xp, g, tgrid, o);
                    const int64_t s = p * nb + i;
                    for (int a = 0; a < 3; ++a) {
                        x_c[s * 3 + a] = st.x[a];
                        xs[i * 3 + a] = st.x[a];
                    }
                    if (jinv)
                        for (int r = 0; r < 3; ++r)
                            for (int c = 0; c < 3; ++c) jinv[s * 9 + 3 * r + c] = st.inv_jac.m[r][c];
                    if (resid) resid[s] = norm(st.g);
                    if (iters) iters[s] = st.iterations;
                    converged[s] = st.converged ? 1 : 0;
                    conv[i] = converged[s];
                }
                dedup(xs.data(), conv.data(), nb, dedup_dist, kp.data());
                if (keep)
                    for (int i = 0; i < nb; ++i) keep[p * nb + i] = kp[i];
            }
        });
    });
}

// dedup_roots (correspondence.cpp:162-176) over m roots xs[m][3].
// Which operation-order variant this build is (oracle/Makefile): "fma" (default), "unfused",
// "invrow0", "pairsum", "gccfma".
const char* orc_variant(void) {
#if defined(ORC_VARIANT_NAME)
    return ORC_VARIANT_NAME;
#else
    return "fma";
#endif
}

int orc_dedup_roots(const double* xs, int m, double dedup_dist, uint8_t* keep) {
    return guard([&] { dedup(xs, nullptr, m, dedup_dist, keep); });
}

// Grid-routed implicit-differentiation VJP. Restates the math of implicit_grad_approx
// (diff.cpp:43-51) and the training root-cotangent block (diff.cpp:336-359):
// u = −J̃ᵀ v; the reference then forms uw_i = u·(B_i x̃*) (:354-356) and pushes it into the
// MLP at x*. Here the skinning weights are the grid itself, so
//   ∂L/∂w_{c,i} += φ_c(x*) · u·(B_i x̃*)          (grad_w, [V][nb])
//   ∂L/∂T_c     += φ_c(x*) · u x̃*ᵀ  (3×4)        (grad_T, [V][12])
// with φ_c the trilinear weights of locate_cell(x*) (skinning.cpp:141-156).
// Roots with sel[p] < 0 contribute nothing. jinv [n][9], x_star [n][3], v [n][3].
int orc_grid_vjp(int nx, int ny, int nz, int nb, const double* bbox6, const double* bones, const double* x_star,
                 const double* jinv, const double* v, const int32_t* sel, int64_t n, double* grad_T,
                 double* grad_w) {
    return guard([&] {
        std::vector<double> dummy(1);
        Grid g = make_grid(dummy.data(), nx, ny, nz, nb, bbox6);
        const auto B = make_bones(bones, nb);
        const int64_t V = g.vertex_count();
        if (grad_T) std::fill(grad_T, grad_T + V * 12, 0.0);
        if (grad_w) std::fill(grad_w, grad_w + V * nb, 0.0);
        for (int64_t p = 0; p < n; ++p) {
            if (sel && sel[p] < 0) continue;
            const V3 xs{{x_star[3 * p], x_star[3 * p + 1], x_star[3 * p + 2]}};
            M3 J;
            for (int r = 0; r < 3; ++r)
                for (int c = 0; c < 3; ++c) J.m[r][c] = jinv[9 * p + 3 * r + c];
            V3 u;  // u = −J̃ᵀ v (diff.cpp:351)
            for (int c = 0; c < 3; ++c)
                u[c] = -dot3(J.m[0][c], v[3 * p], J.m[1][c], v[3 * p + 1], J.m[2][c], v[3 * p + 2]);
            std::vector<double> uw(nb);
            for (int i = 0; i < nb; ++i) uw[i] = dot(u, B[i].apply(xs));  // diff.cpp:354-356
            const Cell c = locate(g, xs, false);
            for (int dk = 0; dk < 2; ++dk) {
                const double wz = dk ? c.tz : 1.0 - c.tz;
                for (int dj = 0; dj < 2; ++dj) {
                    const double wyz = wz * (dj ? c.ty : 1.0 - c.ty);
                    for (int di = 0; di < 2; ++di) {
                        const double phi = wyz * (di ? c.tx : 1.0 - c.tx);
                        const int64_t vi = g.vidx(c.i0 + di, c.j0 + dj, c.k0 + dk);
                        if (grad_T)
                            for (int r = 0; r < 3; ++r) {
                                for (int col = 0; col < 3; ++col)
                                    grad_T[vi * 12 + r * 4 + col] = madd(grad_T[vi * 12 + r * 4 + col], phi * u[r], xs[col]);
                                grad_T[vi * 12 + r * 4 + 3] = madd(grad_T[vi * 12 + r * 4 + 3], phi, u[r]);
                            }
                        if (grad_w)
                            for (int i = 0; i < nb; ++i) grad_w[vi * nb + i] = madd(grad_w[vi * nb + i], phi, uw[i]);
                    }
                }
            }
        }
    });
}

// Exact implicit cotangent (implicit_grad_exact, diff.cpp:31-41) on the grid field:
// u = −J⁻ᵀ v with J = deform_jacobian(x*, grid, B) solved by partial-pivot LU of Jᵀ (:36);
// ok[p]=0 if |det J| < 1e-10 (SingularRootError, :34-35).
int orc_implicit_u_exact(const double* w, int nx, int ny, int nz, int nb, const double* bbox6,
                         const double* bones, const double* x_star, const double* v, int64_t n, double* u_out,
                         uint8_t* ok) {
    return guard([&] {
        Grid g = make_grid(w, nx, ny, nz, nb, bbox6);
        const auto B = make_bones(bones, nb);
        std::vector<double> wb(nb), gb(nb * 3);
        for (int64_t p = 0; p < n; ++p) {
            const V3 xs{{x_star[3 * p], x_star[3 * p + 1], x_star[3 * p + 2]}};
            const M3 J = deform_jacobian(g, B, xs, wb, gb);
            const double det = det3(J);
            if (std::abs(det) < 1e-10) {
                ok[p] = 0;
                for (int a = 0; a < 3; ++a) u_out[3 * p + a] = 0.0;
                continue;
            }
            ok[p] = 1;
            const V3 u = lu_solve_transposed(J, V3{{v[3 * p], v[3 * p + 1], v[3 * p + 2]}});  // diff.cpp:36
            for (int c = 0; c < 3; ++c) u_out[3 * p + c] = -u[c];  // acc.scale(-1.0) (diff.cpp:39)
        }
    });
}

}  // extern "C"
