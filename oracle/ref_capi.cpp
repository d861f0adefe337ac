// ORACLE — TEST INFRASTRUCTURE ONLY (oracle/_ref). A C entry point over the REFERENCE'S OWN hot-path
// sources (/root/reference/proj/src/{geometry,skinning,deformer,correspondence}.cpp, compiled unmodified
// by oracle/ref_build.sh against the minimal Eigen stand-in oracle/eigen_shim): precompute_transform_grid
// → batch_search → CorrespondenceSets exactly as the reference computes them, and init_states. Used by
// tests/ as a second checker and by bench.py's --impl reference / cpu_baseline ("kind": "reference").
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "fskin/correspondence.hpp"
#include "fskin/deformer.hpp"

using namespace fskin;

namespace {
thread_local std::string g_err;

template <typename Fn>
int guard(Fn&& fn) {
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

SkinningVoxelGrid make_grid(const double* w, int nx, int ny, int nz, int nb, const double* bb) {
    SkinningVoxelGrid g(GridDims{nx, ny, nz}, Aabb{Vec3(bb[0], bb[1], bb[2]), Vec3(bb[3], bb[4], bb[5])}, nb);
    std::memcpy(g.raw().data(), w, g.raw().size() * sizeof(double));
    return g;
}

std::vector<RigidTransform> make_bones(const double* b, int nb) {
    std::vector<RigidTransform> out(nb);
    for (int i = 0; i < nb; ++i)
        for (int r = 0; r < 3; ++r) {
            for (int c = 0; c < 3; ++c) out[i].rotation(r, c) = b[12 * i + 4 * r + c];
            out[i].translation(r) = b[12 * i + 4 * r + 3];
        }
    return out;
}
}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_precompute_tgrid(const double* w, int nx, int ny, int nz, int nb, const double* bbox6, const double* bones,
                         int workers, double* tgrid) {
    return guard([&] {
        const SkinningVoxelGrid g = make_grid(w, nx, ny, nz, nb, bbox6);
        const auto B = make_bones(bones, nb);
        const TransformGrid tg = precompute_transform_grid(g, B, workers);
        std::memcpy(tgrid, tg.vertex_transform(0), g.dims().vertex_count() * 12 * sizeof(double));
    });
}

// batch_search (correspondence.cpp:178-192) through the reference's own code: CorrespondenceSets as
// offsets [n+1] + per-root x [3], residual, J~ [9], source_bone, iterations (capacity cap).
int ref_batch_search(const double* w, int nx, int ny, int nz, int nb, const double* bbox6, const double* bones,
                     const double* pts, int64_t n, int max_iters, double conv_eps, double div_eps, double dedup_dist,
                     int workers, int64_t* offsets, double* rx, double* rres, double* rjinv, int32_t* rbone,
                     int32_t* riters, int64_t cap, int64_t* total) {
    return guard([&] {
        const SkinningVoxelGrid g = make_grid(w, nx, ny, nz, nb, bbox6);
        const auto B = make_bones(bones, nb);
        const TransformGrid tg = precompute_transform_grid(g, B, workers);
        std::vector<Vec3> q(static_cast<size_t>(n));
        for (int64_t p = 0; p < n; ++p) q[p] = Vec3(pts[3 * p], pts[3 * p + 1], pts[3 * p + 2]);
        SearchContext ctx;
        ctx.bones = B;
        ctx.grid = &g;
        ctx.tgrid = &tg;
        SearchOptions o;
        o.max_iters = max_iters;
        o.conv_eps = conv_eps;
        o.div_eps = div_eps;
        o.dedup_dist = dedup_dist;
        const std::vector<CorrespondenceSet> sets = batch_search(q, ctx, o, workers);
        int64_t k = 0;
        for (int64_t p = 0; p < n; ++p) {
            offsets[p] = k;
            for (const Root& r : sets[p].roots) {
                if (k < cap) {
                    for (int a = 0; a < 3; ++a) rx[3 * k + a] = r.x(a);
                    rres[k] = r.residual;
                    for (int a = 0; a < 3; ++a)
                        for (int e = 0; e < 3; ++e) rjinv[9 * k + 3 * a + e] = r.inv_jacobian(a, e);
                    rbone[k] = r.source_bone;
                    riters[k] = r.iterations;
                }
                ++k;
            }
        }
        offsets[n] = k;
        *total = k;
        if (k > cap) throw std::invalid_argument("ref: root buffer too small");
    });
}

// init_states (correspondence.cpp:58-70): x0 [n][nb][3], jinv0 [n][nb][9]
int ref_init_states(const double* w, int nx, int ny, int nz, int nb, const double* bbox6, const double* bones,
                    const double* pts, int64_t n, double* x0, double* jinv0) {
    return guard([&] {
        const SkinningVoxelGrid g = make_grid(w, nx, ny, nz, nb, bbox6);
        const auto B = make_bones(bones, nb);
        const TransformGrid tg = precompute_transform_grid(g, B, 1);
        SearchContext ctx;
        ctx.bones = B;
        ctx.grid = &g;
        ctx.tgrid = &tg;
        for (int64_t p = 0; p < n; ++p) {
            const auto st = init_states(Vec3(pts[3 * p], pts[3 * p + 1], pts[3 * p + 2]), ctx, SearchVariant::Voxel);
            for (int i = 0; i < nb; ++i) {
                for (int a = 0; a < 3; ++a) x0[(p * nb + i) * 3 + a] = st[i].x0(a);
                for (int r = 0; r < 3; ++r)
                    for (int c = 0; c < 3; ++c) jinv0[(p * nb + i) * 9 + 3 * r + c] = st[i].inv_jacobian(r, c);
            }
        }
    });
}

}  // extern "C"
