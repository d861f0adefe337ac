// Exercises the reference-facing C++ API (include/fskin/*.hpp) exactly as the reference's
// callers do (cmd_deform / cmd_bench / train: precompute_transform_grid → batch_search,
// fskin_cli.cpp:395-408, diff.cpp:278-289), on inputs written by tests/test_cpp_api.py.
// Writes the CorrespondenceSets as text for the Python side to compare with the oracle,
// and checks the API's own contracts (soundness, error messages, identity pose).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "fskin/correspondence.hpp"
#include "fskin/deformer.hpp"
#include "fskin/diff.hpp"

using namespace fskin;

static int fails = 0;
#define CHECK(c)                                                          \
    do {                                                                  \
        if (!(c)) {                                                       \
            std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c); \
            ++fails;                                                      \
        }                                                                 \
    } while (0)

template <typename Fn>
static void expect_invalid(Fn&& fn, const std::string& msg) {
    try {
        fn();
        std::fprintf(stderr, "expected invalid_argument '%s'\n", msg.c_str());
        ++fails;
    } catch (const std::invalid_argument& e) {
        if (std::string(e.what()).find(msg) == std::string::npos) {
            std::fprintf(stderr, "wrong message '%s' (want '%s')\n", e.what(), msg.c_str());
            ++fails;
        }
    }
}

int main(int argc, char** argv) {
    if (argc < 3) return 2;
    std::ifstream in(argv[1], std::ios::binary);
    int hdr[5];  // nx ny nz nb n
    in.read(reinterpret_cast<char*>(hdr), sizeof(hdr));
    float bb[6];
    in.read(reinterpret_cast<char*>(bb), sizeof(bb));
    int max_iters;
    in.read(reinterpret_cast<char*>(&max_iters), 4);
    const GridDims dims{hdr[0], hdr[1], hdr[2]};
    const int nb = hdr[3], n = hdr[4];
    SkinningVoxelGrid grid(dims, Aabb{{bb[0], bb[1], bb[2]}, {bb[3], bb[4], bb[5]}}, nb);
    std::vector<float> w(grid.raw().size()), b(nb * 12), x(3 * n);
    in.read(reinterpret_cast<char*>(w.data()), w.size() * 4);
    in.read(reinterpret_cast<char*>(b.data()), b.size() * 4);
    in.read(reinterpret_cast<char*>(x.data()), x.size() * 4);
    if (!in) return 3;
    std::copy(w.begin(), w.end(), grid.raw().begin());
    grid.validate();
    std::vector<RigidTransform> bones(nb);
    for (int i = 0; i < nb; ++i)
        for (int r = 0; r < 3; ++r) {
            for (int c = 0; c < 3; ++c) bones[i].rotation(r, c) = b[i * 12 + r * 4 + c];
            bones[i].translation[r] = b[i * 12 + r * 4 + 3];
        }
    std::vector<Vec3> queries(n);
    for (int p = 0; p < n; ++p) queries[p] = Vec3(x[3 * p], x[3 * p + 1], x[3 * p + 2]);

    const TransformGrid tgrid = precompute_transform_grid(grid, bones, 4);
    SearchContext ctx{bones, nullptr, &grid, &tgrid};
    SearchOptions opts = SearchOptions::defaults_for(grid.bbox());
    opts.max_iters = max_iters;
    const std::vector<CorrespondenceSet> sets = batch_search(queries, ctx, opts, 8);
    CHECK(sets.size() == static_cast<size_t>(n));

    std::FILE* f = std::fopen(argv[2], "w");
    for (const auto& s : sets) {
        std::fprintf(f, "%zu", s.roots.size());
        for (const Root& r : s.roots)
            std::fprintf(f, " %d %.9g %.9g %.9g %.9g %d", r.source_bone, r.x.x(), r.x.y(), r.x.z(), r.residual,
                         r.iterations);
        std::fprintf(f, "\n");
    }
    std::fclose(f);

    // soundness through the API's own evaluator
    for (int p = 0; p < n && p < 500; ++p)
        for (const Root& r : sets[p].roots) {
            const Vec3 d = forward_deform(r.x, tgrid);
            CHECK((d - queries[p]).norm() < opts.conv_eps * 1.01);
            CHECK((r.x - queries[p]).norm() >= 0.0);
        }
    // broyden_search on one query equals the batch result
    const CorrespondenceSet one = broyden_search(queries[0], ctx, opts);
    CHECK(one.roots.size() == sets[0].roots.size());
    for (size_t k = 0; k < one.roots.size(); ++k) CHECK(one.roots[k].x == sets[0].roots[k].x);
    // init_states: x0 = B_i^-1 x' (float64; the values are compared with the oracle's by the test)
    const auto st = init_states(queries[1], ctx, SearchVariant::Voxel);
    CHECK(st.size() == static_cast<size_t>(nb));
    for (int i = 0; i < nb; ++i) CHECK((st[i].x0 - bones[i].inverse().apply(queries[1])).norm() < 1e-12);
    if (argc > 3) {
        std::FILE* g = std::fopen(argv[3], "wb");
        for (const auto& s : st) {
            const double x3[3] = {s.x0[0], s.x0[1], s.x0[2]};
            std::fwrite(x3, sizeof(double), 3, g);
        }
        for (const auto& s : st)
            for (int r = 0; r < 3; ++r)
                for (int c = 0; c < 3; ++c) {
                    const double v = s.inv_jacobian(r, c);
                    std::fwrite(&v, sizeof(double), 1, g);
                }
        std::fclose(g);
    }
    // TransformGrid is a value type (deformer.hpp:27-49): a modified copy leaves the original's
    // device mirror alone, and writes through vertex_transform() after a search are seen
    {
        const Vec3 probe = queries[2];
        const Vec3 before = forward_deform_batch({&probe, 1}, tgrid)[0];
        TransformGrid t2 = tgrid;
        for (std::int64_t v = 0; v < t2.dims().vertex_count(); ++v) t2.set_vertex(v, Affine3::from(RigidTransform::identity()));
        const Vec3 id = forward_deform_batch({&probe, 1}, t2)[0];
        CHECK((id - probe).norm() < 1e-5);
        CHECK(forward_deform_batch({&probe, 1}, tgrid)[0] == before);
        double* m = t2.vertex_transform(0);
        for (std::int64_t v = 0; v < t2.dims().vertex_count(); ++v) {
            m = t2.vertex_transform(v);
            m[3] += 1.0;  // translate every vertex by +1 in x, through the raw pointer
        }
        const Vec3 moved = forward_deform_batch({&probe, 1}, t2)[0];
        CHECK(std::abs(moved[0] - probe[0] - 1.0) < 1e-5);
        CHECK(forward_deform_batch({&probe, 1}, tgrid)[0] == before);
    }
    // max_iters beyond 255 (correspondence.cpp:20 accepts any value >= 1)
    {
        SearchOptions o = opts;
        o.max_iters = 300;
        const std::vector<CorrespondenceSet> s300 = batch_search(std::span<const Vec3>(queries).first(200), ctx, o);
        CHECK(s300.size() == 200);
    }
    // lossless precomputation: the weight-grid and transform-grid evaluators agree
    // to 1e-10 in float64; the GPU batch evaluator (float32) to 1e-5
    for (int p = 0; p < 50; ++p) {
        const Vec3 a = forward_deform(queries[p], grid, bones);
        const Vec3 g = forward_deform(queries[p], tgrid);
        CHECK((a - g).norm() < 1e-10);
        CHECK((forward_deform_batch({&queries[p], 1}, tgrid)[0] - g).norm() < 1e-5);
        const Mat3 J = deform_jacobian(queries[p], grid, bones);
        const Mat3 Jb = deform_jacobian_batch({&queries[p], 1}, tgrid)[0];
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) CHECK(std::abs(J(r, c) - Jb(r, c)) < 1e-4);
    }
    // implicit differentiation (diff.cpp:31-51): exact vs approx cotangent at a converged root, and the
    // singular-root error
    {
        int checked = 0;
        double cos_sum = 0.0;
        for (int p = 0; p < n && checked < 200; ++p)
            for (const Root& r : sets[p].roots) {
                if (r.residual > opts.conv_eps / 10) continue;
                const Vec3 v(0.3, -0.7, 0.5);
                const Vec3 ue = implicit_cotangent_exact(r.x, grid, bones, v);
                const Vec3 ua = implicit_cotangent_approx(r.inv_jacobian, v);
                cos_sum += ue.dot(ua) / (ue.norm() * ua.norm());
                ++checked;
                break;
            }
        CHECK(checked > 50);
        CHECK(cos_sum / checked > 0.9);
        SkinningVoxelGrid g1(GridDims{3, 3, 3}, Aabb{{0, 0, 0}, {1, 1, 1}}, 1);
        for (auto& e : g1.raw()) e = 1.0;
        RigidTransform flat;
        flat.rotation = Mat3::Identity() * 1e-4;
        bool threw = false;
        try {
            implicit_cotangent_exact(Vec3(0.5, 0.5, 0.5), g1, {&flat, 1}, Vec3(1, 0, 0));
        } catch (const SingularRootError&) {
            threw = true;
        }
        CHECK(threw);
        // grid gradient through the API: exact and approx agree in direction on the whole batch
        std::vector<int> first(n, -1);
        std::vector<Vec3> cot(n, Vec3(0.1, 0.2, -0.3));
        for (int p = 0; p < n; ++p)
            if (!sets[p].roots.empty()) first[p] = 0;
        const GridGradient ge = implicit_grad_grid(sets, first, cot, grid, bones, true);
        const GridGradient ga = implicit_grad_grid(sets, first, cot, grid, bones, false);
        double dotv = 0, na = 0, nb2 = 0;
        for (size_t e = 0; e < ge.d_weights.size(); ++e) {
            dotv += ge.d_weights[e] * ga.d_weights[e];
            na += ge.d_weights[e] * ge.d_weights[e];
            nb2 += ga.d_weights[e] * ga.d_weights[e];
        }
        CHECK(ge.d_tgrid.size() == static_cast<size_t>(grid.dims().vertex_count()) * 12);
        CHECK(dotv / std::sqrt(na * nb2) > 0.9);
    }
    // SearchVariant::Mlp (correspondence.cpp:77-79): the reference's SkinningMlp init, distilled to a grid
    // (skinning.cpp:195-221); the MLP-variant search through the same API; its root sets vs the voxel
    // variant on the distilled grid (SPEC acceptance 3); init_states of the MLP variant
    if (argc > 5) {
        const SkinningMlp mlp(nb, 7, grid.bbox());
        CHECK(mlp.bone_count() == nb && mlp.widths().front() == 3);
        double wsum = 0.0;
        const VectorXd w0 = mlp.weights(queries[0]);
        for (std::int64_t i = 0; i < w0.size(); ++i) wsum += w0[i];
        CHECK(std::abs(wsum - 1.0) < 1e-12);
        const SkinningVoxelGrid dg = distill(mlp, GridDims{64, 64, 16}, grid.bbox());
        const TransformGrid dtg = precompute_transform_grid(dg, bones);
        const int m = std::min(n, 2000);
        const std::span<const Vec3> q(queries.data(), m);
        SearchOptions mo = opts;
        mo.variant = SearchVariant::Mlp;
        const SearchContext mctx{bones, &mlp, nullptr, nullptr};
        const std::vector<CorrespondenceSet> ms = batch_search(q, mctx, mo);
        const std::vector<CorrespondenceSet> vs = batch_search(q, SearchContext{bones, nullptr, &dg, &dtg}, opts);
        int match = 0;
        for (int p = 0; p < m; ++p) {
            bool ok = ms[p].roots.size() == vs[p].roots.size();
            for (size_t k = 0; ok && k < ms[p].roots.size(); ++k)
                ok = (ms[p].roots[k].x - vs[p].roots[k].x).norm() < 1e-2 * grid.bbox().diagonal();
            match += ok;
        }
        std::printf("mlp vs voxel (64x64x16 distilled): %d / %d root sets match\n", match, m);
        CHECK(match >= 0.99 * m);
        const auto st = init_states(queries[3], mctx, SearchVariant::Mlp);
        CHECK(st.size() == static_cast<size_t>(nb));
        for (int i = 0; i < nb; ++i) CHECK((st[i].x0 - bones[i].inverse().apply(queries[3])).norm() < 1e-12);
        expect_invalid([&] { SearchContext c2 = mctx; c2.mlp = nullptr; batch_search(q, c2, mo); },
                       "search: mlp variant needs a skinning mlp");
        std::FILE* th = std::fopen(argv[4], "wb");
        std::fwrite(mlp.parameters().data(), sizeof(double), mlp.parameters().size(), th);
        std::fclose(th);
        std::FILE* f2 = std::fopen(argv[5], "w");
        for (const auto& sset : ms) {
            std::fprintf(f2, "%zu", sset.roots.size());
            for (const Root& r : sset.roots)
                std::fprintf(f2, " %d %.9g %.9g %.9g %.9g %d", r.source_bone, r.x.x(), r.x.y(), r.x.z(), r.residual,
                             r.iterations);
            std::fprintf(f2, "\n");
        }
        std::fclose(f2);
    }
    // dedup_roots
    std::vector<Root> rr(3);
    rr[0].x = Vec3(0, 0, 0);
    rr[1].x = Vec3(0, 0, 0);
    rr[2].x = Vec3(1, 0, 0);
    CHECK(dedup_roots(rr, 0.5).size() == 2);
    // error contract (correspondence.cpp:19-41, deformer.cpp:64-66)
    expect_invalid([&] { SearchOptions o = opts; o.max_iters = 0; batch_search(queries, ctx, o); },
                   "search: max_iters must be >= 1");
    expect_invalid([&] { SearchOptions o = opts; o.div_eps = o.conv_eps; batch_search(queries, ctx, o); },
                   "search: div_eps must exceed conv_eps");
    expect_invalid([&] { SearchContext c2 = ctx; c2.tgrid = nullptr; batch_search(queries, c2, opts); },
                   "search: voxel variant needs skinning and transform grids");
    expect_invalid([&] { SearchContext c2 = ctx; c2.bones = {}; batch_search(queries, c2, opts); },
                   "search: no bone transforms");
    expect_invalid([&] { precompute_transform_grid(grid, std::span<const RigidTransform>(bones).first(nb - 1)); },
                   "precompute_transform_grid: bone count mismatch");
    expect_invalid([&] { SearchOptions o = opts; o.variant = SearchVariant::Mlp; batch_search(queries, ctx, o); },
                   "search: mlp variant needs a skinning mlp");
    // empty query list → empty result
    CHECK(batch_search(std::span<const Vec3>(), ctx, opts).empty());
    std::printf("fskin_api_check: %d failures\n", fails);
    return fails ? 1 : 0;
}
