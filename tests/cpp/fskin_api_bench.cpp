// End-to-end timing of the reference-facing C++ API (what a reference caller links): per frame
// precompute_transform_grid + batch_search (std::span<const Vec3> queries in, the reference's
// std::vector<CorrespondenceSet> out — f64→f32 conversion, H2D, search, D2H and the host build of the
// result sets all inside the timed loop). Input file as fskin_api_check.cpp's. Prints one JSON line.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <vector>

#include "fskin/correspondence.hpp"
#include "fskin/deformer.hpp"

using namespace fskin;

int main(int argc, char** argv) {
    if (argc < 3) return 2;
    const int frames = std::atoi(argv[2]);
    std::ifstream in(argv[1], std::ios::binary);
    int hdr[5];
    in.read(reinterpret_cast<char*>(hdr), sizeof(hdr));
    float bb[6];
    in.read(reinterpret_cast<char*>(bb), sizeof(bb));
    int max_iters;
    in.read(reinterpret_cast<char*>(&max_iters), 4);
    const int nb = hdr[3], n = hdr[4];
    SkinningVoxelGrid grid(GridDims{hdr[0], hdr[1], hdr[2]}, Aabb{{bb[0], bb[1], bb[2]}, {bb[3], bb[4], bb[5]}}, nb);
    std::vector<float> w(grid.raw().size()), b(nb * 12), x(3 * n);
    in.read(reinterpret_cast<char*>(w.data()), w.size() * 4);
    in.read(reinterpret_cast<char*>(b.data()), b.size() * 4);
    in.read(reinterpret_cast<char*>(x.data()), x.size() * 4);
    if (!in) return 3;
    std::copy(w.begin(), w.end(), grid.raw().begin());
    std::vector<RigidTransform> bones(nb);
    for (int i = 0; i < nb; ++i)
        for (int r = 0; r < 3; ++r) {
            for (int c = 0; c < 3; ++c) bones[i].rotation(r, c) = b[i * 12 + r * 4 + c];
            bones[i].translation[r] = b[i * 12 + r * 4 + 3];
        }
    std::vector<Vec3> queries(n);
    for (int p = 0; p < n; ++p) queries[p] = Vec3(x[3 * p], x[3 * p + 1], x[3 * p + 2]);
    SearchOptions opts = SearchOptions::defaults_for(grid.bbox());
    opts.max_iters = max_iters;
    size_t roots = 0;
    double t_pre = 0, t_search = 0;
    auto frame = [&] {
        const auto a = std::chrono::steady_clock::now();
        const TransformGrid tgrid = precompute_transform_grid(grid, bones);
        const auto b = std::chrono::steady_clock::now();
        const SearchContext ctx{bones, nullptr, &grid, &tgrid};
        const std::vector<CorrespondenceSet> sets = batch_search(queries, ctx, opts);
        t_pre += std::chrono::duration<double>(b - a).count();
        t_search += std::chrono::duration<double>(std::chrono::steady_clock::now() - b).count();
        roots = 0;
        for (const auto& s : sets) roots += s.roots.size();
    };
    frame();
    frame();
    t_pre = t_search = 0;
    const auto t0 = std::chrono::steady_clock::now();
    for (int f = 0; f < frames; ++f) frame();
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::printf("{\"frames\": %d, \"ms_per_frame\": %.4f, \"solves_per_s\": %.6e, \"roots\": %zu, "
                "\"precompute_ms\": %.4f, \"batch_search_ms\": %.4f}\n",
                frames, 1e3 * s / frames, (double)n * nb * frames / s, roots, 1e3 * t_pre / frames,
                1e3 * t_search / frames);
    return 0;
}
