// fsk_io.cpp — the wire and disk formats around the deformer, host C++:
//
//   SKNV weight grids          load_sknv / save_sknv      (proj/src/skinning.cpp:239-288)
//   .bin posed points          load_points_bin            (proj/src/pointio.cpp:43-62)
//   correspondence dumps       save_correspondence_dump   (proj/src/pointio.cpp:97-117)
//   one cmd_deform frame       files → GPU → dump         (proj/tools/fskin_cli.cpp:395-429)
//
// At the 64 M-point scale of BASELINE config 5 the dump is ~10^10 characters of "%.17g" text,
// an order of magnitude more host time than the GPU search: it is formatted by all host cores
// in blocks (std::to_chars, general format, 17 significant digits == printf "%.17g") and
// written in query order. Errors carry the reference's std::runtime_error texts.
#include <cuda_runtime.h>

#include <algorithm>
#include <charconv>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "fsk.h"

namespace {

thread_local std::string g_io_err;

template <typename Fn>
int io_guard(Fn&& fn) {
    try {
        fn();
        return FSK_OK;
    } catch (const std::invalid_argument& e) {
        g_io_err = e.what();
        return FSK_EINVAL;
    } catch (const std::exception& e) {
        g_io_err = e.what();
        return FSK_EIO;
    }
}

void put_g17(std::string& s, double v) {  // printf("%.17g", v)
    char buf[40];
    const auto r = std::to_chars(buf, buf + sizeof(buf), v, std::chars_format::general, 17);
    s.append(buf, r.ptr);
}
void put_int(std::string& s, long long v) {
    char buf[24];
    const auto r = std::to_chars(buf, buf + sizeof(buf), v);
    s.append(buf, r.ptr);
}

struct SknvHeader {
    fsk_grid_desc d;
    int64_t payload;  // floats
};

SknvHeader read_sknv_header(std::ifstream& in, const std::string& path) {  // skinning.cpp:264-282
    char magic[4];
    in.read(magic, 4);
    if (!in || std::memcmp(magic, "SKNV", 4) != 0) throw std::runtime_error(path + ": not a SKNV grid file");
    uint32_t h[5];
    in.read(reinterpret_cast<char*>(h), sizeof(h));
    if (!in) throw std::runtime_error(path + ": not a SKNV grid file");
    if (h[0] != 1u) throw std::runtime_error(path + ": unsupported SKNV version " + std::to_string(h[0]));
    float bb[6];
    in.read(reinterpret_cast<char*>(bb), sizeof(bb));
    if (!in) throw std::runtime_error(path + ": truncated SKNV payload");
    SknvHeader r{};
    r.d.nx = (int32_t)h[1];
    r.d.ny = (int32_t)h[2];
    r.d.nz = (int32_t)h[3];
    r.d.n_bones = (int32_t)h[4];
    for (int a = 0; a < 3; ++a) {
        r.d.bbox_min[a] = bb[a];
        r.d.bbox_max[a] = bb[3 + a];
    }
    // SkinningVoxelGrid's constructor checks (skinning.cpp:60-70)
    if (r.d.nx < 2 || r.d.ny < 2 || r.d.nz < 2)
        throw std::invalid_argument("SkinningVoxelGrid: dims must be >= 2 per axis");
    if (r.d.n_bones < 1) throw std::invalid_argument("SkinningVoxelGrid: n_bones must be >= 1");
    for (int a = 0; a < 3; ++a)
        if (!(bb[3 + a] - bb[a] > 0.f)) throw std::invalid_argument("SkinningVoxelGrid: bbox must have positive extent");
    r.payload = (int64_t)r.d.nx * r.d.ny * r.d.nz * r.d.n_bones;
    return r;
}

}  // namespace

extern "C" {

const char* fsk_io_last_error(void) { return g_io_err.c_str(); }

int fsk_sknv_read(const char* path, fsk_grid_desc* desc, float* weights, int64_t cap) {
    return io_guard([&] {
        if (!path || !desc) throw std::invalid_argument("fsk: null buffer");
        std::ifstream in(path, std::ios::binary);
        if (!in) throw std::runtime_error(std::string("cannot open grid file: ") + path);
        const SknvHeader h = read_sknv_header(in, path);
        *desc = h.d;
        if (!weights) return;  // header only
        if (cap < h.payload) throw std::invalid_argument("fsk: weight buffer too small");
        in.read(reinterpret_cast<char*>(weights), (std::streamsize)(h.payload * sizeof(float)));
        if (!in) throw std::runtime_error(std::string(path) + ": truncated SKNV payload");
    });
}

int fsk_sknv_write(const char* path, const fsk_grid_desc* desc, const float* weights) {
    return io_guard([&] {
        if (!path || !desc || !weights) throw std::invalid_argument("fsk: null buffer");
        std::ofstream out(path, std::ios::binary);
        if (!out) throw std::runtime_error(std::string("cannot write grid file: ") + path);
        out.write("SKNV", 4);
        const uint32_t h[5] = {1u, (uint32_t)desc->nx, (uint32_t)desc->ny, (uint32_t)desc->nz, (uint32_t)desc->n_bones};
        out.write(reinterpret_cast<const char*>(h), sizeof(h));
        float bb[6];  // SKNV stores the bbox in float32 (skinning.cpp:248-252)
        for (int a = 0; a < 3; ++a) {
            bb[a] = (float)desc->bbox_min[a];
            bb[3 + a] = (float)desc->bbox_max[a];
        }
        out.write(reinterpret_cast<const char*>(bb), sizeof(bb));
        const int64_t n = (int64_t)desc->nx * desc->ny * desc->nz * desc->n_bones;
        out.write(reinterpret_cast<const char*>(weights), (std::streamsize)(n * sizeof(float)));
        if (!out) throw std::runtime_error(std::string("short write to grid file: ") + path);
    });
}

// .bin points (pointio.cpp:43-62): raw float32 triples; points == NULL returns the count only
int fsk_points_bin_read(const char* path, float* points, int64_t cap, int64_t* n_out) {
    return io_guard([&] {
        if (!path || !n_out) throw std::invalid_argument("fsk: null buffer");
        std::ifstream in(path, std::ios::binary | std::ios::ate);
        if (!in) throw std::runtime_error(std::string("cannot open points file: ") + path);
        const std::streamsize bytes = in.tellg();
        if (bytes % std::streamsize(3 * sizeof(float)) != 0)
            throw std::runtime_error(std::string(path) + ": size " + std::to_string((long long)bytes) +
                                     " is not a whole number of f32 triples");
        const int64_t n = bytes / (3 * (int64_t)sizeof(float));
        *n_out = n;
        if (!points) return;
        if (cap < n) throw std::invalid_argument("fsk: point buffer too small");
        in.seekg(0);
        in.read(reinterpret_cast<char*>(points), bytes);
        if (!in) throw std::runtime_error(std::string(path) + ": truncated read");
    });
}

int fsk_points_bin_write(const char* path, const float* points, int64_t n) {
    return io_guard([&] {
        if (!path || (n > 0 && !points)) throw std::invalid_argument("fsk: null buffer");
        std::ofstream out(path, std::ios::binary);
        if (!out) throw std::runtime_error(std::string("cannot write points file: ") + path);
        out.write(reinterpret_cast<const char*>(points), (std::streamsize)(n * 3 * sizeof(float)));
        if (!out) throw std::runtime_error(std::string("short write to points file: ") + path);
    });
}

// save_correspondence_dump (pointio.cpp:97-117): per query "x y z count" then per root
// " x y z residual source_bone iterations", all reals "%.17g" of the double values. Formatted
// by `threads` host threads (0 = all cores) in blocks of queries, written in query order.
}  // extern "C"

namespace {
void dump_block(std::ofstream& out, const float* queries, int64_t n, const int64_t* offsets, const fsk_root* roots,
                int T, std::vector<std::string>& buf) {
    constexpr int64_t kBlock = 1 << 18;  // queries per thread per block
    buf.resize(T);
    for (int64_t b0 = 0; b0 < n; b0 += kBlock * T) {
        std::vector<std::thread> pool;
        for (int t = 0; t < T; ++t)
            pool.emplace_back([&, t] {
                std::string& s = buf[t];
                s.clear();
                const int64_t q0 = b0 + (int64_t)t * kBlock, q1 = std::min(n, q0 + kBlock);
                for (int64_t q = q0; q < q1; ++q) {
                    for (int a = 0; a < 3; ++a) {
                        if (a) s.push_back(' ');
                        put_g17(s, (double)queries[3 * q + a]);
                    }
                    s.push_back(' ');
                    put_int(s, (long long)(offsets[q + 1] - offsets[q]));
                    for (int64_t r = offsets[q]; r < offsets[q + 1]; ++r) {
                        const fsk_root& R = roots[r];
                        for (int a = 0; a < 3; ++a) {
                            s.push_back(' ');
                            put_g17(s, (double)R.x[a]);
                        }
                        s.push_back(' ');
                        put_g17(s, (double)R.residual);
                        s.push_back(' ');
                        put_int(s, R.source_bone);
                        s.push_back(' ');
                        put_int(s, R.iterations);
                    }
                    s.push_back('\n');
                }
            });
        for (auto& th : pool) th.join();
        for (int t = 0; t < T; ++t) out.write(buf[t].data(), (std::streamsize)buf[t].size());
    }
}

int host_threads(int threads) { return threads > 0 ? threads : (int)std::max(1u, std::thread::hardware_concurrency()); }

// pinned host block (H2D/D2H at full PCIe rate); plain allocation when no device is usable
struct HostBlock {
    void* p = nullptr;
    size_t bytes = 0;
    bool pinned = false;
    void ensure(size_t b) {
        if (b <= bytes) return;
        release();
        pinned = cudaMallocHost(&p, b) == cudaSuccess;
        if (!pinned) {
            cudaGetLastError();
            p = std::malloc(b);
            if (!p) throw std::runtime_error("fsk: out of host memory");
        }
        bytes = b;
    }
    void release() {
        if (p) pinned ? (void)cudaFreeHost(p) : std::free(p);
        p = nullptr;
        bytes = 0;
    }
    ~HostBlock() { release(); }
    template <typename T>
    T* as() const { return static_cast<T*>(p); }
};
}  // namespace

extern "C" {

int fsk_write_correspondence_dump(const char* path, const float* queries, int64_t n, const int64_t* offsets,
                                  const fsk_root* roots, int32_t threads) {
    return io_guard([&] {
        if (!path || (n > 0 && (!queries || !offsets))) throw std::invalid_argument("fsk: null buffer");
        std::ofstream out(path, std::ios::binary);
        if (!out) throw std::runtime_error(std::string("cannot write correspondence dump: ") + path);
        std::vector<std::string> buf;
        dump_block(out, queries, n, offsets, roots, host_threads(threads), buf);
        if (!out) throw std::runtime_error(std::string("short write to correspondence dump: ") + path);
    });
}

// One cmd_deform frame from files to file (fskin_cli.cpp:395-429 without the occupancy column):
// SKNV grid + .bin points in, correspondence dump out, streamed in blocks of points so host memory
// is bounded by the block size, not by the frame (64M points: ~10^10 dump characters): block k+1 is
// read and searched (fsk_deform_host's chunked H2D / search / D2H pipeline) while block k is
// formatted and written by a writer thread. Root buffers are count-then-allocate: a block's first
// try holds 2 roots per query, a block with more kept roots is re-run with the reported total.
// Returns the query and root counts. FSK_IO_BLOCK_POINTS overrides the block size (testing).
int fsk_deform_files(fsk_ctx* ctx, const char* grid_path, const float* bones, int32_t n_bones,
                     const char* points_path, const fsk_search_opts* opts, const char* dump_path, int64_t* n_queries,
                     int64_t* n_roots) {
    return io_guard([&] {
        if (!ctx || !grid_path || !bones || !points_path || !opts || !dump_path)
            throw std::invalid_argument("fsk: null buffer");
        fsk_grid_desc d{};
        auto rc = [](int r, bool io) {
            if (r != FSK_OK) {
                const char* m = io ? fsk_io_last_error() : fsk_last_error();
                if (r == FSK_EINVAL) throw std::invalid_argument(m);
                throw std::runtime_error(m);
            }
        };
        rc(fsk_sknv_read(grid_path, &d, nullptr, 0), true);
        const int64_t V = (int64_t)d.nx * d.ny * d.nz;
        HostBlock w;
        w.ensure(std::max<int64_t>(1, V * d.n_bones) * sizeof(float));
        rc(fsk_sknv_read(grid_path, &d, w.as<float>(), V * d.n_bones), true);
        int64_t n = 0;
        rc(fsk_points_bin_read(points_path, nullptr, 0, &n), true);
        std::ifstream in(points_path, std::ios::binary);
        if (!in) throw std::runtime_error(std::string("cannot open points file: ") + points_path);
        std::ofstream out(dump_path, std::ios::binary);
        if (!out) throw std::runtime_error(std::string("cannot write correspondence dump: ") + dump_path);
        int64_t blk = int64_t(1) << 23;  // 8M points per block
        if (const char* e = getenv("FSK_IO_BLOCK_POINTS")) blk = std::max<int64_t>(1, atoll(e));
        blk = std::max<int64_t>(1, std::min(blk, n));
        HostBlock pts[2], offs[2], roots[2];
        int64_t cnt[2] = {0, 0}, total = 0;
        std::vector<std::string> text;
        std::thread writer;
        std::string werr;
        auto join = [&] {
            if (writer.joinable()) writer.join();
            if (!werr.empty()) throw std::runtime_error(werr);
        };
        const int T = host_threads(0);
        try {
            for (int64_t p0 = 0, k = 0; p0 < n || (n == 0 && k == 0); p0 += blk, ++k) {
                const int s = (int)(k & 1);
                const int64_t m = std::min(blk, n - p0);
                pts[s].ensure(std::max<int64_t>(1, 3 * m) * sizeof(float));
                offs[s].ensure((m + 1) * sizeof(int64_t));
                in.read(pts[s].as<char>(), (std::streamsize)(m * 3 * sizeof(float)));
                if (!in) throw std::runtime_error(std::string(points_path) + ": truncated read");
                int64_t cap = std::max<int64_t>(1, 2 * m), t = 0;
                for (int attempt = 0;; ++attempt) {  // count-then-allocate
                    roots[s].ensure(cap * sizeof(fsk_root));
                    const int r = fsk_deform_host(ctx, w.as<float>(), &d, bones, n_bones, pts[s].as<float>(), m, opts,
                                                  offs[s].as<int64_t>(), roots[s].as<fsk_root>(), cap, &t, nullptr);
                    if (r == FSK_EINVAL && t > cap && attempt == 0) {
                        cap = t;
                        continue;
                    }
                    rc(r, false);
                    break;
                }
                cnt[s] = t;
                total += t;
                join();  // block k-1 written; its buffers (slot s^1) are free again after this
                writer = std::thread([&, s, m] {
                    try {
                        dump_block(out, pts[s].as<float>(), m, offs[s].as<int64_t>(), roots[s].as<fsk_root>(), T, text);
                    } catch (const std::exception& e) {
                        werr = e.what();
                    }
                });
                if (n == 0) break;
            }
            join();
        } catch (...) {
            if (writer.joinable()) writer.join();
            throw;
        }
        if (!out) throw std::runtime_error(std::string("short write to correspondence dump: ") + dump_path);
        if (n_queries) *n_queries = n;
        if (n_roots) *n_roots = total;
    });
}

}  // extern "C"
