// fskin_api.cpp — the reference's C++ deformer/correspondence API (include/fskin/*.hpp)
// implemented over the C-ABI (include/fsk.h). Hot-path entry points convert f64 → f32,
// run on the GPU and rebuild the reference's value types; errors are rethrown as the
// reference's exception types with its message text (std::invalid_argument for FSK_EINVAL,
// std::runtime_error otherwise). There is no CPU implementation of the search here.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <mutex>
#include <random>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <thread>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "fsk.h"
#include "fskin/correspondence.hpp"
#include "fskin/deformer.hpp"
#include "fskin/diff.hpp"
#include "fskin/geometry.hpp"
#include "fskin/skinning.hpp"

namespace fskin {

namespace {

void check(int rc) {
    if (rc == FSK_OK) return;
    const std::string msg = fsk_last_error();
    if (rc == FSK_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

void cuda_ok(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

/// Per-thread context on device $FSKIN_DEVICE (default 0): fsk contexts are not thread-safe.
struct ThreadCtx {
    fsk_ctx* ctx = nullptr;
    ThreadCtx() {
        const char* d = std::getenv("FSKIN_DEVICE");
        check(fsk_ctx_create(d ? std::atoi(d) : 0, &ctx));
    }
    ~ThreadCtx() {
        if (ctx) fsk_ctx_destroy(ctx);
    }
};
fsk_ctx* ctx() {
    thread_local ThreadCtx t;
    return t.ctx;
}

/// Device buffers of the C++ API come from a small process-wide pool (per device and size): a frame's
/// temporaries and TransformGrid mirrors reuse the previous frame's allocations instead of a
/// cudaMalloc/cudaFree pair (cudaFree synchronizes the device).
struct DevPool {
    std::mutex mu;
    struct Key {
        int dev;
        size_t bytes;
        bool operator<(const Key& o) const { return dev != o.dev ? dev < o.dev : bytes < o.bytes; }
    };
    std::map<Key, std::vector<void*>> free;
    void* get(size_t bytes) {
        int dev = 0;
        cudaGetDevice(&dev);
        {
            std::lock_guard<std::mutex> lk(mu);
            auto it = free.find(Key{dev, bytes});
            if (it != free.end() && !it->second.empty()) {
                void* p = it->second.back();
                it->second.pop_back();
                return p;
            }
        }
        void* p = nullptr;
        cuda_ok(cudaMalloc(&p, bytes), "cudaMalloc");
        return p;
    }
    void put(void* p, size_t bytes) {
        int dev = 0;
        cudaGetDevice(&dev);
        std::lock_guard<std::mutex> lk(mu);
        auto& v = free[Key{dev, bytes}];
        if (v.size() < 8) v.push_back(p);
        else cudaFree(p);
    }
};
DevPool& dev_pool() {
    static DevPool* pool = new DevPool;  // leaked on purpose: outlives thread-local contexts at exit
    return *pool;
}

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    explicit DevBuf(size_t n) {
        ctx();  // selects the device
        bytes = n ? n : 16;
        p = dev_pool().get(bytes);
    }
    ~DevBuf() {
        if (p) dev_pool().put(p, bytes);
    }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    template <typename T>
    T* as() const { return static_cast<T*>(p); }
};

/// Per-thread device and pinned host staging of batch_search, grown on demand and reused across calls
/// (no cudaMalloc / pageable copy per call).
struct Workspace {
    void* dev[4] = {};
    size_t dcap[4] = {};
    void* pin[4] = {};
    size_t pcap[4] = {};
    void* d(int i, size_t bytes) {
        if (dcap[i] < bytes) {
            if (dev[i]) cudaFree(dev[i]);
            dev[i] = nullptr;
            dcap[i] = 0;
            cuda_ok(cudaMalloc(&dev[i], bytes), "cudaMalloc");
            dcap[i] = bytes;
        }
        return dev[i];
    }
    void* h(int i, size_t bytes) {
        if (pcap[i] < bytes) {
            if (pin[i]) cudaFreeHost(pin[i]);
            pin[i] = nullptr;
            pcap[i] = 0;
            cuda_ok(cudaMallocHost(&pin[i], bytes), "cudaMallocHost");
            pcap[i] = bytes;
        }
        return pin[i];
    }
    ~Workspace() {
        for (int i = 0; i < 4; ++i) {
            if (dev[i]) cudaFree(dev[i]);
            if (pin[i]) cudaFreeHost(pin[i]);
        }
    }
};

void h2d(void* dst, const void* src, size_t bytes) {
    if (bytes) cuda_ok(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice), "cudaMemcpy H2D");
}
void d2h(void* dst, const void* src, size_t bytes) {
    if (bytes) cuda_ok(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost), "cudaMemcpy D2H");
}

fsk_grid_desc desc_of(const GridDims& d, const Aabb& bb, int nb) {
    fsk_grid_desc g;
    g.nx = d.nx;
    g.ny = d.ny;
    g.nz = d.nz;
    g.n_bones = nb;
    for (int a = 0; a < 3; ++a) {
        g.bbox_min[a] = bb.min[a];
        g.bbox_max[a] = bb.max[a];
    }
    return g;
}

std::vector<float> bones_f32(std::span<const RigidTransform> bones) {
    std::vector<float> b(bones.size() * 12);
    for (size_t i = 0; i < bones.size(); ++i)
        for (int r = 0; r < 3; ++r) {
            for (int c = 0; c < 3; ++c) b[i * 12 + r * 4 + c] = static_cast<float>(bones[i].rotation(r, c));
            b[i * 12 + r * 4 + 3] = static_cast<float>(bones[i].translation[r]);
        }
    return b;
}

std::vector<float> points_f32(std::span<const Vec3> x) {
    std::vector<float> p(x.size() * 3);
    for (size_t i = 0; i < x.size(); ++i)
        for (int a = 0; a < 3; ++a) p[3 * i + a] = static_cast<float>(x[i][a]);
    return p;
}

// check_context (correspondence.cpp:29-41)
void check_context(const SearchContext& c, SearchVariant variant) {
    if (c.bones.empty()) throw std::invalid_argument("search: no bone transforms");
    if (variant == SearchVariant::Mlp) {
        if (c.mlp == nullptr) throw std::invalid_argument("search: mlp variant needs a skinning mlp");
        if (static_cast<size_t>(c.mlp->bone_count()) != c.bones.size())
            throw std::invalid_argument("search: mlp bone count mismatch");
        return;
    }
    if (c.grid == nullptr || c.tgrid == nullptr)
        throw std::invalid_argument("search: voxel variant needs skinning and transform grids");
    if (static_cast<size_t>(c.grid->bone_count()) != c.bones.size())
        throw std::invalid_argument("search: grid bone count mismatch");
}

fsk_search_opts c_opts(const SearchOptions& o) {
    fsk_search_opts c;
    c.max_iters = o.max_iters;
    c.conv_eps = o.conv_eps;
    c.div_eps = o.div_eps;
    c.dedup_dist = o.dedup_dist;
    c.flags = 0;
    return c;
}

}  // namespace

// ------------------------------------------------------------------------ geometry
RigidTransform RigidTransform::about_axis(const Vec3& pivot, const Vec3& axis, double angle) {
    const double n = axis.norm();
    if (n < 1e-12) throw std::invalid_argument("RigidTransform::about_axis: axis must be nonzero");
    const Vec3 k = axis / n;
    const double c = std::cos(angle), s = std::sin(angle), t = 1.0 - c;
    Mat3 r;
    r(0, 0) = c + t * k[0] * k[0];
    r(0, 1) = t * k[0] * k[1] - s * k[2];
    r(0, 2) = t * k[0] * k[2] + s * k[1];
    r(1, 0) = t * k[1] * k[0] + s * k[2];
    r(1, 1) = c + t * k[1] * k[1];
    r(1, 2) = t * k[1] * k[2] - s * k[0];
    r(2, 0) = t * k[2] * k[0] - s * k[1];
    r(2, 1) = t * k[2] * k[1] + s * k[0];
    r(2, 2) = c + t * k[2] * k[2];
    return {r, pivot - r * pivot};
}

double point_segment_distance(const Vec3& p, const Vec3& a, const Vec3& b) {
    const Vec3 ab = b - a;
    const double len2 = ab.squaredNorm();
    if (len2 < 1e-24) return (p - a).norm();
    const double t = std::clamp((p - a).dot(ab) / len2, 0.0, 1.0);
    return (p - (a + t * ab)).norm();
}

// ------------------------------------------------------------------------ skinning grid (host utilities)
SkinningVoxelGrid::SkinningVoxelGrid(GridDims dims, Aabb bbox, int n_bones)
    : dims_(dims), bbox_(bbox), n_bones_(n_bones) {
    if (dims.nx < 2 || dims.ny < 2 || dims.nz < 2)
        throw std::invalid_argument("SkinningVoxelGrid: dims must be >= 2 per axis");
    if (n_bones < 1) throw std::invalid_argument("SkinningVoxelGrid: n_bones must be >= 1");
    for (int a = 0; a < 3; ++a)
        if (!(bbox.max[a] - bbox.min[a] > 0.0))
            throw std::invalid_argument("SkinningVoxelGrid: bbox must have positive extent");
    data_.assign(static_cast<size_t>(dims.vertex_count()) * n_bones, 0.0);
}

Vec3 SkinningVoxelGrid::cell_size() const {
    const Vec3 e = bbox_.extent();
    return {e.x() / (dims_.nx - 1), e.y() / (dims_.ny - 1), e.z() / (dims_.nz - 1)};
}

Vec3 SkinningVoxelGrid::vertex_position(int i, int j, int k) const {
    const Vec3 h = cell_size();
    return bbox_.min + Vec3(i * h.x(), j * h.y(), k * h.z());
}

void SkinningVoxelGrid::validate() const {
    for (int a = 0; a < 3; ++a)
        if (!(bbox_.max[a] - bbox_.min[a] > 0.0))
            throw std::invalid_argument("SkinningVoxelGrid: bbox must have positive extent");
    const std::int64_t n = dims_.vertex_count();
    for (std::int64_t v = 0; v < n; ++v) {
        const double* w = data_.data() + v * n_bones_;
        double sum = 0.0;
        for (int b = 0; b < n_bones_; ++b) {
            if (w[b] < 0.0)
                throw std::invalid_argument("SkinningVoxelGrid: negative weight at vertex " + std::to_string(v));
            sum += w[b];
        }
        if (std::abs(sum - 1.0) > 1e-5)
            throw std::invalid_argument("SkinningVoxelGrid: weights at vertex " + std::to_string(v) + " sum to " +
                                        std::to_string(sum));
    }
}

namespace {
CellLocator locate(const GridDims& dims, const Aabb& bbox, const Vec3& x, bool lower) {
    const Vec3 p = bbox.clamp(x);
    const Vec3 ext = bbox.extent();
    const int n[3] = {dims.nx, dims.ny, dims.nz};
    int idx[3];
    double t[3];
    for (int a = 0; a < 3; ++a) {
        const double u = (p[a] - bbox.min[a]) / ext[a] * (n[a] - 1);
        int i = (u == u) ? static_cast<int>(std::floor(u)) : 0;
        if (lower && i >= 1 && u == static_cast<double>(i)) i -= 1;
        i = std::max(0, std::min(i, n[a] - 2));
        idx[a] = i;
        t[a] = std::clamp(u - i, 0.0, 1.0);
    }
    return {idx[0], idx[1], idx[2], t[0], t[1], t[2]};
}
}  // namespace

CellLocator locate_cell(const GridDims& dims, const Aabb& bbox, const Vec3& x) { return locate(dims, bbox, x, false); }
CellLocator locate_cell_lower(const GridDims& dims, const Aabb& bbox, const Vec3& x) {
    return locate(dims, bbox, x, true);
}

void trilerp_weights_into(const SkinningVoxelGrid& grid, const Vec3& x, double* out) {
    const CellLocator c = locate_cell(grid.dims(), grid.bbox(), x);
    const int nb = grid.bone_count();
    for (int b = 0; b < nb; ++b) out[b] = 0.0;
    for (int dk = 0; dk < 2; ++dk) {
        const double wz = dk ? c.tz : 1.0 - c.tz;
        for (int dj = 0; dj < 2; ++dj) {
            const double wyz = wz * (dj ? c.ty : 1.0 - c.ty);
            for (int di = 0; di < 2; ++di) {
                const double w = wyz * (di ? c.tx : 1.0 - c.tx);
                const double* v = grid.vertex_weights(c.i0 + di, c.j0 + dj, c.k0 + dk);
                for (int b = 0; b < nb; ++b) out[b] += w * v[b];
            }
        }
    }
}

VectorXd trilerp_weights(const SkinningVoxelGrid& grid, const Vec3& x) {
    VectorXd out(grid.bone_count());
    trilerp_weights_into(grid, x, out.data());
    return out;
}

MatrixXd weight_spatial_gradient(const SkinningVoxelGrid& grid, const Vec3& x) {
    const CellLocator c = locate_cell_lower(grid.dims(), grid.bbox(), x);
    const Vec3 h = grid.cell_size();
    const int nb = grid.bone_count();
    MatrixXd g(nb, 3);
    const double f[3][2] = {{1.0 - c.tx, c.tx}, {1.0 - c.ty, c.ty}, {1.0 - c.tz, c.tz}};
    const double s[3][2] = {{-1.0 / h.x(), 1.0 / h.x()}, {-1.0 / h.y(), 1.0 / h.y()}, {-1.0 / h.z(), 1.0 / h.z()}};
    for (int dk = 0; dk < 2; ++dk)
        for (int dj = 0; dj < 2; ++dj)
            for (int di = 0; di < 2; ++di) {
                const double* v = grid.vertex_weights(c.i0 + di, c.j0 + dj, c.k0 + dk);
                const double gx = s[0][di] * f[1][dj] * f[2][dk];
                const double gy = f[0][di] * s[1][dj] * f[2][dk];
                const double gz = f[0][di] * f[1][dj] * s[2][dk];
                for (int b = 0; b < nb; ++b) {
                    g(b, 0) += gx * v[b];
                    g(b, 1) += gy * v[b];
                    g(b, 2) += gz * v[b];
                }
            }
    return g;
}

void save_sknv(const SkinningVoxelGrid& grid, const std::string& path) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error("cannot write grid file: " + path);
    out.write("SKNV", 4);
    const std::uint32_t hdr[5] = {1u, static_cast<std::uint32_t>(grid.dims().nx), static_cast<std::uint32_t>(grid.dims().ny),
                                  static_cast<std::uint32_t>(grid.dims().nz), static_cast<std::uint32_t>(grid.bone_count())};
    out.write(reinterpret_cast<const char*>(hdr), sizeof(hdr));
    float bb[6];
    for (int a = 0; a < 3; ++a) {
        bb[a] = static_cast<float>(grid.bbox().min[a]);
        bb[3 + a] = static_cast<float>(grid.bbox().max[a]);
    }
    out.write(reinterpret_cast<const char*>(bb), sizeof(bb));
    std::vector<float> buf(grid.raw().begin(), grid.raw().end());
    out.write(reinterpret_cast<const char*>(buf.data()), static_cast<std::streamsize>(buf.size() * sizeof(float)));
    if (!out) throw std::runtime_error("short write to grid file: " + path);
}

SkinningVoxelGrid load_sknv(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error("cannot open grid file: " + path);
    char magic[4];
    in.read(magic, 4);
    if (!in || std::memcmp(magic, "SKNV", 4) != 0) throw std::runtime_error(path + ": not a SKNV grid file");
    std::uint32_t hdr[5];
    in.read(reinterpret_cast<char*>(hdr), sizeof(hdr));
    if (hdr[0] != 1u) throw std::runtime_error(path + ": unsupported SKNV version " + std::to_string(hdr[0]));
    float bb[6];
    in.read(reinterpret_cast<char*>(bb), sizeof(bb));
    GridDims dims{static_cast<int>(hdr[1]), static_cast<int>(hdr[2]), static_cast<int>(hdr[3])};
    SkinningVoxelGrid grid(dims, Aabb{{bb[0], bb[1], bb[2]}, {bb[3], bb[4], bb[5]}}, static_cast<int>(hdr[4]));
    std::vector<float> buf(grid.raw().size());
    in.read(reinterpret_cast<char*>(buf.data()), static_cast<std::streamsize>(buf.size() * sizeof(float)));
    if (!in) throw std::runtime_error(path + ": truncated SKNV payload");
    std::copy(buf.begin(), buf.end(), grid.raw().begin());
    return grid;
}

// ------------------------------------------------------------------------ skinning MLP (host float64 utilities)
namespace {
int64_t mlp_param_count(const std::vector<int>& w) {
    int64_t p = 0;
    for (size_t l = 0; l + 1 < w.size(); ++l) p += (int64_t)w[l + 1] * w[l] + w[l + 1];
    return p;
}
double softplus(double x) { return x > 0 ? x + std::log1p(std::exp(-x)) : std::log1p(std::exp(x)); }  // mlp.cpp
double sigmoid(double x) { return x >= 0 ? 1.0 / (1.0 + std::exp(-x)) : std::exp(x) / (1.0 + std::exp(x)); }

// forward (mlp.cpp:96-138) at one point with optional forward-mode tangents dX (3 columns): logits, and
// d logits / dx when `tangent` (n_out x 3, row-major)
std::vector<double> mlp_forward(const std::vector<int>& w, const std::vector<double>& th, const double* x,
                                std::vector<double>* tangent) {
    std::vector<double> h(x, x + w[0]), dh;
    if (tangent) {
        dh.assign((size_t)w[0] * 3, 0.0);
        for (int a = 0; a < 3 && a < w[0]; ++a) dh[(size_t)a * 3 + a] = 1.0;
    }
    size_t off = 0;
    for (size_t l = 0; l + 1 < w.size(); ++l) {
        const int ni = w[l], no = w[l + 1];
        const double* W = th.data() + off;  // column-major [no x ni]
        const double* b = W + (size_t)no * ni;
        off += (size_t)no * ni + no;
        std::vector<double> z(no), dz(tangent ? (size_t)no * 3 : 0, 0.0);
        for (int i = 0; i < no; ++i) {
            double acc = 0.0;
            for (int j = 0; j < ni; ++j) acc += W[(size_t)j * no + i] * h[j];
            z[i] = acc + b[i];
            if (tangent)
                for (int c = 0; c < 3; ++c) {
                    double t = 0.0;
                    for (int j = 0; j < ni; ++j) t += W[(size_t)j * no + i] * dh[(size_t)j * 3 + c];
                    dz[(size_t)i * 3 + c] = t;
                }
        }
        const bool hidden = l + 2 < w.size();
        if (hidden) {
            for (int i = 0; i < no; ++i) {
                if (tangent)
                    for (int c = 0; c < 3; ++c) dz[(size_t)i * 3 + c] *= sigmoid(z[i]);
                z[i] = softplus(z[i]);
            }
        }
        h.swap(z);
        if (tangent) dh.swap(dz);
    }
    if (tangent) *tangent = dh;
    return h;
}
}  // namespace

SkinningMlp::SkinningMlp(std::vector<int> widths, std::vector<double> parameters)
    : widths_(std::move(widths)), theta_(std::move(parameters)) {
    if (widths_.size() < 2) throw std::invalid_argument("Mlp: need at least input and output widths");
    if (widths_.front() != 3) throw std::invalid_argument("SkinningMlp: network input width must be 3");
    if ((int64_t)theta_.size() != mlp_param_count(widths_))
        throw std::invalid_argument("Mlp::set_parameters: wrong parameter count");
}

SkinningMlp::SkinningMlp(int n_bones, std::uint64_t seed) {
    if (n_bones < 1) throw std::invalid_argument("SkinningMlp: n_bones must be >= 1");
    widths_ = {3, 64, 64, 64, n_bones};
    theta_.assign((size_t)mlp_param_count(widths_), 0.0);
    std::mt19937_64 rng(seed);  // Mlp::Mlp (mlp.cpp:81-94)
    size_t off = 0;
    for (size_t l = 0; l + 1 < widths_.size(); ++l) {
        const int fan_in = widths_[l], no = widths_[l + 1];
        std::normal_distribution<double> dist(0.0, std::sqrt(2.0 / fan_in));
        for (size_t i = 0; i < (size_t)no * fan_in; ++i) theta_[off + i] = dist(rng);  // column-major data()
        off += (size_t)no * fan_in + no;                                             // biases stay zero
    }
    // scale_output_layer(0.05) (skinning.cpp:16, mlp.cpp:225-228)
    const size_t head = theta_.size() - ((size_t)widths_[3] * n_bones + n_bones);
    for (size_t i = head; i < theta_.size(); ++i) theta_[i] *= 0.05;
}

SkinningMlp::SkinningMlp(int n_bones, std::uint64_t seed, const Aabb& domain) : SkinningMlp(n_bones, seed) {
    // condition_input(center, half_extent) (mlp.cpp:230-239): W0.col(j) /= half_j; b0 -= W0 · center
    const int no = widths_[1];
    double* W0 = theta_.data();
    double* b0 = W0 + (size_t)no * 3;
    const Vec3 c = 0.5 * (domain.min + domain.max), h = 0.5 * domain.extent();
    for (int j = 0; j < 3; ++j)
        for (int i = 0; i < no; ++i) W0[(size_t)j * no + i] /= std::max(h[j], 1e-12);
    for (int i = 0; i < no; ++i) b0[i] -= W0[i] * c[0] + W0[(size_t)no + i] * c[1] + W0[(size_t)2 * no + i] * c[2];
}

VectorXd SkinningMlp::weights(const Vec3& x) const {
    const double xv[3] = {x[0], x[1], x[2]};
    std::vector<double> z = mlp_forward(widths_, theta_, xv, nullptr);
    double m = z[0];
    for (double v : z) m = std::max(m, v);
    VectorXd w((int64_t)z.size());
    double sum = 0.0;
    for (size_t i = 0; i < z.size(); ++i) sum += (w[(int64_t)i] = std::exp(z[i] - m));
    for (size_t i = 0; i < z.size(); ++i) w[(int64_t)i] /= sum;
    return w;
}

MatrixXd SkinningMlp::weight_jacobian(const Vec3& x) const {
    const double xv[3] = {x[0], x[1], x[2]};
    std::vector<double> dz;
    mlp_forward(widths_, theta_, xv, &dz);
    const VectorXd w = weights(x);
    const int nb = bone_count();
    MatrixXd J(nb, 3);
    for (int c = 0; c < 3; ++c) {  // softmax head: dw_i = w_i (dz_i - sum_k w_k dz_k)
        double s = 0.0;
        for (int k = 0; k < nb; ++k) s += w[k] * dz[(size_t)k * 3 + c];
        for (int i = 0; i < nb; ++i) J(i, c) = w[i] * (dz[(size_t)i * 3 + c] - s);
    }
    return J;
}

namespace {
struct DevMlp {  // float32 device copy of a network's flat parameters (re-uploaded per call)
    std::vector<float> th;
    std::vector<int32_t> widths;
    std::unique_ptr<DevBuf> buf;
    explicit DevMlp(const SkinningMlp& m) : th(m.parameters().begin(), m.parameters().end()),
                                            widths(m.widths().begin(), m.widths().end()) {
        buf = std::make_unique<DevBuf>(th.size() * sizeof(float));
        h2d(buf->p, th.data(), th.size() * sizeof(float));
    }
};
}  // namespace

SkinningVoxelGrid distill(const SkinningMlp& mlp, GridDims dims, const Aabb& bbox) {
    SkinningVoxelGrid grid(dims, bbox, mlp.bone_count());
    const DevMlp d(mlp);
    const int64_t V = dims.vertex_count();
    DevBuf out(static_cast<size_t>(V) * mlp.bone_count() * sizeof(float));
    const fsk_grid_desc desc = desc_of(dims, bbox, mlp.bone_count());
    check(fsk_distill(ctx(), d.buf->as<float>(), d.widths.data(), (int32_t)d.widths.size(), &desc, out.as<float>(),
                      nullptr));
    std::vector<float> w(static_cast<size_t>(V) * mlp.bone_count());
    d2h(w.data(), out.p, w.size() * sizeof(float));
    std::copy(w.begin(), w.end(), grid.raw().begin());
    return grid;
}

// ------------------------------------------------------------------------ deformer
Affine3 lbs_blend(std::span<const double> weights, std::span<const RigidTransform> bones) {
    if (weights.size() != bones.size()) throw std::invalid_argument("lbs_blend: weight/bone count mismatch");
    Affine3 out = Affine3::zero();
    for (size_t i = 0; i < bones.size(); ++i) {
        out.linear += bones[i].rotation * weights[i];
        out.translation += bones[i].translation * weights[i];
    }
    return out;
}

Vec3 forward_deform(const Vec3& x, const SkinningVoxelGrid& grid, std::span<const RigidTransform> bones) {
    const VectorXd w = trilerp_weights(grid, x);
    return lbs_blend({w.data(), static_cast<size_t>(w.size())}, bones).apply(x);
}

Vec3 forward_deform(const Vec3& x, const SkinningMlp& mlp, std::span<const RigidTransform> bones) {
    const VectorXd w = mlp.weights(x);
    return lbs_blend({w.data(), static_cast<size_t>(w.size())}, bones).apply(x);
}

Mat3 deform_jacobian(const Vec3& x, const SkinningMlp& mlp, std::span<const RigidTransform> bones) {
    const VectorXd w = mlp.weights(x);  // jacobian_from_weights (deformer.cpp:117-141)
    const MatrixXd gw = mlp.weight_jacobian(x);
    Mat3 J = Mat3::Zero();
    for (size_t i = 0; i < bones.size(); ++i) J += w[static_cast<std::int64_t>(i)] * bones[i].rotation;
    for (size_t i = 0; i < bones.size(); ++i) {
        const Vec3 bx = bones[i].apply(x);
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) J(r, c) += bx[r] * gw(static_cast<std::int64_t>(i), c);
    }
    return J;
}

TransformGrid::TransformGrid(GridDims dims, Aabb bbox) : dims_(dims), bbox_(bbox) {
    data_.assign(static_cast<size_t>(dims.vertex_count()) * 12, 0.0);
}

Affine3 TransformGrid::vertex_affine(int i, int j, int k) const {
    const double* m = vertex_transform(vertex_index(i, j, k));
    Affine3 t;
    for (int r = 0; r < 3; ++r) {
        for (int c = 0; c < 3; ++c) t.linear(r, c) = m[r * 4 + c];
        t.translation[r] = m[r * 4 + 3];
    }
    return t;
}

void TransformGrid::set_vertex(std::int64_t v, const Affine3& t) {
    double* m = vertex_transform(v);
    for (int r = 0; r < 3; ++r) {
        for (int c = 0; c < 3; ++c) m[r * 4 + c] = t.linear(r, c);
        m[r * 4 + 3] = t.translation[r];
    }
}

namespace {
std::shared_ptr<void> dev_buffer(size_t bytes) {
    return std::shared_ptr<void>(new DevBuf(bytes), [](void* p) { delete static_cast<DevBuf*>(p); });
}
}  // namespace

void TransformGrid::sync_device() const {
    // caller holds mu_
    const size_t V = static_cast<size_t>(dims_.vertex_count());
    if (!dev_ || !dev64_) {
        dev_ = dev_buffer(V * 12 * sizeof(float));
        dev64_ = dev_buffer(V * 12 * sizeof(double));
        uploaded_.clear();
    }
    if (uploaded_ != data_) {  // host copy changed since the last upload (through any pointer)
        std::vector<float> f(data_.begin(), data_.end());
        h2d(static_cast<DevBuf*>(dev_.get())->p, f.data(), f.size() * sizeof(float));
        h2d(static_cast<DevBuf*>(dev64_.get())->p, data_.data(), data_.size() * sizeof(double));
        uploaded_ = data_;
    }
}

const float* TransformGrid::device_data() const {
    std::lock_guard<std::mutex> lk(mu_);
    sync_device();
    return static_cast<DevBuf*>(dev_.get())->as<float>();
}

const double* TransformGrid::device_data64() const {
    std::lock_guard<std::mutex> lk(mu_);
    sync_device();
    return static_cast<DevBuf*>(dev64_.get())->as<double>();
}

namespace {
/// float32 device copy of a SkinningVoxelGrid's weights (SearchContext::grid), per thread: the
/// search's exact-replay escalation and its initial Jacobians read the weight grid, as the
/// reference's search_one does (correspondence.cpp:43-54). Re-uploaded whenever the grid's values
/// differ from the last upload.
struct WeightsMirror {
    std::vector<float> host;
    std::shared_ptr<void> dev;
    size_t cap = 0;
};

const float* device_weights(const SkinningVoxelGrid& grid) {
    thread_local WeightsMirror m;
    const std::vector<double>& w = grid.raw();
    std::vector<float> f(w.begin(), w.end());
    if (!m.dev || m.cap < f.size()) {
        m.dev = dev_buffer(std::max<size_t>(f.size(), 1) * sizeof(float));
        m.cap = f.size();
        m.host.clear();
    }
    if (f != m.host) {
        h2d(static_cast<DevBuf*>(m.dev.get())->p, f.data(), f.size() * sizeof(float));
        m.host = std::move(f);
    }
    return static_cast<DevBuf*>(m.dev.get())->as<float>();
}
}  // namespace

// K1 on the GPU in float32 (the fast search's grid) and float64 (the reference's
// TransformGrid precision: the host copy and the float64 re-solves read it).
TransformGrid precompute_transform_grid(const SkinningVoxelGrid& grid, std::span<const RigidTransform> bones, int) {
    if (static_cast<int>(bones.size()) != grid.bone_count())
        throw std::invalid_argument("precompute_transform_grid: bone count mismatch");
    TransformGrid tg(grid.dims(), grid.bbox());
    const std::int64_t V = grid.dims().vertex_count();
    const int nb = grid.bone_count();
    const std::vector<float> b = bones_f32(bones);
    const float* dw = device_weights(grid);
    DevBuf db(b.size() * sizeof(float));
    tg.dev_ = dev_buffer(static_cast<size_t>(V) * 12 * sizeof(float));
    tg.dev64_ = dev_buffer(static_cast<size_t>(V) * 12 * sizeof(double));
    h2d(db.p, b.data(), b.size() * sizeof(float));
    const fsk_grid_desc d = desc_of(grid.dims(), grid.bbox(), nb);
    check(fsk_precompute_tgrid(ctx(), dw, &d, db.as<float>(), nb, static_cast<DevBuf*>(tg.dev_.get())->as<float>(),
                               static_cast<DevBuf*>(tg.dev64_.get())->as<double>(), nullptr));
    // the float64 host copy through pinned staging (a pageable D2H of V·96 B is several times slower)
    thread_local struct Pinned {
        void* p = nullptr;
        size_t cap = 0;
        ~Pinned() {
            if (p) cudaFreeHost(p);
        }
    } stage;
    const size_t bytes = tg.data_.size() * sizeof(double);
    if (stage.cap < bytes) {
        if (stage.p) cudaFreeHost(stage.p);
        stage.p = nullptr;
        stage.cap = 0;
        cuda_ok(cudaMallocHost(&stage.p, bytes), "cudaMallocHost");
        stage.cap = bytes;
    }
    cuda_ok(cudaMemcpy(stage.p, static_cast<DevBuf*>(tg.dev64_.get())->p, bytes, cudaMemcpyDeviceToHost), "D2H tgrid");
    std::memcpy(tg.data_.data(), stage.p, bytes);
    tg.uploaded_ = tg.data_;
    return tg;
}

namespace {
void eval_batch(const TransformGrid& tg, std::span<const Vec3> x, float* t12, float* d, float* jac) {
    const size_t n = x.size();
    const std::vector<float> p = points_f32(x);
    DevBuf dx(p.size() * sizeof(float)), dt(n * 12 * sizeof(float)), dd(n * 3 * sizeof(float)), dj(n * 9 * sizeof(float));
    h2d(dx.p, p.data(), p.size() * sizeof(float));
    const fsk_grid_desc desc = desc_of(tg.dims(), tg.bbox(), 1);
    check(fsk_eval_points(ctx(), tg.device_data(), &desc, dx.as<float>(), static_cast<std::int64_t>(n),
                          t12 ? dt.as<float>() : nullptr, d ? dd.as<float>() : nullptr, jac ? dj.as<float>() : nullptr,
                          nullptr));
    if (t12) d2h(t12, dt.p, n * 12 * sizeof(float));
    if (d) d2h(d, dd.p, n * 3 * sizeof(float));
    if (jac) d2h(jac, dj.p, n * 9 * sizeof(float));
}
}  // namespace

// Single-point host evaluation of the float64 host copy (deformer.cpp:79-94): corners in (dk, dj, di)
// order, each of the 12 entries accumulated corner by corner.
void trilerp_transform_into(const TransformGrid& tgrid, const Vec3& x, double* out12) {
    const CellLocator c = locate_cell(tgrid.dims(), tgrid.bbox(), x);
    for (int e = 0; e < 12; ++e) out12[e] = 0.0;
    for (int dk = 0; dk < 2; ++dk) {
        const double fz = dk ? c.tz : 1.0 - c.tz;
        for (int dj = 0; dj < 2; ++dj) {
            const double fyz = fz * (dj ? c.ty : 1.0 - c.ty);
            for (int di = 0; di < 2; ++di) {
                const double f = fyz * (di ? c.tx : 1.0 - c.tx);
                const double* t = tgrid.vertex_transform(tgrid.vertex_index(c.i0 + di, c.j0 + dj, c.k0 + dk));
                for (int e = 0; e < 12; ++e) out12[e] += f * t[e];
            }
        }
    }
}

Affine3 trilerp_transform(const TransformGrid& tgrid, const Vec3& x) {
    double m[12];
    trilerp_transform_into(tgrid, x, m);
    Affine3 t;
    for (int r = 0; r < 3; ++r) {
        for (int c = 0; c < 3; ++c) t.linear(r, c) = m[r * 4 + c];
        t.translation[r] = m[r * 4 + 3];
    }
    return t;
}

std::vector<Vec3> forward_deform_batch(std::span<const Vec3> x, const TransformGrid& tgrid) {
    std::vector<float> d(x.size() * 3);
    if (!x.empty()) eval_batch(tgrid, x, nullptr, d.data(), nullptr);
    std::vector<Vec3> out(x.size());
    for (size_t i = 0; i < x.size(); ++i) out[i] = Vec3(d[3 * i], d[3 * i + 1], d[3 * i + 2]);
    return out;
}

// d = T(x)·[x;1] on the unclamped x (deformer.cpp:107-113), float64 host copy
Vec3 forward_deform(const Vec3& x, const TransformGrid& tgrid) {
    double m[12];
    trilerp_transform_into(tgrid, x, m);
    Vec3 d;
    for (int r = 0; r < 3; ++r) d[r] = m[4 * r] * x[0] + m[4 * r + 1] * x[1] + m[4 * r + 2] * x[2] + m[4 * r + 3];
    return d;
}

std::vector<Mat3> deform_jacobian_batch(std::span<const Vec3> x, const TransformGrid& tgrid) {
    std::vector<float> j(x.size() * 9);
    if (!x.empty()) eval_batch(tgrid, x, nullptr, nullptr, j.data());
    std::vector<Mat3> out(x.size());
    for (size_t i = 0; i < x.size(); ++i)
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) out[i](r, c) = j[9 * i + 3 * r + c];
    return out;
}

// J = Σ_i w_i R_i + Σ_i (B_i x)(∇w_i)ᵀ in bone order (deformer.cpp:117-136), float64 on the host
Mat3 deform_jacobian(const Vec3& x, const SkinningVoxelGrid& grid, std::span<const RigidTransform> bones) {
    const VectorXd w = trilerp_weights(grid, x);
    const MatrixXd gw = weight_spatial_gradient(grid, x);
    Mat3 J = Mat3::Zero();
    for (size_t i = 0; i < bones.size(); ++i) J += w[static_cast<std::int64_t>(i)] * bones[i].rotation;
    for (size_t i = 0; i < bones.size(); ++i) {
        const Vec3 bx = bones[i].apply(x);
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) J(r, c) += bx[r] * gw(static_cast<std::int64_t>(i), c);
    }
    return J;
}

// ------------------------------------------------------------------------ correspondence
SearchOptions SearchOptions::defaults_for(const Aabb& bbox) {
    const double diag = bbox.diagonal();
    SearchOptions o;
    o.conv_eps = 1e-5 * diag;
    o.div_eps = 0.5 * diag;
    o.dedup_dist = 1e-2 * diag;
    return o;
}

void SearchOptions::validate() const {
    if (max_iters < 1) throw std::invalid_argument("search: max_iters must be >= 1");
    if (!(conv_eps > 0.0)) throw std::invalid_argument("search: conv_eps must be > 0");
    if (!(div_eps > conv_eps)) throw std::invalid_argument("search: div_eps must exceed conv_eps");
    if (!(dedup_dist >= 0.0)) throw std::invalid_argument("search: dedup_dist must be >= 0");
}

// init_states (correspondence.cpp:58-70) on the GPU in float64 with the reference's operation order
// (fsk_init_states64: x0 = B_i^-1 x', J~0 from the weight grid's Jacobian) — the oracle's values.
std::vector<InitState> init_states(const Vec3& x_prime, const SearchContext& c, SearchVariant variant) {
    check_context(c, variant);
    const int nb = static_cast<int>(c.bones.size());
    if (variant == SearchVariant::Mlp) {  // float64 host: J from the network's input tangents (:43-54)
        std::vector<InitState> out(nb);
        for (int i = 0; i < nb; ++i) {
            out[i].x0 = c.bones[i].inverse().apply(x_prime);
            const Mat3 J = deform_jacobian(out[i].x0, *c.mlp, c.bones);
            out[i].inv_jacobian = std::abs(J.determinant()) < 1e-8 ? Mat3::Identity() : J.inverse();
        }
        return out;
    }
    const std::vector<float> b = bones_f32(c.bones);
    const double p[3] = {x_prime[0], x_prime[1], x_prime[2]};
    const float* dw = device_weights(*c.grid);
    DevBuf db(b.size() * 4), dp(sizeof(p)), dx(nb * 3 * sizeof(double)), dj(nb * 9 * sizeof(double));
    h2d(db.p, b.data(), b.size() * 4);
    h2d(dp.p, p, sizeof(p));
    const fsk_grid_desc d = desc_of(c.grid->dims(), c.grid->bbox(), nb);
    check(fsk_init_states64(ctx(), dw, &d, db.as<float>(), nb, dp.as<double>(), 1, dx.as<double>(), dj.as<double>(),
                            nullptr));
    std::vector<double> x0(nb * 3), j0(nb * 9);
    d2h(x0.data(), dx.p, x0.size() * sizeof(double));
    d2h(j0.data(), dj.p, j0.size() * sizeof(double));
    std::vector<InitState> out(nb);
    for (int i = 0; i < nb; ++i) {
        out[i].x0 = Vec3(x0[3 * i], x0[3 * i + 1], x0[3 * i + 2]);
        for (int r = 0; r < 3; ++r)
            for (int q = 0; q < 3; ++q) out[i].inv_jacobian(r, q) = j0[9 * i + 3 * r + q];
    }
    return out;
}

namespace {
void fill_set(CorrespondenceSet& set, const Vec3& query, std::span<const std::int64_t> h_offs,
              std::span<const fsk_root> roots, int64_t q);

std::vector<CorrespondenceSet> to_sets(std::span<const Vec3> queries, std::span<const std::int64_t> h_offs,
                                       std::span<const fsk_root> roots) {
    std::vector<CorrespondenceSet> out(queries.size());
    // the reference's batch_search builds its sets inside parallel_for's workers: so does this, over the
    // host cores (contiguous query ranges; the result does not depend on the split)
    const int64_t n = static_cast<int64_t>(queries.size());
    const int T = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(std::thread::hardware_concurrency(), n / 8192)));
    auto fill = [&](int64_t q0, int64_t q1) {
        for (int64_t q = q0; q < q1; ++q) fill_set(out[static_cast<size_t>(q)], queries[q], h_offs, roots, q);
    };
    if (T == 1) {
        fill(0, n);
    } else {
        std::vector<std::thread> pool;
        for (int t = 0; t < T; ++t) pool.emplace_back(fill, n * t / T, n * (t + 1) / T);
        for (auto& th : pool) th.join();
    }
    return out;
}

void fill_set(CorrespondenceSet& set, const Vec3& query, std::span<const std::int64_t> h_offs,
              std::span<const fsk_root> roots, int64_t q) {
    {
        set.query = query;
        set.roots.reserve(static_cast<size_t>(h_offs[q + 1] - h_offs[q]));
        for (std::int64_t k = h_offs[q]; k < h_offs[q + 1]; ++k) {
            const fsk_root& r = roots[static_cast<size_t>(k)];
            Root root;
            root.x = Vec3(r.x[0], r.x[1], r.x[2]);
            root.residual = r.residual;
            for (int a = 0; a < 3; ++a)
                for (int e = 0; e < 3; ++e) root.inv_jacobian(a, e) = r.inv_jacobian[3 * a + e];
            root.source_bone = r.source_bone;
            root.iterations = r.iterations;
            set.roots.push_back(root);
        }
    }
}
}  // namespace

// The voxel search through the per-thread workspace: queries converted into pinned staging, one H2D,
// fsk_batch_search, D2H of offsets and kept roots into pinned staging, CorrespondenceSets built from it.
std::vector<CorrespondenceSet> batch_search_voxel(std::span<const Vec3> queries, const SearchContext& c,
                                                  const fsk_grid_desc& d, const fsk_search_opts& so, const float* dw) {
    thread_local Workspace w;
    const std::int64_t n = static_cast<std::int64_t>(queries.size());
    const int nb = static_cast<int>(c.bones.size());
    const std::vector<float> b = bones_f32(c.bones);
    float* hp = static_cast<float*>(w.h(0, n * 3 * sizeof(float)));
    for (std::int64_t i = 0; i < n; ++i)
        for (int a = 0; a < 3; ++a) hp[3 * i + a] = static_cast<float>(queries[i][a]);
    float* dp = static_cast<float*>(w.d(0, n * 3 * sizeof(float)));
    float* db = static_cast<float*>(w.d(1, b.size() * sizeof(float)));
    std::int64_t* doffs = static_cast<std::int64_t*>(w.d(2, (n + 1) * sizeof(std::int64_t)));
    std::int64_t* hoffs = static_cast<std::int64_t*>(w.h(1, (n + 1) * sizeof(std::int64_t)));
    cuda_ok(cudaMemcpyAsync(dp, hp, n * 3 * sizeof(float), cudaMemcpyHostToDevice, 0), "H2D points");
    h2d(db, b.data(), b.size() * sizeof(float));
    std::int64_t cap = std::min<std::int64_t>(n * nb, 4 * n);  // count-then-allocate: ~1.05 roots are kept per query
    std::vector<std::int64_t> h_offs;
    for (int attempt = 0; attempt < 2; ++attempt) {
        fsk_root* dr = static_cast<fsk_root*>(w.d(3, cap * sizeof(fsk_root)));
        check(fsk_batch_search(ctx(), c.tgrid->device_data(), c.tgrid->device_data64(), dw, &d, db, nb, dp, n, &so,
                               doffs, dr, cap, nullptr));
        cuda_ok(cudaMemcpyAsync(hoffs, doffs, (n + 1) * sizeof(std::int64_t), cudaMemcpyDeviceToHost, 0), "D2H offsets");
        cuda_ok(cudaStreamSynchronize(0), "cudaStreamSynchronize");
        const std::int64_t total = hoffs[n];
        if (total > cap) {  // more kept roots than records: search again into exactly that many
            cap = total;
            continue;
        }
        fsk_root* hr = static_cast<fsk_root*>(w.h(2, std::max<std::int64_t>(1, total) * sizeof(fsk_root)));
        if (total > 0) {
            cuda_ok(cudaMemcpyAsync(hr, dr, total * sizeof(fsk_root), cudaMemcpyDeviceToHost, 0), "D2H roots");
            cuda_ok(cudaStreamSynchronize(0), "cudaStreamSynchronize");
        }
        return to_sets(queries, std::span<const std::int64_t>(hoffs, n + 1), std::span<const fsk_root>(hr, total));
    }
    throw std::runtime_error("fsk: root count changed between identical searches");
}

// batch_search (correspondence.cpp:178-192) on the GPU. Voxel variant: K1's grids (the TransformGrid's
// device mirrors), SearchContext::grid's weights for J~0 and the float64 replay, K2 + dedup + compaction;
// root records count-then-allocate (4 per query first, the exact count on a rerun). Mlp variant: the
// network at every Broyden iterate on the tensor cores (fsk_search_fwd_mlp), compacted likewise.
std::vector<CorrespondenceSet> batch_search(std::span<const Vec3> queries, const SearchContext& c,
                                            const SearchOptions& opts, int) {
    check_context(c, opts.variant);
    opts.validate();
    const std::int64_t n = static_cast<std::int64_t>(queries.size());
    if (n == 0) {
        const std::int64_t zero = 0;
        return to_sets(queries, {&zero, 1}, {});
    }
    const int nb = static_cast<int>(c.bones.size());
    const fsk_search_opts so = c_opts(opts);
    if (opts.variant == SearchVariant::Mlp) {
        const std::vector<float> b = bones_f32(c.bones);
        const std::vector<float> p = points_f32(queries);
        DevBuf db(b.size() * 4), dp(p.size() * 4), offs((n + 1) * 8);
        h2d(db.p, b.data(), b.size() * 4);
        h2d(dp.p, p.data(), p.size() * 4);
        std::vector<std::int64_t> h_offs(n + 1);
        std::vector<fsk_root> roots;
        const DevMlp net(*c.mlp);
        DevBuf xc(n * nb * 12), ji(n * nb * 36), rs(n * nb * 4), it(n * nb * 4), cv(n * nb), kp(n * nb), nr(n * 4);
        fsk_search_out o{xc.as<float>(), ji.as<float>(), rs.as<float>(), it.as<std::int32_t>(), cv.as<std::uint8_t>(),
                         kp.as<std::uint8_t>(), nr.as<std::int32_t>(), nullptr};
        check(fsk_search_fwd_mlp(ctx(), net.buf->as<float>(), net.widths.data(), (int32_t)net.widths.size(),
                                 db.as<float>(), nb, dp.as<float>(), n, &so, &o, nullptr));
        std::int64_t total = 0;
        const int rc = fsk_compact_roots(ctx(), &o, n, nb, offs.as<std::int64_t>(), nullptr, 0, &total, nullptr);
        if (rc != FSK_OK && total == 0) check(rc);
        DevBuf dr(std::max<std::int64_t>(1, total) * sizeof(fsk_root));
        check(fsk_compact_roots(ctx(), &o, n, nb, offs.as<std::int64_t>(), dr.as<fsk_root>(), total, &total, nullptr));
        d2h(h_offs.data(), offs.p, h_offs.size() * 8);
        roots.resize(static_cast<size_t>(total));
        if (total > 0) d2h(roots.data(), dr.p, roots.size() * sizeof(fsk_root));
        return to_sets(queries, h_offs, roots);
    }
    const fsk_grid_desc d = desc_of(c.tgrid->dims(), c.tgrid->bbox(), nb);
    // SearchContext::grid's weights go to the search like the reference's (J~0 from the weight grid,
    // correspondence.cpp:43-54): the escalated solves then replay the reference's operation order
    const float* dw = device_weights(*c.grid);
    return batch_search_voxel(queries, c, d, so, dw);
}

CorrespondenceSet broyden_search(const Vec3& x_prime, const SearchContext& c, const SearchOptions& opts) {
    return batch_search({&x_prime, 1}, c, opts)[0];
}

// ------------------------------------------------------------------------ implicit differentiation
SingularRootError::SingularRootError(double det)
    : std::runtime_error("implicit gradient: deformation Jacobian is singular (det " + std::to_string(det) + ")") {}

Vec3 implicit_cotangent_exact(const Vec3& x_star, const SkinningVoxelGrid& grid, std::span<const RigidTransform> bones,
                              const Vec3& cotangent) {
    if (static_cast<int>(bones.size()) != grid.bone_count()) throw std::invalid_argument("deform vjp: bone count mismatch");
    const std::vector<float> b = bones_f32(bones);
    const float xv[6] = {static_cast<float>(x_star[0]), static_cast<float>(x_star[1]), static_cast<float>(x_star[2]),
                         static_cast<float>(cotangent[0]), static_cast<float>(cotangent[1]),
                         static_cast<float>(cotangent[2])};
    const float* dw = device_weights(grid);
    DevBuf db(b.size() * 4), dx(sizeof(xv)), du(3 * sizeof(double)), dok(1), ddet(sizeof(double));
    h2d(db.p, b.data(), b.size() * 4);
    h2d(dx.p, xv, sizeof(xv));
    const fsk_grid_desc d = desc_of(grid.dims(), grid.bbox(), grid.bone_count());
    check(fsk_implicit_u_exact(ctx(), dw, &d, db.as<float>(), grid.bone_count(), dx.as<float>(), dx.as<float>() + 3, 1,
                               du.as<double>(), dok.as<std::uint8_t>(), ddet.as<double>(), nullptr));
    double u[3], det;
    std::uint8_t ok;
    d2h(u, du.p, sizeof(u));
    d2h(&ok, dok.p, 1);
    d2h(&det, ddet.p, sizeof(det));
    if (!ok) throw SingularRootError(det);
    return Vec3(u[0], u[1], u[2]);
}

Vec3 implicit_cotangent_approx(const Mat3& inv_jacobian, const Vec3& cotangent) {
    return -(inv_jacobian.transpose() * cotangent);
}

GridGradient implicit_grad_grid(std::span<const CorrespondenceSet> sets, std::span<const int> root_of_query,
                                std::span<const Vec3> cotangents, const SkinningVoxelGrid& grid,
                                std::span<const RigidTransform> bones, bool exact) {
    const std::int64_t n = static_cast<std::int64_t>(sets.size());
    if (root_of_query.size() != sets.size() || cotangents.size() != sets.size())
        throw std::invalid_argument("implicit_grad_grid: one root index and one cotangent per query");
    const int nb = grid.bone_count();
    if (static_cast<int>(bones.size()) != nb) throw std::invalid_argument("deform vjp: bone count mismatch");
    std::vector<fsk_root> recs;
    std::vector<std::int64_t> ridx(static_cast<size_t>(n), -1);
    std::vector<float> v(static_cast<size_t>(3 * n));
    for (std::int64_t q = 0; q < n; ++q) {
        for (int a = 0; a < 3; ++a) v[3 * q + a] = static_cast<float>(cotangents[q][a]);
        const int k = root_of_query[q];
        if (k < 0) continue;
        if (k >= static_cast<int>(sets[q].roots.size())) throw std::invalid_argument("implicit_grad_grid: root index out of range");
        const Root& r = sets[q].roots[k];
        fsk_root f{};
        for (int a = 0; a < 3; ++a) f.x[a] = static_cast<float>(r.x[a]);
        f.residual = static_cast<float>(r.residual);
        for (int a = 0; a < 3; ++a)
            for (int e = 0; e < 3; ++e) f.inv_jacobian[3 * a + e] = static_cast<float>(r.inv_jacobian(a, e));
        f.source_bone = r.source_bone;
        f.iterations = r.iterations;
        ridx[q] = static_cast<std::int64_t>(recs.size());
        recs.push_back(f);
    }
    const std::int64_t V = grid.dims().vertex_count();
    const std::vector<float> b = bones_f32(bones);
    const float* dw = exact ? device_weights(grid) : nullptr;
    DevBuf db(b.size() * 4), dr(std::max<size_t>(recs.size(), 1) * sizeof(fsk_root)), di(ridx.size() * 8 + 8),
        dv(v.size() * 4 + 4), dT(static_cast<size_t>(V) * 12 * sizeof(float)), dW(static_cast<size_t>(V) * nb * sizeof(float)),
        dok(static_cast<size_t>(n) + 1);
    h2d(db.p, b.data(), b.size() * 4);
    h2d(dr.p, recs.data(), recs.size() * sizeof(fsk_root));
    h2d(di.p, ridx.data(), ridx.size() * 8);
    h2d(dv.p, v.data(), v.size() * 4);
    const fsk_grid_desc d = desc_of(grid.dims(), grid.bbox(), nb);
    if (exact)
        check(fsk_search_bwd_exact_roots(ctx(), dw, &d, db.as<float>(), nb, dr.as<fsk_root>(), di.as<std::int64_t>(),
                                         dv.as<float>(), n, dT.as<float>(), dok.as<std::uint8_t>(), 1, nullptr));
    else
        check(fsk_search_bwd_roots(ctx(), &d, dr.as<fsk_root>(), di.as<std::int64_t>(), dv.as<float>(), n, dT.as<float>(),
                                   1, nullptr));
    check(fsk_grad_weights(ctx(), &d, dT.as<float>(), db.as<float>(), nb, dW.as<float>(), nullptr));
    std::vector<float> t(static_cast<size_t>(V) * 12), w(static_cast<size_t>(V) * nb);
    d2h(t.data(), dT.p, t.size() * 4);
    d2h(w.data(), dW.p, w.size() * 4);
    GridGradient out;
    out.d_tgrid.assign(t.begin(), t.end());
    out.d_weights.assign(w.begin(), w.end());
    if (exact && n > 0) {
        std::vector<std::uint8_t> ok(static_cast<size_t>(n));
        d2h(ok.data(), dok.p, ok.size());
        for (std::int64_t q = 0; q < n; ++q) out.skipped += (ridx[q] >= 0 && !ok[q]) ? 1 : 0;
    }
    return out;
}

std::vector<Root> dedup_roots(std::vector<Root> roots, double dedup_dist) {
    std::vector<Root> kept;
    kept.reserve(roots.size());
    for (Root& r : roots) {
        bool dup = false;
        for (const Root& k : kept)
            if ((r.x - k.x).norm() < dedup_dist) {
                dup = true;
                break;
            }
        if (!dup) kept.push_back(std::move(r));
    }
    return kept;
}

}  // namespace fskin
