// ORACLE — TEST INFRASTRUCTURE ONLY. Not part of the product (see fskin_oracle.cpp).
//
// Double-precision restatement of the reference's MLP stages next to the deformer hot path
// (SURVEY §8(f) rows 1 and 2):
//   * Mlp::forward / backward with softplus hidden units and a linear head
//     (proj/src/mlp.cpp:115-163), softplus / sigmoid / softmax / softmax_vjp (:10-45),
//     parameter order of Mlp::parameters() (:207-219: per layer W column-major, then b);
//   * distill(SkinningMlp, dims, bbox) (proj/src/skinning.cpp:195-221) with
//     SkinningMlp::weights_batch (:47-51) and SkinningVoxelGrid::vertex_position (:77-80);
//   * the VJP of distill: dL/dtheta = sum_v backward(softmax_vjp(w_v, dL/dw_v)) — the chain the
//     training step takes through the skinning network (diff.cpp:348-359, with the grid
//     vertices in place of the roots);
//   * OccupancyMlp::occupancy_batch (proj/src/shape.cpp:218-228) and posed_occupancy_batch
//     (:242-269): max over each query's roots, first root wins ties, argmax -1 when empty.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace orc_mlp {

thread_local std::string g_err;

double softplus(double x) { return std::max(x, 0.0) + std::log1p(std::exp(-std::abs(x))); }  // mlp.cpp:10-13
double sigmoid(double x) {                                                                     // mlp.cpp:15-21
    if (x >= 0.0) return 1.0 / (1.0 + std::exp(-x));
    const double e = std::exp(x);
    return e / (1.0 + e);
}
void softmax_inplace(double* z, int n) {  // mlp.cpp:32-36
    double m = z[0];
    for (int i = 1; i < n; ++i) m = std::max(m, z[i]);
    double s = 0.0;
    for (int i = 0; i < n; ++i) {
        z[i] = std::exp(z[i] - m);
        s += z[i];
    }
    for (int i = 0; i < n; ++i) z[i] /= s;
}

struct Net {
    std::vector<int> w;                      // widths
    std::vector<const double*> W, b;         // W[l]: (w[l+1] x w[l]) column-major
    Net(const double* theta, const int* widths, int nw) : w(widths, widths + nw) {
        if (nw < 2) throw std::invalid_argument("Mlp: need at least input and output widths");
        const double* p = theta;
        for (int l = 0; l + 1 < nw; ++l) {
            W.push_back(p);
            p += (int64_t)w[l + 1] * w[l];
            b.push_back(p);
            p += w[l + 1];
        }
    }
    int layers() const { return (int)W.size(); }
    double Wat(int l, int r, int c) const { return W[l][(int64_t)c * w[l + 1] + r]; }
    // forward of one input column (mlp.cpp:115-138); pre/act kept for backward
    void forward(const double* x, std::vector<std::vector<double>>& pre, std::vector<std::vector<double>>& act) const {
        pre.assign(layers(), {});
        act.assign(layers(), {});
        std::vector<double> h(x, x + w[0]);
        for (int l = 0; l < layers(); ++l) {
            std::vector<double> z(w[l + 1]);
            for (int r = 0; r < w[l + 1]; ++r) {
                double s = 0.0;
                for (int c = 0; c < w[l]; ++c) s += Wat(l, r, c) * h[c];
                z[r] = s + b[l][r];
            }
            pre[l] = z;
            if (l + 1 < layers()) {
                for (auto& v : z) v = softplus(v);
                act[l] = z;
            }
            h = z;
        }
    }
    // backward of one column (mlp.cpp:140-163): accumulates dtheta
    void backward(const double* x, const std::vector<std::vector<double>>& pre,
                  const std::vector<std::vector<double>>& act, std::vector<double> delta, double* dtheta) const {
        std::vector<int64_t> off(layers());
        int64_t o = 0;
        for (int l = 0; l < layers(); ++l) {
            off[l] = o;
            o += (int64_t)w[l + 1] * w[l] + w[l + 1];
        }
        for (int l = layers() - 1; l >= 0; --l) {
            const double* in = l == 0 ? x : act[l - 1].data();
            double* dW = dtheta + off[l];
            double* db = dW + (int64_t)w[l + 1] * w[l];
            for (int c = 0; c < w[l]; ++c)
                for (int r = 0; r < w[l + 1]; ++r) dW[(int64_t)c * w[l + 1] + r] += delta[r] * in[c];
            for (int r = 0; r < w[l + 1]; ++r) db[r] += delta[r];
            if (l == 0) break;
            std::vector<double> d(w[l]);
            for (int c = 0; c < w[l]; ++c) {
                double s = 0.0;
                for (int r = 0; r < w[l + 1]; ++r) s += Wat(l, r, c) * delta[r];
                d[c] = s * sigmoid(pre[l - 1][c]);  // softplus' = sigmoid(pre)
            }
            delta = std::move(d);
        }
    }
    int64_t n_params() const {
        int64_t n = 0;
        for (int l = 0; l < layers(); ++l) n += (int64_t)w[l + 1] * w[l] + w[l + 1];
        return n;
    }
};

template <typename F>
void parallel_for(int64_t n, int workers, F&& f) {  // parallel.hpp:17-33 (contiguous ranges)
    workers = std::max(1, std::min<int>(workers, (int)std::max<int64_t>(1, n)));
    std::vector<std::thread> pool;
    for (int t = 0; t < workers; ++t) pool.emplace_back([&, t] { f(n * t / workers, n * (t + 1) / workers, t); });
    for (auto& th : pool) th.join();
}

void vertex_position(int64_t v, int nx, int ny, int nz, const double* bbox6, double* x) {  // skinning.cpp:72-80
    const int64_t i = v % nx, j = (v / nx) % ny, k = v / ((int64_t)nx * ny);
    const int n[3] = {nx, ny, nz};
    const int64_t id[3] = {i, j, k};
    for (int a = 0; a < 3; ++a) x[a] = bbox6[a] + (double)id[a] * ((bbox6[3 + a] - bbox6[a]) / (n[a] - 1));
}

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

}  // namespace orc_mlp

using namespace orc_mlp;

extern "C" {

const char* orc_mlp_last_error(void) { return g_err.c_str(); }

// Mlp::forward on a row-major batch X [B][in] -> out [B][out] (mlp.cpp:115-138)
int orc_mlp_forward(const double* theta, const int* widths, int nw, const double* X, int64_t B, double* out,
                    int workers) {
    return guard([&] {
        const Net net(theta, widths, nw);
        parallel_for(B, workers, [&](int64_t b0, int64_t b1, int) {
            std::vector<std::vector<double>> pre, act;
            for (int64_t p = b0; p < b1; ++p) {
                net.forward(X + p * widths[0], pre, act);
                std::copy(pre.back().begin(), pre.back().end(), out + p * widths[nw - 1]);
            }
        });
    });
}

// distill (skinning.cpp:195-221): weights [V][nb] = softmax(net(vertex_position(v)))
int orc_distill(const double* theta, const int* widths, int nw, int nx, int ny, int nz, const double* bbox6,
                double* weights, int workers) {
    return guard([&] {
        if (nx < 2 || ny < 2 || nz < 2) throw std::invalid_argument("distill: dims must be >= 2 per axis");
        if (widths[0] != 3) throw std::invalid_argument("SkinningMlp: network input width must be 3");
        const Net net(theta, widths, nw);
        const int nb = widths[nw - 1];
        parallel_for((int64_t)nx * ny * nz, workers, [&](int64_t v0, int64_t v1, int) {
            std::vector<std::vector<double>> pre, act;
            for (int64_t v = v0; v < v1; ++v) {
                double x[3];
                vertex_position(v, nx, ny, nz, bbox6, x);
                net.forward(x, pre, act);
                std::vector<double> z = pre.back();
                softmax_inplace(z.data(), nb);
                std::copy(z.begin(), z.end(), weights + v * nb);
            }
        });
    });
}

// VJP of distill: dtheta = sum_v backward(softmax_vjp(w_v, dw_v)) (mlp.cpp:38-41, :140-163)
int orc_distill_vjp(const double* theta, const int* widths, int nw, int nx, int ny, int nz, const double* bbox6,
                    const double* dw, double* dtheta, int workers) {
    return guard([&] {
        const Net net(theta, widths, nw);
        const int nb = widths[nw - 1];
        const int64_t P = net.n_params();
        workers = std::max(1, workers);
        std::vector<std::vector<double>> part(workers, std::vector<double>(P, 0.0));
        parallel_for((int64_t)nx * ny * nz, workers, [&](int64_t v0, int64_t v1, int t) {
            std::vector<std::vector<double>> pre, act;
            for (int64_t v = v0; v < v1; ++v) {
                double x[3];
                vertex_position(v, nx, ny, nz, bbox6, x);
                net.forward(x, pre, act);
                std::vector<double> w = pre.back();
                softmax_inplace(w.data(), nb);
                double dot = 0.0;
                for (int i = 0; i < nb; ++i) dot += w[i] * dw[v * nb + i];
                std::vector<double> dz(nb);
                for (int i = 0; i < nb; ++i) dz[i] = w[i] * (dw[v * nb + i] - dot);
                net.backward(x, pre, act, dz, part[t].data());
            }
        });
        for (int64_t i = 0; i < P; ++i) {
            double s = 0.0;
            for (int t = 0; t < workers; ++t) s += part[t][i];
            dtheta[i] = s;
        }
    });
}

// posed_occupancy_batch (shape.cpp:242-269) over CorrespondenceSets given as offsets [n+1]
// and root positions [M][3]; the network input is (x, pose) (occupancy_batch, :218-228).
int orc_posed_occupancy(const double* theta, const int* widths, int nw, const double* pose, int n_pose,
                        const int64_t* offsets, const double* roots_x, int64_t n, double* pred, int32_t* argmax,
                        int workers) {
    return guard([&] {
        const Net net(theta, widths, nw);
        if (widths[0] < 3 || widths[nw - 1] != 1)
            throw std::invalid_argument("occupancy mlp: expected input >= 3, scalar output");
        if (n_pose != widths[0] - 3)
            throw std::invalid_argument("occupancy mlp: pose vector length " + std::to_string(n_pose) +
                                        ", field conditioned on " + std::to_string(widths[0] - 3));
        parallel_for(n, workers, [&](int64_t q0, int64_t q1, int) {
            std::vector<std::vector<double>> pre, act;
            std::vector<double> in(widths[0]);
            for (int64_t q = q0; q < q1; ++q) {
                pred[q] = 0.0;
                argmax[q] = -1;
                bool first = true;
                for (int64_t r = offsets[q]; r < offsets[q + 1]; ++r) {
                    for (int a = 0; a < 3; ++a) in[a] = roots_x[3 * r + a];
                    for (int a = 0; a < n_pose; ++a) in[3 + a] = pose[a];
                    net.forward(in.data(), pre, act);
                    const double occ = sigmoid(pre.back()[0]);
                    if (first || occ > pred[q]) {
                        pred[q] = occ;
                        argmax[q] = (int32_t)(r - offsets[q]);
                        first = false;
                    }
                }
            }
        });
    });
}

}  // extern "C"
