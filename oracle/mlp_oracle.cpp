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
//   * the MLP variant of the search (SearchVariant::Mlp): eval_deform via
//     forward_deform(x, mlp, bones) (deformer.cpp:22-26, correspondence.cpp:77-79), the initial
//     Jacobian deform_jacobian(x, mlp, bones) (deformer.cpp:117-141) with
//     SkinningMlp::weight_jacobian (skinning.cpp:53-64, Mlp::input_tangent mlp.cpp:142-155),
//     iterate (correspondence.cpp:97-124), search_one / dedup_roots (:126-176).
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
    // weights w = softmax(net(x)) and dw/dx [nb][3] (SkinningMlp::weight_jacobian,
    // skinning.cpp:53-64: Mlp::input_tangent then the softmax Jacobian)
    void weights_and_jacobian(const double* x, std::vector<double>& w, std::vector<double>& dw) const {
        std::vector<std::vector<double>> pre, act;
        forward(x, pre, act);
        const int nb = w_out();
        w = pre.back();
        softmax_inplace(w.data(), nb);
        dw.assign((size_t)nb * 3, 0.0);
        for (int c = 0; c < 3; ++c) {
            std::vector<double> t(this->w[0], 0.0);
            t[c] = 1.0;
            for (int l = 0; l < layers(); ++l) {
                std::vector<double> u(this->w[l + 1]);
                for (int r = 0; r < this->w[l + 1]; ++r) {
                    double acc = 0.0;
                    for (int k = 0; k < this->w[l]; ++k) acc += Wat(l, r, k) * t[k];
                    u[r] = acc;
                }
                if (l + 1 < layers())
                    for (int r = 0; r < this->w[l + 1]; ++r) u[r] *= sigmoid(pre[l][r]);
                t = std::move(u);
            }
            double dot = 0.0;
            for (int i = 0; i < nb; ++i) dot += w[i] * t[i];
            for (int i = 0; i < nb; ++i) dw[(size_t)i * 3 + c] = w[i] * (t[i] - dot);
        }
    }
    int w_out() const { return w.back(); }
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

// ---------------------------------------------------------------- MLP-variant search
namespace {
struct MB {  // rigid bone [R|t] (row-major 3x4)
    double R[9], t[3];
};
// forward_deform(x, mlp, bones) = lbs_blend(w(x), B)·x (deformer.cpp:9-19, :22-26)
void mlp_deform(const Net& net, const std::vector<MB>& B, const double* x, double* d, std::vector<double>& w,
                std::vector<double>* dw) {
    if (dw) {
        net.weights_and_jacobian(x, w, *dw);
    } else {
        std::vector<std::vector<double>> pre, act;
        net.forward(x, pre, act);
        w = pre.back();
        softmax_inplace(w.data(), (int)w.size());
    }
    double M[9] = {0}, T[3] = {0};
    for (size_t i = 0; i < B.size(); ++i) {
        for (int e = 0; e < 9; ++e) M[e] += w[i] * B[i].R[e];
        for (int e = 0; e < 3; ++e) T[e] += w[i] * B[i].t[e];
    }
    for (int r = 0; r < 3; ++r) d[r] = M[3 * r] * x[0] + M[3 * r + 1] * x[1] + M[3 * r + 2] * x[2] + T[r];
}
}  // namespace

// SkinningMlp::weights / weight_jacobian at points x [n][3]: w [n][nb], dw [n][nb][3]
int orc_mlp_weights_jacobian(const double* theta, const int* widths, int nw, const double* x, int64_t n, double* w_out,
                             double* dw_out, int workers) {
    return guard([&] {
        const Net net(theta, widths, nw);
        const int nb = widths[nw - 1];
        parallel_for(n, workers, [&](int64_t p0, int64_t p1, int) {
            std::vector<double> w, dw;
            for (int64_t p = p0; p < p1; ++p) {
                net.weights_and_jacobian(x + 3 * p, w, dw);
                std::copy(w.begin(), w.end(), w_out + p * nb);
                std::copy(dw.begin(), dw.end(), dw_out + p * nb * 3);
            }
        });
    });
}

// batch_search with SearchVariant::Mlp (correspondence.cpp:126-192), dense per-(point, init)
// outputs like orc_batch_search.
int orc_batch_search_mlp(const double* theta, const int* widths, int nw, const double* bones, int n_bones,
                         const double* x_prime, int64_t n, int max_iters, double conv_eps, double div_eps,
                         double dedup_dist, int workers, double* x_c, double* jinv, double* resid, int32_t* iters,
                         uint8_t* converged, uint8_t* keep) {
    return guard([&] {
        if (n_bones < 1) throw std::invalid_argument("search: no bone transforms");
        if (widths[0] != 3) throw std::invalid_argument("SkinningMlp: network input width must be 3");
        if (widths[nw - 1] != n_bones) throw std::invalid_argument("search: mlp bone count mismatch");
        if (max_iters < 1) throw std::invalid_argument("search: max_iters must be >= 1");
        if (!(conv_eps > 0.0)) throw std::invalid_argument("search: conv_eps must be > 0");
        if (!(div_eps > conv_eps)) throw std::invalid_argument("search: div_eps must exceed conv_eps");
        if (!(dedup_dist >= 0.0)) throw std::invalid_argument("search: dedup_dist must be >= 0");
        const Net net(theta, widths, nw);
        std::vector<MB> B(n_bones);
        for (int i = 0; i < n_bones; ++i)
            for (int r = 0; r < 3; ++r) {
                for (int c = 0; c < 3; ++c) B[i].R[3 * r + c] = bones[12 * i + 4 * r + c];
                B[i].t[r] = bones[12 * i + 4 * r + 3];
            }
        const int nb = n_bones;
        parallel_for(n, workers, [&](int64_t p0, int64_t p1, int) {
            std::vector<double> w, dw;
            for (int64_t p = p0; p < p1; ++p) {
                const double* xp = x_prime + 3 * p;
                std::vector<double> xs(3 * nb);
                std::vector<uint8_t> cv(nb);
                for (int i = 0; i < nb; ++i) {
                    const MB& b = B[i];
                    // x0 = B_i^-1 x' = Rᵀ x' + (−Rᵀ t) (geometry.hpp:58-61)
                    double x[3], it[3];
                    for (int a = 0; a < 3; ++a) it[a] = -(b.R[a] * b.t[0] + b.R[3 + a] * b.t[1] + b.R[6 + a] * b.t[2]);
                    for (int a = 0; a < 3; ++a) x[a] = b.R[a] * xp[0] + b.R[3 + a] * xp[1] + b.R[6 + a] * xp[2] + it[a];
                    // J = Σ w_i R_i + Σ (B_i x)(∇w_i)ᵀ (deformer.cpp:117-128), inverse or I (:43-54)
                    double d[3];
                    mlp_deform(net, B, x, d, w, &dw);
                    double J[9] = {0};
                    for (int k = 0; k < nb; ++k)
                        for (int e = 0; e < 9; ++e) J[e] += w[k] * B[k].R[e];
                    for (int k = 0; k < nb; ++k) {
                        double bx[3];
                        for (int r = 0; r < 3; ++r)
                            bx[r] = B[k].R[3 * r] * x[0] + B[k].R[3 * r + 1] * x[1] + B[k].R[3 * r + 2] * x[2] + B[k].t[r];
                        for (int r = 0; r < 3; ++r)
                            for (int c = 0; c < 3; ++c) J[3 * r + c] += bx[r] * dw[(size_t)k * 3 + c];
                    }
                    double Ji[9];
                    const double c00 = J[4] * J[8] - J[5] * J[7], c01 = J[2] * J[7] - J[1] * J[8],
                                 c02 = J[1] * J[5] - J[2] * J[4], c10 = J[5] * J[6] - J[3] * J[8],
                                 c11 = J[0] * J[8] - J[2] * J[6], c12 = J[2] * J[3] - J[0] * J[5],
                                 c20 = J[3] * J[7] - J[4] * J[6], c21 = J[1] * J[6] - J[0] * J[7],
                                 c22 = J[0] * J[4] - J[1] * J[3];
                    const double det = J[0] * c00 + J[1] * c10 + J[2] * c20;
                    if (std::abs(det) < 1e-8) {
                        for (int e = 0; e < 9; ++e) Ji[e] = (e % 4 == 0) ? 1.0 : 0.0;
                    } else {
                        const double cc[9] = {c00, c01, c02, c10, c11, c12, c20, c21, c22};
                        for (int e = 0; e < 9; ++e) Ji[e] = cc[e] / det;
                    }
                    double g[3] = {d[0] - xp[0], d[1] - xp[1], d[2] - xp[2]};
                    // iterate (correspondence.cpp:97-124)
                    int k_it = 0;
                    bool conv = false;
                    double err = std::sqrt(g[0] * g[0] + g[1] * g[1] + g[2] * g[2]);
                    if (err < conv_eps) conv = true;
                    for (int k = 0; !conv && k < max_iters; ++k) {
                        if (err > div_eps) break;
                        double dx[3];
                        for (int r = 0; r < 3; ++r) dx[r] = -(Ji[3 * r] * g[0] + Ji[3 * r + 1] * g[1] + Ji[3 * r + 2] * g[2]);
                        for (int a = 0; a < 3; ++a) x[a] += dx[a];
                        mlp_deform(net, B, x, d, w, nullptr);
                        double dg[3];
                        for (int a = 0; a < 3; ++a) {
                            const double gn = d[a] - xp[a];
                            dg[a] = gn - g[a];
                            g[a] = gn;
                        }
                        k_it = k + 1;
                        err = std::sqrt(g[0] * g[0] + g[1] * g[1] + g[2] * g[2]);
                        if (err < conv_eps) {
                            conv = true;
                            break;
                        }
                        double jdg[3];
                        for (int r = 0; r < 3; ++r) jdg[r] = Ji[3 * r] * dg[0] + Ji[3 * r + 1] * dg[1] + Ji[3 * r + 2] * dg[2];
                        const double den = dx[0] * jdg[0] + dx[1] * jdg[1] + dx[2] * jdg[2];
                        if (std::abs(den) > 1e-18) {
                            double q[3], wr[3];
                            for (int r = 0; r < 3; ++r) q[r] = (dx[r] - jdg[r]) / den;
                            for (int c = 0; c < 3; ++c) wr[c] = dx[0] * Ji[c] + dx[1] * Ji[3 + c] + dx[2] * Ji[6 + c];
                            for (int r = 0; r < 3; ++r)
                                for (int c = 0; c < 3; ++c) Ji[3 * r + c] += q[r] * wr[c];
                        }
                    }
                    const int64_t s = p * nb + i;
                    for (int a = 0; a < 3; ++a) x_c[3 * s + a] = xs[3 * i + a] = x[a];
                    if (jinv)
                        for (int e = 0; e < 9; ++e) jinv[9 * s + e] = Ji[e];
                    if (resid) resid[s] = err;
                    if (iters) iters[s] = k_it;
                    converged[s] = cv[i] = conv ? 1 : 0;
                }
                // dedup_roots (correspondence.cpp:162-176) over the converged inits in bone order
                std::vector<int> kept;
                for (int i = 0; i < nb; ++i) {
                    uint8_t kk = 0;
                    if (cv[i]) {
                        kk = 1;
                        for (int j : kept) {
                            const double e0 = xs[3 * i] - xs[3 * j], e1 = xs[3 * i + 1] - xs[3 * j + 1],
                                         e2 = xs[3 * i + 2] - xs[3 * j + 2];
                            if (std::sqrt(e0 * e0 + e1 * e1 + e2 * e2) < dedup_dist) {
                                kk = 0;
                                break;
                            }
                        }
                        if (kk) kept.push_back(i);
                    }
                    if (keep) keep[p * nb + i] = kk;
                }
            }
        });
    });
}

}  // extern "C"
