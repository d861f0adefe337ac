// ORACLE-SIDE ANALYSIS TOOL — TEST INFRASTRUCTURE ONLY (see fskin_oracle.cpp header).
//
// Emulates the GPU solver's arithmetic precision on the CPU to study where FP32 Broyden
// trajectories part from the f64 oracle (correspondence.cpp:97-124 restated in a scalar
// type R over a transform grid stored in type G). Used by tests/test_precision_study.py
// and DESIGN.md's precision analysis; never by the product.
#include <cmath>
#include <cstdint>
#include <thread>
#include <vector>

namespace {

template <typename R, typename G>
struct Emu {
    int nx, ny, nz;
    R lo[3], hi[3], scale[3];
    const G* tg;  // [V][12]

    void locate(const R x[3], bool lower, int idx[3], R t[3]) const {
        const int n[3] = {nx, ny, nz};
        for (int a = 0; a < 3; ++a) {
            R p = x[a] < lo[a] ? lo[a] : x[a];
            p = p > hi[a] ? hi[a] : p;
            const R u = (p - lo[a]) * scale[a];
            int i = (u == u) ? (int)std::floor(u) : 0;
            if (lower && i >= 1 && u == (R)i) i -= 1;
            i = i < 0 ? 0 : (i > n[a] - 2 ? n[a] - 2 : i);
            idx[a] = i;
            R tt = u - (R)i;
            t[a] = tt < 0 ? 0 : (tt > 1 ? 1 : tt);
        }
    }
    const G* vtx(int i, int j, int k) const { return tg + ((int64_t(k) * ny + j) * nx + i) * 12; }
    void trilerp(const R x[3], R T[12]) const {
        int c[3];
        R t[3];
        locate(x, false, c, t);
        for (int e = 0; e < 12; ++e) T[e] = 0;
        for (int dk = 0; dk < 2; ++dk) {
            const R wz = dk ? t[2] : 1 - t[2];
            for (int dj = 0; dj < 2; ++dj) {
                const R wyz = wz * (dj ? t[1] : 1 - t[1]);
                for (int di = 0; di < 2; ++di) {
                    const R w = wyz * (di ? t[0] : 1 - t[0]);
                    const G* m = vtx(c[0] + di, c[1] + dj, c[2] + dk);
                    for (int e = 0; e < 12; ++e) T[e] += w * (R)m[e];
                }
            }
        }
    }
    void jacobian(const R x[3], R J[9]) const {
        R T[12];
        trilerp(x, T);
        int c[3];
        R t[3];
        locate(x, true, c, t);
        R Gm[9] = {0};
        for (int dk = 0; dk < 2; ++dk)
            for (int dj = 0; dj < 2; ++dj)
                for (int di = 0; di < 2; ++di) {
                    const R fx = di ? t[0] : 1 - t[0], fy = dj ? t[1] : 1 - t[1], fz = dk ? t[2] : 1 - t[2];
                    const R g[3] = {(di ? scale[0] : -scale[0]) * fy * fz, fx * (dj ? scale[1] : -scale[1]) * fz,
                                    fx * fy * (dk ? scale[2] : -scale[2])};
                    const G* m = vtx(c[0] + di, c[1] + dj, c[2] + dk);
                    for (int r = 0; r < 3; ++r) {
                        const R y = (R)m[4 * r] * x[0] + (R)m[4 * r + 1] * x[1] + (R)m[4 * r + 2] * x[2] + (R)m[4 * r + 3];
                        for (int q = 0; q < 3; ++q) Gm[3 * r + q] += y * g[q];
                    }
                }
        for (int r = 0; r < 3; ++r)
            for (int q = 0; q < 3; ++q) J[3 * r + q] = T[4 * r + q] + Gm[3 * r + q];
    }
    void deform(const R x[3], R d[3]) const {
        R T[12];
        trilerp(x, T);
        for (int r = 0; r < 3; ++r) d[r] = T[4 * r] * x[0] + T[4 * r + 1] * x[1] + T[4 * r + 2] * x[2] + T[4 * r + 3];
    }
};

template <typename R>
void inv_or_id(const R J[9], R Ji[9]) {
    const R c00 = J[4] * J[8] - J[5] * J[7], c01 = J[2] * J[7] - J[1] * J[8], c02 = J[1] * J[5] - J[2] * J[4];
    const R c10 = J[5] * J[6] - J[3] * J[8], c11 = J[0] * J[8] - J[2] * J[6], c12 = J[2] * J[3] - J[0] * J[5];
    const R c20 = J[3] * J[7] - J[4] * J[6], c21 = J[1] * J[6] - J[0] * J[7], c22 = J[0] * J[4] - J[1] * J[3];
    const R det = J[0] * c00 + J[1] * c10 + J[2] * c20;
    if (std::fabs(det) < (R)1e-8) {
        for (int e = 0; e < 9; ++e) Ji[e] = (e % 4 == 0) ? 1 : 0;
        return;
    }
    const R inv = 1 / det;
    const R c[9] = {c00, c01, c02, c10, c11, c12, c20, c21, c22};
    for (int e = 0; e < 9; ++e) Ji[e] = c[e] * inv;
}

struct EscRule {
    int cap = 1 << 30;  // stop the low-precision pass after this many iterations (escalate)
    int min_div_iters = 1 << 30;  // escalate unconverged solves with iters >= this
    double conv_band = 0, div_band = 0, det_guard = 0, den_guard = 0;
};

// R: Broyden algebra and trilerp (J~, dx, dg, T); X: position x, residual g = T·[x;1] − x'
// and the threshold tests; G: grid storage. (R, X, G) = (f32, f64, f32) is the "f64 state"
// variant of the FP32 pass.
template <typename R, typename G, typename X = R>
void solve(const Emu<R, G>& E, const double* B12, const double* xpd, int max_iters, X conv, X div, double* xo,
           uint8_t* cv, int32_t* it, const EscRule* rule = nullptr, uint8_t* esc = nullptr, double* jn = nullptr) {
    bool e = false;
    auto near = [&](X v, X thr, double band) { return band > 0 && std::fabs((double)v / (double)thr - 1.0) < band; };
    const X xp[3] = {(X)xpd[0], (X)xpd[1], (X)xpd[2]};
    X Rm[9], t[3];
    for (int r = 0; r < 3; ++r) {
        for (int c = 0; c < 3; ++c) Rm[3 * r + c] = (X)B12[4 * r + c];
        t[r] = (X)B12[4 * r + 3];
    }
    X x[3];
    for (int a = 0; a < 3; ++a) {
        const X rt = Rm[a] * t[0] + Rm[3 + a] * t[1] + Rm[6 + a] * t[2];
        x[a] = Rm[a] * xp[0] + Rm[3 + a] * xp[1] + Rm[6 + a] * xp[2] + (-rt);
    }
    auto deform = [&](const X xx[3], X d[3]) {
        const R xr[3] = {(R)xx[0], (R)xx[1], (R)xx[2]};
        R T[12];
        E.trilerp(xr, T);
        for (int r = 0; r < 3; ++r)
            d[r] = (X)T[4 * r] * xx[0] + (X)T[4 * r + 1] * xx[1] + (X)T[4 * r + 2] * xx[2] + (X)T[4 * r + 3];
    };
    R J[9], Ji[9];
    X d[3], g[3];
    double amp = 0, cosmin = 1;  // sensitivity diagnostics: largest relative rank-1 update, smallest |cos(dx, J~dg)|
    double err_prev = 0, step_last = 0;  // residual before the last step, length of the last step
    {
        const R xr[3] = {(R)x[0], (R)x[1], (R)x[2]};
        E.jacobian(xr, J);
    }
    if (rule) {
        const R det = J[0] * (J[4] * J[8] - J[5] * J[7]) - J[1] * (J[3] * J[8] - J[5] * J[6]) + J[2] * (J[3] * J[7] - J[4] * J[6]);
        if (std::fabs((double)det) < rule->det_guard) e = true;
    }
    inv_or_id(J, Ji);
    deform(x, d);
    for (int a = 0; a < 3; ++a) g[a] = d[a] - xp[a];
    X err = std::sqrt(g[0] * g[0] + g[1] * g[1] + g[2] * g[2]);
    int iters = 0;
    bool conv_ok = err < conv;
    if (rule && (near(err, conv, rule->conv_band) || near(err, div, rule->div_band))) e = true;
    if (!conv_ok) {
        for (int k = 0; k < max_iters; ++k) {
            if (rule && k >= rule->cap) { e = true; break; }
            if (err > div) break;
            R dx[3];
            const R gr[3] = {(R)g[0], (R)g[1], (R)g[2]};
            for (int r = 0; r < 3; ++r) dx[r] = -(Ji[3 * r] * gr[0] + Ji[3 * r + 1] * gr[1] + Ji[3 * r + 2] * gr[2]);
            for (int a = 0; a < 3; ++a) x[a] += (X)dx[a];
            err_prev = (double)err;
            step_last = std::sqrt((double)dx[0] * dx[0] + (double)dx[1] * dx[1] + (double)dx[2] * dx[2]);
            deform(x, d);
            X gn[3];
            R dg[3];
            for (int a = 0; a < 3; ++a) {
                gn[a] = d[a] - xp[a];
                dg[a] = (R)(gn[a] - g[a]);
                g[a] = gn[a];
            }
            iters = k + 1;
            err = std::sqrt(g[0] * g[0] + g[1] * g[1] + g[2] * g[2]);
            if (rule && (near(err, conv, rule->conv_band) || near(err, div, rule->div_band))) e = true;
            if (err < conv) {
                conv_ok = true;
                break;
            }
            R jdg[3];
            for (int r = 0; r < 3; ++r) jdg[r] = Ji[3 * r] * dg[0] + Ji[3 * r + 1] * dg[1] + Ji[3 * r + 2] * dg[2];
            const R den = dx[0] * jdg[0] + dx[1] * jdg[1] + dx[2] * jdg[2];
            if (rule && std::fabs((double)den) < rule->den_guard) e = true;
            {
                const double nd = std::sqrt((double)dx[0] * dx[0] + (double)dx[1] * dx[1] + (double)dx[2] * dx[2]);
                const double nj = std::sqrt((double)jdg[0] * jdg[0] + (double)jdg[1] * jdg[1] + (double)jdg[2] * jdg[2]);
                if (nd > 0 && nj > 0) cosmin = std::fmin(cosmin, std::fabs((double)den) / (nd * nj));
            }
            if (std::fabs(den) > (R)1e-18) {
                R q[3], w[3];
                for (int r = 0; r < 3; ++r) q[r] = (dx[r] - jdg[r]) / den;
                for (int c = 0; c < 3; ++c) w[c] = dx[0] * Ji[c] + dx[1] * Ji[3 + c] + dx[2] * Ji[6 + c];
                double um = 0, jm = 0;
                for (int r = 0; r < 3; ++r)
                    for (int c = 0; c < 3; ++c) {
                        um = std::fmax(um, std::fabs((double)(q[r] * w[c])));
                        jm = std::fmax(jm, std::fabs((double)Ji[3 * r + c]));
                    }
                if (jm > 0) amp = std::fmax(amp, um / jm);
                for (int r = 0; r < 3; ++r)
                    for (int c = 0; c < 3; ++c) Ji[3 * r + c] += q[r] * w[c];
            }
        }
    }
    if (rule && !conv_ok && iters >= rule->min_div_iters) e = true;
    for (int a = 0; a < 3; ++a) xo[a] = (double)x[a];
    *cv = conv_ok;
    *it = iters;
    if (esc) *esc = e;
    if (jn) {
        double m = 0;
        for (int q = 0; q < 9; ++q) m = std::fmax(m, std::fabs((double)Ji[q]));
        jn[0] = m;
        jn[1] = amp;
        jn[2] = cosmin;
        for (int q = 0; q < 9; ++q) jn[3 + q] = (double)Ji[q];  // final J~
        double nx = 0;  // |J~ g| at the end: the step a further iteration would take
        for (int r = 0; r < 3; ++r) {
            const double v = (double)Ji[3 * r] * (double)g[0] + (double)Ji[3 * r + 1] * (double)g[1] +
                             (double)Ji[3 * r + 2] * (double)g[2];
            nx += v * v;
        }
        jn[12] = (double)err / (double)conv;
        jn[13] = std::sqrt(nx) / (double)conv;
        jn[14] = err_prev / (double)conv;
        jn[15] = step_last / (double)conv;
    }
}

template <typename R, typename G, typename X = R>
void run(const double* tg64, int nx, int ny, int nz, const double* bbox, const double* bones, int nb, const double* x,
         int64_t n, int max_iters, double conv, double div, int workers, double* xo, uint8_t* cv, int32_t* it,
         const EscRule* rule = nullptr, uint8_t* esc = nullptr, double* jn = nullptr) {
    const int64_t V = int64_t(nx) * ny * nz;
    std::vector<G> tg(V * 12);
    for (int64_t e = 0; e < V * 12; ++e) tg[e] = (G)tg64[e];
    Emu<R, G> E;
    E.nx = nx; E.ny = ny; E.nz = nz; E.tg = tg.data();
    const int n3[3] = {nx, ny, nz};
    for (int a = 0; a < 3; ++a) {
        E.lo[a] = (R)bbox[a];
        E.hi[a] = (R)bbox[3 + a];
        E.scale[a] = (R)((double)(n3[a] - 1) / ((double)(R)bbox[3 + a] - (double)(R)bbox[a]));
    }
    std::vector<std::thread> pool;
    for (int w = 0; w < workers; ++w)
        pool.emplace_back([&, w] {
            for (int64_t p = n * w / workers; p < n * (w + 1) / workers; ++p)
                for (int i = 0; i < nb; ++i) {
                    const int64_t s = p * nb + i;
                    solve<R, G, X>(E, bones + 12 * i, x + 3 * p, max_iters, (X)conv, (X)div, xo + 3 * s, cv + s, it + s,
                                rule, esc ? esc + s : nullptr, jn ? jn + 16 * s : nullptr);
                }
        });
    for (auto& t : pool) t.join();
}

}  // namespace

extern "C" int orc_emul_search(int mode, const double* tgrid, int nx, int ny, int nz, const double* bbox6,
                               const double* bones, int nb, const double* x, int64_t n, int max_iters, double conv,
                               double div, int workers, double* x_c, uint8_t* converged, int32_t* iters) {
    // mode 0: f64 state, f64 grid; 1: f32 state, f32 grid (the GPU kernel); 2: f64 state, f32 grid;
    // 3: f32 trilerp and Broyden algebra, f64 position and residual, f32 grid
    switch (mode) {
        case 0: run<double, double>(tgrid, nx, ny, nz, bbox6, bones, nb, x, n, max_iters, conv, div, workers, x_c, converged, iters); break;
        case 1: run<float, float>(tgrid, nx, ny, nz, bbox6, bones, nb, x, n, max_iters, conv, div, workers, x_c, converged, iters); break;
        case 2: run<double, float>(tgrid, nx, ny, nz, bbox6, bones, nb, x, n, max_iters, conv, div, workers, x_c, converged, iters); break;
        case 3: run<float, float, double>(tgrid, nx, ny, nz, bbox6, bones, nb, x, n, max_iters, conv, div, workers, x_c, converged, iters); break;
        default: return 1;
    }
    return 0;
}

// Hybrid (the GPU design): float32 pass with an iteration cap and escalation flags; the
// escalation mask is returned so the caller can substitute the f64 (mode 0) results.
extern "C" int orc_emul_hybrid(const double* tgrid, int nx, int ny, int nz, const double* bbox6, const double* bones,
                               int nb, const double* x, int64_t n, int max_iters, double conv, double div, int workers,
                               int cap, int min_div_iters, double conv_band, double div_band, double det_guard,
                               double den_guard, double* x_c, uint8_t* converged, int32_t* iters, uint8_t* esc,
                               double* jinv_diag /* [n][nb][16]: max|J~|, amp, cos_min, J~, err/conv, |J~g|/conv, err_prev/conv, |dx_last|/conv */, int mixed_state) {
    EscRule r;
    r.cap = cap;
    r.min_div_iters = min_div_iters;
    r.conv_band = conv_band;
    r.div_band = div_band;
    r.det_guard = det_guard;
    r.den_guard = den_guard;
    if (mixed_state)
        run<float, float, double>(tgrid, nx, ny, nz, bbox6, bones, nb, x, n, max_iters, conv, div, workers, x_c, converged, iters, &r, esc, jinv_diag);
    else
        run<float, float>(tgrid, nx, ny, nz, bbox6, bones, nb, x, n, max_iters, conv, div, workers, x_c, converged, iters, &r, esc, jinv_diag);
    return 0;
}
