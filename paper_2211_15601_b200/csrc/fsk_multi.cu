// fsk_multi.cu — single-process multi-GPU form of the deformer C-ABI:
// the reference is one C++ process (parallel_for over host threads, parallel.hpp:17-33), so
// its drop-in drives every GPU of the box from one process: one fsk_ctx, stream and host
// thread per device, points sharded in contiguous ranges (the parallel_for partition,
// parallel.hpp:28-29). The pose inputs (weight grid, bones) reach the devices by one NCCL
// broadcast from device 0; the solves themselves exchange nothing — each reads only the
// immutable grid and bones; the backward sums dL/dT [V][12] over the
// devices with one NCCL all-reduce (ncclCommInitAll communicator, NVLink/NVSwitch), in the
// deterministic mode as exact int64 fixed-point sums under a shared scale.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <barrier>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "fsk.h"
#include "fsk_ctx.h"

struct fsk_multi {
    std::vector<int> dev;
    std::vector<fsk_ctx*> ctx;
    std::vector<cudaStream_t> st;
    std::vector<ncclComm_t> comm;  // created on first collective use
    // per-device staging (device buffers)
    struct Buf {
        float *w = nullptr, *b = nullptr, *p = nullptr, *gx = nullptr, *gT = nullptr, *gw = nullptr;
        int64_t *offs = nullptr, *ridx = nullptr, *acc = nullptr;
        fsk_root* roots = nullptr;
        size_t cw = 0, cb = 0, cp = 0, cgx = 0, cgT = 0, cgw = 0, coffs = 0, cridx = 0, croots = 0, cacc = 0;
    };
    std::vector<Buf> buf;
};

namespace fsk {
namespace {

template <typename T>
T* grow(T*& p, size_t& cap, size_t n) {
    n = std::max<size_t>(n, 1);
    if (cap < n) {
        if (p) cudaFree(p);
        p = nullptr;
        cuda_check(cudaMalloc(&p, n * sizeof(T)), "cudaMalloc");
        cap = n;
    }
    return p;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) fail(FSK_ECUDA, std::string(what) + ": " + ncclGetErrorString(r));
}

// Run fn(r) on one host thread per device (device set, errors collected; first one rethrown).
template <typename Fn>
void per_device(fsk_multi* m, Fn&& fn) {
    const int R = (int)m->dev.size();
    std::vector<Error> errs(R);
    std::vector<char> bad(R, 0);
    std::vector<std::thread> th;
    for (int r = 0; r < R; ++r)
        th.emplace_back([&, r] {
            try {
                cuda_check(cudaSetDevice(m->dev[r]), "cudaSetDevice");
                fn(r);
            } catch (const Error& e) {
                errs[r] = e;
                bad[r] = 1;
            } catch (const std::exception& e) {
                errs[r] = Error{FSK_ECUDA, e.what()};
                bad[r] = 1;
            }
        });
    for (auto& t : th) t.join();
    for (int r = 0; r < R; ++r)
        if (bad[r]) throw errs[r];
}

void rc_check(int rc) {
    if (rc != FSK_OK) fail(rc, fsk_last_error());
}

void ensure_comm(fsk_multi* m) {  // one communicator per device, NVLink/NVSwitch (created on first use)
    if (!m->comm.empty()) return;
    m->comm.resize(m->dev.size());
    nccl_check(ncclCommInitAll(m->comm.data(), (int)m->dev.size(), m->dev.data()), "ncclCommInitAll");
}

}  // namespace
}  // namespace fsk

using namespace fsk;

extern "C" {

int fsk_multi_create(int32_t n_devices, const int32_t* devices, fsk_multi** out) {
    return guard([&] {
        if (!out || n_devices < 1 || !devices) fail(FSK_EINVAL, "fsk_multi: need at least one device");
        auto* m = new fsk_multi;
        try {
            for (int r = 0; r < n_devices; ++r) {
                for (int q = 0; q < r; ++q)
                    if (devices[q] == devices[r]) fail(FSK_EINVAL, "fsk_multi: duplicate device");
                fsk_ctx* c = nullptr;
                rc_check(fsk_ctx_create(devices[r], &c));
                m->ctx.push_back(c);
                m->dev.push_back(devices[r]);
                cudaStream_t s = nullptr;
                cuda_check(cudaSetDevice(devices[r]), "cudaSetDevice");
                cuda_check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
                m->st.push_back(s);
            }
            m->buf.resize(n_devices);
        } catch (...) {
            fsk_multi_destroy(m);
            throw;
        }
        *out = m;
    });
}

int fsk_multi_destroy(fsk_multi* m) {
    return guard([&] {
        if (!m) return;
        for (auto c : m->comm) ncclCommDestroy(c);
        for (size_t r = 0; r < m->dev.size(); ++r) {
            cudaSetDevice(m->dev[r]);
            if (r < m->buf.size()) {
                auto& b = m->buf[r];
                for (void* p : {(void*)b.w, (void*)b.b, (void*)b.p, (void*)b.gx, (void*)b.gT, (void*)b.gw,
                                (void*)b.offs, (void*)b.ridx, (void*)b.roots, (void*)b.acc})
                    if (p) cudaFree(p);
            }
            if (r < m->st.size() && m->st[r]) cudaStreamDestroy(m->st[r]);
            if (r < m->ctx.size()) fsk_ctx_destroy(m->ctx[r]);
        }
        delete m;
    });
}

int32_t fsk_multi_device_count(const fsk_multi* m) { return m ? (int32_t)m->dev.size() : 0; }

int fsk_multi_deform_host(fsk_multi* m, const float* weights, const fsk_grid_desc* desc, const float* bones,
                          int32_t n_bones_pose, const float* points, int64_t n, const fsk_search_opts* opts,
                          int64_t* offsets, fsk_root* roots, int64_t cap, int64_t* total_out) {
    return guard([&] {
        if (!m || !desc || !opts || !offsets || !total_out || !weights || !bones || (n > 0 && !points))
            fail(FSK_EINVAL, "fsk: null buffer");
        if (n < 0) fail(FSK_EINVAL, "fsk: negative point count");
        const int R = (int)m->dev.size();
        const int64_t V = (int64_t)desc->nx * desc->ny * desc->nz;
        const int nb = desc->n_bones;
        if (n_bones_pose != nb) fail(FSK_EINVAL, "precompute_transform_grid: bone count mismatch");
        ensure_comm(m);
        // pose inputs: host -> device 0 once, then one grouped ncclBroadcast over NVLink to the other
        // devices (the weight grid and bones are broadcast, every device runs K1 locally)
        for (int r = 0; r < R; ++r) {
            cuda_check(cudaSetDevice(m->dev[r]), "cudaSetDevice");
            auto& b = m->buf[r];
            grow(b.w, b.cw, V * nb);
            grow(b.b, b.cb, (size_t)nb * 12);
        }
        cuda_check(cudaSetDevice(m->dev[0]), "cudaSetDevice");
        cuda_check(cudaMemcpyAsync(m->buf[0].w, weights, V * nb * sizeof(float), cudaMemcpyHostToDevice, m->st[0]),
                   "H2D weights");
        cuda_check(cudaMemcpyAsync(m->buf[0].b, bones, nb * 12 * sizeof(float), cudaMemcpyHostToDevice, m->st[0]),
                   "H2D bones");
        if (R > 1) {
            nccl_check(ncclGroupStart(), "ncclGroupStart");
            for (int r = 0; r < R; ++r) {
                cuda_check(cudaSetDevice(m->dev[r]), "cudaSetDevice");
                nccl_check(ncclBroadcast(m->buf[0].w, m->buf[r].w, (size_t)V * nb, ncclFloat, 0, m->comm[r], m->st[r]),
                           "ncclBroadcast weights");
                nccl_check(ncclBroadcast(m->buf[0].b, m->buf[r].b, (size_t)nb * 12, ncclFloat, 0, m->comm[r], m->st[r]),
                           "ncclBroadcast bones");
            }
            nccl_check(ncclGroupEnd(), "ncclGroupEnd");
        }
        std::vector<int64_t> cnt(R, 0), base(R, 0);
        std::barrier sync(R);
        per_device(m, [&](int r) {
            auto& b = m->buf[r];
            cudaStream_t st = m->st[r];
            const int64_t p0 = n * r / R, p1 = n * (r + 1) / R, k = p1 - p0;  // parallel.hpp:28-29
            try {
                if (k > 0)
                    cuda_check(cudaMemcpyAsync(grow(b.p, b.cp, 3 * k), points + 3 * p0, 3 * k * sizeof(float),
                                               cudaMemcpyHostToDevice, st),
                               "H2D points");
                grow(b.offs, b.coffs, k + 1);
                // count-then-allocate: room for 4 kept roots per query first (about 1.05 are kept); a shard
                // with more is searched again into a buffer of exactly its count
                int64_t rcap = std::max<int64_t>(1, std::min<int64_t>(k * nb, 4 * k));
                int64_t c = 0;
                for (int attempt = 0; attempt < 2; ++attempt) {
                    grow(b.roots, b.croots, rcap);
                    rc_check(fsk_deform(m->ctx[r], b.w, desc, b.b, n_bones_pose, b.p, k, opts, nullptr, b.offs,
                                        b.roots, rcap, st));
                    cuda_check(cudaMemcpyAsync(&c, b.offs + k, sizeof(int64_t), cudaMemcpyDeviceToHost, st), "D2H count");
                    cuda_check(cudaStreamSynchronize(st), "cudaStreamSynchronize");
                    if (c <= rcap) break;
                    rcap = c;
                }
                cnt[r] = c;
            } catch (...) {
                cnt[r] = -1;
                sync.arrive_and_drop();
                throw;
            }
            sync.arrive_and_wait();
            for (int q = 0; q < R; ++q)
                if (cnt[q] < 0) return;  // another device failed: its error is reported
            int64_t bs = 0;
            for (int q = 0; q < r; ++q) bs += cnt[q];
            base[r] = bs;
            int64_t total = 0;
            for (int q = 0; q < R; ++q) total += cnt[q];
            // the roots gather straight into the caller's host buffer, one D2H per device in parallel
            if (total <= cap && cnt[r] > 0) {
                if (!roots) fail(FSK_EINVAL, "fsk: null buffer");
                cuda_check(cudaMemcpyAsync(roots + bs, b.roots, cnt[r] * sizeof(fsk_root), cudaMemcpyDeviceToHost, st),
                           "D2H roots");
            }
            if (k > 0)
                cuda_check(cudaMemcpyAsync(offsets + p0, b.offs, k * sizeof(int64_t), cudaMemcpyDeviceToHost, st),
                           "D2H offsets");
            cuda_check(cudaStreamSynchronize(st), "cudaStreamSynchronize");
            if (bs)
                for (int64_t i = p0; i < p1; ++i) offsets[i] += bs;  // shard-local -> global root index
        });
        int64_t total = 0;
        for (int r = 0; r < R; ++r) total += cnt[r];
        offsets[n] = total;
        *total_out = total;
        if (total > cap) fail(FSK_EINVAL, "fsk: root buffer too small");
    });
}

int fsk_multi_grad_weights_host(fsk_multi* m, const fsk_grid_desc* desc, const float* bones, int32_t n_bones_pose,
                                const fsk_root* roots, const int64_t* root_index, const float* grad_xc, int64_t n,
                                float* grad_w, int deterministic) {
    return guard([&] {
        if (!m || !desc || !bones || !grad_w || (n > 0 && (!roots || !root_index || !grad_xc)))
            fail(FSK_EINVAL, "fsk: null buffer");
        if (n < 0) fail(FSK_EINVAL, "fsk: negative point count");
        if (n_bones_pose != desc->n_bones) fail(FSK_EINVAL, "precompute_transform_grid: bone count mismatch");
        const int R = (int)m->dev.size();
        const int64_t V = (int64_t)desc->nx * desc->ny * desc->nz;
        const int nb = desc->n_bones;
        ensure_comm(m);
        // per shard: the selected roots (compacted host-side into one record per query), the
        // cotangents, K3 into dL/dT, then sum dL/dT over the devices (NCCL), dL/dw on device 0.
        // Deterministic mode: every device rounds to int64 fixed point with the SAME scale (max term
        // all-reduced over the devices, n = all points) and the int64 sums are all-reduced exactly, so
        // the gradient is bitwise the one-device result for any device count.
        std::vector<std::vector<fsk_root>> sel(R);
        std::vector<std::vector<int64_t>> ridx(R);
        for (int r = 0; r < R; ++r) {
            const int64_t p0 = n * r / R, p1 = n * (r + 1) / R;
            sel[r].reserve(p1 - p0);
            ridx[r].resize(p1 - p0);
            for (int64_t p = p0; p < p1; ++p) {
                if (root_index[p] < 0) {
                    ridx[r][p - p0] = -1;
                } else {
                    ridx[r][p - p0] = (int64_t)sel[r].size();
                    sel[r].push_back(roots[root_index[p]]);
                }
            }
        }
        per_device(m, [&](int r) {
            auto& b = m->buf[r];
            cudaStream_t st = m->st[r];
            const int64_t p0 = n * r / R, p1 = n * (r + 1) / R, k = p1 - p0;
            grow(b.roots, b.croots, sel[r].size());
            grow(b.ridx, b.cridx, k);
            grow(b.gx, b.cgx, 3 * k + 4);  // + the max term (deterministic mode)
            grow(b.gT, b.cgT, V * 12);
            if (!sel[r].empty())
                cuda_check(cudaMemcpyAsync(b.roots, sel[r].data(), sel[r].size() * sizeof(fsk_root),
                                           cudaMemcpyHostToDevice, st),
                           "H2D roots");
            if (k > 0) {
                cuda_check(cudaMemcpyAsync(b.ridx, ridx[r].data(), k * sizeof(int64_t), cudaMemcpyHostToDevice, st),
                           "H2D root index");
                cuda_check(cudaMemcpyAsync(b.gx, grad_xc + 3 * p0, 3 * k * sizeof(float), cudaMemcpyHostToDevice, st),
                           "H2D cotangents");
            }
            if (!deterministic) {
                rc_check(fsk_search_bwd_roots(m->ctx[r], desc, b.roots, b.ridx, b.gx, k, b.gT, 0, st));
            } else {
                const fsk_bwd_src src{nullptr, nullptr, nullptr, 0, b.roots, b.ridx};
                rc_check(fsk_search_bwd_max_term(m->ctx[r], desc, &src, b.gx, k, b.gx + 3 * k, st));
            }
        });
        if (deterministic) {
            // global max term, then each shard's int64 sums with the shared scale, summed exactly
            nccl_check(ncclGroupStart(), "ncclGroupStart");
            for (int r = 0; r < R; ++r) {
                const int64_t k = n * (r + 1) / R - n * r / R;
                cuda_check(cudaSetDevice(m->dev[r]), "cudaSetDevice");
                float* mt = m->buf[r].gx + 3 * k;
                nccl_check(ncclAllReduce(mt, mt, 1, ncclFloat, ncclMax, m->comm[r], m->st[r]), "ncclAllReduce max");
            }
            nccl_check(ncclGroupEnd(), "ncclGroupEnd");
            per_device(m, [&](int r) {
                auto& b = m->buf[r];
                const int64_t p0 = n * r / R, k = n * (r + 1) / R - p0;
                grow(b.acc, b.cacc, V * 12);
                cuda_check(cudaMemsetAsync(b.acc, 0, V * 12 * sizeof(int64_t), m->st[r]), "cudaMemsetAsync");
                const fsk_bwd_src src{nullptr, nullptr, nullptr, 0, b.roots, b.ridx};
                rc_check(fsk_search_bwd_fixed(m->ctx[r], desc, &src, b.gx, k, n, b.gx + 3 * k, b.acc, m->st[r]));
            });
            nccl_check(ncclGroupStart(), "ncclGroupStart");
            for (int r = 0; r < R; ++r) {
                cuda_check(cudaSetDevice(m->dev[r]), "cudaSetDevice");
                nccl_check(ncclAllReduce(m->buf[r].acc, m->buf[r].acc, (size_t)V * 12, ncclInt64, ncclSum, m->comm[r],
                                         m->st[r]),
                           "ncclAllReduce int64");
            }
            nccl_check(ncclGroupEnd(), "ncclGroupEnd");
            const int64_t k0 = n / R;  // device 0's shard size: its max-term slot
            cuda_check(cudaSetDevice(m->dev[0]), "cudaSetDevice");
            rc_check(fsk_fixed_to_float(m->ctx[0], m->buf[0].acc, V * 12, n, m->buf[0].gx + 3 * k0, m->buf[0].gT,
                                        m->st[0]));
        } else {
            // dL/dT summed over the devices: one all-reduce, ranks grouped from this thread
            nccl_check(ncclGroupStart(), "ncclGroupStart");
            for (int r = 0; r < R; ++r) {
                cuda_check(cudaSetDevice(m->dev[r]), "cudaSetDevice");
                nccl_check(ncclAllReduce(m->buf[r].gT, m->buf[r].gT, (size_t)V * 12, ncclFloat, ncclSum, m->comm[r],
                                         m->st[r]),
                           "ncclAllReduce");
            }
            nccl_check(ncclGroupEnd(), "ncclGroupEnd");
        }
        auto& b0 = m->buf[0];
        cudaStream_t st0 = m->st[0];
        cuda_check(cudaSetDevice(m->dev[0]), "cudaSetDevice");
        grow(b0.b, b0.cb, (size_t)nb * 12);
        grow(b0.gw, b0.cgw, V * nb);
        cuda_check(cudaMemcpyAsync(b0.b, bones, nb * 12 * sizeof(float), cudaMemcpyHostToDevice, st0), "H2D bones");
        rc_check(fsk_grad_weights(m->ctx[0], desc, b0.gT, b0.b, n_bones_pose, b0.gw, st0));
        cuda_check(cudaMemcpyAsync(grad_w, b0.gw, V * nb * sizeof(float), cudaMemcpyDeviceToHost, st0), "D2H grad_w");
        for (int r = 0; r < R; ++r) {
            cuda_check(cudaSetDevice(m->dev[r]), "cudaSetDevice");
            cuda_check(cudaStreamSynchronize(m->st[r]), "cudaStreamSynchronize");
        }
    });
}

}  // extern "C"
