// Multi-GPU synthesis inside one process (gm_synthesize_multi, gridmdp_b200.h).
//
// Replaces the reference's execution substrate — parallel_for over contiguous
// row ranges (include/gridmdp/parallel.hpp:23-51) under run_backward
// (src/synthesis.cpp:165-195) — by contiguous state shards, one host thread +
// one stream per device (SURVEY.md §8 e):
//   * stage (i): each device builds the rows of its states (gm_build_shard), no
//     communication;
//   * stage (ii): each device steps its states (gm_step_device) reading the full
//     V_{k+1}; after each step V_k is exchanged: only the cutoff-bounded halos
//     (the state intervals the peers' slabs read, gm_shard_reach, fixed for the
//     model) when they move at most half of what an all-gather moves, else an
//     in-place all-gather of the equal-sized shards.
// Transports: NCCL (ncclAllGather / grouped ncclSend+ncclRecv on each device's
// stream; NVLink / NVSwitch on a B200 node), loaded at run time, or CUDA peer
// copies after a host barrier (any device list, including one device repeated,
// which is how the sharded path is exercised on a single GPU).
// Per-row arithmetic does not depend on the shard, so results are bit-identical
// to gm_synthesize for any device count.
#include "gridmdp_b200.h"

#include "gm_internal.hpp"

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <barrier>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace {

// ------------------------------------------------------------------ NCCL (dlopen)

struct Nccl {
    ncclResult_t (*commInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*groupStart)() = nullptr;
    ncclResult_t (*groupEnd)() = nullptr;
    const char* (*errorString)(ncclResult_t) = nullptr;
    std::string why;
    bool ok = false;
};

const Nccl& nccl() {
    static Nccl N;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = nullptr;
        for (const char* name : {"libnccl.so.2", "libnccl.so"})
            if ((h = dlopen(name, RTLD_NOW | RTLD_LOCAL))) break;
        if (!h) {
            N.why = std::string("NCCL not loadable: ") + dlerror();
            return;
        }
        auto sym = [&](auto& fn, const char* name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
            if (!fn && N.why.empty()) N.why = std::string("NCCL symbol missing: ") + name;
        };
        sym(N.commInitAll, "ncclCommInitAll");
        sym(N.commDestroy, "ncclCommDestroy");
        sym(N.allGather, "ncclAllGather");
        sym(N.send, "ncclSend");
        sym(N.recv, "ncclRecv");
        sym(N.groupStart, "ncclGroupStart");
        sym(N.groupEnd, "ncclGroupEnd");
        sym(N.errorString, "ncclGetErrorString");
        N.ok = N.why.empty();
    });
    return N;
}

void nck(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        gmi_throw(GM_ERR_CUDA, std::string(what) + ": " + (nccl().errorString ? nccl().errorString(r) : "NCCL error"));
}

void cck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        cudaGetLastError();
        gmi_throw(e == cudaErrorMemoryAllocation ? GM_ERR_MEMORY : GM_ERR_CUDA,
                  std::string(what) + ": " + cudaGetErrorString(e));
    }
}

void sck(gm_code rc, const gm_status& st) {
    if (rc != GM_OK) gmi_throw(rc, st.msg);
}

// ------------------------------------------------------------------ plans

struct Range {
    int peer;
    int64_t a, b; // flat state range [a, b)
};

// Equal contiguous state ranges, padded to `per` (sharded.py ShardPlan).
struct Shards {
    int64_t n_x = 0, per = 0;
    int n = 0;
    int64_t x0(int r) const { return std::min(n_x, r * per); }
    int64_t x1(int r) const { return std::min(n_x, x0(r) + per); }
};

// Halo plan (sharded.py halo_plan): device j sends device r the part of its
// states inside r's reach interval.
struct Exchange {
    bool halo = false;
    int64_t halo_states = 0, ag_states = 0;
    std::vector<std::vector<Range>> sends, recvs; // per device
};

Exchange plan_exchange(const Shards& S, const std::vector<std::pair<int64_t, int64_t>>& reach, int mode) {
    Exchange X;
    X.sends.resize(static_cast<size_t>(S.n));
    X.recvs.resize(static_cast<size_t>(S.n));
    std::vector<std::vector<Range>> hs(static_cast<size_t>(S.n)), hr(static_cast<size_t>(S.n));
    for (int r = 0; r < S.n; ++r) {
        X.ag_states += S.n_x - (S.x1(r) - S.x0(r));
        for (int j = 0; j < S.n; ++j) {
            if (j == r) continue;
            const int64_t a = std::max(S.x0(j), reach[static_cast<size_t>(r)].first);
            const int64_t b = std::min(S.x1(j), reach[static_cast<size_t>(r)].second);
            if (a < b) {
                hs[static_cast<size_t>(j)].push_back({r, a, b});
                hr[static_cast<size_t>(r)].push_back({j, a, b});
                X.halo_states += b - a;
            }
        }
    }
    X.halo = mode == GM_XCHG_HALO || (mode == GM_XCHG_AUTO && 2 * X.halo_states <= X.ag_states);
    if (X.halo) {
        X.sends = std::move(hs);
        X.recvs = std::move(hr);
    } else {
        for (int r = 0; r < S.n; ++r)
            for (int j = 0; j < S.n; ++j)
                if (j != r && S.x0(j) < S.x1(j)) {
                    X.sends[static_cast<size_t>(j)].push_back({r, S.x0(j), S.x1(j)});
                    X.recvs[static_cast<size_t>(r)].push_back({j, S.x0(j), S.x1(j)});
                }
    }
    return X;
}

// ------------------------------------------------------------------ per-device state

struct Dev {
    int device = 0;
    gm_model* model = nullptr;
    gm_matrix* tm = nullptr;
    cudaStream_t s = nullptr;
    double* vals = nullptr;   // (T+1) x P, column k at vals + k * P
    uint32_t* pol = nullptr;  // T x per
    uint32_t* wst = nullptr;  // T x per
    std::vector<cudaEvent_t> step_ev; // one per step (peer transport)
    cudaEvent_t t0 = nullptr, t1 = nullptr, t2 = nullptr;
    float build_ms = 0.f, sweep_ms = 0.f;
    ~Dev() {
        if (model) {
            cudaSetDevice(device);
            if (s) cudaStreamSynchronize(s);
            if (tm) gm_matrix_free(tm);
            gm_model_free(model);
        }
        cudaFree(vals);
        cudaFree(pol);
        cudaFree(wst);
        for (cudaEvent_t e : step_ev) cudaEventDestroy(e);
        for (cudaEvent_t e : {t0, t1, t2})
            if (e) cudaEventDestroy(e);
        if (s) cudaStreamDestroy(s);
    }
};

struct Job {
    gm_model* m = nullptr;
    int n = 0;
    std::vector<int> devices;
    int exchange = GM_XCHG_AUTO, transport = GM_XPORT_NCCL;
    Shards S;
    int T = 0;
    bool reach = false, matrix = false;
    int64_t P = 0; // padded V length per * n
    std::vector<std::unique_ptr<Dev>> dev;
    std::vector<std::pair<int64_t, int64_t>> reach_iv;
    Exchange X;
    std::vector<ncclComm_t> comms;
    gm_result* res = nullptr;
    double *h_vals = nullptr;
    uint32_t *h_pol = nullptr, *h_wst = nullptr;
    std::barrier<> bar;
    std::atomic<bool> failed{false};
    std::mutex mu;
    gm_status err{};
    explicit Job(int n_) : n(n_), bar(n_) {}

    void fail(const gm_status& st) {
        std::lock_guard<std::mutex> lk(mu);
        if (!failed.exchange(true)) err = st;
    }
    // A collective point: every thread arrives; true when no thread has failed.
    bool sync_ok() {
        bar.arrive_and_wait();
        return !failed.load();
    }
};

// Runs `f` with the C ABI's error mapping; records the first failure.
template <class F>
bool step_guard(Job& J, F&& f) {
    gm_status st{};
    if (gmi_guarded(&st, std::function<void()>(f)) != GM_OK) {
        J.fail(st);
        return false;
    }
    return true;
}

void exchange_peer(Job& J, int d, int k) {
    Dev& D = *J.dev[static_cast<size_t>(d)];
    for (const Range& r : J.X.recvs[static_cast<size_t>(d)]) {
        Dev& src = *J.dev[static_cast<size_t>(r.peer)];
        cck(cudaStreamWaitEvent(D.s, src.step_ev[static_cast<size_t>(k)], 0), "peer wait");
        const size_t off = static_cast<size_t>(k) * static_cast<size_t>(J.P) + static_cast<size_t>(r.a);
        cck(cudaMemcpyPeerAsync(D.vals + off, D.device, src.vals + off, src.device, static_cast<size_t>(r.b - r.a) * 8,
                                D.s),
            "peer copy");
    }
}

// The store transport: the peers that read this device's states wrote them into its
// column k during their step k (gmi_step_device_mirrored); wait for those steps.
void exchange_store(Job& J, int d, int k) {
    Dev& D = *J.dev[static_cast<size_t>(d)];
    for (const Range& r : J.X.recvs[static_cast<size_t>(d)])
        cck(cudaStreamWaitEvent(D.s, J.dev[static_cast<size_t>(r.peer)]->step_ev[static_cast<size_t>(k)], 0),
            "store wait");
}

// This device's pass-2 epilogue targets for step k: every peer column whose read
// interval (the exchange plan's send ranges) holds some of this device's states.
gmk::GmMirror mirrors_for(Job& J, int d, int k) {
    gmk::GmMirror mir;
    for (const Range& r : J.X.sends[static_cast<size_t>(d)]) {
        if (mir.n == gmk::kMaxMirrors) throw std::runtime_error("store transport: more than 8 peers per device");
        mir.dst[mir.n] = J.dev[static_cast<size_t>(r.peer)]->vals + static_cast<size_t>(k) * static_cast<size_t>(J.P);
        mir.lo[mir.n] = r.a;
        mir.hi[mir.n] = r.b;
        ++mir.n;
    }
    return mir;
}

void exchange_nccl(Job& J, int d, int k) {
    Dev& D = *J.dev[static_cast<size_t>(d)];
    const Nccl& N = nccl();
    double* col = D.vals + static_cast<size_t>(k) * static_cast<size_t>(J.P);
    if (!J.X.halo) { // in place: this device's chunk sits at d * per
        nck(N.allGather(col + static_cast<size_t>(d) * static_cast<size_t>(J.S.per), col, static_cast<size_t>(J.S.per),
                        ncclDouble, J.comms[static_cast<size_t>(d)], D.s),
            "ncclAllGather");
        return;
    }
    nck(N.groupStart(), "ncclGroupStart");
    for (const Range& r : J.X.sends[static_cast<size_t>(d)])
        nck(N.send(col + r.a, static_cast<size_t>(r.b - r.a), ncclDouble, r.peer, J.comms[static_cast<size_t>(d)], D.s),
            "ncclSend");
    for (const Range& r : J.X.recvs[static_cast<size_t>(d)])
        nck(N.recv(col + r.a, static_cast<size_t>(r.b - r.a), ncclDouble, r.peer, J.comms[static_cast<size_t>(d)], D.s),
            "ncclRecv");
    nck(N.groupEnd(), "ncclGroupEnd");
}

void device_main(Job& J, int d) {
    Dev& D = *J.dev[static_cast<size_t>(d)];
    const int64_t x0 = J.S.x0(d), x1 = J.S.x1(d);
    const size_t P = static_cast<size_t>(J.P), per = static_cast<size_t>(J.S.per);
    const int T = J.T;
    // setup: model on this device, stream, tables
    bool ok = step_guard(J, [&] {
        cck(cudaSetDevice(D.device), "cudaSetDevice");
        gm_status st{};
        sck(gm_model_clone(J.m, &D.model, &st), st);
        cck(cudaStreamCreateWithFlags(&D.s, cudaStreamNonBlocking), "stream");
        sck(gm_model_set_stream(D.model, D.s, 0, &st), st);
        for (cudaEvent_t* e : {&D.t0, &D.t1, &D.t2}) cck(cudaEventCreate(e), "event");
        D.step_ev.resize(static_cast<size_t>(T));
        for (cudaEvent_t& e : D.step_ev) cck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
        cck(cudaMalloc(&D.vals, std::max<size_t>(P * (T + 1), 1) * 8), "value table");
        cck(cudaMalloc(&D.pol, std::max<size_t>(per * T, 1) * 4), "policy table");
        cck(cudaMalloc(&D.wst, std::max<size_t>(per * T, 1) * 4), "worst table");
        cck(cudaMemsetAsync(D.vals, 0, P * (T + 1) * 8, D.s), "value table");
        if (!J.reach) { // terminal column: 1 for safety, 0 for reach (synthesis.cpp:177-181)
            std::vector<double> ones(static_cast<size_t>(J.S.n_x), 1.0);
            cck(cudaMemcpyAsync(D.vals + P * T, ones.data(), ones.size() * 8, cudaMemcpyHostToDevice, D.s), "terminal");
            cck(cudaStreamSynchronize(D.s), "terminal");
        }
        if (J.n > 1 && J.exchange != GM_XCHG_ALLGATHER) {
            int64_t lo = 0, hi = 0;
            sck(gm_shard_reach(D.model, x0, x1, &lo, &hi, &st), st);
            J.reach_iv[static_cast<size_t>(d)] = {lo, hi};
        }
    });
    if (!J.sync_ok()) return;
    if (d == 0 && J.n > 1) { // the exchange plan from every device's reach (fixed for the model)
        if (J.exchange == GM_XCHG_ALLGATHER)
            for (int r = 0; r < J.n; ++r) J.reach_iv[static_cast<size_t>(r)] = {0, J.S.n_x};
        J.X = plan_exchange(J.S, J.reach_iv, J.exchange);
    }
    if (!J.sync_ok()) return;
    // stage (i): this device's rows (matrix mode), fused target-hit vector
    ok = step_guard(J, [&] {
        gm_status st{};
        cck(cudaEventRecord(D.t0, D.s), "event");
        if (J.matrix) sck(gm_build_shard(D.model, x0, x1, &D.tm, &st), st);
        cck(cudaEventRecord(D.t1, D.s), "event");
    });
    if (!J.sync_ok()) return;
    // stage (ii): T backward steps, V exchanged after each
    // NCCL also runs for one device (a one-rank in-place all-gather): the transport
    // is then exercised on any machine with a GPU
    const bool use_nccl = J.transport == GM_XPORT_NCCL, use_store = J.transport == GM_XPORT_STORE;
    for (int k = T - 1; k >= 0; --k) {
        ok = step_guard(J, [&] {
            gm_status st{};
            if (use_store && J.n > 1) {
                const gmk::GmMirror mir = mirrors_for(J, d, k);
                sck(gmi_step_device_mirrored(D.model, D.tm, x0, x1, D.vals + P * (k + 1), D.vals + P * k + x0,
                                             D.pol + per * k, D.wst + per * k, D.s, &mir, &st),
                    st);
            } else {
                sck(gm_step_device(D.model, D.tm, x0, x1, D.vals + P * (k + 1), D.vals + P * k + x0, D.pol + per * k,
                                   D.wst + per * k, D.s, &st),
                    st);
            }
            if (k == T - 1) { // device errors (domain, quadrature) surface after the first step
                cck(cudaStreamSynchronize(D.s), "bellman step");
                sck(gm_check_device_errors(D.model, &st), st);
            }
            if (J.n > 1 && !use_nccl) cck(cudaEventRecord(D.step_ev[static_cast<size_t>(k)], D.s), "step event");
        });
        if (k == T - 1 || !use_nccl) {
            // the first step is a collective error check; the peer transport needs every
            // device's step event recorded before it is waited on
            if (!J.sync_ok()) return;
        }
        if (J.n > 1 || use_nccl) {
            ok = step_guard(J, [&] {
                if (use_nccl) exchange_nccl(J, d, k);
                else if (use_store) exchange_store(J, d, k);
                else exchange_peer(J, d, k);
            });
            if (!ok) { // NCCL peers cannot continue without this device: stop everyone at the next sync
                if (use_nccl) return;
            }
        }
    }
    ok = step_guard(J, [&] {
        cck(cudaEventRecord(D.t2, D.s), "event");
        // this device's columns into the host result (column-major n_x x (T+1) / n_x x T)
        if (x1 > x0 && T > 0) {
            const size_t w = static_cast<size_t>(x1 - x0);
            const size_t nx = static_cast<size_t>(J.S.n_x);
            cck(cudaMemcpy2DAsync(J.h_vals + x0, nx * 8, D.vals + x0, P * 8, w * 8, static_cast<size_t>(T),
                                  cudaMemcpyDeviceToHost, D.s),
                "values");
            cck(cudaMemcpy2DAsync(J.h_pol + x0, nx * 4, D.pol, per * 4, w * 4, static_cast<size_t>(T),
                                  cudaMemcpyDeviceToHost, D.s),
                "policy");
            cck(cudaMemcpy2DAsync(J.h_wst + x0, nx * 4, D.wst, per * 4, w * 4, static_cast<size_t>(T),
                                  cudaMemcpyDeviceToHost, D.s),
                "worst");
        }
        cck(cudaStreamSynchronize(D.s), "sweep");
        gm_status st{};
        sck(gm_check_device_errors(D.model, &st), st);
        cck(cudaEventElapsedTime(&D.build_ms, D.t0, D.t1), "timing");
        cck(cudaEventElapsedTime(&D.sweep_ms, D.t1, D.t2), "timing");
    });
    (void)ok;
}

} // namespace

gm_code gm_synthesize_multi(gm_model* m, int32_t n_dev, const int32_t* devices, int32_t exchange, int32_t transport,
                            gm_result** out, gm_multi_stats* stats, gm_status* st) {
    return gmi_guarded(st, [&] {
        if (n_dev < 1) throw std::out_of_range("synthesize_multi: at least one device");
        if (exchange < GM_XCHG_AUTO || exchange > GM_XCHG_ALLGATHER)
            gmi_throw(GM_ERR_CONFIG, "synthesize_multi: unknown exchange");
        if (transport != GM_XPORT_NCCL && transport != GM_XPORT_PEER && transport != GM_XPORT_STORE)
            gmi_throw(GM_ERR_CONFIG, "synthesize_multi: unknown transport");
        if (transport == GM_XPORT_STORE && n_dev > gmk::kMaxMirrors + 1)
            gmi_throw(GM_ERR_CONFIG, "synthesize_multi: the store transport handles at most 9 devices");
        gm_sizes sz;
        gm_status s2{};
        sck(gm_model_sizes(m, &sz, &s2), s2);
        // the reference's budget check (synthesis.cpp:217-223) on the whole model
        if (sz.mode == GM_MODE_MATRIX && sz.mem_budget != 0 && sz.memory_estimate > static_cast<uint64_t>(sz.mem_budget))
            gmi_throw(GM_ERR_MEMORY, "matrix mode needs " + std::to_string(sz.memory_estimate) +
                                         " bytes but the budget is " + std::to_string(sz.mem_budget) + "; use ofa mode");
        int count = 0;
        if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
            cudaGetLastError();
            gmi_throw(GM_ERR_CUDA, "no CUDA device available: the B200 engine has no CPU fallback");
        }
        Job J(n_dev);
        J.m = m;
        J.exchange = exchange;
        J.transport = transport;
        for (int i = 0; i < n_dev; ++i) {
            const int dv = devices ? devices[i] : i;
            if (dv < 0 || dv >= count) throw std::out_of_range("synthesize_multi: device " + std::to_string(dv));
            J.devices.push_back(dv);
        }
        J.S.n_x = sz.n_states;
        J.S.n = n_dev;
        J.S.per = (sz.n_states + n_dev - 1) / n_dev;
        J.P = J.S.per * n_dev;
        J.T = sz.horizon;
        J.reach = sz.spec_kind != GM_SAFETY;
        J.matrix = sz.mode == GM_MODE_MATRIX;
        J.reach_iv.assign(static_cast<size_t>(n_dev), {0, 0});
        if (transport == GM_XPORT_NCCL) {
            const Nccl& N = nccl();
            if (!N.ok) gmi_throw(GM_ERR_CUDA, N.why + " (use the peer transport)");
            std::vector<int> sorted = J.devices;
            std::sort(sorted.begin(), sorted.end());
            if (std::adjacent_find(sorted.begin(), sorted.end()) != sorted.end())
                gmi_throw(GM_ERR_CONFIG, "synthesize_multi: NCCL needs distinct devices (the peer transport accepts repeats)");
            J.comms.resize(static_cast<size_t>(n_dev));
            nck(N.commInitAll(J.comms.data(), n_dev, J.devices.data()), "ncclCommInitAll");
        }
        if (transport == GM_XPORT_PEER || transport == GM_XPORT_STORE) // direct NVLink access between the pairs
            for (int a : J.devices)
                for (int b : J.devices) {
                    if (a == b) continue;
                    int can = 0;
                    if (cudaDeviceCanAccessPeer(&can, a, b) == cudaSuccess && can) {
                        cudaSetDevice(a);
                        if (cudaDeviceEnablePeerAccess(b, 0) != cudaSuccess) cudaGetLastError(); // already enabled
                    } else if (transport == GM_XPORT_STORE) {
                        cudaGetLastError();
                        gmi_throw(GM_ERR_CUDA, "synthesize_multi: the store transport needs peer access between "
                                               "devices " + std::to_string(a) + " and " + std::to_string(b));
                    }
                }
        // absorbing flags (spec.cpp:51-60) from the caller's model, then the host result
        std::vector<uint8_t> absorbing(static_cast<size_t>(sz.n_states));
        cck(cudaSetDevice(J.devices[0]), "cudaSetDevice");
        sck(gm_absorbing_states(m, absorbing.data(), &s2), s2);
        std::unique_ptr<gm_result, void (*)(gm_result*)> res(gmi_result_new(m, sz.mode, absorbing.data()), gm_result_free);
        gmi_result_tables(res.get(), &J.h_vals, &J.h_pol, &J.h_wst);
        for (int i = 0; i < n_dev; ++i) {
            J.dev.emplace_back(new Dev);
            J.dev.back()->device = J.devices[static_cast<size_t>(i)];
        }
        {
            std::vector<std::thread> th;
            for (int i = 0; i < n_dev; ++i) th.emplace_back(device_main, std::ref(J), i);
            for (auto& t : th) t.join();
        }
        for (ncclComm_t c : J.comms) nccl().commDestroy(c);
        if (J.failed) gmi_throw(J.err.code, J.err.msg);
        if (stats) {
            std::memset(stats, 0, sizeof *stats);
            for (auto& D : J.dev) {
                stats->build_ms = std::max(stats->build_ms, static_cast<double>(D->build_ms));
                stats->sweep_ms = std::max(stats->sweep_ms, static_cast<double>(D->sweep_ms));
            }
            stats->halo_states = J.X.halo_states;
            stats->allgather_states = J.X.ag_states;
            stats->exchange_used = (n_dev > 1 || transport == GM_XPORT_NCCL) ? (J.X.halo ? GM_XCHG_HALO : GM_XCHG_ALLGATHER) : 0;
            stats->transport_used = transport;
            stats->n_devices = n_dev;
        }
        J.dev.clear();
        cudaSetDevice(J.devices[0]);
        *out = res.release();
    });
}
