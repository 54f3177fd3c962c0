// C ABI of libgridmdp_b200.so (include/gridmdp_b200.h): model lifetime, device
// residency, stage (i)/(ii) orchestration over the kernels in gm_kernels.cu,
// and the reference's container formats (io.cpp:142-256).
#include "gridmdp_b200.h"

#include "gm_host.hpp"
#include "gm_internal.hpp"
#include "gm_jit.hpp"
#include "gm_kernels.cuh"

#include <cuda_runtime.h>

#include <atomic>
#include <charconv>
#include <climits>
#include <cstring>
#include <exception>
#include <functional>
#include <fstream>
#include <map>
#include <memory>
#include <mutex>
#include <sstream>
#include <thread>
#include <tuple>
#include <vector>

using namespace gmh;

// ===========================================================================
// status plumbing
// ===========================================================================

namespace {

void put_status(gm_status* st, int code, const std::string& msg, int64_t row = -1, int parse = 0) {
    if (!st) return;
    st->code = code;
    st->is_parse = parse;
    st->first_bad_row = row;
    std::strncpy(st->msg, msg.c_str(), sizeof(st->msg) - 1);
    st->msg[sizeof(st->msg) - 1] = '\0';
}

struct DomainAt : DomainErr {
    int64_t row;
    DomainAt(const std::string& m, int64_t r) : DomainErr(m), row(r) {}
};

template <class F>
gm_code guarded(gm_status* st, F&& f) {
    put_status(st, GM_OK, "");
    try {
        f();
        return GM_OK;
    } catch (const ParseErr& e) {
        put_status(st, GM_ERR_CONFIG, e.what(), -1, 1);
        return GM_ERR_CONFIG;
    } catch (const ConfigErr& e) {
        put_status(st, GM_ERR_CONFIG, e.what());
        return GM_ERR_CONFIG;
    } catch (const MemoryErr& e) {
        put_status(st, GM_ERR_MEMORY, e.what());
        return GM_ERR_MEMORY;
    } catch (const DomainAt& e) {
        put_status(st, GM_ERR_DOMAIN, e.what(), e.row);
        return GM_ERR_DOMAIN;
    } catch (const DomainErr& e) {
        put_status(st, GM_ERR_DOMAIN, e.what());
        return GM_ERR_DOMAIN;
    } catch (const IoErr& e) {
        put_status(st, GM_ERR_IO, e.what());
        return GM_ERR_IO;
    } catch (const std::out_of_range& e) {
        put_status(st, GM_ERR_RANGE, e.what());
        return GM_ERR_RANGE;
    } catch (const CudaErr& e) {
        put_status(st, GM_ERR_CUDA, e.what());
        return GM_ERR_CUDA;
    } catch (const std::bad_alloc&) {
        put_status(st, GM_ERR_MEMORY, "host allocation failed");
        return GM_ERR_MEMORY;
    } catch (const std::exception& e) {
        put_status(st, GM_ERR_OTHER, e.what());
        return GM_ERR_OTHER;
    }
}

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        cudaGetLastError();
        if (e == cudaErrorMemoryAllocation)
            throw MemoryErr(std::string(what) + ": device allocation failed (" + cudaGetErrorString(e) + ")");
        throw CudaErr(std::string(what) + ": " + cudaGetErrorString(e));
    }
}

// Large device blocks (stored matrices: tens of GB) are cached on release and
// reused by the next allocation of a similar size on the same device, so
// repeated synthesize/build calls do not pay cudaMalloc/cudaFree of the matrix
// (hundreds of ms at 100 GB). On allocation failure the cache is flushed first.
constexpr size_t kCacheMin = 1ULL << 20; // smaller blocks: cudaMalloc/cudaFree (cudaFree synchronises the device)
std::mutex g_cache_mu;
std::multimap<size_t, std::pair<int, void*>> g_cache; // bytes -> (device, ptr)

void flush_cache() {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    int cur = 0;
    cudaGetDevice(&cur);
    for (auto& kv : g_cache) {
        cudaSetDevice(kv.second.first);
        cudaFree(kv.second.second);
    }
    g_cache.clear();
    cudaSetDevice(cur);
}

size_t cached_bytes() {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_cache_mu);
    size_t s = 0;
    for (auto& kv : g_cache)
        if (kv.second.first == dev) s += kv.first;
    return s;
}

void* dev_alloc(size_t bytes, size_t& got, const char* what) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (bytes >= kCacheMin) {
        std::lock_guard<std::mutex> lk(g_cache_mu);
        for (auto it = g_cache.lower_bound(bytes); it != g_cache.end() && it->first <= bytes + bytes / 4; ++it) {
            if (it->second.first != dev) continue;
            void* p = it->second.second;
            got = it->first;
            g_cache.erase(it);
            return p;
        }
    }
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        flush_cache();
        e = cudaMalloc(&p, bytes);
    }
    ck(e, what);
    got = bytes;
    return p;
}

void dev_free(void* p, size_t bytes) {
    if (!p) return;
    if (bytes >= kCacheMin) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceSynchronize(); // no queued kernel may still use the block once it is reusable
        std::lock_guard<std::mutex> lk(g_cache_mu);
        g_cache.emplace(bytes, std::make_pair(dev, p));
        return;
    }
    cudaFree(p);
}

template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;      // elements usable
    size_t bytes = 0;  // allocated bytes
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void release() {
        dev_free(p, bytes);
        p = nullptr;
        n = 0;
        bytes = 0;
    }
    void ensure(size_t count, const char* what) {
        if (count <= n && p) return;
        release();
        if (count == 0) count = 1;
        // +16 bytes: bulk async copies may read a 16-byte aligned superset of the last row
        p = static_cast<T*>(dev_alloc(count * sizeof(T) + 16, bytes, what));
        n = count;
    }
};

// ---------------------------------------------------------------- timing
std::atomic<long long> g_launches{0};
std::mutex g_tmu;
bool g_timing = false;
double g_total_ms[gmk::KF_COUNT] = {};
double g_last_ms[gmk::KF_COUNT] = {};
long long g_fam_launches[gmk::KF_COUNT] = {};
std::vector<std::tuple<int, cudaEvent_t, cudaEvent_t>> g_pending;
std::vector<cudaEvent_t> g_pool;

cudaEvent_t take_event() {
    if (!g_pool.empty()) {
        cudaEvent_t e = g_pool.back();
        g_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    ck(cudaEventCreate(&e), "cudaEventCreate");
    return e;
}

void collect_timing() {
    std::lock_guard<std::mutex> lk(g_tmu);
    for (auto& [fam, a, b] : g_pending) {
        cudaEventSynchronize(b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        g_total_ms[fam] += ms;
        g_last_ms[fam] = ms;
        g_pool.push_back(a);
        g_pool.push_back(b);
    }
    g_pending.clear();
}

struct Launch {
    int fam;
    cudaStream_t s;
    cudaEvent_t a = nullptr, b = nullptr;
    Launch(int f, cudaStream_t st) : fam(f), s(st) {
        ++g_launches;
        {
            std::lock_guard<std::mutex> lk(g_tmu);
            ++g_fam_launches[fam];
        }
        if (g_timing) {
            std::lock_guard<std::mutex> lk(g_tmu);
            a = take_event();
            b = take_event();
            cudaEventRecord(a, s);
        }
    }
    ~Launch() {
        if (a) {
            cudaEventRecord(b, s);
            std::lock_guard<std::mutex> lk(g_tmu);
            g_pending.emplace_back(fam, a, b);
        }
    }
};

} // namespace

// ===========================================================================
// opaque handles
// ===========================================================================

struct gm_model {
    Model M;
    GmDev D{};
    int device = -1;
    cudaStream_t stream = nullptr;
    cudaStream_t own_stream = nullptr; // the model's stream when a caller stream is in use
    DevBuf<GmIns> d_prog;
    DevBuf<double> d_lits;
    DevBuf<int> d_lines;
    DevBuf<uint8_t> d_absorb;
    DevBuf<unsigned long long> d_err;
    // step scratch
    DevBuf<double> d_mass[2], d_t0x[2], d_vin, d_chunk;
    DevBuf<long long> d_origin[2];
    DevBuf<uint8_t> d_rowflag[2];
    DevBuf<long long> d_reach; // origin min / max (gm_shard_reach)
    cudaStream_t aux = nullptr; // producer stream of the row-prologue pipeline
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_ready[2] = {}, ev_used[2] = {};
    bool dev_ready = false;
    bool absorb_ready = false;
    // run-time compiled row kernels (gm_jit.cpp): state of the last row-kernel launch
    bool jit_used = false;
    double jit_compile_s = 0.0;
    std::string jit_why;
    // device time of the last gm_synthesize* (stage i / stage ii), ms
    double last_build_ms = 0.0, last_sweep_ms = 0.0;
    // OFA row prologue results (per-axis cell masses, origins, T0x, row flags) of the
    // rows [ofa_r0, ofa_r0 + ofa_n), kept across the steps of a sweep: a step depends
    // on V only, so steps 2..T recompute every row's T(x'|x,u) from the cached 1-D
    // masses (Σ W_d doubles per row, never the R-wide row) without re-running the
    // dynamics and the CDFs. Invalidated when the spec changes (refresh_device).
    DevBuf<double> ofa_mass, ofa_t0x;
    DevBuf<long long> ofa_origin;
    DevBuf<uint8_t> ofa_flag;
    int64_t ofa_r0 = -1, ofa_n = 0, ofa_chunk = 0;
    bool ofa_valid = false;
    bool ofa_cache_steps = false; // set by the multi-step drivers (run_backward, gm_step_device)
};

// Row kernels with the dynamics compiled for this model, or nullptr (interpreter).
// GM_JIT=1 forces run-time compiled kernels, 0 disables them; unset: used when
// the launch covers >= 2^21 rows (a first compile costs 2-5 s, cached per process).
// Run-time compilation costs 2-8 s on first use (then cached in the process and on
// disk), so it is used for launches big enough to repay it: >= 2^21 rows, or >= 2^32
// row entries (the C5 half-matrix shard, 1.97 M rows x 7,000: build 26.1 -> 19.1 ms)
static bool jit_worth_it(const gm_model* m, int64_t rows) {
    return rows >= (int64_t(1) << 21) || static_cast<double>(rows) * static_cast<double>(m->D.R) >= 4294967296.0;
}

static const gmj::Kernels* jit_kernels(gm_model* m, int want, int64_t rows) {
    std::string why;
    if (m->M.noise.family == GM_CUSTOM) { // the quadrature kernels interpret the pdf
        m->jit_used = false;
        m->jit_why = "not used: custom densities run the bytecode interpreter";
        return nullptr;
    }
    const char* env = std::getenv("GM_JIT");
    if (!env && !jit_worth_it(m, rows)) {
        m->jit_used = false;
        m->jit_why = "not used: fewer than 2^21 rows and 2^32 row entries in the launch (GM_JIT=1 forces it)";
        return nullptr;
    }
    // the build kernel is specialised to the row shape when it qualifies (GM_JIT_SHAPE=0: off)
    static const char* js = std::getenv("GM_JIT_SHAPE");
    const std::string shape =
        (want & gmj::WANT_BUILD_QS) && !(js && js[0] == '0') ? gmj::shape_defines(m->D) : std::string();
    const gmj::Kernels* k = gmj::kernels_for(m->M.prog, m->M.X.dim(), m->M.U.dim(), m->M.W.dim(), want, &why, shape,
                                             gmk::build_ctas(m->D, true));
    m->jit_used = k != nullptr;
    m->jit_why = k ? std::string() : why;
    m->jit_compile_s = k ? k->compile_s : 0.0;
    return k;
}

// The OFA consumer compiled for the model's row shape (gm_jit.cpp ofa_kernel), or
// nullptr: same policy as jit_kernels (GM_JIT=1 forces, 0 disables, unset:
// jit_worth_it); GM_OFA_SHAPE=0 keeps the ahead-of-time consumers.
static const gmk::OfaJit* ofa_jit(gm_model* m, int64_t rows, gmk::OfaJit& out) {
    static const char* off = std::getenv("GM_OFA_SHAPE");
    if (off && off[0] == '0') return nullptr;
    const char* env = std::getenv("GM_JIT");
    // a sweep runs the consumer once per step (C3b, 0.28 M rows x 7,776 x 8 steps:
    // 21.0 -> 14.0 ms with the per-group kernel)
    const int64_t steps = m->ofa_cache_steps ? std::max(1, m->M.spec.horizon) : 1;
    if ((env && env[0] == '0') || (!env && !jit_worth_it(m, rows * steps))) return nullptr;
    if (m->M.noise.family == GM_CUSTOM) return nullptr;
    std::string why;
    double cs = 0.0;
    out.shape = gmj::ofa_kernel(gmj::ofa_shape_defines(m->D), &cs, &why, &out.packed, &out.group);
    return out.shape ? &out : nullptr;
}

struct gm_matrix {
    int device = -1;
    int64_t row_begin = 0, row_end = 0, R = 0;
    int64_t pitch = 0; // row stride of `probs` in doubles (>= R, zero padding)
    DevBuf<double> probs;
    DevBuf<long long> origins;
    DevBuf<double> t0x; // optional (shard builds for reach specs)
    bool has_t0x = false;
    bool masked = false;
    // read_matrix containers carry their own shape (io.cpp:262-276), checked against a model
    bool has_meta = false;
    Grid X;
    int64_t n_u = 0, n_w = 0;
    std::vector<int64_t> extents;
};

// Host tables that are filled by copies: resize() leaves the elements
// uninitialised (no zero pass over hundreds of MB before the device copy).
template <class T>
struct NoInitAlloc : std::allocator<T> {
    using value_type = T;
    template <class U>
    struct rebind {
        using other = NoInitAlloc<U>;
    };
    NoInitAlloc() = default;
    template <class U>
    NoInitAlloc(const NoInitAlloc<U>&) noexcept {}
    template <class U>
    void construct(U* p) noexcept {
        ::new (static_cast<void*>(p)) U;
    }
    template <class U, class... A>
    void construct(U* p, A&&... a) {
        ::new (static_cast<void*>(p)) U(std::forward<A>(a)...);
    }
};
template <class T>
using HostVec = std::vector<T, NoInitAlloc<T>>;

struct gm_result {
    Model meta; // grids, spec, gamma for the container
    int mode = 0;
    int64_t n_x = 0;
    int T = 0;
    HostVec<double> values;      // n_x x (T+1), column-major
    HostVec<uint32_t> policy;    // n_x x T, column-major
    HostVec<uint32_t> worst;     // n_x x T, column-major
    HostVec<uint8_t> absorbing;  // n_x (reach) or empty
};

namespace {

struct ManifestR { // io.cpp:72-121
    std::map<std::string, std::string> kv;
    ManifestR(std::istream& is, const char* magic) {
        std::string line;
        if (!std::getline(is, line)) throw IoErr("empty container");
        std::istringstream head(line);
        std::string mg;
        int version = 0;
        head >> mg >> version;
        if (mg != magic) throw IoErr("bad magic line '" + line + "'");
        if (version != 1) throw IoErr("unsupported container version " + std::to_string(version));
        while (std::getline(is, line)) {
            if (line == "payload") return;
            const auto eq = line.find('=');
            if (eq == std::string::npos || line.empty() || line.back() != ';')
                throw IoErr("malformed manifest line '" + line + "'");
            auto trim = [](std::string s) {
                const auto b = s.find_first_not_of(" \t");
                const auto e = s.find_last_not_of(" \t");
                return b == std::string::npos ? std::string{} : s.substr(b, e - b + 1);
            };
            kv[trim(line.substr(0, eq))] = trim(line.substr(eq + 1, line.size() - eq - 2));
        }
        throw IoErr("missing payload marker");
    }
    bool has(const std::string& k) const { return kv.count(k) != 0; }
    const std::string& str(const std::string& k) const {
        auto it = kv.find(k);
        if (it == kv.end()) throw IoErr("manifest key '" + k + "' missing");
        return it->second;
    }
    int64_t integer(const std::string& k) const { return std::stoll(str(k)); }
    double number(const std::string& k) const { return std::stod(str(k)); }
    std::vector<double> vec(const std::string& k) const {
        const std::string& s = str(k);
        if (s.size() < 2 || s.front() != '{' || s.back() != '}')
            throw IoErr("manifest key '" + k + "' is not a vector");
        std::vector<double> out;
        std::istringstream iss(s.substr(1, s.size() - 2));
        std::string item;
        while (std::getline(iss, item, ',')) out.push_back(std::stod(item));
        return out;
    }
    Grid grid(const std::string& prefix) const {
        if (integer(prefix + ".dim") == 0) return grid_from({}, {}, {});
        return grid_from(vec(prefix + ".lb"), vec(prefix + ".ub"), vec(prefix + ".eta"));
    }
};

std::vector<int> line_offsets(const GmDev& D) {
    // relative flat offset of every slab line (all axes but the last, row-major)
    std::vector<int> out(static_cast<size_t>(D.n_lines), 0);
    const int lead = D.n - 1; // real axes before the last
    for (int L = 0; L < D.n_lines; ++L) {
        long long rem = L, off = 0;
        for (int d = lead - 1; d >= 0; --d) {
            const long long j = rem % D.W[d];
            rem /= D.W[d];
            off += j * D.xstride[d];
        }
        out[static_cast<size_t>(L)] = static_cast<int>(off);
    }
    return out;
}

void ensure_device(gm_model* m) {
    if (m->dev_ready) {
        ck(cudaSetDevice(m->device), "cudaSetDevice");
        return;
    }
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) {
        cudaGetLastError();
        throw CudaErr("no CUDA device available: the B200 engine has no CPU fallback");
    }
    int dev = 0;
    ck(cudaGetDevice(&dev), "cudaGetDevice");
    m->device = dev;
    ck(cudaStreamCreateWithFlags(&m->stream, cudaStreamNonBlocking), "cudaStreamCreate");
    const Program& P = m->M.prog;
    m->d_prog.ensure(P.code.size(), "program");
    if (!P.code.empty())
        ck(cudaMemcpy(m->d_prog.p, P.code.data(), P.code.size() * sizeof(GmIns), cudaMemcpyHostToDevice), "program");
    m->d_lits.ensure(P.lits.size(), "literals");
    if (!P.lits.empty())
        ck(cudaMemcpy(m->d_lits.p, P.lits.data(), P.lits.size() * sizeof(double), cudaMemcpyHostToDevice), "literals");
    m->d_err.ensure(1, "error slot");
    const unsigned long long none = ULLONG_MAX;
    ck(cudaMemcpy(m->d_err.p, &none, sizeof none, cudaMemcpyHostToDevice), "error slot");
    m->dev_ready = true;
}

// descriptor refresh after spec/model changes; uploads the line table and
// absorbing flags (absorbing_states, spec.cpp:51-60 -> k_absorb)
void refresh_device(gm_model* m) {
    ensure_device(m);
    m->ofa_valid = false; // T0x and the absorbed-row flags depend on the spec
    if (m->M.R > INT_MAX) throw MemoryErr("row width exceeds the device limit");
    m->D = m->M.device_descriptor();
    {
        // slab offsets (line table, element tables, V gathers) are 32-bit relative to
        // the row's 64-bit origin: the slab's flat span must fit
        long long span = 0;
        for (int d = 0; d < m->D.n; ++d) span += static_cast<long long>(m->D.W[d] - 1) * m->D.xstride[d];
        if (span > INT_MAX) throw MemoryErr("slab span exceeds the device's 32-bit offset range");
    }
    m->D.prog = m->d_prog.p;
    m->D.lits = m->d_lits.p;
    const std::vector<int> lines = line_offsets(m->D);
    m->d_lines.ensure(lines.size(), "line table");
    ck(cudaMemcpy(m->d_lines.p, lines.data(), lines.size() * sizeof(int), cudaMemcpyHostToDevice), "line table");
    m->D.line_off = m->d_lines.p;
    m->D.absorb = nullptr;
    if (m->M.spec.reach()) {
        m->d_absorb.ensure(static_cast<size_t>(m->M.n_x()), "absorbing flags");
        {
            Launch L(gmk::KF_MISC, m->stream);
            gmk::absorb_flags(m->D, m->d_absorb.p, m->stream);
        }
        m->D.absorb = m->d_absorb.p;
    }
    ck(cudaStreamSynchronize(m->stream), "absorbing flags");
    m->absorb_ready = true;
}

void prepare(gm_model* m) {
    if (!m->dev_ready || !m->absorb_ready) refresh_device(m);
    else ck(cudaSetDevice(m->device), "cudaSetDevice");
}

// Raises the reference's DomainError for the lowest failing row, if any.
void raise_device_error(gm_model* m) {
    unsigned long long row = ULLONG_MAX;
    ck(cudaMemcpy(&row, m->d_err.p, sizeof row, cudaMemcpyDeviceToHost), "error slot");
    if (row == ULLONG_MAX) return;
    const unsigned long long none = ULLONG_MAX;
    ck(cudaMemcpy(m->d_err.p, &none, sizeof none, cudaMemcpyHostToDevice), "error slot");
    std::vector<double> mu;
    try {
        m->M.row_image(static_cast<int64_t>(row), mu);
    } catch (const DomainErr& e) {
        throw DomainAt(e.what(), static_cast<int64_t>(row));
    }
    if (m->M.noise.family == GM_CUSTOM)
        throw DomainAt("adaptive_simpson: quadrature did not converge", static_cast<int64_t>(row));
    throw DomainAt("inc_beta: continued fraction did not converge", static_cast<int64_t>(row));
}

int64_t chunk_rows(const gm_model* m) {
    // 32 MB of per-axis masses per scratch buffer: two buffers stay L2-resident
    // next to V while the prologue of chunk c+1 overlaps the consumer of chunk c
    const int64_t per_row = static_cast<int64_t>(m->D.sumW) * 8 + 8 + 8 + 1;
    int64_t c = (32LL << 20) / std::max<int64_t>(per_row, 1);
    c = std::max<int64_t>(c, 4096);
    return c;
}

void ensure_scratch(gm_model* m, int64_t chunk) {
    for (int b = 0; b < 2; ++b) {
        m->d_mass[b].ensure(static_cast<size_t>(chunk) * std::max(m->D.sumW, 1), "mass scratch");
        m->d_origin[b].ensure(static_cast<size_t>(chunk), "origin scratch");
        m->d_t0x[b].ensure(static_cast<size_t>(chunk), "t0x scratch");
        m->d_rowflag[b].ensure(static_cast<size_t>(chunk), "row flags");
    }
    if (!m->aux) {
        int lo = 0, hi = 0; // the producer (row prologue) gets the higher priority
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        ck(cudaStreamCreateWithPriority(&m->aux, cudaStreamNonBlocking, hi), "aux stream");
        for (cudaEvent_t* e : {&m->ev_fork, &m->ev_join, &m->ev_ready[0], &m->ev_ready[1], &m->ev_used[0],
                               &m->ev_used[1]})
            ck(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "pipeline events");
    }
}

// Producer/consumer pipeline over row chunks: the row prologue of chunk c runs on
// the aux stream into scratch buffer c&1 while the consumer of chunk c-1 runs on
// `s`; `consume(c0, cn, buf)` enqueues the consumer of one chunk on `s`.
template <class Produce, class Consume>
void pipeline(gm_model* m, int64_t n, int64_t chunk, cudaStream_t s, Produce&& produce, Consume&& consume) {
    ck(cudaEventRecord(m->ev_fork, s), "fork");
    ck(cudaStreamWaitEvent(m->aux, m->ev_fork, 0), "fork");
    int64_t c = 0;
    for (int64_t c0 = 0; c0 < n; c0 += chunk, ++c) {
        const int64_t cn = std::min(chunk, n - c0);
        const int b = static_cast<int>(c & 1);
        if (c >= 2) ck(cudaStreamWaitEvent(m->aux, m->ev_used[b], 0), "reuse");
        produce(c0, cn, b);
        ck(cudaEventRecord(m->ev_ready[b], m->aux), "ready");
        ck(cudaStreamWaitEvent(s, m->ev_ready[b], 0), "ready");
        consume(c0, cn, b);
        ck(cudaEventRecord(m->ev_used[b], s), "used");
    }
    ck(cudaEventRecord(m->ev_join, m->aux), "join");
    ck(cudaStreamWaitEvent(s, m->ev_join, 0), "join");
}

// A matrix used with a model must have its row shape (and, when read from a
// container, its grid, input / disturbance counts and window).
void check_matrix_model(const gm_matrix* tm, const gm_model* m) {
    bool ok = tm->R == m->M.R && tm->pitch == m->D.pitch && tm->row_end <= m->M.rows();
    if (ok && tm->has_meta)
        ok = tm->X.lb == m->M.X.lb && tm->X.ub == m->M.X.ub && tm->X.eta == m->M.X.eta && tm->n_u == m->M.n_u() &&
             tm->n_w == m->M.n_w() && tm->extents == m->M.extents;
    if (!ok) throw ConfigErr("the transition matrix does not match the model (grid, counts or window)");
}

// Stage (i) for rows [r0, r1): origins + probabilities (+ T0x for reach shards)
void build_rows(gm_model* m, int64_t r0, int64_t r1, gm_matrix* tm, bool want_t0x) {
    const int64_t n = r1 - r0;
    tm->device = m->device;
    tm->row_begin = r0;
    tm->row_end = r1;
    tm->R = m->M.R;
    tm->pitch = m->D.pitch;
    const uint64_t cells = mul_checked(static_cast<uint64_t>(n), static_cast<uint64_t>(tm->pitch), "matrix size");
    tm->probs.ensure(cells, "matrix payload");
    tm->origins.ensure(static_cast<size_t>(n), "matrix origins");
    if (want_t0x) {
        tm->t0x.ensure(static_cast<size_t>(n), "target-hit vector");
        tm->has_t0x = true;
    }
    const gmj::Kernels* J =
        jit_kernels(m, gmk::build_uses_qs(m->D) ? gmj::WANT_BUILD_QS : gmj::WANT_BUILD_NOQS, n);
    {
        Launch L(gmk::KF_BUILD, m->stream);
        static const char* sl = std::getenv("GM_BUILD_SLICES");
        const int64_t slices = sl ? std::max(1, std::atoi(sl)) : 1;
        const int64_t per = (n + slices - 1) / slices;
        for (int64_t c0 = 0; c0 < n; c0 += per) {
            const int64_t cn = std::min(per, n - c0);
            gmk::build(m->D, r0 + c0, cn, tm->origins.p + c0, want_t0x ? tm->t0x.p + c0 : nullptr,
                       tm->probs.p + c0 * tm->pitch, m->d_err.p, m->stream, J ? J->build_ws : nullptr);
        }
    }
    ck(cudaStreamSynchronize(m->stream), "build");
    raise_device_error(m);
}

// OFA step from cached row prologue results. The first step of rows [r0, r0+n) runs
// the usual prologue / consumer pipeline with the prologue writing into the cache
// (one slot per chunk); later steps launch only the consumers. Off when GM_OFA_CACHE=0,
// for one-off steps (m->ofa_cache_steps unset) or when the cache would not leave a
// quarter of the device free. Returns false when the caller must run the plain path.
bool ofa_cached_step(gm_model* m, int64_t r0, int64_t n, const double* v_next, cudaStream_t s) {
    static const char* env = std::getenv("GM_OFA_CACHE");
    if ((env && env[0] == '0') || !m->ofa_cache_steps || m->M.noise.family == GM_CUSTOM) return false;
    const int64_t chunk = std::min(chunk_rows(m), n);
    const size_t sumW = static_cast<size_t>(std::max(m->D.sumW, 1));
    const bool hit = m->ofa_valid && m->ofa_r0 == r0 && m->ofa_n == n && m->ofa_chunk == chunk;
    if (!hit) {
        const uint64_t need = static_cast<uint64_t>(n) * (sumW * 8 + 8 + 8 + 1);
        size_t free_b = 0, total_b = 0;
        ck(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
        free_b += cached_bytes();
        if (need + total_b / 4 > free_b) return false;
        m->ofa_valid = false;
        m->ofa_mass.ensure(static_cast<size_t>(n) * sumW, "OFA mass cache");
        m->ofa_origin.ensure(static_cast<size_t>(n), "OFA origin cache");
        m->ofa_t0x.ensure(static_cast<size_t>(n), "OFA target-hit cache");
        m->ofa_flag.ensure(static_cast<size_t>(n), "OFA row-flag cache");
    }
    const bool reach = m->M.spec.reach();
    double* vin = m->d_vin.p;
    gmk::OfaJit jo;
    const gmk::OfaJit* JO = ofa_jit(m, n, jo);
    if (hit) {
        for (int64_t c0 = 0; c0 < n; c0 += chunk) {
            const int64_t cn = std::min(chunk, n - c0);
            Launch L(gmk::KF_EXPECT_OFA, s);
            gmk::expect_ofa(m->D, cn, m->ofa_mass.p + c0 * sumW, m->ofa_origin.p + c0, m->ofa_t0x.p + c0,
                            m->ofa_flag.p + c0, v_next, vin + c0, s, JO);
        }
        return true;
    }
    // first step: the pipeline of the plain path, prologue results written to the cache
    ensure_scratch(m, chunk); // the aux stream and events
    const gmj::Kernels* J = jit_kernels(m, gmj::WANT_PROLOGUE, n);
    ck(cudaEventRecord(m->ev_fork, s), "fork");
    ck(cudaStreamWaitEvent(m->aux, m->ev_fork, 0), "fork");
    int64_t c = 0;
    for (int64_t c0 = 0; c0 < n; c0 += chunk, ++c) {
        const int64_t cn = std::min(chunk, n - c0);
        const int b = static_cast<int>(c & 1);
        {
            Launch L(gmk::KF_PROLOGUE, m->aux);
            gmk::prologue(m->D, r0 + c0, cn, gmk::PF_SKIP_ABSORBED | gmk::PF_MASSES | (reach ? gmk::PF_T0X : 0),
                          m->ofa_origin.p + c0, m->ofa_t0x.p + c0, m->ofa_flag.p + c0, m->ofa_mass.p + c0 * sumW,
                          m->d_err.p, m->aux, J ? J->prologue : nullptr);
        }
        ck(cudaEventRecord(m->ev_ready[b], m->aux), "ready");
        ck(cudaStreamWaitEvent(s, m->ev_ready[b], 0), "ready");
        Launch L(gmk::KF_EXPECT_OFA, s);
        gmk::expect_ofa(m->D, cn, m->ofa_mass.p + c0 * sumW, m->ofa_origin.p + c0, m->ofa_t0x.p + c0,
                        m->ofa_flag.p + c0, v_next, vin + c0, s, JO);
    }
    ck(cudaEventRecord(m->ev_join, m->aux), "join");
    ck(cudaStreamWaitEvent(s, m->ev_join, 0), "join");
    m->ofa_r0 = r0;
    m->ofa_n = n;
    m->ofa_chunk = chunk;
    m->ofa_valid = true;
    return true;
}

// One backward step over states [x0, x1) (bellman_impl, synthesis.cpp:61-143).
// v_next: full device V (absorbing zeroed); outputs indexed from x0.
// `mir`: the pass-2 epilogue also stores the values into other devices' tables
// (gm_multi.cpp, the "store" transport).
void step_states(gm_model* m, gm_matrix* tm, int64_t x0, int64_t x1, const double* v_next,
                 double* v_out, uint32_t* pol, uint32_t* wst, cudaStream_t s, const gmk::GmMirror* mir = nullptr) {
    const int64_t nuw = m->M.n_u() * m->M.n_w();
    const int64_t r0 = x0 * nuw, r1 = x1 * nuw;
    const int64_t n = r1 - r0;
    m->d_vin.ensure(static_cast<size_t>(std::max<int64_t>(n, 1)), "v_in workspace");
    if (tm) {
        check_matrix_model(tm, m);
        if (m->M.spec.reach() && !tm->has_t0x)
            throw ConfigErr("bellman step: a reach specification needs the matrix's target-hit vector");
        if (tm->row_begin <= r0 && tm->row_end >= r1 && n > 0 && gmk::step_warp_applies(m->D)) {
            Launch L(gmk::KF_EXPECT_MATRIX, s);
            const int64_t rb = r0 - tm->row_begin;
            if (gmk::step_warp(m->D, x0, x1 - x0, tm->probs.p + rb * m->D.pitch, tm->origins.p + rb,
                               tm->has_t0x ? tm->t0x.p + rb : nullptr, v_next, m->d_vin.p, v_out, pol, wst, s, mir))
                return; // both passes done, one warp per state
        }
        if (tm->row_begin <= r0 && tm->row_end >= r1 && n > 0 && !(mir && mir->n) && gmk::step_small_applies(m->D)) {
            Launch L(gmk::KF_EXPECT_MATRIX, s);
            if (gmk::step_small(m->D, x0, x1 - x0, tm->probs.p, r0 - tm->row_begin, tm->origins.p,
                                tm->has_t0x ? tm->t0x.p : nullptr, v_next, m->d_vin.p, v_out, pol, wst, s))
                return; // both passes done (small states)
        }
        if (tm->row_begin > r0 || tm->row_end < r1)
            throw ConfigErr("bellman step: the matrix does not cover the requested states");
        Launch L(gmk::KF_EXPECT_MATRIX, s);
        gmk::expect_matrix(m->D, tm->row_begin, r0 - tm->row_begin, r1 - tm->row_begin, tm->probs.p,
                           tm->origins.p, tm->has_t0x ? tm->t0x.p : nullptr, v_next, m->d_vin.p, s);
    } else if (n > 0 && m->M.noise.family == GM_CUSTOM) {
        // custom densities: rows of a chunk are integrated into a transient matrix
        // (k_build_custom) and dotted with V by the stored-matrix kernel
        const int64_t pitch = m->D.pitch;
        const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(n, (64LL << 20) / 8 / std::max<int64_t>(pitch, 1)));
        ensure_scratch(m, chunk);
        m->d_chunk.ensure(static_cast<size_t>(chunk * pitch), "custom row chunk");
        const bool reach = m->M.spec.reach();
        for (int64_t c0 = 0; c0 < n; c0 += chunk) {
            const int64_t cn = std::min(chunk, n - c0);
            {
                Launch L(gmk::KF_PROLOGUE, s);
                gmk::build_custom(m->D, r0 + c0, cn, m->d_origin[0].p, reach ? m->d_t0x[0].p : nullptr, m->d_chunk.p,
                                  m->d_err.p, s);
            }
            Launch L(gmk::KF_EXPECT_MATRIX, s);
            gmk::expect_matrix(m->D, r0 + c0, 0, cn, m->d_chunk.p, m->d_origin[0].p, reach ? m->d_t0x[0].p : nullptr,
                               v_next, m->d_vin.p + c0, s);
        }
    } else if (n > 0 && ofa_cached_step(m, r0, n, v_next, s)) {
        // consumer only, from the prologue results cached by an earlier step of the sweep
    } else if (n > 0) {
        const int64_t chunk = std::min(chunk_rows(m), n);
        ensure_scratch(m, chunk);
        const bool reach = m->M.spec.reach();
        const gmj::Kernels* J = jit_kernels(m, gmj::WANT_PROLOGUE, n);
        gmk::OfaJit jo;
        const gmk::OfaJit* JO = ofa_jit(m, n, jo);
        pipeline(
            m, n, chunk, s,
            [&](int64_t c0, int64_t cn, int b) {
                Launch L(gmk::KF_PROLOGUE, m->aux);
                gmk::prologue(m->D, r0 + c0, cn, gmk::PF_SKIP_ABSORBED | gmk::PF_MASSES | (reach ? gmk::PF_T0X : 0),
                              m->d_origin[b].p, m->d_t0x[b].p, m->d_rowflag[b].p, m->d_mass[b].p, m->d_err.p,
                              m->aux, J ? J->prologue : nullptr);
            },
            [&](int64_t c0, int64_t cn, int b) {
                Launch L(gmk::KF_EXPECT_OFA, s);
                gmk::expect_ofa(m->D, cn, m->d_mass[b].p, m->d_origin[b].p, m->d_t0x[b].p, m->d_rowflag[b].p,
                                v_next, m->d_vin.p + c0, s, JO);
            });
    }
    Launch L(gmk::KF_MAXMIN, s);
    gmk::maxmin(m->D, x0, x1 - x0, m->d_vin.p, v_out, pol, wst, s, mir);
}

void ensure_t0x(gm_model* m, gm_matrix* tm) {
    if (!m->M.spec.reach() || tm->has_t0x) return;
    const int64_t n = tm->row_end - tm->row_begin;
    tm->t0x.ensure(static_cast<size_t>(std::max<int64_t>(n, 1)), "target-hit vector");
    const int64_t chunk = chunk_rows(m);
    ensure_scratch(m, std::min(chunk, std::max<int64_t>(n, 1)));
    const gmj::Kernels* J = jit_kernels(m, gmj::WANT_PROLOGUE, n);
    for (int64_t c0 = 0; c0 < n; c0 += chunk) {
        const int64_t cn = std::min(chunk, n - c0);
        Launch L(gmk::KF_PROLOGUE, m->stream);
        if (m->M.noise.family == GM_CUSTOM) {
            gmk::build_custom(m->D, tm->row_begin + c0, cn, m->d_origin[0].p, tm->t0x.p + c0, nullptr, m->d_err.p,
                              m->stream);
            continue;
        }
        gmk::prologue(m->D, tm->row_begin + c0, cn, gmk::PF_SKIP_ABSORBED | gmk::PF_T0X, m->d_origin[0].p,
                      tm->t0x.p + c0, m->d_rowflag[0].p, nullptr, m->d_err.p, m->stream, J ? J->prologue : nullptr);
    }
    ck(cudaStreamSynchronize(m->stream), "target hit");
    raise_device_error(m);
    tm->has_t0x = true;
}

// run_backward (synthesis.cpp:165-195) over all states on one device. The host
// tables are sized by a helper thread while the device builds and sweeps, and
// each column goes to the host (aux stream) as soon as its step is done, under
// the next step's kernels: the result is ready shortly after the last step.
// CUDA events bracketing stage (i) / stage (ii) of one synthesis on the model's stream.
struct PhaseTimer {
    gm_model* m;
    cudaEvent_t e[3] = {};
    explicit PhaseTimer(gm_model* mm) : m(mm) {
        for (cudaEvent_t& x : e) ck(cudaEventCreate(&x), "phase events");
    }
    ~PhaseTimer() {
        for (cudaEvent_t x : e) cudaEventDestroy(x);
    }
    void mark(int i) { ck(cudaEventRecord(e[i], m->stream), "phase event"); }
    void finish() {
        float a = 0.f, b = 0.f;
        ck(cudaEventSynchronize(e[2]), "phase event");
        ck(cudaEventElapsedTime(&a, e[0], e[1]), "phase time");
        ck(cudaEventElapsedTime(&b, e[1], e[2]), "phase time");
        m->last_build_ms = a;
        m->last_sweep_ms = b;
    }
};

gm_result* run_backward(gm_model* m, gm_matrix* tm, PhaseTimer* pt = nullptr) {
    const int64_t n_x = m->M.n_x();
    // OFA prologue results cached across the T steps; released when the sweep ends
    struct CacheScope {
        gm_model* m;
        explicit CacheScope(gm_model* mm) : m(mm) { m->ofa_cache_steps = true; }
        ~CacheScope() {
            m->ofa_cache_steps = false;
            m->ofa_valid = false;
            m->ofa_mass.release();
            m->ofa_origin.release();
            m->ofa_t0x.release();
            m->ofa_flag.release();
        }
    } cache_scope(m);
    const int T = m->M.spec.horizon;
    const bool reach = m->M.spec.reach();
    const size_t nx = static_cast<size_t>(n_x);
    DevBuf<double> vals;
    DevBuf<uint32_t> pol, wst;
    vals.ensure(nx * (T + 1), "value table");
    pol.ensure(nx * T, "policy table");
    wst.ensure(nx * T, "worst-disturbance table");
    std::unique_ptr<gm_result> r(new gm_result);
    r->meta = m->M;
    r->mode = tm ? GM_MODE_MATRIX : GM_MODE_OFA;
    r->n_x = n_x;
    r->T = T;
    std::exception_ptr sizer_err; // e.g. std::bad_alloc: rethrown on this thread after the join
    std::thread sizer([&] {
        try {
            r->values.resize(nx * (T + 1));
            r->policy.resize(nx * T);
            r->worst.resize(nx * T);
            std::fill(r->values.begin() + static_cast<std::ptrdiff_t>(nx) * T, r->values.end(), reach ? 0.0 : 1.0);
        } catch (...) {
            sizer_err = std::current_exception();
        }
    });
    struct Joiner {
        std::thread& t;
        ~Joiner() {
            if (t.joinable()) t.join();
        }
    } joiner{sizer};
    {
        std::vector<double> term(nx, reach ? 0.0 : 1.0);
        ck(cudaMemcpy(vals.p + nx * T, term.data(), term.size() * 8, cudaMemcpyHostToDevice), "terminal column");
    }
    ensure_scratch(m, 4096); // the aux stream
    cudaEvent_t done[2];
    for (cudaEvent_t& e : done) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "step events");
    struct EvFree {
        cudaEvent_t* e;
        ~EvFree() {
            cudaEventDestroy(e[0]);
            cudaEventDestroy(e[1]);
        }
    } evfree{done};
    auto join_sizer = [&] {
        if (sizer.joinable()) sizer.join();
        if (sizer_err) std::rethrow_exception(sizer_err);
    };
    auto copy_column = [&](int k, cudaEvent_t ready) {
        join_sizer();
        ck(cudaStreamWaitEvent(m->aux, ready, 0), "column wait");
        ck(cudaMemcpyAsync(r->values.data() + nx * k, vals.p + nx * k, nx * 8, cudaMemcpyDeviceToHost, m->aux),
           "values");
        ck(cudaMemcpyAsync(r->policy.data() + nx * k, pol.p + nx * k, nx * 4, cudaMemcpyDeviceToHost, m->aux),
           "policy");
        ck(cudaMemcpyAsync(r->worst.data() + nx * k, wst.p + nx * k, nx * 4, cudaMemcpyDeviceToHost, m->aux), "worst");
        ck(cudaStreamSynchronize(m->aux), "column copy");
    };
    // small tables (<= 64 MB) stay on the device until the sweep ends: the T steps are
    // enqueued back to back with no host synchronisation between them (launch-bound
    // configurations); larger ones stream each column out under the next step
    const bool defer = (nx * (T + 1) * 8 + 2 * nx * T * 4) <= (size_t(64) << 20);
    if (pt) pt->mark(1);
    for (int k = T - 1; k >= 0; --k) {
        step_states(m, tm, 0, n_x, vals.p + nx * (k + 1), vals.p + nx * k, pol.p + nx * k, wst.p + nx * k, m->stream);
        ck(cudaEventRecord(done[k & 1], m->stream), "step event");
        if (k == T - 1) {
            ck(cudaStreamSynchronize(m->stream), "bellman step");
            raise_device_error(m);
        } else if (!defer) {
            copy_column(k + 1, done[(k + 1) & 1]); // step k runs meanwhile
        }
    }
    if (pt) pt->mark(2);
    ck(cudaStreamSynchronize(m->stream), "bellman sweep");
    raise_device_error(m);
    if (pt) pt->finish();
    if (defer && T > 0) {
        join_sizer();
        ck(cudaMemcpy(r->values.data(), vals.p, nx * T * 8, cudaMemcpyDeviceToHost), "values");
        ck(cudaMemcpy(r->policy.data(), pol.p, nx * T * 4, cudaMemcpyDeviceToHost), "policy");
        ck(cudaMemcpy(r->worst.data(), wst.p, nx * T * 4, cudaMemcpyDeviceToHost), "worst");
    } else if (T > 0) {
        copy_column(0, done[0]);
    }
    join_sizer();
    if (reach) {
        r->absorbing.resize(nx);
        ck(cudaMemcpy(r->absorbing.data(), m->d_absorb.p, nx, cudaMemcpyDeviceToHost), "absorbing");
    }
    return r.release();
}

// ---------------------------------------------------------------- containers

void put_u64(std::ostream& os, uint64_t v) {
    char b[8];
    for (int i = 0; i < 8; ++i) b[i] = static_cast<char>((v >> (8 * i)) & 0xff);
    os.write(b, 8);
}
void put_u32(std::ostream& os, uint32_t v) {
    char b[4];
    for (int i = 0; i < 4; ++i) b[i] = static_cast<char>((v >> (8 * i)) & 0xff);
    os.write(b, 4);
}
void put_f64(std::ostream& os, double v) {
    uint64_t u;
    std::memcpy(&u, &v, 8);
    put_u64(os, u);
}

void grid_lines(std::ostream& os, const char* prefix, const Grid& g) {
    os << prefix << ".dim = " << g.dim() << ";\n";
    if (g.dim() == 0) return;
    os << prefix << ".lb = " << fmt_vec(g.lb) << ";\n";
    os << prefix << ".ub = " << fmt_vec(g.ub) << ";\n";
    os << prefix << ".eta = " << fmt_vec(g.eta) << ";\n";
}

const char* kind_name(int k) {
    return k == GM_SPEC_SAFETY ? "safety" : k == GM_SPEC_REACH ? "reachability" : "reach-avoid";
}

} // namespace

// ===========================================================================
// C ABI
// ===========================================================================

extern "C" {

static void apply_overrides(Cfg& c, const gm_overrides* ov) {
    if (!ov) return;
    if (ov->threads >= 0) c.threads = ov->threads;
    if (ov->mode && *ov->mode) c.mode = ov->mode;
    if (ov->mem_budget >= 0) c.mem_budget = static_cast<uint64_t>(ov->mem_budget);
    if (ov->seed >= 0) c.seed = static_cast<uint64_t>(ov->seed);
    if (ov->runs >= 0) c.runs = ov->runs;
    if (ov->time_steps >= 0) c.time_steps = ov->time_steps;
    if (ov->output && *ov->output) c.output = ov->output;
}

static gm_code make_model(const Cfg& c0, const gm_overrides* ov, gm_model** out, gm_status* st) {
    return guarded(st, [&] {
        Cfg c = c0;
        apply_overrides(c, ov);
        auto* m = new gm_model;
        try {
            m->M = build_model_from_cfg(c);
        } catch (...) {
            delete m;
            throw;
        }
        *out = m;
    });
}

gm_code gm_model_create(const gm_model_desc* d, gm_model** out, gm_status* st) {
    return guarded(st, [&] {
        auto grid = [](const gm_grid_desc& g) {
            if (g.dim < 0 || g.dim > GM_MAX_DIMS) throw ConfigErr("model_create: grid dimension out of range");
            if (g.dim == 0) return grid_from({}, {}, {});
            return grid_from(std::vector<double>(g.lb, g.lb + g.dim), std::vector<double>(g.ub, g.ub + g.dim),
                             std::vector<double>(g.eta, g.eta + g.dim));
        };
        const Grid X = grid(d->state), U = grid(d->input), W = grid(d->disturbance);
        const int n = X.dim(), mm = U.dim(), p = W.dim();
        auto expr = [&](const gm_expr_desc& e, int nn, int m2, int p2, const std::string& what) {
            if (e.n_nodes <= 0 || !e.nodes) throw ConfigErr(what + ": empty expression");
            std::vector<XNode> nodes(static_cast<size_t>(e.n_nodes));
            for (int32_t i = 0; i < e.n_nodes; ++i) {
                const gm_expr_node& s = e.nodes[i];
                XNode& x = nodes[static_cast<size_t>(i)];
                if (s.op < 0 || s.op > static_cast<int>(XOp::variable))
                    throw ConfigErr(what + ": node " + std::to_string(i) + " has an unknown operator");
                x.op = static_cast<XOp>(s.op);
                x.value = s.value;
                x.vclass = static_cast<uint8_t>(s.var_class);
                x.vindex = s.var_index;
                for (int k = 0; k < 3; ++k) x.kid[k] = s.kid[k];
            }
            return expr_from_nodes(std::move(nodes), e.root, nn, m2, p2, what);
        };
        std::vector<Expr> dyn;
        for (int32_t i = 0; i < d->n_dynamics; ++i)
            dyn.push_back(expr(d->dynamics[i], n, mm, p, "dynamics.x" + std::to_string(i)));
        const int nd = d->noise_dim;
        if (nd < 0 || nd > GM_MAX_DIMS) throw ConfigErr("model_create: noise dimension out of range");
        std::vector<double> p1(d->param1, d->param1 + (d->param1 ? nd : 0));
        std::vector<double> p2(d->param2, d->param2 + (d->param2 ? nd : 0));
        Expr pdf;
        if (d->noise_family == GM_NOISE_CUSTOM) pdf = expr(d->custom_pdf, n, 0, 0, "noise.pdf");
        SpecV spec;
        if (d->spec_kind < GM_SAFETY || d->spec_kind > GM_REACH_AVOID) throw ConfigErr("model_create: unknown spec kind");
        spec.kind = d->spec_kind;
        spec.horizon = d->horizon;
        if (d->target_lo && d->target_hi)
            spec.target = BoxV{std::vector<double>(d->target_lo, d->target_lo + n),
                               std::vector<double>(d->target_hi, d->target_hi + n)};
        if (d->avoid_lo && d->avoid_hi)
            spec.avoid = BoxV{std::vector<double>(d->avoid_lo, d->avoid_lo + n),
                              std::vector<double>(d->avoid_hi, d->avoid_hi + n)};
        auto* m = new gm_model;
        try {
            m->M = build_model_from_parts(X, U, W, std::move(dyn), d->noise_family, d->noise_mode ? 1 : 0, d->gamma, p1,
                                          p2, std::move(pdf), spec, d->mode == GM_MODE_OFA ? GM_MODE_OFA_ : GM_MODE_MATRIX_,
                                          d->threads, d->mem_budget);
        } catch (...) {
            delete m;
            throw;
        }
        *out = m;
    });
}

gm_code gm_model_save_config(const gm_model* m, const char* path, gm_status* st) {
    return guarded(st, [&] {
        std::ofstream os(path);
        if (!os) throw IoErr(std::string("cannot open '") + path + "' for writing");
        os << save_config_text(m->M.cfg);
        if (!os) throw IoErr(std::string("failed while writing '") + path + "'");
    });
}

gm_code gm_model_load(const char* path, const gm_overrides* ov, gm_model** out, gm_status* st) {
    Cfg c;
    const gm_code rc = guarded(st, [&] { c = load_cfg_file(path ? path : ""); });
    if (rc != GM_OK) return rc;
    return make_model(c, ov, out, st);
}

gm_code gm_model_parse(const char* text, const char* name, const gm_overrides* ov, gm_model** out,
                       gm_status* st) {
    Cfg c;
    const gm_code rc = guarded(st, [&] { c = parse_cfg_text(text ? text : "", name ? name : "<config>"); });
    if (rc != GM_OK) return rc;
    return make_model(c, ov, out, st);
}

void gm_model_free(gm_model* m) {
    if (!m) return;
    if (m->dev_ready) {
        cudaSetDevice(m->device);
        cudaStreamSynchronize(m->stream);
        if (m->aux) {
            cudaStreamSynchronize(m->aux);
            cudaStreamDestroy(m->aux);
            for (cudaEvent_t e : {m->ev_fork, m->ev_join, m->ev_ready[0], m->ev_ready[1], m->ev_used[0], m->ev_used[1]})
                cudaEventDestroy(e);
        }
        cudaStreamDestroy(m->own_stream ? m->own_stream : m->stream);
    }
    delete m;
}

gm_code gm_model_set_spec(gm_model* m, int32_t kind, int32_t horizon, const double* tlo, const double* thi,
                          const double* alo, const double* ahi, gm_status* st) {
    return guarded(st, [&] {
        const int n = m->M.X.dim();
        SpecV s;
        s.kind = kind;
        s.horizon = horizon;
        if (tlo && thi) s.target = BoxV{std::vector<double>(tlo, tlo + n), std::vector<double>(thi, thi + n)};
        if (alo && ahi) s.avoid = BoxV{std::vector<double>(alo, alo + n), std::vector<double>(ahi, ahi + n)};
        m->M.spec = s;
        m->absorb_ready = false;
    });
}

gm_code gm_model_set_options(gm_model* m, int32_t mode, int64_t mem_budget, gm_status* st) {
    return guarded(st, [&] {
        if (mode >= 0) m->M.mode = mode;
        if (mem_budget >= 0) m->M.mem_budget = static_cast<uint64_t>(mem_budget);
    });
}

gm_code gm_model_sizes(const gm_model* m, gm_sizes* o, gm_status* st) {
    return guarded(st, [&] {
        std::memset(o, 0, sizeof *o);
        const Model& M = m->M;
        o->n_dim = M.X.dim();
        o->m_dim = M.U.dim();
        o->p_dim = M.W.dim();
        o->n_states = M.n_x();
        o->n_inputs = M.n_u();
        o->n_disturbances = M.n_w();
        o->pairs = M.n_x() * M.n_u();
        o->spec_kind = M.spec.kind;
        o->horizon = M.spec.horizon;
        o->mode = M.mode;
        o->threads = M.threads;
        o->gamma = M.noise.gamma;
        o->mem_budget = static_cast<int64_t>(M.mem_budget);
        for (int d = 0; d < M.X.dim() && d < GM_MAX_DIMS; ++d) {
            o->counts[d] = M.X.count[d];
            o->strides[d] = M.X.stride[d];
            o->extents[d] = M.extents[d];
        }
        o->row_width = M.R;
        o->rows_per_thread_group = tpr_for_width(M.R);
        try { // memory_estimate raises MemoryError only when asked for (abstraction.cpp:37-48)
            o->rows = M.rows();
            o->memory_estimate = M.memory_estimate();
        } catch (const MemoryErr&) {
            o->rows = 0;
            o->memory_estimate = 0;
            o->size_overflow = 1;
        }
    });
}

gm_code gm_absorbing_states(gm_model* m, uint8_t* flags, gm_status* st) {
    return guarded(st, [&] {
        prepare(m);
        const size_t n = static_cast<size_t>(m->M.n_x());
        if (!m->M.spec.reach()) {
            std::memset(flags, 0, n);
            return;
        }
        ck(cudaMemcpy(flags, m->d_absorb.p, n, cudaMemcpyDeviceToHost), "absorbing flags");
    });
}

gm_code gm_dynamics_image(const gm_model* m, int64_t row, double* mu_out, gm_status* st) {
    return guarded(st, [&] {
        if (row < 0 || row >= m->M.rows()) throw std::out_of_range("dynamics_image: row out of range");
        std::vector<double> mu;
        m->M.row_image(row, mu);
        std::memcpy(mu_out, mu.data(), mu.size() * 8);
    });
}

const char* gm_model_output_path(const gm_model* m) { return m->M.cfg.output.c_str(); }

int64_t gm_model_program_size(const gm_model* m) { return static_cast<int64_t>(m->M.prog.code.size()); }

gm_code gm_model_jit_compile(const gm_model* m, int32_t kind, double* seconds, gm_status* st) {
    return guarded(st, [&] {
        // kind 2 with the model's row-shape specialisation, as the launcher compiles it
        const char* js = std::getenv("GM_JIT_SHAPE");
        const std::string shape = kind == 3 ? gmj::ofa_shape_defines(m->M.device_descriptor())
                                  : kind == 2 && !(js && js[0] == '0') ? gmj::shape_defines(m->M.device_descriptor())
                                                                       : std::string();
        if (kind == 3 && shape.empty()) throw ConfigErr("the model's row shape does not qualify for the OFA kernel");
        const std::string err = gmj::compile_only(m->M.prog, m->M.X.dim(), m->M.U.dim(), m->M.W.dim(), kind, seconds,
                                                  shape, gmk::build_ctas(m->M.device_descriptor(), true));
        if (!err.empty()) throw std::runtime_error(err);
    });
}

int32_t gm_model_jit_status(const gm_model* m, double* compile_s, char* why, int64_t why_len) {
    if (compile_s) *compile_s = m->jit_compile_s;
    if (why && why_len > 0) {
        std::strncpy(why, m->jit_why.c_str(), static_cast<size_t>(why_len - 1));
        why[why_len - 1] = '\0';
    }
    return m->jit_used ? 1 : 0;
}

gm_code gm_set_device(int32_t device, gm_status* st) {
    return guarded(st, [&] { ck(cudaSetDevice(device), "cudaSetDevice"); });
}

gm_code gm_model_set_stream(gm_model* m, void* stream, int32_t use_own, gm_status* st) {
    return guarded(st, [&] {
        ensure_device(m);
        if (!m->own_stream) m->own_stream = m->stream;
        m->stream = use_own ? m->own_stream : static_cast<cudaStream_t>(stream);
    });
}

int64_t gm_launch_count(void) { return g_launches.load(); }

double gm_last_kernel_ms(int32_t family) {
    collect_timing();
    if (family < 0 || family >= gmk::KF_COUNT) return 0.0;
    return g_last_ms[family];
}

void gm_enable_kernel_timing(int32_t on) {
    collect_timing();
    g_timing = on != 0;
}

double gm_kernel_ms_total(int32_t family) {
    collect_timing();
    if (family < 0 || family >= gmk::KF_COUNT) return 0.0;
    return g_total_ms[family];
}

const char* gm_last_kernel_variant(int32_t family) { return gmk::last_variant(family); }

int64_t gm_kernel_launches(int32_t family) {
    if (family < 0 || family >= gmk::KF_COUNT) return 0;
    std::lock_guard<std::mutex> lk(g_tmu);
    return g_fam_launches[family];
}

void gm_reset_kernel_stats(void) {
    collect_timing();
    std::lock_guard<std::mutex> lk(g_tmu);
    for (int i = 0; i < gmk::KF_COUNT; ++i) {
        g_total_ms[i] = 0;
        g_last_ms[i] = 0;
        g_fam_launches[i] = 0;
    }
}

// ---------------------------------------------------------------- stage (i)

gm_code gm_build_matrix(gm_model* m, int64_t r0, int64_t r1, gm_matrix** out, gm_status* st) {
    return guarded(st, [&] {
        const int64_t rows = m->M.rows();
        if (r0 < 0 || r1 > rows || r0 > r1) throw std::out_of_range("build_matrix: row range outside the model");
        prepare(m);
        auto tm = std::make_unique<gm_matrix>();
        build_rows(m, r0, r1, tm.get(), false);
        *out = tm.release();
    });
}

gm_code gm_build_shard(gm_model* m, int64_t x0, int64_t x1, gm_matrix** out, gm_status* st) {
    return guarded(st, [&] {
        if (x0 < 0 || x1 > m->M.n_x() || x0 > x1) throw std::out_of_range("build_shard: state range outside the grid");
        check_spec(m->M.spec, m->M.X);
        prepare(m);
        const int64_t nuw = m->M.n_u() * m->M.n_w();
        if (*out) { // rebuild in place
            (*out)->has_t0x = false;
            (*out)->masked = false;
            build_rows(m, x0 * nuw, x1 * nuw, *out, m->M.spec.reach());
            return;
        }
        auto tm = std::make_unique<gm_matrix>();
        build_rows(m, x0 * nuw, x1 * nuw, tm.get(), m->M.spec.reach());
        *out = tm.release();
    });
}

gm_code gm_build_shard_host(gm_model* m, int64_t x0, int64_t x1, gm_matrix** out, int64_t* origins_host,
                            double* t0x_host, gm_status* st) {
    return guarded(st, [&] {
        if (x0 < 0 || x1 > m->M.n_x() || x0 > x1) throw std::out_of_range("build_shard: state range outside the grid");
        check_spec(m->M.spec, m->M.X);
        prepare(m);
        const int64_t nuw = m->M.n_u() * m->M.n_w();
        const int64_t r0 = x0 * nuw, n = (x1 - x0) * nuw;
        const bool reach = m->M.spec.reach();
        std::unique_ptr<gm_matrix> fresh;
        gm_matrix* tm = *out;
        if (!tm) {
            fresh = std::make_unique<gm_matrix>();
            tm = fresh.get();
        }
        tm->device = m->device;
        tm->row_begin = r0;
        tm->row_end = r0 + n;
        tm->R = m->M.R;
        tm->pitch = m->D.pitch;
        tm->masked = false;
        tm->has_t0x = false;
        tm->probs.ensure(mul_checked(static_cast<uint64_t>(n), static_cast<uint64_t>(tm->pitch), "matrix size"),
                         "matrix payload");
        tm->origins.ensure(static_cast<size_t>(n), "matrix origins");
        if (reach) {
            tm->t0x.ensure(static_cast<size_t>(n), "target-hit vector");
            tm->has_t0x = true;
        }
        ensure_scratch(m, 4096); // the aux stream and events of the producer pipeline
        const gmj::Kernels* J =
            jit_kernels(m, gmk::build_uses_qs(m->D) ? gmj::WANT_BUILD_QS : gmj::WANT_BUILD_NOQS, n);
        // GM_BUILD_HOST_DIRECT=1 with pinned (device-accessible) host buffers: the build
        // kernel writes each row's origin / T0x to the host itself, next to the device
        // copy, in one launch. Measured slower (C2b: 49 ms vs 21 ms end to end; the
        // scattered 8-byte host writes throttle the kernel), so the sliced copies are the
        // default
        auto mapped = [](void* p) -> void* {
            if (!p) return nullptr;
            cudaPointerAttributes a{};
            if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
                cudaGetLastError();
                return nullptr;
            }
            return a.type == cudaMemoryTypeHost ? a.devicePointer : nullptr;
        };
        void* oh = mapped(origins_host);
        void* th = reach ? mapped(t0x_host) : nullptr;
        static const char* direct_env = std::getenv("GM_BUILD_HOST_DIRECT");
        const bool direct = (direct_env && direct_env[0] == '1') && m->M.noise.family != GM_CUSTOM &&
                            (origins_host == nullptr || oh) && (!reach || t0x_host == nullptr || th) &&
                            (oh || th);
        if (direct) {
            GmDev Dv = m->D;
            Dv.origin_host = static_cast<long long*>(oh);
            Dv.t0x_host = static_cast<double*>(th);
            {
                Launch L(gmk::KF_BUILD, m->stream);
                gmk::build(Dv, r0, n, tm->origins.p, reach ? tm->t0x.p : nullptr, tm->probs.p, m->d_err.p, m->stream,
                           J ? J->build_ws : nullptr);
            }
            ck(cudaStreamSynchronize(m->stream), "build");
            raise_device_error(m);
            if (fresh) *out = fresh.release();
            return;
        }
        // pageable buffers: the rows in a few slices, slice k's origins / T0x travel to
        // the host on the aux stream while slice k+1 builds
        const int64_t slices = n >= (int64_t(1) << 16) ? 4 : 1;
        const int64_t per = (n + slices - 1) / slices;
        cudaEvent_t ev[4];
        for (int64_t k = 0; k < slices; ++k) ck(cudaEventCreateWithFlags(&ev[k], cudaEventDisableTiming), "event");
        for (int64_t k = 0; k < slices; ++k) {
            const int64_t c0 = k * per, cn = std::min(per, n - c0);
            if (cn <= 0) break;
            {
                Launch L(gmk::KF_BUILD, m->stream);
                gmk::build(m->D, r0 + c0, cn, tm->origins.p + c0, reach ? tm->t0x.p + c0 : nullptr,
                           tm->probs.p + c0 * tm->pitch, m->d_err.p, m->stream, J ? J->build_ws : nullptr);
            }
            ck(cudaEventRecord(ev[k], m->stream), "slice event");
            ck(cudaStreamWaitEvent(m->aux, ev[k], 0), "slice wait");
            if (origins_host)
                ck(cudaMemcpyAsync(origins_host + c0, tm->origins.p + c0, static_cast<size_t>(cn) * 8,
                                   cudaMemcpyDeviceToHost, m->aux),
                   "origins");
            if (t0x_host && reach)
                ck(cudaMemcpyAsync(t0x_host + c0, tm->t0x.p + c0, static_cast<size_t>(cn) * 8, cudaMemcpyDeviceToHost,
                                   m->aux),
                   "t0x");
        }
        ck(cudaStreamSynchronize(m->stream), "build");
        ck(cudaStreamSynchronize(m->aux), "copies");
        for (int64_t k = 0; k < slices; ++k) cudaEventDestroy(ev[k]);
        raise_device_error(m);
        if (fresh) *out = fresh.release();
    });
}

gm_code gm_shard_reach(gm_model* m, int64_t x0, int64_t x1, int64_t* lo, int64_t* hi, gm_status* st) {
    return guarded(st, [&] {
        if (x0 < 0 || x1 > m->M.n_x() || x0 > x1) throw std::out_of_range("shard_reach: state range outside the grid");
        prepare(m);
        *lo = *hi = x0;
        if (x1 == x0) return;
        if (m->M.noise.family == GM_CUSTOM) { // conservative: the whole grid
            *lo = 0;
            *hi = m->M.n_x();
            return;
        }
        const int64_t nuw = m->M.n_u() * m->M.n_w();
        const int64_t r0 = x0 * nuw, n = (x1 - x0) * nuw;
        const int64_t chunk = std::min(chunk_rows(m), n);
        ensure_scratch(m, chunk);
        m->d_reach.ensure(2, "reach bounds");
        const long long init[2] = {LLONG_MAX, -1};
        ck(cudaMemcpyAsync(m->d_reach.p, init, sizeof init, cudaMemcpyHostToDevice, m->stream), "reach init");
        const gmj::Kernels* J = jit_kernels(m, gmj::WANT_PROLOGUE, n);
        // rows of absorbed states are skipped by the step for reach specs (synthesis.cpp:86-89)
        const int flags = m->M.spec.reach() ? gmk::PF_SKIP_ABSORBED : 0;
        for (int64_t c0 = 0; c0 < n; c0 += chunk) {
            const int64_t cn = std::min(chunk, n - c0);
            Launch L(gmk::KF_MISC, m->stream);
            gmk::prologue(m->D, r0 + c0, cn, flags, m->d_origin[0].p, nullptr, m->d_rowflag[0].p, nullptr, m->d_err.p,
                          m->stream, J ? J->prologue : nullptr);
            gmk::origin_minmax(m->d_origin[0].p, m->d_rowflag[0].p, cn, m->d_reach.p, m->stream);
        }
        long long mm[2];
        ck(cudaMemcpyAsync(mm, m->d_reach.p, sizeof mm, cudaMemcpyDeviceToHost, m->stream), "reach bounds");
        ck(cudaStreamSynchronize(m->stream), "shard reach");
        raise_device_error(m);
        if (mm[1] < 0) return; // every row absorbed: the step reads nothing
        int64_t span = 0; // the slab's last post-state relative to its origin
        for (int d = 0; d < m->D.n; ++d) span += (m->D.W[d] - 1) * m->D.xstride[d];
        *lo = mm[0];
        *hi = std::min<int64_t>(m->M.n_x(), mm[1] + span + 1);
    });
}

gm_code gm_mask_absorbing(gm_model* m, gm_matrix* tm, gm_status* st) {
    return guarded(st, [&] {
        if (!m->M.spec.reach()) return; // abstraction.cpp:323
        prepare(m);
        const Model& M = m->M;
        const int n = M.X.dim();
        std::vector<long long> off(static_cast<size_t>(n) + 1, 0);
        for (int d = 0; d < n; ++d) off[d + 1] = off[d] + M.X.count[d];
        auto member = [&](const BoxV& b) {
            std::vector<uint8_t> f(static_cast<size_t>(off[n]), 0);
            if (b.dim() != n) return f;
            for (int d = 0; d < n; ++d)
                for (int64_t j = 0; j < M.X.count[d]; ++j) {
                    const double rep = M.X.rep(d, j);
                    f[static_cast<size_t>(off[d] + j)] = (rep >= b.lo[d] && rep <= b.hi[d]) ? 1 : 0;
                }
            return f;
        };
        const auto inT = member(M.spec.target);
        const bool haveA = M.spec.avoid.dim() > 0;
        const auto inA = haveA ? member(M.spec.avoid) : std::vector<uint8_t>{};
        DevBuf<uint8_t> dT, dA;
        DevBuf<long long> dOff;
        dT.ensure(inT.size(), "mask flags");
        ck(cudaMemcpy(dT.p, inT.data(), inT.size(), cudaMemcpyHostToDevice), "mask flags");
        if (haveA) {
            dA.ensure(inA.size(), "mask flags");
            ck(cudaMemcpy(dA.p, inA.data(), inA.size(), cudaMemcpyHostToDevice), "mask flags");
        }
        dOff.ensure(off.size(), "mask offsets");
        ck(cudaMemcpy(dOff.p, off.data(), off.size() * sizeof(long long), cudaMemcpyHostToDevice), "mask offsets");
        {
            Launch L(gmk::KF_MASK, m->stream);
            gmk::mask(m->D, 0, tm->row_end - tm->row_begin, tm->probs.p, tm->origins.p, dT.p,
                      haveA ? dA.p : nullptr, dOff.p, m->stream);
        }
        ck(cudaStreamSynchronize(m->stream), "mask");
        tm->masked = true;
    });
}

gm_code gm_build_target_hit(gm_model* m, int64_t r0, int64_t r1, double* t0x_out, gm_status* st) {
    return guarded(st, [&] {
        check_spec(m->M.spec, m->M.X);
        if (!m->M.spec.reach())
            throw ConfigErr("build_target_hit requires a reachability or reach-avoid spec");
        if (r0 < 0 || r1 > m->M.rows() || r0 > r1) throw std::out_of_range("build_target_hit: row range");
        prepare(m);
        gm_matrix tmp;
        tmp.row_begin = r0;
        tmp.row_end = r1;
        ensure_t0x(m, &tmp);
        if (r1 > r0)
            ck(cudaMemcpy(t0x_out, tmp.t0x.p, static_cast<size_t>(r1 - r0) * 8, cudaMemcpyDeviceToHost), "t0x");
    });
}

gm_code gm_matrix_copy_rows(const gm_matrix* tm, int64_t r0, int64_t r1, int64_t* origins, double* probs,
                            gm_status* st) {
    return guarded(st, [&] {
        if (r0 < tm->row_begin || r1 > tm->row_end || r0 > r1) throw std::out_of_range("matrix rows out of range");
        ck(cudaSetDevice(tm->device), "cudaSetDevice");
        const int64_t a = r0 - tm->row_begin, n = r1 - r0;
        if (n == 0) return;
        if (origins)
            ck(cudaMemcpy(origins, tm->origins.p + a, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToHost), "origins");
        if (probs)
            ck(cudaMemcpy2D(probs, static_cast<size_t>(tm->R) * 8, tm->probs.p + a * tm->pitch,
                            static_cast<size_t>(tm->pitch) * 8, static_cast<size_t>(tm->R) * 8, static_cast<size_t>(n),
                            cudaMemcpyDeviceToHost),
               "probs");
    });
}

gm_code gm_matrix_copy_t0x(const gm_matrix* tm, int64_t r0, int64_t r1, double* t0x, gm_status* st) {
    return guarded(st, [&] {
        if (!tm->has_t0x) throw ConfigErr("matrix carries no target-hit vector");
        if (r0 < tm->row_begin || r1 > tm->row_end || r0 > r1) throw std::out_of_range("matrix rows out of range");
        ck(cudaSetDevice(tm->device), "cudaSetDevice");
        if (r1 > r0)
            ck(cudaMemcpy(t0x, tm->t0x.p + (r0 - tm->row_begin), static_cast<size_t>(r1 - r0) * 8,
                          cudaMemcpyDeviceToHost),
               "t0x");
    });
}

int64_t gm_matrix_pitch(const gm_matrix* tm) { return tm->pitch; }

gm_code gm_matrix_info(const gm_matrix* tm, int64_t* rb, int64_t* re, int64_t* R, const double** probs,
                       const int64_t** origins, gm_status* st) {
    return guarded(st, [&] {
        if (rb) *rb = tm->row_begin;
        if (re) *re = tm->row_end;
        if (R) *R = tm->R;
        if (probs) *probs = tm->probs.p;
        if (origins) *origins = reinterpret_cast<const int64_t*>(tm->origins.p);
    });
}

gm_code gm_matrix_write(const gm_matrix* tm, const gm_model* m, const char* path, gm_status* st) {
    return guarded(st, [&] {
        // write_matrix, io.cpp:236-256
        if (tm->row_begin != 0 || tm->row_end != m->M.rows())
            throw IoErr("write_matrix needs the whole matrix (rows 0..rows)");
        std::ofstream os(path, std::ios::binary);
        if (!os) throw IoErr(std::string("cannot open '") + path + "' for writing");
        const Model& M = m->M;
        os << "gridmdp-matrix" << ' ' << 1 << '\n';
        grid_lines(os, "states", M.X);
        os << "n_inputs = " << M.n_u() << ";\n";
        os << "n_disturbances = " << M.n_w() << ";\n";
        std::string w = "{";
        for (size_t d = 0; d < M.extents.size(); ++d) {
            if (d) w += ", ";
            w += std::to_string(M.extents[d]);
        }
        os << "window = " << w << "};\n";
        const int64_t rows = tm->row_end - tm->row_begin;
        os << "array.origins = i64 " << rows << " 1;\n";
        os << "array.probs = f64 " << rows << " " << tm->R << ";\n";
        os << "payload\n";
        ck(cudaSetDevice(tm->device), "cudaSetDevice");
        std::vector<long long> org(static_cast<size_t>(rows));
        if (rows) ck(cudaMemcpy(org.data(), tm->origins.p, org.size() * 8, cudaMemcpyDeviceToHost), "origins");
        for (long long o : org) put_u64(os, static_cast<uint64_t>(o));
        const int64_t blk = std::max<int64_t>(1, (64LL << 20) / 8 / std::max<int64_t>(tm->R, 1));
        std::vector<double> buf;
        for (int64_t r = 0; r < rows; r += blk) {
            const int64_t n = std::min(blk, rows - r);
            buf.resize(static_cast<size_t>(n * tm->R));
            ck(cudaMemcpy2D(buf.data(), static_cast<size_t>(tm->R) * 8, tm->probs.p + r * tm->pitch,
                            static_cast<size_t>(tm->pitch) * 8, static_cast<size_t>(tm->R) * 8, static_cast<size_t>(n),
                            cudaMemcpyDeviceToHost),
               "probs");
            for (double v : buf) put_f64(os, v);
        }
        if (!os) throw IoErr(std::string("failed while writing '") + path + "'");
    });
}

gm_code gm_matrix_write_prism(const gm_matrix* tm, const gm_model* m, const char* path, gm_status* st) {
    return guarded(st, [&] {
        // export_prism, io.cpp:289-317
        if (tm->row_begin != 0 || tm->row_end != m->M.rows())
            throw IoErr("export_prism needs the whole matrix (rows 0..rows)");
        std::ofstream os(path);
        if (!os) throw IoErr(std::string("cannot open '") + path + "' for writing");
        ck(cudaSetDevice(tm->device), "cudaSetDevice");
        const Model& M = m->M;
        const int64_t rows = tm->row_end - tm->row_begin, R = tm->R;
        DevBuf<unsigned long long> cnt;
        cnt.ensure(1, "count");
        // padding is zero, so the count over rows x pitch is the count over the rows
        const unsigned long long transitions = gmk::count_positive(tm->probs.p, rows * tm->pitch, cnt.p, nullptr);
        const int64_t choices = M.n_u() * M.n_w();
        os << M.n_x() << ' ' << rows << ' ' << transitions << '\n';
        const Grid& g = M.X;
        const int n = g.dim();
        std::vector<long long> org;
        std::vector<double> buf;
        const int64_t blk = std::max<int64_t>(1, (64LL << 20) / 8 / std::max<int64_t>(R, 1));
        std::string line;
        char num[64];
        for (int64_t r0 = 0; r0 < rows; r0 += blk) {
            const int64_t nb = std::min(blk, rows - r0);
            org.resize(static_cast<size_t>(nb));
            buf.resize(static_cast<size_t>(nb * R));
            ck(cudaMemcpy(org.data(), tm->origins.p + r0, org.size() * 8, cudaMemcpyDeviceToHost), "origins");
            ck(cudaMemcpy2D(buf.data(), static_cast<size_t>(R) * 8, tm->probs.p + r0 * tm->pitch,
                            static_cast<size_t>(tm->pitch) * 8, static_cast<size_t>(R) * 8, static_cast<size_t>(nb),
                            cudaMemcpyDeviceToHost),
               "probs");
            for (int64_t i = 0; i < nb; ++i) {
                const int64_t r = r0 + i, src = r / choices, choice = r % choices;
                // visit_slab (abstraction.hpp:130-149): row-major over the extents
                int64_t o[GMD_MAXD], j[GMD_MAXD] = {0}, rem = org[static_cast<size_t>(i)], flat = 0;
                for (int d = 0; d < n; ++d) {
                    o[d] = rem / g.stride[d];
                    rem %= g.stride[d];
                    flat += o[d] * g.stride[d];
                }
                const double* row = buf.data() + i * R;
                for (int64_t k = 0;; ) {
                    if (row[k] > 0.0) {
                        line = std::to_string(src);
                        line += ' ';
                        line += std::to_string(choice);
                        line += ' ';
                        line += std::to_string(flat);
                        line += ' ';
                        auto res = std::to_chars(num, num + sizeof num, row[k]);
                        line.append(num, res.ptr);
                        line += '\n';
                        os << line;
                    }
                    ++k;
                    int d = n - 1;
                    for (; d >= 0; --d) {
                        flat += g.stride[d];
                        if (++j[d] < M.extents[d]) break;
                        flat -= M.extents[d] * g.stride[d];
                        j[d] = 0;
                    }
                    if (d < 0) break;
                }
            }
        }
        if (!os) throw IoErr(std::string("failed while writing '") + path + "'");
    });
}

void gm_matrix_free(gm_matrix* tm) {
    if (!tm) return;
    if (tm->device >= 0) cudaSetDevice(tm->device);
    delete tm;
}

gm_code gm_matrix_read(const char* path, gm_matrix** out, gm_status* st) {
    return guarded(st, [&] {
        // read_matrix, io.cpp:258-283
        std::ifstream is(path, std::ios::binary);
        if (!is) throw IoErr(std::string("cannot open '") + path + "'");
        ManifestR mf(is, "gridmdp-matrix");
        auto tm = std::make_unique<gm_matrix>();
        tm->has_meta = true;
        tm->X = mf.grid("states");
        tm->n_u = mf.integer("n_inputs");
        tm->n_w = mf.integer("n_disturbances");
        int64_t R = 1;
        for (double w : mf.vec("window")) {
            tm->extents.push_back(static_cast<int64_t>(w));
            R *= tm->extents.back();
        }
        const int64_t rows = tm->X.total * tm->n_u * tm->n_w;
        int count = 0;
        if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
            cudaGetLastError();
            throw CudaErr("no CUDA device available: the B200 engine has no CPU fallback");
        }
        ck(cudaGetDevice(&tm->device), "cudaGetDevice");
        tm->row_begin = 0;
        tm->row_end = rows;
        tm->R = R;
        tm->pitch = row_pitch(R);
        tm->probs.ensure(mul_checked(static_cast<uint64_t>(rows), static_cast<uint64_t>(tm->pitch), "matrix size"),
                         "matrix payload");
        tm->origins.ensure(static_cast<size_t>(std::max<int64_t>(rows, 1)), "matrix origins");
        if (tm->pitch != R) ck(cudaMemset(tm->probs.p, 0, static_cast<size_t>(rows * tm->pitch) * 8), "padding");
        // little-endian payloads (io.cpp:30-70) on a little-endian host: bulk reads
        std::vector<long long> org(static_cast<size_t>(rows));
        is.read(reinterpret_cast<char*>(org.data()), static_cast<std::streamsize>(org.size() * 8));
        if (!is) throw IoErr("truncated payload");
        if (rows) ck(cudaMemcpy(tm->origins.p, org.data(), org.size() * 8, cudaMemcpyHostToDevice), "origins");
        const int64_t blk = std::max<int64_t>(1, (64LL << 20) / 8 / std::max<int64_t>(R, 1));
        std::vector<double> buf;
        for (int64_t r = 0; r < rows; r += blk) {
            const int64_t n = std::min(blk, rows - r);
            buf.resize(static_cast<size_t>(n * R));
            is.read(reinterpret_cast<char*>(buf.data()), static_cast<std::streamsize>(buf.size() * 8));
            if (!is) throw IoErr("truncated payload");
            ck(cudaMemcpy2D(tm->probs.p + r * tm->pitch, static_cast<size_t>(tm->pitch) * 8, buf.data(),
                            static_cast<size_t>(R) * 8, static_cast<size_t>(R) * 8, static_cast<size_t>(n),
                            cudaMemcpyHostToDevice),
               "probs");
        }
        char extra;
        if (is.get(extra)) throw IoErr("trailing bytes after the declared payload");
        *out = tm.release();
    });
}

gm_code gm_matrix_upload(const gm_model* mc, int64_t row_begin, int64_t rows, const int64_t* origins,
                         const double* probs, gm_matrix** out, gm_status* st) {
    return guarded(st, [&] {
        gm_model* m = const_cast<gm_model*>(mc); // device residency only
        if (row_begin < 0 || rows < 0 || row_begin + rows > m->M.rows())
            throw std::out_of_range("matrix_upload: row range outside the model");
        prepare(m);
        auto tm = std::make_unique<gm_matrix>();
        tm->device = m->device;
        tm->row_begin = row_begin;
        tm->row_end = row_begin + rows;
        tm->R = m->M.R;
        tm->pitch = m->D.pitch;
        const int64_t R = tm->R;
        tm->probs.ensure(mul_checked(static_cast<uint64_t>(rows), static_cast<uint64_t>(tm->pitch), "matrix size"),
                         "matrix payload");
        tm->origins.ensure(static_cast<size_t>(std::max<int64_t>(rows, 1)), "matrix origins");
        if (tm->pitch != R) ck(cudaMemset(tm->probs.p, 0, static_cast<size_t>(rows * tm->pitch) * 8), "padding");
        if (rows) {
            ck(cudaMemcpy(tm->origins.p, origins, static_cast<size_t>(rows) * 8, cudaMemcpyHostToDevice), "origins");
            ck(cudaMemcpy2D(tm->probs.p, static_cast<size_t>(tm->pitch) * 8, probs, static_cast<size_t>(R) * 8,
                            static_cast<size_t>(R) * 8, static_cast<size_t>(rows), cudaMemcpyHostToDevice),
               "probs");
        }
        *out = tm.release();
    });
}

// ---------------------------------------------------------------- stage (ii)

gm_code gm_bellman_step(gm_model* m, gm_matrix* tm, const double* t0x, const double* v_next, double* v_out,
                        uint32_t* pol, uint32_t* wst, gm_status* st) {
    return guarded(st, [&] {
        check_spec(m->M.spec, m->M.X);
        prepare(m);
        const int64_t n_x = m->M.n_x();
        if (tm && (tm->row_begin != 0 || tm->row_end != m->M.rows()))
            throw ConfigErr("bellman_step: the matrix must cover every row");
        if (tm && t0x && m->M.spec.reach()) {
            const size_t n = static_cast<size_t>(tm->row_end - tm->row_begin);
            tm->t0x.ensure(std::max<size_t>(n, 1), "target-hit vector");
            ck(cudaMemcpy(tm->t0x.p, t0x, n * 8, cudaMemcpyHostToDevice), "t0x");
            tm->has_t0x = true;
        }
        if (tm) ensure_t0x(m, tm);
        DevBuf<double> vn, vo;
        DevBuf<uint32_t> dp, dw;
        vn.ensure(static_cast<size_t>(n_x), "v_next");
        vo.ensure(static_cast<size_t>(n_x), "v_out");
        dp.ensure(static_cast<size_t>(n_x), "policy");
        dw.ensure(static_cast<size_t>(n_x), "worst");
        ck(cudaMemcpyAsync(vn.p, v_next, static_cast<size_t>(n_x) * 8, cudaMemcpyHostToDevice, m->stream), "v_next");
        {
            Launch L(gmk::KF_MISC, m->stream);
            gmk::zero_absorbing(m->D, vn.p, m->stream);
        }
        step_states(m, tm, 0, n_x, vn.p, vo.p, dp.p, dw.p, m->stream);
        ck(cudaStreamSynchronize(m->stream), "bellman step");
        raise_device_error(m);
        ck(cudaMemcpy(v_out, vo.p, static_cast<size_t>(n_x) * 8, cudaMemcpyDeviceToHost), "v_out");
        if (pol) ck(cudaMemcpy(pol, dp.p, static_cast<size_t>(n_x) * 4, cudaMemcpyDeviceToHost), "policy");
        if (wst) ck(cudaMemcpy(wst, dw.p, static_cast<size_t>(n_x) * 4, cudaMemcpyDeviceToHost), "worst");
    });
}

gm_code gm_step_device(gm_model* m, gm_matrix* tm, int64_t x0, int64_t x1, const double* d_v_next, double* d_v_out,
                       uint32_t* d_pol, uint32_t* d_wst, void* stream, gm_status* st) {
    return guarded(st, [&] {
        if (x0 < 0 || x1 > m->M.n_x() || x0 > x1) throw std::out_of_range("step_device: state range");
        prepare(m);
        if (tm) ensure_t0x(m, tm);
        m->ofa_cache_steps = true; // sharded sweeps step the same rows T times (freed with the model)
        step_states(m, tm, x0, x1, d_v_next, d_v_out, d_pol, d_wst, static_cast<cudaStream_t>(stream));
    });
}

gm_code gm_store_probe(double* d_buf, int64_t n, uint64_t seed, void* stream, gm_status* st) {
    return guarded(st, [&] { gmk::store_probe(d_buf, n, seed, static_cast<cudaStream_t>(stream)); });
}

gm_code gm_model_release_ofa_cache(gm_model* m, gm_status* st) {
    return guarded(st, [&] {
        if (m->dev_ready) ck(cudaSetDevice(m->device), "cudaSetDevice");
        m->ofa_valid = false;
        m->ofa_mass.release();
        m->ofa_origin.release();
        m->ofa_t0x.release();
        m->ofa_flag.release();
    });
}

gm_code gm_copy_row_values(gm_model* m, double* out, int64_t n, gm_status* st) {
    return guarded(st, [&] {
        prepare(m);
        if (n < 0 || static_cast<size_t>(n) > m->d_vin.n) throw std::out_of_range("copy_row_values: size");
        ck(cudaStreamSynchronize(m->stream), "sync");
        if (n) ck(cudaMemcpy(out, m->d_vin.p, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToHost), "v_in");
    });
}

gm_code gm_check_device_errors(gm_model* m, gm_status* st) {
    return guarded(st, [&] {
        prepare(m);
        raise_device_error(m);
    });
}

gm_code gm_zero_absorbing_device(gm_model* m, double* d_v, void* stream, gm_status* st) {
    return guarded(st, [&] {
        prepare(m);
        Launch L(gmk::KF_MISC, static_cast<cudaStream_t>(stream));
        gmk::zero_absorbing(m->D, d_v, static_cast<cudaStream_t>(stream));
    });
}

gm_code gm_synthesize(gm_model* m, gm_result** out, gm_status* st) {
    return guarded(st, [&] {
        check_spec(m->M.spec, m->M.X);
        if (m->M.mode == GM_MODE_MATRIX_) {
            const uint64_t need = m->M.memory_estimate();
            if (m->M.mem_budget != 0 && need > m->M.mem_budget) {
                std::ostringstream os;
                os << "matrix mode needs " << need << " bytes but the budget is " << m->M.mem_budget
                   << "; use ofa mode";
                throw MemoryErr(os.str());
            }
            prepare(m);
            size_t free_b = 0, total_b = 0;
            ck(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
            free_b += cached_bytes(); // released matrices kept for reuse count as free
            const uint64_t dev_need = need + static_cast<uint64_t>(m->M.rows()) * 16 +
                                      static_cast<uint64_t>(m->M.rows()) * static_cast<uint64_t>(m->D.pitch - m->M.R) * 8;
            if (dev_need > static_cast<uint64_t>(free_b)) {
                std::ostringstream os;
                os << "matrix mode needs " << dev_need << " bytes of device memory but only " << free_b
                   << " are free; use ofa mode";
                throw MemoryErr(os.str());
            }
            PhaseTimer pt(m);
            pt.mark(0);
            gm_matrix tm;
            build_rows(m, 0, m->M.rows(), &tm, m->M.spec.reach());
            *out = run_backward(m, &tm, &pt);
        } else {
            prepare(m);
            PhaseTimer pt(m);
            pt.mark(0);
            *out = run_backward(m, nullptr, &pt);
        }
    });
}

gm_code gm_synthesize_with_matrix(gm_model* m, gm_matrix* tm, const double* t0x, gm_result** out, gm_status* st) {
    return guarded(st, [&] {
        check_spec(m->M.spec, m->M.X);
        prepare(m);
        check_matrix_model(tm, m);
        if (tm->row_begin != 0 || tm->row_end != m->M.rows())
            throw ConfigErr("synthesize_with_matrix: the matrix must cover every row");
        if (m->M.spec.reach()) {
            gm_status s2;
            if (gm_mask_absorbing(m, tm, &s2) != GM_OK) throw CudaErr(s2.msg);
            if (t0x) {
                tm->t0x.ensure(static_cast<size_t>(std::max<int64_t>(tm->row_end - tm->row_begin, 1)), "t0x");
                ck(cudaMemcpy(tm->t0x.p, t0x, static_cast<size_t>(tm->row_end - tm->row_begin) * 8,
                              cudaMemcpyHostToDevice),
                   "t0x");
                tm->has_t0x = true;
            }
            ensure_t0x(m, tm); // t0x NULL: built on demand (synthesis.hpp:49-50)
        }
        *out = run_backward(m, tm);
    });
}

gm_code gm_result_shape(const gm_result* r, int64_t* n_x, int32_t* T, int32_t* has_abs, int32_t* mode,
                        gm_status* st) {
    return guarded(st, [&] {
        if (n_x) *n_x = r->n_x;
        if (T) *T = r->T;
        if (has_abs) *has_abs = r->absorbing.empty() ? 0 : 1;
        if (mode) *mode = r->mode;
    });
}

gm_code gm_result_copy(const gm_result* r, double* values, uint32_t* policy, uint32_t* worst, uint8_t* absorbing,
                       gm_status* st) {
    return guarded(st, [&] {
        if (values) std::memcpy(values, r->values.data(), r->values.size() * 8);
        if (policy) std::memcpy(policy, r->policy.data(), r->policy.size() * 4);
        if (worst) std::memcpy(worst, r->worst.data(), r->worst.size() * 4);
        if (absorbing && !r->absorbing.empty()) std::memcpy(absorbing, r->absorbing.data(), r->absorbing.size());
    });
}

gm_code gm_result_data(const gm_result* r, const double** values, const uint32_t** policy, const uint32_t** worst,
                       const uint8_t** absorbing, gm_status* st) {
    return guarded(st, [&] {
        if (values) *values = r->values.data();
        if (policy) *policy = r->policy.data();
        if (worst) *worst = r->worst.data();
        if (absorbing) *absorbing = r->absorbing.empty() ? nullptr : r->absorbing.data();
    });
}

gm_code gm_result_from_tables(const gm_model* m, const double* values, const uint32_t* policy, const uint32_t* worst,
                              gm_result** out, gm_status* st) {
    return guarded(st, [&] {
        auto* r = new gm_result;
        r->meta = m->M;
        r->mode = m->M.mode;
        r->n_x = m->M.n_x();
        r->T = m->M.spec.horizon;
        const size_t nx = static_cast<size_t>(r->n_x);
        r->values.assign(values, values + nx * (r->T + 1));
        r->policy.assign(policy, policy + nx * r->T);
        r->worst.assign(worst, worst + nx * r->T);
        if (m->M.spec.reach()) {
            r->absorbing.resize(nx);
            const Grid& g = m->M.X;
            for (size_t i = 0; i < nx; ++i) {
                const std::vector<double> p = grid_point(g, static_cast<int64_t>(i));
                r->absorbing[i] = (m->M.spec.target.contains(p) ||
                                   (m->M.spec.avoid.dim() > 0 && m->M.spec.avoid.contains(p)))
                                      ? 1
                                      : 0;
            }
        }
        *out = r;
    });
}

gm_code gm_model_last_times(const gm_model* m, double* build_ms, double* sweep_ms, gm_status* st) {
    return guarded(st, [&] {
        if (build_ms) *build_ms = m->last_build_ms;
        if (sweep_ms) *sweep_ms = m->last_sweep_ms;
    });
}

gm_code gm_model_clone(const gm_model* m, gm_model** out, gm_status* st) {
    return guarded(st, [&] {
        auto* c = new gm_model;
        c->M = m->M; // host description only: device state is created on first use
        *out = c;
    });
}

gm_code gm_result_write(const gm_result* r, const char* path, gm_status* st) {
    return guarded(st, [&] {
        // write_results, io.cpp:142-179
        std::ofstream os(path, std::ios::binary);
        if (!os) throw IoErr(std::string("cannot open '") + path + "' for writing");
        const Model& M = r->meta;
        const int64_t n_x = r->n_x;
        const int T = r->T;
        os << "gridmdp-results" << ' ' << 1 << '\n';
        os << "mode = " << (r->mode == GM_MODE_MATRIX ? "matrix" : "ofa") << ";\n";
        os << "gamma = " << fmt_shortest(M.noise.gamma) << ";\n";
        os << "spec.type = " << kind_name(M.spec.kind) << ";\n";
        os << "spec.time_steps = " << T << ";\n";
        if (M.spec.target.dim() > 0) {
            os << "target.lb = " << fmt_vec(M.spec.target.lo) << ";\n";
            os << "target.ub = " << fmt_vec(M.spec.target.hi) << ";\n";
        }
        if (M.spec.avoid.dim() > 0) {
            os << "avoid.lb = " << fmt_vec(M.spec.avoid.lo) << ";\n";
            os << "avoid.ub = " << fmt_vec(M.spec.avoid.hi) << ";\n";
        }
        grid_lines(os, "states", M.X);
        grid_lines(os, "inputs", M.U);
        grid_lines(os, "disturbances", M.W);
        os << "array.values = f64 " << n_x << " " << (T + 1) << ";\n";
        os << "array.policy = u32 " << n_x << " " << T << ";\n";
        os << "array.worst_dist = u32 " << n_x << " " << T << ";\n";
        os << "array.absorbing = u8 " << r->absorbing.size() << " 1;\n";
        os << "payload\n";
        const size_t nx = static_cast<size_t>(n_x);
        std::string buf;
        buf.reserve(nx * (T + 1) * 8);
        auto flush = [&] {
            os.write(buf.data(), static_cast<std::streamsize>(buf.size()));
            buf.clear();
        };
        for (size_t i = 0; i < nx; ++i)
            for (int k = 0; k <= T; ++k) {
                uint64_t u;
                std::memcpy(&u, &r->values[static_cast<size_t>(k) * nx + i], 8);
                for (int b = 0; b < 8; ++b) buf.push_back(static_cast<char>((u >> (8 * b)) & 0xff));
            }
        flush();
        for (size_t i = 0; i < nx; ++i)
            for (int k = 0; k < T; ++k) {
                const uint32_t u = r->policy[static_cast<size_t>(k) * nx + i];
                for (int b = 0; b < 4; ++b) buf.push_back(static_cast<char>((u >> (8 * b)) & 0xff));
            }
        flush();
        for (size_t i = 0; i < nx; ++i)
            for (int k = 0; k < T; ++k) {
                const uint32_t u = r->worst[static_cast<size_t>(k) * nx + i];
                for (int b = 0; b < 4; ++b) buf.push_back(static_cast<char>((u >> (8 * b)) & 0xff));
            }
        flush();
        for (uint8_t b : r->absorbing) buf.push_back(static_cast<char>(b));
        flush();
        if (!os) throw IoErr(std::string("failed while writing '") + path + "'");
    });
}

void gm_result_free(gm_result* r) { delete r; }

void gm_release_cached_memory(void) { flush_cache(); }

} // extern "C"

// ---------------------------------------------------------------- internal hooks (gm_internal.hpp)

gm_code gmi_step_device_mirrored(gm_model* m, gm_matrix* tm, int64_t x0, int64_t x1, const double* d_v_next,
                                  double* d_v_out, uint32_t* d_pol, uint32_t* d_wst, void* stream,
                                  const gmk::GmMirror* mir, gm_status* st) {
    return guarded(st, [&] {
        if (x0 < 0 || x1 > m->M.n_x() || x0 > x1) throw std::out_of_range("step_device: state range");
        if (mir && (mir->n < 0 || mir->n > gmk::kMaxMirrors)) throw std::out_of_range("step_device: mirror count");
        prepare(m);
        if (tm) ensure_t0x(m, tm);
        m->ofa_cache_steps = true;
        step_states(m, tm, x0, x1, d_v_next, d_v_out, d_pol, d_wst, static_cast<cudaStream_t>(stream), mir);
    });
}

gm_result* gmi_result_new(const gm_model* m, int mode, const uint8_t* absorbing) {
    std::unique_ptr<gm_result> r(new gm_result);
    r->meta = m->M;
    r->mode = mode;
    r->n_x = m->M.n_x();
    r->T = m->M.spec.horizon;
    const size_t nx = static_cast<size_t>(r->n_x);
    r->values.resize(nx * (r->T + 1));
    r->policy.resize(nx * r->T);
    r->worst.resize(nx * r->T);
    const bool reach = m->M.spec.reach();
    std::fill(r->values.begin() + static_cast<std::ptrdiff_t>(nx) * r->T, r->values.end(), reach ? 0.0 : 1.0);
    if (reach) r->absorbing.assign(absorbing, absorbing + nx);
    return r.release();
}

void gmi_result_tables(gm_result* r, double** values, uint32_t** policy, uint32_t** worst) {
    *values = r->values.data();
    *policy = r->policy.data();
    *worst = r->worst.data();
}

gm_code gmi_guarded(gm_status* st, const std::function<void()>& f) { return guarded(st, f); }

[[noreturn]] void gmi_throw(int code, const std::string& msg) {
    switch (code) {
        case GM_ERR_CONFIG: throw ConfigErr(msg);
        case GM_ERR_MEMORY: throw MemoryErr(msg);
        case GM_ERR_DOMAIN: throw DomainErr(msg);
        case GM_ERR_IO: throw IoErr(msg);
        case GM_ERR_RANGE: throw std::out_of_range(msg);
        case GM_ERR_CUDA: throw CudaErr(msg);
        default: throw std::runtime_error(msg);
    }
}


// ===========================================================================
// results reader (read_results, io.cpp:181-230) and the closed-loop simulator
// (simulate / roll_one / write_trajectory_csv, sim.cpp:16-154)
// ===========================================================================

struct gm_sim {
    int n = 0, m = 0, p = 0, T = 0;
    int32_t runs = 0;
    bool traj = false;
    std::vector<uint8_t> sat;
    std::vector<int32_t> steps;
    std::vector<double> states, inputs, dists; // [run][k][d], T+1 / T / T rows per run
};

namespace {


// contains(grid, x), grid.cpp:67-75
bool grid_contains(const Grid& g, const std::vector<double>& x) {
    if (static_cast<int>(x.size()) != g.dim()) return false;
    for (int d = 0; d < g.dim(); ++d) {
        const double t = (x[d] - g.lb[d]) / g.eta[d];
        if (t < -0.5 - 1e-9 || t > static_cast<double>(g.count[d] - 1) + 0.5 + 1e-9) return false;
    }
    return true;
}

void put_shortest(std::ostream& os, double v) { // std::to_chars, sim.cpp:109-114
    char buf[32];
    auto r = std::to_chars(buf, buf + sizeof buf, v);
    os.write(buf, r.ptr - buf);
}

} // namespace

extern "C" {

gm_code gm_result_read(const char* path, gm_result** out, gm_status* st) {
    return guarded(st, [&] {
        std::ifstream is(path, std::ios::binary);
        if (!is) throw IoErr(std::string("cannot open '") + path + "'");
        ManifestR mf(is, "gridmdp-results");
        auto r = std::make_unique<gm_result>();
        r->mode = mf.str("mode") == "matrix" ? GM_MODE_MATRIX : GM_MODE_OFA;
        r->meta.noise.gamma = mf.number("gamma");
        const std::string kind = mf.str("spec.type");
        if (kind == "safety") r->meta.spec.kind = GM_SPEC_SAFETY;
        else if (kind == "reachability" || kind == "reach") r->meta.spec.kind = GM_SPEC_REACH;
        else if (kind == "reach-avoid" || kind == "reach_avoid") r->meta.spec.kind = GM_SPEC_REACH_AVOID;
        else throw ConfigErr("unknown spec type '" + kind + "'");
        r->meta.spec.horizon = static_cast<int>(mf.integer("spec.time_steps"));
        if (mf.has("target.lb")) r->meta.spec.target = BoxV{mf.vec("target.lb"), mf.vec("target.ub")};
        if (mf.has("avoid.lb")) r->meta.spec.avoid = BoxV{mf.vec("avoid.lb"), mf.vec("avoid.ub")};
        r->meta.X = mf.grid("states");
        r->meta.U = mf.grid("inputs");
        r->meta.W = mf.grid("disturbances");
        std::istringstream vshape(mf.str("array.values"));
        std::string tag;
        int64_t n_x = 0;
        int cols = 0;
        vshape >> tag >> n_x >> cols;
        if (tag != "f64" || n_x != r->meta.X.total || cols != r->meta.spec.horizon + 1)
            throw IoErr("values array shape disagrees with the manifest");
        std::istringstream ashape(mf.str("array.absorbing"));
        int64_t n_abs = 0;
        int one = 0;
        ashape >> tag >> n_abs >> one;
        if (tag != "u8" || (n_abs != 0 && n_abs != n_x)) throw IoErr("absorbing array shape disagrees with the manifest");
        const int T = r->meta.spec.horizon;
        r->n_x = n_x;
        r->T = T;
        const size_t nx = static_cast<size_t>(n_x);
        std::vector<char> buf(nx * (T + 1) * 8);
        auto get = [&](size_t bytes) {
            buf.resize(bytes);
            is.read(buf.data(), static_cast<std::streamsize>(bytes));
            if (!is) throw IoErr("truncated payload");
        };
        // state-major on disk (io.cpp:171-177), column-major in memory
        get(nx * (T + 1) * 8);
        r->values.resize(nx * (T + 1));
        for (size_t i = 0; i < nx; ++i)
            for (int k = 0; k <= T; ++k)
                std::memcpy(&r->values[static_cast<size_t>(k) * nx + i], &buf[(i * (T + 1) + k) * 8], 8);
        for (HostVec<uint32_t>* dst : {&r->policy, &r->worst}) {
            get(nx * T * 4);
            dst->resize(nx * T);
            for (size_t i = 0; i < nx; ++i)
                for (int k = 0; k < T; ++k)
                    std::memcpy(&(*dst)[static_cast<size_t>(k) * nx + i], &buf[(i * T + k) * 4], 4);
        }
        r->absorbing.resize(static_cast<size_t>(n_abs));
        if (n_abs > 0) {
            is.read(reinterpret_cast<char*>(r->absorbing.data()), n_abs);
            if (!is) throw IoErr("truncated payload");
        }
        char extra;
        if (is.get(extra)) throw IoErr("trailing bytes after the declared payload");
        *out = r.release();
    });
}

gm_code gm_query_policy(const gm_result* r, const double* x, int32_t n, int32_t k, double* u_out, gm_status* st) {
    return guarded(st, [&] {
        // query_policy, synthesis.cpp:230-239
        if (k < 1 || k > r->T) {
            std::ostringstream os;
            os << "query_policy: step " << k << " outside [1, " << r->T << "]";
            throw std::out_of_range(os.str());
        }
        const int64_t ix = grid_index(r->meta.X, std::vector<double>(x, x + n)); // point_to_index
        const uint32_t iu = r->policy[static_cast<size_t>(k - 1) * static_cast<size_t>(r->n_x) + static_cast<size_t>(ix)];
        const std::vector<double> u = grid_point(r->meta.U, static_cast<int64_t>(iu)); // index_to_point
        std::copy(u.begin(), u.end(), u_out);
    });
}

gm_code gm_result_value_at(const gm_result* r, const double* x, int32_t n, int32_t k, double* v, gm_status* st) {
    return guarded(st, [&] {
        if (k < 0 || k > r->T) throw std::out_of_range("value_at: step outside [0, T]");
        const std::vector<double> p(x, x + n);
        const int64_t ix = grid_index(r->meta.X, p); // point_to_index (out_of_range outside)
        *v = r->values[static_cast<size_t>(k) * static_cast<size_t>(r->n_x) + static_cast<size_t>(ix)];
    });
}

gm_code gm_model_sim_defaults(const gm_model* m, int32_t* runs, uint64_t* seed, gm_status* st) {
    return guarded(st, [&] {
        *runs = m->M.cfg.runs;
        *seed = m->M.cfg.seed;
    });
}

gm_code gm_simulate(gm_model* m, const gm_result* res, const double* x0, int32_t n_x0, int32_t runs, uint64_t seed,
                    int32_t worst_case, int32_t want_traj, gm_sim** out, gm_status* st) {
    return guarded(st, [&] {
        const Model& M = m->M;
        const SpecV& spec = res->meta.spec; // cmd_simulate passes res.spec (gridmdp_main.cpp:130)
        check_spec(spec, M.X);               // validate_spec, sim.cpp:88
        if (runs < 1) throw ConfigErr("simulate: need at least one run");
        const std::vector<double> x(x0, x0 + std::max(n_x0, 0));
        if (!grid_contains(M.X, x)) throw std::out_of_range("simulate: x0 lies outside the quantized region");
        if (spec.horizon > res->T || res->meta.X.total != M.X.total)
            throw ConfigErr("simulate: synthesis result does not match the model/spec");
        prepare(m);
        const int n = M.X.dim(), mu = M.U.dim(), p = M.W.dim(), T = spec.horizon;
        gmk::SimArgs A{};
        A.runs = runs;
        A.T = T;
        A.reach = spec.reach() ? 1 : 0;
        A.has_avoid = spec.avoid.dim() > 0 ? 1 : 0;
        A.worst_case = worst_case ? 1 : 0;
        A.seed = seed;
        if (M.noise.family == GM_CUSTOM) { // custom_sup_estimate (noise.cpp:307-333) on the host
            const int nd = M.X.dim();
            int per_dim = 17;
            int64_t total = 1;
            for (int d = 0; d < nd; ++d) total *= per_dim;
            if (total > 100000) per_dim = 5;
            std::vector<double> pt(static_cast<size_t>(nd));
            std::vector<int64_t> idx(static_cast<size_t>(nd), 0);
            double sup = 0.0;
            for (;;) {
                for (int d = 0; d < nd; ++d) {
                    const double t = per_dim == 1 ? 0.5 : static_cast<double>(idx[d]) / (per_dim - 1);
                    pt[d] = M.noise.p1[d] + t * (M.noise.p2[d] - M.noise.p1[d]);
                }
                sup = std::max(sup, eval_expr(M.noise.pdf, pt.data(), nullptr, nullptr));
                int d = nd - 1;
                for (; d >= 0; --d) {
                    if (++idx[d] < per_dim) break;
                    idx[d] = 0;
                }
                if (d < 0) break;
            }
            if (!(sup > 0.0)) throw DomainErr("sample: custom density appears to be zero on its support");
            A.custom_sup = sup * 1.5;
        }
        for (int d = 0; d < n; ++d) {
            A.x0[d] = x[d];
            if (spec.target.dim() == n) { A.tlo[d] = spec.target.lo[d]; A.thi[d] = spec.target.hi[d]; }
            if (spec.avoid.dim() == n) { A.alo[d] = spec.avoid.lo[d]; A.ahi[d] = spec.avoid.hi[d]; }
        }
        const Grid& RX = res->meta.X;
        const Grid& RU = res->meta.U;
        for (int d = 0; d < RX.dim() && d < GMD_MAXD; ++d) {
            A.rs_lb[d] = RX.lb[d];
            A.rs_eta[d] = RX.eta[d];
            A.rs_count[d] = RX.count[d];
            A.rs_stride[d] = RX.stride[d];
        }
        A.ru_dim = RU.dim();
        for (int d = 0; d < RU.dim() && d < GMD_MAXD; ++d) {
            A.ru_lb[d] = RU.lb[d];
            A.ru_eta[d] = RU.eta[d];
            A.ru_stride[d] = RU.stride[d];
        }
        A.rs_n = res->n_x;
        const size_t nT = static_cast<size_t>(res->n_x) * static_cast<size_t>(res->T);
        DevBuf<uint32_t> d_pol, d_wst;
        d_pol.ensure(std::max<size_t>(nT, 1), "policy table");
        d_wst.ensure(std::max<size_t>(nT, 1), "worst-disturbance table");
        if (nT) {
            ck(cudaMemcpy(d_pol.p, res->policy.data(), nT * 4, cudaMemcpyHostToDevice), "policy table");
            ck(cudaMemcpy(d_wst.p, res->worst.data(), nT * 4, cudaMemcpyHostToDevice), "worst-disturbance table");
        }
        A.policy = d_pol.p;
        A.worst = d_wst.p;
        const size_t R = static_cast<size_t>(runs);
        DevBuf<uint8_t> d_sat;
        DevBuf<int> d_steps;
        DevBuf<double> d_st, d_in, d_ds;
        d_sat.ensure(R, "run flags");
        d_steps.ensure(R, "run steps");
        A.satisfied = d_sat.p;
        A.steps = d_steps.p;
        if (want_traj) {
            d_st.ensure(R * (T + 1) * std::max(n, 1), "trajectories");
            d_in.ensure(R * T * std::max(mu, 1), "trajectories");
            d_ds.ensure(R * T * std::max(p, 1), "trajectories");
            A.states = d_st.p;
            A.inputs = mu ? d_in.p : nullptr;
            A.dists = p ? d_ds.p : nullptr;
        }
        A.err = m->d_err.p;
        {
            Launch L(gmk::KF_MISC, m->stream);
            gmk::simulate(m->D, A, m->stream);
        }
        ck(cudaStreamSynchronize(m->stream), "simulate");
        unsigned long long bad = ULLONG_MAX;
        ck(cudaMemcpy(&bad, m->d_err.p, sizeof bad, cudaMemcpyDeviceToHost), "error slot");
        if (bad != ULLONG_MAX) {
            const unsigned long long none = ULLONG_MAX;
            ck(cudaMemcpy(m->d_err.p, &none, sizeof none, cudaMemcpyHostToDevice), "error slot");
            throw DomainErr("simulate: the dynamics hit a domain error in run " + std::to_string(bad));
        }
        auto s = std::make_unique<gm_sim>();
        s->n = n;
        s->m = mu;
        s->p = p;
        s->T = T;
        s->runs = runs;
        s->traj = want_traj != 0;
        s->sat.resize(R);
        s->steps.resize(R);
        ck(cudaMemcpy(s->sat.data(), d_sat.p, R, cudaMemcpyDeviceToHost), "run flags");
        ck(cudaMemcpy(s->steps.data(), d_steps.p, R * 4, cudaMemcpyDeviceToHost), "run steps");
        if (want_traj) {
            s->states.resize(R * (T + 1) * n);
            s->inputs.resize(R * T * mu);
            s->dists.resize(R * T * p);
            if (n) ck(cudaMemcpy(s->states.data(), d_st.p, s->states.size() * 8, cudaMemcpyDeviceToHost), "trajectories");
            if (mu) ck(cudaMemcpy(s->inputs.data(), d_in.p, s->inputs.size() * 8, cudaMemcpyDeviceToHost), "trajectories");
            if (p) ck(cudaMemcpy(s->dists.data(), d_ds.p, s->dists.size() * 8, cudaMemcpyDeviceToHost), "trajectories");
        }
        *out = s.release();
    });
}

gm_code gm_sim_summary(const gm_sim* s, int32_t* runs, int64_t* satisfied, double* rate, gm_status* st) {
    return guarded(st, [&] {
        int64_t ok = 0;
        for (uint8_t b : s->sat) ok += b;
        *runs = s->runs;
        *satisfied = ok;
        if (s->runs < 1) throw ConfigErr("empirical_rate: empty batch");
        *rate = static_cast<double>(ok) / static_cast<double>(s->runs); // empirical_rate, sim.cpp:103-108
    });
}

gm_code gm_sim_copy(const gm_sim* s, uint8_t* satisfied, int32_t* steps, double* states, double* inputs,
                    double* dists, gm_status* st) {
    return guarded(st, [&] {
        if (satisfied) std::memcpy(satisfied, s->sat.data(), s->sat.size());
        if (steps) std::memcpy(steps, s->steps.data(), s->steps.size() * 4);
        if ((states || inputs || dists) && !s->traj) throw ConfigErr("simulate: trajectories were not recorded");
        if (states) std::memcpy(states, s->states.data(), s->states.size() * 8);
        if (inputs) std::memcpy(inputs, s->inputs.data(), s->inputs.size() * 8);
        if (dists) std::memcpy(dists, s->dists.data(), s->dists.size() * 8);
    });
}

gm_code gm_sim_write_csv(const gm_sim* s, const char* path, gm_status* st) {
    return guarded(st, [&] {
        // write_trajectory_csv, sim.cpp:117-154
        if (s->runs < 1) throw ConfigErr("write_trajectory_csv: empty batch");
        if (!s->traj) throw ConfigErr("simulate: trajectories were not recorded");
        std::ofstream os(path);
        if (!os) throw IoErr(std::string("cannot open '") + path + "' for writing");
        os << "run,k";
        for (int d = 0; d < s->n; ++d) os << ",x" << d;
        for (int d = 0; d < s->m; ++d) os << ",u" << d;
        for (int d = 0; d < s->p; ++d) os << ",w" << d;
        os << ",flag\n";
        const size_t T = static_cast<size_t>(s->T);
        for (size_t r = 0; r < static_cast<size_t>(s->runs); ++r) {
            const int steps = s->steps[r];
            for (int k = 0; k <= steps; ++k) {
                os << r << ',' << k;
                for (int d = 0; d < s->n; ++d) {
                    os << ',';
                    put_shortest(os, s->states[(r * (T + 1) + k) * s->n + d]);
                }
                for (int d = 0; d < s->m; ++d) {
                    os << ',';
                    if (k < steps) put_shortest(os, s->inputs[(r * T + k) * s->m + d]);
                }
                for (int d = 0; d < s->p; ++d) {
                    os << ',';
                    if (k < steps) put_shortest(os, s->dists[(r * T + k) * s->p + d]);
                }
                os << ',' << (s->sat[r] ? 1 : 0) << '\n';
            }
        }
        if (!os) throw IoErr(std::string("failed while writing '") + path + "'");
    });
}

void gm_sim_free(gm_sim* s) { delete s; }

} // extern "C"
