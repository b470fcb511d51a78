// host.cu -- C-ABI implementation (include/bode.h): argument validation with
// the reference's error semantics, device buffers, multi-GPU sharding,
// H2D/compute/D2H pipelining and the device-resident outer loop.
//
// Reference behaviour mirrored here:
//   integrateBatch validation order  batch_driver.cpp:42-50
//   ToleranceSettings::validate      ode_problem.hpp:46-53
//   contiguous static partition      batch_driver.cpp:68-73 (here: across GPUs)
//   outerLoop window schedule        batch_driver.cpp:99-105
//   per-system stats merge           batch_driver.cpp:109-110, ode_problem.hpp:72-80
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <link.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/bode.h"
#include "dispatch.h"

namespace {

using bode::DevStats;
using bode::DevTol;
using bode::KernelEntry;

thread_local std::string g_last_error;
std::atomic<long long> g_launches{0};
std::atomic<int> g_block_override{0};
std::atomic<int> g_force_wide{0};  // one-system-per-block kernels even where lane kernels exist
std::atomic<long long> g_attempt_budget{0};  // per-window attempts per system (0: none)
std::atomic<int> g_shard_layout{0};  // 0: contiguous shards (the reference's), 1: block-cyclic
std::atomic<int> g_persistent{0};  // dynamic-refill kernels where compiled (opt-in)
std::atomic<double> g_repack_threshold{0.7};  // outer loop: re-pack below this efficiency
std::atomic<int> g_presort_param{-2};  // outer loop: sort by |g[row]| first (-1 off, -2 auto)

// The parameter row that is a system's stiffness (its spectral radius up to a
// constant) for the built-in problems: expDecay's g0 (the reference's
// specRadHint, problems.cpp:140-142). -1: none known.
int stiffness_param_row(const bode_problem_t* p) {
    return p->kind == BODE_PROBLEM_EXPDECAY && p->param_dim >= 1 ? 0 : -1;
}

int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

#define BODE_CUDA(call)                                                                   \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess)                                                            \
            return fail(BODE_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

const double kPleiadesIC[28] = {
    // data/pleiades_ic.txt (FNV-1a 0x5583feb418028048, problems.hpp:29):
    // x1..x7, y1..y7, x'1..x'7, y'1..y'7
    3.0,  3.0, -1.0, -3.0, 2.0, -2.0, 2.0,  3.0,  -3.0, 2.0, 0.0,  0.0,   -4.0, 4.0,
    0.0,  0.0, 0.0,  0.0,  0.0, 1.75, -1.5, 0.0,  0.0,  0.0, -1.25, 1.0, 0.0,  0.0};

DevTol to_dev(const bode_tol_t* t, int dim) {
    DevTol d;
    d.eps = t->eps;
    d.abs_tol = t->abs_tol;
    d.rel_tol = t->rel_tol;
    d.uround = t->uround;
    d.tiny = t->tiny;
    d.safety = t->safety;
    d.p1 = t->p1;
    d.errcon = t->errcon;
    d.pgrow = t->pgrow;
    d.pshrnk = t->pshrnk;
    d.h_min_floor = t->h_min_floor;
    d.kappa = t->kappa;
    d.powtab = nullptr;
    d.rkc_coef = nullptr;
    static const int refill_min = [] {
        const char* s = std::getenv("BODE_REFILL_MIN");  // tuning knob, default 8
        const int v = s ? std::atoi(s) : 8;
        return v < 1 ? 1 : v > 32 ? 32 : v;
    }();
    d.refill_min = refill_min;
    d.stride = 0;
    d.dim = dim;
    d.scratch = nullptr;
    d.max_attempts = g_attempt_budget.load();
    d.trace = nullptr;
    d.trace_cap = 0;
    d.trace_count = nullptr;
    return d;
}

// ---- host libm pow tables for the EXACT policy (arith.cuh pow_glibc) ----
// glibc's pow reads __pow_log_data and __exp_data (hidden symbols); they are
// located in the loaded libm by content signature and copied verbatim, so
// the device evaluates pow over exactly the host's tables. Only the x86-64
// FMA build of pow is restated, so this also requires the ifunc condition
// that selects it (FMA and AVX2).
struct PowTabSearch {
    const double* log_head = nullptr;
    const double* exp_head = nullptr;
    const uint64_t* exp_tab = nullptr;
};

const unsigned char* find8(const unsigned char* h, size_t n, const void* pat, size_t m) {
    for (size_t i = 0; i + m <= n; i += 8)
        if (std::memcmp(h + i, pat, m) == 0) return h + i;
    return nullptr;
}

int powtab_cb(struct dl_phdr_info* info, size_t, void* data) {
    if (!info->dlpi_name || !std::strstr(info->dlpi_name, "libm.so")) return 0;
    auto* s = static_cast<PowTabSearch*>(data);
    const double log_sig[3] = {0x1.62e42fefa3800p-1, 0x1.ef35793c76730p-45, -0.5};
    const double exp_sig[2] = {0x1.71547652b82fep+7, 0x1.8p52};
    const uint64_t tab_sig[4] = {0x0ull, 0x3ff0000000000000ull, 0x3c9b3b4f1a88bf6eull,
                                 0x3feff63da9fb3335ull};
    for (int j = 0; j < info->dlpi_phnum; ++j) {
        const ElfW(Phdr)& ph = info->dlpi_phdr[j];
        if (ph.p_type != PT_LOAD || !(ph.p_flags & PF_R) || (ph.p_flags & PF_X)) continue;
        uintptr_t b = (info->dlpi_addr + ph.p_vaddr + 7) & ~uintptr_t(7);
        const auto* base = reinterpret_cast<const unsigned char*>(b);
        const size_t n = ph.p_memsz & ~size_t(7);
        if (!s->log_head) s->log_head = (const double*)find8(base, n, log_sig, sizeof log_sig);
        if (!s->exp_head) s->exp_head = (const double*)find8(base, n, exp_sig, sizeof exp_sig);
        if (!s->exp_tab) s->exp_tab = (const uint64_t*)find8(base, n, tab_sig, sizeof tab_sig);
    }
    return 1;
}

// host copy of the 785-double table image, or empty when unavailable
const std::vector<double>& host_powtab() {
    static std::vector<double> img;
    static std::once_flag once;
    std::call_once(once, [] {
        __builtin_cpu_init();
        if (!__builtin_cpu_supports("fma") || !__builtin_cpu_supports("avx2")) return;
        dlopen("libm.so.6", RTLD_NOW | RTLD_GLOBAL);  // make sure it is mapped
        PowTabSearch s;
        dl_iterate_phdr(powtab_cb, &s);
        if (!s.log_head || !s.exp_head || !s.exp_tab) return;
        img.resize(785);
        std::memcpy(img.data(), s.log_head, 9 * sizeof(double));
        std::memcpy(img.data() + 9, s.log_head + 9, 512 * sizeof(double));
        std::memcpy(img.data() + 521, s.exp_head, 8 * sizeof(double));
        std::memcpy(img.data() + 529, s.exp_tab, 256 * sizeof(double));
    });
    return img;
}

// First compiled kernel for (problem, solver, policy). Several lane-group
// widths may be compiled for one problem; BODE_LANES=<L> (tuning knob, e.g.
// for A/B measurements) prefers the variant with that width. All variants
// give bitwise-identical results.
// Kernels registered at load time by problem libraries built against
// include/bode_problem.cuh (bode_register_kernels). Function-local statics, so
// registration from another library's static initializers is order-safe.
std::mutex& registry_mutex() {
    static std::mutex m;
    return m;
}
std::deque<KernelEntry>& registry() {  // deque: entries never move once added
    static std::deque<KernelEntry>* v = new std::deque<KernelEntry>();
    return *v;
}

template <class Seq>
const KernelEntry* find_in(const Seq& tab, const bode_problem_t* p, int solver, int arith,
                           int want_lanes, int want_maxreg, const KernelEntry** first) {
    for (const KernelEntry& e : tab) {
        if (e.kind == p->kind && e.dim == p->dim && e.param_dim == p->param_dim &&
            e.solver == solver && e.arith == arith) {
            const int cap = e.maxreg > 0 ? e.maxreg : 255;
            if ((want_lanes == 0 || e.lanes == want_lanes) &&
                (want_maxreg < 0 || cap == want_maxreg))
                return &e;
            if (!*first) *first = &e;
        }
    }
    return nullptr;
}

const KernelEntry* find_entry(const bode_problem_t* p, int solver, int arith) {
    int n = 0;
    const KernelEntry* tab = bode::kernel_table(&n);
    static const int want_lanes = [] {
        const char* s = std::getenv("BODE_LANES");
        return s ? std::atoi(s) : 0;
    }();
    static const int want_maxreg = [] {  // BODE_MAXREG=<cap> (255 = uncapped)
        const char* s = std::getenv("BODE_MAXREG");
        return s ? std::atoi(s) : -1;
    }();
    struct Span {
        const KernelEntry *b, *e;
        const KernelEntry* begin() const { return b; }
        const KernelEntry* end() const { return e; }
    };
    // one system per block (wide.cuh) for a problem kind with a run-time
    // dimension: when no lane-group kernel is compiled for p->dim, or forced
    auto wide = [&]() -> const KernelEntry* {
        for (int i = 0; i < n; ++i)
            if (tab[i].wide && tab[i].kind == p->kind && tab[i].param_dim == p->param_dim &&
                tab[i].solver == solver && tab[i].arith == arith)
                return &tab[i];
        return nullptr;
    };
    if (g_force_wide.load())
        if (const KernelEntry* e = wide()) return e;
    const KernelEntry* first = nullptr;
    if (const KernelEntry* e =
            find_in(Span{tab, tab + n}, p, solver, arith, want_lanes, want_maxreg, &first))
        return e;
    {
        std::lock_guard<std::mutex> lock(registry_mutex());
        if (const KernelEntry* e =
                find_in(registry(), p, solver, arith, want_lanes, want_maxreg, &first))
            return e;
    }
    if (first) return first;
    // a run-time-dimension lane kernel that holds p->dim (the smallest such
    // capacity), else one system per block
    const KernelEntry* pad = nullptr;
    for (int i = 0; i < n; ++i) {
        const KernelEntry& e = tab[i];
        if (e.cap >= p->dim && e.kind == p->kind && e.param_dim == p->param_dim &&
            e.solver == solver && e.arith == arith && (!pad || e.cap < pad->cap))
            pad = &e;
    }
    return pad ? pad : wide();
}

// The one-system-per-block entry for (kind, solver, arith), if any.
const KernelEntry* find_wide(const bode_problem_t* p, int solver, int arith) {
    int n = 0;
    const KernelEntry* tab = bode::kernel_table(&n);
    for (int i = 0; i < n; ++i)
        if (tab[i].wide && tab[i].kind == p->kind && tab[i].param_dim == p->param_dim &&
            tab[i].solver == solver && tab[i].arith == arith)
            return &tab[i];
    return nullptr;
}

int check_problem_shape(const bode_problem_t* p) {
    if (p == nullptr) return fail(BODE_E_INVALID_SHAPE, "problem is NULL");
    if (p->dim < 1) return fail(BODE_E_INVALID_SHAPE, "problem dim must be positive");
    if (p->param_dim < 0) return fail(BODE_E_INVALID_SHAPE, "negative param_dim");
    if (p->kind == BODE_PROBLEM_HEAT && p->dim < 2)
        return fail(BODE_E_INVALID_SHAPE, "heatEquation: need at least two interior points");
    return BODE_OK;
}

// Common validation of integrateBatch (batch_driver.cpp:42-50).
int validate_call(const bode_problem_t* p, int solver, int arith, double t, double t_end,
                  int64_t num, const void* g, const void* y, const bode_tol_t* tol,
                  const KernelEntry** entry) {
    if (!(t_end > t)) return fail(BODE_E_INVALID_INTERVAL, "integrateBatch: tNext must exceed t");
    int rc = check_problem_shape(p);
    if (rc) return rc;
    if (num < 1) return fail(BODE_E_INVALID_SHAPE, "numSystems must be positive");
    if (y == nullptr) return fail(BODE_E_INVALID_SHAPE, "state array is NULL");
    if (p->param_dim > 0 && g == nullptr)
        return fail(BODE_E_INVALID_SHAPE, "parameter array is NULL but param_dim > 0");
    if (tol == nullptr) return fail(BODE_E_INVALID_SHAPE, "tolerance settings are NULL");
    rc = bode_tol_validate(tol);
    if (rc) return rc;
    if (solver != BODE_SOLVER_RKCK && solver != BODE_SOLVER_RKC)
        return fail(BODE_E_INVALID_SHAPE, "unknown solver");
    if (arith != BODE_ARITH_EXACT && arith != BODE_ARITH_FAST)
        return fail(BODE_E_INVALID_SHAPE, "unknown arithmetic policy");
    *entry = find_entry(p, solver, arith);
    if (*entry == nullptr)
        return fail(BODE_E_UNSUPPORTED, "no device kernel compiled for this problem/dim/solver");
    return BODE_OK;
}

// RKC stage-coefficient tables (rkc.cuh), one per (device, policy, kappa),
// built on first use by the device generator itself.
int rkc_table_for(const KernelEntry* e, double kappa, cudaStream_t s, const double** out) {
    struct Key {
        int dev, arith;
        double kappa;
        const double* tab;
    };
    static std::mutex m;
    static std::vector<Key> cache;
    int dev = 0;
    BODE_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(m);
    for (const Key& k : cache)
        if (k.dev == dev && k.arith == e->arith && k.kappa == kappa) {
            *out = k.tab;
            return BODE_OK;
        }
    double* tab = nullptr;
    BODE_CUDA(cudaMalloc(&tab, bode::rkc_table_doubles() * sizeof(double)));
    BODE_CUDA((cudaError_t)e->prepare(e->fn, dev, 0));
    BODE_CUDA((cudaError_t)e->build_rkc_table(tab, kappa, s));
    BODE_CUDA(cudaStreamSynchronize(s));
    cache.push_back({dev, e->arith, kappa, tab});
    *out = tab;
    return BODE_OK;
}

// Work counters for persistent launches: a per-device ring, zeroed on the
// launch stream right before use (safe unless > kCounters launches overlap).
constexpr int kCounters = 256;
int claim_counter(cudaStream_t s, unsigned long long** out) {
    static std::mutex m;
    static unsigned long long* pool[64] = {nullptr};
    static int next[64] = {0};
    int dev = 0;
    BODE_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(m);
    if (!pool[dev]) BODE_CUDA(cudaMalloc(&pool[dev], kCounters * sizeof(unsigned long long)));
    unsigned long long* c = pool[dev] + next[dev];
    next[dev] = (next[dev] + 1) % kCounters;
    BODE_CUDA(cudaMemsetAsync(c, 0, sizeof(unsigned long long), s));
    *out = c;
    return BODE_OK;
}

int block_for(const KernelEntry* e) {
    int b = g_block_override.load();
    if (b <= 0) b = e->default_block;
    return b;
}

// One window of a one-system-per-block kernel (wide.cuh): the system's
// kWideVecs state-length vectors in dynamic shared memory when they fit,
// otherwise in a stream-ordered per-block scratch; a grid-stride loop over
// the systems with the grid sized to the resident capacity.
// Threads per block of the one-system-per-block kernels: one per component
// up to 512 (wide_block), but 256 when shared memory then admits two or more
// blocks per SM -- 1.14-1.51x for 1024 < n <= 1750 (r02bt/r02bu); with one
// block per SM, or the vectors in the global scratch, 512 stays faster.
int wide_threads(const void* fn, int n, size_t smem, bool in_smem, int* block) {
    *block = bode::wide_block(n);
    if (in_smem && *block > 256) {
        int per_sm = 0;
        BODE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, smem));
        if (per_sm >= 2) *block = 256;
    }
    return BODE_OK;
}

int launch_wide(const KernelEntry* e, cudaStream_t s, const double* g, double* y, DevStats* st,
                long long num, double t, double tEnd, DevTol tol, int merge) {
    const int n = tol.dim;
    if (n < 2) return fail(BODE_E_INVALID_SHAPE, "run-time-dimension kernel needs dim >= 2");
    int dev = 0, sms = 0;
    BODE_CUDA(cudaGetDevice(&dev));
    BODE_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const size_t vec_bytes = (size_t)bode::kWideVecs * (size_t)n * sizeof(double);
    const bool in_smem = vec_bytes <= (size_t)bode::kWideSmemMax;
    const size_t smem = in_smem ? vec_bytes : 0;
    BODE_CUDA((cudaError_t)e->prepare(e->fn, dev, (int)smem));
    int block = 0;
    if (int rc = wide_threads(e->fn, n, smem, in_smem, &block)) return rc;
    long long grid = 1;
    if (in_smem) {
        int per_sm = 0;
        BODE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, e->fn, block, smem));
        grid = std::min<long long>(num, (long long)std::max(per_sm, 1) * sms);
    } else {
        // global scratch: at most two blocks per SM, within a 4 GiB budget
        const long long budget = std::max<long long>(1, (4LL << 30) / (long long)vec_bytes);
        grid = std::min<long long>(num, std::min<long long>(2LL * sms, budget));
        BODE_CUDA(cudaMallocAsync((void**)&tol.scratch, (size_t)grid * vec_bytes, s));
    }
    cudaError_t le = (cudaError_t)e->launch(e->fn, dim3((unsigned)grid), dim3(block), smem, s, g,
                                            y, st, num, t, tEnd, tol, merge);
    if (tol.scratch != nullptr) BODE_CUDA(cudaFreeAsync(tol.scratch, s));
    BODE_CUDA(le);
    g_launches.fetch_add(1);
    return BODE_OK;
}

// Launch one window over `num` systems resident on the current device.
int launch_window(const KernelEntry* e, cudaStream_t s, const double* g, double* y,
                  DevStats* st, long long num, double t, double tEnd, const DevTol& tol_in,
                  int merge, long long stride = 0) {
    DevTol tol = tol_in;
    tol.stride = stride;
    tol.powtab = bode::device_powtab();
    tol.rkc_coef = nullptr;
    if (e->build_rkc_table != nullptr) {
        int rc = rkc_table_for(e, tol.kappa, s, &tol.rkc_coef);
        if (rc) return rc;
    }
    if (e->wide) return launch_wide(e, s, g, y, st, num, t, tEnd, tol, merge);
    const int block = block_for(e);
    const long long threads = num * e->lanes;
    const long long grid = (threads + block - 1) / block;
    const size_t smem = (size_t)e->smem_per_thread * block;
    // (a traced launch always takes the static schedule)
    const bool persistent =
        e->launch_persistent != nullptr && g_persistent.load() && tol.trace == nullptr;
    const bool budget = tol.max_attempts > 0 || tol.trace != nullptr;  // the instrumented instance
    const void* fn = persistent ? (budget ? e->bpfn : e->pfn) : (budget ? e->bfn : e->fn);
    if (fn == nullptr)
        return fail(BODE_E_UNSUPPORTED, "no kernel instance with the attempt-budget check");
    {
        // current device and the per-device smem attribute, in the runtime that
        // owns the kernel (idempotent and cheap, so done on every launch)
        int dev = 0;
        BODE_CUDA(cudaGetDevice(&dev));
        BODE_CUDA((cudaError_t)e->prepare(fn, dev, (int)smem));
    }
    if (persistent) {
        int dev = 0, sms = 0, per_sm = 0;
        BODE_CUDA(cudaGetDevice(&dev));
        BODE_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        BODE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, block, smem));
        const long long pgrid = std::max<long long>(1, std::min<long long>(grid, (long long)per_sm * sms));
        unsigned long long* counter = nullptr;
        int rc = claim_counter(s, &counter);
        if (rc) return rc;
        BODE_CUDA((cudaError_t)e->launch_persistent(fn, dim3((unsigned)pgrid), dim3(block), smem,
                                                    s, g, y, st, num, t, tEnd, tol, merge,
                                                    counter));
    } else {
        BODE_CUDA((cudaError_t)e->launch(fn, dim3((unsigned)grid), dim3(block), smem, s, g, y, st,
                                         num, t, tEnd, tol, merge));
    }
    g_launches.fetch_add(1);
    BODE_CUDA(cudaGetLastError());
    return BODE_OK;
}

#ifndef BODE_MAX_CHUNKS
#define BODE_MAX_CHUNKS 32
#endif
constexpr int kMaxChunks = BODE_MAX_CHUNKS;  // host-pointer pipeline depth per shard

// Device buffers, streams and events of one shard, leased exclusively for one
// call: concurrent or nested calls (from another host thread, or from a sink)
// never share state, and several shards may live on one device. Leases are
// pooled per device, so a warm call does no cudaMalloc.
struct Lease {
    int device = 0;
    double* y = nullptr;
    double* g = nullptr;
    DevStats* st = nullptr;
    long long* ord = nullptr;  // outer loop: position -> original index after re-packing
    double* ysnap[2] = {nullptr, nullptr};  // outer loop: staged snapshots (caller's order)
    size_t y_cap = 0, g_cap = 0, st_cap = 0, ord_cap = 0, ysnap_cap[2] = {0, 0};
    cudaStream_t streams[3] = {nullptr, nullptr, nullptr};  // H2D, compute, D2H
    cudaEvent_t events[2 * kMaxChunks] = {};                 // per chunk: H2D done, kernel done
    cudaEvent_t snap_ready[2] = {};   // snapshot slot staged in ysnap (compute stream)
    cudaEvent_t snap_copied[2] = {};  // snapshot slot's D2H finished (D2H stream)
};

class LeasePool {
  public:
    // On the caller's current device (== device).
    int acquire(int device, Lease** out) {
        {
            std::lock_guard<std::mutex> lock(m_);
            if (!free_[device].empty()) {
                *out = free_[device].back();
                free_[device].pop_back();
                return BODE_OK;
            }
        }
        Lease* L = new Lease;
        L->device = device;
        for (auto& s : L->streams)
            BODE_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        for (auto& ev : L->events) BODE_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        for (int i = 0; i < 2; ++i) {
            BODE_CUDA(cudaEventCreateWithFlags(&L->snap_ready[i], cudaEventDisableTiming));
            BODE_CUDA(cudaEventCreateWithFlags(&L->snap_copied[i], cudaEventDisableTiming));
        }
        *out = L;
        return BODE_OK;
    }
    void release(Lease* L) {
        // nothing may still be in flight on a lease handed to the next caller
        // (error paths return early)
        cudaSetDevice(L->device);
        for (auto& s : L->streams) cudaStreamSynchronize(s);
        std::lock_guard<std::mutex> lock(m_);
        free_[L->device].push_back(L);
    }

  private:
    std::mutex m_;
    std::vector<Lease*> free_[64];
};

LeasePool& lease_pool() {
    static LeasePool* p = new LeasePool();  // outlives static destructors
    return *p;
}

struct LeaseGuard {
    Lease* L = nullptr;
    LeaseGuard() = default;
    LeaseGuard(const LeaseGuard&) = delete;
    LeaseGuard& operator=(const LeaseGuard&) = delete;
    ~LeaseGuard() {
        if (L) lease_pool().release(L);
    }
};

// Pinned host staging for the outer loop's asynchronous snapshots, kept
// across calls (pinning gigabytes costs far more than a window).
class PinnedCache {
  public:
    int acquire(size_t bytes, void** out) {
        {
            std::lock_guard<std::mutex> lock(m_);
            for (size_t i = 0; i < free_.size(); ++i)
                if (free_[i].second >= bytes) {
                    *out = free_[i].first;
                    sizes_.push_back(free_[i]);
                    free_.erase(free_.begin() + i);
                    return BODE_OK;
                }
        }
        void* p = nullptr;
        BODE_CUDA(cudaHostAlloc(&p, bytes, cudaHostAllocPortable));
        std::lock_guard<std::mutex> lock(m_);
        sizes_.push_back({p, bytes});
        *out = p;
        return BODE_OK;
    }
    void release(void* p) {
        std::lock_guard<std::mutex> lock(m_);
        for (size_t i = 0; i < sizes_.size(); ++i)
            if (sizes_[i].first == p) {
                free_.push_back(sizes_[i]);
                sizes_.erase(sizes_.begin() + i);
                return;
            }
    }

  private:
    std::mutex m_;
    std::vector<std::pair<void*, size_t>> free_, sizes_;  // idle / handed out
};

PinnedCache& pinned_cache() {
    static PinnedCache* p = new PinnedCache();
    return *p;
}

template <class T>
int ensure(T** p, size_t* cap, size_t count) {
    if (count <= *cap) return BODE_OK;
    if (*p) cudaFree(*p);
    *p = nullptr;
    *cap = 0;
    BODE_CUDA(cudaMalloc((void**)p, std::max<size_t>(count, 1) * sizeof(T)));
    *cap = count;
    return BODE_OK;
}

bool host_pinned(const void* ptr) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

// A run of consecutive systems of the caller's batch [begin, begin + count)
// held at column `local` of a shard's device SoA arrays.
struct Range {
    int64_t begin, count, local;
};

struct Shard {
    int device;
    int64_t begin, count;       // first system and the shard's system count
    std::vector<Range> ranges;  // one (contiguous) or several (block-cyclic)
};

// The shard's transfer chunks: each range, the single range of a contiguous
// shard split into `nch` column chunks (the host-pointer pipeline).
std::vector<Range> shard_chunks(const Shard& sh, int nch) {
    if (sh.ranges.size() > 1) return sh.ranges;
    std::vector<Range> v;
    const int64_t cb = sh.count / nch, crem = sh.count % nch;
    int64_t off = 0;
    for (int c = 0; c < nch; ++c) {
        const int64_t nk = cb + (c < crem ? 1 : 0);
        v.push_back({sh.begin + off, nk, off});
        off += nk;
    }
    return v;
}

// Shards (batch_driver.cpp:68-73), the reference's `workers`: shard d runs on
// device (current + d) mod device_count, so a one-process-per-GPU caller
// (torchrun rank r with cuda:r current) and num_gpus = 1 stays on its own GPU,
// and num_gpus above the device count puts several shards on one device (as
// workers above the core count share cores). Results are bitwise independent
// of the shard count and layout (batch_driver.hpp:16-21).
//  * contiguous (default, the reference's partition): shard d holds one range;
//  * block-cyclic (bode_set_shard_layout(1)): blocks of B systems dealt round
//    robin, at most kMaxChunks per shard, so a batch sorted by stiffness (cost)
//    still gives every device the same mix (SURVEY.md 7.4 hard part 7).
std::vector<Shard> make_shards(int64_t num, int gpus) {
    std::vector<Shard> v;
    int cur = 0, n = 1;
    if (cudaGetDevice(&cur) != cudaSuccess) cur = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n < 1) n = 1;
    if (gpus > 1 && g_shard_layout.load() == 1) {
        const int64_t per = (int64_t)gpus * kMaxChunks;
        const int64_t blk = std::max<int64_t>(4096, (num + per - 1) / per);
        for (int d = 0; d < gpus; ++d) v.push_back({(cur + d) % n, 0, 0, {}});
        for (int64_t b = 0, i = 0; b < num; b += blk, ++i) {
            Shard& sh = v[(size_t)(i % gpus)];
            const int64_t len = std::min<int64_t>(blk, num - b);
            if (sh.ranges.empty()) sh.begin = b;
            sh.ranges.push_back({b, len, sh.count});
            sh.count += len;
        }
        v.erase(std::remove_if(v.begin(), v.end(), [](const Shard& s) { return s.count == 0; }),
                v.end());
        return v;
    }
    const int64_t base = num / gpus, rem = num % gpus;
    int64_t b = 0;
    for (int d = 0; d < gpus; ++d) {
        const int64_t len = base + (d < rem ? 1 : 0);
        if (len > 0) v.push_back({(cur + d) % n, b, len, {{b, len, 0}}});
        b += len;
    }
    return v;
}

// Restores the calling thread's current device when a host entry point
// returns (the shard loop switches devices).
struct DeviceRestore {
    int dev = -1;
    DeviceRestore() {
        if (cudaGetDevice(&dev) != cudaSuccess) dev = -1;
    }
    ~DeviceRestore() {
        if (dev >= 0) cudaSetDevice(dev);
    }
};

constexpr int kMaxShards = 4096;

int check_devices(int gpus) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n < 1) {
        cudaGetLastError();
        return fail(BODE_E_NO_DEVICE, "no CUDA device available (there is no CPU fallback)");
    }
    if (gpus < 1) return fail(BODE_E_INVALID_SHAPE, "workers (num_gpus) must be positive");
    if (gpus > kMaxShards) return fail(BODE_E_INVALID_SHAPE, "workers (num_gpus) above 4096");
    if (n > 64) return fail(BODE_E_UNSUPPORTED, "more than 64 visible devices");
    return BODE_OK;
}

// One shard of a host-pointer window, pipelined in chunks over three streams
// with one role each: H2D copies back to back on streams[0], the kernels on
// streams[1] (chunk k waits for its H2D), D2H copies on streams[2] (chunk k
// waits for its kernel). With pinned host memory both PCIe directions then run
// continuously and overlap the compute; the window costs about
// max(H2D, D2H) + one chunk's kernel.
int run_shard_window(const KernelEntry* e, const bode_problem_t* p, const Shard& sh,
                     int64_t num, const double* g, double* y, bode_stats_t* stats, double t,
                     double tEnd, const DevTol& tol) {
    BODE_CUDA(cudaSetDevice(sh.device));
    LeaseGuard guard;
    int rc = lease_pool().acquire(sh.device, &guard.L);
    if (rc) return rc;
    Lease& B = *guard.L;
    const int N = p->dim, P = p->param_dim;
    if ((rc = ensure(&B.y, &B.y_cap, (size_t)sh.count * N))) return rc;
    if (P > 0 && (rc = ensure(&B.g, &B.g_cap, (size_t)sh.count * P))) return rc;
    if (stats && (rc = ensure(&B.st, &B.st_cap, (size_t)sh.count))) return rc;

    // A stiffness parameter known up front (bode_set_presort_param; expDecay's
    // g0 by default): sort the shard by it on the device, integrate, restore
    // the caller's order. Systems are independent, so the results are bitwise
    // unchanged; warps then hold systems of similar cost.
    const int presort_sel = g_presort_param.load();
    const int row = presort_sel == -2 ? stiffness_param_row(p) : presort_sel;
    if (row >= 0 && row < P && g != nullptr && sh.count >= 1024) {
        const long long cnt = sh.count;
        cudaStream_t s = B.streams[1];
        if ((rc = ensure(&B.ord, &B.ord_cap, (size_t)cnt))) return rc;
        for (const Range& rg : sh.ranges) {
            BODE_CUDA(cudaMemcpy2DAsync(B.y + rg.local, cnt * sizeof(double), y + rg.begin,
                                        num * sizeof(double), rg.count * sizeof(double), N,
                                        cudaMemcpyHostToDevice, s));
            BODE_CUDA(cudaMemcpy2DAsync(B.g + rg.local, cnt * sizeof(double), g + rg.begin,
                                        num * sizeof(double), rg.count * sizeof(double), P,
                                        cudaMemcpyHostToDevice, s));
        }
        if ((rc = bode::init_order(B.ord, cnt, s))) return fail(rc, "order init failed");
        if ((rc = bode::repack_by(N, P, cnt, B.y, B.g, nullptr, B.ord, row, s)))
            return fail(rc, "presort failed");
        if ((rc = launch_window(e, s, B.g, B.y, stats ? B.st : nullptr, cnt, t, tEnd, tol, 0)))
            return rc;
        if ((rc = bode::unpack(N, P, cnt, B.y, nullptr, stats ? B.st : nullptr, B.ord, nullptr, s)))
            return fail(rc, "unpack failed");
        for (const Range& rg : sh.ranges) {
            BODE_CUDA(cudaMemcpy2DAsync(y + rg.begin, num * sizeof(double), B.y + rg.local,
                                        cnt * sizeof(double), rg.count * sizeof(double), N,
                                        cudaMemcpyDeviceToHost, s));
            if (stats)
                BODE_CUDA(cudaMemcpyAsync(stats + rg.begin, B.st + rg.local,
                                          rg.count * sizeof(DevStats), cudaMemcpyDeviceToHost, s));
        }
        BODE_CUDA(cudaStreamSynchronize(s));
        return BODE_OK;
    }

    const bool pinned = host_pinned(y);
    const int64_t min_chunk = 1 << 16;
    const int nchunks =
        pinned ? (int)std::min<int64_t>(kMaxChunks, std::max<int64_t>(1, sh.count / min_chunk)) : 1;
    const std::vector<Range> chunks = shard_chunks(sh, nchunks);
    cudaStream_t sh2d = B.streams[0], sk = B.streams[1], sd2h = B.streams[2];
    for (size_t k = 0; k < chunks.size(); ++k) {
        const int64_t nk = chunks[k].count, off = chunks[k].local;
        double* dy = B.y + off * N;
        double* dg = P > 0 ? B.g + off * P : nullptr;
        DevStats* dst = stats ? B.st + off : nullptr;
        const int64_t src = chunks[k].begin;
        cudaEvent_t in_done = B.events[2 * k], k_done = B.events[2 * k + 1];
        BODE_CUDA(cudaMemcpy2DAsync(dy, nk * sizeof(double), y + src, num * sizeof(double),
                                    nk * sizeof(double), N, cudaMemcpyHostToDevice, sh2d));
        if (P > 0)
            BODE_CUDA(cudaMemcpy2DAsync(dg, nk * sizeof(double), g + src, num * sizeof(double),
                                        nk * sizeof(double), P, cudaMemcpyHostToDevice, sh2d));
        BODE_CUDA(cudaEventRecord(in_done, sh2d));
        BODE_CUDA(cudaStreamWaitEvent(sk, in_done, 0));
        rc = launch_window(e, sk, dg, dy, dst, nk, t, tEnd, tol, 0);
        if (rc) return rc;
        BODE_CUDA(cudaEventRecord(k_done, sk));
        BODE_CUDA(cudaStreamWaitEvent(sd2h, k_done, 0));
        BODE_CUDA(cudaMemcpy2DAsync(y + src, num * sizeof(double), dy, nk * sizeof(double),
                                    nk * sizeof(double), N, cudaMemcpyDeviceToHost, sd2h));
        if (stats)
            BODE_CUDA(cudaMemcpyAsync(stats + src, dst, nk * sizeof(DevStats),
                                      cudaMemcpyDeviceToHost, sd2h));
    }
    for (auto& s : B.streams) BODE_CUDA(cudaStreamSynchronize(s));
    return BODE_OK;
}

// Runs f(shard index) for every shard: one host thread per device in use,
// each taking its device's shards in order.
template <class F>
int for_each_shard(const std::vector<Shard>& shards, F&& f) {
    if (shards.size() == 1) return f(size_t(0));
    std::vector<int> devs;
    for (const Shard& s : shards)
        if (std::find(devs.begin(), devs.end(), s.device) == devs.end()) devs.push_back(s.device);
    std::vector<int> rcs(shards.size(), BODE_OK);
    std::vector<std::string> msgs(shards.size());
    auto run_device = [&](int dev) {
        for (size_t i = 0; i < shards.size(); ++i) {
            if (shards[i].device != dev) continue;
            rcs[i] = f(i);
            if (rcs[i]) {
                msgs[i] = g_last_error;
                return;
            }
        }
    };
    if (devs.size() == 1) {
        run_device(devs[0]);
    } else {
        std::vector<std::thread> pool;
        for (int d : devs) pool.emplace_back(run_device, d);
        for (auto& th : pool) th.join();
    }
    for (size_t i = 0; i < shards.size(); ++i)
        if (rcs[i]) return fail(rcs[i], msgs[i]);
    return BODE_OK;
}

// Delivers outer-loop snapshots to the caller's sink from one library thread,
// in window order, while the next windows compute: job k waits for its
// snapshot's D2H events, then calls sink(t_k, staging). done() tells the
// producer when a staging slot may be overwritten.
class SinkWorker {
  public:
    struct Job {
        int64_t k;
        double t;
        const double* y;
        std::vector<std::pair<int, cudaEvent_t>> events;  // (device, D2H done)
    };
    SinkWorker(bode_sink_fn fn, void* user, int64_t num, int dim)
        : fn_(fn), user_(user), num_(num), dim_(dim), th_([this] { loop(); }) {}
    ~SinkWorker() { finish(); }
    void push(Job j) {
        std::lock_guard<std::mutex> lock(m_);
        q_.push_back(std::move(j));
        cv_.notify_all();
    }
    // blocks until the sink for window k has returned
    void wait_done(int64_t k) {
        std::unique_lock<std::mutex> lock(m_);
        cv_.wait(lock, [&] { return done_ >= k || failed_; });
    }
    void finish() {
        {
            std::lock_guard<std::mutex> lock(m_);
            stop_ = true;
            cv_.notify_all();
        }
        if (th_.joinable()) th_.join();
    }
    bool failed() const { return failed_; }

  private:
    void loop() {
        for (;;) {
            Job j;
            {
                std::unique_lock<std::mutex> lock(m_);
                cv_.wait(lock, [&] { return stop_ || !q_.empty(); });
                if (q_.empty()) return;
                j = std::move(q_.front());
                q_.pop_front();
            }
            bool ok = true;
            for (auto& de : j.events) {
                ok = ok && cudaSetDevice(de.first) == cudaSuccess &&
                     cudaEventSynchronize(de.second) == cudaSuccess;
            }
            if (ok) fn_(j.t, j.y, num_, dim_, user_);
            std::lock_guard<std::mutex> lock(m_);
            if (!ok) failed_ = true;
            done_ = j.k;
            cv_.notify_all();
        }
    }
    bode_sink_fn fn_;
    void* user_;
    int64_t num_;
    int dim_;
    std::mutex m_;
    std::condition_variable cv_;
    std::deque<Job> q_;
    int64_t done_ = 0;
    bool stop_ = false;
    bool failed_ = false;
    std::thread th_;
};

}  // namespace

namespace bode {
// Device copy of the host libm pow tables on the current device (uploaded
// once per device), or null when the host pow is not the restated variant.
const double* device_powtab() {
    static std::mutex m;
    static const double* dev[64] = {nullptr};
    static bool tried[64] = {false};
    const auto& img = host_powtab();
    if (img.empty()) return nullptr;
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= 64) return nullptr;
    std::lock_guard<std::mutex> lock(m);
    if (!tried[d]) {
        tried[d] = true;
        double* p = nullptr;
        if (cudaMalloc(&p, img.size() * sizeof(double)) == cudaSuccess &&
            cudaMemcpy(p, img.data(), img.size() * sizeof(double), cudaMemcpyHostToDevice) ==
                cudaSuccess)
            dev[d] = p;
    }
    return dev[d];
}
}  // namespace bode

extern "C" {

int bode_pow_exact_available(void) { return host_powtab().empty() ? 0 : 1; }


const char* bode_version(void) { return "bode 0.1.0 (sm_100a, FP64)"; }
const char* bode_last_error(void) { return g_last_error.c_str(); }

int bode_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

void bode_tol_default(bode_tol_t* t) {  // ode_problem.hpp:33-44
    t->eps = 1.0e-10;
    t->abs_tol = 1.0e-10;
    t->rel_tol = 1.0e-6;
    t->uround = 2.22e-16;
    t->tiny = 1.0e-30;
    t->safety = 0.9;
    t->p1 = 0.1;
    t->errcon = 1.89e-4;
    t->pgrow = -0.2;
    t->pshrnk = -0.25;
    t->h_min_floor = 1.0e-20;
    t->kappa = 2.0 / 13.0;
}

int bode_tol_validate(const bode_tol_t* t) {  // ode_problem.hpp:46-53
    if (t == nullptr) return fail(BODE_E_INVALID_SHAPE, "tolerance settings are NULL");
    if (!(t->eps > 0.0 && t->abs_tol > 0.0 && t->rel_tol > 0.0))
        return fail(BODE_E_INVALID_SHAPE, "ToleranceSettings: eps/absTol/relTol must be positive");
    if (!(t->safety > 0.0 && t->safety < 1.0) || !(t->p1 > 0.0 && t->p1 < 1.0))
        return fail(BODE_E_INVALID_SHAPE, "ToleranceSettings: safety and p1 must lie in (0, 1)");
    if (!(t->uround > 0.0 && t->tiny > 0.0 && t->h_min_floor > 0.0 && t->kappa >= 0.0))
        return fail(BODE_E_INVALID_SHAPE, "ToleranceSettings: bad auxiliary constants");
    return BODE_OK;
}

int bode_problem_init(bode_problem_t* p, int32_t kind, int32_t dim) {
    if (p == nullptr) return fail(BODE_E_INVALID_SHAPE, "problem is NULL");
    p->kind = kind;
    p->reserved = 0;
    switch (kind) {
        case BODE_PROBLEM_PLEIADES: p->dim = 28; p->param_dim = 0; break;
        case BODE_PROBLEM_HEAT:
            if (dim < 2) return fail(BODE_E_INVALID_SHAPE, "heatEquation: need at least two interior points");
            p->dim = dim; p->param_dim = 0; break;
        case BODE_PROBLEM_EXPDECAY: p->dim = 1; p->param_dim = 1; break;
        case BODE_PROBLEM_HARMONIC: p->dim = 2; p->param_dim = 0; break;
        case BODE_PROBLEM_RICCATI:
        case BODE_PROBLEM_SINT: p->dim = 1; p->param_dim = 0; break;
        case BODE_PROBLEM_DIAG:
            if (dim < 1) return fail(BODE_E_INVALID_SHAPE, "dim must be positive");
            p->dim = dim; p->param_dim = dim; break;
        case BODE_PROBLEM_ZERO:
        case BODE_PROBLEM_CONST:
            if (dim < 1) return fail(BODE_E_INVALID_SHAPE, "dim must be positive");
            p->dim = dim; p->param_dim = 0; break;
        default: {  // a registered problem: dim/param_dim from its kernels
            std::lock_guard<std::mutex> lock(registry_mutex());
            const KernelEntry* hit = nullptr;
            for (const KernelEntry& e : registry())
                if (e.kind == kind && (dim <= 0 || e.dim == dim)) {
                    hit = &e;
                    break;
                }
            if (hit == nullptr) return fail(BODE_E_INVALID_SHAPE, "unknown problem kind");
            p->dim = hit->dim;
            p->param_dim = hit->param_dim;
        }
    }
    return BODE_OK;
}

int bode_register_kernels(const void* table, int32_t count, int32_t entry_bytes) {
    if (table == nullptr || count < 1)
        return fail(BODE_E_INVALID_SHAPE, "bode_register_kernels: empty table");
    if (entry_bytes != (int32_t)sizeof(KernelEntry))
        return fail(BODE_E_UNSUPPORTED,
                    "bode_register_kernels: entry layout differs from this libbode "
                    "(rebuild the problem library against this include/)");
    const KernelEntry* es = static_cast<const KernelEntry*>(table);
    for (int32_t i = 0; i < count; ++i) {
        const KernelEntry& e = es[i];
        if (e.fn == nullptr || e.launch == nullptr || e.prepare == nullptr || e.dim < 1 ||
            e.param_dim < 0 || e.lanes < 1 || 32 % e.lanes != 0 || e.dim % e.lanes != 0 ||
            (e.solver != BODE_SOLVER_RKCK && e.solver != BODE_SOLVER_RKC) ||
            (e.arith != BODE_ARITH_EXACT && e.arith != BODE_ARITH_FAST) ||
            (e.solver == BODE_SOLVER_RKC && e.build_rkc_table == nullptr))
            return fail(BODE_E_INVALID_SHAPE, "bode_register_kernels: malformed entry");
    }
    std::lock_guard<std::mutex> lock(registry_mutex());
    for (int32_t i = 0; i < count; ++i) registry().push_back(es[i]);
    return BODE_OK;
}

int bode_registered_count(void) {
    std::lock_guard<std::mutex> lock(registry_mutex());
    return (int)registry().size();
}

int bode_problem_supported(const bode_problem_t* p, int32_t solver, int32_t arith) {
    return (p && find_entry(p, solver, arith)) ? 1 : 0;
}

int bode_stats_summary(const bode_stats_t* st, int64_t num, bode_stats_summary_t* out) {
    if (st == nullptr || out == nullptr || num < 1)
        return fail(BODE_E_INVALID_SHAPE, "stats summary: NULL pointer or num < 1");
    bode_stats_summary_t r{};
    r.num = num;
    r.attempts_argmax = 0;
    double warp_max_sum = 0.0;
    for (int64_t w = 0; w < num; w += 32) {
        int64_t wmax = 0;
        const int64_t wend = std::min<int64_t>(num, w + 32);
        for (int64_t i = w; i < wend; ++i) {
            const int64_t a = st[i].steps_accepted + st[i].steps_rejected;
            r.attempts_total += a;
            if (a > r.attempts_max) {
                r.attempts_max = a;
                r.attempts_argmax = i;
            }
            r.rhs_evals_total += st[i].rhs_evals;
            r.rhs_evals_max = std::max<int64_t>(r.rhs_evals_max, st[i].rhs_evals);
            wmax = std::max<int64_t>(wmax, st[i].rhs_evals);
            r.underflow_count += st[i].underflow ? 1 : 0;
            r.budget_exhausted_count += st[i].budget_exhausted ? 1 : 0;
        }
        warp_max_sum += (double)(wend - w) * (double)wmax;
    }
    r.attempts_mean = (double)r.attempts_total / (double)num;
    r.lockstep_efficiency = warp_max_sum > 0 ? (double)r.rhs_evals_total / warp_max_sum : 1.0;
    *out = r;
    return BODE_OK;
}

int64_t bode_num_windows(double t0, double t_end, double h_outer) {
    const double ratio = (t_end - t0) / h_outer;  // batch_driver.cpp:99-100
    const long n = static_cast<long>(std::ceil(ratio - 1e-9));
    return std::max(1L, n);
}

double bode_window_end(double t0, double t_end, double h_outer, int64_t k) {
    const int64_t n = bode_num_windows(t0, t_end, h_outer);  // batch_driver.cpp:105
    return (k == n) ? t_end : t0 + static_cast<double>(k) * h_outer;
}

int bode_set_block_size(int32_t threads) {
    if (threads != 0 && (threads < 32 || threads > bode::kMaxBlock || threads % 32 != 0))
        return fail(BODE_E_INVALID_SHAPE, "block size must be 0 or a multiple of 32 in [32, 256]");
    g_block_override.store(threads);
    return BODE_OK;
}

int64_t bode_launch_count(void) { return g_launches.load(); }

int bode_set_attempt_budget(int64_t max_attempts) {
    if (max_attempts < 0) return fail(BODE_E_INVALID_SHAPE, "attempt budget must be >= 0");
    g_attempt_budget.store(max_attempts);
    return BODE_OK;
}

// StepObserver for one system (ode_problem.hpp:85-94): the system's window on
// the device with the instrumented kernel instance recording every attempt.
int bode_trace_steps(const bode_problem_t* p, int32_t solver, int32_t arith, double t,
                     double t_end, const double* g, double* y, const bode_tol_t* tol,
                     bode_stats_t* stats, bode_step_record_t* records, int64_t capacity,
                     int64_t* count) {
    const KernelEntry* e = nullptr;
    int rc = validate_call(p, solver, arith, t, t_end, 1, g, y, tol, &e);
    if (rc) return rc;
    if (records == nullptr || capacity < 0 || count == nullptr)
        return fail(BODE_E_INVALID_SHAPE, "trace: records/count NULL or negative capacity");
    if ((rc = check_devices(1))) return rc;
    const int N = p->dim, P = p->param_dim;
    double *dy = nullptr, *dg = nullptr;
    DevStats* dst = nullptr;
    bode::StepRec* drec = nullptr;
    unsigned long long* dn = nullptr;
    auto release = [&]() {
        cudaFree(dy);
        cudaFree(dg);
        cudaFree(dst);
        cudaFree(drec);
        cudaFree(dn);
    };
    cudaError_t ce = cudaMalloc(&dy, N * sizeof(double));
    if (ce == cudaSuccess && P > 0) ce = cudaMalloc(&dg, P * sizeof(double));
    if (ce == cudaSuccess) ce = cudaMalloc(&dst, sizeof(DevStats));
    if (ce == cudaSuccess) ce = cudaMalloc(&drec, std::max<int64_t>(capacity, 1) * sizeof(bode::StepRec));
    if (ce == cudaSuccess) ce = cudaMalloc(&dn, sizeof(unsigned long long));
    if (ce == cudaSuccess) ce = cudaMemcpy(dy, y, N * sizeof(double), cudaMemcpyHostToDevice);
    if (ce == cudaSuccess && P > 0) ce = cudaMemcpy(dg, g, P * sizeof(double), cudaMemcpyHostToDevice);
    if (ce == cudaSuccess) ce = cudaMemset(dn, 0, sizeof(unsigned long long));
    if (ce != cudaSuccess) {
        release();
        return fail(BODE_E_CUDA, std::string("trace setup: ") + cudaGetErrorString(ce));
    }
    DevTol dt = to_dev(tol, N);
    dt.trace = drec;
    dt.trace_cap = capacity;
    dt.trace_count = dn;
    rc = launch_window(e, 0, dg, dy, dst, 1, t, t_end, dt, 0);
    unsigned long long n = 0;
    if (rc == BODE_OK) {
        ce = cudaMemcpy(&n, dn, sizeof(n), cudaMemcpyDeviceToHost);
        const int64_t kept = std::min<int64_t>((int64_t)n, capacity);
        if (ce == cudaSuccess && kept > 0)
            ce = cudaMemcpy(records, drec, kept * sizeof(bode::StepRec), cudaMemcpyDeviceToHost);
        if (ce == cudaSuccess) ce = cudaMemcpy(y, dy, N * sizeof(double), cudaMemcpyDeviceToHost);
        if (ce == cudaSuccess && stats) ce = cudaMemcpy(stats, dst, sizeof(DevStats), cudaMemcpyDeviceToHost);
        if (ce != cudaSuccess) rc = fail(BODE_E_CUDA, std::string("trace: ") + cudaGetErrorString(ce));
    }
    release();
    *count = (int64_t)n;
    return rc;
}

int bode_use_device(int32_t device) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n < 1) {
        cudaGetLastError();
        return fail(BODE_E_NO_DEVICE, "no CUDA device available (there is no CPU fallback)");
    }
    if (device < 0 || device >= n) return fail(BODE_E_INVALID_SHAPE, "device index out of range");
    BODE_CUDA(cudaSetDevice(device));
    return BODE_OK;
}

int bode_set_shard_layout(int32_t layout) {
    if (layout != 0 && layout != 1) return fail(BODE_E_INVALID_SHAPE, "shard layout must be 0 or 1");
    g_shard_layout.store(layout);
    return BODE_OK;
}

int bode_set_wide(int32_t mode) {
    g_force_wide.store(mode ? 1 : 0);
    return BODE_OK;
}

int bode_set_persistent(int32_t enable) {
    g_persistent.store(enable ? 1 : 0);
    return BODE_OK;
}

int bode_set_repack_threshold(double threshold) {
    if (!(threshold >= 0.0 && threshold <= 1.0))
        return fail(BODE_E_INVALID_SHAPE, "repack threshold must lie in [0, 1]");
    g_repack_threshold.store(threshold);
    return BODE_OK;
}

int bode_set_presort_param(int32_t param_row) {
    if (param_row < -2) return fail(BODE_E_INVALID_SHAPE, "presort parameter row must be >= -2");
    g_presort_param.store(param_row);
    return BODE_OK;
}

int bode_order_init(int64_t* order_dev, int64_t num, void* stream) {
    if (order_dev == nullptr || num < 1) return fail(BODE_E_INVALID_SHAPE, "order: bad arguments");
    int rc = check_devices(1);
    if (rc) return rc;
    rc = bode::init_order(reinterpret_cast<long long*>(order_dev), num,
                          static_cast<cudaStream_t>(stream));
    return rc ? fail(rc, "order init failed") : BODE_OK;
}

int bode_repack_by_cost(const bode_problem_t* p, int64_t num, double* y_dev, double* g_dev,
                        bode_stats_t* stats_dev, int64_t* order_dev, void* stream) {
    int rc = check_problem_shape(p);
    if (rc) return rc;
    if (num < 1 || y_dev == nullptr || stats_dev == nullptr || order_dev == nullptr ||
        (p->param_dim > 0 && g_dev == nullptr))
        return fail(BODE_E_INVALID_SHAPE, "repack: bad arguments");
    if ((rc = check_devices(1))) return rc;
    rc = bode::repack_by_cost(p->dim, p->param_dim, num, y_dev, g_dev,
                              reinterpret_cast<DevStats*>(stats_dev),
                              reinterpret_cast<long long*>(order_dev),
                              static_cast<cudaStream_t>(stream));
    return rc ? fail(rc, "repack failed") : BODE_OK;
}

int bode_repack_by_param(const bode_problem_t* p, int64_t num, double* y_dev, double* g_dev,
                         bode_stats_t* stats_dev, int64_t* order_dev, int32_t param_row,
                         void* stream) {
    int rc = check_problem_shape(p);
    if (rc) return rc;
    if (num < 1 || y_dev == nullptr || g_dev == nullptr || order_dev == nullptr ||
        param_row < 0 || param_row >= p->param_dim)
        return fail(BODE_E_INVALID_SHAPE, "repack_by_param: bad arguments");
    if ((rc = check_devices(1))) return rc;
    rc = bode::repack_by(p->dim, p->param_dim, num, y_dev, g_dev,
                         reinterpret_cast<DevStats*>(stats_dev),
                         reinterpret_cast<long long*>(order_dev), param_row,
                         static_cast<cudaStream_t>(stream));
    return rc ? fail(rc, "repack failed") : BODE_OK;
}

int bode_unpack(const bode_problem_t* p, int64_t num, double* y_dev, double* g_dev,
                bode_stats_t* stats_dev, int64_t* order_dev, void* stream) {
    int rc = check_problem_shape(p);
    if (rc) return rc;
    if (num < 1 || y_dev == nullptr || order_dev == nullptr)
        return fail(BODE_E_INVALID_SHAPE, "unpack: bad arguments");
    if ((rc = check_devices(1))) return rc;
    rc = bode::unpack(p->dim, p->param_dim, num, y_dev, g_dev,
                      reinterpret_cast<DevStats*>(stats_dev),
                      reinterpret_cast<long long*>(order_dev), nullptr,
                      static_cast<cudaStream_t>(stream));
    return rc ? fail(rc, "unpack failed") : BODE_OK;
}

int bode_lockstep_efficiency(const bode_problem_t* p, int32_t solver, int32_t arith, int64_t num,
                             const bode_stats_t* stats_dev, double* efficiency, void* stream) {
    int rc = check_problem_shape(p);
    if (rc) return rc;
    if (num < 1 || stats_dev == nullptr || efficiency == nullptr)
        return fail(BODE_E_INVALID_SHAPE, "lockstep efficiency: bad arguments");
    const KernelEntry* e = find_entry(p, solver, arith);
    if (e == nullptr) return fail(BODE_E_UNSUPPORTED, "no device kernel for this problem");
    if ((rc = check_devices(1))) return rc;
    rc = bode::lockstep_efficiency(reinterpret_cast<const DevStats*>(stats_dev), num,
                                   32 / e->lanes, efficiency, static_cast<cudaStream_t>(stream));
    return rc ? fail(rc, "lockstep efficiency failed") : BODE_OK;
}

// One window of a device-resident batch sorted by a stiffness parameter: the
// caller's arrays are copied into a stream-ordered scratch, sorted there
// (bode_repack_by_param), integrated, unpacked and copied back, all on the
// caller's stream (asynchronous; the caller's g is only read). Bitwise the
// unsorted window.
int presorted_device_window(const KernelEntry* e, const bode_problem_t* p, cudaStream_t s,
                            const double* g_dev, double* y_dev, DevStats* st_dev, int merge,
                            int64_t num, double t, double t_end, const DevTol& dt, int row) {
    const int N = p->dim, P = p->param_dim;
    const size_t n = (size_t)num;
    auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
    const size_t by = al(n * N * sizeof(double)), bg = al(n * P * sizeof(double)),
                 bs = al(n * sizeof(DevStats)), bo = al(n * sizeof(long long));
    char* base = nullptr;
    BODE_CUDA(cudaMallocAsync((void**)&base, by + bg + bs + bo, s));
    double* wy = reinterpret_cast<double*>(base);
    double* wg = reinterpret_cast<double*>(base + by);
    DevStats* wst = st_dev ? reinterpret_cast<DevStats*>(base + by + bg) : nullptr;
    long long* word = reinterpret_cast<long long*>(base + by + bg + bs);
    int rc = BODE_OK;
    cudaError_t ce = cudaMemcpyAsync(wy, y_dev, n * N * sizeof(double), cudaMemcpyDeviceToDevice, s);
    if (ce == cudaSuccess)
        ce = cudaMemcpyAsync(wg, g_dev, n * P * sizeof(double), cudaMemcpyDeviceToDevice, s);
    if (ce == cudaSuccess && wst && merge)
        ce = cudaMemcpyAsync(wst, st_dev, n * sizeof(DevStats), cudaMemcpyDeviceToDevice, s);
    if (ce != cudaSuccess) rc = fail(BODE_E_CUDA, std::string("presort copy: ") + cudaGetErrorString(ce));
    if (!rc && (rc = bode::init_order(word, num, s))) rc = fail(rc, "order init failed");
    if (!rc && (rc = bode::repack_by(N, P, num, wy, wg, (wst && merge) ? wst : nullptr, word, row, s)))
        rc = fail(rc, "presort failed");
    if (!rc) rc = launch_window(e, s, wg, wy, wst, num, t, t_end, dt, merge);
    if (!rc && (rc = bode::unpack(N, P, num, wy, nullptr, wst, word, nullptr, s)))
        rc = fail(rc, "unpack failed");
    if (!rc) {
        ce = cudaMemcpyAsync(y_dev, wy, n * N * sizeof(double), cudaMemcpyDeviceToDevice, s);
        if (ce == cudaSuccess && wst)
            ce = cudaMemcpyAsync(st_dev, wst, n * sizeof(DevStats), cudaMemcpyDeviceToDevice, s);
        if (ce != cudaSuccess) rc = fail(BODE_E_CUDA, std::string("presort copy back: ") + cudaGetErrorString(ce));
    }
    cudaFreeAsync(base, s);
    return rc;
}

int bode_int_driver_device(const bode_problem_t* p, int32_t solver, int32_t arith, double t,
                           double t_end, int64_t num, const double* g_dev, double* y_dev,
                           const bode_tol_t* tol, bode_stats_t* stats_dev, int32_t merge_stats,
                           void* stream) {
    const KernelEntry* e = nullptr;
    int rc = validate_call(p, solver, arith, t, t_end, num, g_dev, y_dev, tol, &e);
    if (rc) return rc;
    if ((rc = check_devices(1))) return rc;
    // a stiffness parameter known up front (bode_set_presort_param; expDecay's g0
    // by default): sort by it around the window
    const int presort_sel = g_presort_param.load();
    const int row = presort_sel == -2 ? stiffness_param_row(p) : presort_sel;
    if (row >= 0 && row < p->param_dim && g_dev != nullptr && num >= 1024)
        return presorted_device_window(e, p, (cudaStream_t)stream, g_dev, y_dev,
                                       (DevStats*)stats_dev, merge_stats ? 1 : 0, num, t, t_end,
                                       to_dev(tol, p->dim), row);
    return launch_window(e, (cudaStream_t)stream, g_dev, y_dev, (DevStats*)stats_dev, num, t,
                         t_end, to_dev(tol, p->dim), merge_stats ? 1 : 0);
}

int bode_int_driver(const bode_problem_t* p, int32_t solver, int32_t arith, double t,
                    double t_end, int64_t num, const double* g, double* y, const bode_tol_t* tol,
                    bode_stats_t* stats, int32_t num_gpus) {
    const KernelEntry* e = nullptr;
    int rc = validate_call(p, solver, arith, t, t_end, num, g, y, tol, &e);
    if (rc) return rc;
    if ((rc = check_devices(num_gpus))) return rc;
    const DevTol dt = to_dev(tol, p->dim);
    DeviceRestore restore;
    const auto shards = make_shards(num, num_gpus);
    return for_each_shard(shards, [&](size_t i) {
        return run_shard_window(e, p, shards[i], num, g, y, stats, t, t_end, dt);
    });
}

int bode_outer_loop(const bode_problem_t* p, int32_t solver, int32_t arith, double t0,
                    double t_end, double h_outer, int64_t num, const double* g, double* y,
                    const bode_tol_t* tol, bode_stats_t* stats, int32_t num_gpus,
                    bode_sink_fn sink, void* user, int32_t* outer_steps) {
    if (!(t_end > t0)) return fail(BODE_E_INVALID_INTERVAL, "outerLoop: tEnd must exceed t0");
    if (!(h_outer > 0.0)) return fail(BODE_E_INVALID_INTERVAL, "outerLoop: hOuter must be positive");
    const KernelEntry* e = nullptr;
    int rc = validate_call(p, solver, arith, t0, t_end, num, g, y, tol, &e);
    if (rc) return rc;
    if ((rc = check_devices(num_gpus))) return rc;
    const DevTol dt = to_dev(tol, p->dim);
    DeviceRestore restore;
    const auto shards = make_shards(num, num_gpus);
    const int N = p->dim, P = p->param_dim;
    const int64_t nwin = bode_num_windows(t0, t_end, h_outer);

    // One lease per shard for the whole call; y stays resident across windows
    // (SURVEY 8f row 1). With pinned host memory the first window's upload and
    // the last window's download are pipelined with its kernels in column
    // chunks of the shard's SoA arrays (launches with a row stride): H2D on
    // streams[0], kernels on streams[1], D2H on streams[2], per-chunk events.
    std::vector<LeaseGuard> leases(shards.size());
    rc = for_each_shard(shards, [&](size_t i) {
        const Shard& sh = shards[i];
        BODE_CUDA(cudaSetDevice(sh.device));
        int r = lease_pool().acquire(sh.device, &leases[i].L);
        if (r) return r;
        Lease& B = *leases[i].L;
        if ((r = ensure(&B.y, &B.y_cap, (size_t)sh.count * N))) return r;
        if (P > 0 && (r = ensure(&B.g, &B.g_cap, (size_t)sh.count * P))) return r;
        if ((r = ensure(&B.st, &B.st_cap, (size_t)sh.count))) return r;
        if ((r = ensure(&B.ord, &B.ord_cap, (size_t)sh.count))) return r;
        if (sink != nullptr && nwin > 1)
            for (int slot = 0; slot < 2; ++slot)
                if ((r = ensure(&B.ysnap[slot], &B.ysnap_cap[slot], (size_t)sh.count * N)))
                    return r;
        if ((r = bode::init_order(B.ord, sh.count, B.streams[1]))) return fail(r, "order init failed");
        return BODE_OK;
    });
    if (rc) return rc;

    // Snapshots of windows 1..n-1 (batch_driver.cpp:104-114) are asynchronous:
    // after window k's kernel the state is staged on the device (ysnap[k%2],
    // in the caller's order), its D2H into pinned staging[k%2] runs on the D2H
    // stream while window k+1 computes, and a library thread hands it to the
    // sink once the copy lands. A slot is reused at window k+2, after the sink
    // for window k returned. The final window's state goes to y as before.
    void* staging[2] = {nullptr, nullptr};
    struct StagingGuard {
        void** s;
        ~StagingGuard() {
            for (int i = 0; i < 2; ++i)
                if (s[i]) pinned_cache().release(s[i]);
        }
    } staging_guard{staging};
    std::unique_ptr<SinkWorker> worker;
    if (sink != nullptr && nwin > 1) {
        for (int i = 0; i < 2; ++i)
            if ((rc = pinned_cache().acquire((size_t)num * N * sizeof(double), &staging[i])))
                return rc;
        worker.reset(new SinkWorker(sink, user, num, N));
    }

    double t = t0;
    const bool pinned = host_pinned(y);
    std::vector<char> repacked(shards.size(), 0);
    const double threshold = g_repack_threshold.load();
    const int presort_sel = g_presort_param.load();
    const int presort_row = presort_sel == -2 ? stiffness_param_row(p) : presort_sel;
    for (int64_t k = 1; k <= nwin; ++k) {
        const double tk = (k == nwin) ? t_end : t0 + static_cast<double>(k) * h_outer;
        const bool last = k == nwin;
        const bool async_snap = worker != nullptr && !last;
        const int slot = (int)(k % 2);
        if (async_snap && k > 2) {
            worker->wait_done(k - 2);  // staging[slot] is free again
            if (worker->failed()) return fail(BODE_E_CUDA, "snapshot copy failed");
        }
        double* host_snap = async_snap ? static_cast<double*>(staging[slot]) : nullptr;
        rc = for_each_shard(shards, [&](size_t si) {
            const Shard& sh = shards[si];
            BODE_CUDA(cudaSetDevice(sh.device));
            Lease& B = *leases[si].L;
            cudaStream_t sh2d = B.streams[0], s = B.streams[1], sd2h = B.streams[2];
            const long long cnt = sh.count;
            const bool first = k == 1;
            const int nch = pinned ? (int)std::min<int64_t>(kMaxChunks, std::max<int64_t>(1, cnt / (1 << 16)))
                                   : 1;
            // sort by a stiffness parameter before the first window: needs the
            // whole shard uploaded first, so that upload is not chunked
            const bool presort = first && presort_row >= 0 && presort_row < P && cnt >= 1024;
            // the final download can ride along per chunk unless the batch is re-packed
            const bool chunked_out = last && !repacked[si] && !presort && nch > 1;
            const bool chunked = (first && !presort && nch > 1) || chunked_out;
            int r = BODE_OK;
            if (first && !chunked) {  // upload in one piece (per range)
                for (const Range& rg : sh.ranges) {
                    BODE_CUDA(cudaMemcpy2DAsync(B.y + rg.local, cnt * sizeof(double),
                                                y + rg.begin, num * sizeof(double),
                                                rg.count * sizeof(double), N,
                                                cudaMemcpyHostToDevice, s));
                    if (P > 0)
                        BODE_CUDA(cudaMemcpy2DAsync(B.g + rg.local, cnt * sizeof(double),
                                                    g + rg.begin, num * sizeof(double),
                                                    rg.count * sizeof(double), P,
                                                    cudaMemcpyHostToDevice, s));
                }
            }
            if (presort) {
                // before window 1 the stats hold nothing yet (window 1 overwrites them)
                if ((r = bode::repack_by(N, P, cnt, B.y, B.g, nullptr, B.ord, presort_row, s)))
                    return fail(r, "presort failed");
                repacked[si] = 1;
            }
            if (chunked) {
                const std::vector<Range> chunks = shard_chunks(sh, nch);
                for (size_t c = 0; c < chunks.size(); ++c) {
                    const long long nk = chunks[c].count, off = chunks[c].local;
                    const int64_t src = chunks[c].begin;
                    cudaEvent_t in_done = B.events[2 * c], k_done = B.events[2 * c + 1];
                    if (first) {
                        BODE_CUDA(cudaMemcpy2DAsync(B.y + off, cnt * sizeof(double),
                                                    y + src, num * sizeof(double),
                                                    nk * sizeof(double), N,
                                                    cudaMemcpyHostToDevice, sh2d));
                        if (P > 0)
                            BODE_CUDA(cudaMemcpy2DAsync(B.g + off, cnt * sizeof(double),
                                                        g + src, num * sizeof(double),
                                                        nk * sizeof(double), P,
                                                        cudaMemcpyHostToDevice, sh2d));
                        BODE_CUDA(cudaEventRecord(in_done, sh2d));
                        BODE_CUDA(cudaStreamWaitEvent(s, in_done, 0));
                    }
                    r = launch_window(e, s, P > 0 ? B.g + off : nullptr, B.y + off, B.st + off,
                                      nk, t, tk, dt, first ? 0 : 1, cnt);
                    if (r) return r;
                    if (chunked_out) {
                        BODE_CUDA(cudaEventRecord(k_done, s));
                        BODE_CUDA(cudaStreamWaitEvent(sd2h, k_done, 0));
                        BODE_CUDA(cudaMemcpy2DAsync(y + src, num * sizeof(double),
                                                    B.y + off, cnt * sizeof(double),
                                                    nk * sizeof(double), N,
                                                    cudaMemcpyDeviceToHost, sd2h));
                        if (stats)
                            BODE_CUDA(cudaMemcpyAsync(stats + src, B.st + off,
                                                      nk * sizeof(DevStats),
                                                      cudaMemcpyDeviceToHost, sd2h));
                    }
                }
            } else {
                r = launch_window(e, s, P > 0 ? B.g : nullptr, B.y, B.st, cnt, t, tk, dt,
                                  first ? 0 : 1);
                if (r) return r;
            }
            if (last && repacked[si]) {  // back to the caller's order, in place
                if ((r = bode::unpack(N, P, cnt, B.y, P > 0 ? B.g : nullptr, B.st, B.ord,
                                      nullptr, s)))
                    return fail(r, "unpack failed");
                repacked[si] = 0;
            }
            if (async_snap) {
                // stage the snapshot (caller's order) once slot's previous D2H is done
                double* ys = B.ysnap[slot];
                BODE_CUDA(cudaStreamWaitEvent(s, B.snap_copied[slot], 0));
                if (repacked[si]) {
                    if ((r = bode::unpack(N, P, cnt, B.y, nullptr, nullptr, B.ord, ys, s)))
                        return fail(r, "snapshot unpack failed");
                } else {
                    BODE_CUDA(cudaMemcpyAsync(ys, B.y, (size_t)cnt * N * sizeof(double),
                                              cudaMemcpyDeviceToDevice, s));
                }
                BODE_CUDA(cudaEventRecord(B.snap_ready[slot], s));
                BODE_CUDA(cudaStreamWaitEvent(sd2h, B.snap_ready[slot], 0));
                for (const Range& rg : sh.ranges)
                    BODE_CUDA(cudaMemcpy2DAsync(host_snap + rg.begin, num * sizeof(double),
                                                ys + rg.local, cnt * sizeof(double),
                                                rg.count * sizeof(double), N,
                                                cudaMemcpyDeviceToHost, sd2h));
                BODE_CUDA(cudaEventRecord(B.snap_copied[slot], sd2h));
            }
            if (last && !chunked_out) {
                for (const Range& rg : sh.ranges) {
                    BODE_CUDA(cudaMemcpy2DAsync(y + rg.begin, num * sizeof(double),
                                                B.y + rg.local, cnt * sizeof(double),
                                                rg.count * sizeof(double), N,
                                                cudaMemcpyDeviceToHost, s));
                    if (stats)
                        BODE_CUDA(cudaMemcpyAsync(stats + rg.begin, B.st + rg.local,
                                                  rg.count * sizeof(DevStats),
                                                  cudaMemcpyDeviceToHost, s));
                }
            }
            if (!last && threshold > 0.0 && cnt >= 1024) {
                // re-pack when the cost history says warps idle behind stragglers
                double eff = 1.0;
                if ((r = bode::lockstep_efficiency(B.st, cnt, 32 / e->lanes, &eff, s)))
                    return fail(r, "lockstep efficiency failed");
                if (eff < threshold) {
                    if ((r = bode::repack_by_cost(N, P, cnt, B.y, P > 0 ? B.g : nullptr, B.st,
                                                  B.ord, s)))
                        return fail(r, "repack failed");
                    repacked[si] = 1;
                }
            }
            if (last)
                for (auto& st : B.streams) BODE_CUDA(cudaStreamSynchronize(st));
            return BODE_OK;
        });
        if (rc) return rc;
        if (async_snap) {
            SinkWorker::Job j{k, tk, host_snap, {}};
            for (size_t si = 0; si < shards.size(); ++si)
                j.events.push_back({shards[si].device, leases[si].L->snap_copied[slot]});
            worker->push(std::move(j));
        }
        t = tk;
    }
    if (worker) {
        worker->wait_done(nwin - 1);
        const bool bad = worker->failed();
        worker->finish();
        if (bad) return fail(BODE_E_CUDA, "snapshot copy failed");
    }
    if (sink) sink(t_end, y, num, N, user);  // the final state, in y (batch_driver.cpp:112)
    if (outer_steps) *outer_steps = (int32_t)nwin;
    return BODE_OK;
}

// Fixed-step harnesses (rkck.cpp:168-181, rkc.cpp:290-306), host pointers.
// integrateFixed on a one-system-per-block kernel: vectors in shared memory
// when they fit, else a per-block global scratch (as launch_wide).
int fixed_wide(const KernelEntry* e, const bode_problem_t* p, double t0, double t_end,
               int64_t num_steps, int32_t stages, double kappa, int64_t num, const double* g,
               double* y) {
    const int n = p->dim;
    int dev = 0, sms = 0;
    BODE_CUDA(cudaGetDevice(&dev));
    BODE_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const size_t vec_bytes = (size_t)bode::kWideVecs * (size_t)n * sizeof(double);
    const bool in_smem = vec_bytes <= (size_t)bode::kWideSmemMax;
    const size_t smem = in_smem ? vec_bytes : 0;
    BODE_CUDA((cudaError_t)e->prepare(e->ffn, dev, (int)smem));
    int block = 0;
    if (int rc = wide_threads(e->ffn, n, smem, in_smem, &block)) return rc;
    long long grid = 1;
    if (in_smem) {
        int per_sm = 0;
        BODE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, e->ffn, block, smem));
        grid = std::min<long long>(num, (long long)std::max(per_sm, 1) * sms);
    } else {
        const long long budget = std::max<long long>(1, (4LL << 30) / (long long)vec_bytes);
        grid = std::min<long long>(num, std::min<long long>(2LL * sms, budget));
    }
    double *dy = nullptr, *scratch = nullptr;
    BODE_CUDA(cudaMalloc(&dy, (size_t)num * n * sizeof(double)));
    if (!in_smem) BODE_CUDA(cudaMalloc(&scratch, (size_t)grid * vec_bytes));
    BODE_CUDA(cudaMemcpy(dy, y, (size_t)num * n * sizeof(double), cudaMemcpyHostToDevice));
    cudaError_t le = (cudaError_t)e->launch_fixed_wide(e->ffn, dim3((unsigned)grid), dim3(block),
                                                       smem, 0, nullptr, dy, num, t0, t_end, num_steps,
                                                       stages, kappa, n, scratch);
    g_launches.fetch_add(1);
    if (le == cudaSuccess) le = cudaMemcpy(y, dy, (size_t)num * n * sizeof(double), cudaMemcpyDeviceToHost);
    cudaFree(dy);
    if (scratch) cudaFree(scratch);
    BODE_CUDA(le);
    return BODE_OK;
}

int bode_integrate_fixed(const bode_problem_t* p, int32_t solver, int32_t arith, double t0,
                         double t_end, int64_t num_steps, int32_t stages, double kappa,
                         int64_t num, const double* g, double* y) {
    if (!(t_end > t0) || num_steps < 1)
        return fail(BODE_E_INVALID_INTERVAL, "integrateFixed: bad interval or step count");
    if (solver == BODE_SOLVER_RKC && stages < 2)
        return fail(BODE_E_INVALID_STAGE_COUNT, "rkc::coefficients: need at least two stages");
    bode_tol_t tol;
    bode_tol_default(&tol);
    const KernelEntry* e = nullptr;
    int rc = validate_call(p, solver, arith, t0, t_end, num, g, y, &tol, &e);
    if (rc) return rc;
    if (e->cap > 0 || e->wide) {  // run-time dimension: the one-system-per-block harness
        const KernelEntry* w = e->wide ? e : find_wide(p, solver, arith);
        if (w == nullptr) return fail(BODE_E_UNSUPPORTED, "no fixed-step kernel for this problem");
        if ((rc = check_devices(1))) return rc;
        return fixed_wide(w, p, t0, t_end, num_steps, stages, kappa, num, g, y);
    }
    if (e->launch_fixed == nullptr) {  // e.g. the lane-pair Pleiades kernel: try the others
        int n = 0;
        const KernelEntry* tab = bode::kernel_table(&n);
        for (int i = 0; i < n; ++i)
            if (tab[i].kind == p->kind && tab[i].dim == p->dim && tab[i].param_dim == p->param_dim &&
                tab[i].solver == solver && tab[i].arith == arith && tab[i].launch_fixed) {
                e = &tab[i];
                break;
            }
    }
    if (e->launch_fixed == nullptr)
        return fail(BODE_E_UNSUPPORTED, "no fixed-step kernel for this problem/solver");
    if ((rc = check_devices(1))) return rc;
    int dev = 0;  // the calling thread's current device
    BODE_CUDA(cudaGetDevice(&dev));
    const int N = p->dim, P = p->param_dim;
    double *dy = nullptr, *dg = nullptr;
    BODE_CUDA(cudaMalloc(&dy, (size_t)num * N * sizeof(double)));
    if (P > 0) BODE_CUDA(cudaMalloc(&dg, (size_t)num * P * sizeof(double)));
    BODE_CUDA(cudaMemcpy(dy, y, (size_t)num * N * sizeof(double), cudaMemcpyHostToDevice));
    if (P > 0) BODE_CUDA(cudaMemcpy(dg, g, (size_t)num * P * sizeof(double), cudaMemcpyHostToDevice));
    const int block = 128;
    const long long grid = (num * e->lanes + block - 1) / block;
    BODE_CUDA((cudaError_t)e->prepare(e->ffn, dev, 0));
    BODE_CUDA((cudaError_t)e->launch_fixed(e->ffn, dim3((unsigned)grid), dim3(block), 0, dg, dy,
                                           num, t0, t_end, num_steps, stages, kappa));
    g_launches.fetch_add(1);
    BODE_CUDA(cudaMemcpy(y, dy, (size_t)num * N * sizeof(double), cudaMemcpyDeviceToHost));
    cudaFree(dy);
    if (dg) cudaFree(dg);
    return BODE_OK;
}

// ---- synthetic inputs (problems.cpp:158-191) ----
uint64_t bode_splitmix64_at(uint64_t seed, uint64_t k) {
    uint64_t z = seed + (k + 1) * 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

double bode_unit_symmetric_at(uint64_t seed, uint64_t k) {
    const double u01 = static_cast<double>(bode_splitmix64_at(seed, k) >> 11) * 0x1.0p-53;
    return 2.0 * u01 - 1.0;
}

int bode_perturb_initial_conditions(const double* base, int32_t dim, double magnitude,
                                    uint64_t seed, int64_t count, double* out) {
    return bode_perturb_initial_conditions_range(base, dim, magnitude, seed, 0, count, out);
}

// Systems [first, first + count) of the reference's perturbation stream
// (counter k = i*dim + j, problems.cpp:175-187) as a local SoA array of
// `count` columns: a rank builds exactly its own shard of a global batch.
int bode_perturb_initial_conditions_range(const double* base, int32_t dim, double magnitude,
                                          uint64_t seed, int64_t first, int64_t count,
                                          double* out) {
    if (count < 1) return fail(BODE_E_INVALID_SHAPE, "perturbInitialConditions: count must be positive");
    if (first < 0) return fail(BODE_E_INVALID_SHAPE, "perturbInitialConditions: negative first system");
    if (dim < 1 || base == nullptr) return fail(BODE_E_INVALID_SHAPE, "perturbInitialConditions: empty base state");
    if (!(magnitude >= 0.0 && magnitude <= 0.1))
        return fail(BODE_E_INVALID_SHAPE, "perturbInitialConditions: magnitude outside [0, 0.1]");
    const unsigned hw = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
    const int64_t workers = std::min<int64_t>(hw, std::max<int64_t>(1, count / 65536));
    auto body = [&](int64_t lo, int64_t hi) {
        for (int j = 0; j < dim; ++j)
            for (int64_t i = lo; i < hi; ++i) {
                const uint64_t k = static_cast<uint64_t>(first + i) * static_cast<uint64_t>(dim) + j;
                const double u = bode_unit_symmetric_at(seed, k);
                out[i + count * j] = base[j] * (1.0 + u * magnitude);
            }
    };
    if (workers <= 1) {
        body(0, count);
    } else {
        std::vector<std::thread> pool;
        for (int64_t w = 0; w < workers; ++w)
            pool.emplace_back(body, count * w / workers, count * (w + 1) / workers);
        for (auto& th : pool) th.join();
    }
    return BODE_OK;
}

void bode_pleiades_ic(double out[28]) { std::memcpy(out, kPleiadesIC, sizeof(kPleiadesIC)); }

void bode_heat_initial_condition(int32_t n, double* u) {  // problems.cpp:124-132
    const double dx = 1.0 / (n + 1);
    for (int i = 0; i < n; ++i) {
        const double x = (i + 1) * dx;
        u[i] = 4.0 * x * (1.0 - x);
    }
}

}  // extern "C"
