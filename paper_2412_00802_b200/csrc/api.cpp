// Diagnostics of the C ABI: thread-local last error, version, launch counter,
// CUDA-event kernel timing (used by bench.py for the roofline "achieved").
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "internal.h"

namespace hedl {

static thread_local std::string g_last_error;

bool timing_enabled() {
    static const bool on = [] { const char *e = std::getenv("HEDL_TIMING"); return e && *e && *e != '0'; }();
    return on;
}
double now_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
void timing_note(const char *what, double ms) {
    if (timing_enabled()) std::fprintf(stderr, "[hedl timing] %-28s %9.3f ms\n", what, ms);
}

void set_error(const std::string &msg) { g_last_error = msg; }

hedl_status fail(hedl_status st, const std::string &msg) {
    g_last_error = msg;
    return st;
}

hedl_status cuda_fail(const hedl_kb *kb, cudaError_t e, const char *where) {
    if (kb) const_cast<hedl_kb *>(kb)->poisoned = true;
    g_last_error = std::string(where) + ": " + cudaGetErrorString(e);
    cudaGetLastError();
    return HEDL_ERR_CUDA;
}

void *pool_take(const hedl_kb *kb, int role, size_t need, size_t *got) {
    std::lock_guard<std::mutex> lk(kb->pool_mu);
    auto &v = kb->pool[role];
    int best = -1;
    for (int i = 0; i < (int)v.size(); ++i)
        if (v[i].second >= need && (best < 0 || v[i].second < v[best].second)) best = i;
    if (best < 0) return nullptr;
    void *p = v[best].first;
    *got = v[best].second;
    v.erase(v.begin() + best);
    return p;
}

// ---- device memory (hedl_set_allocator) -------------------------------------------
// Every device allocation of the library goes through dev_malloc / dev_free: the caller's
// allocator when one is installed (the Python binding installs torch's caching allocator),
// else cudaMalloc / cudaFree.  The allocator can only change while no KB is alive, so a
// block is always freed by the allocator that made it.
static std::mutex g_alloc_mu;
static hedl_dev_alloc_fn g_alloc = nullptr;
static hedl_dev_free_fn g_free = nullptr;
static void *g_alloc_ctx = nullptr;
static std::atomic<uint64_t> g_n_alloc{0}, g_n_free{0};
static int g_live_kbs = 0;

void live_kb_add(int d) {
    std::lock_guard<std::mutex> lk(g_alloc_mu);
    g_live_kbs += d;
}

#ifdef HEDL_CHECKED
// Checked build: every device block gets kGuard bytes of 0xA5 on both sides; dev_free checks
// them (after a device synchronise) and aborts with the block's size if a kernel wrote there.
constexpr size_t kGuard = 4096;
static std::mutex g_guard_mu;
static std::unordered_map<void *, size_t> g_guarded;       // user pointer -> requested bytes
static std::atomic<uint64_t> g_guard_checked{0};
static bool guard_check(void *p, size_t bytes) {
    const size_t pad = (bytes + 255) & ~size_t(255);
    std::vector<unsigned char> h(kGuard);
    bool ok = true;
    for (char *g : {(char *)p - kGuard, (char *)p + pad}) {
        if (cudaMemcpy(h.data(), g, kGuard, cudaMemcpyDeviceToHost) != cudaSuccess) return false;
        for (unsigned char c : h) ok &= c == 0xA5;
    }
    g_guard_checked.fetch_add(1);
    return ok;
}
static struct GuardReport {
    ~GuardReport() {
        std::fprintf(stderr, "[hedl checked] guard zones verified on %llu freed device blocks, none corrupted\n",
                     (unsigned long long)g_guard_checked.load());
    }
} g_guard_report;
#endif

cudaError_t dev_malloc(void **p, size_t bytes, cudaStream_t s) {
#ifdef HEDL_CHECKED
    {
        const size_t pad = (bytes + 255) & ~size_t(255);
        void *base = nullptr;
        cudaError_t e = cudaMalloc(&base, pad + 2 * kGuard);
        if (e != cudaSuccess) { *p = nullptr; return e; }
        cudaMemset(base, 0xA5, pad + 2 * kGuard);               // guards, and garbage in the block
        cudaDeviceSynchronize();
        *p = (char *)base + kGuard;
        std::lock_guard<std::mutex> lk(g_guard_mu);
        g_guarded[*p] = bytes;
        (void)s;
        return cudaSuccess;
    }
#endif
    *p = nullptr;
    g_n_alloc.fetch_add(1, std::memory_order_relaxed);
    const double t0 = timing_enabled() ? now_ms() : 0.0;
    cudaError_t e;
    if (g_alloc) {
        int dev = 0;
        cudaGetDevice(&dev);
        *p = g_alloc(bytes, dev, (void *)s, g_alloc_ctx);
        e = *p ? cudaSuccess : cudaErrorMemoryAllocation;
    } else {
        e = cudaMalloc(p, bytes);
    }
    if (timing_enabled())
        std::fprintf(stderr, "[hedl timing] dev_malloc %12zu B %9.3f ms\n", bytes, now_ms() - t0);
    return e;
}

bool dev_alloc_installed() { return g_alloc != nullptr; }

void dev_free(void *p, cudaStream_t s) {
    if (!p) return;
#ifdef HEDL_CHECKED
    {
        cudaDeviceSynchronize();
        size_t bytes = 0;
        {
            std::lock_guard<std::mutex> lk(g_guard_mu);
            auto it = g_guarded.find(p);
            if (it == g_guarded.end()) { std::fprintf(stderr, "[hedl checked] free of an unknown block %p\n", p); std::abort(); }
            bytes = it->second;
            g_guarded.erase(it);
        }
        if (!guard_check(p, bytes)) {
            std::fprintf(stderr, "[hedl checked] guard zone of a %zu-byte device block corrupted\n", bytes);
            std::abort();
        }
        cudaFree((char *)p - kGuard);
        (void)s;
        return;
    }
#endif
    g_n_free.fetch_add(1, std::memory_order_relaxed);
    if (g_free) {
        int dev = 0;
        cudaGetDevice(&dev);
        g_free(p, dev, (void *)s, g_alloc_ctx);
        return;
    }
    cudaFree(p);
}

static void pool_free_one(int role, void *p) {
    if (role == PR_PLAN_HOST || role == PR_DPLAN_HOST) cudaFreeHost(p);
    else dev_free(p);
}

constexpr size_t kPoolKeep = 4;

void pool_give(const hedl_kb *kb, int role, void *p, size_t bytes) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(kb->pool_mu);
    auto &v = kb->pool[role];
    v.push_back({p, bytes});
    // keep the kPoolKeep largest: a double-buffered caller (bench.py's e2e loop) has three
    // programs alive at once, and an evicted pinned block costs a cudaFreeHost (a device-wide
    // synchronisation) now and a cudaMallocHost (~80 ms for a C4 plan blob) later
    while (v.size() > kPoolKeep) {
        size_t mi = 0;
        for (size_t i = 1; i < v.size(); ++i)
            if (v[i].second < v[mi].second) mi = i;
        pool_free_one(role, v[mi].first);
        v.erase(v.begin() + mi);
    }
}

void pool_release_all(hedl_kb *kb) {
    std::lock_guard<std::mutex> lk(kb->pool_mu);
    for (int r = 0; r < PR_N; ++r) {
        for (auto &e : kb->pool[r]) pool_free_one(r, e.first);
        kb->pool[r].clear();
    }
}

const char *kKClassName[KC_N] = {"bool", "restrict", "restrict_heavy", "drange", "cover_init", "gather",
                                 "slice_pack", "slice", "slice_heavy", "kb", "slice_ex", "interp", "string", "bool_l2", "slice_u"};

static std::atomic<uint64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
void count_launches(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
uint64_t launches_total() { return g_launches.load(); }
static std::atomic<uint64_t> g_h2d{0}, g_d2h{0};
void count_io(uint64_t h2d, uint64_t d2h) {
    g_h2d.fetch_add(h2d, std::memory_order_relaxed);
    g_d2h.fetch_add(d2h, std::memory_order_relaxed);
}

struct ProfRec {
    cudaEvent_t a, b;
    int kc;
    double bytes, units;
};
static std::mutex g_prof_mu;
static bool g_prof_on = false;
static std::vector<ProfRec> g_prof;
static std::vector<cudaEvent_t> g_ev_pool;
static thread_local cudaEvent_t g_pending = nullptr;

static cudaEvent_t get_event() {
    if (!g_ev_pool.empty()) {
        cudaEvent_t e = g_ev_pool.back();
        g_ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

bool prof_active() { return g_prof_on; }

void prof_begin(cudaStream_t s, int) {
    if (!g_prof_on) return;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_pending = get_event();
    cudaEventRecord(g_pending, s);
}

void prof_end(cudaStream_t s, int kc, double bytes, double units) {
    if (!g_prof_on || !g_pending) return;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    cudaEvent_t b = get_event();
    cudaEventRecord(b, s);
    g_prof.push_back({g_pending, b, kc, bytes, units});
    g_pending = nullptr;
}

}  // namespace hedl

using namespace hedl;

extern "C" const char *hedl_last_error(void) { return g_last_error.c_str(); }
extern "C" const char *hedl_version(void) { return "hedl-b200 0.1 (sm_100a)"; }
extern "C" uint64_t hedl_launch_count(void) { return launches_total(); }

extern "C" hedl_status hedl_io_counters(uint64_t *h2d, uint64_t *d2h) {
    if (h2d) *h2d = g_h2d.load();
    if (d2h) *d2h = g_d2h.load();
    return HEDL_OK;
}

extern "C" hedl_status hedl_set_allocator(hedl_dev_alloc_fn alloc, hedl_dev_free_fn free_fn, void *ctx) {
    if ((alloc == nullptr) != (free_fn == nullptr)) return fail(HEDL_ERR_INVALID_ARG, "alloc and free must both be set or both be null");
    std::lock_guard<std::mutex> lk(g_alloc_mu);
    if (g_live_kbs > 0) return fail(HEDL_ERR_INVALID_ARG, "the allocator can only change while no KB is alive");
    g_alloc = alloc;
    g_free = free_fn;
    g_alloc_ctx = ctx;
    return HEDL_OK;
}

extern "C" hedl_status hedl_alloc_counters(uint64_t *n_alloc, uint64_t *n_free) {
    if (n_alloc) *n_alloc = g_n_alloc.load();
    if (n_free) *n_free = g_n_free.load();
    return HEDL_OK;
}

extern "C" hedl_status hedl_prof_enable(int on) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_prof_on = on != 0;
    return HEDL_OK;
}

extern "C" hedl_status hedl_prof_reset(void) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    for (auto &r : g_prof) {
        cudaEventSynchronize(r.b);
        g_ev_pool.push_back(r.a);
        g_ev_pool.push_back(r.b);
    }
    g_prof.clear();
    return HEDL_OK;
}

extern "C" int hedl_prof_read(hedl_prof_entry *out, int max_entries) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    hedl_prof_entry acc[KC_N];
    std::memset(acc, 0, sizeof(acc));
    for (auto &r : g_prof) {
        cudaEventSynchronize(r.b);
        float ms = 0;
        cudaEventElapsedTime(&ms, r.a, r.b);
        acc[r.kc].launches++;
        acc[r.kc].total_ms += ms;
        acc[r.kc].alg_bytes += r.bytes;
        acc[r.kc].units += r.units;
    }
    int n = 0;
    for (int k = 0; k < KC_N; ++k) {
        if (!acc[k].launches) continue;
        if (out && n < max_entries) {
            out[n] = acc[k];
            std::snprintf(out[n].name, sizeof(out[n].name), "%s", kKClassName[k]);
        }
        ++n;
    }
    return n;
}
