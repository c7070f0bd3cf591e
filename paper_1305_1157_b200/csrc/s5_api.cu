// s5_api.cu -- host driver and C-ABI of libs5.so (see include/s5.h).
//
// The driver replaces the reference's recursion over SortJobs
// (samplesort.py:273-434, scheduler.py) with level-synchronous device
// segment lists: every level launches the wide pipeline, the fused narrow
// kernel and the warp base case over all live segments at once, and reads
// back only the next level's list counters (one 64-byte D2H per level).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstddef>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <immintrin.h>

#include <atomic>
#include <condition_variable>
#include <functional>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/s5.h"
#include "s5_kernels.cuh"

using namespace s5;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define S5_CUDA(call)                                                                  \
    do {                                                                               \
        cudaError_t e_ = (call);                                                       \
        if (e_ != cudaSuccess)                                                         \
            return fail(S5_E_CUDA, "%s failed: %s", #call, cudaGetErrorString(e_));    \
    } while (0)

struct Cfg {
    uint32_t v, alpha, classifier, small_max, local_max, narrow_max, flags, dmax, wide_dcap;
    uint32_t wide_target, local_target;
    uint64_t seed;
};

#ifndef S5_ROOT_STAGES
#define S5_ROOT_STAGES 3
#endif
constexpr uint32_t kRootStages = S5_ROOT_STAGES;  // bulk-copy stages of the root scatter
constexpr uint32_t kTreeAhead = 1024;  // tree CTAs launched ahead of the level's host read
constexpr uint32_t kLocalThreads = 512;   // segments of <= 4096 strings
using LocalCfg = LocalSmem<kLocalThreads>;
constexpr uint32_t kLocalXSThreads = 64;  // <= 512
using LocalXSCfg = LocalSmem<kLocalXSThreads>;
constexpr uint32_t kLocalSThreads = 128;  // <= 1024
using LocalSCfg = LocalSmem<kLocalSThreads>;
constexpr uint32_t kLocalMThreads = 256;  // <= 2048
using LocalMCfg = LocalSmem<kLocalMThreads>;
#ifndef S5_NARROW_DEFAULT
#define S5_NARROW_DEFAULT 4096
#endif
// segments of (local_max, kNarrowDefault] strings take the one-CTA S^5 step
// (off by default: measured slower than the wide pipeline at level 1, DESIGN 8)
constexpr uint32_t kNarrowDefault = S5_NARROW_DEFAULT;

int resolve(const s5_config* c, Cfg* o) {
    o->v = c && c->v ? c->v : 8191;
    o->alpha = c && c->alpha ? c->alpha : 4;
    o->classifier = c ? c->classifier : 0;
    o->small_max = c && c->small_max ? c->small_max : 32;
    o->narrow_max = c && c->narrow_max ? c->narrow_max : kNarrowDefault;
    o->local_max = c && c->local_max ? c->local_max : LocalCfg::maxn;
    uint32_t wv = c && c->wide_v ? c->wide_v : 511;
    uint32_t wd = 0;
    while (wd < 31 && ((1u << wd) - 1) < wv) ++wd;
    if (((1u << wd) - 1) != wv || wd > kWideDMax)
        return fail(S5_E_INVALID, "wide_v must be 2**d - 1 with d <= %u, got %u", kWideDMax, wv);
    o->wide_dcap = wd;
    o->wide_target = c ? c->wide_target : 0;
    o->local_target = c && c->local_target ? c->local_target : 8;
    if (o->local_target > 32) return fail(S5_E_INVALID, "local_target must be <= 32");
    o->flags = c ? c->flags : 0;
    o->seed = c ? c->seed : 1;
    uint32_t d = 0;
    while (d < 31 && ((1u << d) - 1) < o->v) ++d;
    if (o->v < 1 || ((1u << d) - 1) != o->v)
        return fail(S5_E_INVALID, "need 2**d - 1 splitters, got v=%u", o->v);
    o->dmax = d;
    if (o->classifier > 1) return fail(S5_E_INVALID, "classifier must be 0 (unroll) or 1 (equal)");
    if (o->small_max < 1 || o->small_max > 32)
        return fail(S5_E_INVALID, "small_max must be in [1, 32]");
    if (o->narrow_max < o->small_max || o->narrow_max > kNarrowMaxSize)
        return fail(S5_E_INVALID, "narrow_max must be in [small_max, %u]", kNarrowMaxSize);
    if (o->local_max > LocalCfg::maxn) o->local_max = LocalCfg::maxn;
    if (o->local_max < o->small_max) o->local_max = o->small_max;
    if (o->local_max > o->narrow_max) o->local_max = o->narrow_max;
    if (o->alpha > 64) return fail(S5_E_INVALID, "alpha must be <= 64");
    return 0;
}

uint64_t align_up(uint64_t x, uint64_t a = 256) { return (x + a - 1) / a * a; }

struct Layout {
    uint64_t off[2], key[2], key2[2], lists[2][NCLS], cta_start, tree_off, hist_off, tree_pool, hist_pool,
        ctl, hints, bkt, pos, total;
    uint32_t cap[NCLS];
    uint64_t tree_cap, hist_cap;
};

Layout make_layout(uint64_t n, const Cfg& c) {
    Layout L{};
    uint64_t at = 0;
    auto take = [&](uint64_t bytes) {
        uint64_t p = at;
        at = align_up(at + bytes);
        return p;
    };
    L.cap[SMALL] = static_cast<uint32_t>(n / 2 + 1);
    L.cap[LOCAL_W] = static_cast<uint32_t>(n / (c.small_max + 1) + 1);
    L.cap[LOCAL_XS] = static_cast<uint32_t>(n / (std::min(c.local_max, kWarpLocalMax) + 1) + 1);
    L.cap[LOCAL_S] = static_cast<uint32_t>(n / (std::min(c.local_max, LocalXSCfg::maxn) + 1) + 1);
    L.cap[LOCAL_M] = static_cast<uint32_t>(n / (std::min(c.local_max, LocalSCfg::maxn) + 1) + 1);
    L.cap[LOCAL] = static_cast<uint32_t>(n / (std::min(c.local_max, LocalMCfg::maxn) + 1) + 1);
    L.cap[NARROW] = static_cast<uint32_t>(n / (c.local_max + 1) + 1);
    L.cap[WIDE] = static_cast<uint32_t>(n / (c.narrow_max + 1) + 1);
    for (int s = 0; s < 2; ++s) L.off[s] = take(n * 4);
    for (int s = 0; s < 2; ++s) L.key[s] = take(n * 8);
    for (int b = 0; b < 2; ++b)
        for (int q = 0; q < NCLS; ++q) L.lists[b][q] = take(uint64_t(L.cap[q]) * sizeof(Seg));
    L.cta_start = take((uint64_t(L.cap[WIDE]) + 1) * 4);
    L.tree_off = take(uint64_t(L.cap[WIDE]) * 8);
    L.hist_off = take(uint64_t(L.cap[WIDE]) * 8);
    // wide segments have > narrow_max strings; v+1 <= size/8, and at most
    // ceil(size/64K) <= 296 rows of k <= size/4 counters (see choose_d)
    L.tree_cap = n / 4 + uint64_t(L.cap[WIDE]) * (2 + kLutWords) + 16;
    L.hist_cap = n + n / 2 + 4 * uint64_t(L.cap[WIDE]) + 65536;
    if (const char* e = getenv("S5_TEST_POOL_WORDS")) {  // tests: force the overflow path
        L.tree_cap = std::min<uint64_t>(L.tree_cap, strtoull(e, nullptr, 10));
        L.hist_cap = std::min<uint64_t>(L.hist_cap, strtoull(e, nullptr, 10));
    }
    L.tree_pool = take(L.tree_cap * 8);
    L.hist_pool = take(L.hist_cap * 4);
    L.hints = take(n * sizeof(uint2));
    L.bkt = take(n * 2);
    L.ctl = take(sizeof(Ctl));
    for (int s = 0; s < 2; ++s) L.key2[s] = take(n > c.narrow_max ? n * 8 : 0);
    // flags bit13 (arenas >= 4 GiB): the string-index -> arena-position table
    L.pos = take((c.flags & 8192) ? n * 8 : 0);
    L.total = at;
    return L;
}

template <typename K>
int set_smem(K kernel, int bytes) {
    if (bytes > 232448) return fail(S5_E_CUDA, "shared memory request of %d bytes", bytes);
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess)
        return fail(S5_E_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    return 0;
}

constexpr int kWideTreeSmem = kWideSampleCap * 8 + (1 << kWideDMax) * 12;
// k_wide_tree: sample of <= alpha * v keys (power of two >= 64) + node ranges
inline uint32_t wide_sample_words(const Cfg& c) {
    const uint32_t dw = std::min(c.dmax, c.wide_dcap);
    const uint32_t m = std::min<uint32_t>(kWideSampleCap, c.alpha * ((1u << dw) - 1));
    uint32_t M = 64;
    while (M < m) M <<= 1;
    return M;
}
inline int wide_tree_smem(const Cfg& c) {
    return wide_sample_words(c) * 8 + (1 << std::min(c.dmax, c.wide_dcap)) * 12;
}
constexpr int kWideSmem = (1 << kWideDMax) * 8 + ((2 << kWideDMax) + 2) * 4 + (1 << kWideDMax) * 8 + (kLutCells + 1) * 2 + 16;
inline int wide_smem(uint32_t dcap) {
    return (1 << dcap) * 8 + ((2 << dcap) + 2) * 4 + (1 << dcap) * 8 + (kLutCells + 1) * 2 + 16;
}

int init_attributes() {
    static std::once_flag once;
    static int rc = 0;
    std::call_once(once, [] {
        rc = set_smem(k_narrow<false>, NarrowSmem::total);
        if (!rc) rc = set_smem(k_narrow<true>, NarrowSmem::total);
        if (!rc) rc = set_smem(k_wide_tree<kTreeThreads>, kWideTreeSmem);
        if (!rc) rc = set_smem(k_wide_tree<kTreeThreadsFew>, kWideTreeSmem);
        if (!rc) rc = set_smem(k_wide_count<false>, kWideSmem);
        if (!rc) rc = set_smem(k_wide_count<true>, kWideSmem);
        if (!rc) rc = set_smem(k_wide_count<false, true>, kWideSmem);
        if (!rc) rc = set_smem(k_wide_count<false, false, true>, kWideSmem);
        if (!rc) rc = set_smem(k_wide_count<false, true, true>, kWideSmem);
        if (!rc) rc = set_smem(k_wide_scatter, WideScatterSmem::total);
        if (!rc) rc = set_smem(k_wide_scatter_tma<1024, 4096>, WideTmaSmem<4096>::bytes(kWideDMax));
        if (!rc) rc = set_smem(k_wide_scatter_tma<1024, 4096, kRootStages>,
                               WideTmaSmem<4096, kRootStages>::bytes(kWideDMax));
        if (!rc) rc = set_smem(k_wide_scatter_tma<512, 2048>, WideTmaSmem<2048>::bytes(kWideDMax));
        if (!rc) rc = set_smem(k_build_tree, 227 * 1024);
        if (!rc) rc = set_smem(k_local<kLocalThreads>, LocalCfg::total);
        if (!rc) rc = set_smem(k_local<kLocalSThreads>, LocalSCfg::total);
        if (!rc) rc = set_smem(k_local<kLocalXSThreads>, LocalXSCfg::total);
        if (!rc) rc = set_smem(k_local<kLocalXSThreads, true>, LocalXSCfg::total);
        if (!rc) rc = set_smem(k_local<kLocalSThreads, true>, LocalSCfg::total);
        if (!rc) rc = set_smem(k_local<kLocalMThreads>, LocalMCfg::total);
    });
    return rc;
}

// ctl and seq are mapped (zero-copy, usable from every device under UVA):
// the level loop's control block is published by k_publish and read by a
// host spin on seq instead of a copy + stream synchronisation
struct Pinned {
    Ctl* ctl = nullptr;
    uint32_t* seq = nullptr;
    uint32_t next = 0;
    ~Pinned() {  // thread exit (the mapped block is per thread)
        if (ctl) cudaFreeHost(ctl);
        if (seq) cudaFreeHost(seq);
    }
};

Pinned& pinned() {
    thread_local Pinned p;
    if (!p.ctl || !p.seq) {
        const unsigned fl = cudaHostAllocMapped | cudaHostAllocPortable;
        if (!p.ctl && cudaHostAlloc(&p.ctl, sizeof(Ctl), fl) != cudaSuccess) p.ctl = nullptr;
        if (!p.seq && cudaHostAlloc(&p.seq, 64, fl) != cudaSuccess) p.seq = nullptr;
        if (p.seq) *p.seq = 0;
    }
    return p;
}

// Serialises sorts on one device: the side streams and their fork/join
// events (Side) are shared by every caller on the device, so one sort's
// enqueue sequence must not interleave with another's.
struct DevSortLock {
    std::mutex mu;
};

// Error-path cleanup of sort_impl: timing events destroyed on every return;
// on an error return the caller's stream is drained first, so no kernel of
// the failed call is still reading the workspace when the caller reuses it.
struct SortScope {
    cudaStream_t st = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    bool ok = false;
    ~SortScope() {
        if (!ok) cudaStreamSynchronize(st);
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
    }
};

// copy of the device control block into mapped host memory, then the
// sequence number (system-scope fence between them)
__global__ void k_publish(const Ctl* __restrict__ src, Ctl* dst, uint32_t* seq, uint32_t val) {
    constexpr uint32_t W = sizeof(Ctl) / 4;
    const uint32_t* a = reinterpret_cast<const uint32_t*>(src);
    volatile uint32_t* b = reinterpret_cast<volatile uint32_t*>(dst);
    for (uint32_t i = threadIdx.x; i < W; i += blockDim.x) b[i] = a[i];
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) *reinterpret_cast<volatile uint32_t*>(seq) = val;
}

// wait for k_publish(val): spin on the mapped word; a failed stream ends the
// wait with its error
int wait_published(Pinned& hp, uint32_t val, cudaStream_t st) {
    const volatile uint32_t* q = hp.seq;
    for (uint32_t spins = 0; *q != val; ++spins) {
        if ((spins & 1023) == 1023) {
            const cudaError_t e = cudaStreamQuery(st);
            if (e != cudaSuccess && e != cudaErrorNotReady)
                return fail(S5_E_CUDA, "level kernels: %s", cudaGetErrorString(e));
            if (e == cudaSuccess && *q != val)  // stream drained: the word must be there
                return fail(S5_E_INTERNAL, "control block not published");
        }
#if defined(__x86_64__)
        __builtin_ia32_pause();
#endif
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    return 0;
}

// One instance per CUDA device (the library's cached buffers live on the
// device that was current when they were made).
std::mutex& registry_mutex() {
    static std::mutex m;
    return m;
}
template <class T>
std::map<int, T>& registry() {
    static std::map<int, T> r;  // node-based: references stay valid
    return r;
}
template <class T>
T& per_device() {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(registry_mutex());
    return registry<T>()[dev];
}

int grid_for(uint64_t n, int threads, int max_blocks = 148 * 16) {
    uint64_t b = (n + threads - 1) / threads;
    return static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(b, max_blocks)));
}

// Launch bookkeeping; with cfg flags bit1, CUDA events around every launch
// give per-kernel device time on the launching stream.
// Side streams of a device: the size classes of one level work on disjoint
// segments, so the one-CTA classes run concurrently with each other and
// with the level's wide step (fork/join by events; the per-kernel profiling
// mode keeps everything on the caller's stream).
struct Side {
    static constexpr int kLanes = 7;
    cudaStream_t s[kLanes] = {};
    cudaEvent_t fork = nullptr, join[kLanes] = {};
    bool ok = false;
};

Side* side_streams() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    std::lock_guard<std::mutex> g(registry_mutex());
    Side& sd = registry<Side>()[dev];
    if (!sd.ok) {
        bool good = cudaEventCreateWithFlags(&sd.fork, cudaEventDisableTiming) == cudaSuccess;
        for (int i = 0; good && i < Side::kLanes; ++i)
            good = cudaStreamCreateWithFlags(&sd.s[i], cudaStreamNonBlocking) == cudaSuccess &&
                   cudaEventCreateWithFlags(&sd.join[i], cudaEventDisableTiming) == cudaSuccess;
        if (!good) return nullptr;
        sd.ok = true;
    }
    return &sd;
}

struct Prof {
    bool on = false;
    cudaStream_t st = nullptr;
    uint64_t launches = 0;
    uint32_t count[16] = {};
    struct Rec { int k; uint32_t level; uint64_t strings; cudaEvent_t a, b; };
    std::vector<Rec> recs;
    uint64_t elems[16] = {};
    uint32_t level = 0;
    void begin(int k, uint64_t strings = 0) {
        ++launches;
        ++count[k];
        elems[k] += strings;
        if (!on) return;
        Rec r{k, level, strings, nullptr, nullptr};
        cudaEventCreate(&r.a);
        cudaEventCreate(&r.b);
        cudaEventRecord(r.a, st);
        recs.push_back(r);
    }
    void end() {
        if (on && !recs.empty()) cudaEventRecord(recs.back().b, st);
    }
    cudaEvent_t origin = nullptr;
    void finish(s5_stats* stats) {
        if (stats) {
            stats->launches = launches;
            for (int k = 0; k < 16; ++k) {
                stats->kern_launches[k] = count[k];
                stats->kern_strings[k] = elems[k];
            }
        }
        uint32_t nrec = 0;
        for (auto& r : recs) {
            float ms = 0, t0 = 0;
            if (stats && cudaEventSynchronize(r.b) == cudaSuccess &&
                cudaEventElapsedTime(&ms, r.a, r.b) == cudaSuccess) {
                stats->kern_ms[r.k] += ms;
                if (origin) cudaEventElapsedTime(&t0, origin, r.a);
                if (nrec < S5_MAX_LAUNCH_RECS)
                    stats->launch_recs[nrec++] = s5_launch_rec{static_cast<uint32_t>(r.k), r.level,
                                                               r.strings, ms, t0};
            }
            cudaEventDestroy(r.a);
            cudaEventDestroy(r.b);
        }
        recs_total = recs.size();
        recs.clear();
    }
    size_t recs_total = 0;
    ~Prof() {  // error returns: events of unfinished records
        for (auto& r : recs) {
            cudaEventDestroy(r.a);
            cudaEventDestroy(r.b);
        }
    }
};

}  // namespace

namespace {

// Persistent host worker pool for the staging copies (thread start-up per
// chunk would cost more than the copies themselves).
class Pool {
    std::vector<std::thread> th_;
    std::mutex job_mu_;  // one job at a time: callers on other devices queue here
    std::mutex mu_;
    std::condition_variable go_, done_;
    std::function<void(unsigned)> job_;
    uint64_t gen_ = 0;
    unsigned left_ = 0;
    bool stop_ = false;
    unsigned T_ = 1;

    Pool() {
        T_ = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
        for (unsigned i = 1; i < T_; ++i) th_.emplace_back([this, i] { loop(i); });
    }
    ~Pool() {
        {
            std::lock_guard<std::mutex> g(mu_);
            stop_ = true;
        }
        go_.notify_all();
        for (auto& t : th_) t.join();
    }
    void loop(unsigned i) {
        uint64_t seen = 0;
        for (;;) {
            std::function<void(unsigned)> f;
            {
                std::unique_lock<std::mutex> lk(mu_);
                go_.wait(lk, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
                f = job_;
            }
            f(i);
            std::lock_guard<std::mutex> g(mu_);
            if (--left_ == 0) done_.notify_one();
        }
    }

public:
    static Pool& get() {
        static Pool p;
        return p;
    }
    // f(begin, end) over T contiguous parts of [0, n)
    void par_for(uint64_t n, const std::function<void(uint64_t, uint64_t)>& f) {
        const unsigned T = n < (1u << 16) ? 1u : T_;
        if (T == 1) {
            f(0, n);
            return;
        }
        // the job slot (job_, left_, gen_) belongs to one caller until every
        // worker has finished its part: concurrent callers (threads driving
        // different GPUs through the host paths) wait for it
        std::lock_guard<std::mutex> job(job_mu_);
        auto part = [&, T](unsigned i) { f(n * i / T, n * (i + 1) / T); };
        {
            std::lock_guard<std::mutex> g(mu_);
            job_ = part;
            left_ = T_ - 1;
            ++gen_;
        }
        go_.notify_all();
        part(0);
        std::unique_lock<std::mutex> lk(mu_);
        done_.wait(lk, [&] { return left_ == 0; });
    }
    unsigned threads() const { return T_; }
    // f(tid, T) once on every pool thread (tid 0 = the caller)
    void run_all(const std::function<void(unsigned, unsigned)>& f) {
        if (T_ == 1) {
            f(0, 1);
            return;
        }
        std::lock_guard<std::mutex> job(job_mu_);
        const unsigned T = T_;
        auto part = [&, T](unsigned i) { f(i, T); };
        {
            std::lock_guard<std::mutex> g(mu_);
            job_ = part;
            left_ = T_ - 1;
            ++gen_;
        }
        go_.notify_all();
        part(0);
        std::unique_lock<std::mutex> lk(mu_);
        done_.wait(lk, [&] { return left_ == 0; });
    }
};

// Host staging kernels.  The output streams are written once and not read
// again by this thread, so AVX2 non-temporal stores skip the read-for-
// ownership of every destination line (half the host memory traffic).
bool has_avx2() {
    static const bool v = (__builtin_cpu_init(), __builtin_cpu_supports("avx2"));
    return v;
}

// int64 handles -> u32 offsets with the range check; true if any is outside [0, lim).
// NT: non-temporal stores (a staging buffer larger than the host cache);
// otherwise plain stores, so a small staging slot stays cached for the DMA read
template <bool NT = true>
__attribute__((target("avx2"))) bool narrow_u32_avx2(const int64_t* src, uint32_t* dst, uint64_t n,
                                                     uint64_t lim) {
    uint64_t i = 0, bad = 0;
    for (; i < n && (reinterpret_cast<uintptr_t>(dst + i) & 31); ++i) {
        bad |= static_cast<uint64_t>(src[i]) >= lim;
        dst[i] = static_cast<uint32_t>(src[i]);
    }
    const __m256i zero = _mm256_setzero_si256();
    const __m256i top = _mm256_set1_epi64x(static_cast<long long>(lim) - 1);
    const __m256i lows = _mm256_setr_epi32(0, 2, 4, 6, 1, 3, 5, 7);
    __m256i badv = zero;
    for (; i + 8 <= n; i += 8) {
        const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i));
        const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 4));
        badv = _mm256_or_si256(badv, _mm256_or_si256(_mm256_cmpgt_epi64(zero, a), _mm256_cmpgt_epi64(a, top)));
        badv = _mm256_or_si256(badv, _mm256_or_si256(_mm256_cmpgt_epi64(zero, b), _mm256_cmpgt_epi64(b, top)));
        const __m128i la = _mm256_castsi256_si128(_mm256_permutevar8x32_epi32(a, lows));
        const __m128i lb = _mm256_castsi256_si128(_mm256_permutevar8x32_epi32(b, lows));
        if (NT) _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i), _mm256_set_m128i(lb, la));
        else _mm256_store_si256(reinterpret_cast<__m256i*>(dst + i), _mm256_set_m128i(lb, la));
    }
    for (; i < n; ++i) {
        bad |= static_cast<uint64_t>(src[i]) >= lim;
        dst[i] = static_cast<uint32_t>(src[i]);
    }
    if (NT) _mm_sfence();
    return bad || !_mm256_testz_si256(badv, badv);
}

template <typename T>
__attribute__((target("avx2"))) void widen_avx2(const T* src, int64_t* dst, uint64_t n) {
    uint64_t i = 0;
    for (; i < n && (reinterpret_cast<uintptr_t>(dst + i) & 31); ++i) dst[i] = src[i];
    for (; i + 4 <= n; i += 4) {
        __m256i v;
        if (sizeof(T) == 4) {
            v = _mm256_cvtepu32_epi64(_mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i)));
        } else if (sizeof(T) == 2) {
            v = _mm256_cvtepu16_epi64(_mm_loadl_epi64(reinterpret_cast<const __m128i*>(src + i)));
        } else {
            uint32_t x;
            memcpy(&x, src + i, 4);
            v = _mm256_cvtepu8_epi64(_mm_cvtsi32_si128(static_cast<int>(x)));
        }
        _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i), v);
    }
    for (; i < n; ++i) dst[i] = src[i];
    _mm_sfence();
}

template <bool NT = true>
bool narrow_u32(const int64_t* src, uint32_t* dst, uint64_t n, uint64_t lim) {
    if (has_avx2()) return narrow_u32_avx2<NT>(src, dst, n, lim);
    uint64_t bad = 0;
    for (uint64_t i = 0; i < n; ++i) {
        bad |= static_cast<uint64_t>(src[i]) >= lim;
        dst[i] = static_cast<uint32_t>(src[i]);
    }
    return bad;
}

template <typename T>
void widen(const T* src, int64_t* dst, uint64_t n) {
    if (has_avx2()) return widen_avx2<T>(src, dst, n);
    for (uint64_t i = 0; i < n; ++i) dst[i] = src[i];
}

void par_memcpy(void* dst, const void* src, uint64_t bytes) {
    Pool::get().par_for(bytes, [&](uint64_t a, uint64_t b) {
        memcpy(static_cast<char*>(dst) + a, static_cast<const char*>(src) + a, b - a);
    });
}

__global__ void k_widen32(const uint32_t* __restrict__ a, int64_t* __restrict__ b, uint64_t n) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x)
        b[i] = a[i];
}

template <typename T>
__global__ void k_shrink(const int64_t* __restrict__ a, T* __restrict__ b, uint64_t n) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x)
        b[i] = static_cast<T>(a[i]);
}

__global__ void k_max64(const int64_t* __restrict__ a, uint64_t n, unsigned long long* out) {
    unsigned long long m = 0;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x)
        m = max(m, static_cast<unsigned long long>(a[i]));
    for (int x = 16; x > 0; x >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, x));
    if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

struct HostPath {
    std::mutex mu;
    void* dbuf = nullptr;
    uint64_t dbytes = 0;
    static constexpr int kStages = 3;
    void* stage[kStages] = {};
    cudaEvent_t ev[kStages] = {};
    uint64_t piece = 0;  // elements per staged piece (S5_HOST_PIECE overrides)
    unsigned long long* dmax = nullptr;
    unsigned long long* hmax = nullptr;
    void* xbuf = nullptr;  // narrowing scratch of the standalone transfer entries
    uint64_t xbytes = 0;
    static constexpr uint64_t kChunk = 32ull << 20;  // bytes per staging buffer
    // staging ring (S5_HOST_RING, default: both directions): R pinned slots of
    // P bytes (default 48 x 2 MiB); the copy engine and the host workers each
    // run ahead on their own pieces -- no barrier per piece as in the
    // three-stage path (config 2 e2e 12.5-13.3 -> 11.2-11.4 ms, same box,
    // profiles/e2e_ring.py)
    static constexpr int kRingMax = 64;
    int ring = -1;  // -1: not configured yet
    char* rbuf = nullptr;
    uint64_t rP = 0;
    int rR = 0;
    cudaEvent_t rev[kRingMax] = {};
    std::atomic<int64_t> rready[kRingMax];
    std::atomic<int64_t> rfreed[kRingMax];
};

HostPath& host_path() { return per_device<HostPath>(); }

struct PartScratch {  // s5_partition
    std::mutex mu;
    void* d = nullptr;
    uint64_t bytes = 0;
    unsigned long long* h = nullptr;
};

int host_path_init(HostPath& H) {
    if (H.stage[0]) return 0;
    const char* e = getenv("S5_HOST_PIECE");
    H.piece = e ? strtoull(e, nullptr, 10) : (8ull << 20);
    H.piece = std::max<uint64_t>(1, std::min(H.piece, HostPath::kChunk / 8));
    for (int i = 0; i < HostPath::kStages; ++i) {
        S5_CUDA(cudaHostAlloc(&H.stage[i], HostPath::kChunk, cudaHostAllocDefault));
        S5_CUDA(cudaEventCreateWithFlags(&H.ev[i], cudaEventDisableTiming));
    }
    S5_CUDA(cudaMalloc(&H.dmax, sizeof(unsigned long long)));
    S5_CUDA(cudaHostAlloc(&H.hmax, sizeof(unsigned long long), cudaHostAllocDefault));
    // bit 0: downloads through the ring, bit 1: uploads too, bit 2: plain
    // (cached) narrowing stores into the ring instead of non-temporal ones
    const char* r = getenv("S5_HOST_RING");
    H.ring = Pool::get().threads() >= 2 ? (r ? atoi(r) : 3) : 0;  // a scheduler + at least one worker
    if (H.ring) {
        const char* p = getenv("S5_RING_PIECE");
        const char* q = getenv("S5_RING_SLOTS");
        H.rP = p ? strtoull(p, nullptr, 10) : (2ull << 20);
        H.rP = std::max<uint64_t>(64 << 10, std::min<uint64_t>(H.rP, 16ull << 20)) & ~uint64_t(255);
        H.rR = q ? atoi(q) : 48;
        H.rR = std::max(2, std::min(H.rR, HostPath::kRingMax));
        S5_CUDA(cudaHostAlloc(&H.rbuf, H.rP * H.rR, cudaHostAllocDefault));
        for (int i = 0; i < H.rR; ++i) S5_CUDA(cudaEventCreateWithFlags(&H.rev[i], cudaEventDisableTiming));
    }
    return 0;
}

// The staging ring.  The caller's thread (pool thread 0) schedules the DMA
// in piece order on the caller's stream and retires finished copies by
// event queries; the other pool threads claim pieces in order and narrow
// (H2D) or widen (D2H) them.  Slot s holds pieces s, s + R, ...; per slot
// `rready` is the last piece made ready for the other side and `rfreed` the
// last piece whose slot use is over.  A worker never waits for the others,
// only for its own piece's slot or copy.
struct RingPiece {
    const char* d;   // device source (D2H)
    int64_t* h;      // host destination (D2H)
    uint64_t count;
    uint32_t w;
};

template <typename Sched, typename Work>
int ring_run(HostPath& H, uint64_t K, Sched&& sched_step, Work&& work) {
    const int R = H.rR;
    for (int s = 0; s < R; ++s) {
        H.rready[s].store(static_cast<int64_t>(s) - R, std::memory_order_relaxed);
        H.rfreed[s].store(static_cast<int64_t>(s) - R, std::memory_order_relaxed);
    }
    std::atomic<uint64_t> next{0};
    std::atomic<int> abort{0};
    std::atomic<int> err{0};
    Pool::get().run_all([&](unsigned tid, unsigned) {
        if (tid == 0) {
            if (int e = sched_step(abort)) {
                err.store(e);
                abort.store(1);
            }
            return;
        }
        for (;;) {
            const uint64_t k = next.fetch_add(1, std::memory_order_relaxed);
            if (k >= K) return;
            if (!work(k, abort)) return;
        }
    });
    return err.load();
}

int host_upload_ring(HostPath& H, const int64_t* h_handles, uint64_t n, uint64_t arena_len,
                     uint32_t* d32, cudaStream_t st) {
    const int R = H.rR;
    const uint64_t E = H.rP / 4;
    const uint64_t K = (n + E - 1) / E;
    std::atomic<bool> bad{false};
    auto sched = [&](std::atomic<int>& abort) -> int {
        uint64_t issued = 0, retired = 0;
        while (retired < K) {
            bool progress = false;
            if (issued < K) {
                const int s = static_cast<int>(issued % R);
                if (H.rready[s].load(std::memory_order_acquire) == static_cast<int64_t>(issued)) {
                    const uint64_t len = std::min(E, n - issued * E);
                    S5_CUDA(cudaMemcpyAsync(d32 + issued * E, H.rbuf + uint64_t(s) * H.rP, len * 4,
                                            cudaMemcpyHostToDevice, st));
                    S5_CUDA(cudaEventRecord(H.rev[s], st));
                    ++issued;
                    progress = true;
                }
            }
            if (retired < issued) {
                const int s = static_cast<int>(retired % R);
                const cudaError_t q = cudaEventQuery(H.rev[s]);
                if (q == cudaSuccess) {
                    H.rfreed[s].store(static_cast<int64_t>(retired), std::memory_order_release);
                    ++retired;
                    progress = true;
                } else if (q != cudaErrorNotReady) {
                    return fail(S5_E_CUDA, "staging DMA failed: %s", cudaGetErrorString(q));
                }
            }
            if (!progress) _mm_pause();
            if (abort.load(std::memory_order_relaxed)) return 0;
        }
        return 0;
    };
    auto work = [&](uint64_t k, std::atomic<int>& abort) -> bool {
        const int s = static_cast<int>(k % R);
        const int64_t want = static_cast<int64_t>(k) - R;
        while (H.rfreed[s].load(std::memory_order_acquire) != want)
            if (abort.load(std::memory_order_relaxed)) return false; else _mm_pause();
        const uint64_t len = std::min(E, n - k * E);
        uint32_t* dst = reinterpret_cast<uint32_t*>(H.rbuf + uint64_t(s) * H.rP);
        if ((H.ring & 4) ? narrow_u32<false>(h_handles + k * E, dst, len, arena_len)
                         : narrow_u32<true>(h_handles + k * E, dst, len, arena_len))
            bad.store(true, std::memory_order_relaxed);
        H.rready[s].store(static_cast<int64_t>(k), std::memory_order_release);
        return true;
    };
    if (int e = ring_run(H, K, sched, work)) return e;
    if (bad.load()) return fail(S5_E_RANGE, "handle outside the arena");
    return 0;
}

int host_download_ring(HostPath& H, const std::vector<RingPiece>& pieces, cudaStream_t st) {
    const int R = H.rR;
    const uint64_t K = pieces.size();
    auto sched = [&](std::atomic<int>& abort) -> int {
        uint64_t issued = 0, retired = 0;
        while (retired < K) {
            bool progress = false;
            if (issued < K) {
                const int s = static_cast<int>(issued % R);
                if (H.rfreed[s].load(std::memory_order_acquire) == static_cast<int64_t>(issued) - R) {
                    const RingPiece& P = pieces[issued];
                    S5_CUDA(cudaMemcpyAsync(H.rbuf + uint64_t(s) * H.rP, P.d, P.count * P.w,
                                            cudaMemcpyDeviceToHost, st));
                    S5_CUDA(cudaEventRecord(H.rev[s], st));
                    ++issued;
                    progress = true;
                }
            }
            if (retired < issued) {
                const int s = static_cast<int>(retired % R);
                const cudaError_t q = cudaEventQuery(H.rev[s]);
                if (q == cudaSuccess) {
                    H.rready[s].store(static_cast<int64_t>(retired), std::memory_order_release);
                    ++retired;
                    progress = true;
                } else if (q != cudaErrorNotReady) {
                    return fail(S5_E_CUDA, "staging DMA failed: %s", cudaGetErrorString(q));
                }
            }
            if (!progress) _mm_pause();
            if (abort.load(std::memory_order_relaxed)) return 0;
        }
        return 0;
    };
    auto work = [&](uint64_t k, std::atomic<int>& abort) -> bool {
        const int s = static_cast<int>(k % R);
        while (H.rready[s].load(std::memory_order_acquire) != static_cast<int64_t>(k))
            if (abort.load(std::memory_order_relaxed)) return false; else _mm_pause();
        const RingPiece& P = pieces[k];
        const char* sp = H.rbuf + uint64_t(s) * H.rP;
        switch (P.w) {
            case 1: widen(reinterpret_cast<const uint8_t*>(sp), P.h, P.count); break;
            case 2: widen(reinterpret_cast<const uint16_t*>(sp), P.h, P.count); break;
            case 4: widen(reinterpret_cast<const uint32_t*>(sp), P.h, P.count); break;
            default: memcpy(P.h, sp, P.count * 8);
        }
        H.rfreed[s].store(static_cast<int64_t>(k), std::memory_order_release);
        return true;
    };
    return ring_run(H, K, sched, work);
}

int host_scratch(HostPath& H, uint64_t bytes) {
    if (bytes <= H.xbytes) return 0;
    if (H.xbuf) cudaFree(H.xbuf);
    H.xbuf = nullptr;
    H.xbytes = 0;
    S5_CUDA(cudaMalloc(&H.xbuf, bytes));
    H.xbytes = bytes;
    return 0;
}

// H2D: narrow + range-check into pinned staging (host workers), DMA, widen
// on the device; chunk i is narrowed while chunk i-1 is in flight
int host_upload(HostPath& H, const int64_t* h_handles, uint64_t n, uint64_t arena_len,
                uint32_t* d32, int64_t* dh, cudaStream_t st) {
    if (H.ring & 2) {
        if (int e = host_upload_ring(H, h_handles, n, arena_len, d32, st)) {
            cudaStreamSynchronize(st);
            return e;
        }
        if (dh) k_widen32<<<grid_for(n, 256), 256, 0, st>>>(d32, dh, n);
        S5_CUDA(cudaStreamSynchronize(st));
        return 0;
    }
    Pool& pool = Pool::get();
    const uint64_t per = H.piece;
    constexpr int NS = HostPath::kStages;
    std::atomic<bool> bad{false};
    uint64_t ci = 0;
    for (uint64_t off = 0; off < n; off += per, ++ci) {
        const uint64_t len = std::min(per, n - off);
        const int b = static_cast<int>(ci % NS);
        if (ci >= NS) S5_CUDA(cudaEventSynchronize(H.ev[b]));
        uint32_t* s32 = static_cast<uint32_t*>(H.stage[b]);
        const int64_t* src = h_handles + off;
        pool.par_for(len, [&](uint64_t a, uint64_t e) {
            if (narrow_u32(src + a, s32 + a, e - a, arena_len)) bad.store(true, std::memory_order_relaxed);
        });
        S5_CUDA(cudaMemcpyAsync(d32 + off, s32, len * 4, cudaMemcpyHostToDevice, st));
        S5_CUDA(cudaEventRecord(H.ev[b], st));
    }
    if (dh) k_widen32<<<grid_for(n, 256), 256, 0, st>>>(d32, dh, n);
    S5_CUDA(cudaStreamSynchronize(st));
    if (bad.load()) return fail(S5_E_RANGE, "handle outside the arena");
    return 0;
}

// D2H: handles narrowed to u32 and the LCP array to the narrowest width
// holding its maximum on the device, DMA, widened into the caller's arrays
// (chunk i widened while chunk i+1 is in flight)
int host_download(HostPath& H, const int64_t* dh, uint64_t n, const int64_t* dl, uint64_t nl,
                  uint32_t* d32, void* dn, int64_t* h_handles, int64_t* h_lcp, cudaStream_t st,
                  uint64_t* bytes) {
    Pool& pool = Pool::get();
    const uint64_t per = H.piece;
    constexpr int NS = HostPath::kStages;
    if (n) k_shrink<uint32_t><<<grid_for(n, 256), 256, 0, st>>>(dh, d32, n);
    uint32_t w = 8;
    if (dl && h_lcp && nl) {
        S5_CUDA(cudaMemsetAsync(H.dmax, 0, sizeof(unsigned long long), st));
        k_max64<<<grid_for(nl, 256), 256, 0, st>>>(dl, nl, H.dmax);
        S5_CUDA(cudaMemcpyAsync(H.hmax, H.dmax, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
        S5_CUDA(cudaStreamSynchronize(st));
        const unsigned long long mx = *H.hmax;
        w = mx <= 0xFFull ? 1 : mx <= 0xFFFFull ? 2 : mx <= 0xFFFFFFFFull ? 4 : 8;
        const int g = grid_for(nl, 256);
        if (w == 1) k_shrink<uint8_t><<<g, 256, 0, st>>>(dl, static_cast<uint8_t*>(dn), nl);
        if (w == 2) k_shrink<uint16_t><<<g, 256, 0, st>>>(dl, static_cast<uint16_t*>(dn), nl);
        if (w == 4) k_shrink<uint32_t><<<g, 256, 0, st>>>(dl, static_cast<uint32_t*>(dn), nl);
    }
    S5_CUDA(cudaGetLastError());
    if (H.ring & 1) {
        std::vector<RingPiece> rp;
        const uint64_t e4 = H.rP / 4;
        for (uint64_t off = 0; off < n; off += e4)
            rp.push_back({reinterpret_cast<const char*>(d32 + off), h_handles + off, std::min(e4, n - off), 4});
        if (dl && h_lcp && nl) {
            const char* src = w == 8 ? reinterpret_cast<const char*>(dl) : static_cast<const char*>(dn);
            const uint64_t ew = H.rP / w;
            for (uint64_t off = 0; off < nl; off += ew)
                rp.push_back({src + off * w, h_lcp + off, std::min(ew, nl - off), w});
        }
        *bytes = n * 4 + (dl && h_lcp ? nl * w : 0);
        if (rp.empty()) return 0;
        const int e = host_download_ring(H, rp, st);
        S5_CUDA(cudaStreamSynchronize(st));
        return e;
    }
    struct Piece { const char* d; int64_t* h; uint64_t count; uint32_t w; };
    std::vector<Piece> pieces;
    for (uint64_t off = 0; off < n; off += per)
        pieces.push_back({reinterpret_cast<const char*>(d32 + off), h_handles + off,
                          std::min(per, n - off), 4});
    if (dl && h_lcp && nl) {
        const char* src = w == 8 ? reinterpret_cast<const char*>(dl) : static_cast<const char*>(dn);
        for (uint64_t off = 0; off < nl; off += per)
            pieces.push_back({src + off * w, h_lcp + off, std::min(per, nl - off), w});
    }
    *bytes = n * 4 + (dl && h_lcp ? nl * w : 0);
    if (pieces.empty()) return 0;
    auto issue = [&](uint64_t k) -> int {
        int b = static_cast<int>(k % NS);
        S5_CUDA(cudaMemcpyAsync(H.stage[b], pieces[k].d, pieces[k].count * pieces[k].w,
                                cudaMemcpyDeviceToHost, st));
        S5_CUDA(cudaEventRecord(H.ev[b], st));
        return 0;
    };
    for (uint64_t k = 0; k + 1 < NS && k < pieces.size(); ++k)
        if (int e = issue(k)) return e;
    for (uint64_t k = 0; k < pieces.size(); ++k) {
        if (k + NS - 1 < pieces.size())
            if (int e = issue(k + NS - 1)) return e;
        const int b = static_cast<int>(k % NS);
        S5_CUDA(cudaEventSynchronize(H.ev[b]));
        const Piece P = pieces[k];
        const void* sp = H.stage[b];
        pool.par_for(P.count, [&](uint64_t a, uint64_t e) {
            switch (P.w) {
                case 1: widen(static_cast<const uint8_t*>(sp) + a, P.h + a, e - a); break;
                case 2: widen(static_cast<const uint16_t*>(sp) + a, P.h + a, e - a); break;
                case 4: widen(static_cast<const uint32_t*>(sp) + a, P.h + a, e - a); break;
                default: memcpy(P.h + a, static_cast<const int64_t*>(sp) + a, (e - a) * 8);
            }
        });
    }
    S5_CUDA(cudaStreamSynchronize(st));
    return 0;
}

}  // namespace

extern "C" {

int s5_version(void) { return 1; }

const char* s5_last_error(void) { return g_err.c_str(); }

uint64_t s5_workspace_bytes(uint64_t n, uint64_t arena_len, const s5_config* cfg) {
    Cfg c;
    if (resolve(cfg, &c)) return 0;
    if (arena_len >= (1ull << 32)) c.flags |= 8192;  // index mode: + the position table
    return make_layout(n, c).total;
}

static int sort_impl(const uint8_t* d_arena, uint64_t arena_len, int64_t* d_handles, uint64_t n,
                     uint64_t depth, int64_t* d_lcp, const s5_config* cfg, void* d_ws,
                     uint64_t ws_bytes, void* stream_, s5_stats* stats, s5_audit_fn audit,
                     void* audit_user) {
    Cfg c;
    if (int rc = resolve(cfg, &c)) return rc;
    if (stats) memset(stats, 0, sizeof(*stats));
    if (n <= 1) return 0;
    if (!d_arena || !d_handles) return fail(S5_E_INVALID, "null arena or handles");
    if (reinterpret_cast<uintptr_t>(d_arena) % 8)
        return fail(S5_E_INVALID, "device arena must be 8-byte aligned");
    if (arena_len == 0) return fail(S5_E_INVALID, "empty arena with n > 1 handles");
    // arenas of >= 4 GiB (or flags bit13) sort string indices through a
    // position table (SortArgs::pos, index mode)
    if (arena_len >= (1ull << 32)) c.flags |= 8192;
    const bool indexed = (c.flags & 8192) != 0;
    if (indexed && audit) return fail(S5_E_INVALID, "the audit replay is not available in index mode");
    if (arena_len >= (1ull << 32) && (c.flags & 512))
        return fail(S5_E_INVALID, "u32 input offsets (flags bit9) cannot name an arena of >= 4 GiB");
    if (n >= (1ull << 31)) return fail(S5_E_RANGE, "n must be < 2^31");
    if (depth >= arena_len) return fail(S5_E_RANGE, "depth beyond arena");
    Layout L = make_layout(n, c);
    if (!d_ws || ws_bytes < L.total)
        return fail(S5_E_WORKSPACE, "workspace of %llu bytes, need %llu",
                    (unsigned long long)ws_bytes, (unsigned long long)L.total);
    if (int rc = init_attributes()) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream_);
    char* ws = static_cast<char*>(d_ws);
    Pinned& hp = pinned();
    if (!hp.ctl || !hp.seq) return fail(S5_E_CUDA, "pinned host allocation failed");

    // one sort at a time per device (shared side streams); events and the
    // stream drain of an error return handled by the scope
    DevSortLock& dsl = per_device<DevSortLock>();
    std::lock_guard<std::mutex> dev_lock(dsl.mu);
    SortScope scope;
    scope.st = st;
    if (stats) {
        S5_CUDA(cudaEventCreate(&scope.ev0));
        S5_CUDA(cudaEventCreate(&scope.ev1));
        S5_CUDA(cudaEventRecord(scope.ev0, st));
    }
    cudaEvent_t ev0 = scope.ev0, ev1 = scope.ev1;

    SortArgs A{};
    A.arena = d_arena;
    for (int s = 0; s < 2; ++s) {
        A.off[s] = reinterpret_cast<uint32_t*>(ws + L.off[s]);
        A.key[s] = reinterpret_cast<uint64_t*>(ws + L.key[s]);
        A.key2[s] = reinterpret_cast<uint64_t*>(ws + L.key2[s]);
    }
    A.pos = indexed ? reinterpret_cast<int64_t*>(ws + L.pos) : nullptr;
    A.k2_cap = n > c.narrow_max;  // the key2 arrays exist (make_layout)
    {
        int dev = 0, sms = 0;
        S5_CUDA(cudaGetDevice(&dev));
        S5_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        A.sm_count = static_cast<uint32_t>(sms);
        if (const char* e = getenv("S5_SM_ROUND")) A.sm_count = static_cast<uint32_t>(atoi(e));  // tuning
    }
    A.out = d_handles;
    A.lcp = d_lcp;
    A.hint_list = reinterpret_cast<uint2*>(ws + L.hints);
    A.hint_cap = static_cast<uint32_t>(n);
    for (int q = 0; q < NCLS; ++q) A.cap[q] = L.cap[q];
    A.ctl = reinterpret_cast<Ctl*>(ws + L.ctl);
    A.small_max = c.small_max;
    A.local_max = c.local_max;
    A.local_w_max = std::min(c.local_max, kWarpLocalMax);
    A.local_xs_max = std::min(c.local_max, LocalXSCfg::maxn);
    A.local_s_max = std::min(c.local_max, LocalSCfg::maxn);
    A.local_m_max = std::min(c.local_max, LocalMCfg::maxn);
    A.wide_dcap = c.wide_dcap;
    A.local_target = c.local_target;
    A.wide_chunk = kWideChunkMin;
    A.wide_sample = wide_sample_words(c);
    if (const char* e = getenv("S5_WIDE_CHUNK")) A.wide_chunk = std::max(1024, atoi(e));  // tuning
    A.wide_target = std::max<uint32_t>(16, c.wide_target ? c.wide_target : c.local_max / 8);
    A.narrow_max = c.narrow_max;
    A.dmax = c.dmax;
    A.alpha = c.alpha;
    A.flags = c.flags;
    A.seed = c.seed;

    WidePlan P{};
    P.cta_start = reinterpret_cast<uint32_t*>(ws + L.cta_start);
    P.tree_off = reinterpret_cast<uint64_t*>(ws + L.tree_off);
    P.hist_off = reinterpret_cast<uint64_t*>(ws + L.hist_off);
    P.tree_pool = reinterpret_cast<uint64_t*>(ws + L.tree_pool);
    P.hist_pool = reinterpret_cast<uint32_t*>(ws + L.hist_pool);
    P.tree_cap = L.tree_cap;
    P.bkt = reinterpret_cast<uint16_t*>(ws + L.bkt);
    P.hist_cap = L.hist_cap;

    Prof prof;
    prof.on = stats && (c.flags & 2);
    prof.st = st;
    prof.origin = ev0;
    // a wide root (table classifier) gathers its keys inside the level-0 count
    // kernel; otherwise a separate gather pass
    A.arena_len = arena_len;
    const bool fuse_root = !audit && !c.classifier && n > c.narrow_max && !(c.flags & 64);
    // flags bit9: the input is n u32 offsets in the first 4n bytes of d_handles
    // (the multi-GPU exchange payload); every level-0 read of it (tree sample,
    // fused count or k_gather) completes before the first handle is written
    const uint32_t* in32 = (c.flags & 512) ? reinterpret_cast<const uint32_t*>(d_handles) : nullptr;
    unsigned long long fetches_total = 0, hints_total = 0;
    uint32_t level = 0;
    // a second attempt only after a failed root prefix skip (Ctl::skip_fail: the
    // sample's common prefix did not hold for every string; level 0 wrote nothing)
    for (int attempt = 0;; ++attempt) {
    bool retry = false;
    // level 0: cached keys at the common depth, root segment
    int cur = 0;
    for (int q = 0; q < NCLS; ++q) A.next[q] = reinterpret_cast<Seg*>(ws + L.lists[cur][q]);
    S5_CUDA(cudaMemsetAsync(A.ctl, 0, sizeof(Ctl), st));
    A.k2_depth = static_cast<uint32_t>(depth);
    if (!fuse_root) {
        prof.begin(S5_K_GATHER, n);
        k_gather<<<grid_for(n, 256), 256, 0, st>>>(d_handles, in32, static_cast<uint32_t>(n),
                                                    depth, arena_len, A);
        prof.end();
    }
    prof.begin(S5_K_INIT);
    k_init_root<<<1, 32, 0, st>>>(A, static_cast<uint32_t>(n), static_cast<uint32_t>(depth));
    prof.end();
    S5_CUDA(cudaGetLastError());

    fetches_total = hints_total = 0;
    bool wide_before = true;  // the previous level ran S^5 steps (wide or narrow segments)
    for (level = 0;; ++level) {
        prof.level = level;
        A.root = level == 0 && fuse_root && !in32 ? d_handles : nullptr;
        A.root32 = level == 0 && fuse_root ? in32 : nullptr;
        const uint32_t tag = ++hp.next;
        k_publish<<<1, 32, 0, st>>>(A.ctl, hp.ctl, hp.seq, tag);
        ++prof.launches;
        // the wide plan reads this level's segment count on the device, so it
        // runs while the host waits for the published control block
        P.segs = reinterpret_cast<const Seg*>(ws + L.lists[cur][WIDE]);
        P.nsegs = 0;
        prof.begin(S5_K_WIDE_PLAN);
        k_wide_plan<<<1, 1024, 0, st>>>(A, P);
        prof.end();
        // ... and so do the splitter trees: enqueued behind the plan, they are
        // built while the host wakes up, reads the block and launches the rest
        // of the level (the segment count comes from the control block; grid
        // = an upper bound, surplus CTAs return)
        A.k2_stage = fuse_root && level == 0 ? 1u : 0u;
        // (only S^5 steps emit wide children: none can exist behind a level without one)
        const uint32_t tree_ub = level == 0 ? 1u : !wide_before ? 0u
                                                 : std::min<uint32_t>(L.cap[WIDE], kTreeAhead);
        prof.begin(S5_K_WIDE_TREE);
        if (level == 0)  // one segment: its CTA's sample sort is the level's critical path
            k_wide_tree<kTreeThreadsFew><<<1, kTreeThreadsFew, wide_tree_smem(c), st>>>(A, P, 0, 0);
        else if (tree_ub)
            k_wide_tree<kTreeThreads><<<tree_ub, kTreeThreads, wide_tree_smem(c), st>>>(A, P, 0, 0);
        prof.end();
        S5_CUDA(cudaGetLastError());
        if (int e = wait_published(hp, tag, st)) return e;
        Ctl h;
        memcpy(&h, hp.ctl, sizeof(Ctl));
        // second key words: gathered at the root, read at level 1 when the root
        // tree chose to carry them (ctl->k2)
        A.k2_stage = !fuse_root ? 0u : level == 0 ? 1u : (level == 1 && h.k2) ? 2u : 0u;
        if (level == 1 && h.skip_fail) {  // redo the sort without the root prefix skip
            if (attempt) return fail(S5_E_INTERNAL, "root prefix skip failed twice");
            retry = true;
            break;
        }
        if (level == 1) A.k2_depth = static_cast<uint32_t>(depth) + h.skip;  // the root's depth
        if (h.err & ERR_RANGE) return fail(S5_E_RANGE, "handle outside the arena");
        if (h.err & ERR_LIST) return fail(S5_E_INTERNAL, "segment list overflow");
        // plan_err is sticky and must be checked before the `!live` break: the
        // plan of this level's wide segments ran before the host read the
        // block, and when it overflowed (wide_ctas = 0) every wide kernel of
        // the level skipped its work -- the sort must fail, not finish early
        if ((h.err | h.plan_err) & ERR_POOL) return fail(S5_E_INTERNAL, "wide pool overflow");
        fetches_total = h.fetches;
        hints_total = h.hints;
        uint32_t m[NCLS];
        uint64_t live = 0, live_elems = 0;
        for (int q = 0; q < NCLS; ++q) {
            m[q] = h.n_list[q];
            live += m[q];
            live_elems += h.elems[q];
        }
        if (!live) break;
        // every level splits a segment or moves one 8 bytes deeper (a wide
        // segment of strings sharing P more bytes takes P / 8 levels), so the
        // level count is bounded by the splits plus the deepest advance
        if (level >= n + arena_len / 8 + 1024) return fail(S5_E_INTERNAL, "no progress");
        if (audit && level > 0) {
            // debug replay of the reference's audit hook (samplesort.py:235-236, :431-432):
            // the children emitted by the previous level, with both sides' offsets
            std::vector<Seg> hs(live);
            std::vector<uint32_t> side0(n), side1(n);
            uint64_t at = 0;
            for (int q = 0; q < NCLS; ++q) {
                if (m[q])
                    S5_CUDA(cudaMemcpyAsync(hs.data() + at, ws + L.lists[cur][q],
                                            uint64_t(m[q]) * sizeof(Seg), cudaMemcpyDeviceToHost, st));
                at += m[q];
            }
            S5_CUDA(cudaMemcpyAsync(side0.data(), A.off[0], n * 4, cudaMemcpyDeviceToHost, st));
            S5_CUDA(cudaMemcpyAsync(side1.data(), A.off[1], n * 4, cudaMemcpyDeviceToHost, st));
            S5_CUDA(cudaStreamSynchronize(st));
            audit(audit_user, level, reinterpret_cast<const s5_segment*>(hs.data()), hs.size(),
                  side0.data(), side1.data(), n);
        }
        if (stats && level < S5_MAX_LEVELS) {
            stats->wide_elems[level] = h.elems[WIDE];
            stats->narrow_elems[level] = h.elems[NARROW];
            stats->small_elems[level] = h.elems[SMALL];
            stats->local_elems[level] = h.elems[LOCAL] + h.elems[LOCAL_S] + h.elems[LOCAL_M] +
                                        h.elems[LOCAL_XS] + h.elems[LOCAL_W];
            stats->local_steps += m[LOCAL] + m[LOCAL_S] + m[LOCAL_M] + m[LOCAL_XS] + m[LOCAL_W];
            stats->n_per_pass[level] = live_elems;
            stats->wide_steps += m[WIDE];
            stats->narrow_steps += m[NARROW];
            stats->small_segments += m[SMALL];
        }
        // swap lists: this level reads `cur`, emits into the other
        const Seg* segs[NCLS];
        for (int q = 0; q < NCLS; ++q) segs[q] = reinterpret_cast<const Seg*>(ws + L.lists[cur][q]);
        cur ^= 1;
        for (int q = 0; q < NCLS; ++q) A.next[q] = reinterpret_cast<Seg*>(ws + L.lists[cur][q]);
        S5_CUDA(cudaMemsetAsync(A.ctl, 0, offsetof(Ctl, fetches), st));
        Side* sd = prof.on ? nullptr : side_streams();
        bool lane_used[Side::kLanes] = {};
        if (sd) S5_CUDA(cudaEventRecord(sd->fork, st));
        auto lane = [&](int i) -> cudaStream_t {
            if (!sd) return st;
            if (!lane_used[i]) cudaStreamWaitEvent(sd->s[i], sd->fork, 0);
            lane_used[i] = true;
            return sd->s[i];
        };

        wide_before = m[WIDE] + m[NARROW] > 0;
        if (m[WIDE]) {
            P.segs = segs[WIDE];
            P.nsegs = m[WIDE];
            if (m[WIDE] > tree_ub) {  // the trees beyond the launch made ahead of the host read
                prof.begin(S5_K_WIDE_TREE);
                k_wide_tree<kTreeThreads><<<m[WIDE] - tree_ub, kTreeThreads, wide_tree_smem(c), st>>>(
                    A, P, tree_ub, m[WIDE]);
                prof.end();
            }
            // upper bound on CTAs; surplus CTAs exit on ctl->wide_ctas
            uint32_t ub = static_cast<uint32_t>(std::min<uint64_t>(
                uint64_t(m[WIDE]) * kWideCtasMax, n / A.wide_chunk + m[WIDE]));
            const int wsm = wide_smem(c.wide_dcap);
            prof.begin(S5_K_WIDE_COUNT, h.elems[WIDE]);
            // level 0 of a fused root: the tree kernel may have moved the segment
            // behind the sample's common prefix (Ctl::skip) -- the SKIP instantiation
            // checks every string against it, the other one returns at once
            const bool may_skip = level == 0 && fuse_root && !(c.flags & 16384);
            if (c.classifier) {
                k_wide_count<true><<<ub, kWideThreads, wsm, st>>>(A, P);
            } else if (indexed && level == 0) {  // fills the position table
                k_wide_count<false, true><<<ub, kWideThreads, wsm, st>>>(A, P);
                if (may_skip) k_wide_count<false, true, true><<<ub, kWideThreads, wsm, st>>>(A, P);
            } else {
                k_wide_count<false><<<ub, kWideThreads, wsm, st>>>(A, P);
                if (may_skip) k_wide_count<false, false, true><<<ub, kWideThreads, wsm, st>>>(A, P);
            }
            prof.end();
            dim3 cg(m[WIDE], ((2u << std::min(c.dmax, c.wide_dcap)) + 31) / 32);
            prof.begin(S5_K_WIDE_COLSCAN);
            if (m[WIDE] <= 8)  // the root: 8 buckets per CTA, so ~kc/8 CTAs share the rows
                k_wide_colscan_g<32, 8><<<dim3(m[WIDE], cg.y * 4), 1024, 0, st>>>(A, P);
            else if (m[WIDE] <= 32)  // few, large segments: many rows per column
                k_wide_colscan<32><<<cg, 1024, 0, st>>>(A, P);
            else
                k_wide_colscan<8><<<cg, 256, 0, st>>>(A, P);
            prof.end();
            prof.begin(S5_K_WIDE_BSCAN);
            k_wide_bscan<<<m[WIDE], 256, 0, st>>>(A, P);
            prof.end();
            prof.begin(S5_K_WIDE_SCATTER, h.elems[WIDE]);
            // tiles brought in by the bulk-copy engine (one tile in flight while
            // the other is written out) for few huge segments (the root: 4096-string
            // tiles) and for small segments (2048, three CTAs per SM); register-
            // staged 4096-string tiles at two CTAs per SM in between
            if ((c.flags & 32) || m[WIDE] <= 8)
                k_wide_scatter_tma<1024, 4096, kRootStages>
                    <<<ub, 1024, WideTmaSmem<4096, kRootStages>::bytes(c.wide_dcap), st>>>(A, P);
            else if ((c.flags & 128) || h.elems[WIDE] < uint64_t(m[WIDE]) * 32768)  // small segments
                k_wide_scatter_tma<512, 2048>
                    <<<ub, 512, WideTmaSmem<2048>::bytes(c.wide_dcap), st>>>(A, P);
            else
                k_wide_scatter<<<ub, kWideThreads, WideScatterSmem::bytes(c.wide_dcap, A.k2_cap != 0), st>>>(A, P);
            prof.end();
        }
        if (m[NARROW]) {
            prof.begin(S5_K_NARROW, h.elems[NARROW]);
            if (c.classifier)
                k_narrow<true><<<m[NARROW], kNarrowThreads, NarrowSmem::total, lane(6)>>>(A, segs[NARROW]);
            else
                k_narrow<false><<<m[NARROW], kNarrowThreads, NarrowSmem::total, lane(6)>>>(A, segs[NARROW]);
            prof.end();
        }
        if (m[LOCAL_W]) {
            prof.begin(S5_K_LOCAL_W, h.elems[LOCAL_W]);
            k_local_w<<<(m[LOCAL_W] + kWarpLocalWarps - 1) / kWarpLocalWarps, kWarpLocalWarps * 32, 0,
                        lane(5)>>>(A, segs[LOCAL_W], m[LOCAL_W]);
            prof.end();
        }
        if (m[LOCAL_XS]) {
            prof.begin(S5_K_LOCAL_XS, h.elems[LOCAL_XS]);
            if (h.w32)  // high-entropy keys (root sample): 32-bit sort words
                k_local<kLocalXSThreads, true>
                    <<<m[LOCAL_XS], kLocalXSThreads, LocalXSCfg::total, lane(0)>>>(A, segs[LOCAL_XS]);
            else
                k_local<kLocalXSThreads>
                    <<<m[LOCAL_XS], kLocalXSThreads, LocalXSCfg::total, lane(0)>>>(A, segs[LOCAL_XS]);
            prof.end();
        }
        if (m[LOCAL_S]) {
            prof.begin(S5_K_LOCAL_S, h.elems[LOCAL_S]);
            if (h.w32)
                k_local<kLocalSThreads, true>
                    <<<m[LOCAL_S], kLocalSThreads, LocalSCfg::total, lane(1)>>>(A, segs[LOCAL_S]);
            else
                k_local<kLocalSThreads>
                    <<<m[LOCAL_S], kLocalSThreads, LocalSCfg::total, lane(1)>>>(A, segs[LOCAL_S]);
            prof.end();
        }
        if (m[LOCAL_M]) {
            prof.begin(S5_K_LOCAL_M, h.elems[LOCAL_M]);
            k_local<kLocalMThreads>
                <<<m[LOCAL_M], kLocalMThreads, LocalMCfg::total, lane(2)>>>(A, segs[LOCAL_M]);
            prof.end();
        }
        if (m[LOCAL]) {
            prof.begin(S5_K_LOCAL, h.elems[LOCAL]);
            k_local<kLocalThreads>
                <<<m[LOCAL], kLocalThreads, LocalCfg::total, lane(3)>>>(A, segs[LOCAL]);
            prof.end();
        }
        if (m[SMALL]) {
            uint32_t blocks = (m[SMALL] + 7) / 8;
            prof.begin(S5_K_SMALL, h.elems[SMALL]);
            k_small<<<blocks, 256, 0, lane(4)>>>(A, segs[SMALL], m[SMALL]);
            prof.end();
        }
        for (int i = 0; sd && i < Side::kLanes; ++i) {
            if (!lane_used[i]) continue;
            S5_CUDA(cudaEventRecord(sd->join[i], sd->s[i]));
            S5_CUDA(cudaStreamWaitEvent(st, sd->join[i], 0));
        }
        S5_CUDA(cudaGetLastError());
    }
    if (!retry) break;
    c.flags |= 16384;
    A.flags = c.flags;
    }
    if (d_lcp && !(c.flags & 1)) {
        prof.begin(S5_K_LCP_FIX, hints_total);
        if (hints_total)
            k_lcp_fix<<<grid_for(hints_total, 256), 256, 0, st>>>(d_arena, d_handles, d_lcp,
                                                                  A.hint_list, hints_total);
        prof.end();
        S5_CUDA(cudaGetLastError());
    }
    if (stats) {
        S5_CUDA(cudaEventRecord(ev1, st));
        S5_CUDA(cudaEventSynchronize(ev1));
        S5_CUDA(cudaEventElapsedTime(&stats->ms_total, ev0, ev1));
        stats->levels = level;
        stats->key_fetches = fetches_total;
        stats->boundary_lcps = hints_total;
    }
    prof.finish(stats);
    if (stats) stats->n_launch_recs = static_cast<uint32_t>(std::min<size_t>(prof.recs_total, S5_MAX_LAUNCH_RECS));
    scope.ok = true;
    return 0;
}

int s5_sort(const uint8_t* d_arena, uint64_t arena_len, int64_t* d_handles, uint64_t n,
            uint64_t depth, int64_t* d_lcp, const s5_config* cfg, void* d_ws, uint64_t ws_bytes,
            void* stream, s5_stats* stats) {
    return sort_impl(d_arena, arena_len, d_handles, n, depth, d_lcp, cfg, d_ws, ws_bytes, stream,
                     stats, nullptr, nullptr);
}

int s5_sort_audit(const uint8_t* d_arena, uint64_t arena_len, int64_t* d_handles, uint64_t n,
                  uint64_t depth, int64_t* d_lcp, const s5_config* cfg, void* d_ws,
                  uint64_t ws_bytes, void* stream, s5_stats* stats, s5_audit_fn fn, void* user) {
    return sort_impl(d_arena, arena_len, d_handles, n, depth, d_lcp, cfg, d_ws, ws_bytes, stream,
                     stats, fn, user);
}

// Host-buffer entry: handles and LCP move through two pinned staging chunks
// so the host memcpy of chunk i overlaps the DMA of chunk i-1 (H2D) and the
// DMA of chunk i+1 overlaps the copy-out of chunk i (D2H).

// Host-buffer entry.  Offsets are 32-bit (arena < 4 GiB), so the handles
// cross PCIe as u32 (narrowed on the host while they are staged, with the
// range check the device would do) and come back as u32; the LCP array
// comes back in the narrowest of 1/2/4/8 bytes that holds its maximum.
// Host workers narrow/widen chunk i while the DMA of chunk i+-1 runs.
int s5_sort_host(const uint8_t* d_arena, uint64_t arena_len, int64_t* h_handles, uint64_t n,
                 uint64_t depth, int64_t* h_lcp, const s5_config* cfg, void* stream_,
                 s5_stats* stats) {
    HostPath& H = host_path();
    std::lock_guard<std::mutex> lock(H.mu);
    if (n <= 1) {
        if (stats) memset(stats, 0, sizeof(*stats));
        return 0;
    }
    Cfg c;
    if (int rc = resolve(cfg, &c)) return rc;
    // arenas of >= 4 GiB (or flags bit13): int64 handles both ways, index mode
    const bool indexed = arena_len >= (1ull << 32) || (c.flags & 8192);
    if (indexed) c.flags |= 8192;
    uint64_t ws = make_layout(n, c).total;
    uint64_t need = 2 * align_up(n * 8) + 2 * align_up(n * 4) + ws;
    if (need > H.dbytes) {
        if (H.dbuf) cudaFree(H.dbuf);
        H.dbuf = nullptr;
        H.dbytes = 0;
        S5_CUDA(cudaMalloc(&H.dbuf, need));
        H.dbytes = need;
    }
    if (int rc = host_path_init(H)) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream_);
    char* base = static_cast<char*>(H.dbuf);
    int64_t* dh = reinterpret_cast<int64_t*>(base);
    int64_t* dl = reinterpret_cast<int64_t*>(base + align_up(n * 8));
    uint32_t* d32 = reinterpret_cast<uint32_t*>(base + 2 * align_up(n * 8));
    void* dn = base + 2 * align_up(n * 8) + align_up(n * 4);
    void* dws = base + 2 * align_up(n * 8) + 2 * align_up(n * 4);

    // the u32 offsets land in the first 4n bytes of dh and the sort reads them
    // in place (flags bit9: no widening pass, half the root's handle reads)
    s5_config cc{};
    if (cfg) cc = *cfg;
    else cc.seed = 1;
    auto t0 = std::chrono::steady_clock::now();
    if (indexed) {
        cc.flags |= 8192;
        S5_CUDA(cudaMemcpyAsync(dh, h_handles, n * 8, cudaMemcpyHostToDevice, st));
    } else {
        cc.flags |= 512;
        if (int rc = host_upload(H, h_handles, n, arena_len, reinterpret_cast<uint32_t*>(dh), nullptr, st))
            return rc;
    }
    auto t1 = std::chrono::steady_clock::now();
    int rc = s5_sort(d_arena, arena_len, dh, n, depth, h_lcp ? dl : nullptr, &cc, dws, ws,
                     stream_, stats);
    if (rc) return rc;
    S5_CUDA(cudaStreamSynchronize(st));
    auto t2 = std::chrono::steady_clock::now();
    uint64_t d2h_bytes = 0;
    if (indexed) {
        S5_CUDA(cudaMemcpyAsync(h_handles, dh, n * 8, cudaMemcpyDeviceToHost, st));
        if (h_lcp) S5_CUDA(cudaMemcpyAsync(h_lcp, dl, (n - 1) * 8, cudaMemcpyDeviceToHost, st));
        S5_CUDA(cudaStreamSynchronize(st));
        d2h_bytes = n * 8 + (h_lcp ? (n - 1) * 8 : 0);
    } else if (int e = host_download(H, dh, n, h_lcp ? dl : nullptr, n - 1, d32, dn, h_handles, h_lcp,
                                     st, &d2h_bytes)) {
        return e;
    }
    auto t3 = std::chrono::steady_clock::now();
    if (stats) {
        stats->host_h2d_ms = std::chrono::duration<float, std::milli>(t1 - t0).count();
        stats->host_sort_ms = std::chrono::duration<float, std::milli>(t2 - t1).count();
        stats->host_d2h_ms = std::chrono::duration<float, std::milli>(t3 - t2).count();
        stats->host_h2d_bytes = indexed ? n * 8 : n * 4;
        stats->host_d2h_bytes = d2h_bytes;
    }
    return 0;
}

// Host-buffer transfers on their own (the multi-GPU path's shards): the same
// u32 / narrowest-LCP staging as s5_sort_host.
int s5_upload_handles(const int64_t* h_handles, uint64_t n, uint64_t arena_len, int64_t* d_handles,
                      void* stream) {
    HostPath& H = host_path();
    std::lock_guard<std::mutex> lock(H.mu);
    if (n == 0) return 0;
    if (arena_len > 0xFFFFFFFFull) return fail(S5_E_RANGE, "offsets are 32-bit (arena < 4 GiB)");
    if (int rc = host_path_init(H)) return rc;
    if (int rc = host_scratch(H, align_up(n * 4))) return rc;
    return host_upload(H, h_handles, n, arena_len, static_cast<uint32_t*>(H.xbuf), d_handles,
                       static_cast<cudaStream_t>(stream));
}

int s5_download(const int64_t* d_handles, uint64_t n, const int64_t* d_lcp, uint64_t n_lcp,
                int64_t* h_handles, int64_t* h_lcp, void* stream) {
    HostPath& H = host_path();
    std::lock_guard<std::mutex> lock(H.mu);
    if (int rc = host_path_init(H)) return rc;
    if (int rc = host_scratch(H, align_up(n * 4) + align_up(n_lcp * 4))) return rc;
    uint32_t* d32 = static_cast<uint32_t*>(H.xbuf);
    void* dn = static_cast<char*>(H.xbuf) + align_up(n * 4);
    uint64_t bytes = 0;
    return host_download(H, d_handles, n, h_lcp ? d_lcp : nullptr, n_lcp, d32, dn, h_handles, h_lcp,
                         static_cast<cudaStream_t>(stream), &bytes);
}

int s5_pack_keys(const uint8_t* d_arena, uint64_t arena_len, const int64_t* d_handles,
                 uint64_t n, uint64_t depth, uint64_t* d_keys, void* stream) {
    (void)arena_len;
    if (!n) return 0;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    k_pack_keys<<<grid_for(n, 256), 256, 0, st>>>(d_arena, d_handles, n, depth, d_keys);
    S5_CUDA(cudaGetLastError());
    return 0;
}

int s5_adjacent_lcp(const uint8_t* d_arena, uint64_t arena_len, const int64_t* d_sorted,
                    uint64_t n, int64_t* d_lcp, void* stream) {
    (void)arena_len;
    if (n <= 1) return 0;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    k_adjacent_lcp<<<grid_for(n - 1, 256), 256, 0, st>>>(d_arena, d_sorted, n - 1, d_lcp);
    S5_CUDA(cudaGetLastError());
    return 0;
}

int s5_first_unsorted(const uint8_t* d_arena, uint64_t arena_len, const int64_t* d_handles,
                      uint64_t n, int64_t* d_result, void* stream) {
    (void)arena_len;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    S5_CUDA(cudaMemsetAsync(d_result, 0xFF, 8, st));  // -1 == ULLONG_MAX
    if (n <= 1) return 0;
    k_first_unsorted<<<grid_for(n - 1, 256), 256, 0, st>>>(
        d_arena, d_handles, n - 1, reinterpret_cast<unsigned long long*>(d_result));
    S5_CUDA(cudaGetLastError());
    return 0;
}

int s5_partition(const uint8_t* d_arena, uint64_t arena_len, const int64_t* d_handles, uint64_t n,
                 const int64_t* d_splitters, uint32_t nsplit, int64_t* d_out, uint64_t* h_counts,
                 void* stream) {
    (void)arena_len;
    const uint32_t G = nsplit + 1;
    if (G > kPartMaxRanks) return fail(S5_E_INVALID, "at most %u ranks", kPartMaxRanks);
    if (n >= (1ull << 31)) return fail(S5_E_RANGE, "n must be < 2^31");
    if (!h_counts) return fail(S5_E_INVALID, "null counts");
    if (n == 0) {
        for (uint32_t d = 0; d < G; ++d) h_counts[d] = 0;
        return 0;
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (nsplit == 0) {  // one rank: everything stays
        S5_CUDA(cudaMemcpyAsync(d_out, d_handles, n * 8, cudaMemcpyDeviceToDevice, st));
        S5_CUDA(cudaStreamSynchronize(st));
        h_counts[0] = n;
        return 0;
    }
    const uint32_t C = static_cast<uint32_t>(std::min<uint64_t>(1184, std::max<uint64_t>(1, n / 2048)));
    const uint32_t chunk = static_cast<uint32_t>((n + C - 1) / C);
    const uint64_t need = align_up(n * 2) + align_up(uint64_t(C) * G * 4) + align_up(G * 8ull);
    PartScratch& X = per_device<PartScratch>();
    std::lock_guard<std::mutex> lock(X.mu);
    if (need > X.bytes) {
        if (X.d) cudaFree(X.d);
        X.d = nullptr;
        X.bytes = 0;
        S5_CUDA(cudaMalloc(&X.d, need));
        X.bytes = need;
    }
    if (!X.h) S5_CUDA(cudaHostAlloc(&X.h, kPartMaxRanks * 8, cudaHostAllocDefault));
    unsigned long long* h_tot = X.h;
    char* p = static_cast<char*>(X.d);
    uint16_t* dest = reinterpret_cast<uint16_t*>(p);
    uint32_t* rows = reinterpret_cast<uint32_t*>(p + align_up(n * 2));
    auto* tot = reinterpret_cast<unsigned long long*>(p + align_up(n * 2) + align_up(uint64_t(C) * G * 4));
    k_part_count<<<C, kPartThreads, 0, st>>>(d_arena, d_handles, static_cast<uint32_t>(n),
                                             d_splitters, nsplit, chunk, dest, rows);
    k_part_scan<<<1, 1024, 0, st>>>(rows, C, G, tot);
    k_part_scatter<<<C, kPartThreads, 0, st>>>(d_handles, static_cast<uint32_t>(n), chunk, G, dest,
                                               rows, tot, d_out);
    S5_CUDA(cudaGetLastError());
    S5_CUDA(cudaMemcpyAsync(h_tot, tot, G * 8ull, cudaMemcpyDeviceToHost, st));
    S5_CUDA(cudaStreamSynchronize(st));
    for (uint32_t d = 0; d < G; ++d) h_counts[d] = h_tot[d];
    return 0;
}

namespace {
struct AuxScratch {
    std::mutex mu;
    void* d = nullptr;
    uint64_t bytes = 0;
    void* d2 = nullptr;  // materialisation: lengths and prefix sums
    uint64_t bytes2 = 0;
    unsigned long long* h = nullptr;  // pinned: two results
};
AuxScratch& aux() { return per_device<AuxScratch>(); }
int aux_reserve(AuxScratch& X, uint64_t bytes) {
    if (!X.h) S5_CUDA(cudaHostAlloc(&X.h, 16, cudaHostAllocDefault));
    if (bytes <= X.bytes) return 0;
    if (X.d) cudaFree(X.d);
    X.d = nullptr;
    X.bytes = 0;
    S5_CUDA(cudaMalloc(&X.d, bytes));
    X.bytes = bytes;
    return 0;
}
// ordered zero positions of a[0, len) (+ shift) into pos; returns their count
int zero_positions(const uint8_t* a, uint64_t len, int64_t* pos, int64_t shift, char* scratch,
                   unsigned long long* h_tmp, cudaStream_t st, uint64_t* count) {
    const uint64_t blocks = (len + kScanChunk - 1) / kScanChunk;
    auto* counts = reinterpret_cast<uint32_t*>(scratch);
    auto* base = reinterpret_cast<unsigned long long*>(scratch + align_up(blocks * 4));
    k_term_count<1><<<blocks, kScanThreads, 0, st>>>(a, nullptr, len, counts, nullptr);
    k_scan_small<uint32_t><<<1, 1024, 0, st>>>(counts, blocks, base);
    k_term_write<<<blocks, kScanThreads, 0, st>>>(a, len, base, pos, shift);
    S5_CUDA(cudaGetLastError());
    S5_CUDA(cudaMemcpyAsync(h_tmp, base + blocks, 8, cudaMemcpyDeviceToHost, st));
    S5_CUDA(cudaStreamSynchronize(st));
    *count = *h_tmp;
    return 0;
}
uint64_t zero_scratch_bytes(uint64_t len) {
    const uint64_t blocks = (len + kScanChunk - 1) / kScanChunk;
    return align_up(blocks * 4) + align_up((blocks + 1) * 8);
}
// lengths of n strings into d_len: a short SWAR walk, then (only if some
// string is longer than 64 bytes) the ordered terminator compaction + search
int lengths_into(AuxScratch& X, const uint8_t* d_arena, uint64_t arena_len, const int64_t* d_h,
                 uint64_t n, int64_t* d_len, cudaStream_t st) {
    if (int rc = aux_reserve(X, 64)) return rc;
    auto* longer = static_cast<unsigned long long*>(X.d);
    S5_CUDA(cudaMemsetAsync(longer, 0, 8, st));
    // walk cap from the arena bytes per handle (line arenas: a few times the
    // mean string; suffix arenas, ~1 byte per handle: short, then the search);
    // the device arena's pad covers the over-read
    const uint64_t per = (arena_len / std::max<uint64_t>(n, 1) + 7) / 8;
    const uint32_t words = static_cast<uint32_t>(std::min<uint64_t>(14, 2 + 2 * per));
    k_lengths_walk<<<grid_for(n, 256), 256, 0, st>>>(d_arena, d_h, n, words, d_len, longer);
    S5_CUDA(cudaMemcpyAsync(X.h, longer, 8, cudaMemcpyDeviceToHost, st));
    S5_CUDA(cudaStreamSynchronize(st));
    if (X.h[0] == 0) return 0;
    const uint64_t zs = zero_scratch_bytes(arena_len);
    if (int rc = aux_reserve(X, zs + align_up(arena_len * 8))) return rc;
    char* scratch = static_cast<char*>(X.d);
    auto* pos = reinterpret_cast<int64_t*>(scratch + zs);
    uint64_t z = 0;
    if (int rc = zero_positions(d_arena, arena_len, pos, 0, scratch, X.h, st, &z)) return rc;
    k_lengths<<<grid_for(n, 256), 256, 0, st>>>(d_h, n, pos, z, d_len);
    S5_CUDA(cudaGetLastError());
    return 0;
}
}  // namespace

int s5_ingest_lines(const uint8_t* d_raw, uint64_t len, uint8_t* d_arena, int64_t* d_handles,
                    uint64_t* h_n, uint64_t* h_arena_len, int64_t* h_nul_offset, void* stream) {
    if (!h_n || !h_arena_len || !h_nul_offset) return fail(S5_E_INVALID, "null result pointer");
    *h_n = 0;
    *h_arena_len = 0;
    *h_nul_offset = -1;
    if (len == 0) return 0;
    if (len >= 0xFFFFFFFFull) return fail(S5_E_RANGE, "input of %llu bytes: offsets are 32-bit",
                                         static_cast<unsigned long long>(len));
    AuxScratch& X = aux();
    std::lock_guard<std::mutex> lock(X.mu);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const uint64_t blocks = (len + kScanChunk - 1) / kScanChunk;
    if (int rc = aux_reserve(X, zero_scratch_bytes(len) + 16)) return rc;
    char* scratch = static_cast<char*>(X.d);
    auto* counts = reinterpret_cast<uint32_t*>(scratch);
    auto* base = reinterpret_cast<unsigned long long*>(scratch + align_up(blocks * 4));
    auto* nul = reinterpret_cast<unsigned long long*>(scratch + zero_scratch_bytes(len));
    S5_CUDA(cudaMemsetAsync(nul, 0xFF, 8, st));
    // newlines -> terminators, counted per CTA; the first embedded 0 recorded
    k_term_count<0><<<blocks, kScanThreads, 0, st>>>(d_raw, d_arena, len, counts, nul);
    k_scan_small<uint32_t><<<1, 1024, 0, st>>>(counts, blocks, base);
    // string k+1 starts right after terminator k; string 0 at offset 0
    S5_CUDA(cudaMemsetAsync(d_handles, 0, 8, st));
    k_term_write<<<blocks, kScanThreads, 0, st>>>(d_arena, len, base, d_handles + 1, 1);
    S5_CUDA(cudaGetLastError());
    S5_CUDA(cudaMemcpyAsync(X.h, nul, 8, cudaMemcpyDeviceToHost, st));
    S5_CUDA(cudaMemcpyAsync(X.h + 1, base + blocks, 8, cudaMemcpyDeviceToHost, st));
    uint8_t last = 0;
    S5_CUDA(cudaMemcpyAsync(&last, d_raw + len - 1, 1, cudaMemcpyDeviceToHost, st));
    S5_CUDA(cudaStreamSynchronize(st));
    if (X.h[0] != ~0ull) {
        *h_nul_offset = static_cast<int64_t>(X.h[0]);
        return fail(S5_E_INVALID, "input contains byte 0 at offset %llu", X.h[0]);
    }
    uint64_t nterm = X.h[1];
    uint64_t alen = len;
    if (last != '\n') {  // the last line has no newline: append its terminator
        S5_CUDA(cudaMemsetAsync(d_arena + len, 0, 1, st));
        ++nterm;
        ++alen;
    }
    S5_CUDA(cudaStreamSynchronize(st));
    *h_n = nterm;
    *h_arena_len = alen;
    return 0;
}

int s5_string_lengths(const uint8_t* d_arena, uint64_t arena_len, const int64_t* d_handles,
                      uint64_t n, int64_t* d_len, void* stream) {
    if (n == 0) return 0;
    AuxScratch& X = aux();
    std::lock_guard<std::mutex> lock(X.mu);
    return lengths_into(X, d_arena, arena_len, d_handles, n, d_len, static_cast<cudaStream_t>(stream));
}

int s5_materialize(const uint8_t* d_arena, uint64_t arena_len, const int64_t* d_sorted, uint64_t n,
                   uint8_t* d_out, uint64_t out_cap, int64_t* d_out_handles, uint64_t* h_out_len,
                   void* stream) {
    if (!h_out_len) return fail(S5_E_INVALID, "null result pointer");
    *h_out_len = 0;
    if (n == 0) return 0;
    AuxScratch& X = aux();
    std::lock_guard<std::mutex> lock(X.mu);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const uint64_t nb = (n + 1023) / 1024;
    // lengths and prefix sums in their own buffer (lengths_into reuses the aux scratch)
    const uint64_t need = align_up(n * 8) + align_up(nb * 8) + align_up((nb + 1) * 8);
    if (need > X.bytes2) {
        if (X.d2) cudaFree(X.d2);
        X.d2 = nullptr;
        X.bytes2 = 0;
        S5_CUDA(cudaMalloc(&X.d2, need));
        X.bytes2 = need;
    }
    auto* len = static_cast<int64_t*>(X.d2);
    auto* tot = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(len) + align_up(n * 8));
    auto* bb = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(tot) + align_up(nb * 8));
    if (int rc = lengths_into(X, d_arena, arena_len, d_sorted, n, len, st)) return rc;
    // exclusive prefix of (length + 1): the new handles
    k_scan_len_block<<<nb, 1024, 0, st>>>(len, n, d_out_handles, tot);
    k_scan_small<unsigned long long><<<1, 1024, 0, st>>>(tot, nb, bb);
    k_scan_len_add<<<grid_for(n, 256), 256, 0, st>>>(d_out_handles, n, bb);
    S5_CUDA(cudaGetLastError());
    S5_CUDA(cudaMemcpyAsync(X.h, bb + nb, 8, cudaMemcpyDeviceToHost, st));
    S5_CUDA(cudaStreamSynchronize(st));
    *h_out_len = X.h[0];
    if (X.h[0] > out_cap)
        return fail(S5_E_WORKSPACE, "output of %llu bytes, capacity %llu", X.h[0],
                    static_cast<unsigned long long>(out_cap));
    k_gather_strings<<<grid_for(n * 32, 256), 256, 0, st>>>(d_arena, d_sorted, len, d_out_handles, n,
                                                            d_out);
    S5_CUDA(cudaGetLastError());
    return 0;
}

int s5_classify(const uint64_t* d_keys, uint64_t n, const uint64_t* d_in_order, uint32_t v,
                uint32_t classifier, uint16_t* d_buckets, void* stream) {
    uint32_t d = 0;
    while (d < 31 && ((1u << d) - 1) < v) ++d;
    if (v < 1 || ((1u << d) - 1) != v || d > kMaxTreeD)
        return fail(S5_E_INVALID, "need 2**d - 1 splitters (d <= %u), got %u", kMaxTreeD, v);
    if (classifier > 2) return fail(S5_E_INVALID, "classifier must be 0, 1 or 2");
    if (!n) return 0;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int smem = (1 << d) * 8 * 2 + (kLutCells + 1) * 2 + 16;
    if (smem > 48 * 1024) {
        if (int rc = set_smem(k_classify<0>, smem)) return rc;
        if (int rc = set_smem(k_classify<1>, smem)) return rc;
        if (int rc = set_smem(k_classify<2>, smem)) return rc;
    }
    const int g = grid_for(n, 256, 296);
    if (classifier == 1)
        k_classify<1><<<g, 256, smem, st>>>(d_keys, n, d_in_order, d, d_buckets);
    else if (classifier == 2)
        k_classify<2><<<g, 256, smem, st>>>(d_keys, n, d_in_order, d, d_buckets);
    else
        k_classify<0><<<g, 256, smem, st>>>(d_keys, n, d_in_order, d, d_buckets);
    S5_CUDA(cudaGetLastError());
    return 0;
}

int s5_build_tree(const uint64_t* d_sorted_sample, uint32_t m, uint32_t v,
                  uint64_t* d_level_order, uint64_t* d_in_order, void* stream) {
    uint32_t d = 0;
    while (d < 31 && ((1u << d) - 1) < v) ++d;
    if (v < 1 || ((1u << d) - 1) != v || d > kMaxTreeD)
        return fail(S5_E_INVALID, "need 2**d - 1 splitters (d <= %u), got %u", kMaxTreeD, v);
    if (m < 1) return fail(S5_E_INVALID, "empty sample");
    uint64_t smem = uint64_t(m) * 8 + (uint64_t(1) << d) * 12;
    if (smem > 227 * 1024) return fail(S5_E_INVALID, "sample too large for one CTA");
    if (int rc = init_attributes()) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    k_build_tree<<<1, 1024, smem, st>>>(d_sorted_sample, m, d, d_level_order, d_in_order);
    S5_CUDA(cudaGetLastError());
    return 0;
}

int s5_host_markov_text(const double* cdf, const double* u, uint64_t n, uint32_t sigma,
                        uint8_t* out) {
    if (sigma < 1 || sigma > 255) return fail(S5_E_INVALID, "sigma must be in [1, 255]");
    uint32_t a = 0, b = sigma > 1 ? 1 : 0;  // virtual sym[-2] = 0, sym[-1] = 1
    const uint64_t row = sigma;
    for (uint64_t i = 0; i < n; ++i) {
        const double* c = cdf + (uint64_t(a) * sigma + b) * row;
        double x = u[i];
        uint32_t lo = 0, hi = sigma;  // smallest s with c[s] >= x
        while (lo < hi) {
            uint32_t mid = (lo + hi) >> 1;
            if (c[mid] >= x) hi = mid; else lo = mid + 1;
        }
        uint32_t s = lo < sigma ? lo : sigma - 1;
        out[i] = static_cast<uint8_t>(0x40 + s);
        a = b;
        b = s;
    }
    return 0;
}

int s5_host_copy_pieces(uint8_t* dst, const int64_t* dst_start, const int64_t* src_start,
                        const int64_t* lengths, const uint8_t* blob, uint64_t m) {
    Pool::get().par_for(m, [&](uint64_t a, uint64_t b) {
        for (uint64_t i = a; i < b; ++i)
            memcpy(dst + dst_start[i], blob + src_start[i], static_cast<size_t>(lengths[i]));
    });
    return 0;
}

static void (*g_multi_release)() = nullptr;  // set by s5_multi.cuh

int s5_release_caches(void) {
    int cur = 0;
    cudaGetDevice(&cur);
    if (g_multi_release) g_multi_release();
    std::lock_guard<std::mutex> g(registry_mutex());
    for (auto& kv : registry<HostPath>()) {
        HostPath& H = kv.second;
        std::lock_guard<std::mutex> l(H.mu);
        cudaSetDevice(kv.first);
        if (H.dbuf) cudaFree(H.dbuf);
        if (H.xbuf) cudaFree(H.xbuf);
        if (H.dmax) cudaFree(H.dmax);
        if (H.hmax) cudaFreeHost(H.hmax);
        for (int i = 0; i < HostPath::kStages; ++i) {
            if (H.stage[i]) cudaFreeHost(H.stage[i]);
            if (H.ev[i]) cudaEventDestroy(H.ev[i]);
            H.stage[i] = nullptr;
            H.ev[i] = nullptr;
        }
        H.dbuf = H.xbuf = nullptr;
        H.dbytes = H.xbytes = 0;
        H.dmax = nullptr;
        H.hmax = nullptr;
    }
    for (auto& kv : registry<AuxScratch>()) {
        AuxScratch& X = kv.second;
        std::lock_guard<std::mutex> l(X.mu);
        cudaSetDevice(kv.first);
        if (X.d) cudaFree(X.d);
        if (X.d2) cudaFree(X.d2);
        if (X.h) cudaFreeHost(X.h);
        X.d = X.d2 = nullptr;
        X.h = nullptr;
        X.bytes = X.bytes2 = 0;
    }
    for (auto& kv : registry<PartScratch>()) {
        PartScratch& X = kv.second;
        std::lock_guard<std::mutex> l(X.mu);
        cudaSetDevice(kv.first);
        if (X.d) cudaFree(X.d);
        if (X.h) cudaFreeHost(X.h);
        X.d = nullptr;
        X.h = nullptr;
        X.bytes = 0;
    }
    for (auto& kv : registry<Side>()) {
        Side& sd = kv.second;
        if (!sd.ok) continue;
        cudaSetDevice(kv.first);
        for (int i = 0; i < Side::kLanes; ++i) {
            cudaStreamDestroy(sd.s[i]);
            cudaEventDestroy(sd.join[i]);
        }
        cudaEventDestroy(sd.fork);
        sd = Side{};
    }
    cudaSetDevice(cur);
    return 0;
}

}  // extern "C"

#include "s5_multi.cuh"
