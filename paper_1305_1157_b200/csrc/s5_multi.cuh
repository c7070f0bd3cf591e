// s5_sort_multi: the p-way split of pS^5 (samplesort.py:369-434, :437-444)
// with p = GPUs of one process.  Included at the end of
// s5_api.cu: composes the library's own entry points (s5_partition, s5_sort,
// s5_adjacent_lcp) with peer copies over NVLink; one host thread per shard.
#pragma once

#include <atomic>
#include <chrono>
#include <string>
#include <thread>

namespace {

constexpr uint32_t kMultiMaxGpus = 64;      // one host thread per shard
constexpr uint32_t kMultiOversample = 64;   // samples per shard and destination ...
constexpr uint32_t kMultiMinSamples = 2048;  // ... and at least this many per shard (slice balance)

__device__ __forceinline__ uint64_t multi_mix(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

// s sample handles of one shard, drawn by a hash of (seed, slot).
__global__ void k_multi_sample(const int64_t* __restrict__ h, uint64_t n, uint32_t s, uint64_t seed,
                               int64_t* __restrict__ out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < s) out[i] = h[multi_mix(seed + i) % n];
}

// same[i]: sorted sample strings i and i+1 are identical (both end right
// behind their common prefix).
__global__ void k_multi_same(const uint8_t* __restrict__ arena, const int64_t* __restrict__ s,
                             const int64_t* __restrict__ lcp, uint32_t m, uint8_t* __restrict__ same) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i + 1 < m) same[i] = arena[s[i] + lcp[i]] == 0 && arena[s[i + 1] + lcp[i]] == 0;
}

// The exchange payload: int64 arena offsets below 4 GiB cross NVLink as u32.
__global__ void k_multi_narrow(const int64_t* __restrict__ in, uint64_t n, uint32_t* __restrict__ out) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += stride)
        out[i] = static_cast<uint32_t>(in[i]);
}

struct MultiSlot {  // device scratch of shard g, kept between calls
    int dev = -1;
    void* d = nullptr;
    uint64_t bytes = 0;
    void* ws = nullptr;
    uint64_t ws_bytes = 0;
};
struct MultiState {
    std::mutex mu;  // one s5_sort_multi at a time
    MultiSlot slot[kMultiMaxGpus];
    MultiSlot samp;  // the sample sort's scratch on devices[0] (d only)
};
MultiState& multi_state() {
    static MultiState s;
    return s;
}
int multi_reserve(void** p, uint64_t* have, uint64_t need) {
    if (need <= *have && *p) return 0;
    if (*p) cudaFree(*p);
    *p = nullptr;
    *have = 0;
    S5_CUDA(cudaMalloc(p, need ? need : 16));
    *have = need ? need : 16;
    return 0;
}

void multi_release() {
    MultiState& M = multi_state();
    std::lock_guard<std::mutex> lock(M.mu);
    for (MultiSlot& X : M.slot) {
        if (X.dev >= 0) cudaSetDevice(X.dev);
        if (X.d) cudaFree(X.d);
        if (X.ws) cudaFree(X.ws);
        X = MultiSlot{};
    }
    if (M.samp.d) {
        cudaSetDevice(M.samp.dev);
        cudaFree(M.samp.d);
    }
    M.samp = MultiSlot{};
}
const bool g_multi_release_set = (g_multi_release = multi_release, true);

// One persistent host thread per shard slot (a thread keeps its device's
// per-thread library state -- the mapped control block of s5_sort -- between
// calls instead of allocating it per call).  run(G, devices, fn) executes
// fn(g) on thread g with devices[g] current; the first failure's code and
// message are re-raised on the calling thread.  Threads are detached and the
// pool is never destroyed (no join at process exit).
struct MultiPool {
    std::mutex mu;
    std::condition_variable go, done;
    std::function<int(int)> job;
    const int* devices = nullptr;
    uint64_t gen = 0;
    int G = 0, left = 0, nthreads = 0;
    std::vector<int> rc;
    std::vector<std::string> msg;

    void worker(int g, uint64_t seen) {
        for (;;) {
            std::unique_lock<std::mutex> lk(mu);
            go.wait(lk, [&] { return gen != seen; });
            seen = gen;
            if (g >= G) continue;  // not part of this job
            const std::function<int(int)> f = job;
            const int dev = devices[g];
            lk.unlock();
            int r = 0;
            std::string m;
            if (cudaSetDevice(dev) != cudaSuccess) {
                r = S5_E_CUDA;
                m = "cudaSetDevice failed";
            } else {
                r = f(g);
                if (r) m = s5_last_error();
            }
            lk.lock();
            rc[g] = r;
            msg[g] = m;
            if (--left == 0) done.notify_all();
        }
    }
    int run(int G_, const int* devs, std::function<int(int)> f) {
        std::unique_lock<std::mutex> lk(mu);
        for (; nthreads < G_; ++nthreads) std::thread(&MultiPool::worker, this, nthreads, gen).detach();
        G = G_;
        devices = devs;
        job = std::move(f);
        rc.assign(G_, 0);
        msg.assign(G_, std::string());
        left = G_;
        ++gen;
        go.notify_all();
        done.wait(lk, [&] { return left == 0; });
        job = nullptr;
        for (int g = 0; g < G_; ++g)
            if (rc[g]) return fail(rc[g], "shard %d (device %d): %s", g, devs[g], msg[g].c_str());
        return 0;
    }
};
MultiPool& multi_pool() {
    static MultiPool* p = new MultiPool;
    return *p;
}
template <class F>
int multi_par(int G, const int* devices, F fn) {
    return multi_pool().run(G, devices, std::function<int(int)>(fn));
}

}  // namespace

extern "C" int s5_sort_multi(int n_gpus, const int* devices, const uint8_t* const* d_arenas,
                             uint64_t arena_len, int64_t* const* d_handle_shards,
                             const uint64_t* shard_n, int64_t* const* d_out_handles,
                             int64_t* const* d_out_lcp, const uint64_t* out_capacity,
                             uint64_t* out_counts, const s5_config* cfg, s5_stats* stats) {
    if (n_gpus < 1 || uint32_t(n_gpus) > kMultiMaxGpus)
        return fail(S5_E_INVALID, "n_gpus must be in 1..%u", kMultiMaxGpus);
    if (!devices || !d_arenas || !d_handle_shards || !shard_n || !d_out_handles || !out_capacity ||
        !out_counts)
        return fail(S5_E_INVALID, "null argument");
    const int G = n_gpus;
    const auto t0 = std::chrono::steady_clock::now();
    int cur = 0;
    S5_CUDA(cudaGetDevice(&cur));
    struct Restore {
        int d;
        ~Restore() { cudaSetDevice(d); }
    } restore{cur};
    MultiState& M = multi_state();
    std::lock_guard<std::mutex> lock(M.mu);

    const bool trace = getenv("S5_MULTI_TRACE") != nullptr;  // phase wall times on stderr
    auto mark = [&](const char* what) {
        if (trace)
            fprintf(stderr, "s5_sort_multi %-10s %8.3f ms\n", what,
                    std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - t0).count());
    };
    uint64_t total = 0;
    for (int g = 0; g < G; ++g) {
        if (shard_n[g] >= (1ull << 31)) return fail(S5_E_RANGE, "shard %d: n must be < 2^31", g);
        total += shard_n[g];
        out_counts[g] = 0;
    }
    if (stats) *stats = s5_stats{};
    if (total == 0) return 0;
    if (G == 1) {  // one device: nothing to split or exchange
        const uint64_t n = shard_n[0];
        if (n > out_capacity[0])
            return fail(S5_E_WORKSPACE, "slice 0 holds %llu strings, capacity %llu",
                        (unsigned long long)n, (unsigned long long)out_capacity[0]);
        S5_CUDA(cudaSetDevice(devices[0]));
        MultiSlot& X = M.slot[0];
        if (X.dev != devices[0]) {
            if (X.dev >= 0) cudaSetDevice(X.dev);
            if (X.d) cudaFree(X.d);
            if (X.ws) cudaFree(X.ws);
            S5_CUDA(cudaSetDevice(devices[0]));
            X = MultiSlot{};
            X.dev = devices[0];
        }
        S5_CUDA(cudaMemcpyAsync(d_out_handles[0], d_handle_shards[0], n * 8, cudaMemcpyDeviceToDevice,
                                nullptr));
        if (n > 1) {
            const uint64_t wsb = s5_workspace_bytes(n, arena_len, cfg);
            if (int r = multi_reserve(&X.ws, &X.ws_bytes, wsb)) return r;
            if (int r = s5_sort(d_arenas[0], arena_len, d_out_handles[0], n, 0,
                                d_out_lcp ? d_out_lcp[0] : nullptr, cfg, X.ws, X.ws_bytes, nullptr, stats))
                return r;
        }
        S5_CUDA(cudaDeviceSynchronize());
        out_counts[0] = n;
        if (stats)
            stats->ms_total =
                std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - t0).count();
        return 0;
    }
    const bool narrow = arena_len < (1ull << 32);  // u32 payload; index-mode arenas send int64
    const uint32_t S = std::max(kMultiOversample * uint32_t(G), kMultiMinSamples);  // samples per shard
    const uint32_t nsplit = uint32_t(G) - 1;
    s5_config c = cfg ? *cfg : s5_config{};
    const uint64_t seed = c.seed ? c.seed : 1;

    // Scratch per shard: [samples S] [splitters G-1] [pair 2] [grouped n_g] [payload n_g]
    auto off_spl = [&](void* d) { return static_cast<int64_t*>(d) + S; };
    auto off_pair = [&](void* d) { return static_cast<int64_t*>(d) + S + kMultiMaxGpus; };
    auto off_grp = [&](void* d) { return static_cast<int64_t*>(d) + S + kMultiMaxGpus + 2; };
    for (int g = 0; g < G; ++g) {
        MultiSlot& X = M.slot[g];
        S5_CUDA(cudaSetDevice(devices[g]));
        if (X.dev != devices[g]) {  // the slot moved to another device
            if (X.d || X.ws) {
                if (X.dev >= 0) cudaSetDevice(X.dev);
                if (X.d) cudaFree(X.d);
                if (X.ws) cudaFree(X.ws);
                S5_CUDA(cudaSetDevice(devices[g]));
            }
            X = MultiSlot{};
            X.dev = devices[g];
        }
        const uint64_t need = (uint64_t(S) + kMultiMaxGpus + 2 + 2 * shard_n[g]) * 8 + 64;
        if (int rc = multi_reserve(&X.d, &X.bytes, need)) return rc;
    }

    // direct NVLink copies between distinct devices (otherwise cudaMemcpyPeer
    // stages through the host); already-enabled pairs are fine
    for (int a = 0; a < G; ++a)
        for (int b = 0; b < G; ++b) {
            if (devices[a] == devices[b]) continue;
            bool seen = false;  // each ordered pair once
            for (int k = 0; k < b && !seen; ++k) seen = devices[k] == devices[b];
            for (int k = 0; k < a && !seen; ++k) seen = devices[k] == devices[a];
            if (seen) continue;
            int can = 0;
            if (cudaDeviceCanAccessPeer(&can, devices[a], devices[b]) != cudaSuccess || !can) {
                cudaGetLastError();
                continue;
            }
            S5_CUDA(cudaSetDevice(devices[a]));
            const cudaError_t e = cudaDeviceEnablePeerAccess(devices[b], 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
                return fail(S5_E_CUDA, "cudaDeviceEnablePeerAccess(%d -> %d): %s", devices[a],
                            devices[b], cudaGetErrorString(e));
            cudaGetLastError();
        }

    // 1. samples of every non-empty shard -> host -> first device
    std::vector<int64_t> samp;
    samp.reserve(uint64_t(S) * G);
    for (int g = 0; g < G; ++g) {
        if (!shard_n[g]) continue;
        S5_CUDA(cudaSetDevice(devices[g]));
        int64_t* d_s = static_cast<int64_t*>(M.slot[g].d);
        k_multi_sample<<<(S + 255) / 256, 256>>>(d_handle_shards[g], shard_n[g], S,
                                                 seed * 1000003ull + uint64_t(g) * S, d_s);
        S5_CUDA(cudaGetLastError());
        const size_t at = samp.size();
        samp.resize(at + S);
        S5_CUDA(cudaMemcpy(samp.data() + at, d_s, S * 8ull, cudaMemcpyDeviceToHost));
    }
    mark("samples");
    // 2. splitters: G-1 evenly spaced strings of the (string, handle)-sorted sample
    std::vector<int64_t> spl(nsplit);
    if (nsplit) {
        const uint32_t m = static_cast<uint32_t>(samp.size());
        S5_CUDA(cudaSetDevice(devices[0]));
        // [sample m] [lcp m] [same m] [workspace], kept between calls
        const uint64_t wsb = s5_workspace_bytes(m, arena_len, &c);
        MultiSlot& T = M.samp;
        if (T.dev != devices[0]) {
            if (T.d) {
                cudaSetDevice(T.dev);
                cudaFree(T.d);
                S5_CUDA(cudaSetDevice(devices[0]));
            }
            T = MultiSlot{};
            T.dev = devices[0];
        }
        if (int r = multi_reserve(&T.d, &T.bytes, align_up(m * 8ull) * 2 + align_up(m) + wsb + 256))
            return r;
        void* d_tmp = T.d;
        int64_t* d_s = static_cast<int64_t*>(d_tmp);
        int64_t* d_l = reinterpret_cast<int64_t*>(static_cast<char*>(d_tmp) + align_up(m * 8ull));
        uint8_t* d_same = reinterpret_cast<uint8_t*>(static_cast<char*>(d_tmp) + 2 * align_up(m * 8ull));
        void* d_ws = static_cast<char*>(d_tmp) + 2 * align_up(m * 8ull) + align_up(m);
        S5_CUDA(cudaMemcpy(d_s, samp.data(), m * 8ull, cudaMemcpyHostToDevice));
        if (int rc = s5_sort(d_arenas[0], arena_len, d_s, m, 0, d_l, &c, d_ws, wsb, nullptr, nullptr))
            return rc;
        k_multi_same<<<(m + 255) / 256, 256>>>(d_arenas[0], d_s, d_l, m, d_same);
        S5_CUDA(cudaGetLastError());
        std::vector<uint8_t> same(m);
        S5_CUDA(cudaMemcpy(samp.data(), d_s, m * 8ull, cudaMemcpyDeviceToHost));
        S5_CUDA(cudaMemcpy(same.data(), d_same, m - 1, cudaMemcpyDeviceToHost));
        // identical strings order by handle, so the splitter list is
        // non-decreasing in s5_partition's (string, handle) order
        for (uint32_t a = 0; a < m;) {
            uint32_t b = a;
            while (b + 1 < m && same[b]) ++b;
            if (b > a) std::sort(samp.begin() + a, samp.begin() + b + 1);
            a = b + 1;
        }
        for (uint32_t j = 0; j < nsplit; ++j)
            spl[j] = samp[std::min<uint64_t>(uint64_t(j + 1) * m / G, m - 1)];
    }

    mark("splitters");
    // 3. group every shard by destination; 4. payload ready for the peers
    std::vector<uint64_t> counts(uint64_t(G) * G, 0);  // counts[src * G + dst]
    int rc = multi_par(G, devices, [&](int g) -> int {
        const uint64_t n = shard_n[g];
        if (!n) return 0;
        MultiSlot& X = M.slot[g];
        int64_t* d_spl = off_spl(X.d);
        int64_t* d_grp = off_grp(X.d);
        if (nsplit) S5_CUDA(cudaMemcpy(d_spl, spl.data(), nsplit * 8ull, cudaMemcpyHostToDevice));
        if (int r = s5_partition(d_arenas[g], arena_len, d_handle_shards[g], n, d_spl, nsplit, d_grp,
                                 &counts[uint64_t(g) * G], nullptr))
            return r;
        if (narrow) {
            uint32_t* d_pay = reinterpret_cast<uint32_t*>(d_grp + n);
            k_multi_narrow<<<static_cast<unsigned>(std::min<uint64_t>((n + 1023) / 1024, 1184)), 256>>>(
                d_grp, n, d_pay);
            S5_CUDA(cudaGetLastError());
        }
        S5_CUDA(cudaDeviceSynchronize());
        return 0;
    });
    if (rc) return rc;
    std::vector<uint64_t> sizes(G, 0);
    for (int d = 0; d < G; ++d) {
        for (int g = 0; g < G; ++g) sizes[d] += counts[uint64_t(g) * G + d];
        if (sizes[d] > out_capacity[d])
            return fail(S5_E_WORKSPACE, "slice %d holds %llu strings, capacity %llu", d,
                        (unsigned long long)sizes[d], (unsigned long long)out_capacity[d]);
        if (sizes[d] >= (1ull << 31)) return fail(S5_E_RANGE, "slice %d: n must be < 2^31", d);
    }

    mark("partition");
    // 5. exchange (peer copies into the destination's output buffer) and local sorts
    std::vector<s5_stats> st(stats ? G : 0);
    rc = multi_par(G, devices, [&](int d) -> int {
        const uint64_t m = sizes[d];
        if (!m) return 0;
        MultiSlot& X = M.slot[d];
        const uint64_t esz = narrow ? 4 : 8;
        char* dst = reinterpret_cast<char*>(d_out_handles[d]);
        uint64_t at = 0;
        for (int g = 0; g < G; ++g) {
            const uint64_t cnt = counts[uint64_t(g) * G + d];
            if (!cnt) continue;
            uint64_t lo = 0;
            for (int k = 0; k < d; ++k) lo += counts[uint64_t(g) * G + k];
            const int64_t* grp = off_grp(M.slot[g].d);
            const char* src = narrow ? reinterpret_cast<const char*>(grp + shard_n[g]) + lo * 4
                                     : reinterpret_cast<const char*>(grp + lo);
            S5_CUDA(cudaMemcpyPeerAsync(dst + at * esz, devices[d], src, devices[g], cnt * esz, nullptr));
            at += cnt;
        }
        S5_CUDA(cudaDeviceSynchronize());
        if (m == 1) {
            if (narrow) {
                uint32_t v = 0;
                S5_CUDA(cudaMemcpy(&v, dst, 4, cudaMemcpyDeviceToHost));
                const int64_t w = v;
                S5_CUDA(cudaMemcpy(dst, &w, 8, cudaMemcpyHostToDevice));
            }
            return 0;
        }
        s5_config cc = c;
        if (narrow) cc.flags |= 512u;  // bit9: u32 offsets in, int64 handles out
        const uint64_t wsb = s5_workspace_bytes(m, arena_len, &cc);
        if (int r = multi_reserve(&X.ws, &X.ws_bytes, wsb)) return r;
        if (int r = s5_sort(d_arenas[d], arena_len, d_out_handles[d], m, 0,
                            d_out_lcp ? d_out_lcp[d] : nullptr, &cc, X.ws, X.ws_bytes, nullptr,
                            stats ? &st[d] : nullptr))
            return r;
        S5_CUDA(cudaDeviceSynchronize());
        return 0;
    });
    if (rc) return rc;

    mark("sorts");
    // 6. the LCP across each slice boundary, on the left device
    if (d_out_lcp) {
        for (int d = 0; d < G; ++d) {
            if (!sizes[d]) continue;
            int nxt = -1;
            for (int r = d + 1; r < G && nxt < 0; ++r)
                if (sizes[r]) nxt = r;
            if (nxt < 0) break;
            if (!d_out_lcp[d])
                return fail(S5_E_INVALID, "null LCP buffer for slice %d", d);
            S5_CUDA(cudaSetDevice(devices[d]));
            int64_t* pair = off_pair(M.slot[d].d);
            S5_CUDA(cudaMemcpy(pair, d_out_handles[d] + sizes[d] - 1, 8, cudaMemcpyDeviceToDevice));
            S5_CUDA(cudaMemcpyPeer(pair + 1, devices[d], d_out_handles[nxt], devices[nxt], 8));
            if (int r = s5_adjacent_lcp(d_arenas[d], arena_len, pair, 2, d_out_lcp[d] + sizes[d] - 1,
                                        nullptr))
                return r;
            S5_CUDA(cudaDeviceSynchronize());
        }
    }
    mark("boundaries");
    for (int d = 0; d < G; ++d) out_counts[d] = sizes[d];
    if (stats) {
        int big = 0;
        for (int d = 1; d < G; ++d)
            if (sizes[d] > sizes[big]) big = d;
        *stats = st[big];
        uint64_t launches = 0, fetches = 0;
        for (int d = 0; d < G; ++d) {
            launches += st[d].launches + (shard_n[d] ? 4 : 0);
            fetches += st[d].key_fetches;
        }
        stats->launches = launches;
        stats->key_fetches = fetches;
        stats->ms_total = std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - t0).count();
    }
    return 0;
}
