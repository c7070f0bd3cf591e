// s5_kernels.cuh -- sm_100a kernels of the level-synchronous S^5 string sort.
//
// Data in HBM (one sort call, n strings):
//   arena   u8[N + pad]                     read-only, 8-byte aligned
//   off[2]  u32[n]  key[2] u64[n]           ping-pong (offset, cached 8-byte key)
//   out     i64[n]  (the caller's handles)  final order, written once per string
//   lcp     i64[n-1]                        exact LCPs; bucket boundaries whose
//           neighbours finish in different CTAs are listed in hint_list
// A segment {begin, size, depth, side} is a range of off/key[side] whose
// strings share `depth` leading bytes and whose keys hold bytes
// [depth, depth+8).  Each level processes every live segment once:
//   wide   (size > narrow_max): multi-CTA S^5 step -- plan, tree, count,
//          column scan, bucket scan + emit, scatter (samplesort.py:369-434)
//   narrow (size <= narrow_max): one fused CTA S^5 step (samplesort.py:213-238)
//   small  (size <= small_max <= 32): warp sort on cached keys with refills
//          and LCP emission (replaces basesort.py's mkqs/insertion tiers)
#pragma once

#include <cstdint>

#include "s5_device.cuh"

namespace s5 {

struct Seg {
    uint32_t begin, size, depth, side;
};

constexpr int NCLS_MAX = 8;

// Device control block: next-level list counters, error bits, statistics.
struct Ctl {
    uint32_t n_list[NCLS_MAX];  // next-level segment counts per size class
    uint32_t err;        // bit0 handle range, bit1 list overflow, bit2 pool overflow
    unsigned long long elems[NCLS_MAX];  // strings in next-level lists, per class
    unsigned long long fetches;   // arena key gathers
    unsigned long long hints;     // boundary LCP hints appended to the hint list
    uint32_t wide_ctas;           // plan: CTAs of the current wide launch
    uint32_t k2;                  // root tree: carry second key words to level 1
    uint32_t w32;                 // root tree: high-entropy keys, 32-bit local sort words
    unsigned long long tree_words, hist_words;  // plan: pool use of the current level
    uint32_t plan_err;            // plan: ERR_POOL (sticky; the plan runs before the level's reset)
    // Root prefix skip: the root sample's keys share `skip` leading bytes
    // (value skip_prefix, no terminator among them), so level 0 classifies
    // the 8 bytes after them -- "http://" costs URL-like data no level of its
    // own.  The level-0 count checks every string against the prefix; one
    // mismatch sets skip_fail, the level-0 scatter then writes nothing and
    // the host restarts the sort without the skip.
    uint32_t skip, skip_fail;
    unsigned long long skip_prefix;
};

enum : uint32_t { ERR_RANGE = 1, ERR_LIST = 2, ERR_POOL = 4 };
enum : int { WIDE = 0, NARROW = 1, SMALL = 2, LOCAL = 3, LOCAL_S = 4, LOCAL_M = 5, LOCAL_XS = 6,
              LOCAL_W = 7, NCLS = 8 };

struct SortArgs {
    const uint8_t* arena;
    uint32_t* off[2];
    uint64_t* key[2];
    int64_t* out;
    int64_t* lcp;
    uint2* hint_list;      // (position, depth) of LCPs left for k_lcp_fix
    uint32_t hint_cap;
    Seg* next[NCLS];
    uint32_t cap[NCLS];
    Ctl* ctl;
    uint32_t small_max, local_w_max, local_xs_max, local_s_max, local_m_max, local_max, narrow_max;
    uint32_t dmax;         // log2(cfg.v + 1)
    uint32_t wide_dcap;    // wide steps use d <= wide_dcap (<= kWideDMax)
    uint32_t wide_target;  // wide steps aim at children of about this size
    uint32_t local_target; // unused (the local tier sorts whole segments)
    uint32_t wide_chunk;   // strings per wide CTA at least (kWideChunkMin)
    uint32_t wide_sample;  // power-of-two bound of a wide step's sample (k_wide_tree smem)
    uint32_t alpha;
    uint32_t flags;        // s5_config flags (bit2: no common-prefix skip)
    uint64_t seed;
    const int64_t* root;   // level 0 only: the caller's handles (gather fused into the count)
    const uint32_t* root32; // ... or, with cfg flags bit9, the caller's handles as u32 offsets
    uint64_t arena_len;
    // Second key words (string bytes depth+8..depth+15), gathered by the root
    // count while its reads are in arena order and carried to level 1, whose
    // equality buckets then need no random arena refetch.  k2_stage: 1 at the
    // root (count fills key2[0], scatter carries it to key2[1]), 2 at level 1
    // (scatter reads key2[1] for segments still at the root depth).  Active
    // only when the root tree set ctl->k2 (k_wide_tree's estimate).
    uint64_t* key2[2];
    uint32_t k2_stage;
    uint32_t k2_depth;
    // Below the root the same arrays carry an equality bucket's second word
    // one level: a segment with Seg.side bit 1 set ("k2-valid") has in
    // key2[side & 1] the string bytes [depth+8, depth+16).  The wide scatter
    // fetches 16 bytes for the strings of an equality bucket (one random
    // access, like the 8-byte refetch) and flags the child; the child's own
    // equality buckets then take their next key from key2 instead of the
    // arena -- every other level of a shared-prefix chain without a random
    // fetch.  k2_cap: the arrays exist (n > narrow_max).
    uint32_t k2_cap;
    uint32_t sm_count;  // SMs of the device (wide_geom rounds a huge segment's CTAs to whole waves)
    // Arenas of >= 4 GiB (the reference's handles are int64 offsets,
    // strings.py:3-7): the u32 offset arrays hold each string's index in the
    // caller's array and `pos` (a copy of the handles, filled by level 0)
    // maps it to the arena position -- one more load per key refetch, none
    // on the key-only paths.  Null for arenas below 4 GiB.
    int64_t* pos;
};

// arena position / final handle of the string an offset word names
__device__ __forceinline__ uint64_t apos(const int64_t* pos, uint32_t o) {
    return pos ? static_cast<uint64_t>(__ldg(pos + o)) : o;
}
__device__ __forceinline__ uint64_t apos(const SortArgs& A, uint32_t o) { return apos(A.pos, o); }
__device__ __forceinline__ int64_t ahandle(const SortArgs& A, uint32_t o) {
    return static_cast<int64_t>(apos(A.pos, o));
}

// ping-pong side of a segment, and its second-key-word flag (see SortArgs)
__device__ __forceinline__ uint32_t sd(const Seg& s) { return s.side & 1u; }
__device__ __forceinline__ bool k2v(const Seg& s) { return (s.side & 2u) != 0; }

// second key words of the root (k2_stage 1: gathered by the count, carried by
// the scatter) and of level 1 (k2_stage 2, segments still at the root depth)
__device__ __forceinline__ uint32_t k2_mode(const SortArgs& A, const Seg& s) {
    if (!A.k2_stage || !A.ctl->k2) return 0;
    if (A.k2_stage == 1) return 1;
    return s.depth == A.k2_depth ? 2u : 0u;
}

// What a distribution step does with second key words: 1 / 2 the root's
// carry (k2_mode), 3 = the segment is k2-valid (equality buckets read their
// next key from key2), 4 = fetch 16 bytes for equality buckets and flag the
// children k2-valid, 0 = plain 8-byte refetch.
enum : uint32_t { K2_NONE = 0, K2_ROOT = 1, K2_LEVEL1 = 2, K2_USE = 3, K2_MAKE = 4 };
__device__ __forceinline__ uint32_t k2_kind(const SortArgs& A, const Seg& s) {
    const uint32_t m = k2_mode(A, s);
    if (m) return m;
    if (k2v(s)) return K2_USE;
    return A.k2_cap ? K2_MAKE : K2_NONE;
}

constexpr uint32_t kNarrowThreads = 512;
constexpr uint32_t kNarrowDMax = 8;           // v <= 255, k <= 511
constexpr uint32_t kNarrowMaxSize = 1u << 20;  // no per-string shared memory
constexpr uint32_t kNarrowSampleCap = 2048;
constexpr uint32_t kWideThreads = 512;
constexpr uint32_t kWideDMax = 10;            // v <= 1023, k <= 2047
constexpr uint32_t kWideTile = 4096;          // scatter tile staged in shared memory
constexpr uint32_t kWideSampleCap = 8192;
constexpr uint32_t kMaxTreeD = 13;            // standalone tree / classify surfaces
constexpr uint32_t kWideChunkMin = 16384;     // strings per CTA at least
constexpr uint32_t kWideCtasMax = 1184;       // 8 waves of 148 SMs
constexpr uint32_t kWideFrontier = 1u << 20;  // max C x k open bucket cursors
constexpr int kWideItems = 4;                 // interleaved descents per thread
// per wide segment after the level-order tree: in-order splitters, the
// classification table (kLutCells + 1 u16) and (pf, lb) -- built once in
// k_wide_tree
constexpr uint32_t kLutTabWords = (kLutCells + 1 + 3) / 4;
constexpr uint32_t kLutWords = kLutTabWords + 2;

__host__ __device__ __forceinline__ uint32_t ceil_log2(uint32_t x) {
    uint32_t d = 0;
    while ((1u << d) < x) ++d;
    return d;
}

// Splitter tree depth for a segment: about 16 strings per inner bucket.
__host__ __device__ __forceinline__ uint32_t choose_d(uint32_t size, uint32_t dmax) {
    uint32_t d = ceil_log2((size + 15) / 16);
    if (d < 1) d = 1;
    return d < dmax ? d : dmax;
}

__device__ __forceinline__ int size_class(const SortArgs& A, uint32_t size) {
    return size <= A.small_max     ? SMALL
         : size <= A.local_w_max   ? LOCAL_W
         : size <= A.local_xs_max  ? LOCAL_XS
         : size <= A.local_s_max   ? LOCAL_S
         : size <= A.local_m_max   ? LOCAL_M
         : size <= A.local_max     ? LOCAL
         : size <= A.narrow_max    ? NARROW : WIDE;
}

__device__ __forceinline__ void emit_child(const SortArgs& A, uint32_t begin, uint32_t size,
                                           uint32_t depth, uint32_t side, int cls = -1) {
    if (cls < 0) cls = size_class(A, size);
    uint32_t idx = atomicAdd(&A.ctl->n_list[cls], 1u);
    if (idx < A.cap[cls]) {
        A.next[cls][idx] = Seg{begin, size, depth, side};
        atomicAdd(&A.ctl->elems[cls], static_cast<unsigned long long>(size));
    } else {
        atomicOr(&A.ctl->err, ERR_LIST);
    }
}

// ---------------------------------------------------------------------------
// block-level building blocks

// In-place ascending bitonic sort of s[0..M), M a power of two.
template <uint32_t THREADS>
__device__ void bitonic_sort_smem(uint64_t* s, uint32_t M) {
    for (uint32_t k = 2; k <= M; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = threadIdx.x; i < M; i += THREADS) {
                uint32_t ixj = i ^ j;
                if (ixj > i) {
                    uint64_t a = s[i], b = s[ixj];
                    bool up = (i & k) == 0;
                    if ((a > b) == up) {
                        s[i] = b;
                        s[ixj] = a;
                    }
                }
            }
            __syncthreads();
        }
    }
}

// select_splitters + _fill_level_order (classifier.py:85-126), level by level:
// node i covers sample range [na[i], nb[i]] with fallback sample[nf[i]];
// its splitter is the range middle, equal samples are skipped with binary
// searches (the sample is sorted), an empty range yields the fallback for the
// whole subtree (D5).  Produces exactly the reference's splitters.
template <uint32_t THREADS>
__device__ __noinline__ void build_tree_levels(const uint64_t* sample, uint32_t m, uint32_t d,
                                  uint64_t* tree, int32_t* na, int32_t* nb, uint32_t* nf) {
    if (threadIdx.x == 0) {
        na[1] = 0;
        nb[1] = static_cast<int32_t>(m) - 1;
        nf[1] = 0;
        tree[0] = 0;
    }
    __syncthreads();
    for (uint32_t l = 0; l < d; ++l) {
        uint32_t first = 1u << l;
        for (uint32_t i = first + threadIdx.x; i < 2 * first; i += THREADS) {
            int32_t a = na[i], b = nb[i];
            uint32_t f = nf[i];
            uint64_t x;
            int32_t la = 1, lb = 0, ra = 1, rb = 0;
            uint32_t cf = f;
            if (a > b) {
                x = sample[f];
            } else {
                int32_t mm = (a + b) >> 1;
                x = sample[mm];
                int32_t lo = a, hi = mm;  // first index in [a, mm] with sample >= x
                while (lo < hi) {
                    int32_t mid = (lo + hi) >> 1;
                    if (sample[mid] < x) lo = mid + 1; else hi = mid;
                }
                int32_t b2 = lo - 1;
                lo = mm + 1;
                hi = b + 1;  // first index in (mm, b] with sample > x
                while (lo < hi) {
                    int32_t mid = (lo + hi) >> 1;
                    if (sample[mid] <= x) lo = mid + 1; else hi = mid;
                }
                la = a; lb = b2; ra = lo; rb = b;
                cf = static_cast<uint32_t>(mm);
            }
            tree[i] = x;
            if (l + 1 < d) {
                na[2 * i] = la; nb[2 * i] = lb; nf[2 * i] = cf;
                na[2 * i + 1] = ra; nb[2 * i + 1] = rb; nf[2 * i + 1] = cf;
            }
        }
        __syncthreads();
    }
}

// Exclusive scan of h[0..k) in place, h[k] = total.  All threads call.
template <uint32_t THREADS>
__device__ __noinline__ void block_exclusive_scan(uint32_t* h, uint32_t k, uint32_t* warp_sums) {
    const uint32_t per = (k + THREADS) / THREADS;  // covers k+1 slots
    uint32_t lo = threadIdx.x * per;
    uint32_t sum = 0;
    for (uint32_t j = 0; j < per; ++j) {
        uint32_t idx = lo + j;
        if (idx < k) sum += h[idx];
    }
    uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t incl = sum;
    for (uint32_t o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) warp_sums[w] = incl;
    __syncthreads();
    if (w == 0) {
        constexpr uint32_t NW = THREADS / 32;
        uint32_t x = lane < NW ? warp_sums[lane] : 0;
        for (uint32_t o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane < NW) warp_sums[lane] = x;  // inclusive
    }
    __syncthreads();
    uint32_t run = incl - sum + (w ? warp_sums[w - 1] : 0);
    for (uint32_t j = 0; j < per; ++j) {
        uint32_t idx = lo + j;
        if (idx < k) {
            uint32_t c = h[idx];
            h[idx] = run;
            run += c;
        } else if (idx == k) {
            h[idx] = run;
        }
    }
    __syncthreads();
}

// block_exclusive_scan of a tile's bucket counts fused with the per-CTA
// cursor step of the distribution: gb[b] = cur[b] (the tile's global base of
// bucket b), cur[b] += count of b.  All threads call; ends with a barrier.
template <uint32_t THREADS>
__device__ __forceinline__ void tile_scan(uint32_t* h, uint32_t k, uint32_t* cur, uint32_t* gb,
                                          uint32_t* warp_sums) {
    const uint32_t per = (k + THREADS) / THREADS;  // covers k+1 slots
    const uint32_t lo = threadIdx.x * per;
    uint32_t sum = 0;
    for (uint32_t j = 0; j < per; ++j) {
        const uint32_t idx = lo + j;
        if (idx < k) sum += h[idx];
    }
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t incl = sum;
    for (uint32_t o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) warp_sums[w] = incl;
    __syncthreads();
    if (w == 0) {
        constexpr uint32_t NW = THREADS / 32;
        uint32_t x = lane < NW ? warp_sums[lane] : 0;
        for (uint32_t o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane < NW) warp_sums[lane] = x;  // inclusive
    }
    __syncthreads();
    uint32_t run = incl - sum + (w ? warp_sums[w - 1] : 0);
    for (uint32_t j = 0; j < per; ++j) {
        const uint32_t idx = lo + j;
        if (idx < k) {
            const uint32_t c = h[idx];
            h[idx] = run;
            run += c;
            const uint32_t r = cur[idx];
            gb[idx] = r;
            cur[idx] = r + c;
        } else if (idx == k) {
            h[idx] = run;
        }
    }
    __syncthreads();
}

struct EmitScratch {
    uint32_t cnt[NCLS];
    uint32_t base[NCLS];
    uint32_t elems[NCLS];
    uint32_t hints;
    unsigned long long hint_base;
};

// whole-warp sum, one native 32-bit shared atomic per warp (64-bit shared
// atomics compile to CAS spin loops)
__device__ __forceinline__ void warp_add(uint32_t* dst, uint32_t v) {
    v = __reduce_add_sync(0xffffffffu, v);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(dst, v);
}

__device__ __forceinline__ void push_hint(const SortArgs& A, EmitScratch* es, uint32_t pos,
                                          uint32_t depth) {
    unsigned long long slot = es->hint_base + atomicAdd(&es->hints, 1u);
    if (slot < A.hint_cap) A.hint_list[slot] = make_uint2(pos, depth);
    else atomicOr(&A.ctl->err, ERR_LIST);
}

// reserve es->hints list slots for this CTA (all threads call)
__device__ __forceinline__ void reserve_hints(const SortArgs& A, EmitScratch* es) {
    __syncthreads();
    if (threadIdx.x == 0) {
        es->hint_base = es->hints ? atomicAdd(&A.ctl->hints,
                                              static_cast<unsigned long long>(es->hints)) : 0;
        es->hints = 0;
    }
    __syncthreads();
}

// Per-bucket epilogue of one S^5 step, aggregated per CTA: LCP hint at every
// bucket's left boundary (bucket_layout boundaries, classifier.py:284-304),
// and a child segment for every unfinished bucket of >= 2 strings with the
// reference's depth rule for equality buckets (+8) and finished rule (D8:
// equality bucket of a terminated splitter = identical strings).  Children
// are counted in shared memory first, so each CTA reserves its list slots
// with one global atomic per size class.  `tree` may be shared or global.
// KEEP_SMALL: buckets of <= small_max strings are finished by the calling CTA
// itself (k_local) instead of becoming children.
template <uint32_t THREADS, bool KEEP_SMALL = false>
__device__ __forceinline__ void emit_block(const SortArgs& A, const Seg& s, const uint32_t* starts, uint32_t k,
                           const uint64_t* tree, uint32_t d, EmitScratch* es) {
    if (threadIdx.x < NCLS) {
        es->cnt[threadIdx.x] = 0;
        es->elems[threadIdx.x] = 0;
    }
    if (threadIdx.x == 0) es->hints = 0;
    const bool make2 = k2_kind(A, s) == K2_MAKE;  // the scatter fetches 16 bytes for them
    __syncthreads();
    uint32_t my_hints = 0;
    uint32_t my_elems[NCLS] = {};
    for (uint32_t b = threadIdx.x; b < k; b += THREADS) {
        uint32_t st = starts[b], cnt = starts[b + 1] - st;
        if (!cnt) continue;
        if (!KEEP_SMALL && st > 0 && A.lcp) ++my_hints;
        bool odd = b & 1;
        bool fin = cnt == 1 || (odd && has_zero_byte(tree[node_of_rank(b >> 1, d)]));
        if (!fin && !(KEEP_SMALL && cnt <= A.small_max)) {
            int cls = size_class(A, cnt);
            atomicAdd(&es->cnt[cls], 1u);
            my_elems[cls] += cnt;
        }
    }
    warp_add(&es->hints, my_hints);
    for (int q = 0; q < NCLS; ++q) warp_add(&es->elems[q], my_elems[q]);
    __syncthreads();
    if (threadIdx.x < NCLS) {
        uint32_t q = threadIdx.x, c = es->cnt[q];
        es->base[q] = c ? atomicAdd(&A.ctl->n_list[q], c) : 0;
        if (c && es->base[q] + c > A.cap[q]) atomicOr(&A.ctl->err, ERR_LIST);
        if (es->elems[q]) atomicAdd(&A.ctl->elems[q], static_cast<unsigned long long>(es->elems[q]));
        es->cnt[q] = 0;
    }
    if (threadIdx.x == 0) {
        es->hint_base = es->hints ? atomicAdd(&A.ctl->hints,
                                              static_cast<unsigned long long>(es->hints)) : 0;
        es->hints = 0;
    }
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < k; b += THREADS) {
        uint32_t st = starts[b], cnt = starts[b + 1] - st;
        if (!KEEP_SMALL && cnt && st > 0 && A.lcp) push_hint(A, es, s.begin + st - 1, s.depth);
        if (cnt < 2 || (KEEP_SMALL && cnt <= A.small_max)) continue;
        bool odd = b & 1;
        if (odd && has_zero_byte(tree[node_of_rank(b >> 1, d)])) continue;
        int cls = size_class(A, cnt);
        uint32_t slot = es->base[cls] + atomicAdd(&es->cnt[cls], 1u);
        if (slot < A.cap[cls])
            A.next[cls][slot] = Seg{s.begin + st, cnt, s.depth + (odd ? 8u : 0u),
                                    (sd(s) ^ 1u) | (odd && make2 ? 2u : 0u)};
    }
}

// Element epilogue: final slot for finished buckets (handle + identical-string
// LCP), refetched key at depth+8 for equality buckets, plain move otherwise.
__device__ __forceinline__ void place(const SortArgs& A, const Seg& s, uint32_t b, bool fin,
                                      uint32_t p, uint32_t bucket_end, uint32_t o, uint64_t k,
                                      unsigned long long& fetches, uint32_t kind = K2_NONE,
                                      uint32_t src = 0) {
    uint32_t dst = s.begin + p;
    uint32_t ns = sd(s) ^ 1u;
    if (fin) {
        A.out[dst] = ahandle(A, o);
        if ((b & 1) && A.lcp && p + 1 < bucket_end) A.lcp[dst] = s.depth + zero_index(k);
    } else if (b & 1) {
        A.off[ns][dst] = o;
        if (kind == K2_USE) {  // the carried word (src = the string's index on this side)
            A.key[ns][dst] = A.key2[sd(s)][src];
        } else if (kind == K2_MAKE) {  // 16 bytes: the next key and the one after
            uint64_t k0, k1;
            load_key2(A.arena, apos(A, o) + s.depth + 8, k0, k1);
            A.key[ns][dst] = k0;
            A.key2[ns][dst] = k1;
            ++fetches;
        } else {
            A.key[ns][dst] = load_key(A.arena, apos(A, o) + s.depth + 8);
            ++fetches;
        }
    } else {
        A.off[ns][dst] = o;
        A.key[ns][dst] = k;
    }
}

// place() with second key words (mode = k2_kind; 1: root, 2: level 1, else
// place()'s own kinds; src = the string's absolute source index)
__device__ __forceinline__ void place_k2(const SortArgs& A, const Seg& s, uint32_t b, bool fin,
                                         uint32_t p, uint32_t bucket_end, uint32_t o, uint64_t k,
                                         uint32_t mode, uint32_t src, unsigned long long& fetches) {
    if (mode != K2_ROOT && mode != K2_LEVEL1) {
        place(A, s, b, fin, p, bucket_end, o, k, fetches, mode, src);
        return;
    }
    const uint32_t dst = s.begin + p;
    const uint32_t ns = sd(s) ^ 1u;
    if (fin) {
        A.out[dst] = ahandle(A, o);
        if ((b & 1) && A.lcp && p + 1 < bucket_end) A.lcp[dst] = s.depth + zero_index(k);
    } else if (b & 1) {  // equality bucket: its next key is the carried word
        A.off[ns][dst] = o;
        A.key[ns][dst] = A.key2[mode - 1][src];
    } else {
        A.off[ns][dst] = o;
        A.key[ns][dst] = k;
        if (mode == 1) A.key2[1][dst] = A.key2[0][src];
    }
}


// level-0 input handle i of the caller's array (int64, or u32 offsets with
// cfg flags bit9 -- the multi-GPU exchange's payload), streamed once
__device__ __forceinline__ int64_t root_handle(const SortArgs& A, uint32_t i) {
    return A.root32 ? static_cast<int64_t>(__ldcs(A.root32 + i)) : __ldcs(A.root + i);
}

// ---------------------------------------------------------------------------
// level 0: gather keys at the common depth (pack_keys, strings.py:176-182)

__global__ void k_gather(const int64_t* __restrict__ handles, const uint32_t* __restrict__ h32,
                         uint32_t n, uint64_t depth, uint64_t arena_len, SortArgs A) {
    uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        int64_t h = h32 ? static_cast<int64_t>(h32[i]) : handles[i];
        if (h < 0 || static_cast<uint64_t>(h) + depth >= arena_len) {
            atomicOr(&A.ctl->err, ERR_RANGE);
            h = 0;
        }
        if (A.pos) A.pos[i] = h;
        A.off[0][i] = A.pos ? i : static_cast<uint32_t>(h);
        A.key[0][i] = load_key(A.arena, static_cast<uint64_t>(h) + depth);
    }
}

__global__ void k_init_root(SortArgs A, uint32_t n, uint32_t depth) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        emit_child(A, 0, n, depth, 0);
        A.ctl->fetches += n;
    }
}

// ---------------------------------------------------------------------------
// small tier: one warp per segment of <= 32 strings.  Bitonic sort of
// (run, key); pairs of equal unterminated keys stay in a run whose keys are
// refilled at depth+8 (the mkqs equal-partition refill, basesort.py:146-150);
// each adjacent pair's LCP is emitted the moment it is resolved:
//   keys differ            -> depth + equal leading bytes
//   keys equal, terminated -> depth + bytes before the terminator (|s|)

__device__ __forceinline__ bool comp_less(uint32_t ra, uint64_t ka, uint32_t rb, uint64_t kb) {
    return ra < rb || (ra == rb && ka < kb);
}

template <bool UNROLL = true>
__device__ __forceinline__ void warp_bitonic(uint32_t& run, uint64_t& key, uint32_t& off,
                                             uint32_t lane) {
#pragma unroll (UNROLL ? 5 : 1)
    for (uint32_t k = 2; k <= 32; k <<= 1) {
#pragma unroll (UNROLL ? 5 : 1)
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            uint32_t orun = __shfl_xor_sync(0xffffffffu, run, j);
            uint64_t okey = __shfl_xor_sync(0xffffffffu, key, j);
            uint32_t ooff = __shfl_xor_sync(0xffffffffu, off, j);
            bool up = (lane & k) == 0;
            bool lower = (lane & j) == 0;
            bool take = (lower == up) ? comp_less(orun, okey, run, key)
                                      : comp_less(run, key, orun, okey);
            if (take) {
                run = orun;
                key = okey;
                off = ooff;
            }
        }
    }
}

__global__ void __launch_bounds__(256) k_small(SortArgs A, const Seg* __restrict__ segs,
                                               uint32_t nsegs) {
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    if (warp >= nsegs) return;
    const Seg s = segs[warp];
    const bool valid = lane < s.size;
    const bool pair_valid = lane + 1 < s.size;
    uint32_t o = valid ? A.off[sd(s)][s.begin + lane] : 0u;
    uint64_t k = valid ? A.key[sd(s)][s.begin + lane] : ~0ull;
    uint32_t run = valid ? 0u : 0xFFFFFFFFu;
    uint64_t depth = s.depth;
    bool resolved = false;
    uint64_t my_lcp = 0;
    unsigned long long fetches = 0;
    for (;;) {
        warp_bitonic(run, k, o, lane);
        uint64_t nk = __shfl_down_sync(0xffffffffu, k, 1);
        uint32_t nrun = __shfl_down_sync(0xffffffffu, run, 1);
        if (pair_valid && !resolved && nrun == run) {
            if (k != nk) {
                my_lcp = depth + diff_bytes(k, nk);
                resolved = true;
            } else if (has_zero_byte(k)) {
                my_lcp = depth + zero_index(k);
                resolved = true;
            }
        }
        uint32_t unres = __ballot_sync(0xffffffffu, pair_valid && !resolved);
        if (!unres) break;
        bool prev_unres = lane > 0 && ((unres >> (lane - 1)) & 1u);
        uint32_t starts = __ballot_sync(0xffffffffu, !prev_unres);
        uint32_t le = starts & (lane == 31 ? 0xffffffffu : ((2u << lane) - 1u));
        uint32_t run_start = 31u - __clz(le);
        bool active = ((unres >> lane) & 1u) || prev_unres;
        depth += 8;
        if (active) {
            k = load_key(A.arena, apos(A, o) + depth);
            ++fetches;
        }
        run = valid ? run_start : 0xFFFFFFFFu;
    }
    if (valid) A.out[s.begin + lane] = ahandle(A, o);
    if (pair_valid && A.lcp) A.lcp[s.begin + lane] = static_cast<int64_t>(my_lcp);
    for (uint32_t x = 16; x > 0; x >>= 1) fetches += __shfl_xor_sync(0xffffffffu, fetches, x);
    if (lane == 0 && fetches) atomicAdd(&A.ctl->fetches, fetches);
}

// ---------------------------------------------------------------------------
// local tier: one CTA finishes a segment of <= THREADS*8 strings.  Instead of
// another sample/classify/distribute round, the CTA sorts the whole segment
// by its cached keys with a register bitonic network: the key bytes after the
// segment's common prefix and the string's slot (12 bits) are packed into one
// u64, so every compare-exchange is a plain integer min/max.  Runs of equal
// keys are the reference's equality buckets (classifier.py:297-303): identical
// terminated strings finish, two-string runs take one direct walk, runs of
// <= small_max strings one warp, longer runs leave as children at depth + 8.
// Every LCP of the segment is produced here (adjacent keys of different runs
// differ at the segment depth), so the local tier emits no k_lcp_fix hints.
// Replaces the sequential S^5 step + base case (samplesort.py:213-238,
// basesort.py:123-173) for segments that fit one CTA.

// Stages J = jtop..1 of a bitonic merge with block size K on the 64 entries
// at positions base + lane (a) and base + 32 + lane (b) of one warp, in
// registers; ascending where (position & K) == 0.
__device__ __forceinline__ void bitonic_reg_stages(uint64_t& a, uint64_t& b, uint32_t lane,
                                                   uint32_t base, uint32_t K, uint32_t jtop) {
    const bool upa = ((base + lane) & K) == 0, upb = ((base + 32 + lane) & K) == 0;
#pragma unroll 1
    for (uint32_t J = jtop; J > 0; J >>= 1) {
        if (J == 32) {
            if ((a > b) == upa) { uint64_t t = a; a = b; b = t; }
        } else {
            uint64_t oa = __shfl_xor_sync(0xffffffffu, a, J);
            uint64_t ob = __shfl_xor_sync(0xffffffffu, b, J);
            bool lower = (lane & J) == 0;
            a = (lower == upa) ? (oa < a ? oa : a) : (oa > a ? oa : a);
            b = (lower == upb) ? (ob < b ? ob : b) : (ob > b ? ob : b);
        }
    }
}

// Ascending sort of s[0..M), M a power of two >= 64: bitonic network whose
// stages with partner distance <= 32 run in registers (one warp per 64
// entries, shuffles), only the wider stages go through shared memory --
// log2(M/64) * (log2(M) - 5) / 2 + log2(M/64) barriers in total.
template <uint32_t THREADS>
__device__ __noinline__ void sort_sample(uint64_t* s, uint32_t M) {
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t runs = M / 64;
    for (uint32_t r = warp; r < runs; r += THREADS / 32) {
        uint64_t a = s[r * 64 + lane], b = s[r * 64 + 32 + lane];
#pragma unroll 1
        for (uint32_t K = 2; K <= 64; K <<= 1) bitonic_reg_stages(a, b, lane, r * 64, K, K >> 1);
        s[r * 64 + lane] = a;
        s[r * 64 + 32 + lane] = b;
    }
    __syncthreads();
    for (uint32_t K = 128; K <= M; K <<= 1) {
        for (uint32_t J = K >> 1; J >= 64; J >>= 1) {
            for (uint32_t i = threadIdx.x; i < M / 2; i += THREADS) {
                uint32_t lo = ((i & ~(J - 1)) << 1) | (i & (J - 1)), hi = lo + J;
                uint64_t x = s[lo], y = s[hi];
                if ((x > y) == ((lo & K) == 0)) { s[lo] = y; s[hi] = x; }
            }
            __syncthreads();
        }
        for (uint32_t r = warp; r < runs; r += THREADS / 32) {
            uint64_t a = s[r * 64 + lane], b = s[r * 64 + 32 + lane];
            bitonic_reg_stages(a, b, lane, r * 64, K, 32);
            s[r * 64 + lane] = a;
            s[r * 64 + 32 + lane] = b;
        }
        __syncthreads();
    }
}

// Shared-memory slot of sort position e: the low four bits are XORed with
// bits 3..6, which makes both access patterns of block_sort8 -- eight
// consecutive positions per thread, and consecutive positions per lane --
// free of bank conflicts.
__device__ __forceinline__ uint32_t swz(uint32_t e) { return e ^ ((e >> 3) & 15u); }

// in-thread bitonic stage with partner distance JJ < 8
template <uint32_t JJ>
__device__ __forceinline__ void bitonic_thread_stage(uint64_t (&w)[8], uint32_t t, uint32_t K) {
#pragma unroll
    for (uint32_t j = 0; j < 8; ++j) {
        if (j & JJ) continue;
        const bool asc = (((t << 3) | j) & K) == 0;
        const uint64_t a = w[j], b = w[j | JJ];
        const bool x = (a > b) == asc;
        w[j] = x ? b : a;
        w[j | JJ] = x ? a : b;
    }
}

// Ascending sort of THREADS*8 distinct u64 held eight per thread (thread t
// holds positions 8t..8t+7): partner distances < 8 inside a thread, < 256
// across lanes by shuffles, wider ones through shared memory `sb`.
template <uint32_t THREADS>
__device__ __forceinline__ void block_sort8(uint64_t (&w)[8], uint64_t* sb) {
    constexpr uint32_t N = THREADS * 8;
    const uint32_t t = threadIdx.x, lane = t & 31;
#pragma unroll 1
    for (uint32_t K = 2; K <= N; K <<= 1) {
        uint32_t J = K >> 1;
        if (J >= 256) {
#pragma unroll
            for (uint32_t j = 0; j < 8; ++j) sb[swz(t * 8 + j)] = w[j];
            __syncthreads();
#pragma unroll 1
            for (; J >= 256; J >>= 1) {
#pragma unroll 1
                for (uint32_t i = t; i < N / 2; i += THREADS) {
                    const uint32_t lo = ((i & ~(J - 1)) << 1) | (i & (J - 1));
                    const uint32_t a = swz(lo), b = swz(lo + J);
                    const uint64_t x = sb[a], y = sb[b];
                    if ((x > y) == ((lo & K) == 0)) { sb[a] = y; sb[b] = x; }
                }
                __syncthreads();
            }
#pragma unroll
            for (uint32_t j = 0; j < 8; ++j) w[j] = sb[swz(t * 8 + j)];
        }
        const bool asc = ((t << 3) & K) == 0;
#pragma unroll 1
        for (; J >= 8; J >>= 1) {
            const uint32_t m = J >> 3;
            const bool keep_min = ((lane & m) == 0) == asc;
#pragma unroll
            for (uint32_t j = 0; j < 8; ++j) {
                const uint64_t o = __shfl_xor_sync(0xffffffffu, w[j], m);
                if ((o < w[j]) == keep_min) w[j] = o;
            }
        }
        if (J >= 4) bitonic_thread_stage<4>(w, t, K);
        if (J >= 2) bitonic_thread_stage<2>(w, t, K);
        bitonic_thread_stage<1>(w, t, K);
    }
}

// Ascending sort of the 8 words of one thread (bitonic network, 24
// compare-exchanges with compile-time directions).
template <typename T>
__device__ __forceinline__ void sort8_regs(T (&w)[8]) {
#pragma unroll
    for (uint32_t K = 2; K <= 8; K <<= 1) {
#pragma unroll
        for (uint32_t J = K >> 1; J > 0; J >>= 1) {
#pragma unroll
            for (uint32_t j = 0; j < 8; ++j) {
                if (j & J) continue;
                const bool asc = (j & K) == 0 || K == 8;
                const T a = w[j], b = w[j | J];
                const bool x = (a > b) == asc;
                w[j] = x ? b : a;
                w[j | J] = x ? a : b;
            }
        }
    }
}

// the eight words of thread t at positions 8t..8t+7 of a shared array, as
// four 16-byte accesses
__device__ __forceinline__ void store8(uint64_t* sb, uint32_t my, const uint64_t (&w)[8]) {
    ulonglong2* q = reinterpret_cast<ulonglong2*>(sb + my);
#pragma unroll
    for (uint32_t j = 0; j < 4; ++j) q[j] = make_ulonglong2(w[2 * j], w[2 * j + 1]);
}

__device__ __forceinline__ void load8(const uint64_t* sb, uint32_t my, uint64_t (&w)[8]) {
    const ulonglong2* q = reinterpret_cast<const ulonglong2*>(sb + my);
#pragma unroll
    for (uint32_t j = 0; j < 4; ++j) {
        const ulonglong2 x = q[j];
        w[2 * j] = x.x;
        w[2 * j + 1] = x.y;
    }
}

// Sorts the 256 words of one warp (8 per lane, lane l holds positions
// 8l..8l+7, each lane's eight already ascending): bitonic merges of runs of
// 8, 16, .., 128 in registers -- the first stage of each merge compares
// position p with the block's mirror position (partner lane l ^ (g-1),
// element 7-j), so both runs stay ascending; then half-cleaners by shuffle
// and inside the thread.  No shared memory, no barriers.
template <typename T>
__device__ __forceinline__ void warp_merge256(T (&w)[8], uint32_t lane) {
#pragma unroll 1
    for (uint32_t g = 2; g <= 32; g <<= 1) {  // lanes per merged run
        {
            T o[8];
#pragma unroll
            for (uint32_t j = 0; j < 8; ++j) o[j] = __shfl_xor_sync(0xffffffffu, w[7 - j], g - 1);
            const bool lo_half = (lane & (g >> 1)) == 0;
#pragma unroll
            for (uint32_t j = 0; j < 8; ++j) {
                const bool lt = o[j] < w[j];
                w[j] = (lt == lo_half) ? o[j] : w[j];
            }
        }
#pragma unroll 1
        for (uint32_t m = g >> 2; m > 0; m >>= 1) {
            const bool keep_min = (lane & m) == 0;
#pragma unroll
            for (uint32_t j = 0; j < 8; ++j) {
                const T o = __shfl_xor_sync(0xffffffffu, w[j], m);
                if ((o < w[j]) == keep_min) w[j] = o;
            }
        }
#pragma unroll
        for (uint32_t J = 4; J > 0; J >>= 1) {
#pragma unroll
            for (uint32_t j = 0; j < 8; ++j) {
                if (j & J) continue;
                const T a = w[j], b = w[j | J];
                const bool x = a > b;
                w[j] = x ? b : a;
                w[j | J] = x ? a : b;
            }
        }
    }
}

// Ascending merge sort of the first n_live positions (a multiple of 8; the
// words beyond the live ones are ~0) held eight per thread (thread t holds
// positions 8t..8t+7): each thread sorts its eight in registers, then
// log2(n_live/8) rounds merge sorted runs pairwise through shared memory --
// every thread finds where its eight outputs start by a merge-path binary
// search and merges them serially (one shared load per output, no
// divergence).  O(n log n) work, no padding to a power of two; positions
// >= n_live are never touched.
template <uint32_t THREADS, typename T = uint64_t>
__device__ __forceinline__ void block_merge_sort8(T (&w)[8], T* sb, uint32_t n_live) {
    const uint32_t my = 8 * threadIdx.x;
    const bool live = my < n_live;
    if (8 * (threadIdx.x & ~31u) < n_live) {  // warp holds live words: runs of 256 in registers
        sort8_regs(w);
        warp_merge256(w, threadIdx.x & 31);
    }
#pragma unroll 1
    for (uint32_t width = 256; width < n_live; width <<= 1) {
        if (live) {
#pragma unroll
            for (uint32_t j = 0; j < 8; ++j) sb[swz(my + j)] = w[j];
        }
        __syncthreads();
        if (live) {
            const uint32_t a0 = my & ~(2 * width - 1);
            const uint32_t a1 = min(a0 + width, n_live), b1 = min(a0 + 2 * width, n_live);
            const uint32_t diag = my - a0, la = a1 - a0, lb = b1 - a1;
            uint32_t lo = diag > lb ? diag - lb : 0, hi = diag < la ? diag : la;
#pragma unroll 1
            while (lo < hi) {
                const uint32_t mid = (lo + hi) >> 1;
                if (sb[swz(a0 + mid)] <= sb[swz(a1 + diag - 1 - mid)]) lo = mid + 1;
                else hi = mid;
            }
            uint32_t ia = a0 + lo, ib = a1 + diag - lo;
            T va = ia < a1 ? sb[swz(ia)] : static_cast<T>(~T(0));
            T vb = ib < b1 ? sb[swz(ib)] : static_cast<T>(~T(0));
#pragma unroll
            for (uint32_t j = 0; j < 8; ++j) {
                const bool pa = va <= vb;  // an exhausted side holds ~0 (live words are smaller)
                w[j] = pa ? va : vb;
                ia += pa;
                ib += !pa;
                const uint32_t nx = pa ? ia : ib;
                const T nv = (pa ? ia < a1 : ib < b1) ? sb[swz(nx)] : static_cast<T>(~T(0));
                va = pa ? nv : va;
                vb = pa ? vb : nv;
            }
        }
        __syncthreads();
    }
}

// Runs of 3..32 strings whose keys agree below `depth` (the tie list of a
// segment), finished by one warp, several runs per pass: the runs ties[q],
// ties[q+1], ... are packed into the 32 lanes, each in an aligned block of
// its size rounded up to a power of two, while they fit.  One bitonic sort
// of (run, 16 string bytes) over the widest block then orders every packed
// run at once, with refills 16 bytes deeper while pairs stay unresolved (the
// mkqs equal-partition refill, basesort.py:146-150, as warp rounds); writes
// the pair LCPs, the order and the final handles.  A pass costs one network
// and one arena round trip per 16 bytes whatever it holds, so URL-like
// segments (many runs of 3-8 strings) take a fraction of the passes.
// Run ids are 2 x the run's first lane; lanes that hold no string (block
// padding, alignment holes, the tail) carry 2 x lane + 1, so every tuple's
// id grows with its lane and the sort leaves each run in its own lanes.
// Plain pointers, not the SortArgs: a reference to the kernel's parameter
// block makes every thread copy it to local memory (measured: ~19 B of DRAM
// writes per string on the local tier).  Returns (this lane's arena fetches,
// runs consumed).
__device__ __noinline__ uint2 tie_batch_warp(const uint8_t* __restrict__ arena, int64_t* out,
                                             int64_t* lcp, uint32_t begin, const uint32_t* ties,
                                             uint32_t q, uint32_t qend, const uint32_t* off1,
                                             uint16_t* perm, uint64_t depth, uint32_t lane,
                                             const int64_t* __restrict__ pos) {
    uint32_t fetches = 0;
    // packing (uniform over the warp: every lane walks the same list entries)
    uint32_t used = 0, cursor = 0, P = 2;
    uint32_t my_r0 = 0, my_start = 0, my_g = 0;
#pragma unroll 1
    while (q + used < qend) {
        const uint32_t x = ties[q + used];
        const uint32_t g = (x >> 13) & 0x3FFFu, B = g <= 2 ? 2u : 1u << (32 - __clz(g - 1));
        const uint32_t st = (cursor + B - 1) & ~(B - 1);
        if (st + B > 32) break;
        if (lane >= st && lane < st + g) {
            my_r0 = x & 0x1FFFu;
            my_start = st;
            my_g = g;
        }
        cursor = st + B;
        P = B > P ? B : P;
        ++used;
    }
    const bool valid = my_g != 0;
    const bool pair_valid = valid && lane + 1 < my_start + my_g;
    const uint32_t at = my_r0 + lane - my_start;  // sorted position of this lane (valid lanes)
    uint32_t e = valid ? perm[at] : 0u;
    uint32_t run = valid ? 2 * my_start : 2 * lane + 1;
    uint64_t k0 = ~0ull, k1 = ~0ull;
    bool resolved = false, active = valid;
    for (;; depth += 16) {  // 16 string bytes per round
        if (active) {
            load_key2(arena, apos(pos, off1[e]) + depth, k0, k1);
            ++fetches;
        }
        // bitonic sort of (run, k0, k1), payload e -- skipped when every
        // open run reads the same 16 bytes (identical strings so far)
        const uint32_t lead = (run >> 1) & 31u;
        const uint64_t l0 = __shfl_sync(0xffffffffu, k0, lead);
        const uint64_t l1 = __shfl_sync(0xffffffffu, k1, lead);
        const bool same = !active || (k0 == l0 && k1 == l1);
#pragma unroll 1
        for (uint32_t K = __all_sync(0xffffffffu, same) ? 64u : 2u; K <= P; K <<= 1) {
#pragma unroll 1
            for (uint32_t J = K >> 1; J > 0; J >>= 1) {
                uint32_t orun = __shfl_xor_sync(0xffffffffu, run, J);
                uint64_t o0 = __shfl_xor_sync(0xffffffffu, k0, J);
                uint64_t o1 = __shfl_xor_sync(0xffffffffu, k1, J);
                uint32_t oe = __shfl_xor_sync(0xffffffffu, e, J);
                bool olt = orun < run || (orun == run && (o0 < k0 || (o0 == k0 && o1 < k1)));
                bool mlt = run < orun || (run == orun && (k0 < o0 || (k0 == o0 && k1 < o1)));
                // every P-block ends ascending (the last merge), blocks alternate before
                const bool up = (lane & K) == 0 || K == P;
                bool take = (((lane & J) == 0) == up) ? olt : mlt;
                if (take) { run = orun; k0 = o0; k1 = o1; e = oe; }
            }
        }
        uint64_t n0 = __shfl_down_sync(0xffffffffu, k0, 1);
        uint64_t n1 = __shfl_down_sync(0xffffffffu, k1, 1);
        uint32_t nrun = __shfl_down_sync(0xffffffffu, run, 1);
        if (pair_valid && !resolved && nrun == run) {
            uint64_t l = 0;
            if (k0 != n0) { l = depth + diff_bytes(k0, n0); resolved = true; }
            else if (has_zero_byte(k0)) { l = depth + zero_index(k0); resolved = true; }
            else if (k1 != n1) { l = depth + 8 + diff_bytes(k1, n1); resolved = true; }
            else if (has_zero_byte(k1)) { l = depth + 8 + zero_index(k1); resolved = true; }
            if (resolved && lcp) lcp[begin + at] = l;
        }
        uint32_t unres = __ballot_sync(0xffffffffu, pair_valid && !resolved);
        if (!unres) break;
        bool prev_unres = lane > 0 && ((unres >> (lane - 1)) & 1u);
        uint32_t starts = __ballot_sync(0xffffffffu, !prev_unres);
        uint32_t le = starts & (lane == 31 ? 0xffffffffu : ((2u << lane) - 1u));
        active = ((unres >> lane) & 1u) || prev_unres;
        if (valid) run = 2 * (31u - __clz(le));
    }
    if (valid) {
        perm[at] = static_cast<uint16_t>(e);
        out[begin + at] = static_cast<int64_t>(apos(pos, off1[e]));
    }
    return make_uint2(fetches, used);
}

// strings.py:64-74 (_compare_from) + :56-61 (_lcp_pair) in one walk from a
// depth both strings are known to share, 16 bytes per step.
// strings.py:64-74 (_compare_from) + :56-61 (_lcp_pair) in one walk from a
// depth both strings are known to share, 16 bytes per step.  (Rounds of 16,
// 32, then 64 bytes were measured slower: config 4 +7 %.)
__device__ __forceinline__ int walk_compare(const uint8_t* __restrict__ arena, uint64_t a,
                                         uint64_t b, uint64_t depth, uint64_t* lcp_out,
                                         unsigned long long& fetches) {
#pragma unroll 1
    for (;; depth += 16) {
        uint64_t ka[2], kb[2];
        load_key2(arena, a + depth, ka[0], ka[1]);
        load_key2(arena, b + depth, kb[0], kb[1]);
        fetches += 2;
#pragma unroll
        for (uint32_t t = 0; t < 2; ++t) {
            if (ka[t] != kb[t]) {
                if (lcp_out) *lcp_out = depth + 8 * t + diff_bytes(ka[t], kb[t]);
                return ka[t] < kb[t] ? -1 : 1;
            }
            if (has_zero_byte(ka[t])) {
                if (lcp_out) *lcp_out = depth + 8 * t + zero_index(ka[t]);
                return 0;
            }
        }
    }
}

// block-wide min and max of one u64 per thread (all threads call)
template <uint32_t THREADS>
__device__ __forceinline__ void block_minmax(uint64_t& mn, uint64_t& mx, uint64_t (*red)[32]) {
    for (uint32_t x = 16; x > 0; x >>= 1) {
        uint64_t a = __shfl_xor_sync(0xffffffffu, mn, x), b = __shfl_xor_sync(0xffffffffu, mx, x);
        mn = a < mn ? a : mn;
        mx = b > mx ? b : mx;
    }
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) { red[0][w] = mn; red[1][w] = mx; }
    __syncthreads();
    mn = red[0][0];
    mx = red[1][0];
#pragma unroll 1
    for (uint32_t q = 1; q < THREADS / 32; ++q) {
        mn = red[0][q] < mn ? red[0][q] : mn;
        mx = red[1][q] > mx ? red[1][q] : mx;
    }
    __syncthreads();
}

// block-wide OR of one u64 per thread (all threads call): one redux per
// 32-bit half and warp, then the warps' words through shared memory
template <uint32_t THREADS>
__device__ __forceinline__ uint64_t block_or64(uint64_t x, uint64_t (*red)[32]) {
    const uint32_t lo = __reduce_or_sync(0xffffffffu, static_cast<uint32_t>(x));
    const uint32_t hi = __reduce_or_sync(0xffffffffu, static_cast<uint32_t>(x >> 32));
    x = (static_cast<uint64_t>(hi) << 32) | lo;
    if (THREADS == 32) return x;
    const uint32_t w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) red[0][w] = x;
    __syncthreads();
    x = 0;
#pragma unroll
    for (uint32_t q = 0; q < THREADS / 32; ++q) x |= red[0][q];
    __syncthreads();
    return x;
}

// run boundaries: bit p of the bitmap marks the first position of a run
__device__ __forceinline__ uint32_t run_end(const uint32_t* bits, uint32_t p) {
    uint32_t q = p + 1, wi = q >> 5;
    uint32_t b = bits[wi] & (~0u << (q & 31));
    while (!b) b = bits[++wi];
    return wi * 32 + __ffs(b) - 1;
}

__device__ __forceinline__ uint32_t run_begin(const uint32_t* bits, uint32_t p) {
    uint32_t wi = p >> 5;
    uint32_t b = bits[wi] & ((2u << (p & 31)) - 1u);
    while (!b) b = bits[--wi];
    return wi * 32 + 31 - __clz(b);
}

template <uint32_t THREADS>
struct LocalSmem {
    static constexpr uint32_t maxn = THREADS * 8;
    static constexpr uint32_t total = maxn * 8      // sort buffer, later run lists
                                    + maxn * 8      // key1: key by slot
                                    + maxn * 4      // off1: offset by slot
                                    + maxn * 2      // perm: sorted position -> slot
                                    + 2 * (maxn / 32 + 1) * 4;  // run-start bitmaps
};

// candidate runs of the truncated sort words up to this length are split by
// the cached full keys in shared memory
constexpr uint32_t kTruncFix = 64;

template <uint32_t THREADS, bool W32 = false>
__global__ void __launch_bounds__(THREADS, (THREADS >= 512 ? 2 : THREADS >= 256 ? 4 : THREADS >= 128 ? 8 : 16))
k_local(SortArgs A, const Seg* __restrict__ segs) {
    using LS = LocalSmem<THREADS>;
    constexpr uint32_t N = LS::maxn;
    extern __shared__ __align__(16) uint8_t sm[];
    uint64_t* sb = reinterpret_cast<uint64_t*>(sm);
    uint64_t* key1 = sb + N;
    uint32_t* off1 = reinterpret_cast<uint32_t*>(key1 + N);
    uint16_t* perm = reinterpret_cast<uint16_t*>(off1 + N);
    uint32_t* bits = reinterpret_cast<uint32_t*>(perm + N);
    uint32_t* bits2 = bits + N / 32 + 1;
    uint32_t* ties = reinterpret_cast<uint32_t*>(sb);   // run lists reuse the sort buffer
    uint32_t* kids = ties + N;
    uint16_t* pairs = reinterpret_cast<uint16_t*>(sb) + 3 * N;
    __shared__ EmitScratch es;
    __shared__ uint64_t red[2][32];
    __shared__ uint32_t nties, nkids, npairs;

    Seg s = segs[blockIdx.x];
    const uint32_t depth0 = s.depth;  // the carried second words hold [depth0+8, depth0+16)
    const uint32_t t = threadIdx.x, lane = t & 31;
    const uint32_t* __restrict__ goff = A.off[sd(s)] + s.begin;
    const uint64_t* __restrict__ gkey = A.key[sd(s)] + s.begin;

    // the segment in registers (coalesced)
    uint64_t rk[8];
    uint32_t ro[8];
#pragma unroll
    for (uint32_t j = 0; j < 8; ++j) {
        uint32_t i = t + j * THREADS;
        rk[j] = i < s.size ? gkey[i] : 0;
        ro[j] = i < s.size ? goff[i] : 0;
    }
    // keys and offsets by slot; the min/max reduction's barrier publishes them
#pragma unroll
    for (uint32_t j = 0; j < 8; ++j) {
        uint32_t i = t + j * THREADS;
        key1[i] = rk[j];
        off1[i] = ro[j];
    }
    // common prefix of the segment's keys; whole equal words advance the
    // depth in-CTA (the equality-bucket chain of long shared prefixes,
    // classifier.py:297-303, without a level per 8 bytes); all-identical
    // terminated keys finish here
    // (the common prefix of all keys = that of every key with the first one:
    // the leading zeros of the OR of the XORs, one redux per warp)
    unsigned long long fetches = 0;
    uint32_t L;
    const uint32_t o0 = goff[0];
    uint64_t k0 = gkey[0];
    for (;;) {
        uint64_t x = 0;
#pragma unroll
        for (uint32_t j = 0; j < 8; ++j)
            if (t + j * THREADS < s.size) x |= rk[j] ^ k0;
        x = block_or64<THREADS>(x, red);
        if (x == 0) {
            if (has_zero_byte(k0)) {  // identical strings: any order, lcp = |s|
#pragma unroll
                for (uint32_t j = 0; j < 8; ++j) {
                    uint32_t i = t + j * THREADS;
                    if (i < s.size) {
                        A.out[s.begin + i] = ahandle(A, ro[j]);
                        if (A.lcp && i + 1 < s.size) A.lcp[s.begin + i] = s.depth + zero_index(k0);
                    }
                }
                for (uint32_t x = 16; x > 0; x >>= 1)
                    fetches += __shfl_xor_sync(0xffffffffu, fetches, x);
                if (lane == 0 && fetches) atomicAdd(&A.ctl->fetches, fetches);
                return;
            }
            L = 8;
        } else {
            L = static_cast<uint32_t>(__clzll(static_cast<long long>(x))) >> 3;
        }
        // default: skip whole equal words only; flags bit3 also skips a partial
        // common prefix of >= 4 bytes; bit2 disables the skip
        if ((A.flags & 4) || L < ((A.flags & 8) ? 4u : 8u)) break;
        s.depth += L;
#pragma unroll
        for (uint32_t j = 0; j < 8; ++j) {
            if (t + j * THREADS < s.size) {
                rk[j] = load_key(A.arena, apos(A, ro[j]) + s.depth);
                key1[t + j * THREADS] = rk[j];
                ++fetches;
            }
        }
        k0 = load_key(A.arena, apos(A, o0) + s.depth);
    }
    if (L > 7) L = 7;  // all keys equal (skip disabled): one run either way
    // sort words: key bytes after the common prefix, slot in the low 12 bits.
    // With L >= 2 the word holds the whole key (exact); with L < 2 the key's
    // last 12 (L = 0) or 4 (L = 1) bits are dropped, so runs of equal words
    // are only candidate ties, resolved from the segment depth
    // Sort words: the key bytes after the common prefix with the slot in the
    // low bits.  W32 (CTAs of <= 128 threads, launched when the root sample
    // found high-entropy keys, ctl->w32): 32-bit words of SB slot bits and
    // the next KB = 32 - SB key bits -- single-instruction compare-exchanges;
    // the words hold the whole key when L >= 6, else equal words are
    // candidate runs ranked by the full keys below, skipped when the sort
    // left none.  Otherwise 64-bit words (52 key bits, the whole key when
    // L >= 2).
    static_assert(!W32 || THREADS <= 128, "32-bit words need <= 1024 strings");
    constexpr uint32_t SB = THREADS == 128 ? 10u : THREADS == 64 ? 9u : 12u;
    constexpr uint32_t KB = 32u - SB;  // key bits in a 32-bit word
    constexpr bool use32 = W32;
    bool cand_any = true;  // use32: the sort left candidate runs
    if (use32 && !(A.flags & 16)) {
        uint32_t* sb32 = reinterpret_cast<uint32_t*>(sb);
        uint32_t w[8];
        {
            uint64_t kk[8];
            load8(key1, 8 * t, kk);  // key1 published by the last prefix barrier
#pragma unroll
            for (uint32_t j = 0; j < 8; ++j) {
                const uint32_t i = 8 * t + j;
                w[j] = i < s.size ? ((static_cast<uint32_t>((kk[j] << (8 * L)) >> (64 - KB)) << SB) | i) : ~0u;
            }
        }
        block_merge_sort8<THREADS, uint32_t>(w, sb32, (s.size + 7) & ~7u);
        *reinterpret_cast<uint4*>(sb32 + 8 * t) = make_uint4(w[0], w[1], w[2], w[3]);
        *reinterpret_cast<uint4*>(sb32 + 8 * t + 4) = make_uint4(w[4], w[5], w[6], w[7]);
        __syncthreads();
        if (t == 0) {
            bits[N / 32] = 1u;
            nties = 0;
            nkids = 0;
            npairs = 0;
        }
        bool cand = false;
#pragma unroll 1
        for (uint32_t p = t; p < N; p += THREADS) {
            const uint32_t wp = sb32[p];
            const bool st = p == 0 || p >= s.size || (wp >> SB) != (sb32[p - 1] >> SB);
            cand |= !st;
            const uint32_t b = __ballot_sync(0xffffffffu, st);
            if (lane == 0) bits[p >> 5] = b;
            if (p < s.size) perm[p] = static_cast<uint16_t>(wp & ((1u << SB) - 1u));
        }
        cand_any = __syncthreads_or(cand);
    } else {
    uint64_t w[8];
    if (A.flags & 16) {  // power-of-two bitonic network over the whole CTA
#pragma unroll
        for (uint32_t j = 0; j < 8; ++j) {
            uint32_t i = t + j * THREADS;
            w[j] = i < s.size ? (((rk[j] << (8 * L)) & ~0xFFFull) | i) : ~0ull;
        }
        block_sort8<THREADS>(w, sb);
    } else {  // merge sort of the live positions (slot i at position i)
        load8(key1, 8 * t, w);  // key1 published by the last min/max barrier
#pragma unroll
        for (uint32_t j = 0; j < 8; ++j) {
            const uint32_t i = 8 * t + j;
            w[j] = i < s.size ? (((w[j] << (8 * L)) & ~0xFFFull) | i) : ~0ull;
        }
        block_merge_sort8<THREADS>(w, sb, (s.size + 7) & ~7u);
    }
    store8(sb, 8 * t, w);
    __syncthreads();

    // runs of equal words: start bitmap (positions >= size all start runs)
    if (t == 0) {
        bits[N / 32] = 1u;
        nties = 0;
        nkids = 0;
        npairs = 0;
    }
#pragma unroll 1
    for (uint32_t p = t; p < N; p += THREADS) {
        const uint64_t wp = sb[p];
        const bool st = p == 0 || p >= s.size || (wp >> 12) != (sb[p - 1] >> 12);
        const uint32_t b = __ballot_sync(0xffffffffu, st);
        if (lane == 0) bits[p >> 5] = b;
        if (p < s.size) perm[p] = static_cast<uint16_t>(wp & 0xFFFu);
    }
    __syncthreads();
    }
    // key bytes after the prefix the words hold whole; whole keys in the
    // words, or no candidate run (every run is one string)
    const uint32_t kept = use32 ? KB / 8 : 6u;
    const bool exact = use32 ? (8 * (8 - L) <= KB || !cand_any) : L >= 2;
    const uint32_t* rb = bits;
    if (!exact) {
        // truncated words: candidate runs of <= kTruncFix strings are put in
        // full-key order (rank by the cached keys) and split where the full
        // keys differ, which makes them exact runs; longer candidate runs stay
        // whole and leave as children at the same depth (their keys share
        // >= 6 bytes, so the child's words are exact)
        uint16_t* perm2 = reinterpret_cast<uint16_t*>(sb) + 3 * N;
#pragma unroll 1
        for (uint32_t p = t; p < s.size; p += THREADS) {
            const uint32_t r0 = run_begin(bits, p), r1 = run_end(bits, p);
            const uint32_t slot = perm[p];
            uint32_t r = p - r0;
            if (r1 - r0 >= 2 && r1 - r0 <= kTruncFix) {
                const uint64_t k = key1[(slot)];
                r = 0;
#pragma unroll 1
                for (uint32_t q = r0; q < r1; ++q) {
                    const uint64_t y = key1[(perm[q])];
                    r += (y < k) || (y == k && q < p);
                }
            }
            perm2[r0 + r] = static_cast<uint16_t>(slot);
        }
        __syncthreads();
#pragma unroll 1
        for (uint32_t p = t; p < N; p += THREADS) {
            bool st = true;
            if (p < s.size) {
                const uint32_t slot = perm2[p];
                st = (bits[p >> 5] >> (p & 31)) & 1u;
                if (!st && run_end(bits, p) - run_begin(bits, p) <= kTruncFix)
                    st = key1[(slot)] != key1[(perm2[p - 1])];
                perm[p] = static_cast<uint16_t>(slot);
            }
            const uint32_t b = __ballot_sync(0xffffffffu, st);
            if (lane == 0) bits2[p >> 5] = b;
        }
        if (t == 0) bits2[N / 32] = 1u;
        __syncthreads();
        rb = bits2;
    }

    // per position: finished strings go out, children to the other side,
    // LCPs at run boundaries and inside identical runs; ties are listed
    const uint32_t tmax = A.small_max;
    const uint32_t ns = sd(s) ^ 1u;
    const uint64_t depth = s.depth;
#pragma unroll 1
    for (uint32_t p = t; p < s.size; p += THREADS) {
        const uint32_t slot = perm[p];
        const uint64_t k = key1[(slot)];
        const uint32_t o = off1[slot];
        const uint32_t r0 = run_begin(rb, p), r1 = run_end(rb, p);
        const uint32_t g = r1 - r0;
        // keys of the run are equal: exact words, a re-ranked short run, or a
        // terminator inside the bytes the truncated words kept whole ([0, L+6):
        // the run's strings are then identical -- short duplicates finish here)
        const bool rexact = exact || g <= kTruncFix || zero_index(k) < L + kept;
        const uint32_t dst = s.begin + p;
        if (A.lcp && p + 1 == r1 && r1 < s.size)
            A.lcp[dst] = depth + diff_bytes(k, key1[(perm[r1])]);
        if (g == 1 || (rexact && has_zero_byte(k))) {
            A.out[dst] = ahandle(A, o);
            if (A.lcp && p + 1 < r1) A.lcp[dst] = depth + zero_index(k);
        } else if (g > 2 && g > tmax) {
            A.off[ns][dst] = o;
            if (rexact && k2v(s) && depth == depth0) {  // the carried word (slot = input index)
                A.key[ns][dst] = A.key2[sd(s)][s.begin + slot];
            } else if (rexact) {
                A.key[ns][dst] = load_key(A.arena, apos(A, o) + depth + 8);
                ++fetches;
            } else {
                A.key[ns][dst] = k;
            }
            if (p == r0) kids[atomicAdd(&nkids, 1u)] = r0 | (g << 13) | (rexact ? 1u << 31 : 0u);
        } else if (p == r0) {
            if (g == 2)
                pairs[atomicAdd(&npairs, 1u)] = static_cast<uint16_t>(p);
            else
                ties[atomicAdd(&nties, 1u)] = r0 | (g << 13);
        }
    }
    __syncthreads();
    // runs of two strings: one direct walk each, spread over all threads
    const uint32_t np = npairs;
    for (uint32_t q = t; q < np; q += THREADS) {
        const uint32_t p = pairs[q], sa = perm[p], sb2 = perm[p + 1];
        uint64_t l;
        const int c = walk_compare(A.arena, apos(A, off1[sa]), apos(A, off1[sb2]), depth + 8, &l, fetches);
        if (A.lcp) A.lcp[s.begin + p] = l;
        A.out[s.begin + p] = ahandle(A, off1[c > 0 ? sb2 : sa]);
        A.out[s.begin + p + 1] = ahandle(A, off1[c > 0 ? sa : sb2]);
    }
    // runs of 3..small_max strings: one warp each
    const uint32_t nt = nties, nk = nkids;
    {  // each warp takes a contiguous share of the list, several runs per pass
        constexpr uint32_t NWP = THREADS / 32;
        const uint32_t share = (nt + NWP - 1) / NWP;
        uint32_t q = (t >> 5) * share;
        const uint32_t qend = min(nt, q + share);
        while (q < qend) {
            const uint2 r = tie_batch_warp(A.arena, A.out, A.lcp, s.begin, ties, q, qend, off1, perm,
                                           depth + 8, lane, A.pos);
            fetches += r.x;
            q += r.y;
        }
    }
    // children: one list reservation per size class per CTA
    if (nk) {
        if (t < NCLS) {
            es.cnt[t] = 0;
            es.elems[t] = 0;
        }
        __syncthreads();
        for (uint32_t q = t; q < nk; q += THREADS) {
            const uint32_t g = (kids[q] >> 13) & 0x3FFFu;
            const int cls = size_class(A, g);
            atomicAdd(&es.cnt[cls], 1u);
            atomicAdd(&es.elems[cls], g);
        }
        __syncthreads();
        if (t < NCLS) {
            const uint32_t c = es.cnt[t];
            es.base[t] = c ? atomicAdd(&A.ctl->n_list[t], c) : 0;
            if (c && es.base[t] + c > A.cap[t]) atomicOr(&A.ctl->err, ERR_LIST);
            if (es.elems[t])
                atomicAdd(&A.ctl->elems[t], static_cast<unsigned long long>(es.elems[t]));
            es.cnt[t] = 0;
        }
        __syncthreads();
        for (uint32_t q = t; q < nk; q += THREADS) {
            const uint32_t x = kids[q], r0 = x & 0x1FFFu, g = (x >> 13) & 0x3FFFu;
            const uint32_t cdepth = static_cast<uint32_t>(depth) + ((x >> 31) ? 8u : 0u);
            const int cls = size_class(A, g);
            const uint32_t at = es.base[cls] + atomicAdd(&es.cnt[cls], 1u);
            if (at < A.cap[cls]) A.next[cls][at] = Seg{s.begin + r0, g, cdepth, ns};
        }
    }
    for (uint32_t x = 16; x > 0; x >>= 1) fetches += __shfl_xor_sync(0xffffffffu, fetches, x);
    if (lane == 0 && fetches) atomicAdd(&A.ctl->fetches, fetches);
}

// Warp tier: one warp finishes a segment of <= 256 strings (8 per lane) with
// the local tier's algorithm at warp scope -- the sort words are merged in
// registers (sort8_regs + warp_merge256), so there are no shared-memory sort
// rounds and no block barriers; 4 segments per CTA (a CTA lives as long as
// its slowest warp: with 8 the achieved occupancy of URL-like levels was 25 %;
// 4 and 2 measure the same, k_local_w -11 % on config 3, -7 % on 2 and 5).
constexpr uint32_t kWarpLocalMax = 256;
#ifndef S5_WARP_LOCAL_WARPS
#define S5_WARP_LOCAL_WARPS 4
#endif
constexpr uint32_t kWarpLocalWarps = S5_WARP_LOCAL_WARPS;

struct WarpLocalSmem {
    uint64_t key1[kWarpLocalMax];
    uint32_t off1[kWarpLocalMax];
    uint16_t perm[kWarpLocalMax];
    uint16_t perm2[kWarpLocalMax];
    uint32_t bits[kWarpLocalMax / 32 + 1];
    uint32_t bits2[kWarpLocalMax / 32 + 1];
    uint32_t ties[kWarpLocalMax / 3 + 1];
    uint16_t pairs[kWarpLocalMax / 2];
    uint32_t nties, npairs;
};

__global__ void __launch_bounds__(kWarpLocalWarps * 32) k_local_w(SortArgs A, const Seg* __restrict__ segs,
                                                                  uint32_t nsegs) {
    __shared__ WarpLocalSmem wsm[kWarpLocalWarps];
    const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint32_t si = blockIdx.x * kWarpLocalWarps + wid;
    if (si >= nsegs) return;  // warp scope only: no block barriers below
    WarpLocalSmem& W = wsm[wid];
    Seg s = segs[si];
    const uint32_t depth0 = s.depth;
    const uint32_t* __restrict__ goff = A.off[sd(s)] + s.begin;
    const uint64_t* __restrict__ gkey = A.key[sd(s)] + s.begin;
    uint64_t rk[8];
    uint32_t ro[8];
#pragma unroll
    for (uint32_t j = 0; j < 8; ++j) {
        const uint32_t i = lane + 32 * j;
        rk[j] = i < s.size ? gkey[i] : 0;
        ro[j] = i < s.size ? goff[i] : 0;
    }
    unsigned long long fetches = 0;
    uint32_t L;
    uint64_t k0 = __shfl_sync(0xffffffffu, rk[0], 0);
    for (;;) {  // common-prefix skip, as in k_local (OR of the XORs with the first key)
        uint64_t x = 0;
#pragma unroll
        for (uint32_t j = 0; j < 8; ++j)
            if (lane + 32 * j < s.size) x |= rk[j] ^ k0;
        x = block_or64<32>(x, nullptr);
        if (x == 0) {
            if (has_zero_byte(k0)) {  // identical strings
#pragma unroll
                for (uint32_t j = 0; j < 8; ++j) {
                    const uint32_t i = lane + 32 * j;
                    if (i < s.size) {
                        A.out[s.begin + i] = ahandle(A, ro[j]);
                        if (A.lcp && i + 1 < s.size) A.lcp[s.begin + i] = s.depth + zero_index(k0);
                    }
                }
                L = 9;  // done
                break;
            }
            L = 8;
        } else {
            L = static_cast<uint32_t>(__clzll(static_cast<long long>(x))) >> 3;
        }
        if ((A.flags & 4) || L < ((A.flags & 8) ? 4u : 8u)) break;
        s.depth += L;
#pragma unroll
        for (uint32_t j = 0; j < 8; ++j) {
            if (lane + 32 * j < s.size) {
                rk[j] = load_key(A.arena, apos(A, ro[j]) + s.depth);
                ++fetches;
            }
        }
        k0 = __shfl_sync(0xffffffffu, rk[0], 0);
    }
    if (L <= 8) {
        if (L > 7) L = 7;
        // 32-bit sort words: the 3 key bytes after the common prefix, the
        // slot in the low 8 bits (min/max compare-exchanges and one shuffle
        // per word instead of 64-bit compares, four selects and two
        // shuffles).  The words hold the whole key when L >= 5; otherwise
        // equal words are candidate runs, ranked by the full cached keys
        // below -- skipped when the sort left none.
        bool exact = L >= 5;
        uint32_t w[8];
#pragma unroll
        for (uint32_t j = 0; j < 8; ++j) {
            const uint32_t i = lane + 32 * j;
            W.key1[i] = rk[j];
            W.off1[i] = ro[j];
            w[j] = i < s.size ? ((static_cast<uint32_t>((rk[j] << (8 * L)) >> 40) << 8) | i) : ~0u;
        }
        sort8_regs(w);
        warp_merge256(w, lane);
        // run starts of the sorted words (lane l holds positions 8l..8l+7)
        const uint32_t prev = __shfl_up_sync(0xffffffffu, w[7], 1);
        uint32_t fl = 0;
#pragma unroll
        for (uint32_t j = 0; j < 8; ++j) {
            const uint32_t p = 8 * lane + j;
            const uint32_t pw = j ? w[j - 1] : prev;
            const bool st = p == 0 || p >= s.size || (w[j] >> 8) != (pw >> 8);
            fl |= (st ? 1u : 0u) << j;
            if (p < s.size) W.perm[p] = static_cast<uint16_t>(w[j] & 0xFFu);
        }
        if (!exact && !__any_sync(0xffffffffu, fl != 0xFFu)) exact = true;  // every run is one string
        uint32_t word = fl << (8 * (lane & 3));
        word |= __shfl_xor_sync(0xffffffffu, word, 1);
        word |= __shfl_xor_sync(0xffffffffu, word, 2);
        if ((lane & 3) == 0) W.bits[lane >> 2] = word;
        if (lane == 0) {
            W.bits[kWarpLocalMax / 32] = 1u;
            W.nties = 0;
            W.npairs = 0;
        }
        __syncwarp();
        const uint32_t* rb = W.bits;
        if (!exact) {  // candidate runs of truncated words: rank by the full keys
#pragma unroll 1
            for (uint32_t p = lane; p < s.size; p += 32) {
                const uint32_t r0 = run_begin(W.bits, p), r1 = run_end(W.bits, p);
                const uint32_t slot = W.perm[p];
                uint32_t r = p - r0;
                if (r1 - r0 >= 2 && r1 - r0 <= kTruncFix) {
                    const uint64_t k = W.key1[slot];
                    r = 0;
#pragma unroll 1
                    for (uint32_t q = r0; q < r1; ++q) {
                        const uint64_t y = W.key1[W.perm[q]];
                        r += (y < k) || (y == k && q < p);
                    }
                }
                W.perm2[r0 + r] = static_cast<uint16_t>(slot);
            }
            __syncwarp();
#pragma unroll 1
            for (uint32_t p = lane; p < kWarpLocalMax; p += 32) {
                bool st = true;
                if (p < s.size) {
                    const uint32_t slot = W.perm2[p];
                    st = (W.bits[p >> 5] >> (p & 31)) & 1u;
                    if (!st && run_end(W.bits, p) - run_begin(W.bits, p) <= kTruncFix)
                        st = W.key1[slot] != W.key1[W.perm2[p - 1]];
                }
                const uint32_t b = __ballot_sync(0xffffffffu, st);
                if (lane == 0) W.bits2[p >> 5] = b;
            }
            __syncwarp();
            for (uint32_t p = lane; p < s.size; p += 32) W.perm[p] = W.perm2[p];
            if (lane == 0) W.bits2[kWarpLocalMax / 32] = 1u;
            __syncwarp();
            rb = W.bits2;
        }
        // per position, as in k_local; children are emitted one by one
        const uint32_t tmax = A.small_max;
        const uint32_t ns = sd(s) ^ 1u;
        const uint64_t depth = s.depth;
#pragma unroll 1
        for (uint32_t p = lane; p < s.size; p += 32) {
            const uint32_t slot = W.perm[p];
            const uint64_t k = W.key1[slot];
            const uint32_t o = W.off1[slot];
            const uint32_t r0 = run_begin(rb, p), r1 = run_end(rb, p);
            const uint32_t g = r1 - r0;
            // (the words kept key bytes [L, L+3) whole: a terminator there
            // makes the run's strings identical)
            const bool rexact = exact || g <= kTruncFix || zero_index(k) < L + 3;
            const uint32_t dst = s.begin + p;
            if (A.lcp && p + 1 == r1 && r1 < s.size)
                A.lcp[dst] = depth + diff_bytes(k, W.key1[W.perm[r1]]);
            if (g == 1 || (rexact && has_zero_byte(k))) {
                A.out[dst] = ahandle(A, o);
                if (A.lcp && p + 1 < r1) A.lcp[dst] = depth + zero_index(k);
            } else if (g > 2 && g > tmax) {
                A.off[ns][dst] = o;
                if (rexact && k2v(s) && depth == depth0) {  // the carried word
                    A.key[ns][dst] = A.key2[sd(s)][s.begin + slot];
                } else if (rexact) {
                    A.key[ns][dst] = load_key(A.arena, apos(A, o) + depth + 8);
                    ++fetches;
                } else {
                    A.key[ns][dst] = k;
                }
                if (p == r0)
                    emit_child(A, s.begin + r0, g, static_cast<uint32_t>(depth) + (rexact ? 8u : 0u), ns);
            } else if (p == r0) {
                if (g == 2)
                    W.pairs[atomicAdd(&W.npairs, 1u)] = static_cast<uint16_t>(p);
                else
                    W.ties[atomicAdd(&W.nties, 1u)] = r0 | (g << 13);
            }
        }
        __syncwarp();
        for (uint32_t q = lane; q < W.npairs; q += 32) {  // pairs spread over the lanes
            const uint32_t p = W.pairs[q], sa = W.perm[p], sb2 = W.perm[p + 1];
            uint64_t l;
            const int c = walk_compare(A.arena, apos(A, W.off1[sa]), apos(A, W.off1[sb2]), depth + 8, &l, fetches);
            if (A.lcp) A.lcp[s.begin + p] = l;
            A.out[s.begin + p] = ahandle(A, W.off1[c > 0 ? sb2 : sa]);
            A.out[s.begin + p + 1] = ahandle(A, W.off1[c > 0 ? sa : sb2]);
        }
        const uint32_t nt = W.nties;
        for (uint32_t q = 0; q < nt;) {  // several runs per pass
            const uint2 r = tie_batch_warp(A.arena, A.out, A.lcp, s.begin, W.ties, q, nt, W.off1,
                                           W.perm, depth + 8, lane, A.pos);
            fetches += r.x;
            q += r.y;
        }
    }
    for (uint32_t x = 16; x > 0; x >>= 1) fetches += __shfl_xor_sync(0xffffffffu, fetches, x);
    if (lane == 0 && fetches) atomicAdd(&A.ctl->fetches, fetches);
}

// ---------------------------------------------------------------------------
// narrow tier: the whole S^5 step of one segment in one CTA (the reference's
// sequential step, samplesort.py:213-238, at the fan-out of the wide tier):
// sample + splitter tree in shared memory, a counting pass over the keys
// (shared histogram), the bucket starts and children (bucket_layout), then a
// distribution pass that classifies every key again and takes its slot from
// a per-bucket cursor (warp-aggregated shared atomics; order inside a bucket
// is free, the reference's distribution is not stable either).  Both passes
// stream the segment through a ring of shared-memory tiles filled by the
// bulk-copy engine, so the loads of the next tiles are in flight while one
// is classified.  No per-string shared memory: the segment size is not
// bounded by it.  Replaces the six-kernel wide pipeline (tree, count, column
// scan, bucket scan, scatter + the u16 bucket array in HBM) for the segments
// below the root.  A segment whose sample is one unterminated key is checked
// in full and, when every key is equal, its keys are refetched 8 bytes deeper
// in place (the equality-bucket chain of a long shared prefix without a
// level per 8 bytes, as in k_local).

constexpr uint32_t kNarrowTile = 2048;
constexpr uint32_t kNarrowStages = 3;

struct NarrowStage {
    uint64_t key[kNarrowTile + 2];
    uint32_t off[kNarrowTile + 4];
};

struct NarrowSmem {
    static constexpr uint32_t ring_bytes = kNarrowStages * sizeof(NarrowStage);  // 72 KB
    static constexpr uint32_t sample_bytes = kNarrowSampleCap * 8;                // aliases the ring
    static constexpr uint32_t big_bytes = ring_bytes > sample_bytes ? ring_bytes : sample_bytes;
    static constexpr uint32_t tree_bytes = (1u << kNarrowDMax) * 8;
    static constexpr uint32_t node_bytes = (1u << kNarrowDMax) * 12;
    static constexpr uint32_t hist_words = (2u << kNarrowDMax) + 2;  // k + 1
    // in-order splitters + the classification table (lut_build)
    static constexpr uint32_t lut_bytes = (1u << kNarrowDMax) * 8 + (kLutCells + 1 + 7) / 8 * 16;
    static constexpr uint32_t total = big_bytes + tree_bytes + node_bytes + 2 * hist_words * 4 + 8 * kNarrowStages +
                                      lut_bytes;
};

template <bool EQUAL>
__global__ void __launch_bounds__(kNarrowThreads, 2)
k_narrow(SortArgs A, const Seg* __restrict__ segs) {
    constexpr uint32_t T = kNarrowThreads, TILE = kNarrowTile, NS = kNarrowStages;
    constexpr uint32_t IT = TILE / T;  // keys per thread and tile
    extern __shared__ __align__(16) uint8_t sm[];
    NarrowStage* ring = reinterpret_cast<NarrowStage*>(sm);
    uint64_t* sample = reinterpret_cast<uint64_t*>(sm);
    uint64_t* tree = reinterpret_cast<uint64_t*>(sm + NarrowSmem::big_bytes);
    int32_t* na = reinterpret_cast<int32_t*>(sm + NarrowSmem::big_bytes + NarrowSmem::tree_bytes);
    int32_t* nb = na + (1u << kNarrowDMax);
    uint32_t* nf = reinterpret_cast<uint32_t*>(nb + (1u << kNarrowDMax));
    uint32_t* hist = nf + (1u << kNarrowDMax);
    uint32_t* cur = hist + NarrowSmem::hist_words;
    uint64_t* bar = reinterpret_cast<uint64_t*>(cur + NarrowSmem::hist_words);
    uint64_t* spl = bar + kNarrowStages;  // in-order splitters, then the table
    __shared__ uint32_t warp_sums[32];
    __shared__ uint64_t red[2][32];
    __shared__ EmitScratch es;

    Seg s = segs[blockIdx.x];
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t* off = A.off[sd(s)] + s.begin;
    uint64_t* key = A.key[sd(s)] + s.begin;  // rewritten in place by the prefix skip
    uint32_t dw = A.dmax < kNarrowDMax ? A.dmax : kNarrowDMax;
    uint32_t d = ceil_log2((s.size + A.wide_target - 1) / A.wide_target);
    d = d < 1 ? 1 : (d > dw ? dw : d);
    const uint32_t v = (1u << d) - 1, k = 2 * v + 1;
    uint32_t m = A.alpha * v;
    if (m > kNarrowSampleCap) m = kNarrowSampleCap;
    uint32_t M = 64;
    while (M < m) M <<= 1;
    unsigned long long fetches = 0;

    // stage 1: sample (classifier.py:76-82), sorted; the common-prefix skip
    for (;;) {
        const uint64_t sseed = segment_seed(A.seed, s.begin, s.size, s.depth);
        for (uint32_t t = threadIdx.x; t < M; t += T)
            sample[t] = t < m ? __ldcg(key + sample_index(sseed, t, s.size)) : ~0ull;
        __syncthreads();
        sort_sample<T>(sample, M);
        const uint64_t s0 = sample[0];
        if (s0 != sample[m - 1] || has_zero_byte(s0) || (A.flags & 4)) break;
        // the sample is one unterminated key: is every key equal?
        uint64_t mn = ~0ull, mx = 0;
        for (uint32_t i = threadIdx.x; i < s.size; i += T) {
            const uint64_t x = __ldcg(key + i);
            mn = x < mn ? x : mn;
            mx = x > mx ? x : mx;
        }
        block_minmax<T>(mn, mx, red);
        if (mn != mx) break;  // no: an ordinary step (one dominant equality bucket)
        s.depth += 8;
        s.side &= 1u;  // carried second key words belong to the old depth: not valid any more
        for (uint32_t i = threadIdx.x; i < s.size; i += T) {
            key[i] = load_key(A.arena, apos(A, off[i]) + s.depth);
            ++fetches;
        }
        // generic-proxy writes, read next by the sample and the bulk copies
        asm volatile("fence.proxy.async;\n" ::: "memory");
        __syncthreads();
    }
    build_tree_levels<T>(sample, m, d, tree, na, nb, nf);  // ends with a barrier
    // classification table: ~3 shared loads per key instead of d dependent
    // ones (same buckets as the tree descent, classify_lut)
    const LutTree LT = lut_build<T>(tree, d, spl, reinterpret_cast<uint16_t*>(spl + v));
    for (uint32_t b = threadIdx.x; b <= k; b += T) hist[b] = 0;
    if (threadIdx.x == 0) {
        for (uint32_t q = 0; q < NS; ++q) mbar_init(&bar[q], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();  // the sample's shared memory is the ring from here on

    // one ring sequence over both passes: tile q of the segment's pass A
    // (keys), then of pass B (keys + offsets); slot q % NS, parity (q / NS) & 1
    const uint32_t ntiles = (s.size + TILE - 1) / TILE;
    auto issue = [&](uint32_t q) {
        const bool pass_b = q >= ntiles;
        const uint32_t base = (pass_b ? q - ntiles : q) * TILE;
        const uint32_t cnt = min(TILE, s.size - base);
        NarrowStage& S = ring[q % NS];
        uint32_t tx = 0;
        bulk_in(S.key, key + base, cnt, &bar[q % NS], tx);
        if (pass_b) bulk_in(S.off, off + base, cnt, &bar[q % NS], tx);
        mbar_expect_tx(&bar[q % NS], tx);
    };
    if (threadIdx.x == 0)
        for (uint32_t q = 0; q < NS && q < 2 * ntiles; ++q) issue(q);

    // stage 2: classify + count (samplesort.py:51-113), tile by tile
    for (uint32_t q = 0; q < ntiles; ++q) {
        const uint32_t base = q * TILE, cnt = min(TILE, s.size - base);
        const uint32_t shk = elem_shift(key + base, 8);
        mbar_wait(&bar[q % NS], (q / NS) & 1u);
        const NarrowStage& S = ring[q % NS];
        uint64_t kk[IT];
        uint32_t bb[IT];
#pragma unroll
        for (uint32_t j = 0; j < IT; ++j) {
            const uint32_t e = j * T + threadIdx.x;
            kk[j] = e < cnt ? S.key[e + shk] : 0;
        }
        if (EQUAL) {
            classify_iw<true, IT>(kk, tree, d, bb);
        } else {
#pragma unroll
            for (uint32_t j = 0; j < IT; ++j) bb[j] = classify_lut(kk[j], LT);
        }
#pragma unroll
        for (uint32_t j = 0; j < IT; ++j)
            if (j * T + threadIdx.x < cnt) atomicAdd(&hist[bb[j]], 1u);
        __syncthreads();  // every read of this slot is done: refill it
        if (threadIdx.x == 0 && q + NS < 2 * ntiles) {
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            issue(q + NS);
        }
    }

    // stage 3: bucket starts and children (bucket_layout, classifier.py:284-304)
    block_exclusive_scan<T>(hist, k, warp_sums);
    for (uint32_t b = threadIdx.x; b <= k; b += T) cur[b] = hist[b];
    emit_block<T>(A, s, hist, k, tree, d, &es);
    __syncthreads();

    // stage 4: distribution (samplesort.py:146-152): classify again, slot
    // from the bucket's cursor
    const uint32_t k2m = k2_kind(A, s);
    for (uint32_t t = 0; t < ntiles; ++t) {
        const uint32_t q = ntiles + t;
        const uint32_t base = t * TILE, cnt = min(TILE, s.size - base);
        const uint32_t shk = elem_shift(key + base, 8), sho = elem_shift(off + base, 4);
        mbar_wait(&bar[q % NS], (q / NS) & 1u);
        const NarrowStage& S = ring[q % NS];
        uint64_t kk[IT];
        uint32_t oo[IT], bb[IT];
#pragma unroll
        for (uint32_t j = 0; j < IT; ++j) {
            const uint32_t e = j * T + threadIdx.x;
            kk[j] = e < cnt ? S.key[e + shk] : 0;
            oo[j] = e < cnt ? S.off[e + sho] : 0;
        }
        if (EQUAL) {
            classify_iw<true, IT>(kk, tree, d, bb);
        } else {
#pragma unroll
            for (uint32_t j = 0; j < IT; ++j) bb[j] = classify_lut(kk[j], LT);
        }
        uint32_t rr[IT];
#pragma unroll
        for (uint32_t j = 0; j < IT; ++j)
            rr[j] = j * T + threadIdx.x < cnt ? atomicAdd(&cur[bb[j]], 1u) : 0u;
#pragma unroll
        for (uint32_t j = 0; j < IT; ++j) {
            const uint32_t e = j * T + threadIdx.x;
            const uint32_t b = bb[j], r = rr[j];
            if (e < cnt) {
                const uint32_t st = hist[b], end = hist[b + 1];
                const bool fin = end - st == 1 || ((b & 1) && has_zero_byte(kk[j]));
                place_k2(A, s, b, fin, r, end, oo[j], kk[j], k2m, s.begin + base + e, fetches);
            }
        }
        __syncthreads();
        if (threadIdx.x == 0 && q + NS < 2 * ntiles) {
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            issue(q + NS);
        }
    }
    for (uint32_t x = 16; x > 0; x >>= 1) fetches += __shfl_xor_sync(0xffffffffu, fetches, x);
    if (lane == 0 && fetches) atomicAdd(&A.ctl->fetches, fetches);
}

// ---------------------------------------------------------------------------
// wide tier (segments > narrow_max): the fully parallel step of
// samplesort.py:369-434 with CTAs as workers.

struct WidePlan {
    const Seg* segs;
    uint32_t nsegs;
    uint32_t* cta_start;   // [nsegs + 1]
    uint64_t* tree_off;    // [nsegs]  u64 words into tree_pool
    uint64_t* hist_off;    // [nsegs]  u32 words into hist_pool: C rows of k, then k+1 starts
    uint64_t* tree_pool;
    uint32_t* hist_pool;
    uint16_t* bkt;         // [n] bucket of every string of the level's wide segments
    uint64_t tree_cap, hist_cap;
};

struct WideGeom {
    uint32_t d, v, k, C;
};

// Wide step geometry: the fan-out aims at children of ~wide_target strings
// (the next level then finishes them in k_local), capped at wide_dcap; the
// CTA count keeps each CTA's contiguous chunk >= kWideChunkMin strings and the
// write frontier (C x k cursors) small enough to stay resident in L2.
__device__ __forceinline__ WideGeom wide_geom(const Seg& s, const SortArgs& A) {
    WideGeom g;
    uint32_t dcap = A.dmax < A.wide_dcap ? A.dmax : A.wide_dcap;
    uint32_t d = ceil_log2((s.size + A.wide_target - 1) / A.wide_target);
    g.d = d < 1 ? 1 : (d > dcap ? dcap : d);
    g.v = (1u << g.d) - 1;
    g.k = 2 * g.v + 1;
    uint32_t c = (s.size + A.wide_chunk - 1) / A.wide_chunk;
    uint32_t cmax = kWideFrontier / g.k;
    cmax = cmax < 1 ? 1 : (cmax > kWideCtasMax ? kWideCtasMax : cmax);
    g.C = c < 1 ? 1 : (c > cmax ? cmax : c);
    // a segment that fills the machine on its own (the root): whole waves of
    // CTAs -- 512 equal chunks on 148 SMs left the count's second wave (3 CTAs
    // per SM resident) and the scatter's fourth (1 per SM) mostly empty
    if (A.sm_count && g.C >= A.sm_count) g.C -= g.C % A.sm_count;
    return g;
}

// Exclusive scans of CTA counts and pool sizes over the wide segments.
__global__ void __launch_bounds__(1024) k_wide_plan(SortArgs A, WidePlan P) {
    // the level's wide segment count straight from the control block: the
    // plan is enqueued before the host has read it (overlapping the level gap)
    const uint32_t nsegs = A.ctl->n_list[WIDE];
    __shared__ unsigned long long s_carry[3];
    __shared__ unsigned long long s_w[3][32];
    if (threadIdx.x == 0) s_carry[0] = s_carry[1] = s_carry[2] = 0;
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (uint32_t base = 0; base < nsegs; base += 1024) {
        uint32_t i = base + threadIdx.x;
        unsigned long long x[3] = {0, 0, 0};
        if (i < nsegs) {
            WideGeom g = wide_geom(P.segs[i], A);
            x[0] = g.C;
            x[1] = 2 * g.v + 1 + kLutWords;
            x[2] = static_cast<unsigned long long>(g.C) * g.k + g.k + 2;  // + the solo flag
        }
        unsigned long long incl[3];
        for (int q = 0; q < 3; ++q) {
            unsigned long long y = x[q];
            for (uint32_t o = 1; o < 32; o <<= 1) {
                unsigned long long z = __shfl_up_sync(0xffffffffu, y, o);
                if (lane >= o) y += z;
            }
            incl[q] = y;
            if (lane == 31) s_w[q][w] = y;
        }
        __syncthreads();
        if (w == 0) {
            for (int q = 0; q < 3; ++q) {
                unsigned long long y = s_w[q][lane];
                for (uint32_t o = 1; o < 32; o <<= 1) {
                    unsigned long long z = __shfl_up_sync(0xffffffffu, y, o);
                    if (lane >= o) y += z;
                }
                s_w[q][lane] = y;
            }
        }
        __syncthreads();
        if (i < nsegs) {
            unsigned long long e[3];
            for (int q = 0; q < 3; ++q)
                e[q] = s_carry[q] + incl[q] - x[q] + (w ? s_w[q][w - 1] : 0ull);
            P.cta_start[i] = static_cast<uint32_t>(e[0]);
            P.tree_off[i] = e[1];
            P.hist_off[i] = e[2];
        }
        __syncthreads();
        if (threadIdx.x == 0)
            for (int q = 0; q < 3; ++q) s_carry[q] += s_w[q][31];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        P.cta_start[nsegs] = static_cast<uint32_t>(s_carry[0]);
        A.ctl->wide_ctas = static_cast<uint32_t>(s_carry[0]);
        A.ctl->tree_words = s_carry[1];
        A.ctl->hist_words = s_carry[2];
        if (s_carry[1] > P.tree_cap || s_carry[2] > P.hist_cap) {
            atomicOr(&A.ctl->plan_err, ERR_POOL);
            A.ctl->wide_ctas = 0;  // skip the level's wide kernels; host reports the error
        }
    }
}

// Sample + splitter tree per wide segment (one CTA each).
#ifndef S5_TREE_THREADS
#define S5_TREE_THREADS 512
#endif
constexpr uint32_t kTreeThreads = S5_TREE_THREADS;  // one CTA per wide segment

// TT threads per CTA: kTreeThreads in general, kTreeThreadsFew for levels
// with few wide segments (the root), where the one CTA's sample sort is on
// the critical path of the level
constexpr uint32_t kTreeThreadsFew = 1024;

// The level driver enqueues this kernel right behind the plan, before the
// host has read the level's control block (the trees are built while the
// host wakes up and launches the rest of the level): `nsegs` = 0 then, and the
// segment count comes from the control block (not yet reset for the level);
// a level with more wide segments than that launch's grid gets a second
// launch (seg_base, nsegs from the host) for the rest.
template <uint32_t TT>
__global__ void __launch_bounds__(TT) k_wide_tree(SortArgs A, WidePlan P, uint32_t seg_base,
                                                 uint32_t nsegs) {
    extern __shared__ __align__(16) uint8_t sm[];
    if (A.ctl->wide_ctas == 0) return;
    const uint32_t si = seg_base + blockIdx.x;
    if (si >= (nsegs ? nsegs : A.ctl->n_list[WIDE])) return;
    const uint32_t dw = A.dmax < A.wide_dcap ? A.dmax : A.wide_dcap;
    uint64_t* sample = reinterpret_cast<uint64_t*>(sm);
    int32_t* na = reinterpret_cast<int32_t*>(sm + A.wide_sample * 8);
    int32_t* nb = na + (1u << dw);
    uint32_t* nf = reinterpret_cast<uint32_t*>(nb + (1u << dw));
    const Seg s = P.segs[si];
    const WideGeom g = wide_geom(s, A);
    uint32_t m = A.alpha * g.v;
    if (m > kWideSampleCap) m = kWideSampleCap;
    uint32_t M = 64;
    while (M < m) M <<= 1;
    const uint64_t* __restrict__ key = A.key[sd(s)] + s.begin;
    const uint64_t sseed = segment_seed(A.seed, s.begin, s.size, s.depth);
    __shared__ uint32_t bytemask[8][8];  // root: byte values seen per key position
    // level 0 may sample twice: when the first sample's keys share 2..7 whole
    // bytes, the segment moves that many bytes deeper (Ctl::skip) and the
    // splitters come from a second sample of the keys behind the prefix
    uint32_t skip = 0;
#pragma unroll 1
    for (uint32_t pass = 0;; ++pass) {
        if (threadIdx.x < 64) bytemask[threadIdx.x >> 3][threadIdx.x & 7] = 0;
        __syncthreads();
        for (uint32_t t = threadIdx.x; t < M; t += TT) {
            uint64_t x = ~0ull;
            if (t < m) {
                const uint32_t idx = sample_index(sseed, t, s.size);
                if (A.root || A.root32) {  // level 0: keys are not gathered yet
                    const int64_t h = root_handle(A, s.begin + idx);
                    x = (h >= 0 && static_cast<uint64_t>(h) + s.depth + skip < A.arena_len)
                            ? load_key(A.arena, static_cast<uint64_t>(h) + s.depth + skip) : 0;
                } else {
                    x = key[idx];
                }
                if (A.k2_stage == 1 && t < 256) {  // 256 random samples suffice for the estimate
#pragma unroll
                    for (uint32_t j = 0; j < 8; ++j) {
                        const uint32_t v = static_cast<uint32_t>(x >> (56 - 8 * j)) & 0xFFu;
                        atomicOr(&bytemask[j][v >> 5], 1u << (v & 31));
                    }
                }
            }
            sample[t] = x;
        }
        __syncthreads();
        if (pass == 1 || A.k2_stage != 1 || !(A.root || A.root32) || (A.flags & 16384)) break;
        sort_sample<TT>(sample, M);
        const uint64_t lo_k = sample[0], hi_k = sample[m - 1];
        uint32_t L = lo_k == hi_k ? 8u : diff_bytes(lo_k, hi_k);
        const uint32_t z = zero_index(lo_k);
        L = L < z ? L : z;
        __syncthreads();  // every thread has read the extremes: the sample may be redrawn
        if (L < 2 || L > 7) {
            skip = 0xFFFFFFFFu;  // sorted already, no skip
            break;
        }
        skip = L;
        if (threadIdx.x == 0) {
            A.ctl->skip = L;
            A.ctl->skip_prefix = lo_k >> (64 - 8 * L);
            const_cast<Seg*>(P.segs)[si].depth = s.depth + L;
        }
    }
    if (A.k2_stage == 1 && threadIdx.x == 0) {
        // distinct 8-byte keys <= product of the distinct byte values per
        // position; far fewer than the strings -> level 1 is dominated by
        // equality buckets, whose next words are cheapest to read now
        double est = 1.0;
        for (uint32_t j = 0; j < 8; ++j) {
            uint32_t c = 0;
            for (uint32_t q = 0; q < 8; ++q) c += __popc(bytemask[j][q]);
            est *= c ? c : 1;
        }
        // (and only when the root's children will be S^5 steps themselves)
        A.ctl->k2 = (A.flags & 256) == 0 && static_cast<double>(s.size) > 16.0 * est &&
                    s.size / (g.v + 1) > A.local_max;
    }
    if (skip != 0xFFFFFFFFu) sort_sample<TT>(sample, M);
    if (A.k2_stage == 1) {
        // the keys' entropy from the root sample: when nearly every sampled
        // key has its own leading 3-byte window, the one-CTA local tiers sort
        // on 32-bit words (a window + the slot) -- low-entropy data (DNA,
        // Markov text, URLs) would only turn them into candidate runs
        uint32_t same = 0;
        for (uint32_t t = 1 + threadIdx.x; t < m; t += TT)
            same += (sample[t] >> 40) == (sample[t - 1] >> 40);
        same = __reduce_add_sync(0xffffffffu, same);
        __shared__ uint32_t s_same;
        if (threadIdx.x == 0) s_same = 0;
        __syncthreads();
        if ((threadIdx.x & 31) == 0) atomicAdd(&s_same, same);
        __syncthreads();
        if (threadIdx.x == 0) A.ctl->w32 = (A.flags & 2048) == 0 && m >= 256 && s_same * 64 <= m;
    }
    uint64_t* tree = P.tree_pool + P.tree_off[si];
    build_tree_levels<TT>(sample, m, g.d, tree, na, nb, nf);
    // classification table for k_wide_count, once per segment
    uint64_t* spl = tree + g.v + 1;
    const LutTree T = lut_build<TT>(tree, g.d, spl, reinterpret_cast<uint16_t*>(spl + g.v));
    if (threadIdx.x == 0) {
        spl[g.v + kLutTabWords] = T.pf;
        spl[g.v + kLutTabWords + 1] = T.lb;
    }
}

__device__ __forceinline__ uint32_t find_seg(const uint32_t* cta_start, uint32_t nsegs,
                                             uint32_t g) {
    uint32_t lo = 0, hi = nsegs;  // last s with cta_start[s] <= g
    while (hi - lo > 1) {
        uint32_t mid = (lo + hi) >> 1;
        if (cta_start[mid] <= g) lo = mid; else hi = mid;
    }
    return lo;
}

// Per-CTA histogram of a contiguous chunk (stage 2, samplesort.py:383-400).
// Every string's bucket is kept (u16, 2 B) so the scatter does not classify
// again.
// Level 0 of k_wide_count with second key words: handle -> (offset, key,
// next word) gather fused with the classification and the histogram.
// SKIP: the segment sits Ctl::skip bytes behind the sort depth (root prefix
// skip); every string's skipped bytes are checked against the prefix.
template <bool K2, bool IDX = false, bool SKIP = false>
__device__ __forceinline__ void root_gather_count(const SortArgs& A, const Seg& s, uint32_t lo,
                                                  uint32_t hi, const LutTree& T, uint32_t* hist,
                                                  uint16_t* __restrict__ bkt) {
    constexpr int R = 4;  // (8 would lift the whole count kernel's register budget)
    const uint32_t skip = SKIP ? A.ctl->skip : 0u;
    const uint64_t prefix = SKIP ? A.ctl->skip_prefix : 0ull;
    bool mismatch = false;
#pragma unroll 1
    for (uint32_t base = lo; base < hi; base += R * kWideThreads) {
        int64_t hh[R];
        uint64_t kk[R], k2w[R];
#pragma unroll
        for (int j = 0; j < R; ++j) {
            const uint32_t i = base + j * kWideThreads + threadIdx.x;
            hh[j] = i < hi ? root_handle(A, s.begin + i) : 0;
        }
#pragma unroll
        for (int j = 0; j < R; ++j) {
            const uint32_t i = base + j * kWideThreads + threadIdx.x;
            if (i < hi && (hh[j] < 0 || static_cast<uint64_t>(hh[j]) + s.depth - skip >= A.arena_len)) {
                atomicOr(&A.ctl->err, ERR_RANGE);
                hh[j] = 0;
            }
            kk[j] = k2w[j] = 0;
            if (i < hi) {
                if (SKIP)  // a terminator inside the skipped bytes fails the check too
                    mismatch |= (load_key(A.arena, static_cast<uint64_t>(hh[j]) + s.depth - skip) >>
                                 (64 - 8 * skip)) != prefix;
                if (K2) load_key2(A.arena, static_cast<uint64_t>(hh[j]) + s.depth, kk[j], k2w[j]);
                else kk[j] = load_key(A.arena, static_cast<uint64_t>(hh[j]) + s.depth);
            }
        }
#pragma unroll
        for (int j = 0; j < R; ++j) {
            const uint32_t i = base + j * kWideThreads + threadIdx.x;
            if (i < hi) {
                if (IDX) {  // index mode: the offset word names the string, pos its arena position
                    A.pos[s.begin + i] = hh[j];
                    A.off[0][s.begin + i] = s.begin + i;
                } else {
                    A.off[0][s.begin + i] = static_cast<uint32_t>(hh[j]);
                }
                A.key[0][s.begin + i] = kk[j];
                if (K2) A.key2[0][s.begin + i] = k2w[j];
                const uint32_t b = classify_lut(kk[j], T);
                atomicAdd(&hist[b], 1u);
                bkt[i] = static_cast<uint16_t>(b);
            }
        }
    }
    if (SKIP && mismatch) atomicOr(&A.ctl->skip_fail, 1u);
}

// IDX: the level-0 launch of index mode; SKIP: the level-0 launch behind a
// root prefix skip.  Their own instantiations: the position table stores and
// the prefix check would cost the common kernel registers and a CTA per SM.
// The tree kernel decides the skip on the device right before, so level 0
// launches both the plain and the SKIP kernel and the wrong one returns.
template <bool EQUAL, bool IDX = false, bool SKIP = false>
__global__ void __launch_bounds__(kWideThreads) k_wide_count(SortArgs A, WidePlan P) {
    extern __shared__ __align__(16) uint8_t sm[];
    const uint32_t G = blockIdx.x;
    if (G >= A.ctl->wide_ctas) return;
    if (A.k2_stage == 1 && (A.ctl->skip != 0) != SKIP) return;
    uint64_t* tree = reinterpret_cast<uint64_t*>(sm);
    uint32_t* hist = reinterpret_cast<uint32_t*>(sm + (1u << A.wide_dcap) * 8);
    uint64_t* splitters = reinterpret_cast<uint64_t*>(hist + (2u << A.wide_dcap) + 2);
    const uint32_t si = find_seg(P.cta_start, P.nsegs, G);
    const Seg s = P.segs[si];
    const WideGeom g = wide_geom(s, A);
    const uint32_t c = G - P.cta_start[si];
    const uint32_t chunk = (s.size + g.C - 1) / g.C;
    const uint32_t lo = c * chunk;
    const uint32_t hi = min(s.size, lo + chunk);
    const uint64_t* tsrc = P.tree_pool + P.tree_off[si];
    if (EQUAL) {
        for (uint32_t i = threadIdx.x; i <= g.v; i += kWideThreads) tree[i] = tsrc[i];
    } else {  // splitters in order + classification table, prepared by k_wide_tree
        const uint64_t* src = tsrc + g.v + 1;
        uint64_t* dst = splitters;  // splitters then lut, contiguous as in the pool
        for (uint32_t i = threadIdx.x; i < g.v + kLutTabWords; i += kWideThreads) dst[i] = src[i];
    }
    for (uint32_t b = threadIdx.x; b < g.k; b += kWideThreads) hist[b] = 0;
    __syncthreads();
    const uint64_t* __restrict__ key = A.key[sd(s)] + s.begin;
    uint16_t* __restrict__ bkt = P.bkt + s.begin;
    if (!EQUAL) {  // table classification (same buckets, fewer dependent loads)
        LutTree T;
        T.s = splitters;
        T.lut = reinterpret_cast<const uint16_t*>(splitters + g.v);
        T.v = g.v;
        T.pf = tsrc[2 * g.v + 1 + kLutTabWords];
        T.lb = static_cast<uint32_t>(tsrc[2 * g.v + 1 + kLutTabWords + 1]);
        if (A.root || A.root32) {  // level 0: handle -> (offset, key) gather fused with the count
            if (IDX || SKIP) {  // index mode (arenas >= 4 GiB) / root prefix skip
                if (A.k2_stage == 1 && A.ctl->k2) root_gather_count<true, IDX, SKIP>(A, s, lo, hi, T, hist, bkt);
                else root_gather_count<false, IDX, SKIP>(A, s, lo, hi, T, hist, bkt);
            } else if (A.k2_stage == 1 && A.ctl->k2) {
                root_gather_count<true>(A, s, lo, hi, T, hist, bkt);
            } else {
                constexpr int R = 8;
#pragma unroll 1
                for (uint32_t base = lo; base < hi; base += R * kWideThreads) {
                    int64_t hh[R];
                    uint64_t kk[R];
#pragma unroll
                    for (int j = 0; j < R; ++j) {
                        const uint32_t i = base + j * kWideThreads + threadIdx.x;
                        hh[j] = i < hi ? root_handle(A, s.begin + i) : 0;
                    }
#pragma unroll
                    for (int j = 0; j < R; ++j) {
                        const uint32_t i = base + j * kWideThreads + threadIdx.x;
                        if (i < hi && (hh[j] < 0 || static_cast<uint64_t>(hh[j]) + s.depth >= A.arena_len)) {
                            atomicOr(&A.ctl->err, ERR_RANGE);
                            hh[j] = 0;
                        }
                        kk[j] = i < hi ? load_key(A.arena, static_cast<uint64_t>(hh[j]) + s.depth) : 0;
                    }
#pragma unroll
                    for (int j = 0; j < R; ++j) {
                        const uint32_t i = base + j * kWideThreads + threadIdx.x;
                        if (i < hi) {
                            A.off[0][s.begin + i] = static_cast<uint32_t>(hh[j]);
                            A.key[0][s.begin + i] = kk[j];
                            const uint32_t b = classify_lut(kk[j], T);
                            atomicAdd(&hist[b], 1u);
                            bkt[i] = static_cast<uint16_t>(b);
                        }
                    }
                }
            }
            __syncthreads();
            uint32_t* row = P.hist_pool + P.hist_off[si] + static_cast<uint64_t>(c) * g.k;
            for (uint32_t b = threadIdx.x; b < g.k; b += kWideThreads) row[b] = hist[b];
            return;
        }
        uint64_t nx[4];  // keys of the next round, loaded one round ahead
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            uint32_t i = lo + j * kWideThreads + threadIdx.x;
            nx[j] = i < hi ? __ldcs(key + i) : 0;
        }
        for (uint32_t base = lo; base < hi; base += 4 * kWideThreads) {
            uint64_t kk[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                kk[j] = nx[j];
                uint32_t i = base + (4 + j) * kWideThreads + threadIdx.x;
                nx[j] = i < hi ? __ldcs(key + i) : 0;
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                uint32_t i = base + j * kWideThreads + threadIdx.x;
                if (i < hi) {
                    uint32_t b = classify_lut(kk[j], T);
                    atomicAdd(&hist[b], 1u);
                    bkt[i] = static_cast<uint16_t>(b);
                }
            }
        }
        __syncthreads();
        uint32_t* row = P.hist_pool + P.hist_off[si] + static_cast<uint64_t>(c) * g.k;
        for (uint32_t b = threadIdx.x; b < g.k; b += kWideThreads) row[b] = hist[b];
        return;
    }
    constexpr int IW = kWideItems;
    for (uint32_t base = lo; base < hi; base += IW * kWideThreads) {
        uint64_t kk[IW];
        uint32_t b[IW];
#pragma unroll
        for (int j = 0; j < IW; ++j) {
            uint32_t i = base + j * kWideThreads + threadIdx.x;
            kk[j] = i < hi ? __ldcs(key + i) : 0;
        }
        classify_iw<EQUAL, IW>(kk, tree, g.d, b);
#pragma unroll
        for (int j = 0; j < IW; ++j) {
            uint32_t i = base + j * kWideThreads + threadIdx.x;
            if (i < hi) {
                atomicAdd(&hist[b[j]], 1u);
                bkt[i] = static_cast<uint16_t>(b[j]);
            }
        }
    }
    __syncthreads();
    uint32_t* row = P.hist_pool + P.hist_off[si] + static_cast<uint64_t>(c) * g.k;
    for (uint32_t b = threadIdx.x; b < g.k; b += kWideThreads) row[b] = hist[b];
}

// Column prefix over the C rows of every bucket (the worker-major cursor scan
// of samplesort.py:402-410); totals land in the bucket-start area.
// One CTA per (segment, 32 buckets): lane = bucket, the NW warps split the C
// rows; per-warp column sums, a prefix over the warps in shared memory, then
// every warp rewrites its rows as running exclusive prefixes (row reads and
// writes are 128-byte coalesced).
template <uint32_t NW>
__global__ void __launch_bounds__(NW * 32) k_wide_colscan(SortArgs A, WidePlan P) {
    __shared__ uint32_t part[NW][33];
    if (A.ctl->wide_ctas == 0) return;
    const uint32_t si = blockIdx.x;
    const Seg s = P.segs[si];
    const WideGeom g = wide_geom(s, A);
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint32_t b = blockIdx.y * 32 + lane;
    if (blockIdx.y * 32 >= g.k) return;
    uint32_t* rows = P.hist_pool + P.hist_off[si];
    const uint32_t R = (g.C + NW - 1) / NW;
    const uint32_t r0 = min(g.C, w * R), r1 = min(g.C, r0 + R);
    uint32_t sum = 0;
    if (b < g.k) {
#pragma unroll 4
        for (uint32_t c = r0; c < r1; ++c) sum += rows[static_cast<uint64_t>(c) * g.k + b];
    }
    part[w][lane] = sum;
    __syncthreads();
    uint32_t run = 0;
    for (uint32_t q = 0; q < w; ++q) run += part[q][lane];
    if (b < g.k) {
        for (uint32_t c = r0; c < r1; ++c) {
            const uint64_t at = static_cast<uint64_t>(c) * g.k + b;
            const uint32_t x = rows[at];
            rows[at] = run;
            run += x;
        }
        if (w == NW - 1) rows[static_cast<uint64_t>(g.C) * g.k + b] = run;
    }
}

// The same scan with BW < 32 buckets per CTA, for levels with few wide
// segments (the root: C ~ 1000 rows x k ~ 1000 buckets would otherwise be
// ~32 CTAs on the level's critical path).  A warp reads G = 32 / BW rows at
// a time (BW consecutive buckets each, whole sectors for BW >= 8); the rows'
// running prefix is a shuffle scan over the G row lanes of each bucket.
template <uint32_t NW, uint32_t BW>
__global__ void __launch_bounds__(NW * 32) k_wide_colscan_g(SortArgs A, WidePlan P) {
    constexpr uint32_t G = 32 / BW;
    __shared__ uint32_t part[NW][BW];
    if (A.ctl->wide_ctas == 0) return;
    const uint32_t si = blockIdx.x;
    const Seg s = P.segs[si];
    const WideGeom g = wide_geom(s, A);
    if (blockIdx.y * BW >= g.k) return;
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint32_t sub = lane / BW, col = lane % BW, b = blockIdx.y * BW + col;
    uint32_t* rows = P.hist_pool + P.hist_off[si];
    const uint32_t R = (g.C + NW - 1) / NW;
    const uint32_t r0 = min(g.C, w * R), r1 = min(g.C, r0 + R);
    uint32_t sum = 0;
    if (b < g.k) {
#pragma unroll 4
        for (uint32_t c = r0 + sub; c < r1; c += G) sum += rows[static_cast<uint64_t>(c) * g.k + b];
    }
#pragma unroll
    for (uint32_t o = BW; o < 32; o <<= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (sub == 0) part[w][col] = sum;
    __syncthreads();
    uint32_t run = 0;
    for (uint32_t q = 0; q < w; ++q) run += part[q][col];
    for (uint32_t c0 = r0; c0 < r1; c0 += G) {  // warp-uniform
        const uint32_t c = c0 + sub;
        const bool ok = b < g.k && c < r1;
        const uint64_t at = static_cast<uint64_t>(c) * g.k + b;
        const uint32_t x = ok ? rows[at] : 0u;
        uint32_t inc = x;
#pragma unroll
        for (uint32_t o = BW; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        if (ok) rows[at] = run + inc - x;
        run += __shfl_sync(0xffffffffu, inc, (G - 1) * BW + col);
    }
    if (w == NW - 1 && sub == 0 && b < g.k) rows[static_cast<uint64_t>(g.C) * g.k + b] = run;
}

// Bucket starts (stage 3) and the per-bucket epilogue (children, LCP hints).
__global__ void __launch_bounds__(256) k_wide_bscan(SortArgs A, WidePlan P) {
    __shared__ uint32_t warp_sums[32];
    if (A.ctl->wide_ctas == 0) return;
    const uint32_t si = blockIdx.x;
    const Seg s = P.segs[si];
    const WideGeom g = wide_geom(s, A);
    uint32_t* starts = P.hist_pool + P.hist_off[si] + static_cast<uint64_t>(g.C) * g.k;
    block_exclusive_scan<256>(starts, g.k, warp_sums);
    const uint64_t* tree = P.tree_pool + P.tree_off[si];
    // one equality bucket of an unterminated splitter holding the whole
    // segment: every key is equal, so the segment stays where it is and only
    // its keys advance 8 bytes (the scatter does that in place, reading the
    // flag starts[k + 1] = bucket + 1) -- the equality-bucket chain of a
    // shared prefix (classifier.py:297-303) without moving a string
    __shared__ uint32_t solo;
    if (threadIdx.x == 0) solo = 0;
    __syncthreads();
    for (uint32_t b = 1 + 2 * threadIdx.x; b < g.k; b += 2 * 256)
        if (starts[b + 1] - starts[b] == s.size && !has_zero_byte(tree[node_of_rank(b >> 1, g.d)]))
            solo = b + 1;
    __syncthreads();
    if (threadIdx.x == 0) starts[g.k + 1] = solo;
    if (solo) {
        // Seg.side bits 8..15 count the levels a segment has stayed whole.  A
        // shared prefix of P bytes costs a wide segment P / 8 levels; from the
        // fourth on, a segment the one-CTA step can hold goes to k_narrow, whose
        // in-place prefix skip walks the rest of the prefix inside one kernel
        if (threadIdx.x == 0) {
            const uint32_t streak = min(255u, ((s.side >> 8) & 0xFFu) + 1u);
            const bool walk = streak >= 4 && s.size <= kNarrowMaxSize && s.size > A.local_max;
            emit_child(A, s.begin, s.size, s.depth + 8,
                       sd(s) | (k2_kind(A, s) == K2_MAKE ? 2u : 0u) | (streak << 8),
                       walk ? static_cast<int>(NARROW) : -1);
        }
        return;
    }
    __shared__ EmitScratch es;
    emit_block<256>(A, s, starts, g.k, tree, g.d, &es);
}

// The scatter of a segment whose keys are all equal (k_wide_bscan's solo
// flag): keys advance 8 bytes in place -- the carried second words when the
// root gathered them, else one arena fetch per string.
__device__ __forceinline__ void advance_keys(const SortArgs& A, const Seg& s, uint32_t lo, uint32_t hi,
                                             uint32_t threads, unsigned long long& fetches) {
    const uint32_t k2m = k2_kind(A, s);
    const uint32_t* __restrict__ off = A.off[sd(s)] + s.begin;
    uint64_t* key = A.key[sd(s)] + s.begin;
    uint64_t* key2 = A.key2[sd(s)] + s.begin;
    for (uint32_t i = lo + threadIdx.x; i < hi; i += threads) {
        if (k2m == K2_ROOT || k2m == K2_LEVEL1) {
            key[i] = __ldcs(A.key2[k2m - 1] + s.begin + i);
        } else if (k2m == K2_USE) {
            key[i] = __ldcs(key2 + i);
        } else if (k2m == K2_MAKE) {  // the child (this range, k2-valid) keeps the word after
            uint64_t k0, k1;
            load_key2(A.arena, apos(A, __ldcs(off + i)) + s.depth + 8, k0, k1);
            key[i] = k0;
            key2[i] = k1;
            ++fetches;
        } else {
            key[i] = load_key(A.arena, apos(A, __ldcs(off + i)) + s.depth + 8);
            ++fetches;
        }
    }
}

// Out-of-place distribution with per-CTA cursors (stage 4, samplesort.py:412-417).
// Tiles of kWideTile strings are first grouped by bucket in shared memory, so
// each bucket's run of a tile leaves as consecutive addresses (coalesced,
// whole sectors) instead of one scattered 4 B + 8 B store per string.
struct WideScatterSmem {
    static constexpr uint32_t kcap = 2u << kWideDMax;
    static constexpr uint32_t total = (3 * kcap + 8) * 4 + kWideTile * (8 + 4 + 2 + 2) + 64 * 4;
    // shared memory for a launch whose trees have depth <= dcap (k2: with the
    // tile's source indices for second key words)
    __host__ __device__ static constexpr uint32_t bytes(uint32_t dcap, bool k2) {
        return (3 * (2u << dcap) + 8) * 4 + kWideTile * (8 + 4 + 2 + (k2 ? 2 : 0)) + 64 * 4;
    }
};

__global__ void __launch_bounds__(kWideThreads) k_wide_scatter(SortArgs A, WidePlan P) {
    extern __shared__ __align__(16) uint8_t sm[];
    const uint32_t G = blockIdx.x;
    if (G >= A.ctl->wide_ctas) return;
    if (A.k2_stage == 1 && A.ctl->skip_fail) return;  // level 0 is redone without the prefix skip
    uint64_t* sk = reinterpret_cast<uint64_t*>(sm);
    uint32_t* so = reinterpret_cast<uint32_t*>(sk + kWideTile);
    uint16_t* sb = reinterpret_cast<uint16_t*>(so + kWideTile);
    uint16_t* sx = sb + kWideTile;  // tile-relative source index (second key words)
    const uint32_t kc = 2u << A.wide_dcap;
    uint32_t* cur = reinterpret_cast<uint32_t*>(A.k2_cap ? sx + kWideTile : sx);
    uint32_t* cnt = cur + kc;
    uint32_t* gb = cnt + kc + 4;
    uint32_t* warp_sums = gb + kc + 4;
    const uint32_t si = find_seg(P.cta_start, P.nsegs, G);
    const Seg s = P.segs[si];
    const WideGeom g = wide_geom(s, A);
    const uint32_t c = G - P.cta_start[si];
    const uint32_t chunk = (s.size + g.C - 1) / g.C;
    const uint32_t lo = c * chunk;
    const uint32_t hi = min(s.size, lo + chunk);
    const uint64_t* tree = P.tree_pool + P.tree_off[si];
    const uint32_t* rows = P.hist_pool + P.hist_off[si];
    const uint32_t* starts = rows + static_cast<uint64_t>(g.C) * g.k;
    if (starts[g.k + 1]) {  // all keys equal: advance them in place
        unsigned long long fetches = 0;
        advance_keys(A, s, lo, hi, kWideThreads, fetches);
        for (uint32_t x = 16; x > 0; x >>= 1) fetches += __shfl_xor_sync(0xffffffffu, fetches, x);
        if ((threadIdx.x & 31) == 0 && fetches) atomicAdd(&A.ctl->fetches, fetches);
        return;
    }
    for (uint32_t b = threadIdx.x; b < g.k; b += kWideThreads) {
        uint32_t st = starts[b], n_b = starts[b + 1] - st;
        bool fin = n_b == 1 || ((b & 1) && has_zero_byte(tree[node_of_rank(b >> 1, g.d)]));
        cur[b] = (st + rows[static_cast<uint64_t>(c) * g.k + b]) | (fin ? 0x80000000u : 0u);
    }
    const uint32_t* __restrict__ off = A.off[sd(s)] + s.begin;
    const uint64_t* __restrict__ key = A.key[sd(s)] + s.begin;
    const uint16_t* __restrict__ bkt = P.bkt + s.begin;
    const uint32_t lane = threadIdx.x & 31;
    unsigned long long fetches = 0;
    const uint32_t k2m = k2_kind(A, s);
    const bool need_src = k2m != K2_NONE && k2m != K2_MAKE;  // sx: the source index of a slot
    constexpr uint32_t IT = kWideTile / kWideThreads;
    uint64_t kk[IT];
    uint32_t oo[IT], br[IT];  // bucket | rank-in-tile << 16
    // tile loads are issued one tile ahead: the loads of tile t+1 are in
    // flight while tile t is written out
    auto load_tile = [&](uint32_t base) {
#pragma unroll
        for (uint32_t j = 0; j < IT; ++j) {
            uint32_t i = base + j * kWideThreads + threadIdx.x;
            if (i < hi) {
                kk[j] = __ldcs(key + i);
                oo[j] = __ldcs(off + i);
                br[j] = __ldcs(bkt + i);
            }
        }
    };
    if (lo < hi) load_tile(lo);
    for (uint32_t base = lo; base < hi; base += kWideTile) {
        for (uint32_t b = threadIdx.x; b <= g.k; b += kWideThreads) cnt[b] = 0;
        __syncthreads();
#pragma unroll
        for (uint32_t j = 0; j < IT; ++j) {
            uint32_t i = base + j * kWideThreads + threadIdx.x;
            if (i < hi) br[j] |= atomicAdd(&cnt[br[j]], 1u) << 16;
        }
        __syncthreads();
        tile_scan<kWideThreads>(cnt, g.k, cur, gb, warp_sums);
#pragma unroll
        for (uint32_t j = 0; j < IT; ++j) {
            uint32_t i = base + j * kWideThreads + threadIdx.x;
            if (i < hi) {
                uint32_t b = br[j] & 0xFFFFu;
                uint32_t p = cnt[b] + (br[j] >> 16);
                sk[p] = kk[j];
                so[p] = oo[j];
                sb[p] = static_cast<uint16_t>(b);
                if (need_src) sx[p] = static_cast<uint16_t>(j * kWideThreads + threadIdx.x);
            }
        }
        if (base + kWideTile < hi) load_tile(base + kWideTile);
        __syncthreads();
        const uint32_t m = min(kWideTile, hi - base);
        for (uint32_t t = threadIdx.x; t < m; t += kWideThreads) {
            uint32_t b = sb[t];
            uint32_t r = gb[b];
            bool fin = r >> 31;
            uint32_t p = (r & 0x7FFFFFFFu) + (t - cnt[b]);
            uint32_t end = fin && (b & 1) ? starts[b + 1] : 0;
            if (k2m)
                place_k2(A, s, b, fin, p, end, so[t], sk[t], k2m, need_src ? s.begin + base + sx[t] : 0u,
                         fetches);
            else
                place(A, s, b, fin, p, end, so[t], sk[t], fetches);
        }
        __syncthreads();
    }
    for (uint32_t x = 16; x > 0; x >>= 1) fetches += __shfl_xor_sync(0xffffffffu, fetches, x);
    if (lane == 0 && fetches) atomicAdd(&A.ctl->fetches, fetches);
}

// Variant of the distribution with the tile inputs brought in by the bulk
// copy engine (cp.async.bulk, completion on an mbarrier): while tile t is
// ranked and written out, tile t+1 is already in flight into the other
// stage -- no register staging, no load latency on the critical path.  The
// write-out reads each string's key and offset straight from the stage
// through a per-tile position -> element permutation.
template <uint32_t TILE>
struct TmaStage {
    uint64_t key[TILE + 2];
    uint32_t off[TILE + 4];
    uint16_t bkt[TILE + 8];
};

template <uint32_t TILE, uint32_t NS = 2>
struct WideTmaSmem {
    // NS stages | perm u16[tile] | cur, cnt, gb u32[kc] | warp sums | NS mbarriers
    __host__ __device__ static constexpr uint32_t bytes(uint32_t dcap) {
        return NS * static_cast<uint32_t>(sizeof(TmaStage<TILE>)) + TILE * 2 +
               (3 * (2u << dcap) + 8) * 4 + 64 * 4 + 8 * NS;
    }
};

template <uint32_t THREADS, uint32_t TILE, uint32_t NS = 2>
__global__ void __launch_bounds__(THREADS) k_wide_scatter_tma(SortArgs A, WidePlan P) {
    constexpr uint32_t kTmaThreads = THREADS, kTmaTile = TILE;
    using TmaStage = s5::TmaStage<TILE>;
    extern __shared__ __align__(16) uint8_t sm[];
    const uint32_t G = blockIdx.x;
    if (G >= A.ctl->wide_ctas) return;
    if (A.k2_stage == 1 && A.ctl->skip_fail) return;  // level 0 is redone without the prefix skip
    TmaStage* stage = reinterpret_cast<TmaStage*>(sm);
    uint16_t* perm = reinterpret_cast<uint16_t*>(sm + NS * sizeof(TmaStage));
    const uint32_t kc = 2u << A.wide_dcap;
    uint32_t* cur = reinterpret_cast<uint32_t*>(perm + kTmaTile);
    uint32_t* cnt = cur + kc;
    uint32_t* gb = cnt + kc + 4;
    uint32_t* warp_sums = gb + kc + 4;
    uint64_t* bar = reinterpret_cast<uint64_t*>(warp_sums + 64);
    const uint32_t si = find_seg(P.cta_start, P.nsegs, G);
    const Seg s = P.segs[si];
    const WideGeom g = wide_geom(s, A);
    const uint32_t c = G - P.cta_start[si];
    const uint32_t chunk = (s.size + g.C - 1) / g.C;
    const uint32_t lo = c * chunk;
    const uint32_t hi = min(s.size, lo + chunk);
    const uint64_t* tree = P.tree_pool + P.tree_off[si];
    const uint32_t* rows = P.hist_pool + P.hist_off[si];
    const uint32_t* starts = rows + static_cast<uint64_t>(g.C) * g.k;
    if (starts[g.k + 1]) {  // all keys equal: advance them in place
        unsigned long long fetches = 0;
        advance_keys(A, s, lo, hi, kTmaThreads, fetches);
        for (uint32_t x = 16; x > 0; x >>= 1) fetches += __shfl_xor_sync(0xffffffffu, fetches, x);
        if ((threadIdx.x & 31) == 0 && fetches) atomicAdd(&A.ctl->fetches, fetches);
        return;
    }
    const uint32_t* __restrict__ off = A.off[sd(s)] + s.begin;
    const uint64_t* __restrict__ key = A.key[sd(s)] + s.begin;
    const uint16_t* __restrict__ bkt = P.bkt + s.begin;
    auto issue = [&](uint32_t base, uint32_t buf) {
        const uint32_t m = min(kTmaTile, hi - base);
        uint32_t tx = 0;
        bulk_in(stage[buf].key, key + base, m, &bar[buf], tx);
        bulk_in(stage[buf].off, off + base, m, &bar[buf], tx);
        bulk_in(stage[buf].bkt, bkt + base, m, &bar[buf], tx);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n"
                     :: "r"(smem_u32(&bar[buf])), "r"(tx) : "memory");
    };
    if (threadIdx.x == 0) {
        for (uint32_t q = 0; q < NS; ++q)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" :: "r"(smem_u32(&bar[q])) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    for (uint32_t b = threadIdx.x; b < g.k; b += kTmaThreads) {
        uint32_t st = starts[b], n_b = starts[b + 1] - st;
        bool fin = n_b == 1 || ((b & 1) && has_zero_byte(tree[node_of_rank(b >> 1, g.d)]));
        cur[b] = (st + rows[static_cast<uint64_t>(c) * g.k + b]) | (fin ? 0x80000000u : 0u);
    }
    __syncthreads();
    if (threadIdx.x == 0)
        for (uint32_t q = 0; q < NS; ++q)
            if (lo + q * kTmaTile < hi) issue(lo + q * kTmaTile, q);
    constexpr uint32_t IT = kTmaTile / kTmaThreads;
    unsigned long long fetches = 0;
    const uint32_t k2m = k2_kind(A, s);
    uint32_t t = 0, buf = 0, phase = 0;
#pragma unroll 1
    for (uint32_t base = lo; base < hi; base += kTmaTile, ++t) {
        const uint32_t m = min(kTmaTile, hi - base);
        const uint32_t shk = elem_shift(key + base, 8), sho = elem_shift(off + base, 4),
                       shb = elem_shift(bkt + base, 2);
        for (uint32_t b = threadIdx.x; b <= g.k; b += kTmaThreads) cnt[b] = 0;
        // wait for the tile's bytes
        asm volatile(
            "{\n .reg .pred p;\n W%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
            " @!p bra W%=;\n}\n" :: "r"(smem_u32(&bar[buf])), "r"(phase) : "memory");
        __syncthreads();
        const TmaStage& S = stage[buf];
        uint32_t br[IT];  // bucket | rank-in-tile << 16
#pragma unroll
        for (uint32_t j = 0; j < IT; ++j) {
            const uint32_t e = threadIdx.x + j * kTmaThreads;
            if (e < m) {
                const uint32_t b = S.bkt[e + shb];
                br[j] = b | (atomicAdd(&cnt[b], 1u) << 16);
            }
        }
        __syncthreads();
        tile_scan<kTmaThreads>(cnt, g.k, cur, gb, warp_sums);
#pragma unroll
        for (uint32_t j = 0; j < IT; ++j) {
            const uint32_t e = threadIdx.x + j * kTmaThreads;
            if (e < m) perm[cnt[br[j] & 0xFFFFu] + (br[j] >> 16)] = static_cast<uint16_t>(e);
        }
        __syncthreads();
        for (uint32_t q = threadIdx.x; q < m; q += kTmaThreads) {
            const uint32_t e = perm[q];
            const uint32_t b = S.bkt[e + shb];
            const uint32_t r = gb[b];
            const bool fin = r >> 31;
            const uint32_t p = (r & 0x7FFFFFFFu) + (q - cnt[b]);
            const uint32_t end = fin && (b & 1) ? starts[b + 1] : 0;
            if (k2m)
                place_k2(A, s, b, fin, p, end, S.off[e + sho], S.key[e + shk], k2m, s.begin + base + e,
                         fetches);
            else
                place(A, s, b, fin, p, end, S.off[e + sho], S.key[e + shk], fetches);
        }
        __syncthreads();  // every read of this stage is done: refill it
        if (threadIdx.x == 0 && base + NS * kTmaTile < hi) {
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            issue(base + NS * kTmaTile, buf);
        }
        if (++buf == NS) {  // stage ring: parity flips each time it wraps
            buf = 0;
            phase ^= 1u;
        }
    }
    for (uint32_t x = 16; x > 0; x >>= 1) fetches += __shfl_xor_sync(0xffffffffu, fetches, x);
    if ((threadIdx.x & 31) == 0 && fetches) atomicAdd(&A.ctl->fetches, fetches);
}

// ---------------------------------------------------------------------------
// LCP at bucket boundaries: the two strings differ within the 8-byte window
// at the recorded depth (they were classified into different buckets).

__global__ void k_lcp_fix(const uint8_t* __restrict__ arena, const int64_t* __restrict__ out,
                          int64_t* __restrict__ lcp, const uint2* __restrict__ hints,
                          uint64_t m) {
    uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < m;
         i += stride) {
        const uint2 h = hints[i];
        uint64_t d = h.y;
        uint64_t a = static_cast<uint64_t>(out[h.x]), b = static_cast<uint64_t>(out[h.x + 1]);
        for (;;) {
            uint64_t ka = load_key(arena, a + d), kb = load_key(arena, b + d);
            if (ka != kb) { lcp[h.x] = static_cast<int64_t>(d + diff_bytes(ka, kb)); break; }
            if (has_zero_byte(ka)) { lcp[h.x] = static_cast<int64_t>(d + zero_index(ka)); break; }
            d += 8;
        }
    }
}

// ---------------------------------------------------------------------------
// standalone operation surfaces (parity tests of the pieces)

__global__ void k_pack_keys(const uint8_t* __restrict__ arena, const int64_t* __restrict__ h,
                            uint64_t n, uint64_t depth, uint64_t* __restrict__ out) {
    uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += stride)
        out[i] = load_key(arena, static_cast<uint64_t>(h[i]) + depth);
}

// lcp of adjacent sorted strings, 8 bytes per step (strings.py:56-61, :99-102)
__global__ void k_adjacent_lcp(const uint8_t* __restrict__ arena, const int64_t* __restrict__ h,
                               uint64_t m, int64_t* __restrict__ out) {
    uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < m;
         i += stride) {
        uint64_t a = static_cast<uint64_t>(h[i]), b = static_cast<uint64_t>(h[i + 1]);
        uint64_t d = 0;
        for (;;) {
            uint64_t ka = load_key(arena, a + d), kb = load_key(arena, b + d);
            if (ka != kb) { out[i] = static_cast<int64_t>(d + diff_bytes(ka, kb)); break; }
            if (has_zero_byte(ka)) { out[i] = static_cast<int64_t>(d + zero_index(ka)); break; }
            d += 8;
        }
    }
}

// _first_unsorted (strings.py:77-82): min i with s[i] > s[i+1]
__global__ void k_first_unsorted(const uint8_t* __restrict__ arena,
                                 const int64_t* __restrict__ h, uint64_t m,
                                 unsigned long long* __restrict__ result) {
    uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < m;
         i += stride) {
        uint64_t a = static_cast<uint64_t>(h[i]), b = static_cast<uint64_t>(h[i + 1]);
        uint64_t d = 0;
        for (;;) {
            uint64_t ka = load_key(arena, a + d), kb = load_key(arena, b + d);
            if (ka != kb) {
                if (ka > kb) atomicMin(result, static_cast<unsigned long long>(i));
                break;
            }
            if (has_zero_byte(ka)) break;
            d += 8;
        }
    }
}

// classify_tree_unrolled / _equal over a key batch: level order built in
// shared memory from the in-order splitters (_fill_level_order).
// MODE 0: branch-free descent, 1: equality descent, 2: table (k_wide_count)
template <int MODE>
__global__ void __launch_bounds__(256) k_classify(const uint64_t* __restrict__ keys, uint64_t n,
                                                  const uint64_t* __restrict__ in_order,
                                                  uint32_t d, uint16_t* __restrict__ out) {
    extern __shared__ __align__(16) uint64_t tree[];
    const uint32_t v = (1u << d) - 1;
    for (uint32_t i = threadIdx.x + 1; i <= v; i += blockDim.x) {
        uint32_t l = 31 - __clz(i);
        tree[i] = in_order[inorder_rank(i, l, d)];
    }
    if (threadIdx.x == 0) tree[0] = 0;
    __syncthreads();
    uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    if (MODE == 2) {
        uint64_t* s = tree + (1u << d);
        uint16_t* lut = reinterpret_cast<uint16_t*>(s + (1u << d));
        const LutTree T = lut_build<256>(tree, d, s, lut);
        for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
             i += stride)
            out[i] = static_cast<uint16_t>(classify_lut(keys[i], T));
        return;
    }
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += stride)
        out[i] = static_cast<uint16_t>(classify<MODE == 1>(keys[i], tree, d));
}

// select_splitters + build_tree from a sorted sample (single CTA).
__global__ void __launch_bounds__(1024) k_build_tree(const uint64_t* __restrict__ sample,
                                                     uint32_t m, uint32_t d,
                                                     uint64_t* __restrict__ level_order,
                                                     uint64_t* __restrict__ in_order) {
    extern __shared__ __align__(16) uint8_t sm[];
    uint64_t* s = reinterpret_cast<uint64_t*>(sm);
    int32_t* na = reinterpret_cast<int32_t*>(sm + static_cast<uint64_t>(m) * 8);
    int32_t* nb = na + (1u << d);
    uint32_t* nf = reinterpret_cast<uint32_t*>(nb + (1u << d));
    for (uint32_t i = threadIdx.x; i < m; i += 1024) s[i] = sample[i];
    __syncthreads();
    build_tree_levels<1024>(s, m, d, level_order, na, nb, nf);
    const uint32_t v = (1u << d) - 1;
    for (uint32_t c = threadIdx.x; c < v; c += 1024) in_order[c] = level_order[node_of_rank(c, d)];
}


// ---------------------------------------------------------------------------
// multi-GPU partition (distributed.py step 3): destination rank
// of every local string = number of the G-1 splitter strings below it in
// (string, handle) order; then a stable-free grouping of the handles by
// destination (contiguous send ranges for the all-to-all).

constexpr uint32_t kPartThreads = 256;
constexpr uint32_t kPartMaxRanks = 1024;

// (string, handle) three-way compare of splitter a with string b whose
// 8-byte keys at depth 0 are equal
__device__ __forceinline__ int part_tail(const uint8_t* __restrict__ arena, int64_t a, int64_t b,
                                         uint64_t key, unsigned long long& fetches) {
    int c = 0;
    if (!has_zero_byte(key))
        c = walk_compare(arena, static_cast<uint64_t>(a), static_cast<uint64_t>(b), 8, nullptr,
                         fetches);
    return c ? c : (a < b ? -1 : (a > b ? 1 : 0));
}

__global__ void __launch_bounds__(kPartThreads) k_part_count(
        const uint8_t* __restrict__ arena, const int64_t* __restrict__ h, uint32_t n,
        const int64_t* __restrict__ spl, uint32_t ns, uint32_t chunk, uint16_t* __restrict__ dest,
        uint32_t* __restrict__ rows) {
    __shared__ uint64_t skey[kPartMaxRanks];
    __shared__ uint32_t hist[kPartMaxRanks];
    const uint32_t G = ns + 1;
    for (uint32_t i = threadIdx.x; i < ns; i += kPartThreads)
        skey[i] = load_key(arena, static_cast<uint64_t>(spl[i]));
    for (uint32_t d = threadIdx.x; d < G; d += kPartThreads) hist[d] = 0;
    __syncthreads();
    const uint32_t lo = blockIdx.x * chunk, hi = min(n, lo + chunk);
    unsigned long long fetches = 0;
    for (uint32_t i = lo + threadIdx.x; i < hi; i += kPartThreads) {
        const int64_t x = h[i];
        const uint64_t k = load_key(arena, static_cast<uint64_t>(x));
        uint32_t a = 0, b = ns;  // first splitter not below the string
#pragma unroll 1
        while (a < b) {
            const uint32_t mid = (a + b) >> 1;
            const uint64_t sk = skey[mid];
            const int c = sk < k ? -1 : (sk > k ? 1 : part_tail(arena, spl[mid], x, k, fetches));
            if (c < 0) a = mid + 1; else b = mid;
        }
        dest[i] = static_cast<uint16_t>(a);
        atomicAdd(&hist[a], 1u);
    }
    __syncthreads();
    for (uint32_t d = threadIdx.x; d < G; d += kPartThreads)
        rows[static_cast<uint64_t>(blockIdx.x) * G + d] = hist[d];
}

// rows[c][d] -> exclusive prefix over c per destination d; starts[d] =
// exclusive prefix of the destination totals, starts[G] = n.  One warp per
// destination, lanes split the rows.
__global__ void __launch_bounds__(1024) k_part_scan(uint32_t* __restrict__ rows, uint32_t C,
                                                    uint32_t G, unsigned long long* __restrict__ tot) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t R = (C + 31) / 32;
    for (uint32_t d = threadIdx.x >> 5; d < G; d += 32) {
        const uint32_t r0 = min(C, lane * R), r1 = min(C, r0 + R);
        uint32_t sum = 0;
        for (uint32_t c = r0; c < r1; ++c) sum += rows[static_cast<uint64_t>(c) * G + d];
        uint32_t incl = sum;
        for (uint32_t o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        uint32_t run = incl - sum;
        for (uint32_t c = r0; c < r1; ++c) {
            const uint64_t at = static_cast<uint64_t>(c) * G + d;
            const uint32_t x = rows[at];
            rows[at] = run;
            run += x;
        }
        if (lane == 31) tot[d] = incl;
    }
}

__global__ void __launch_bounds__(kPartThreads) k_part_scatter(
        const int64_t* __restrict__ h, uint32_t n, uint32_t chunk, uint32_t G,
        const uint16_t* __restrict__ dest, const uint32_t* __restrict__ rows,
        const unsigned long long* __restrict__ tot, int64_t* __restrict__ out) {
    __shared__ uint32_t cur[kPartMaxRanks];
    // destination starts: exclusive prefix of the totals (G is small)
    for (uint32_t d = threadIdx.x; d < G; d += kPartThreads) {
        unsigned long long st = 0;
        for (uint32_t q = 0; q < d; ++q) st += tot[q];
        cur[d] = static_cast<uint32_t>(st) + rows[static_cast<uint64_t>(blockIdx.x) * G + d];
    }
    __syncthreads();
    const uint32_t lo = blockIdx.x * chunk, hi = min(n, lo + chunk);
    for (uint32_t i = lo + threadIdx.x; i < hi; i += kPartThreads) {
        const uint32_t d = dest[i];
        out[atomicAdd(&cur[d], 1u)] = h[i];
    }
}


// ---------------------------------------------------------------------------
// the path's neighbours: line ingest (harness.py:72-95),
// string lengths (strings.py:85-96) and sorted-string materialisation
// (tests/helpers.py:62-68), all built on one ordered compaction of
// terminator positions.

constexpr uint32_t kScanThreads = 256;
constexpr uint32_t kScanChunk = 16384;  // bytes per CTA, 64 per thread

// SWAR masks over the 8 bytes of a little-endian word: bit 7 of byte i set
// iff byte i is 0 (exact: no borrow-induced false positives above a real
// zero matter because every flagged byte is recomputed per byte below)
__device__ __forceinline__ uint64_t zero_bytes(uint64_t w) {
    // exact per-byte zero test: (b | (b + 0x7F)) has bit 7 clear iff b == 0
    const uint64_t low7 = 0x7F7F7F7F7F7F7F7Full;
    return ~(((w & low7) + low7) | w | low7);
}

// ingest: raw bytes -> arena (newline -> 0), terminators counted per CTA,
// first embedded 0 byte recorded; mode 0 = ingest (copy + convert),
// mode 1 = count zeros of an existing arena.  64 bytes per thread, read and
// written as 8-byte words (the chunk bases are 64-byte aligned; the tail of
// the input is handled bytewise).
template <int MODE>
__global__ void __launch_bounds__(kScanThreads) k_term_count(
        const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, uint64_t len,
        uint32_t* __restrict__ counts, unsigned long long* __restrict__ first_nul) {
    constexpr uint32_t B = kScanChunk / kScanThreads;  // 64
    const uint64_t lo = static_cast<uint64_t>(blockIdx.x) * kScanChunk + threadIdx.x * B;
    const uint64_t hi = min(len, lo + B);
    uint32_t c = 0;
    if (hi == lo + B) {
        const uint64_t* s8 = reinterpret_cast<const uint64_t*>(src + lo);
#pragma unroll
        for (uint32_t q = 0; q < B / 8; ++q) {
            uint64_t w = s8[q];
            if (MODE == 0) {
                const uint64_t z = zero_bytes(w);
                if (z) atomicMin(first_nul, static_cast<unsigned long long>(lo + 8 * q + (__ffsll(z) - 1) / 8));
                const uint64_t nl = zero_bytes(w ^ 0x0A0A0A0A0A0A0A0Aull);  // '\n' bytes
                w &= ~((nl >> 7) * 0xFFull);
                reinterpret_cast<uint64_t*>(dst + lo)[q] = w;
            }
            c += __popcll(zero_bytes(w));
        }
    } else {
        for (uint64_t i = lo; i < hi; ++i) {
            uint8_t x = src[i];
            if (MODE == 0) {
                if (x == 0) atomicMin(first_nul, static_cast<unsigned long long>(i));
                if (x == '\n') x = 0;
                dst[i] = x;
            }
            c += x == 0;
        }
    }
    c = __reduce_add_sync(0xffffffffu, c);
    __shared__ uint32_t ws[kScanThreads / 32];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (uint32_t w = 0; w < kScanThreads / 32; ++w) t += ws[w];
        counts[blockIdx.x] = t;
    }
}

// exclusive scan of n values in one CTA (widened to u64); out[n] = total
template <typename T>
__global__ void __launch_bounds__(1024) k_scan_small(const T* __restrict__ in, uint64_t n,
                                                     unsigned long long* __restrict__ out) {
    __shared__ unsigned long long ws[32], carry;
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (uint64_t b = 0; b < n; b += 1024) {
        const uint64_t i = b + threadIdx.x;
        const unsigned long long x = i < n ? static_cast<unsigned long long>(in[i]) : 0;
        unsigned long long v = x;
        for (uint32_t o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += y;
        }
        if (lane == 31) ws[w] = v;
        __syncthreads();
        if (w == 0) {
            unsigned long long y = ws[lane];
            for (uint32_t o = 1; o < 32; o <<= 1) {
                const unsigned long long z = __shfl_up_sync(0xffffffffu, y, o);
                if (lane >= o) y += z;
            }
            ws[lane] = y;
        }
        __syncthreads();
        const unsigned long long excl = carry + v - x + (w ? ws[w - 1] : 0ull);
        if (i < n) out[i] = excl;
        __syncthreads();
        if (threadIdx.x == 1023) carry = excl + x;
        __syncthreads();
    }
    if (threadIdx.x == 0) out[n] = carry;
}

// ordered positions of the zero bytes of a[0, len): pos[k] = (k-th zero) + shift
__global__ void __launch_bounds__(kScanThreads) k_term_write(
        const uint8_t* __restrict__ a, uint64_t len, const unsigned long long* __restrict__ block_base,
        int64_t* __restrict__ pos, int64_t shift) {
    constexpr uint32_t B = kScanChunk / kScanThreads;
    const uint64_t lo = static_cast<uint64_t>(blockIdx.x) * kScanChunk + threadIdx.x * B;
    const uint64_t hi = min(len, lo + B);
    const bool full = hi == lo + B;
    uint64_t zm[B / 8];
    uint32_t c = 0;
#pragma unroll
    for (uint32_t q = 0; q < B / 8; ++q) {
        uint64_t z = 0;
        if (full) {
            z = zero_bytes(reinterpret_cast<const uint64_t*>(a + lo)[q]);
        } else {
            for (uint32_t b = 0; b < 8; ++b) {
                const uint64_t i = lo + 8 * q + b;
                if (i < hi && a[i] == 0) z |= 0x80ull << (8 * b);
            }
        }
        zm[q] = z;
        c += __popcll(z);
    }
    // exclusive prefix of the thread counts in position order
    uint32_t incl = c;
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (uint32_t o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    __shared__ uint32_t ws[kScanThreads / 32];
    if (lane == 31) ws[w] = incl;
    __syncthreads();
    uint32_t before = 0;
    for (uint32_t q = 0; q < w; ++q) before += ws[q];
    unsigned long long k = block_base[blockIdx.x] + before + incl - c;
#pragma unroll
    for (uint32_t q = 0; q < B / 8; ++q) {
        uint64_t z = zm[q];
        while (z) {
            const uint32_t bit = __ffsll(z) - 1;
            pos[k++] = static_cast<int64_t>(lo + 8 * q + bit / 8) + shift;
            z &= z - 1;
        }
    }
}

// length of strings that end within `words` 8-byte words of their start
// (SWAR walk); the others get -1 and are counted in *longer for the search
__global__ void k_lengths_walk(const uint8_t* __restrict__ arena, const int64_t* __restrict__ h,
                               uint64_t n, uint32_t words, int64_t* __restrict__ len,
                               unsigned long long* __restrict__ longer) {
    unsigned long long nl = 0;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t p = static_cast<uint64_t>(h[i]);
        uint64_t a = p & ~7ull;
        uint64_t w = *reinterpret_cast<const uint64_t*>(arena + a);
        w |= (1ull << (8 * (p - a))) - 1;  // bytes before the start are not terminators
        int64_t L = -1;
#pragma unroll 1
        for (uint32_t q = 0; q < words; ++q) {
            const uint64_t z = zero_bytes(w);
            if (z) {
                L = static_cast<int64_t>(a + (__ffsll(z) - 1) / 8 - p);
                break;
            }
            a += 8;
            w = *reinterpret_cast<const uint64_t*>(arena + a);
        }
        len[i] = L;
        nl += L < 0;
    }
    for (uint32_t x = 16; x > 0; x >>= 1) nl += __shfl_xor_sync(0xffffffffu, nl, x);
    if ((threadIdx.x & 31) == 0 && nl) atomicAdd(longer, nl);
}

// length of every string: distance to the first terminator at or after it
__global__ void k_lengths(const int64_t* __restrict__ h, uint64_t n, const int64_t* __restrict__ term,
                          uint64_t nterm, int64_t* __restrict__ len) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        if (len[i] >= 0) continue;  // found by the short walk
        const int64_t x = h[i];
        uint64_t lo = 0, hi = nterm;
        while (lo < hi) {
            const uint64_t mid = (lo + hi) >> 1;
            if (term[mid] < x) lo = mid + 1; else hi = mid;
        }
        len[i] = (lo < nterm ? term[lo] : x) - x;
    }
}

// exclusive scan of (len + 1) over n strings (block-local pass + totals)
__global__ void __launch_bounds__(1024) k_scan_len_block(const int64_t* __restrict__ len, uint64_t n,
                                                         int64_t* __restrict__ out,
                                                         unsigned long long* __restrict__ block_tot) {
    // block totals may exceed 32 bits only for > 4 GiB outputs (rejected on the host)
    __shared__ unsigned long long ws[32];
    const uint64_t i = blockIdx.x * 1024ull + threadIdx.x;
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const unsigned long long x = i < n ? static_cast<unsigned long long>(len[i]) + 1 : 0;
    unsigned long long v = x;
    for (uint32_t o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
    }
    if (lane == 31) ws[w] = v;
    __syncthreads();
    if (w == 0) {
        unsigned long long y = ws[lane];
        for (uint32_t o = 1; o < 32; o <<= 1) {
            const unsigned long long z = __shfl_up_sync(0xffffffffu, y, o);
            if (lane >= o) y += z;
        }
        ws[lane] = y;
    }
    __syncthreads();
    if (i < n) out[i] = static_cast<int64_t>(v - x + (w ? ws[w - 1] : 0ull));
    if (threadIdx.x == 1023) block_tot[blockIdx.x] = ws[31];
}

__global__ void k_scan_len_add(int64_t* __restrict__ out, uint64_t n,
                               const unsigned long long* __restrict__ block_base) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x)
        out[i] += static_cast<int64_t>(block_base[i >> 10]);
}

// one warp per string: its bytes and terminator to the new arena
__global__ void __launch_bounds__(256) k_gather_strings(const uint8_t* __restrict__ arena,
                                                        const int64_t* __restrict__ h,
                                                        const int64_t* __restrict__ len,
                                                        const int64_t* __restrict__ dst, uint64_t n,
                                                        uint8_t* __restrict__ out) {
    const uint32_t lane = threadIdx.x & 31;
    for (uint64_t i = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5; i < n;
         i += (uint64_t(gridDim.x) * blockDim.x) >> 5) {
        const uint64_t a = static_cast<uint64_t>(h[i]), b = static_cast<uint64_t>(dst[i]);
        const uint64_t L = static_cast<uint64_t>(len[i]) + 1;
        for (uint64_t j = lane; j < L; j += 32) out[b + j] = j + 1 < L ? arena[a + j] : 0;
    }
}

}  // namespace s5
