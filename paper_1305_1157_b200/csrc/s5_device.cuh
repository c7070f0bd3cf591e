// s5_device.cuh -- device helpers shared by the S^5 kernels (sm_100a).
//
// Keys follow the reference's packing (strings.py:36-47, D1/D2 of SPEC.md):
// 8 bytes MSB-first, every byte after the first terminator forced to 0, so
// unsigned integer order equals lexicographic order of the 8-byte windows.
#pragma once

#include <cstdint>

namespace s5 {

constexpr uint64_t kOnes = 0x0101010101010101ull;
constexpr uint64_t kHighs = 0x8080808080808080ull;

__device__ __forceinline__ uint64_t bswap64(uint64_t w) {
    uint32_t lo = static_cast<uint32_t>(w), hi = static_cast<uint32_t>(w >> 32);
    return (static_cast<uint64_t>(__byte_perm(lo, 0, 0x0123)) << 32) |
           __byte_perm(hi, 0, 0x0123);
}

// Key of the string window starting at arena[pos]: two aligned 8-byte loads
// and a funnel shift give the bytes in string order (first byte in the least
// significant position); the exact first zero byte is the lowest flagged
// byte of the SWAR zero test (borrows only propagate upward), bytes from it
// on are cleared, and a byte swap yields the MSB-first key.
// Needs arena 8-byte aligned with >= 16 readable bytes past pos.
__device__ __forceinline__ uint64_t load_key(const uint8_t* __restrict__ arena, uint64_t pos) {
    const uint64_t* p = reinterpret_cast<const uint64_t*>(arena + (pos & ~7ull));
    uint64_t lo = __ldg(p);
    uint64_t hi = __ldg(p + 1);
    uint32_t sh = static_cast<uint32_t>(pos & 7) * 8;
    uint64_t w = sh ? (lo >> sh) | (hi << (64 - sh)) : lo;
    uint64_t t = (w - kOnes) & ~w & kHighs;
    if (t) {
        uint32_t j = (__ffsll(static_cast<long long>(t)) - 1) >> 3;  // first zero byte
        w &= (1ull << (8 * j)) - 1;                                    // j == 0 -> 0
    }
    return bswap64(w);
}

// Keys at pos and pos+8 from three aligned loads (16 string bytes per call);
// a terminator in the first window zeroes the second.  Needs >= 24 readable
// bytes past pos (the arena carries a 64-byte zero pad).
__device__ __forceinline__ void load_key2(const uint8_t* __restrict__ arena, uint64_t pos,
                                          uint64_t& k0, uint64_t& k1) {
    const uint64_t* p = reinterpret_cast<const uint64_t*>(arena + (pos & ~7ull));
    uint64_t w0 = __ldg(p), w1 = __ldg(p + 1), w2 = __ldg(p + 2);
    uint32_t sh = static_cast<uint32_t>(pos & 7) * 8;
    uint64_t x0 = sh ? (w0 >> sh) | (w1 << (64 - sh)) : w0;
    uint64_t x1 = sh ? (w1 >> sh) | (w2 << (64 - sh)) : w1;
    uint64_t t0 = (x0 - kOnes) & ~x0 & kHighs;
    if (t0) {
        uint32_t j = (__ffsll(static_cast<long long>(t0)) - 1) >> 3;
        x0 &= (1ull << (8 * j)) - 1;
        x1 = 0;
    } else {
        uint64_t t1 = (x1 - kOnes) & ~x1 & kHighs;
        if (t1) {
            uint32_t j = (__ffsll(static_cast<long long>(t1)) - 1) >> 3;
            x1 &= (1ull << (8 * j)) - 1;
        }
    }
    k0 = bswap64(x0);
    k1 = bswap64(x1);
}

// Index (0..8) of the first zero byte of an MSB-first key; 8 if none.
__device__ __forceinline__ uint32_t zero_index(uint64_t key) {
    uint64_t w = bswap64(key);
    uint64_t t = (w - kOnes) & ~w & kHighs;
    return t ? static_cast<uint32_t>((__ffsll(static_cast<long long>(t)) - 1) >> 3) : 8u;
}

// classifier.py:145-150 (_has_zero_byte)
__device__ __forceinline__ bool has_zero_byte(uint64_t key) { return zero_index(key) < 8; }

// Leading equal bytes of two keys that differ (strings.py:56-61 semantics:
// a shared terminator cannot precede the first difference).
__device__ __forceinline__ uint32_t diff_bytes(uint64_t a, uint64_t b) {
    return static_cast<uint32_t>(__clzll(static_cast<long long>(a ^ b))) >> 3;
}

// Level-order node holding in-order rank c of a perfect tree of depth d
// (inverse of inorder_rank, classifier.py:179-181).
__device__ __forceinline__ uint32_t node_of_rank(uint32_t c, uint32_t d) {
    uint32_t r = c + 1;
    uint32_t tz = __ffs(r) - 1;
    uint32_t l = d - 1 - tz;
    return (1u << l) + (r >> (tz + 1));
}

// In-order rank of level-order node i at level l (classifier.py:179-181).
__device__ __forceinline__ uint32_t inorder_rank(uint32_t i, uint32_t l, uint32_t d) {
    return (2u * (i - (1u << l)) + 1u) * (1u << (d - 1 - l)) - 1u;
}

// Bucket of key k in the tree t[1..v] (level order, v = 2^d - 1):
//   c = #splitters < k; bucket = 2c+1 if splitter c == k else 2c
// (classify_oracle, classifier.py:187-200).
// UNROLL: full branch-free descent + one leaf equality test
//   (_classify_strings_unrolled, samplesort.py:51-83).
// EQUAL: equality test per node with early exit and the duplicate-splitter
//   walk to the first equal slot (_classify_strings_equal, samplesort.py:86-105).
template <bool EQUAL>
__device__ __forceinline__ uint32_t classify(uint64_t k, const uint64_t* t, uint32_t d) {
    if (!EQUAL) {
        uint32_t i = 1;
#pragma unroll 1
        for (uint32_t l = 0; l < d; ++l) i = 2 * i + (k > t[i] ? 1u : 0u);
        uint32_t c = i - (1u << d);
        uint32_t b = 2 * c;
        if (c < (1u << d) - 1 && t[node_of_rank(c, d)] == k) b += 1;
        return b;
    } else {
        uint32_t i = 1;
        for (uint32_t l = 0; l < d; ++l) {
            uint64_t node = t[i];
            if (k == node) {
                uint32_t j = inorder_rank(i, l, d);
                while (j > 0 && t[node_of_rank(j - 1, d)] == k) --j;
                return 2 * j + 1;
            }
            i = 2 * i + (k > node ? 1u : 0u);
        }
        return 2 * (i - (1u << d));
    }
}

// IW interleaved descents (pS^5-Unroll interleaves three, samplesort.py:44,
// :59-73): independent dependency chains keep the shared-memory pipe busy.
template <bool EQUAL, int IW>
__device__ __forceinline__ void classify_iw(const uint64_t (&k)[IW], const uint64_t* t,
                                            uint32_t d, uint32_t (&b)[IW]) {
    if (!EQUAL) {
        uint32_t i[IW];
#pragma unroll
        for (int j = 0; j < IW; ++j) i[j] = 1;
#pragma unroll 1
        for (uint32_t l = 0; l < d; ++l) {
#pragma unroll
            for (int j = 0; j < IW; ++j) i[j] = 2 * i[j] + (k[j] > t[i[j]] ? 1u : 0u);
        }
        const uint32_t v = (1u << d) - 1;
#pragma unroll
        for (int j = 0; j < IW; ++j) {
            uint32_t c = i[j] - (1u << d);
            b[j] = 2 * c + ((c < v && t[node_of_rank(c, d)] == k[j]) ? 1u : 0u);
        }
    } else {
#pragma unroll
        for (int j = 0; j < IW; ++j) b[j] = classify<true>(k[j], t, d);
    }
}

// Table classification: the same bucket as classify_oracle
// (classifier.py:187-200) in ~3 shared loads instead of d dependent ones.
// The in-order splitters s[0..v) share their first `lb` bits (value `pf`);
// the next kLutBits bits of a key index lut, lut[x] = first splitter whose
// bits there are >= x, so the key's splitter count lies in [lut[x],
// lut[x+1]), finished by a (usually empty) binary search.
constexpr uint32_t kLutBits = 12;
constexpr uint32_t kLutCells = 1u << kLutBits;  // lut has kLutCells + 1 entries

struct LutTree {
    const uint64_t* s;
    const uint16_t* lut;
    uint32_t v, lb;
    uint64_t pf;
};

__device__ __forceinline__ uint32_t lut_cell(uint64_t k, uint32_t lb) {
    return static_cast<uint32_t>((k << lb) >> (64 - kLutBits));
}

__device__ __forceinline__ uint32_t classify_lut(uint64_t k, const LutTree& T) {
    if (T.lb == 64) return k < T.pf ? 0u : (k > T.pf ? 2 * T.v : 1u);
    if (T.lb) {
        uint64_t kp = k >> (64 - T.lb);
        if (kp != T.pf) return kp < T.pf ? 0u : 2 * T.v;
    }
    const uint32_t x = lut_cell(k, T.lb);
    uint32_t lo = T.lut[x], hi = T.lut[x + 1];
#pragma unroll 1
    while (lo < hi) {
        uint32_t mid = (lo + hi) >> 1;
        if (T.s[mid] < k) lo = mid + 1; else hi = mid;
    }
    return 2 * lo + ((lo < T.v && T.s[lo] == k) ? 1u : 0u);
}

// Builds s (in order, from the level-order tree t[1..v]) and lut[0..kLutCells];
// all threads call; ends with a barrier.  Returns the table descriptor.
template <uint32_t THREADS>
__device__ __forceinline__ LutTree lut_build(const uint64_t* t, uint32_t d, uint64_t* s,
                                             uint16_t* lut) {
    const uint32_t v = (1u << d) - 1;
    for (uint32_t c = threadIdx.x; c < v; c += THREADS) s[c] = t[node_of_rank(c, d)];
    __syncthreads();
    const uint64_t a = s[0], b = s[v - 1];
    const uint32_t lb = a == b ? 64u : static_cast<uint32_t>(__clzll(static_cast<long long>(a ^ b)));
    if (lb < 64) {
        for (uint32_t x = threadIdx.x; x <= kLutCells; x += THREADS) {
            uint32_t lo = 0, hi = v;
            while (lo < hi) {
                uint32_t mid = (lo + hi) >> 1;
                if (lut_cell(s[mid], lb) < x) lo = mid + 1; else hi = mid;
            }
            lut[x] = static_cast<uint16_t>(lo);
        }
    }
    __syncthreads();
    LutTree T;
    T.s = s;
    T.lut = lut;
    T.v = v;
    T.lb = lb;
    T.pf = lb == 64 ? a : (lb ? a >> (64 - lb) : 0);
    return T;
}

// Stateless sample RNG: splitmix64 finaliser over (seed, segment, index).
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__host__ __device__ __forceinline__ uint64_t segment_seed(uint64_t seed, uint64_t begin,
                                                          uint64_t size, uint64_t depth) {
    return seed * 0x9E3779B97F4A7C15ull ^ begin * 0xD1B54A32D192ED03ull ^
           size * 0x8CB92BA72F3D8DD7ull ^ depth * 0xABC98388FB8FAC03ull;
}

__device__ __forceinline__ uint32_t sample_index(uint64_t sseed, uint32_t t, uint32_t size) {
    uint64_t r = mix64(sseed + (static_cast<uint64_t>(t) + 1) * 0x9E3779B97F4A7C15ull);
    return static_cast<uint32_t>(__umul64hi(r, size));
}

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// ---------------------------------------------------------------------------
// bulk-copy engine (cp.async.bulk global -> shared, completion on an mbarrier)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 16-byte aligned superset of [src, src + bytes) into dst; returns the
// element shift of src inside the copy
template <typename T>
__device__ __forceinline__ uint32_t bulk_in(T* dst, const T* src, uint32_t count, uint64_t* bar,
                                            uint32_t& tx) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(src);
    const uintptr_t a16 = a & ~static_cast<uintptr_t>(15);
    const uint32_t bytes = static_cast<uint32_t>(((a + count * sizeof(T) + 15) & ~static_cast<uintptr_t>(15)) - a16);
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
        :: "r"(smem_u32(dst)), "l"(a16), "r"(bytes), "r"(smem_u32(bar)) : "memory");
    tx += bytes;
    return static_cast<uint32_t>((a - a16) / sizeof(T));
}

__device__ __forceinline__ uint32_t elem_shift(const void* src, uint32_t size) {
    return static_cast<uint32_t>((reinterpret_cast<uintptr_t>(src) & 15) / size);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" :: "r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t tx) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n"
                 :: "r"(smem_u32(bar)), "r"(tx) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n .reg .pred p;\n W%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra W%=;\n}\n" :: "r"(smem_u32(bar)), "r"(phase) : "memory");
}

}  // namespace s5
