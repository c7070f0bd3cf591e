/*
 * s5.h -- C-ABI of libs5.so, the B200 (sm_100a) super scalar string sample
 * sort (S^5, arXiv 1305.1157).
 *
 * The reference package `strsort` is pure Python + numba and has no FFI; its
 * drop-in boundary is the Python entry-point layer.  Each entry point below
 * replaces one reference routine (cited file:line, paths relative to
 * /root/reference/pkg/src/strsort/) and is bound from Python with ctypes by
 * paper_1305_1157_b200/_lib.py; INTEGRATION.md shows the binding a
 * maintainer would add to the reference package itself.
 *
 * Conventions
 *  - All pointers named d_* are device pointers (caller-owned, e.g. torch
 *    tensors' data_ptr()); h_* are host pointers.
 *  - The arena is the reference's byte arena (strings.py:108-144): strings of
 *    bytes 1..255 closed by a 0; its last byte must be 0.  The device copy
 *    must be 8-byte aligned and followed by at least S5_ARENA_PAD readable
 *    zero bytes (arena_len excludes the padding).
 *  - Handles are int64 offsets of string starts (strings.py:3-7).
 *  - Calls are stream-ordered on `stream` (a cudaStream_t, NULL = legacy
 *    default stream) and return 0 or a negative S5_E* code; s5_last_error()
 *    returns a thread-local message for the last failure.
 *  - Arithmetic is integer only (bytes, u32 offsets, u64 keys, i64 outputs).
 */
#ifndef S5_H_
#define S5_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define S5_ARENA_PAD 128

enum {
    S5_OK = 0,
    S5_E_INVALID = -1,   /* bad argument: unterminated arena, bad v, ... (ValueError) */
    S5_E_CUDA = -2,      /* CUDA runtime error (RuntimeError)                          */
    S5_E_WORKSPACE = -3, /* workspace too small                                        */
    S5_E_RANGE = -4,     /* handle outside the arena / n >= 2^31                        */
    S5_E_INTERNAL = -5,  /* internal capacity exceeded (bug)                           */
    S5_E_NCCL = -6       /* reserved: no entry point of this library calls NCCL         */
};

/* SampleSortConfig (samplesort.py:37-45) plus the GPU tiering knobs.
 * Zero fields take defaults. */
typedef struct {
    uint32_t v;           /* max splitters per step, 2^d-1 (default 8191)       */
    uint32_t alpha;       /* oversampling factor (default 4; the reference's 2)  */
    uint32_t classifier;  /* 0 = "unroll", 1 = "equal" (samplesort.py:43)      */
    uint32_t small_max;   /* segments <= small_max: warp base case (<= 32)      */
    uint32_t narrow_max;  /* segments <= narrow_max: one-CTA S^5 step (<= 2^20; 0: 4096 = off) */
    uint32_t flags;       /* bit0: skip the LCP fix-up (debug); bit1: per-kernel timing;
                           * bit2: no common-prefix skip; bit3: also skip partial prefixes
                           * of >= 4 bytes; bit4: bitonic local sort (power-of-two network);
                           * bit5: bulk-copy (TMA) scatter at every level; bit6: separate
                           * gather pass at level 0; bit7: 2048-tile bulk-copy scatter below
                           * the root; bit8: never carry second key words from the root
                           * to level 1 (otherwise chosen from the root sample); bit9: the
                           * input handles are n u32 offsets packed into the first 4n bytes
                           * of d_handles (the multi-GPU exchange payload); the output is
                           * still n int64 handles in d_handles (n >= 2); bit11: never
                           * use 32-bit sort words in the one-CTA local tiers (otherwise
                           * chosen from the root sample's key entropy); bit13: index
                           * mode -- the u32 offset arrays hold string indices and an
                           * int64 position table (8n more workspace bytes) maps them
                           * to the arena; always on for arenas >= 4 GiB (the
                           * reference's handles are int64 offsets, strings.py:3-7);
                           * bit14: no root prefix skip (otherwise, when the root sample's
                           * keys share 2..7 leading bytes, level 0 classifies the 8 bytes
                           * behind them after checking every string against the prefix) */
    uint64_t seed;        /* sample seed (samplesort.py:45)                     */
    uint32_t local_max;   /* segments <= local_max: one CTA finishes them (<=4096)*/
    uint32_t wide_v;      /* splitters of multi-CTA steps, 2^d-1 <= 1023 (511)  */
    uint32_t wide_target; /* multi-CTA steps aim at children of this size (0: local_max / 8) */
    uint32_t local_target; /* unused since the local tier sorts whole segments (ABI) */
} s5_config;

/* Per-call statistics (Counters, counters.py:8-37; SURVEY 8(d) n_p log). */
#define S5_MAX_LEVELS 128
#define S5_MAX_LAUNCH_RECS 512
typedef struct {
    uint32_t kernel;   /* S5_K_* */
    uint32_t level;
    uint64_t strings;  /* strings the launch processed */
    float ms;          /* device time (CUDA events on the stream) */
    float start_ms;    /* launch start relative to the call's first event */
} s5_launch_rec;
typedef struct {
    uint32_t levels;                     /* level-synchronous passes run          */
    uint32_t pad_;
    uint64_t n_per_pass[S5_MAX_LEVELS];  /* strings moved in pass p (n_p)         */
    uint64_t wide_elems[S5_MAX_LEVELS];  /* of which in multi-CTA S^5 steps       */
    uint64_t narrow_elems[S5_MAX_LEVELS];/* of which in one-CTA S^5 steps         */
    uint64_t small_elems[S5_MAX_LEVELS]; /* of which in warp base-case sorts      */
    uint64_t wide_steps;                 /* S^5 steps over >narrow_max segments   */
    uint64_t narrow_steps;               /* one-CTA S^5 steps                     */
    uint64_t small_segments;             /* base-case segments                    */
    uint64_t key_fetches;                /* arena key gathers (fetches counter)   */
    uint64_t boundary_lcps;              /* LCPs finished by the boundary kernel  */
    uint64_t launches;                   /* kernels launched by the call          */
    float ms_total;                      /* device time of the call (CUDA events) */
    float pad2_;
    /* cfg->flags bit1: per-kernel device time (CUDA events around every
     * launch, same stream), indexed by S5_K_* */
    float kern_ms[16];
    uint32_t kern_launches[16];
    uint64_t local_elems[S5_MAX_LEVELS]; /* of which in one-CTA S^5 + base case    */
    uint64_t local_steps;                /* one-CTA S^5 + base-case segments      */
    uint64_t kern_strings[16];           /* strings processed per kernel (S5_K_*)  */
    uint32_t n_launch_recs;              /* flags bit1: per-launch records        */
    uint32_t pad3_;
    float host_h2d_ms, host_sort_ms, host_d2h_ms, pad4_;  /* s5_sort_host phases (wall) */
    s5_launch_rec launch_recs[S5_MAX_LAUNCH_RECS];
    uint64_t host_h2d_bytes, host_d2h_bytes;  /* s5_sort_host: bytes over PCIe       */
} s5_stats;

enum {
    S5_K_GATHER = 0, S5_K_WIDE_PLAN, S5_K_WIDE_TREE, S5_K_WIDE_COUNT, S5_K_WIDE_COLSCAN,
    S5_K_WIDE_BSCAN, S5_K_WIDE_SCATTER, S5_K_NARROW, S5_K_SMALL, S5_K_LCP_FIX, S5_K_INIT,
    S5_K_LOCAL, S5_K_LOCAL_S, S5_K_LOCAL_M, S5_K_LOCAL_XS, S5_K_LOCAL_W, S5_K_COUNT
};

/* Bytes of device workspace s5_sort needs for n strings. */
uint64_t s5_workspace_bytes(uint64_t n, uint64_t arena_len, const s5_config *cfg);

/* parallel_sample_sort (samplesort.py:437-444) / sample_sort (:241-267):
 * permutes d_handles[0..n) in place into sorted order and, if d_lcp is not
 * NULL, writes the LCP array d_lcp[0..n-1) exactly as _adjacent_lcps
 * (strings.py:99-102) defines it.  `depth` is the common prefix every
 * string is known to share (sample_sort's depth argument). */
int s5_sort(const uint8_t *d_arena, uint64_t arena_len, int64_t *d_handles, uint64_t n,
            uint64_t depth, int64_t *d_lcp, const s5_config *cfg, void *d_workspace,
            uint64_t workspace_bytes, void *stream, s5_stats *stats);

/* Debug variant honouring the reference's audit hook (samplesort.py:235-236,
 * :431-432): after every level, fn receives the child segments the level
 * emitted ({begin, size, depth, side}) and host copies of both ping-pong
 * offset arrays; segment i's strings are side_k[begin .. begin+size) with
 * k = side, all sharing `depth` leading bytes (Eq. (1)). Slow: copies 8n bytes
 * per level. */
typedef struct { uint32_t begin, size, depth, side; } s5_segment;
typedef void (*s5_audit_fn)(void *user, uint32_t level, const s5_segment *segs, uint64_t nsegs,
                            const uint32_t *side0, const uint32_t *side1, uint64_t n);
int s5_sort_audit(const uint8_t *d_arena, uint64_t arena_len, int64_t *d_handles, uint64_t n,
                  uint64_t depth, int64_t *d_lcp, const s5_config *cfg, void *d_workspace,
                  uint64_t workspace_bytes, void *stream, s5_stats *stats, s5_audit_fn fn,
                  void *user);

/* Same with host buffers: uploads handles, sorts, downloads handles + LCP
 * through two pinned staging chunks (host memcpy overlapped with the DMA).
 * The arena must already be on the device (d_arena). Allocates its own
 * device buffers (cached between calls); serialised by an internal lock. */
int s5_sort_host(const uint8_t *d_arena, uint64_t arena_len, int64_t *h_handles, uint64_t n,
                 uint64_t depth, int64_t *h_lcp, const s5_config *cfg, void *stream,
                 s5_stats *stats);

/* pack_keys (strings.py:176-182) / _pack_keys (:50-53). */
int s5_pack_keys(const uint8_t *d_arena, uint64_t arena_len, const int64_t *d_handles,
                 uint64_t n, uint64_t depth, uint64_t *d_keys, void *stream);

/* _adjacent_lcps (strings.py:99-102): d_lcp[i] = lcp(s[i], s[i+1]). */
int s5_adjacent_lcp(const uint8_t *d_arena, uint64_t arena_len, const int64_t *d_sorted,
                    uint64_t n, int64_t *d_lcp, void *stream);

/* _first_unsorted (strings.py:77-82) on the device: writes the first i with
 * s[i] > s[i+1] (or -1) to *d_result. */
int s5_first_unsorted(const uint8_t *d_arena, uint64_t arena_len, const int64_t *d_handles,
                      uint64_t n, int64_t *d_result, void *stream);

/* The host-buffer staging of s5_sort_host on its own (the multi-GPU path's
 * shards): int64 handles in host memory -> d_handles (crossing PCIe as u32,
 * range-checked against arena_len); and d_handles[n] (+ d_lcp[n_lcp]) ->
 * host int64 arrays (u32 handles, LCPs in the narrowest width that holds
 * their maximum).  h_lcp may be null. */
int s5_upload_handles(const int64_t *h_handles, uint64_t n, uint64_t arena_len, int64_t *d_handles,
                      void *stream);
int s5_download(const int64_t *d_handles, uint64_t n, const int64_t *d_lcp, uint64_t n_lcp,
                int64_t *h_handles, int64_t *h_lcp, void *stream);

/* Multi-GPU partition step (the reference's only parallel
 * split is the pS^5 worker split, samplesort.py:369-434): the destination
 * rank of each of n local strings is the number of the nsplit splitter
 * strings below it in (string, handle) order; d_out receives the handles
 * grouped by destination (order inside a group unspecified) and
 * h_counts[nsplit+1] the group sizes (host memory).  nsplit < 1024. */
int s5_partition(const uint8_t *d_arena, uint64_t arena_len, const int64_t *d_handles,
                 uint64_t n, const int64_t *d_splitters, uint32_t nsplit, int64_t *d_out,
                 uint64_t *h_counts, void *stream);

/* parallel_sample_sort(arena, handles, workers) with workers = GPUs of this
 * process (samplesort.py:437-444; the p-way split of the fully parallel
 * step, :369-434).  Shard g (shard_n[g]
 * int64 handles on devices[g], left untouched) and a replica of the padded
 * arena d_arenas[g] live on devices[g]; a device may be listed more than
 * once; n_gpus <= 64.  The library draws max(64 * n_gpus, 2048) samples per shard, sorts them on
 * devices[0], picks n_gpus - 1 splitter strings in (string, handle) order,
 * groups every shard by destination (s5_partition), moves group (g -> d)
 * into d_out_handles[d] with peer copies (u32 offsets for arenas below
 * 4 GiB) and sorts slice d in place there (s5_sort).  On return slice d
 * holds out_counts[d] sorted handles and the slices in device-list order are
 * the global order; d_out_lcp (NULL, or one buffer per slice) receives slice
 * d's out_counts[d] - 1 LCPs followed by the LCP to the first string of the
 * next non-empty slice, so the concatenation is _adjacent_lcps of the whole
 * output (strings.py:99-102).  out_capacity[d] = elements d_out_handles[d]
 * (and d_out_lcp[d]) can hold -- the sum of shard_n always suffices;
 * S5_E_WORKSPACE when a slice outgrows it.  Exchange by cudaMemcpyPeer over
 * NVLink instead of the NCCL communicators the survey's sketch names (one
 * process owns every device, so no communicator is needed).  Blocking;
 * uses the devices' default streams; one call at a time per process.
 * stats: the largest slice's sort statistics, launches and key_fetches
 * summed over the slices, ms_total = host wall time of the call. */
int s5_sort_multi(int n_gpus, const int *devices, const uint8_t *const *d_arenas,
                  uint64_t arena_len, int64_t *const *d_handle_shards, const uint64_t *shard_n,
                  int64_t *const *d_out_handles, int64_t *const *d_out_lcp,
                  const uint64_t *out_capacity, uint64_t *out_counts, const s5_config *cfg,
                  s5_stats *stats);

/* load_lines (harness.py:72-95) on the device: d_raw[len] (one string per
 * line) -> d_arena (newlines become terminators; a terminator is appended
 * when the last line has none; capacity len + 1 + S5_ARENA_PAD, pad zeroed by
 * the caller) and d_handles (string starts, capacity len + 2).  Results in
 * host memory: *h_n strings, *h_arena_len bytes.  An input byte 0 is the
 * reference's EmbeddedNul (harness.py:36-39, :75-79): S5_E_INVALID with its
 * offset in *h_nul_offset. */
int s5_ingest_lines(const uint8_t *d_raw, uint64_t len, uint8_t *d_arena, int64_t *d_handles,
                    uint64_t *h_n, uint64_t *h_arena_len, int64_t *h_nul_offset, void *stream);

/* _string_lengths (strings.py:85-96): distance from each handle to the next
 * terminator (ordered compaction of the arena's terminators + binary search). */
int s5_string_lengths(const uint8_t *d_arena, uint64_t arena_len, const int64_t *d_handles,
                      uint64_t n, int64_t *d_len, void *stream);

/* Sorted-string materialisation (tests/helpers.py:62-68 strings_of; SURVEY
 * 8(f) #4): the strings of d_sorted gathered in order into d_out (each with
 * its terminator), their new handles in d_out_handles[n].  *h_out_len gets
 * the bytes needed; S5_E_WORKSPACE if they exceed out_cap (call with
 * out_cap = 0 to size the buffer). */
int s5_materialize(const uint8_t *d_arena, uint64_t arena_len, const int64_t *d_sorted, uint64_t n,
                   uint8_t *d_out, uint64_t out_cap, int64_t *d_out_handles, uint64_t *h_out_len,
                   void *stream);

/* classify_tree_unrolled / classify_tree_equal (classifier.py:259-278):
 * buckets of n keys against v = 2^d-1 sorted splitters (in-order).
 * classifier: 0 branch-free descent, 1 equality descent, 2 12-bit table + binary
 * search (the multi-CTA count kernel's classifier); identical buckets. */
int s5_classify(const uint64_t *d_keys, uint64_t n, const uint64_t *d_in_order, uint32_t v,
                uint32_t classifier, uint16_t *d_buckets, void *stream);

/* select_splitters + build_tree (classifier.py:85-176) on the device, the
 * path the sort uses: from a sorted sample of m keys, v splitters in level
 * order (d_level_order[v+1], slot 0 unused) and in order (d_in_order[v]). */
int s5_build_tree(const uint64_t *d_sorted_sample, uint32_t m, uint32_t v,
                  uint64_t *d_level_order, uint64_t *d_in_order, void *stream);

/* Host helper for the config-5 generator: order-2 Markov text over sigma
 * symbols from cumulative rows cdf[sigma][sigma][sigma] and uniforms u[n]
 * (SURVEY 8(d) recipe 5). */
int s5_host_markov_text(const double *cdf, const double *u, uint64_t n, uint32_t sigma,
                        uint8_t *out);

/* Host helper for the config-3 generator: dst[dst_start[i] + j] =
 * blob[src_start[i] + j] for j < lengths[i], i < m (host worker threads). */
int s5_host_copy_pieces(uint8_t *dst, const int64_t *dst_start, const int64_t *src_start,
                        const int64_t *lengths, const uint8_t *blob, uint64_t m);

/* Frees the library's cached device buffers, pinned staging and side
 * streams on every device (no call may be in flight); they are re-created
 * on demand. */
int s5_release_caches(void);

const char *s5_last_error(void);
int s5_version(void);

#ifdef __cplusplus
}
#endif
#endif /* S5_H_ */
