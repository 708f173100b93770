/*
 * s5g.h -- C ABI of the B200-native S^5 string sorter (libs5gpu.so).
 *
 * Drop-in boundary for the reference's sort entry points
 *   strsort.ssss.s5_sort        /root/reference/pkg/src/strsort/ssss.py:361-387
 *   strsort.parallel.parallel_s5 /root/reference/pkg/src/strsort/parallel.py:468-492
 * and the return convention SortedWithLcp (basecase.py:21-33): the stable
 * content order of the input handles plus an int64 LCP array with
 * lcps[0] = LCP_UNDEF = -1 (strset.py:31).
 *
 * Conventions
 *  - Plain pointers and sizes only.  "device" pointers are CUDA device
 *    memory of the current device; "host" pointers are host memory.
 *  - Return 0 on success, a negative S5G_E* code on failure; the message is
 *    in s5g_last_error() (thread-local).
 *  - Calls are synchronous: all work is complete when they return.
 *  - Threading: any host thread may call any entry point.  Sorts on the
 *    same device are serialised inside the library (they share the
 *    device's side streams, events and staging buffers); sorts on different
 *    devices run concurrently.  Errors are reported per thread.
 *  - Arena: 0-terminated strings back to back; every handle h satisfies
 *    0 <= h < arena_len and the string at h ends at a 0 byte.  The arena
 *    pointer must be 8-byte aligned and readable for S5G_ARENA_PAD bytes
 *    past arena_len (bytes there are never interpreted as characters).
 */
#ifndef S5G_H
#define S5G_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define S5G_VERSION 1
#define S5G_ARENA_PAD 16

#define S5G_OK 0
#define S5G_E_INVALID (-1)      /* bad argument (ValueError) */
#define S5G_E_VARIANT (-2)      /* unknown classify variant (ValueError) */
#define S5G_E_CUDA (-3)         /* CUDA runtime error */
#define S5G_E_WORKSPACE (-4)    /* workspace too small */
#define S5G_E_NCCL (-5)         /* not returned by this version (see s5g_sort_multi) */

#define S5G_VARIANT_UNROLL 0    /* ssss.py:160-169 */
#define S5G_VARIANT_EQUAL 1     /* ssss.py:170-180 */

/* Mirror of strsort.counters.SortStats (counters.py:13-36). */
typedef struct s5g_stats {
    int64_t char_cmps;
    int64_t word_fetches;      /* 8-byte words fetched from the arena (cache fills
                                  of 3 words per string and refill, and the words
                                  of direct comparisons) -- the Theorem-6 counter */
    int64_t merge_buffer_cmps;
    int64_t scratch_words;
    int64_t jobs_enqueued;     /* segments queued (S^5 steps + CTA segments) */
    int64_t jobs_executed;
    int64_t share_events;
} s5g_stats;

/* Step hook, the analogue of step_hook(StepRecord) (ssss.py:215-224,
 * 340-341): called on the host after every device-wide S^5 step with the
 * bucket bounds (2v+2 entries, relative to lo) and the v in-order splitters. */
typedef void (*s5g_step_cb)(void *ctx, int64_t lo, int64_t hi, int64_t depth, int64_t v,
                            const int64_t *bounds, const uint64_t *inorder);

typedef struct s5g_sort_args {
    const uint8_t *arena;      /* device */
    int64_t arena_len;
    const int64_t *handles;    /* device, n; never modified */
    int64_t n;
    int64_t depth;             /* common prefix length of all strings */
    int64_t *out_handles;      /* device, n */
    int64_t *out_lcps;         /* device, n, or NULL */
    uint8_t *out_dchar;        /* device, n, or NULL (needs out_lcps) */
    void *workspace;           /* device, s5g_workspace_bytes() bytes */
    size_t workspace_bytes;
    void *stream;              /* cudaStream_t (NULL = default stream) */
    int32_t variant;           /* S5G_VARIANT_* */
    int32_t v;                 /* splitter cap (tuning only; clamped to 8191) */
    uint64_t seed;             /* sampling seed (tuning only) */
    int64_t t_medium;          /* segments below this may finish in one CTA */
    s5g_stats *stats;          /* host, accumulated into; may be NULL */
    s5g_step_cb step_cb;       /* may be NULL */
    void *step_ctx;
} s5g_sort_args;

/* Sort on device buffers.  Replaces s5_sort (ssss.py:361). */
int s5g_sort(const s5g_sort_args *args);

/* Device workspace needed by s5g_sort for n strings and this t_medium. */
size_t s5g_workspace_bytes(int64_t n, int64_t t_medium);

/* Sort on HOST buffers (copies in, sorts, copies out; device memory is
 * managed internally).  This is the reference-facing end-to-end call:
 * s5_sort(sset, want_lcps=...) with sset.buffer/handles in host memory.
 * out_lcps / out_dchar may be NULL.  Page-locked buffers are copied by DMA
 * directly; pageable ones through a pinned staging ring filled by all host
 * threads.  Device memory comes from a library-owned pool (the device's
 * default pool is left alone) that keeps it between calls. */
int s5g_sort_host(const uint8_t *arena, int64_t arena_len, const int64_t *handles, int64_t n,
                  int64_t depth, int64_t *out_handles, int64_t *out_lcps, uint8_t *out_dchar,
                  int32_t variant, int32_t v, uint64_t seed, int64_t t_medium,
                  s5g_stats *stats);

/* One host process driving several devices: parallel_s5(sset, p)
 * (parallel.py:468-492) with p = num_devices.  A sample-sort partition with
 * G-1 string splitters (sampled prefixes, ties by input position) cuts the
 * output order into G ranges; device k receives the arena, classifies all
 * strings against the splitters, keeps its range (in input order) and sorts
 * it; the host fixes the LCP at each part boundary (_boundary_lcps,
 * parallel.py:447-455).  Buffers are HOST memory as in s5g_sort_host; the
 * output is identical to a one-device sort.  Device ids must name visible
 * devices (S5G_E_INVALID otherwise); a device may appear more than once.
 * The multi-PROCESS form (one process per GPU, NCCL all-to-all over
 * NVLink) is paper_1403_2056_b200.dist; its collectives run in
 * torch.distributed, so their errors surface there, not as S5G_E_NCCL. */
typedef struct s5g_multi_args {
    const uint8_t *arena;      /* host */
    int64_t arena_len;
    const int64_t *handles;    /* host, n */
    int64_t n;
    int64_t depth;
    int64_t *out_handles;      /* host, n */
    int64_t *out_lcps;         /* host, n, or NULL */
    uint8_t *out_dchar;        /* host, n, or NULL (needs out_lcps) */
    int32_t num_devices;       /* p >= 1 */
    const int32_t *device_ids; /* host, num_devices CUDA device ordinals */
    int32_t variant;
    int32_t v;
    uint64_t seed;
    int64_t t_medium;
    s5g_stats *stats;          /* host, accumulated into; may be NULL */
} s5g_multi_args;
int s5g_sort_multi(const s5g_multi_args *args);

/* Return the device memory s5g_sort_host keeps cached between calls. */
void s5g_release_cached_memory(void);

/* --- kernel-level entry points (parity tests of single rows of the path) --- */

/* extract_keys (strset.py:152-170), exact semantics for any depth. */
int s5g_extract_keys(const uint8_t *arena, int64_t arena_len, const int64_t *handles, int64_t n,
                     int64_t depth, uint64_t *out_keys, void *stream);

/* select_splitters (ssss.py:85-146) on a sorted device sample of `count`
 * keys: level-order tree[v+1], inorder[v], term_pos[v] (uint8),
 * eq_bucket[v+1] (uint16, 2*eq_leftmost[node_to_inorder[node]]+1). */
int s5g_select_splitters(const uint64_t *sample, int64_t count, int64_t v, uint64_t *tree,
                         uint64_t *inorder, uint8_t *term_pos, uint16_t *eq_bucket,
                         void *stream);

/* classify_keys (ssss.py:149-181) against a level-order tree (v+1 entries,
 * index 0 unused) and eq_bucket table (v+1, used by the equal variant). */
int s5g_classify(const uint64_t *keys, int64_t n, const uint64_t *tree,
                 const uint16_t *eq_bucket, int64_t v, int32_t variant, uint16_t *out_bucket,
                 void *stream);

/* Multi-GPU partition step (the G-rank form of _phased_step's classify,
 * parallel.py:359-398): out_rank[i] = number of splitters
 * (splitters[splitter_off[j] .. splitter_off[j+1]), splitter_gidx[j]) ordered
 * before (string at handles[i], its global input index) -- full-string
 * comparison, ties broken by global input index, so equal strings keep input
 * order across ranks.  The global index is string_gidx[i], or base_index + i
 * when string_gidx is NULL.  All pointers are device pointers. */
int s5g_partition(const uint8_t *arena, int64_t arena_len, const int64_t *handles, int64_t n,
                  int64_t base_index, const int64_t *string_gidx, const uint8_t *splitters,
                  const int64_t *splitter_off, const int64_t *splitter_gidx, int32_t nsplitters,
                  int32_t *out_rank, void *stream);

/* String lengths (StringSet.ends - handles, strset.py:64-78). */
int s5g_lengths(const uint8_t *arena, int64_t arena_len, const int64_t *handles, int64_t n,
                int64_t *out_len, void *stream);

/* Pack strings with their terminators into dst at dst_off[i] (the send
 * buffer of the multi-GPU exchange).  lengths may be NULL when dst_off has
 * n + 1 entries (sizes = offset differences, as s5g_pack_plan writes). */
int s5g_pack(const uint8_t *arena, int64_t arena_len, const int64_t *handles,
             const int64_t *lengths, const int64_t *dst_off, int64_t n, uint8_t *dst,
             void *stream);

/* load_delimited (strset.py:113-134) on the device: `data` (device, len
 * bytes, writable, readable for S5G_ARENA_PAD bytes past len with the byte at
 * data[len] set to 0 by the caller) becomes the arena in place -- the
 * delimiter is remapped to 0 (error if data holds a 0 byte while delimiter !=
 * 0) -- and out_handles (device, room for len + 1 entries) receives the
 * string starts; *out_n their count.  A trailing terminator is the caller's
 * data[len] = 0 (the reference appends one).  Workspace: 16 + 4*ceil(len /
 * 16384) bytes. */
int s5g_load_delimited(uint8_t *data, int64_t len, int32_t delimiter, int64_t *out_handles,
                       int64_t *out_n, void *workspace, size_t workspace_bytes, void *stream);
/* The same with out_handles sized by the caller: room for `capacity` entries,
 * of which terminators + 1 are written (a receiver that knows that n strings
 * arrived passes n + 1 instead of reserving len + 1 entries);
 * S5G_E_INVALID, with nothing written, if the data holds more. */
int s5g_load_delimited_n(uint8_t *data, int64_t len, int32_t delimiter, int64_t *out_handles,
                         int64_t capacity, int64_t *out_n, void *workspace,
                         size_t workspace_bytes, void *stream);
/* ... and with a rank directory: out_rank64 (device, ceil(len / 64) entries)
 * receives the number of terminators before each 64-byte block of the arena.
 * s5g_rank_positions then maps string starts of this arena (query, device, m
 * entries, each one of out_handles[0 .. n)) to their index in out_handles:
 * out_pos[j] = i with out_handles[i] == query[j] -- one directory entry plus
 * the block's bytes before the handle per query, no search.  The multi-GPU
 * path uses it to carry global indices through the local sort. */
int s5g_load_delimited_rank(uint8_t *data, int64_t len, int32_t delimiter, int64_t *out_handles,
                            int64_t capacity, int64_t *out_n, uint32_t *out_rank64,
                            void *workspace, size_t workspace_bytes, void *stream);
int s5g_rank_positions(const uint8_t *arena, int64_t arena_len, const uint32_t *rank64,
                       const int64_t *query, int64_t m, int64_t *out_pos, void *stream);

/* Stable grouping by destination rank for the all-to-all send buffer
 * (device): out_order[k] = index of the k-th string when strings are ordered
 * by (dest, index); out_counts[g] (device, G entries) = strings for rank g.
 * 1 <= G <= 127.  Workspace: s5g_group_workspace_bytes(n, G). */
size_t s5g_group_workspace_bytes(int64_t n, int32_t G);
int s5g_group_by_dest(const int32_t *dest, int64_t n, int32_t G, int64_t *out_order,
                      int64_t *out_counts, void *workspace, size_t workspace_bytes, void *stream);

/* Positions of sorted handles in their input array, for unique handles below
 * map_len: map (device int32[map_len], scratch) gets map[handles[i]] = i,
 * then out_pos[j] = map[query[j]].  Device pointers. */
int s5g_positions(const int64_t *handles, int64_t n, const int64_t *query, int64_t m,
                  int32_t *map, int64_t map_len, int64_t *out_pos, void *stream);

/* Input position of every sorted handle: out_pos[j] = i with
 * in_handles[i] the string at out_handles[j], for a stable sort's output
 * (equal handles -- the same string -- are matched in input order, so
 * repeated handles are fine).  Two stable radix sorts by handle; O(n), no
 * per-byte map -- or, when in_handles is strictly ascending (the string
 * starts of a received arena; checked on the device), one binary search per
 * string.  max_handle bounds the handles (e.g. arena_len).  Device
 * pointers; workspace: s5g_input_positions_workspace_bytes(n). */
size_t s5g_input_positions_workspace_bytes(int64_t n);
int s5g_input_positions(const int64_t *in_handles, const int64_t *out_handles, int64_t n,
                        int64_t max_handle, int64_t *out_pos, void *workspace,
                        size_t workspace_bytes, void *stream);

/* out[k] = src[idx[k]] (device int64 arrays). */
int s5g_gather_i64(const int64_t *src, const int64_t *idx, int64_t n, int64_t *out, void *stream);

/* Send plan of the multi-GPU exchange: for the strings in send order
 * (handles[order[k]]): out_handles[k], out_off[0..n] (exclusive byte offsets
 * incl. terminators; out_off[n] = total) and out_dest_bytes[g] = bytes for
 * destination g, given counts[g] strings per destination (all device).
 * Workspace: s5g_pack_plan_workspace_bytes(n). */
size_t s5g_pack_plan_workspace_bytes(int64_t n);
int s5g_pack_plan(const uint8_t *arena, int64_t arena_len, const int64_t *handles,
                  const int64_t *order, int64_t n, const int64_t *counts, int32_t G,
                  int64_t *out_handles, int64_t *out_off, int64_t *out_dest_bytes,
                  void *workspace, size_t workspace_bytes, void *stream);

/* dist_stats (strset.py:290-309) of a sorted set from its exact LCP array
 * (device): D and L. */
int s5g_dist_stats(const int64_t *lcps, int64_t n, int64_t *out_D, int64_t *out_L, void *stream);

/* K-way LCP merge of k <= 16 sorted runs (lcpmerge.kway_lcp_merge,
 * lcpmerge.py:385-424, and the merge phase of parallel.partitioned_merge_sort,
 * parallel.py:885-994).  Run j is handles[run_offsets[j] .. run_offsets[j+1])
 * with its LCP array in lcps at the same positions (lcps[run start] is not
 * read) and, when dchar != NULL, its distinguishing characters (fill_dchar
 * convention; the cached comparisons of lcp_compare_cached).  run_offsets is
 * a HOST array of k + 1 entries; everything else is device memory.  All
 * strings share their first `shared` characters.  Output: the stable merge
 * (ties to the earlier run) and its LCP array with out_lcps[0] = shared.
 * Workspace: s5g_merge_workspace_bytes(n, k). */
size_t s5g_merge_workspace_bytes(int64_t n, int32_t k);
int s5g_kway_merge(const uint8_t *arena, int64_t arena_len, int32_t k, const int64_t *run_offsets,
                   const int64_t *handles, const int64_t *lcps, const uint8_t *dchar,
                   int64_t shared, int64_t *out_handles, int64_t *out_lcps, void *workspace,
                   size_t workspace_bytes, void *stream, s5g_stats *stats);

/* fill_dchar (basecase.py:36-42). */
int s5g_fill_dchar(const uint8_t *arena, const int64_t *handles, const int64_t *lcps, int64_t n,
                   uint8_t *out_dchar, void *stream);

/* --- instrumentation ------------------------------------------------------ */

/* Per-kernel-class device time, recorded with CUDA events on the launching
 * stream around every launch of s5g_sort while enabled. */
typedef struct s5g_kernel_profile {
    char name[32];
    int64_t launches;
    int64_t units;     /* elements (or segments / records) the launches covered */
    double ms;         /* summed event-timed duration */
    int64_t bytes;     /* summed algorithmic bytes (DESIGN.md kernel models) */
} s5g_kernel_profile;

/* on = 1: events around every launch, streams as in production (the timeline);
 * on = 2: the same with every kernel on the caller's stream, so each launch's
 * event time is exclusive and the per-kernel sums add up to the sort. */
void s5g_profile_enable(int on);
void s5g_profile_reset(void);
int s5g_profile_read(s5g_kernel_profile *out, int max_entries);
/* Launch timeline of the last sort run with profiling enabled: kernel index
 * (into s5g_profile_read's table), stream (0 = caller's, 1 = side stream of
 * the pipelined finishers), start / end in ms from the sort's first event.
 * Returns the number of launches (entries beyond max_entries are dropped). */
int s5g_profile_timeline(int *kid, int *stream, float *t0, float *t1, int max_entries);
/* Monotonic count of kernels this library has launched (all entry points). */
unsigned long long s5g_launch_count(void);
/* L2 fetch granularity (bytes: 32, 64 or 128) requested for the duration of
 * each sort (cudaLimitMaxL2FetchGranularity; restored afterwards).  Default 32:
 * the sort is dominated by random 8-byte gathers and stores. */
void s5g_set_l2_fetch_granularity(int bytes);
/* Finisher counters accumulated over all sorts on the current device since
 * the last reset: for k_cta_sort<2>, <4>, <8> (entries 4c .. 4c+3 for c =
 * 0, 1, 2): CTAs, CTA-wide rounds, two-word first rounds, group-mode exits.
 * Copies min(n, 12) entries to out; reset != 0 zeroes them afterwards. */
int s5g_finisher_counters(unsigned long long *out, int n, int reset);

const char *s5g_last_error(void);
int s5g_version(void);

#ifdef __cplusplus
}
#endif
#endif /* S5G_H */
