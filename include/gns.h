/*
 * gns.h — C-ABI of the B200-native greeNsort hot path (arXiv 2402.01816).
 *
 * What the library computes: the STABLE ASCENDING sort ("AscLeft") of n
 * contiguous IEEE binary64 keys in device memory, optionally moving a u32
 * payload with each key, by binary divide&conquer merge sort under a buffer
 * budget.  Citations are PAPER.md (= /root/reference/PAPER.md) line numbers:
 *   - sorting = rearrangement into ascending order, stable: ties keep their
 *     input order left to right (§Definition of sorting, Knuth's
 *     definition, target "AscLeft");
 *   - keys compare by IEEE `<`: -0.0 == +0.0, stability fixes their order, and
 *     every output key keeps its input bits;
 *   - per merge level one read-scan with comparisons and one write-scan
 *     (§Merging or partitioning?), alternating between data and a
 *     100% buffer (Nocopy-Mergesort) with Knuth's merge, the left
 *     run winning ties ("Knuthsort");
 *   - buffer fraction 0.5: the left half is sorted into a half-size buffer, the
 *     right half in place, then both are merged back into the data
 *     (Timsort's <=50% buffer merge; Frogsort's "50% or less
 *     local buffer", PAPER.md:13/260/291; buffer sharing between branches as in
 *     Frogsort3) so %RAM = (dataRAM+bufferRAM)/dataRAM
 *      is 1.5 instead of 2.0.
 *
 * Conventions for every entry point:
 *   - Pointers named keys/vals/src/dst/ws are DEVICE pointers.  The caller owns
 *     them; they must stay valid and untouched until the enqueued work on
 *     `stream` completes.
 *   - Alignment: the sorts (gns_sort_f64, _pairs_, _target_,
 *     gns_sort_keys, gns_sort_omit and their _ws forms) need natural alignment
 *     only -- keys 8-byte, vals 4-byte aligned (any view t[i:j] of a torch
 *     tensor).  32-byte aligned arrays take the fast path directly; other
 *     arrays peel the <= 7 head elements before the first 32-byte boundary,
 *     sort the aligned rest and merge the head in place (one extra read +
 *     write pass, gns_peel.cuh).  Keys and vals with no common 32-byte
 *     boundary (e.g. keys[1:] with vals[2:]) route the vals through a
 *     stream-ordered temporary of 4n bytes (the only case that exceeds the
 *     workspace).  The per-step entry points (gns_tile_sort, gns_merge_pass,
 *     gns_merge_inplace_top, gns_merge_two's dst), gns_sort_keys_u64,
 *     gns_sort_f32 and every ws need 32-byte alignment.  Below these:
 *     GNS_ERR_MISALIGNED, data untouched.
 *   - Every call is asynchronous on `stream` (0 = legacy default stream): a
 *     return of GNS_OK means the kernels are enqueued.  No host sync, except
 *     that the non-_ws sorts allocate their buffer stream-ordered
 *     (cudaMallocAsync/cudaFreeAsync on `stream`).
 *   - Argument errors are detected before anything is enqueued: the data is
 *     untouched.  GNS_ERR_CUDA reports a launch/runtime error; the message is
 *     in gns_last_error_string() (thread-local).
 *   - NaN keys are a precondition violation: the contents of keys/vals after
 *     the call are then unspecified, but every access stays inside
 *     keys/vals/the buffer and the call terminates.  With the environment
 *     variable GNS_DEBUG=1 the sorts of f64 keys first count NaNs (one pass
 *     and a host sync) and return GNS_ERR_INVALID_ARGUMENT, data untouched.
 *   - n in {0, 1} returns GNS_OK with no launch; pointers may be NULL if n == 0.
 *   - Reentrant: no global mutable state; concurrent calls on different streams
 *     with disjoint buffers are allowed.
 */
#ifndef GNS_H
#define GNS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *gns_stream_t;   /* == cudaStream_t */

typedef enum {
    GNS_OK = 0,
    GNS_ERR_INVALID_ARGUMENT = 1,      /* NULL pointer with n > 0, n > GNS_MAX_N, bad run_len */
    GNS_ERR_UNSUPPORTED_FRACTION = 2,  /* buffer_fraction not 1.0 and not in [1/64, 0.5]        */
    GNS_ERR_OUT_OF_MEMORY = 3,         /* buffer allocation failed; input untouched            */
    GNS_ERR_CUDA = 4,                  /* CUDA launch/runtime error                             */
    GNS_ERR_WORKSPACE_TOO_SMALL = 5,   /* ws NULL or ws_bytes < gns_workspace_bytes(...)        */
    GNS_ERR_MISALIGNED = 6             /* below the required alignment (see Conventions)        */
} gns_status;

#define GNS_MAX_N ((size_t)0x7FFFFFFF)   /* 2^31 - 1 elements */

/* The four stable API targets of PAPER.md:137-142 (§Definition of sorting,
 * "AscLeft, AscRight, DescLeft and DescRight"): key direction x the memory
 * direction in which ties keep their input order.  AscLeft is the default of
 * every other entry point. */
typedef enum {
    GNS_ASC_LEFT = 0,    /* ascending, ties in input order (left to right)          */
    GNS_ASC_RIGHT = 1,   /* ascending, ties in reverse input order = reverse(DescLeft) */
    GNS_DESC_LEFT = 2,   /* descending, ties in input order                          */
    GNS_DESC_RIGHT = 3   /* descending, ties in reverse input order = reverse(AscLeft) */
} gns_target;

/* ---- the sort (rows a1-a7 of SURVEY.md §8) -------------------------------
 * keys[0:n) (and vals[0:n)) are replaced by their stable ascending sort.
 * buffer_fraction: 1.0 -> buffer of n elements (%RAM 2.0);
 *                  0.5 -> buffer of ceil(n/2) elements rounded up to 32
 *                         (%RAM 1.5 for even n >= 64);
 *                  p in [1/64, 0.5) -> buffer of ceil(p*n) elements rounded up
 *                         to 32 (%RAM ~ 1+p): the right part is sorted first
 *                         (recursively, same buffer), then the left p*n
 *                         elements are sorted into the buffer and merged back
 *                         in place (Frogsort2/3's imbalanced split and shared
 *                         buffer).  More passes, less RAM.
 * For n <= gns_tile_elems() the sort runs in place with no buffer in either mode. */
gns_status gns_sort_f64(double *keys, size_t n, double buffer_fraction, gns_stream_t stream);
gns_status gns_sort_pairs_f64_u32(double *keys, uint32_t *vals, size_t n,
                                  double buffer_fraction, gns_stream_t stream);

/* Caller-owned workspace variants: ws must hold gns_workspace_bytes(...)
 * bytes (32-byte aligned).  ws is the whole bufferRAM of the call. */
size_t gns_workspace_bytes(size_t n, double buffer_fraction, int with_vals);
gns_status gns_sort_f64_ws(double *keys, size_t n, double buffer_fraction,
                           void *ws, size_t ws_bytes, gns_stream_t stream);
gns_status gns_sort_pairs_f64_u32_ws(double *keys, uint32_t *vals, size_t n,
                                     double buffer_fraction, void *ws, size_t ws_bytes,
                                     gns_stream_t stream);

/* NEXT f3: any of the four targets.  vals may be NULL (key-only).  ws may be
 * NULL (buffer allocated stream-ordered) or a workspace of
 * gns_workspace_bytes(n, buffer_fraction, vals != NULL) bytes.  The Right
 * targets add one in-place reversal pass.  Errors as above, plus
 * GNS_ERR_INVALID_ARGUMENT for an unknown target. */
gns_status gns_sort_target_f64(double *keys, uint32_t *vals, size_t n, double buffer_fraction, gns_target target,
                               void *ws, size_t ws_bytes, gns_stream_t stream);

/* NEXT f3: 8-byte key types.  All share the layout of the f64 path (keys
 * 8-byte aligned words, 32-byte aligned array); only the order differs:
 *   GNS_KEY_F64 binary64 under IEEE < (-0.0 == +0.0; NaN is a precondition
 *               violation, R1), GNS_KEY_I64 two's-complement
 *               int64, GNS_KEY_U64 uint64.
 * Stability (ties keep input order for the Left targets) as above: the
 * output is the unique stable permutation, bit-exact. */
typedef enum {
    GNS_KEY_F64 = 0,
    GNS_KEY_I64 = 1,
    GNS_KEY_U64 = 2
} gns_key_type;

/* The general entry point: keys of any gns_key_type, optional u32 payload,
 * any target, optional workspace (as gns_sort_target_f64).  keys points to n
 * 8-byte keys (double / int64_t / uint64_t).  GNS_ERR_INVALID_ARGUMENT for an
 * unknown key_type or target; other errors as above. */
gns_status gns_sort_keys(void *keys, gns_key_type key_type, uint32_t *vals, size_t n, double buffer_fraction,
                         gns_target target, void *ws, size_t ws_bytes, gns_stream_t stream);

/* NEXT f3: 64-bit payloads.  keys (any gns_key_type) are sorted as by
 * gns_sort_keys with the full buffer and any target; vals[n] (uint64_t, e.g.
 * a 64-bit index or pointer) moves with its key.  The payload rides through
 * the sort as a u32 index (the pairs path), then is gathered once (random
 * 8-byte reads) into the free pairs buffer and copied back: %RAM = 2.0 of
 * the 16-byte elements, about one extra HBM pass over the payload.
 * ws: NULL (allocated stream-ordered) or gns_workspace_bytes_u64(n) bytes,
 * 32-byte aligned.  Errors as gns_sort_keys. */
size_t gns_workspace_bytes_u64(size_t n);
gns_status gns_sort_keys_u64(void *keys, gns_key_type key_type, uint64_t *vals, size_t n, gns_target target,
                             void *ws, size_t ws_bytes, gns_stream_t stream);

/* NEXT f3: binary32 keys.  keys[n] (float) are replaced by their stable sort
 * for `target` (IEEE order, -0.0 == +0.0 with stability fixing their order,
 * every key keeps its bits); vals[n] (u32, or NULL) move with them.  Its own
 * 4-byte kernels (csrc/gns_f32.cuh): the same schedule as the f64 full-buffer
 * sort -- one tile-sort pass (8192-key tiles, every level on chip), then one
 * HBM merge pass per level, ping-pong with a buffer of n keys (+ n vals):
 * %RAM 2.0.  ws: NULL (allocated stream-ordered) or
 * gns_workspace_bytes_f32(n, vals != NULL) bytes (0 for n <= 8192), 32-byte
 * aligned.  NaN keys: precondition
 * violation.  Errors as gns_sort_keys. */
size_t gns_workspace_bytes_f32(size_t n, int with_vals);
gns_status gns_sort_f32(float *keys, uint32_t *vals, size_t n, gns_target target, void *ws, size_t ws_bytes,
                        gns_stream_t stream);

/* NEXT f2: Omitsort (§Full adaptivity) on the full buffer
 * (%RAM 2.0; workspace = gns_workspace_bytes(n, 1.0, vals != NULL)).  Same
 * result as gns_sort_keys (the unique stable sort), different schedule: every
 * sorted run carries its location (data or buffer); a pair of runs in
 * different regions first moves the buffer-resident run to the data region
 * (the paper's "copies one to the data region"); a pair whose runs do not
 * overlap (B's first key not before A's last) is not merged at all ("omitted",
 * zero moves); others are merged into the other region.  The tile sort
 * leaves tiles already in order where they are and writes the others to the
 * data array (even number of merge levels) or the buffer (odd), so that an
 * input whose every pair merges ends in the data array.  A run that ends in
 * the buffer is copied back once.  Presorted input moves no key; partially
 * presorted input (long ascending runs) moves only where runs overlap; random
 * input costs ~25 us of planning plus ~5 us per level over gns_sort_keys.
 * Arguments, alignment and errors as gns_sort_keys (ws may be NULL: allocated
 * stream-ordered).
 * Octosort in the same schedule: a strictly reversed tile is
 * kept as a descending run, disjoint descending runs stay descending, a
 * descending run meeting anything else is reversed once; a descending result
 * is reversed at the end (strictly reversed input: one reversal pass). */
gns_status gns_sort_omit(void *keys, gns_key_type key_type, uint32_t *vals, size_t n, gns_target target, void *ws,
                         size_t ws_bytes, gns_stream_t stream);

/* ---- NEXT f4: the steps of the distributed sort (paper_2402_01816_b200.dist,
 * SURVEY.md §8(e); "parallelize over an arbitrary number of processes",
 * PAPER.md:353).  Each rank sorts its shard (gns_sort_keys), the ranks find
 * the exact cuts at global ranks g N / k by rounds of proposals (key, owner
 * rank, position in the owner's sorted shard) counted with gns_split_cuts and
 * summed by one all-reduce (or, faster but unbalanced, cut at sample
 * splitters), exchange the pieces (one NCCL all-to-all-v) and merge the k
 * received sorted runs in rank order (gns_merge_two, a pairwise tree).
 * Global order: (key, rank, position), i.e. stable in the rank-major input
 * order. */

/* cuts[i] = number of keys of sorted_keys[0:n) (this rank's sorted shard,
 * ascending in key_type order) that precede splitter i in the global order:
 * my_rank < spl_rank[i]: keys <= spl_keys[i]; my_rank > spl_rank[i]:
 * keys < spl_keys[i]; my_rank == spl_rank[i]: spl_pos[i] (clamped to [0, n]).
 * All pointers are device pointers; spl_keys holds nsplit 8-byte keys.
 * Asynchronous on `stream`; GNS_ERR_INVALID_ARGUMENT for NULL pointers,
 * nsplit < 0 or an unknown key type. */
gns_status gns_split_cuts(const void *sorted_keys, gns_key_type key_type, size_t n, const void *spl_keys,
                          const int32_t *spl_rank, const int64_t *spl_pos, int nsplit, int my_rank, int64_t *cuts,
                          gns_stream_t stream);

/* Stable merge of two sorted runs a[0:la) and b[0:lb) (ascending in key_type
 * order; a's keys win ties) into dst[0:la+lb), out of place.  a and b may
 * live anywhere (8-byte aligned keys, 4-byte aligned vals, not overlapping
 * dst); dst must be 32-byte aligned.  vals: dst_vals and the vals of every
 * non-empty run, or none (an empty run's pointers may be NULL).  Row a3+a4's
 * kernel in its two-run geometry; one launch, asynchronous. */
gns_status gns_merge_two(const void *a_keys, const uint32_t *a_vals, size_t la, const void *b_keys,
                         const uint32_t *b_vals, size_t lb, void *dst_keys, uint32_t *dst_vals, gns_key_type key_type,
                         gns_stream_t stream);

/* Pass schedule of a sort (host only, no CUDA call). */
typedef struct {
    int tile;                   /* gns_tile_elems(): elements per tile-sort CTA          */
    int merge_tile;             /* elements per merge CTA                                 */
    int merge_passes;           /* HBM merge passes of a 1.0-mode sort of n               */
    int hbm_passes;             /* ceil(element_passes)                                   */
    int launches;               /* kernel launches of the sort                            */
    double element_passes;      /* sum over all steps of elements moved through HBM / n;  */
                                /* 1.0 mode: 1 + merge_passes; 0.5 mode about the same    */
    size_t left_len;            /* 0.5 mode: elements sorted into the buffer (nl)         */
    size_t workspace_bytes;     /* = gns_workspace_bytes(n, fraction, with_vals)          */
    size_t buffer_elems;        /* key(+val) slots in the workspace (bufferRAM / s)       */
    size_t bytes_lower_bound;   /* element_passes * n * 2 * s, s = 8 or 12: algorithmic   */
                                /* bytes (one read-scan + one write-scan per level)       */
} gns_plan_info;
gns_status gns_plan(size_t n, double buffer_fraction, int with_vals, gns_plan_info *out);

/* ---- the steps, exposed for per-step parity tests and per-kernel timing -- */

/* Row a2 (K1): stable sort of each gns_tile_elems()-element tile of src into the same
 * range of dst (dst == src allowed; otherwise the ranges must not overlap).
 * vals may both be NULL (key-only). */
gns_status gns_tile_sort(const double *src_keys, const uint32_t *src_vals,
                         double *dst_keys, uint32_t *dst_vals, size_t n, gns_stream_t stream);

/* Rows a3+a4 (K2+K3): one merge level.  For q = 0,1,..: merges the sorted runs
 * src[2qL : 2qL+L) and src[2qL+L : 2qL+2L) (clipped to n) into dst[2qL : ..).
 * run_len L must be a positive multiple of gns_merge_tile_elems()/2 (so every
 * pair starts on a merge-tile boundary), at most 2^30.  src and dst must not
 * overlap.  ws: >= gns_merge_workspace_bytes(n) bytes (co-rank array). */
size_t gns_merge_workspace_bytes(size_t n);
gns_status gns_merge_pass(const double *src_keys, const uint32_t *src_vals,
                          double *dst_keys, uint32_t *dst_vals, size_t n, size_t run_len,
                          void *ws, size_t ws_bytes, gns_stream_t stream);

/* Row a6 (K2+K4): ordered in-place top merge of the limited-buffer modes.
 * left_keys[0:nl) (a separate buffer) and keys[nl:n) are sorted runs; the
 * stable merge (left wins ties) is written to keys[0:n).  Requires
 * 0 < nl <= n, nl % 32 == 0 and left_* not overlapping keys/vals.
 * ws: >= gns_merge_workspace_bytes(n). */
gns_status gns_merge_inplace_top(double *keys, uint32_t *vals, const double *left_keys,
                                 const uint32_t *left_vals, size_t nl, size_t n,
                                 void *ws, size_t ws_bytes, gns_stream_t stream);

/* ---- launch timing (measurement) ---------------------------
 * gns_timing_begin(max_launches): until gns_timing_end, every kernel this
 * library launches FROM THE CALLING THREAD is bracketed by CUDA events recorded
 * on the launching stream (one before the first launch, one after each).  The
 * events serialise the launches (no programmatic overlap), so use it for
 * per-kernel shares, not for whole-sort timing.  Launches beyond max_launches
 * (1..4096) are not timed.  GNS_ERR_INVALID_ARGUMENT if already on.
 * gns_timing_end(ms, kind, cap): waits for the last event, writes up to cap
 * per-launch durations (milliseconds) and kinds (1 tile sort, 2 merge pass,
 * 3 co-rank partition, 4 in-place dependency ranges, 5 in-place merge,
 * 6 reversal, 7 splitter cuts, 8 sample gather, 9 Omitsort plan, 10 Omitsort
 * tile list + copies, 11 Omitsort final copy, 12 / 13 index and gather of
 * gns_sort_keys_u64, 0 other -- incl. the binary32 kernels) in
 * launch order, turns timing off and returns the number of timed launches
 * (-1 if timing was off or an event failed). */

/* Measurement helper (bench.py, SURVEY §8(a) row a7 "measured %RAM"): the
 * high-water mark in bytes of the current device's default memory pool --
 * the pool the non-_ws sorts allocate their buffer from (cudaMallocAsync) --
 * since the last reset.  reset != 0 resets it to the current usage first and
 * returns 0.  Returns (size_t)-1 on a CUDA error.  Synchronous (no stream
 * work); call it outside timed regions. */
size_t gns_pool_high_water(int reset);
gns_status gns_timing_begin(int max_launches);
int gns_timing_end(float *ms, int *kind, int cap);

/* Compile-time geometry of this build. */
int gns_tile_elems(void);
int gns_merge_tile_elems(void);

const char *gns_status_string(gns_status s);
const char *gns_last_error_string(void);

#ifdef __cplusplus
}
#endif
#endif /* GNS_H */
