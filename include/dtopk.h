/*
 * dtopk.h -- C ABI of the B200-native Dr. Top-k hot path (libdtopk.so).
 *
 * Plain pointers and sizes only: no torch / Python types cross this boundary.
 * Every entry point is stream-ordered on the caller's cudaStream_t, never
 * synchronises the stream, and never allocates device memory: the caller
 * passes a workspace of at least dtopk_workspace_bytes(...) bytes.
 *
 * Reference interfaces replaced (paths under the reference package
 * pkg/src/dtopk/):
 *   dtopk_select            <- pipeline.dr_topk                (pipeline.py:172-220)
 *                              incl. the direct fallback       (pipeline.py:184-191)
 *   dtopk_select_begin/     <- the same call split at the threshold, so a
 *   dtopk_select_finish        multi-GPU caller can all-reduce theta between
 *                              the first top-k and the concatenation
 *                              (distributed.py:162 runs dr_topk per partition;
 *                              the exchange is the one PAPER.md:738-742 disabled)
 *   dtopk_extract_delegates <- delegate.extract_delegates      (delegate.py:142-155)
 *                              and extract_delegates_blocked   (delegate.py:158-191)
 *   dtopk_kth_largest       <- kernels.radix_topk threshold    (kernels.py:109-165),
 *                              used by pipeline.first_topk     (pipeline.py:87-116)
 *   dtopk_qualify           <- pipeline.first_topk qualification (pipeline.py:87-116)
 *   dtopk_concat            <- pipeline.concatenate_filtered    (pipeline.py:119-159)
 *   dtopk_min_at_least      <- radix_topk skip_last relaxation  (kernels.py:161-164)
 *   dtopk_merge_lists,      <- the coordinator's merge of worker lists
 *   dtopk_dsel_*               (distributed.py:191-251)
 *   dtopk_workspace_bytes   <- (no reference counterpart: numpy allocates implicitly)
 *
 * Key spaces: every kernel works on 32-bit *keys* where "larger key" means
 * "selected first".  uint32 largest is the identity map, uint32 smallest is
 * ~x, float32 uses the order-preserving bijection
 *     u = (b >> 31) ? ~b : b | 0x80000000      (then ~u for smallest).
 * Results are returned in the input dtype; indices are int64 positions into
 * the input (plus the caller's index_offset for sharded inputs).
 */
#ifndef DTOPK_H_
#define DTOPK_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  DTOPK_OK = 0,
  DTOPK_EMPTY_INPUT = 1,        /* core.EmptyInput   (core.py:37-38)  */
  DTOPK_INVALID_K = 2,          /* core.InvalidK     (core.py:33-34)  */
  DTOPK_INVALID_BETA = 3,       /* core.InvalidBeta  (core.py:41-42)  */
  DTOPK_INVALID_ARG = 4,        /* ValueError (bad alpha / dtype / alignment) */
  DTOPK_WORKSPACE_TOO_SMALL = 5,
  DTOPK_CUDA_ERROR = 6,
  DTOPK_UNSUPPORTED = 7         /* beta > 32 with subranges of more than 8192 keys */
} dtopk_status;

typedef enum { DTOPK_U32 = 0, DTOPK_F32 = 1 } dtopk_dtype;

/* flags for dtopk_select / dtopk_select_begin */
#define DTOPK_FLAG_EXACT_STATS 1u  /* re-read tie-only subranges so concatenated_len is exact */
#define DTOPK_FLAG_DELEGATES_DONE 2u  /* dtopk_select: K1 already ran via dtopk_delegates_range */

/* Device-resident result header, written by the kernels of one call.
 * Field names follow core.WorkloadStats (core.py:59-93) where they overlap. */
typedef struct {
  uint64_t k_out;                 /* number of (value, index) pairs written (== k unless a
                                     larger external theta was applied)              */
  uint64_t candidate_subranges;   /* subranges with max delegate >= theta              */
  uint64_t fully_qualified;       /* beta-th delegate >= theta     (pipeline.py:104-108) */
  uint64_t partially_qualified;   /* max >= theta > beta-th delegate (pipeline.py:109,205) */
  uint64_t concatenated_len;      /* |C|: elements >= theta of fully qualified subranges */
  uint64_t concat_skipped_fq;     /* work skipped because the first k ties were already placed;
                                     concatenated_len is exact iff this is 0          */
  uint64_t elements_reread;       /* input elements re-read by the concatenation stage */
  uint64_t pool_gt;               /* G: elements strictly above theta                  */
  uint64_t pool_eq;               /* ties at theta collected (capped by k)             */
  uint64_t delegate_bucket;       /* delegates in theta's top-11-bit bucket            */
  uint32_t theta_local;           /* kth(D) in key space                               */
  uint32_t theta;                 /* threshold actually used (max with external theta) */
  uint32_t kth_key;               /* exact k-th key of the answer                      */
  uint32_t path;                  /* 1 = radix select over the pool, 2 = merge, 3 = direct */
  int64_t theta_slot;             /* theta_local as int64, target of an all-reduce(MAX) */
  uint32_t filtered;              /* 1: K1 stored only records of subranges above a sampled floor */
  uint32_t filter_fallback;       /* 1: that floor missed theta's bucket; full K1 + K2 re-ran     */
} dtopk_result;

/* Bytes of workspace needed by dtopk_select for these parameters. */
size_t dtopk_workspace_bytes(uint64_t n, uint64_t k, int alpha, int beta, int direct);

/* Byte offset of the dtopk_result header inside the workspace. */
size_t dtopk_result_offset(void);

/*
 * Full top-k: pipeline.dr_topk (pipeline.py:172-220), delegate path or, with
 * direct != 0, the direct radix top-k fallback (pipeline.py:184-191).
 *   keys          device pointer, 16-byte aligned, n elements of `dtype`
 *   k             1 <= k <= n
 *   largest       1 = top-k largest, 0 = smallest
 *   alpha, beta   resolved by validate_config (core.py:145-174); ignored if direct
 *   out_values    device, k elements of `dtype`, ordered best first
 *   out_indices   device, k int64 positions (+ index_offset); ties broken by
 *                 lowest index, final order (key desc, index asc)
 *   index_offset  added to every output index (global offset of a shard)
 *   ws, ws_bytes  workspace; the dtopk_result header lives at
 *                 ws + dtopk_result_offset()
 *   stage_events  null, or 5 events from dtopk_event_create() recorded at the
 *                 stage boundaries start | Delegate | FirstK | Concat | SecondK
 *                 (core.STAGES, core.py:22-26; pipeline.py:187-219 timers)
 */
dtopk_status dtopk_select(const void* keys, uint64_t n, int dtype, uint64_t k, int largest,
                          int alpha, int beta, int direct, uint32_t flags,
                          void* out_values, int64_t* out_indices, int64_t index_offset,
                          void* ws, size_t ws_bytes, void* stream, void* const* stage_events);

/* A plan fixes every argument of dtopk_select (input, outputs, workspace) and
 * captures the whole launch sequence into a CUDA graph.  The large-pool tail
 * sits behind a device-side conditional node that finish_small sets, so for
 * pools of <= 8192 pairs its kernels are not launched at all.  Replaying the
 * plan is equivalent to calling dtopk_select with the same arguments. */
typedef struct dtopk_plan_s* dtopk_plan;
dtopk_status dtopk_plan_create(const void* keys, uint64_t n, int dtype, uint64_t k, int largest,
                               int alpha, int beta, int direct, uint32_t flags,
                               void* out_values, int64_t* out_indices, int64_t index_offset,
                               void* ws, size_t ws_bytes, dtopk_plan* out_plan);
dtopk_status dtopk_plan_launch(dtopk_plan plan, void* stream);
/* kernels in the always-executed part and in the conditional tail */
void dtopk_plan_kernels(dtopk_plan plan, unsigned long long* main_kernels, unsigned long long* tail_kernels);
void dtopk_plan_destroy(dtopk_plan plan);

/* Streamed host input (distributed.py:97-137 residency / reload plan,
 * PAPER.md:928-932): K1 over K1 chunks [chunk_begin, chunk_end) (2048 keys
 * each, ceil(n / 2048) in all) of the device buffer `keys`, as soon as that
 * range has arrived (chunk_begin == 0 also clears the workspace).  After the
 * last range, dtopk_select with DTOPK_FLAG_DELEGATES_DONE finishes the call.
 * beta <= 8.  The ranges must cover every chunk exactly once. */
dtopk_status dtopk_delegates_range(const void* keys, uint64_t n, int dtype, uint64_t k, int largest,
                                   int alpha, int beta, uint64_t chunk_begin, uint64_t chunk_end,
                                   void* ws, size_t ws_bytes, void* stream);

/* First half of dtopk_select (delegate path only): delegates, theta = kth(D).
 * Afterwards dtopk_result.theta_slot holds theta (int64) in device memory. */
dtopk_status dtopk_select_begin(const void* keys, uint64_t n, int dtype, uint64_t k, int largest,
                                int alpha, int beta, uint32_t flags,
                                void* ws, size_t ws_bytes, void* stream, void* const* stage_events);

/* Second half: uses theta = max(theta_local, *theta_override) when
 * theta_override (device int64*) is non-null.  May emit k_out < k pairs when an
 * external theta is larger than this shard's k-th key. */
dtopk_status dtopk_select_finish(const void* keys, uint64_t n, int dtype, uint64_t k, int largest,
                                 int alpha, int beta, uint32_t flags,
                                 const int64_t* theta_override,
                                 void* out_values, int64_t* out_indices, int64_t index_offset,
                                 void* ws, size_t ws_bytes, void* stream, void* const* stage_events);

/* delegate.extract_delegates: out_delegates[beta*ceil(n/2^alpha)] in key space,
 * subrange-major, non-increasing inside a subrange, zero-padded tail
 * (delegate.py:132-139).  Needs dtopk_workspace_bytes(n, 1, alpha, beta, 0). */
dtopk_status dtopk_extract_delegates(const void* keys, uint64_t n, int dtype, int largest,
                                     int alpha, int beta, uint32_t* out_delegates,
                                     void* ws, size_t ws_bytes, void* stream);

/* Exact k-th largest key of a uint32 key array (radix select, 11/11/10-bit
 * digits); writes it to *out_kth (device).  Needs
 * dtopk_workspace_bytes(n, k, 0, 1, 1). */
dtopk_status dtopk_kth_largest(const uint32_t* keys, uint64_t n, uint64_t k, uint32_t* out_kth,
                               void* ws, size_t ws_bytes, void* stream);

/* ---- Stage operators (stage-level API and its parity tests) ----
 * dtopk_qualify        <- pipeline.first_topk qualification (pipeline.py:87-116):
 *   given the delegate vector (key space, beta per subrange) and theta, writes
 *   in D order the selected delegates (>= theta) and their subrange tags, the
 *   partial ones (selected, subrange not fully qualified) and the fully
 *   qualified subrange ids (d_beta >= theta, ascending); out_counts[3] =
 *   (selected, partial, fully qualified).  Output buffers hold up to
 *   n_delegates (selected / partial) and n_delegates / beta (ids) entries.
 * dtopk_concat         <- pipeline.concatenate_filtered (pipeline.py:119-159):
 *   elements whose key is >= theta of the listed subranges (ascending ids),
 *   subrange-ascending then scan order, in the input dtype; *out_count on the
 *   device.  out_values holds up to n_fq * 2^alpha elements.
 * dtopk_min_at_least   <- the skip_last relaxation of kernels.radix_topk
 *   (kernels.py:161-164): *out_min = min{ key >= edge } (0xffffffff if none).
 * Workspace: dtopk_stage_workspace_bytes(n_delegates) for qualify,
 * dtopk_stage_workspace_bytes(n_fq << alpha) for concat. */
size_t dtopk_stage_workspace_bytes(uint64_t n_elements);
dtopk_status dtopk_qualify(const uint32_t* delegates, uint64_t n_delegates, int beta, uint32_t theta,
                           uint32_t* sel_values, uint32_t* sel_tags, uint32_t* part_values, uint32_t* part_tags,
                           uint32_t* fq_sids, int64_t* out_counts, void* ws, size_t ws_bytes, void* stream);
dtopk_status dtopk_concat(const void* keys, uint64_t n, int dtype, int largest, int alpha, const uint32_t* fq_sids,
                          uint64_t n_fq, uint32_t theta, void* out_values, int64_t* out_count, void* ws,
                          size_t ws_bytes, void* stream);
dtopk_status dtopk_min_at_least(const uint32_t* keys, uint64_t n, uint32_t edge, uint32_t* out_min, void* stream);

/* ---- Multi-GPU candidate merge (distributed.py:191-251 coordinator merge) ----
 * Every rank's candidates are (value bits, global index) lists ordered
 * (key desc, index asc); ranks own contiguous shards in rank order.
 *
 * dtopk_merge_lists: exact first `cap` pairs of the merge of n_lists such lists
 * (list j at offset o_j = in_off[j], or j * in_stride when in_off is null;
 * in_len[j * len_stride] valid pairs, device int64), by a tree of pairwise merge-path
 * rounds; equal keys keep list (= index) order.  Indices of list j start at
 * in_idx + o_j; its values at in_val + o_j * vmul (u32 words), one value every
 * vstride words (vstride 2: the low word of int64 slots).  tmp_val / tmp_idx hold dtopk_merge_tmp_pairs(n_lists, cap) pairs,
 * tmp_len 2 * n_lists int64.  Writes exactly min(cap, sum in_len) pairs. */
size_t dtopk_merge_tmp_pairs(int n_lists, uint64_t cap);
dtopk_status dtopk_merge_lists(int dtype, int largest, const uint32_t* in_val, int vmul, int vstride,
                               const int64_t* in_idx, const int64_t* in_off, int64_t in_stride,
                               const int64_t* in_len, int64_t len_stride, int n_lists, uint64_t cap,
                               uint32_t* out_val,
                               int64_t* out_idx, uint32_t* tmp_val, int64_t* tmp_idx, int64_t* tmp_len,
                               void* stream);

/* Distributed radix select over per-rank candidate lists (merge="select"):
 *   dtopk_dsel_init(state[2], hist[2048], k)
 *   for pass in 0..2: dtopk_dsel_hist -> all_reduce(SUM, hist) -> dtopk_dsel_digit
 *     (after pass 2, gt_eq[0..1] = this rank's candidates above / equal to kth)
 *   all_gather(gt_eq) -> gathered[2 * world]
 *   dtopk_dsel_place -> slots[2k] (own pairs in own slots, zero elsewhere) and the
 *     rank segment table; all_reduce(SUM, slots) assembles the answer, which
 *     dtopk_merge_lists(vstride 2, in_off = seg_off, in_len = seg_len) orders. */
dtopk_status dtopk_dsel_init(int64_t* state, int64_t* hist, uint64_t k, void* stream);
dtopk_status dtopk_dsel_hist(int dtype, int largest, const uint32_t* bits, const int64_t* cnt, uint64_t cap,
                             const int64_t* state, int pass, int64_t* hist, void* stream);
dtopk_status dtopk_dsel_digit(int dtype, int largest, int64_t* state, int64_t* hist, int pass,
                              const uint32_t* bits, const int64_t* cnt, int64_t* gt_eq, void* stream);
dtopk_status dtopk_dsel_place(const int64_t* gathered, const int64_t* state, int rank, int world, uint64_t k,
                              const uint32_t* bits, const int64_t* idx, int64_t* slots, int64_t* seg_off,
                              int64_t* seg_len, void* stream);

/* CUDA timing events for stage_events (cudaEventCreate / Destroy /
 * ElapsedTime; elapsed synchronises on `end`). */
void* dtopk_event_create(void);
void dtopk_event_destroy(void* ev);
float dtopk_event_elapsed_ms(void* start, void* end);

/* Deterministic synthetic input (value i depends only on (seed, i)):
 * dist 0 uniform u32, 1 ascending (i + param), 2 constant param,
 * 3 uniform in [0, param), 4 N(0,1) float32, 5 Pareto(param/1000) float32,
 * 6 rint(N(1e8, 10)) u32 (the reference ND set, data.py:65-75),
 * 7 descending (param - i).  Test/bench data only, not the hot path. */
dtopk_status dtopk_generate(void* out, uint64_t n, int dist, uint64_t seed, uint64_t param, void* stream);

/* Number of SMs the library sizes its persistent grids for (current device). */
int dtopk_num_sms(void);

/* Total kernels this library has launched in the process (for benchmarks). */
unsigned long long dtopk_launch_count(void);

/* Library version string. */
const char* dtopk_version(void);

#ifdef __cplusplus
}
#endif

#endif /* DTOPK_H_ */
