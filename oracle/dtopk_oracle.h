/*
 * dtopk_oracle.h -- CPU restatement of the reference Dr. Top-k path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library; it
 * is the checker, never the product.  The product path (libdtopk.so) has no
 * CPU fallback.
 *
 * Every function cites the reference code it restates (paths under
 * /root/reference/pkg/src/dtopk/).  Parity of this restatement against the
 * reference itself is pinned by tests/golden/ (vectors produced by the
 * reference package in the build container, see tests/golden/make_golden.py).
 */
#ifndef DTOPK_ORACLE_H_
#define DTOPK_ORACLE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  uint64_t delegate_vector_len;          /* core.WorkloadStats fields (core.py:69-74) */
  uint64_t concatenated_len;
  uint64_t fully_qualified_subranges;
  uint64_t partially_qualified_subranges;
  uint64_t elements_read;
  uint64_t elements_written;
  uint32_t theta;                        /* first_topk threshold (pipeline.py:93)      */
  uint32_t threshold;                    /* values[k-1]                                */
  uint64_t pool_len;                     /* |C| + |partial entries|                    */
} oracle_stats;

/* tuning.auto_alpha (tuning.py:74-90) */
int oracle_auto_alpha(uint64_t n, uint64_t k, double const_c, int beta);

/* core.effective_beta (core.py:132-136) */
int oracle_effective_beta(int beta, int alpha);

/* delegate.extract_delegates values (delegate.py:58-155): out[beta*ceil(n/2^alpha)] */
void oracle_extract_delegates(const uint32_t* v, uint64_t n, int alpha, int beta, uint32_t* out);

/* kernels.radix_topk threshold (kernels.py:109-165), 8-bit digits.
 * skip_last=0: exact k-th largest; skip_last=1: min{x >= prefix_bits}.
 * *reads (nullable) accumulates the reference's logical read counter. */
uint32_t oracle_radix_threshold(const uint32_t* vals, uint64_t m, uint64_t k, int skip_last, uint64_t* reads);

/* pipeline.dr_topk (pipeline.py:172-220) on uint32 keys, radix backend.
 * direct != 0 runs the direct fallback (pipeline.py:184-191).
 * out_values[k] non-increasing.  Returns 0 on success, <0 on bad arguments. */
int oracle_dr_topk(const uint32_t* v, uint64_t n, uint64_t k, int alpha, int beta, int skip_last, int direct,
                   uint32_t* out_values, oracle_stats* st);

/* Index restatement of kernels._extract_exact (kernels.py:83-96) applied to
 * the whole input: every key > kth, then the first (k - #gt) keys == kth in
 * index order; emitted ordered by (key desc, index asc). */
void oracle_topk_indices(const uint32_t* keys, uint64_t n, uint64_t k, uint32_t kth, uint32_t* out_keys,
                         int64_t* out_idx);

/* Order-preserving float32 -> uint32 key map; largest=0 also inverts. */
void oracle_f32_to_keys(const uint32_t* bits, uint64_t n, int largest, uint32_t* out);

/* distributed.run_distributed analogue (distributed.py:191-251): equal
 * partitions (plan rule, distributed.py:97-131), one dr_topk per partition on
 * `threads` POSIX threads with auto alpha per partition, merge by sort.
 * Returns 0 on success. */
int oracle_dr_topk_partitioned(const uint32_t* v, uint64_t n, uint64_t k, int beta, double const_c, int workers,
                               uint32_t* out_values);

/* Host twin of the device generator's uniform distribution
 * (csrc/generate.cuh, dist 0): out[i] = splitmix64(key(seed) + offset + i) >> 32,
 * filled on `threads` POSIX threads.  Input preparation for the CPU baseline. */
void oracle_generate_uniform(uint32_t* out, uint64_t n, uint64_t seed, uint64_t offset, int threads);

#ifdef __cplusplus
}
#endif

#endif
