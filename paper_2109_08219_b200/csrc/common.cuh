// common.cuh -- shared device helpers for the Dr. Top-k sm_100a kernels.
//
// Key spaces, PTX wrappers (mbarrier, 1-D TMA bulk copy, acquire/release),
// block scans, the radix-select digit finder, decoupled look-back, and the
// device-resident control block that carries state between the kernels of
// one dtopk_select call (so the host never synchronises mid-pipeline).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/dtopk.h"

#ifndef DTOPK_TAIL_MINB
#define DTOPK_TAIL_MINB 4  // scan_emit min CTAs per SM (register cap 79 -> 64: one wave on large pools; capping k4_read too slowed small k)
#endif

namespace dtopk {

using u32 = uint32_t;
using u64 = uint64_t;
using ull = unsigned long long;

constexpr u32 FULL = 0xffffffffu;

// ---------------------------------------------------------------------------
// Key maps.  All selection runs on u32 keys where a larger key wins.
// ---------------------------------------------------------------------------
enum KeyMode { KM_U32_MAX = 0, KM_U32_MIN = 1, KM_F32_MAX = 2, KM_F32_MIN = 3, KM_KEY = 4 };

template <int M>
__device__ __forceinline__ u32 to_key(u32 b) {
  if constexpr (M == KM_U32_MAX || M == KM_KEY) {
    return b;
  } else if constexpr (M == KM_U32_MIN) {
    return ~b;
  } else {
    u32 u = b ^ ((u32)((int)b >> 31) | 0x80000000u);
    if constexpr (M == KM_F32_MAX) return u;
    return ~u;
  }
}

template <int M>
__device__ __forceinline__ u32 from_key(u32 u) {
  if constexpr (M == KM_U32_MAX || M == KM_KEY) {
    return u;
  } else if constexpr (M == KM_U32_MIN) {
    return ~u;
  } else {
    if constexpr (M == KM_F32_MIN) u = ~u;
    return u ^ ((u & 0x80000000u) ? 0x80000000u : 0xffffffffu);
  }
}

// Radix digits of a key: 11 / 11 / 10 bits, most significant first.
constexpr int NB1 = 2048, NB2 = 2048, NB3 = 1024;
__device__ __forceinline__ u32 dig1(u32 k) { return k >> 21; }
__device__ __forceinline__ u32 dig2(u32 k) { return (k >> 10) & 0x7ffu; }
__device__ __forceinline__ u32 dig3(u32 k) { return k & 0x3ffu; }

// Digits of the delegate threshold theta = kth(D).  Delegates are maxima, so
// they crowd the top of the key range: a linear top-11-bit bucket can hold
// most of D (the max of 2048 uniform keys lands in the top 1/2048 of the
// range with probability 0.63).  The first digit is therefore log-scale in
// the distance from the top, d = ~key: (leading zeros of d, next DSB bits of
// d), 33 x 2^DSB buckets ordered like the keys.  A bucket is a key interval
// [kmin, kmin + 2^r) with r <= 31 - DSB; digit 2 = (key - kmin) >> 13,
// digit 3 = (key - kmin) & 8191.  DSB = 7 (was 6): float32 keys put a whole
// octave of values in one (clz, 6-bit) bucket, so theta's bucket outgrew the
// one-CTA tail on N(0,1) data; 7 bits halve every bucket.
constexpr int DSB = 7;                                  // sub-bits of the first digit
constexpr u32 DSB_MASK = (1u << DSB) - 1u;
// float32 keys are already logarithmic (sign, exponent, mantissa), and their
// maxima crowd near the data's maximum, not near 0xffffffff: for them the first
// digit is linear, the top 13 key bits (16 buckets per octave).  N(0,1) data at
// k = 1024: theta's bucket 33,862 delegates with the log digit, ~3 k linear.
constexpr int DLIN_SHIFT = 19;
constexpr int NBD1 = 8192;  // max(33 x 128 log buckets, 2^13 linear), a multiple of 512 (find_digit reads bin pairs)
constexpr int NBD2 = 4096, NBD3 = 8192;
constexpr int DSH3 = 13;  // digit 2 = (key - kmin) >> 13 (<= 11 bits), digit 3 = low 13 bits
__device__ __forceinline__ u32 ddig1(u32 key) {
  const u32 d = ~key;
  if (d == 0) return (32u << DSB) | DSB_MASK;
  const u32 c = __clz(d);
  const u32 m = c >= 31 ? 0u : (d << (c + 1)) >> (32 - DSB);
  return (c << DSB) | (DSB_MASK - m);
}
// key interval [kmin, kmax] of log bucket b
__device__ __forceinline__ void dbucket_range(u32 b, u32& kmin, u32& kmax) {
  const u32 c = b >> DSB, m = DSB_MASK - (b & DSB_MASK);
  if (c >= 32) {
    kmin = kmax = 0xffffffffu;
    return;
  }
  const u32 lead = 1u << (31 - c);
  u32 dlo, dhi;
  if (c <= 31 - DSB) {
    const u32 r = 31 - DSB - c;
    dlo = lead | (m << r);
    dhi = dlo | ((1u << r) - 1u);
  } else {
    dlo = dhi = lead | (m >> (c - (31 - DSB)));
  }
  kmin = ~dhi;
  kmax = ~dlo;
}

__device__ __forceinline__ u32 ddig(u32 key, bool lin) { return lin ? (key >> DLIN_SHIFT) : ddig1(key); }
__device__ __forceinline__ void dbucket(u32 b, bool lin, u32& kmin, u32& kmax) {
  if (lin) {
    kmin = b << DLIN_SHIFT;
    kmax = kmin | ((1u << DLIN_SHIFT) - 1u);
  } else {
    dbucket_range(b, kmin, kmax);
  }
}

// ---------------------------------------------------------------------------
// Control block (device memory, zeroed once per call).
// ---------------------------------------------------------------------------
struct DigitResult {
  u32 digit;
  u32 valid;
  ull rem;    // rank still sought inside the chosen bucket (1-based)
  ull cnt;    // population of the chosen bucket
  ull above;  // population of all higher buckets
};

struct alignas(16) SelectState {  // 16-byte aligned: find_digit reads the histograms as ulonglong2
  ull hist1[NBD1];  // sized for the delegate digits; the pool select uses NB1/NB2/NB3 of them
  ull hist2[NBD2];
  ull hist3[NBD3];
  ull buf_count;  // pass-2 compaction counter
  DigitResult r1, r2, r3;
  u32 kth;
  u32 done3;
};

enum Path : u32 { PATH_NONE = 0, PATH_SELECT = 1, PATH_MERGE = 2, PATH_DIRECT = 3 };

struct Ctrl {
  dtopk_result res;   // host-visible header (kept first: dtopk_result_offset() == 0)
  SelectState selD;   // theta = kth(delegates)
  SelectState selP;   // tau = kth(pool) or kth(V) on the direct path
  // qualification (K3): ordered records of subranges with max delegate >= theta
  u32 k3_ticket;
  u32 nE;          // class-E records (read by K4)
  ull cand_count;  // records
  ull nA;          // class-A records (one element > theta each)
  ull gt_rec_end;  // 1 + last record index that holds elements > theta
  u32 sup_total;   // records = candidate-superset entries (K2, resolved with theta)
  u32 k2b_done;    // K2b CTAs finished (exact superset of a deferred, large-bucket call)
  ull sumEgt;      // elements > theta found by K4
  // assembly (K5) and tie location (K6)
  u32 k5_ticket;
  u32 ties_full;
  u32 k6_count;
  u32 small_done;  // finish_small wrote the answer
  u32 nT;          // class-T records (tie-only, counted by K4T)
  u32 nTslots;     // T-list slots handed out by K3 (>= nT for beta 2: C entries leave holes)
  u32 k4t_ticket;
  u32 k4t_completed;  // tickets K4T has finished (bounds how far ahead tickets are handed out)
  ull k4t_eq_done; // ties of the word chunks K4T has completed
  // emit and sort of the answer
  u32 em_ticket;
  u32 maxkey;
  u32 sort_lo;
  u32 sort_src;    // 0: sort buffer A holds the input, 1: buffer B
  ull sort_m;      // elements to sort
  u32 big_mode;    // 0 done by finish_small, 1 merge (append ties), 2 sort the pool, 3 radix select
  u32 sort_done;   // last-block counter of sort_scan
  u32 lsd_fallback;
  u32 bk_ticket;     // last-block counter of bucket_scan  // large answer too skewed for the bucket sort: LSD radix sort instead
  // filtered delegate pass (K0 sample -> K1 records -> K2 over records; delegate.cuh)
  u32 filt_on;    // K0: K1 writes records of subranges with d_1 >= filt_t instead of D / meta
  u32 filt_t;     // K0: floor of the sample bucket at ~1.25 k delegates (a lower bound of theta's bucket floor)
  u32 filt_fail;  // K2: the floor was above theta's bucket (or the bucket is huge): full K1 + K2 rerun
  u32 samp_done;  // K0 last-CTA counter
  // theta's first-digit bucket holding a large share of D (tie-heavy input)
  u32 bk_nmin, bk_max;  // K2: ~min and max of the bucket's members (one value: theta without a digit-3 pass)
  u32 trunc;            // pass 3: tie-only superset entries past tie_cut are dropped (enough ties before it)
  u32 tie_cut;          // last K2b segment whose tie-only entries are kept
  u32 tb_done;          // K2c last-CTA counter
  // pool floor (K4h, large E re-reads): the exact k-th-largest bin of the pool's keys
  u32 pfloor;           // keys below it (and above theta) stay out of P_gt; 0 = off
  u32 pf_ticket;        // K4h last-CTA counter
  ull below_floor;      // E keys in (theta, pfloor): counted into |C| by K5
  alignas(16) ull pf_hist[2048];
  alignas(16) ull samp_hist[NBD1];  // K0: first-digit histogram of the sampled subranges' delegates
};

enum BigMode : u32 { BIG_NONE = 0, BIG_MERGE = 1, BIG_SORT_POOL = 2, BIG_SELECT = 3 };

// ---------------------------------------------------------------------------
// PTX wrappers
// ---------------------------------------------------------------------------
__device__ __forceinline__ u32 smem_addr(const void* p) {
  return (u32)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(u64* bar, u32 count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(u64* bar, u32 bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(u64* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(u32 addr, u32 parity) {
  u32 ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(addr), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(u64* bar, u32 parity) {
  const u32 a = smem_addr(bar);
  while (!mbar_try_wait(a, parity)) {
  }
}
// 1-D TMA bulk copy global -> shared, completion signalled on `bar`.
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, u32 bytes, u64* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

// The same copy with an L2 cache-policy hint (createpolicy): K1 streams the
// whole input once, so its lines are marked evict_first and do not push the
// delegates, the workspace and the kernels' code out of the 126 MB L2.
__device__ __forceinline__ u64 l2_policy_evict_first() {
  u64 pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void tma_load_1d_hint(void* dst, const void* src, u32 bytes, u64* bar, u64 policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(policy)
      : "memory");
}

// Bulk prefetch of global memory into L2 (no shared-memory destination).
__device__ __forceinline__ void l2_prefetch_bulk(const void* src, u32 bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

__device__ __forceinline__ u64 ld_acquire(const u64* p) {
  u64 v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(u64* p, u64 v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ u32 ld_volatile_u32(const u32* p) {
  return *(const volatile u32*)p;
}

__device__ __forceinline__ uint4 ld_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// Programmatic dependent launch (PDL): the post-K1 chain is launched with
// programmatic stream serialization, so each kernel's CTAs are scheduled while
// its predecessor still runs and block here until the predecessor's grid has
// completed and its writes are visible.  pdl_trigger lets the next kernel in
// the chain be scheduled as soon as every CTA of this one has started.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ u32 lanemask_lt() {
  u32 m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Warp-aggregated shared-memory histogram increment; all 32 lanes must call.
__device__ __forceinline__ void hist_add_agg(u32* shist, u32 bin, bool pred) {
  const u32 key = pred ? bin : 0xffffffffu;
  const u32 peers = __match_any_sync(FULL, key);
  if (pred && (u32)(__ffs(peers) - 1) == (threadIdx.x & 31)) atomicAdd(&shist[bin], (u32)__popc(peers));
}

// Shared-memory histogram increment for mostly-uniform or mostly-identical
// bins: one atomic when the whole warp hits one bin (tie-heavy inputs), plain
// per-lane atomics otherwise.  All 32 lanes must call.
__device__ __forceinline__ void hist_add_warp(u32* shist, u32 bin, bool pred) {
  const u32 key = pred ? bin : 0xffffffffu;
  int same = 0;
  __match_all_sync(FULL, key, &same);
  if (same) {
    if (pred && (threadIdx.x & 31) == 0) atomicAdd(&shist[bin], 32u);
  } else if (pred) {
    atomicAdd(&shist[bin], 1u);
  }
}

// ---------------------------------------------------------------------------
// top-beta ladders (registers, non-increasing, zero initialised: the
// reference's _rows_ladder semantics, delegate.py:93-107)
// ---------------------------------------------------------------------------
template <int B>
__device__ __forceinline__ void ladder_insert(u32 (&L)[B], u32 x) {
#pragma unroll
  for (int i = 0; i < B; i++) {
    const u32 hi = max(L[i], x);
    x = min(L[i], x);
    L[i] = hi;
  }
}

template <int B>
__device__ __forceinline__ void ladder_merge(u32 (&L)[B], const u32 (&R)[B]) {
  if constexpr (B == 1) {
    L[0] = max(L[0], R[0]);
  } else if constexpr (B == 2) {
    const u32 m1 = max(L[0], R[0]);
    const u32 m2 = max(min(L[0], R[0]), max(L[1], R[1]));
    L[0] = m1;
    L[1] = m2;
  } else {
#pragma unroll
    for (int i = 0; i < B; i++) ladder_insert<B>(L, R[i]);
  }
}

// ---------------------------------------------------------------------------
// Block scans for 256-thread blocks.
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T n = __shfl_up_sync(FULL, v, o);
    if (lane >= o) v += n;
  }
  return v;
}

// Inclusive scan over the first 256 threads; all 256 must call. `scratch` >= 8.
template <typename T>
__device__ __forceinline__ T block_incl_scan_256(T v, T* scratch) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  v = warp_incl_scan(v);
  if (lane == 31) scratch[w] = v;
  __syncthreads();
  T add = 0;
#pragma unroll
  for (int i = 0; i < 8; i++)
    if (i < w) add += scratch[i];
  __syncthreads();
  return v + add;
}

// Radix-select digit finder: among NB buckets (hist in global memory), find
// the bucket b holding the k_rem-th largest key: suffix(b+1) < k_rem <= suffix(b).
// Must be called by all 256 threads of a block; result broadcast via `out` (smem).
template <int NB>
__device__ void find_digit(const ull* hist, ull k_rem, DigitResult* out, ull* scratch) {
  constexpr int PER = NB / 256;
  static_assert(PER % 2 == 0, "find_digit reads bin pairs");
  const int t = threadIdx.x;
  ull loc[PER];
  ull sum = 0;
  // thread t owns bins NB-1-t*PER .. NB-PER-t*PER (descending); 16-byte loads of bin pairs
  const ulonglong2* h2 = reinterpret_cast<const ulonglong2*>(hist + NB - PER - t * PER);
#pragma unroll
  for (int i = 0; i < PER / 2; i++) {
    const ulonglong2 q = __ldcg(&h2[i]);  // bins NB-PER-t*PER + 2i, +2i+1
    loc[PER - 1 - 2 * i] = q.x;
    loc[PER - 2 - 2 * i] = q.y;
  }
#pragma unroll
  for (int i = 0; i < PER; i++) sum += loc[i];
  if (t == 0) out->valid = 0;
  const ull incl = block_incl_scan_256<ull>(sum, scratch);
  ull run = incl - sum;
#pragma unroll
  for (int i = 0; i < PER; i++) {
    const int b = NB - 1 - (t * PER + i);
    if (run < k_rem && run + loc[i] >= k_rem) {
      out->digit = (u32)b;
      out->rem = k_rem - run;
      out->cnt = loc[i];
      out->above = run;
      out->valid = 1;
    }
    run += loc[i];
  }
  __syncthreads();
}

// find_digit over a shared-memory u32 histogram (same contract as find_digit).
// PAD: bin b is stored at b + b / 32 (thread t's PER = 32 bins then start 33 t
// words apart: conflict-free, instead of a 32-way conflict on every read).
template <int NB, bool PAD = false>
__device__ void find_digit_sm(const u32* sh, ull k_rem, DigitResult* out, ull* scratch) {
  constexpr int PER = NB / 256;
  const int t = threadIdx.x;
  u32 loc[PER];
  ull sum = 0;
#pragma unroll
  for (int i = 0; i < PER; i++) {
    const u32 b = (u32)(NB - 1 - (t * PER + i));
    loc[i] = sh[PAD ? b + (b >> 5) : b];
    sum += loc[i];
  }
  if (t == 0) out->valid = 0;
  const ull incl = block_incl_scan_256<ull>(sum, scratch);
  ull run = incl - sum;
#pragma unroll
  for (int i = 0; i < PER; i++) {
    const int b = NB - 1 - (t * PER + i);
    if (run < k_rem && run + loc[i] >= k_rem) {
      out->digit = (u32)b;
      out->rem = k_rem - run;
      out->cnt = loc[i];
      out->above = run;
      out->valid = 1;
    }
    run += loc[i];
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// Decoupled look-back over a chain of u64 tile states:
//   bits 63..62 flag (0 empty, 1 aggregate, 2 inclusive prefix), 61..0 value.
// A tile publishes its aggregate, a whole warp walks back 32 predecessors per
// step (summing aggregates until the nearest inclusive prefix), then the tile
// publishes its own inclusive prefix.
// ---------------------------------------------------------------------------
constexpr u64 LB_VAL = (1ull << 62) - 1;
constexpr u64 LB_AGG = 1ull << 62;
constexpr u64 LB_PRE = 2ull << 62;

__device__ __forceinline__ void lb_publish_agg(u64* st, u64 tile, u64 agg) {
  st_release(&st[tile], (tile == 0 ? LB_PRE : LB_AGG) | agg);
}

// All 32 lanes of one warp call; the exclusive prefix is returned in every lane.
__device__ __forceinline__ u64 lb_warp_prefix(u64* st, u64 tile) {
  const int lane = threadIdx.x & 31;
  u64 excl = 0;
  long long hi = (long long)tile - 1;
  while (hi >= 0) {
    const long long t = hi - lane;
    u64 s = LB_PRE;  // before tile 0 the prefix is 0
    if (t >= 0) {
      do {
        s = ld_acquire(&st[t]);
      } while ((s >> 62) == 0);
    }
    const u32 pre = __ballot_sync(FULL, (s >> 62) == 2);
    const int stop = pre ? __ffs(pre) - 1 : 31;
    u64 v = lane <= stop ? (s & LB_VAL) : 0;
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    excl += v;
    if (pre) break;
    hi -= 32;
  }
  return excl;
}

__device__ __forceinline__ void lb_publish_prefix(u64* st, u64 tile, u64 incl) {
  if (tile != 0) st_release(&st[tile], LB_PRE | incl);
}

}  // namespace dtopk
