// delegate.cuh -- K1: one streaming pass over the input that emits the
// top-beta delegates of every 2^alpha subrange (reference: delegate.py:58-191).
//
// Design (B200):
//  * persistent grid, one 288-thread CTA per SM: warp 8 is a TMA producer that
//    streams 8 KiB chunks (2048 keys) into a 16-stage shared-memory ring with
//    1-D cp.async.bulk + mbarrier completion; each of warps 0-7 owns every 8th
//    stage and reduces whole chunks on its own (no CTA-wide barriers).
//  * consumers read the staged chunk with bank-conflict-free LDS.128, apply the
//    key map on the fly (float->ordered u32, ~x for smallest) and keep a
//    register top-beta ladder per lane; subranges are reduced in registers
//    (W <= 64), with xor-shuffle butterflies (W <= 2048) or as per-chunk
//    partials merged by a tiny second kernel (W > 2048).
//  * the first radix digit (top 11 bits) of every delegate is histogrammed in
//    shared memory and flushed once per CTA: pass 1 of the delegate top-k is
//    fused into the stream, so the delegate vector is read only once more.
#pragma once

#include "common.cuh"

namespace dtopk {

constexpr int K1_CHUNK = 2048;    // keys per stage = one warp's unit of work (8 KiB)
constexpr int K1_LOG_CHUNK = 11;
#ifndef DTOPK_K1_CWARPS
#define DTOPK_K1_CWARPS 8
#endif
#ifndef DTOPK_K1_CPS
#define DTOPK_K1_CPS 1
#endif
constexpr int K1_CWARPS = DTOPK_K1_CWARPS;  // consumer warps
constexpr int K1_CPS = DTOPK_K1_CPS;        // resident CTAs per SM
#ifndef DTOPK_K1_STAGES
#define DTOPK_K1_STAGES 16
#endif
#ifndef DTOPK_K1_EXP
#define DTOPK_K1_EXP 0  // profiling experiments only (tools/k1_exp.cu): 1 = no consumer work, 2 = no emit
#endif
#ifndef DTOPK_K1_PREFETCH
#define DTOPK_K1_PREFETCH 0
#endif
constexpr int K1_STAGES = DTOPK_K1_STAGES;  // stages in flight (a multiple of the consumer warps)
constexpr int K1_PREFETCH = DTOPK_K1_PREFETCH;  // chunks prefetched into L2 ahead of the TMA ring
#ifndef DTOPK_K1_HCOPIES
#define DTOPK_K1_HCOPIES 1
#endif
// copies of the shared first-digit histogram, picked by lane: at small alpha
// every lane emits its own subrange, and the delegates (maxima) crowd into a
// few log-scale bins, so same-address atomics serialise inside a warp
constexpr int K1_HCOPIES = DTOPK_K1_HCOPIES;
constexpr int K1_THREADS = (K1_CWARPS + 1) * 32;
// beta >= 3 ladders are compute-bound at 8 consumer warps (f32 beta 3: 0.86 ms vs
// 0.74 at beta 2); 16 warps (one per ring stage) restore the stream: 0.78 ms
template <int B>
constexpr int k1_cwarps() { return B >= 3 ? 16 : K1_CWARPS; }
template <int B>
constexpr int k1_threads() { return (k1_cwarps<B>() + 1) * 32; }
constexpr size_t K1_SMEM = (size_t)K1_STAGES * K1_CHUNK * 4 + 2 * K1_STAGES * 8 + (size_t)NBD1 * 4 * K1_HCOPIES;

struct K1Args {
  const u32* keys;
  u64 n;
  int alpha;
  u64 S;         // number of subranges = ceil(n / 2^alpha)
  u32* D;        // [S][B] delegates (key space)
  u32* partial;  // [nchunks][B] when alpha > K1_LOG_CHUNK
  ull* hist1;    // global first-digit histogram of D
  int do_hist;
  u32* meta;     // [S] (min(c1, 0xffff) << 16) | (p1 & 0xffff): count and position of the max
  u32* pmeta;    // [2 * nchunks] c1 / p1 of the chunk partials (alpha > K1_LOG_CHUNK)
  // filtered mode (alpha 6..8, beta <= 2; see k0_sample): fmode 0 = always full
  // (D + meta), 1 = records {sid, d_1, d_2, meta} of the subranges with d_1 >=
  // ctrl->filt_t when ctrl->filt_on (else full), 2 = full, only if ctrl->filt_fail
  Ctrl* ctrl;
  int fmode;
  uint4* frec;     // per consumer warp of the grid, a contiguous stream of fcap records
  u32* chunk_cnt;  // [nchunks] (offset of chunk c's records in its warp's stream << 6) | count
  u64 fcap;        // records per warp stream: ceil(nchunks / (grid * 8)) * (2048 >> alpha)
  u64 c_begin, c_end;  // chunks this launch reduces (a streamed host input arrives range by range)
  int lin;             // first digit: linear (float32 keys) or log-scale (uint32)
};

// Per-lane accumulator: top-B ladder, uint4 index p of the running maximum
// (updated only on a strictly larger uint4 maximum, so it names the first
// uint4 that holds d_1) and the running minimum (a subrange is constant iff
// min == max).  Per uint4 and B = 2 this is 13 integer min/max/select ops:
// pairwise sort, top-2 of the four, merge into the ladder.
template <int B>
struct Acc {
  u32 L[B];
  u32 p;
  u32 mn;
  __device__ __forceinline__ void init(u32 p0) {
#pragma unroll
    for (int i = 0; i < B; i++) L[i] = 0;
    p = p0;
    mn = 0xffffffffu;
  }
};

// x: keys for the ladder (absent = 0), y: keys for the minimum (absent = ~0)
template <int B>
__device__ __forceinline__ void acc_keys(Acc<B>& A, const u32 (&x)[4], const u32 (&y)[4], u32 q) {
  if constexpr (B == 1) {
    const u32 t1 = max(max(x[0], x[1]), max(x[2], x[3]));
    A.p = t1 > A.L[0] ? q : A.p;
    A.L[0] = max(A.L[0], t1);
  } else if constexpr (B == 2) {
    const u32 h1 = max(x[0], x[1]), l1 = min(x[0], x[1]);
    const u32 h2 = max(x[2], x[3]), l2 = min(x[2], x[3]);
    const u32 t1 = max(h1, h2), t2 = max(min(h1, h2), max(l1, l2));
    A.p = t1 > A.L[0] ? q : A.p;
    const u32 n1 = max(A.L[0], t1);
    const u32 n2 = max(max(min(A.L[0], t1), A.L[1]), t2);
    A.L[0] = n1;
    A.L[1] = n2;
  } else if constexpr (B == 3 || B == 4) {
    // sort the four keys (t1 >= t2 >= t3 >= t4), then merge the two sorted
    // lists: top-B of L u t without per-key insertion chains
    const u32 h1 = max(x[0], x[1]), l1 = min(x[0], x[1]);
    const u32 h2 = max(x[2], x[3]), l2 = min(x[2], x[3]);
    const u32 t1 = max(h1, h2), m = min(h1, h2), M = max(l1, l2), t4 = min(l1, l2);
    const u32 t2 = max(m, M), t3 = min(m, M);
    A.p = t1 > A.L[0] ? q : A.p;
    if constexpr (B == 3) {
      const u32 a0 = A.L[0], a1 = A.L[1], a2 = A.L[2];
      A.L[0] = max(a0, t1);
      A.L[1] = max(min(a0, t1), max(a1, t2));
      A.L[2] = max(max(a2, t3), max(min(a0, t2), min(a1, t1)));
    } else {
      // bitonic: r_i = max(a_i, t_{3-i}) is bitonic and holds the top 4; sort it
      const u32 r0 = max(A.L[0], t4), r1 = max(A.L[1], t3), r2 = max(A.L[2], t2), r3 = max(A.L[3], t1);
      const u32 s0 = max(r0, r2), s2 = min(r0, r2), s1 = max(r1, r3), s3 = min(r1, r3);
      A.L[0] = max(s0, s1);
      A.L[1] = min(s0, s1);
      A.L[2] = max(s2, s3);
      A.L[3] = min(s2, s3);
    }
  } else {
    const u32 t1 = max(max(x[0], x[1]), max(x[2], x[3]));
    A.p = t1 > A.L[0] ? q : A.p;
#pragma unroll
    for (int c = 0; c < 4; c++) ladder_insert<B>(A.L, x[c]);
  }
  A.mn = min(A.mn, min(min(y[0], y[1]), min(y[2], y[3])));
}

template <int B>
__device__ __forceinline__ void acc_merge(Acc<B>& A, const u32 (&R)[B], u32 rp, u32 rmn) {
  A.p = R[0] > A.L[0] ? rp : A.p;
  A.mn = min(A.mn, rmn);
  ladder_merge<B>(A.L, R);
}

template <int B>
__device__ __forceinline__ void acc_shfl(Acc<B>& A, int off) {
  u32 R[B];
#pragma unroll
  for (int i = 0; i < B; i++) R[i] = __shfl_xor_sync(FULL, A.L[i], off);
  const u32 rp = __shfl_xor_sync(FULL, A.p, off);
  const u32 rmn = __shfl_xor_sync(FULL, A.mn, off);
  acc_merge<B>(A, R, rp, rmn);
}

// beta = 2 merge of a whole warp's accumulators with warp reductions instead
// of five shuffle butterfly levels: d_1 = max, the first lane holding it
// supplies p, d_2 = max over the other lanes' L[0] and that lane's L[1],
// min = min.  (Partial-mask reductions for smaller groups measured slower than
// the butterflies.)  All 32 lanes must call.
template <int B>
__device__ __forceinline__ void acc_warp_b2(Acc<B>& A) {
  if constexpr (B == 2) {
    const int lane = threadIdx.x & 31;
    const u32 m = __reduce_max_sync(FULL, A.L[0]);
    const int first = __ffs(__ballot_sync(FULL, A.L[0] == m)) - 1;
    const u32 m2 = __reduce_max_sync(FULL, lane == first ? A.L[1] : A.L[0]);
    A.p = __shfl_sync(FULL, A.p, first);
    A.mn = __reduce_min_sync(FULL, A.mn);
    A.L[0] = m;
    A.L[1] = m2;
  }
}

// Whole-warp top-B merge for B != 2: B rounds of a warp max over the lanes'
// ladder heads (each lane's ladder is non-increasing); the first lane holding
// the round's max advances, so duplicates count once per copy -- the top-B
// multiset.  p comes from the first lane holding the overall max.  All 32
// lanes must call.
template <int B>
__device__ __forceinline__ void acc_warp_merge(Acc<B>& A) {
  const int lane = threadIdx.x & 31;
  u32 out[B];
  int ptr = 0;
  u32 p0 = 0;
#pragma unroll
  for (int r = 0; r < B; r++) {
    u32 head = 0;
#pragma unroll
    for (int i = 0; i < B; i++) head = ptr == i ? A.L[i] : head;
    const u32 m = __reduce_max_sync(FULL, head);
    const int first = __ffs(__ballot_sync(FULL, head == m)) - 1;
    if (r == 0) p0 = __shfl_sync(FULL, A.p, first);
    ptr += lane == first ? 1 : 0;
    out[r] = m;
  }
  A.mn = __reduce_min_sync(FULL, A.mn);
  A.p = p0;
#pragma unroll
  for (int i = 0; i < B; i++) A.L[i] = out[i];
}

// meta word of a subrange: bit 31 = constant subrange (every key equals d_1),
// bits 0..30 = offset of an occurrence of d_1 inside the subrange (exact and
// unique whenever d_2 < d_1).
__device__ __forceinline__ u32 pack_meta(bool constant, u32 p1) { return (constant ? 0x80000000u : 0u) | (p1 & 0x7fffffffu); }


template <int B>
__device__ __forceinline__ void store_delegates(u32* D, u64 sid, const u32 (&L)[B]) {
  if constexpr (B == 2) {
    *reinterpret_cast<uint2*>(D + sid * 2) = make_uint2(L[0], L[1]);
  } else if constexpr (B == 4) {
    *reinterpret_cast<uint4*>(D + sid * 4) = make_uint4(L[0], L[1], L[2], L[3]);
  } else {
#pragma unroll
    for (int i = 0; i < B; i++) D[sid * B + i] = L[i];
  }
}

// Emit one subrange's delegates: lanes with `leader` write; every lane of the
// warp must call (warp-aggregated histogram).
template <int B>
__device__ __forceinline__ void emit_subrange(const K1Args& a, u32* shist, u64 sid, bool leader,
                                              const u32 (&L)[B], u32 meta, bool one_writer = false) {
  const bool w = leader && sid < a.S;
  if (w && DTOPK_K1_EXP != 4) {
    store_delegates<B>(a.D, sid, L);
    a.meta[sid] = meta;
  }
  if (a.do_hist && DTOPK_K1_EXP != 3) {
    if constexpr (K1_HCOPIES > 1) shist += (threadIdx.x & (K1_HCOPIES - 1)) * NBD1;
    if (one_writer) {  // a single emitting lane: no aggregation needed
      if (w) {
#pragma unroll
        for (int i = 0; i < B; i++) atomicAdd(&shist[ddig(L[i], a.lin)], 1u);
      }
    } else {
#pragma unroll
      for (int i = 0; i < B; i++) {
        // plain shared atomics: measured faster than match_any aggregation, also on all-equal input
        if (w) atomicAdd(&shist[ddig(L[i], a.lin)], 1u);
      }
    }
  }
}

// Filtered emission (alpha >= 6: one call per chunk, every lane calls): the
// delegates still feed the first-digit histogram, but only subranges whose max
// delegate reaches the sampled floor `ft` are stored, as superset-format
// records appended to the warp's own contiguous stream (`wrun` records so far);
// lane 0 stores the chunk's (stream offset, count).  D and meta are not written
// at all.  Measured (tools/k1_alpha.py): at alpha 6 the full D + meta writes
// cost K1 ~90 us, chunk-strided record slots (one partial line per chunk) ~43
// us; dense per-warp streams touch ~4x fewer lines.
template <int B>
__device__ __forceinline__ void emit_filtered(const K1Args& a, u32* shist, u64 c, u64 sid, bool leader,
                                              const u32 (&L)[B], u32 meta, u32 ft, u32& wrun) {
  const bool w = leader && sid < a.S;
  const bool keep = w && L[0] >= ft;
  const u32 q = __ballot_sync(FULL, keep);
  const u32 base = (blockIdx.x * K1_CWARPS + (threadIdx.x >> 5)) * (u32)a.fcap;
  if (keep && DTOPK_K1_EXP != 6)
    a.frec[(u64)base + wrun + __popc(q & lanemask_lt())] = make_uint4((u32)sid, L[0], B >= 2 ? L[1] : 0u, meta);
  if ((threadIdx.x & 31) == 0 && DTOPK_K1_EXP != 5) a.chunk_cnt[c] = (wrun << 6) | __popc(q);
  wrun += __popc(q);
  if (a.do_hist) {
    if constexpr (K1_HCOPIES > 1) shist += (threadIdx.x & (K1_HCOPIES - 1)) * NBD1;
#pragma unroll
    for (int i = 0; i < B; i++)
      if (w) atomicAdd(&shist[ddig(L[i], a.lin)], 1u);
  }
}

template <int MODE, bool TAIL>
__device__ __forceinline__ u32 k1_fetch(const K1Args& a, u64 start, u32 e, u32 cnt, u32 tcnt, u32 smv) {
  if constexpr (!TAIL) {
    return to_key<MODE>(smv);
  } else {
    if (e >= cnt) return 0u;  // absent: zero pad (delegate.py:132-139)
    if (e >= tcnt) return to_key<MODE>(a.keys[start + e]);
    return to_key<MODE>(smv);
  }
}

// Insert the four keys of one uint4 at chunk offset e (p1 records chunk
// offsets).  Absent tail keys (e >= cnt) are zero padded in the ladder --
// inserting 0 into a zero-initialised ladder is a no-op -- and never counted.
// Keys of the uint4 at chunk offset e (TAIL: absent keys become 0 for the
// ladder and ~0 for the minimum).
template <int MODE, bool TAIL>
__device__ __forceinline__ void load_keys(const K1Args& a, u64 start, u32 e, u32 cnt, u32 tcnt, const uint4 v,
                                          u32 (&x)[4], u32 (&y)[4]) {
  const u32 r[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int c = 0; c < 4; c++) {
    x[c] = k1_fetch<MODE, TAIL>(a, start, e + c, cnt, tcnt, r[c]);
    y[c] = (TAIL && e + c >= cnt) ? 0xffffffffu : x[c];
  }
}

// Resolve the exact position of d_1 inside the uint4 p (chunk-relative uint4
// index) by re-reading it from the staged chunk; returns the subrange meta.
template <int MODE, int B, bool TAIL>
__device__ __forceinline__ u32 finalize_meta(const K1Args& a, const uint4* st4, u64 start, u32 cnt, u32 tcnt,
                                             const Acc<B>& A) {
  u32 x[4], y[4];
  load_keys<MODE, TAIL>(a, start, A.p * 4u, cnt, tcnt, st4[A.p], x, y);
  u32 c = 3;
#pragma unroll
  for (int i = 3; i >= 0; i--)
    if (x[i] == A.L[0]) c = (u32)i;
  const u32 e = A.p * 4u + c;
  const u64 wmask = (1ull << a.alpha) - 1;
  return pack_meta(A.mn == A.L[0], (u32)((start + e) & wmask));
}

// One warp reduces one staged chunk of 2048 keys.  No CTA-wide barrier: the
// eight consumer warps run decoupled, each on its own stages.
// `rel`: the stage's empty barrier.  The lane-contiguous path (alpha >= 6,
// full chunks) releases the stage as soon as its last shared-memory read is
// done -- before the subrange butterflies and the delegate stores -- and then
// returns true; otherwise the caller releases it.
template <int MODE, int B, bool TAIL>
__device__ __forceinline__ bool k1_warp_chunk(const K1Args& a, const u32* stage, u64 c, u32* shist, u64* rel,
                                              bool filt, u32 ft, u32& wrun) {
  const int lane = threadIdx.x & 31;
  const u64 start = c << K1_LOG_CHUNK;
  const u32 cnt = TAIL ? (u32)min((u64)K1_CHUNK, a.n - start) : (u32)K1_CHUNK;
  const u32 tcnt = TAIL ? ((cnt * 4u) & ~15u) / 4u : (u32)K1_CHUNK;
  const int alpha = a.alpha;
  const uint4* st4 = reinterpret_cast<const uint4*>(stage);

  if (alpha <= 4) {
    // ---- W <= 16, lane-interleaved: uint4 q = j*32 + lane; a subrange spans W/4 lanes
#pragma unroll 2
    for (int j = 0; j < 16; j++) {
      const u32 q = (u32)j * 32u + (u32)lane;
      u32 x[4], y[4];
      load_keys<MODE, TAIL>(a, start, q * 4u, cnt, tcnt, st4[q], x, y);
      if (alpha == 1) {
        if constexpr (B == 1) {
#pragma unroll
          for (int h = 0; h < 2; h++) {
            const u32 lo = x[2 * h], hi = x[2 * h + 1];
            u32 L0[1] = {max(lo, hi)};
            const u32 mn = min(y[2 * h], y[2 * h + 1]);
            const u32 off = hi > lo ? 1u : 0u;  // first occurrence of the max
            emit_subrange<1>(a, shist, ((start + q * 4u) >> 1) + h, true, L0, pack_meta(mn == L0[0], off));
          }
        }
      } else {
        Acc<B> A;
        A.init(q);
        acc_keys<B>(A, x, y, q);
        const int G = 1 << (alpha - 2);
        for (int off = 1; off < G; off <<= 1) acc_shfl<B>(A, off);
        const u32 meta = finalize_meta<MODE, B, TAIL>(a, st4, start, cnt, tcnt, A);
        emit_subrange<B>(a, shist, (start + q * 4u) >> alpha, (lane & (G - 1)) == 0, A.L, meta);
      }
    }
    return false;
  }

  // ---- lane-contiguous: lane owns keys [lane*64, lane*64+64).  LDS.128 order
  // is rotated by lane inside each subrange-aligned group of >= 8 uint4 so a
  // quarter-warp always hits 8 distinct 16-byte bank groups.  Two accumulators
  // (even / odd uint4) halve the dependent chain through the ladder.
  const u32 q0 = (u32)lane * 16u;
  if (alpha == 5) {
#pragma unroll
    for (int h = 0; h < 2; h++) {
      Acc<B> A0, A1;
      A0.init(q0 + h * 8);
      A1.init(q0 + h * 8);
#pragma unroll
      for (int jj = 0; jj < 8; jj++) {
        const u32 q = q0 + h * 8 + ((jj + lane) & 7);
        u32 x[4], y[4];
        load_keys<MODE, TAIL>(a, start, q * 4u, cnt, tcnt, st4[q], x, y);
        acc_keys<B>((jj & 1) ? A1 : A0, x, y, q);
      }
      acc_merge<B>(A0, A1.L, A1.p, A1.mn);
      const u32 meta = finalize_meta<MODE, B, TAIL>(a, st4, start, cnt, tcnt, A0);
      emit_subrange<B>(a, shist, (start + (q0 + h * 8) * 4u) >> 5, true, A0.L, meta);
    }
    return false;
  }
  Acc<B> A0, A1;
  A0.init(q0);
  A1.init(q0);
#pragma unroll
  for (int jj = 0; jj < 16; jj++) {
    const u32 q = q0 + ((jj + lane) & 15);
    u32 x[4], y[4];
    load_keys<MODE, TAIL>(a, start, q * 4u, cnt, tcnt, st4[q], x, y);
    acc_keys<B>((jj & 1) ? A1 : A0, x, y, q);
  }
  acc_merge<B>(A0, A1.L, A1.p, A1.mn);
  if constexpr (DTOPK_K1_EXP == 2) {
    if (A0.L[0] == 0x12345678u && A0.p == 7u) a.D[c] = A0.mn;
    return false;
  }
  // exact chunk offset of this lane's maximum (first occurrence inside its
  // uint4), read while the stage is still owned; then hand the stage back
  {
    u32 x[4], y[4];
    load_keys<MODE, TAIL>(a, start, A0.p * 4u, cnt, tcnt, st4[A0.p], x, y);
    u32 cc = 3;
#pragma unroll
    for (int i = 3; i >= 0; i--)
      if (x[i] == A0.L[0]) cc = (u32)i;
    A0.p = A0.p * 4u + cc;
  }
  bool released = false;
  if (!TAIL && rel != nullptr) {
    __syncwarp();
    if (lane == 0) mbar_arrive(rel);
    released = true;
  }
  const int G = alpha >= K1_LOG_CHUNK ? 32 : 1 << (alpha - 6);  // lanes per subrange (alpha == 6: 1)
  if (B == 2 && G == 32) {
    acc_warp_b2(A0);  // whole-warp subrange (alpha >= 11): warp reductions
  } else if (B != 2 && G == 32) {
    acc_warp_merge(A0);  // whole-warp subrange, beta != 2: B rounds of warp max over the lanes' ladder heads
  } else {
    for (int off = 1; off < G; off <<= 1) acc_shfl<B>(A0, off);
  }
  const u64 wmask = (1ull << alpha) - 1;
  if (alpha <= K1_LOG_CHUNK) {
    const u32 meta = pack_meta(A0.mn == A0.L[0], (u32)((start + A0.p) & wmask));
    if (B <= 2 && filt)
      emit_filtered<B>(a, shist, c, (start + q0 * 4u) >> alpha, (lane & (G - 1)) == 0, A0.L, meta, ft, wrun);
    else
      emit_subrange<B>(a, shist, (start + q0 * 4u) >> alpha, (lane & (G - 1)) == 0, A0.L, meta, G == 32);
  } else {
    // W > 2048: this chunk is one part of a subrange -> partial ladder + the
    // exact offset of its max inside the subrange + its minimum
    if (lane == 0) {
#pragma unroll
      for (int i = 0; i < B; i++) a.partial[c * B + i] = A0.L[i];
      a.pmeta[2 * c] = (u32)((start + A0.p) & wmask);
      a.pmeta[2 * c + 1] = A0.mn;
    }
  }
  return released;
}

// The (single) ragged last chunk goes through an out-of-line copy so the bounds
// checks do not inflate the register budget of the steady-state loop.
template <int MODE, int B>
__device__ __noinline__ void k1_warp_chunk_tail(const K1Args& a, const u32* stage, u64 c, u32* shist, bool filt,
                                                u32 ft, u32& wrun) {
  k1_warp_chunk<MODE, B, true>(a, stage, c, shist, nullptr, filt, ft, wrun);
}

#ifndef DTOPK_K1_EVICT_FIRST
#define DTOPK_K1_EVICT_FIRST 1  // K1's input stream is marked L2 evict_first
#endif
#ifndef DTOPK_K1_CONTIG
#define DTOPK_K1_CONTIG 0  // 1: CTA b reduces the contiguous chunk range [b R, (b+1) R), R = ceil(nch / grid)
#endif

// Chunk of iteration i of this CTA (iteration i uses ring stage i % K1_STAGES
// and consumer warp i % K1_CWARPS), or ~0 past the CTA's last chunk.
__device__ __forceinline__ u64 k1_chunk_of(u64 i, u64 c0, u64 c1) {
  if (DTOPK_K1_CONTIG) {
    const u64 R = (c1 - c0 + gridDim.x - 1) / gridDim.x;
    const u64 c = c0 + (u64)blockIdx.x * R + i;
    return (i < R && c < c1) ? c : ~0ull;
  }
  const u64 c = c0 + blockIdx.x + i * gridDim.x;
  return c < c1 ? c : ~0ull;
}

template <int MODE, int B>
__global__ void __launch_bounds__(k1_threads<B>(), K1_CPS) k1_delegates(K1Args a) {
  constexpr int CW = k1_cwarps<B>();
  static_assert(K1_STAGES % CW == 0, "each consumer warp owns whole ring stages");
  pdl_trigger();
  if (a.fmode == 2 && !ld_volatile_u32(&a.ctrl->filt_fail)) return;  // fallback pass not needed
#ifdef DTOPK_K1_FORCE_FT  // profiling only (tools/k1_alpha.py): filtered emission with a fixed floor
  const bool filt = a.alpha >= 6 && a.alpha <= 11;
  const u32 ft = DTOPK_K1_FORCE_FT;
#else
  const bool filt = a.fmode == 1 && ld_volatile_u32(&a.ctrl->filt_on) != 0;
  const u32 ft = filt ? ld_volatile_u32(&a.ctrl->filt_t) : 0u;
#endif
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  u32* stages = reinterpret_cast<u32*>(smem_raw);
  u64* full = reinterpret_cast<u64*>(smem_raw + (size_t)K1_STAGES * K1_CHUNK * 4);
  u64* empty = full + K1_STAGES;
  u32* shist = reinterpret_cast<u32*>(empty + K1_STAGES);

  const u64 nch = (a.n + K1_CHUNK - 1) >> K1_LOG_CHUNK;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < NBD1 * K1_HCOPIES; i += k1_threads<B>()) shist[i] = 0;
  if (tid == 0) {
    for (int s = 0; s < K1_STAGES; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();

  // Iteration i of this CTA handles chunk blockIdx.x + i*gridDim.x in stage
  // i % 16, consumed by warp i % 8; the stage's parity flips every 16 iterations.
  if (warp == CW) {
    if (lane == 0) {
      u64 i = 0;
      const u64 pol = l2_policy_evict_first();
      for (u64 c = k1_chunk_of(0, a.c_begin, a.c_end); c != ~0ull; c = k1_chunk_of(++i, a.c_begin, a.c_end)) {
        const u32 s = (u32)(i % K1_STAGES);
        const u32 ph = (u32)(i / K1_STAGES) & 1u;
        mbar_wait(&empty[s], ph ^ 1u);
        const u64 start = c << K1_LOG_CHUNK;
        const u64 cnt = min((u64)K1_CHUNK, a.n - start);
        const u32 bytes = (u32)(cnt * 4u) & ~15u;
        if constexpr (K1_PREFETCH > 0) {
          const u64 cp = c + (u64)K1_PREFETCH * gridDim.x;
          if (cp < nch && ((cp + 1) << K1_LOG_CHUNK) <= a.n) l2_prefetch_bulk(a.keys + (cp << K1_LOG_CHUNK), K1_CHUNK * 4u);
        }
        if (bytes) {
          mbar_arrive_expect_tx(&full[s], bytes);
          if constexpr (DTOPK_K1_EVICT_FIRST)
            tma_load_1d_hint(stages + (size_t)s * K1_CHUNK, a.keys + start, bytes, &full[s], pol);
          else
            tma_load_1d(stages + (size_t)s * K1_CHUNK, a.keys + start, bytes, &full[s]);
        } else {
          mbar_arrive(&full[s]);
        }
      }
    }
  } else {
    u64 i = warp;
    u32 wrun = 0;  // records in this warp's stream (filtered mode)
    for (u64 c = k1_chunk_of(i, a.c_begin, a.c_end); c != ~0ull; i += CW, c = k1_chunk_of(i, a.c_begin, a.c_end)) {
      const u32 s = (u32)(i % K1_STAGES);
      const u32 ph = (u32)(i / K1_STAGES) & 1u;
      mbar_wait(&full[s], ph);
      const u32* st = stages + (size_t)s * K1_CHUNK;
      if constexpr (DTOPK_K1_EXP == 1) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        continue;
      }
      bool released = false;
      if (((c + 1) << K1_LOG_CHUNK) <= a.n)
        released = k1_warp_chunk<MODE, B, false>(a, st, c, shist, &empty[s], filt, ft, wrun);
      else
        k1_warp_chunk_tail<MODE, B>(a, st, c, shist, filt, ft, wrun);
      if (!released) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
      }
    }
  }
  __syncthreads();
  if (a.do_hist) {
    for (int i = tid; i < NBD1; i += k1_threads<B>()) {
      u32 v = 0;
#pragma unroll
      for (int h = 0; h < K1_HCOPIES; h++) v += shist[h * NBD1 + i];
      if (v) atomicAdd(&a.hist1[i], (ull)v);
    }
  }
}

// K0: sample for the filtered delegate pass.  1/K0_GROUP of the K1 chunks
// (2048 keys), as K0_REGIONS runs of consecutive chunks at hashed offsets (one
// run per 1/K0_REGIONS of the input: a few hundred TLB entries instead of one
// per sampled chunk, which made a scattered sample latency-bound), each chunk
// read by one warp with coalesced 16-byte loads (uint4 j*32 + lane, all 16 in flight), its
// subranges (alpha 6..8) are reduced to their top-B delegates with shuffles and
// histogrammed on the first radix digit; the last CTA picks the floor of the
// bucket holding sample rank r_s ~ (1.25 k + 64) * f (+4 sigma), f = sampled
// share of D.  With probability ~1 that floor lies at or below theta's bucket
// floor (K2 verifies it exactly and falls back to the full pass otherwise), so
// K1 need only store subranges whose max delegate reaches it.  The filter
// stays off when the chosen buckets hold more than a quarter of the sample
// (tie-heavy / narrow-range input: the floor would keep most subranges).
// Reads 1/K0_GROUP of the input.
#ifndef DTOPK_K0_R
#define DTOPK_K0_R 1.25  // sample rank of the floor, in units of k (theta is at rank k of D)
#endif
constexpr int K0_GROUP = 512;
constexpr int K0_REGIONS = 64;
__host__ __device__ __forceinline__ u64 k0_run(u64 nch_full) {
  const u64 L = nch_full / (K0_REGIONS * K0_GROUP);
  return L ? L : 1;
}

// top-2 (or top-1) merge of two ladders
template <int B>
__device__ __forceinline__ void k0_merge(u32& a0, u32& a1, u32 b0, u32 b1) {
  if (B >= 2) a1 = max(min(a0, b0), max(a1, b1));
  a0 = max(a0, b0);
}

template <int MODE, int B>
__global__ void __launch_bounds__(256) k0_sample(const u32* __restrict__ keys, int alpha, u64 S, u64 k, u64 nD,
                                                 Ctrl* ctrl, u64 nch_full) {
  __shared__ u32 sh[NBD1];
  __shared__ ull scratch[8];
  __shared__ DigitResult res;
  __shared__ int am_last;
  const int tid = threadIdx.x, lane = tid & 31;
  for (int i = tid; i < NBD1; i += 256) sh[i] = 0;
  __syncthreads();
  // K0_REGIONS runs of L consecutive chunks, one per 1/K0_REGIONS of the input at
  // a hashed offset: few pages (TLB entries) touched, 1/K0_GROUP of the chunks
  const u64 slot = nch_full / K0_REGIONS, L = k0_run(nch_full);
  const u64 ng = K0_REGIONS * L;
  const u64 gw = ((u64)blockIdx.x * 256 + tid) >> 5, nw = ((u64)gridDim.x * 256) >> 5;
  for (u64 g = gw; g < ng; g += nw) {
    const u64 r = g / L;
    const u64 c = r * slot + (((u32)r * 0x9E3779B1u) >> 16) % (slot - L + 1) + g % L;
    const uint4* p = reinterpret_cast<const uint4*>(keys + (c << K1_LOG_CHUNK));
    uint4 v[16];
#pragma unroll
    for (int j = 0; j < 16; j++) v[j] = ld_nc_v4(p + j * 32 + lane);
    u32 t0[16], t1[16];  // this lane's top-B of uint4 j*32 + lane
#pragma unroll
    for (int j = 0; j < 16; j++) {
      const u32 x[4] = {to_key<MODE>(v[j].x), to_key<MODE>(v[j].y), to_key<MODE>(v[j].z), to_key<MODE>(v[j].w)};
      const u32 h1 = max(x[0], x[1]), l1 = min(x[0], x[1]), h2 = max(x[2], x[3]), l2 = min(x[2], x[3]);
      t0[j] = max(h1, h2);
      t1[j] = max(min(h1, h2), max(l1, l2));
    }
    // alpha 6: 16 lanes per subrange and instruction; 7: 32; 8: 32 lanes x 2 instructions
    const int G = alpha == 6 ? 16 : 32;
    const int per = alpha >= 8 ? 2 : 1;
#pragma unroll
    for (int j = 0; j < 16; j += 2) {
      u32 a0 = t0[j], a1 = t1[j], b0 = t0[j + 1], b1 = t1[j + 1];
      if (per == 2) {
        k0_merge<B>(a0, a1, b0, b1);
      }
      for (int o = 1; o < G; o <<= 1) {
        k0_merge<B>(a0, a1, __shfl_xor_sync(FULL, a0, o), __shfl_xor_sync(FULL, a1, o));
        if (per == 1) k0_merge<B>(b0, b1, __shfl_xor_sync(FULL, b0, o), __shfl_xor_sync(FULL, b1, o));
      }
      if ((lane & (G - 1)) == 0) {
        atomicAdd(&sh[ddig(a0, MODE >= 2)], 1u);
        if (B >= 2) atomicAdd(&sh[ddig(a1, MODE >= 2)], 1u);
        if (per == 1) {
          atomicAdd(&sh[ddig(b0, MODE >= 2)], 1u);
          if (B >= 2) atomicAdd(&sh[ddig(b1, MODE >= 2)], 1u);
        }
      }
    }
  }
  __syncthreads();
  for (int i = tid; i < NBD1; i += 256)
    if (sh[i]) atomicAdd(&ctrl->samp_hist[i], (ull)sh[i]);
  __threadfence();
  __syncthreads();
  if (tid == 0) am_last = atomicAdd(&ctrl->samp_done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  const ull ns = K0_REGIONS * k0_run(nch_full) * (2048ull >> alpha) * (u64)B;  // sampled delegates
  const double f = (double)ns / (double)nD;
  const double R = (double)k * DTOPK_K0_R + 64.0;
  const ull rs = (ull)ceil(R * f + 4.0 * sqrt(R * f) + 8.0);
  find_digit<NBD1>(ctrl->samp_hist, rs, &res, scratch);
  if (tid == 0) {
    const bool on = ns > 0 && rs <= ns && res.valid && (res.above + res.cnt) * 4 <= ns;
    u32 kmin, kmax;
    dbucket(res.digit, MODE >= 2, kmin, kmax);
    ctrl->filt_t = kmin;
    ctrl->filt_on = on ? 1u : 0u;
    ctrl->res.filtered = on ? 1u : 0u;
  }
}

// Merge per-chunk partial ladders into per-subrange delegates (alpha > 13).
template <int B>
__global__ void __launch_bounds__(256) k1_merge(const u32* __restrict__ partial, const u32* __restrict__ pmeta,
                                                u64 nch, int alpha, u64 S, u32* __restrict__ D,
                                                u32* __restrict__ meta, ull* __restrict__ hist1, int lin) {
  pdl_trigger();
  __shared__ u32 shist[NBD1];
  for (int i = threadIdx.x; i < NBD1; i += 256) shist[i] = 0;
  __syncthreads();
  const u64 cps = 1ull << (alpha - K1_LOG_CHUNK);
  const u64 stride = (u64)gridDim.x * 256;
  const u64 s_end = (S + 31) & ~31ull;  // keep whole warps in the loop for hist_add_agg
  for (u64 s = (u64)blockIdx.x * 256 + threadIdx.x; s < s_end; s += stride) {
    Acc<B> A;
    A.init(0);
    if (s < S) {
      const u64 c_end = min(nch, (s + 1) * cps);
      for (u64 c = s * cps; c < c_end; c++) {
        u32 R[B];
#pragma unroll
        for (int i = 0; i < B; i++) R[i] = partial[c * B + i];
        acc_merge<B>(A, R, pmeta[2 * c], pmeta[2 * c + 1]);
      }
      store_delegates<B>(D, s, A.L);
      meta[s] = pack_meta(A.mn == A.L[0], A.p);
    }
    u32 L[B];
#pragma unroll
    for (int i = 0; i < B; i++) L[i] = A.L[i];
#pragma unroll
    for (int i = 0; i < B; i++) hist_add_agg(shist, ddig(L[i], lin), s < S);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < NBD1; i += 256) {
    const u32 v = shist[i];
    if (v) atomicAdd(&hist1[i], (ull)v);
  }
}

// Generic top-beta for 8 < beta <= 32: one warp per subrange, per-lane
// insertion ladders (the reference's _rows_ladder, delegate.py:93-107), then a
// beta-round warp arg-max merge.  Cold path: correctness over speed.
template <int MODE>
__global__ void __launch_bounds__(256) k1_generic(const u32* __restrict__ keys, u64 n, int alpha, int beta,
                                                  u64 S, u32* __restrict__ D, u32* __restrict__ meta,
                                                  ull* __restrict__ hist1) {
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const u64 gw = ((u64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const u64 nw = ((u64)gridDim.x * blockDim.x) >> 5;
  const u64 W = 1ull << alpha;
  for (u64 s = gw; s < S; s += nw) {
    u32 L[32];
    for (int i = 0; i < 32; i++) L[i] = 0;
    for (u64 e = lane; e < W; e += 32) {
      const u64 i = s * W + e;
      const u32 x = i < n ? to_key<MODE>(keys[i]) : 0u;
      if (x <= L[beta - 1]) continue;
      int p = beta - 1;
      while (p > 0 && x > L[p - 1]) {
        L[p] = L[p - 1];
        p--;
      }
      L[p] = x;
    }
    int ptr = 0;
    u32 d1 = 0;
    for (int r = 0; r < beta; r++) {
      const u32 head = ptr < beta ? L[ptr] : 0u;
      const u32 m = __reduce_max_sync(FULL, head);
      const u32 win = __ballot_sync(FULL, head == m);
      if (lane == __ffs(win) - 1) ptr++;
      if (r == 0) d1 = m;
      if (lane == 0) {
        D[s * beta + r] = m;
        atomicAdd(&hist1[ddig(m, MODE >= 2)], 1ull);
      }
    }
    // position of the first max and constant-subrange flag: second pass (cold path)
    u32 pos = 0xffffffffu, mn = 0xffffffffu;
    for (u64 e = lane; e < W; e += 32) {
      const u64 i = s * W + e;
      if (i < n) {
        const u32 x = to_key<MODE>(keys[i]);
        mn = min(mn, x);
        if (x == d1) pos = min(pos, (u32)e);
      }
    }
    pos = __reduce_min_sync(FULL, pos);
    mn = __reduce_min_sync(FULL, mn);
    if (lane == 0) meta[s] = pack_meta(mn == d1, pos);
  }
}

}  // namespace dtopk
