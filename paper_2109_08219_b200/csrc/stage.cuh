// stage.cuh -- the reference's stage operators as standalone device entries
// (dtopk_qualify, dtopk_concat, dtopk_min_at_least) and the large-beta
// delegate kernel.  These serve the stage-level API (pipeline.first_topk,
// pipeline.concatenate_filtered) and its parity tests; the fused pipeline
// (K1..K6) does the same work without materialising these vectors.
//
//   first_topk qualification   pipeline.py:87-116
//   concatenate_filtered       pipeline.py:119-159
//   relaxed theta (skip_last)  kernels.py:161-164: min{ d : d >= kth & ~0xff }
//   _rows_ladder, any beta     delegate.py:93-107, 120-127
//
// Ordered compaction is three kernels: per-tile counts, one exclusive scan of
// the tile counts (single CTA), and a re-evaluating emit that writes each
// element at its tile offset plus its rank inside the tile.
#pragma once

#include <cub/block/block_radix_sort.cuh>

#include "common.cuh"

namespace dtopk {

constexpr int STG_THREADS = 256;
constexpr int STG_PER = 16;
constexpr int STG_TILE = STG_THREADS * STG_PER;  // elements per tile
constexpr int STG_STREAMS = 3;                   // qualify: selected, partial, fully qualified

// Exclusive rank of this thread's count inside the CTA, plus the CTA total.
__device__ __forceinline__ u32 stg_block_excl(u32 v, u32* scratch, u32& total) {
  const u32 incl = block_incl_scan_256<u32>(v, scratch);
  __shared__ u32 s_tot;
  if (threadIdx.x == 255) s_tot = incl;
  __syncthreads();
  total = s_tot;
  return incl - v;
}

// ---------------------------------------------------------------- qualify
// Element i of D (key space, subrange-major, beta per subrange):
//   selected  d_i >= theta                      (values + tags, D order)
//   partial   selected and d_beta(s) < theta    (values + tags)
//   fully q.  d_beta(s) >= theta, once per s    (subrange ids, ascending)
__device__ __forceinline__ void qual_flags(const u32* __restrict__ D, u64 nD, int beta, u32 theta, u64 i, bool& sel,
                                           bool& part, bool& fq) {
  sel = part = fq = false;
  if (i >= nD) return;
  const u64 s = i / (u64)beta;
  const bool full = D[s * beta + beta - 1] >= theta;
  sel = D[i] >= theta;
  part = sel && !full;
  fq = full && (i == s * beta);
}

__global__ void __launch_bounds__(STG_THREADS) qual_count(const u32* __restrict__ D, u64 nD, int beta, u32 theta,
                                                          u32* __restrict__ tile_cnt) {
  __shared__ u32 scratch[8];
  const u64 base = (u64)blockIdx.x * STG_TILE + (u64)threadIdx.x * STG_PER;
  u32 c[STG_STREAMS] = {0, 0, 0};
  for (int j = 0; j < STG_PER; j++) {
    bool s, p, f;
    qual_flags(D, nD, beta, theta, base + j, s, p, f);
    c[0] += s;
    c[1] += p;
    c[2] += f;
  }
  for (int q = 0; q < STG_STREAMS; q++) {
    u32 tot;
    stg_block_excl(c[q], scratch, tot);
    if (threadIdx.x == 0) tile_cnt[(u64)blockIdx.x * STG_STREAMS + q] = tot;
    __syncthreads();
  }
}

// Exclusive scan of `ntiles` x `nstreams` counts (in place, per stream) by one
// CTA; totals to out_total[nstreams] (int64).
__global__ void __launch_bounds__(STG_THREADS) stg_scan(u32* __restrict__ tile_cnt, u64 ntiles, int nstreams,
                                                        int64_t* __restrict__ out_total) {
  __shared__ ull scratch[8];
  for (int q = 0; q < nstreams; q++) {
    const u64 per = (ntiles + STG_THREADS - 1) / STG_THREADS;
    const u64 t0 = (u64)threadIdx.x * per, t1 = min(ntiles, t0 + per);
    ull sum = 0;
    for (u64 t = t0; t < t1; t++) sum += tile_cnt[t * nstreams + q];
    const ull incl = block_incl_scan_256<ull>(sum, scratch);
    ull run = incl - sum;
    for (u64 t = t0; t < t1; t++) {
      const u32 c = tile_cnt[t * nstreams + q];
      tile_cnt[t * nstreams + q] = (u32)run;  // offsets fit: outputs are < 2^32 elements per stream here
      run += c;
    }
    if (threadIdx.x == STG_THREADS - 1) out_total[q] = (int64_t)incl;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(STG_THREADS) qual_emit(const u32* __restrict__ D, u64 nD, int beta, u32 theta,
                                                         const u32* __restrict__ tile_off, u32* __restrict__ sel_val,
                                                         u32* __restrict__ sel_tag, u32* __restrict__ part_val,
                                                         u32* __restrict__ part_tag, u32* __restrict__ fq_sid) {
  __shared__ u32 scratch[8];
  const u64 base = (u64)blockIdx.x * STG_TILE + (u64)threadIdx.x * STG_PER;
  u32 c[STG_STREAMS] = {0, 0, 0};
  for (int j = 0; j < STG_PER; j++) {
    bool s, p, f;
    qual_flags(D, nD, beta, theta, base + j, s, p, f);
    c[0] += s;
    c[1] += p;
    c[2] += f;
  }
  u32 o[STG_STREAMS];
  for (int q = 0; q < STG_STREAMS; q++) {
    u32 tot;
    o[q] = tile_off[(u64)blockIdx.x * STG_STREAMS + q] + stg_block_excl(c[q], scratch, tot);
    __syncthreads();
  }
  for (int j = 0; j < STG_PER; j++) {
    const u64 i = base + j;
    bool s, p, f;
    qual_flags(D, nD, beta, theta, i, s, p, f);
    const u32 tag = (u32)(i / (u64)beta);
    if (s) {
      sel_val[o[0]] = D[i];
      sel_tag[o[0]++] = tag;
    }
    if (p) {
      part_val[o[1]] = D[i];
      part_tag[o[1]++] = tag;
    }
    if (f) fq_sid[o[2]++] = tag;
  }
}

// ---------------------------------------------------------------- concat
// Virtual element j of the fully qualified subranges (subrange-ascending, scan
// order): subrange fq[j >> alpha], offset j & (W-1); kept when its key >= theta.
template <int MODE>
__device__ __forceinline__ bool concat_elem(const u32* __restrict__ raw, u64 n, int alpha,
                                            const u32* __restrict__ fq, u64 nv, u32 theta, u64 j, u32& bits) {
  if (j >= nv) return false;
  const u64 pos = ((u64)fq[j >> alpha] << alpha) | (j & ((1ull << alpha) - 1));
  if (pos >= n) return false;
  bits = raw[pos];
  return to_key<MODE>(bits) >= theta;
}

template <int MODE>
__global__ void __launch_bounds__(STG_THREADS) concat_count(const u32* __restrict__ raw, u64 n, int alpha,
                                                            const u32* __restrict__ fq, u64 nv, u32 theta,
                                                            u32* __restrict__ tile_cnt) {
  __shared__ u32 scratch[8];
  const u64 base = (u64)blockIdx.x * STG_TILE + (u64)threadIdx.x * STG_PER;
  u32 c = 0, b;
  for (int j = 0; j < STG_PER; j++) c += concat_elem<MODE>(raw, n, alpha, fq, nv, theta, base + j, b);
  u32 tot;
  stg_block_excl(c, scratch, tot);
  if (threadIdx.x == 0) tile_cnt[blockIdx.x] = tot;
}

template <int MODE>
__global__ void __launch_bounds__(STG_THREADS) concat_emit(const u32* __restrict__ raw, u64 n, int alpha,
                                                           const u32* __restrict__ fq, u64 nv, u32 theta,
                                                           const u32* __restrict__ tile_off, u32* __restrict__ out) {
  __shared__ u32 scratch[8];
  const u64 base = (u64)blockIdx.x * STG_TILE + (u64)threadIdx.x * STG_PER;
  u32 c = 0, b;
  for (int j = 0; j < STG_PER; j++) c += concat_elem<MODE>(raw, n, alpha, fq, nv, theta, base + j, b);
  u32 tot;
  u32 o = tile_off[blockIdx.x] + stg_block_excl(c, scratch, tot);
  for (int j = 0; j < STG_PER; j++)
    if (concat_elem<MODE>(raw, n, alpha, fq, nv, theta, base + j, b)) out[o++] = b;
}

// ---------------------------------------------------------------- min >= edge
__global__ void __launch_bounds__(STG_THREADS) min_at_least(const u32* __restrict__ keys, u64 n, u32 edge,
                                                            u32* __restrict__ out) {
  u32 m = 0xffffffffu;
  bool any = false;
  for (u64 i = (u64)blockIdx.x * STG_THREADS + threadIdx.x; i < n; i += (u64)gridDim.x * STG_THREADS) {
    const u32 x = keys[i];
    if (x >= edge) {
      m = min(m, x);
      any = true;
    }
  }
  m = __reduce_min_sync(FULL, m);
  any = __any_sync(FULL, any);
  if ((threadIdx.x & 31) == 0 && any) atomicMin(out, m);
}

// ---------------------------------------------------------------- beta > 32
// One CTA per subrange (W <= K1B_MAXW): the subrange's keys are sorted
// descending in shared memory (CUB block radix sort of ~key) and the first
// beta are its delegates; meta from the sorted pairs (position of the first
// occurrence of the max, constant flag).  _rows_ladder's result for any beta.
constexpr int K1B_THREADS = 256, K1B_ITEMS = 32, K1B_MAXW = K1B_THREADS * K1B_ITEMS;  // 8192 keys

template <int MODE>
__global__ void __launch_bounds__(K1B_THREADS) k1_bigbeta(const u32* __restrict__ keys, u64 n, int alpha, int beta,
                                                          u64 S, u32* __restrict__ D, u32* __restrict__ meta,
                                                          ull* __restrict__ hist1) {
  typedef cub::BlockRadixSort<u32, K1B_THREADS, K1B_ITEMS, u32> Sorter;
  __shared__ typename Sorter::TempStorage tmp;
  __shared__ u32 s_first, s_min;
  const u64 W = 1ull << alpha;
  for (u64 s = blockIdx.x; s < S; s += gridDim.x) {
    u32 k[K1B_ITEMS], p[K1B_ITEMS];
    u32 mn = 0xffffffffu;
#pragma unroll
    for (int j = 0; j < K1B_ITEMS; j++) {
      const u64 e = (u64)threadIdx.x * K1B_ITEMS + j;  // blocked arrangement
      const u64 i = s * W + e;
      const bool in = e < W && i < n;
      const bool pad = e < W && i >= n;  // zero-padded tail (delegate.py:132-139)
      const u32 key = in ? to_key<MODE>(keys[i]) : 0u;
      if (in) mn = min(mn, key);
      // sort by ~key ascending (= key descending); absent slots (e >= W) sort last
      k[j] = (in || pad) ? ~key : 0xffffffffu;
      p[j] = (u32)e;
      if (!(in || pad)) p[j] = 0xffffffffu;
    }
    if (threadIdx.x == 0) {
      s_first = 0xffffffffu;
      s_min = 0xffffffffu;
    }
    __syncthreads();
    mn = __reduce_min_sync(FULL, mn);
    if ((threadIdx.x & 31) == 0) atomicMin(&s_min, mn);
    Sorter(tmp).Sort(k, p);  // stable: equal keys keep position order
#pragma unroll
    for (int j = 0; j < K1B_ITEMS; j++) {
      const u32 r = threadIdx.x * K1B_ITEMS + j;  // rank after the sort (blocked)
      if (r < (u32)beta) {
        const u32 key = ~k[j];
        D[s * beta + r] = key;
        atomicAdd(&hist1[ddig(key, MODE >= 2)], 1ull);
        if (r == 0) s_first = p[j];
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      // constant subrange: every present key equals d_1 (padding is not a key, as in K1)
      const u32 d1 = D[s * beta];
      meta[s] = ((s_min == d1) ? 0x80000000u : 0u) | (s_first & 0x7fffffffu);
    }
    __syncthreads();
  }
}

}  // namespace dtopk
