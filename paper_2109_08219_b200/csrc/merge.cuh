// merge.cuh -- device side of the multi-GPU candidate merge (ShardedTopK).
//
// Reference: the coordinator's final top-k over the gathered worker lists
// (distributed.py:191-251).  Here every rank holds a list of
// (value bits, global index) pairs ordered (key desc, index asc); ranks own
// contiguous shards in rank order, so for two lists A (lower ranks) and B
// (higher ranks) every index of A is below every index of B and the merged
// order on equal keys is "A first".  The exact global top-k is therefore a
// merge, not a selection: a tree of pairwise merge-path rounds, each keeping
// the first `cap` outputs of every pair (merge_round).
//
// merge="select" first decides how many pairs each rank contributes (a
// distributed radix select over the candidates' keys, three histogram
// all-reduces of 11/11/10-bit digits: dsel_hist / dsel_digit), then every rank
// writes its contribution into its own slots of a zeroed k-slot buffer
// (dsel_place) that one all-reduce(SUM) assembles; the rank segments are then
// merged by the same rounds.
//
// Nothing here synchronises the host: list lengths, offsets and the select
// state live in device memory, so the whole sharded step can be captured in
// one CUDA graph together with the NCCL collectives between the kernels.
#pragma once

#include "common.cuh"

namespace dtopk {

constexpr int MG_THREADS = 256;
constexpr int MG_PER = 8;
constexpr int MG_TILE = MG_THREADS * MG_PER;  // outputs per CTA

// Value bits of list element i (values are u32 bits; `vstride` 2 reads the low
// word of an int64 slot array, the all-reduce-assembled select buffer).
__device__ __forceinline__ u32 mg_bits(const u32* v, int vstride, long long i) { return v[i * vstride]; }

// Number of elements of A among the first d outputs of merge(A, B) (A first on
// equal keys): the smallest i with key(A[i]) < key(B[d-1-i]), found by one warp
// probing 32 candidates per step (log32 of the range dependent loads).
template <int M>
__device__ long long warp_corank(const u32* a, const u32* b, int vstride, long long la, long long lb, long long d) {
  const int lane = threadIdx.x & 31;
  long long lo = d > lb ? d - lb : 0;
  long long hi = d < la ? d : la;
  // invariant: answer in [lo, hi]
  while (hi - lo > 0) {
    const long long span = hi - lo;
    const long long step = (span + 31) / 32;
    const long long i = lo + (long long)lane * step;  // probe A[i] vs B[d-1-i]
    bool after = true;                                 // A[i] comes after B[d-1-i] (i beyond the answer)
    if (i < hi) {
      const u32 ka = to_key<M>(mg_bits(a, vstride, i));
      const u32 kb = to_key<M>(mg_bits(b, vstride, d - 1 - i));
      after = ka < kb;
    }
    const unsigned m = __ballot_sync(FULL, after);
    // first lane whose probe is "after": answer in (probe_{l-1}, probe_l]
    const int l = m ? __ffs(m) - 1 : 32;
    const long long nlo = l == 0 ? lo : lo + (long long)(l - 1) * step + 1;
    long long nhi = l >= 32 ? hi : lo + (long long)l * step;
    if (nhi > hi) nhi = hi;
    lo = nlo;
    hi = nhi;
    if (step == 1) break;
  }
  return lo;
}

struct MergeArgs {
  const u32* in_val;          // value bits of the input lists
  int vmul;                   // u32 words per unit of list offset (2: offsets count int64 words)
  int vstride;                // u32 words between consecutive values: 1 (u32 array) or 2 (int64 slots)
  const long long* in_idx;    // global indices
  const long long* in_off;    // element offset of list j (null: j * in_stride)
  long long in_stride;
  const long long* in_len;    // valid length of list j at in_len[j * len_stride] (device)
  long long len_stride;
  int n_lists;
  long long cap;              // outputs kept per pair (k)
  u32* out_val;
  long long* out_idx;
  long long out_stride;       // output list j starts at j * out_stride
  long long* out_len;         // written: min(cap, len_a + len_b) per pair
};

// One merge round: pair j = blockIdx.y merges lists 2j and 2j+1 (an odd last
// list is copied), tile blockIdx.x of MG_TILE outputs.  A and B tiles are staged
// as keys in shared memory; each thread merges MG_PER consecutive outputs.
template <int M>
__global__ void __launch_bounds__(MG_THREADS) merge_round(MergeArgs a) {
  __shared__ u32 ska[MG_TILE], skb[MG_TILE];
  __shared__ long long s_a0, s_a1;
  pdl_wait();
  const int j = blockIdx.y;
  const int ia = 2 * j, ib = 2 * j + 1;
  const long long lia = a.in_len[ia * a.len_stride];
  const long long lib = ib < a.n_lists ? a.in_len[ib * a.len_stride] : 0;
  const long long la = lia < a.cap ? lia : a.cap;
  const long long lb = lib < a.cap ? lib : a.cap;
  const long long m = la + lb < a.cap ? la + lb : a.cap;
  if (blockIdx.x == 0 && threadIdx.x == 0) a.out_len[j] = m;
  const long long d0 = (long long)blockIdx.x * MG_TILE;
  if (d0 >= m) return;
  const long long d1 = d0 + MG_TILE < m ? d0 + MG_TILE : m;
  const long long offa = a.in_off ? a.in_off[ia] : (long long)ia * a.in_stride;
  const long long offb = ib < a.n_lists ? (a.in_off ? a.in_off[ib] : (long long)ib * a.in_stride) : 0;
  const u32* va = a.in_val + offa * a.vmul;
  const u32* vb = a.in_val + offb * a.vmul;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    const long long c = warp_corank<M>(va, vb, a.vstride, la, lb, d0);
    if ((threadIdx.x & 31) == 0) s_a0 = c;
  } else if (warp == 1) {
    const long long c = warp_corank<M>(va, vb, a.vstride, la, lb, d1);
    if ((threadIdx.x & 31) == 0) s_a1 = c;
  }
  __syncthreads();
  const long long a0 = s_a0, a1 = s_a1;
  const long long b0 = d0 - a0, b1 = d1 - a1;
  const int na = (int)(a1 - a0), nb = (int)(b1 - b0);
  for (int t = threadIdx.x; t < na; t += MG_THREADS) ska[t] = to_key<M>(mg_bits(va, a.vstride, a0 + t));
  for (int t = threadIdx.x; t < nb; t += MG_THREADS) skb[t] = to_key<M>(mg_bits(vb, a.vstride, b0 + t));
  __syncthreads();
  // per-thread co-rank inside the tile (binary search over shared memory)
  const int dd = threadIdx.x * MG_PER;
  const int nt = (int)(d1 - d0);
  if (dd >= nt) return;
  int lo = dd > nb ? dd - nb : 0, hi = dd < na ? dd : na;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (ska[mid] >= skb[dd - 1 - mid])
      lo = mid + 1;
    else
      hi = mid;
  }
  int x = lo, y = dd - lo;
  const long long* ia_idx = a.in_idx + offa;
  const long long* ib_idx = a.in_idx + offb;
  u32* ov = a.out_val + (long long)j * a.out_stride + d0;
  long long* oi = a.out_idx + (long long)j * a.out_stride + d0;
#pragma unroll
  for (int q = 0; q < MG_PER; q++) {
    const int o = dd + q;
    if (o >= nt) break;
    const bool take_a = x < na && (y >= nb || ska[x] >= skb[y]);
    if (take_a) {
      ov[o] = from_key<M>(ska[x]);
      oi[o] = ia_idx[a0 + x];
      x++;
    } else {
      ov[o] = from_key<M>(skb[y]);
      oi[o] = ib_idx[b0 + y];
      y++;
    }
  }
}

// ---------------------------------------------------------------------------
// Distributed radix select over the per-rank candidate lists.
// state[0] = prefix of the kth key so far, state[1] = rank still sought
// (1-based) under that prefix; initialised by dsel_init.
// ---------------------------------------------------------------------------
constexpr int DSEL_BINS = 2048;

__device__ __forceinline__ void dsel_digit_of(int pass, int& shift, int& nb) {
  shift = pass == 0 ? 21 : (pass == 1 ? 10 : 0);
  nb = pass == 2 ? 10 : 11;
}

__global__ void dsel_init(long long* state, long long* hist, long long k) {
  pdl_wait();
  for (int t = threadIdx.x; t < DSEL_BINS; t += blockDim.x) hist[t] = 0;
  if (threadIdx.x == 0) {
    state[0] = 0;
    state[1] = k;
  }
}

// Histogram of the digit `pass` of the valid candidates (first *cnt of `bits`,
// ordered key desc) under the current prefix.  The list is sorted, so equal
// digits come in runs: a thread walks 16 consecutive keys and adds one count per
// run to a shared histogram, flushed once per CTA.
template <int M>
__global__ void __launch_bounds__(256) dsel_hist(const u32* bits, const long long* cnt, const long long* state,
                                                 int pass, long long* hist) {
  __shared__ u32 sh[DSEL_BINS];
  pdl_wait();
  for (int t = threadIdx.x; t < DSEL_BINS; t += blockDim.x) sh[t] = 0;
  __syncthreads();
  int shift, nb;
  dsel_digit_of(pass, shift, nb);
  const long long n = *cnt;
  const u32 prefix = (u32)state[0];
  const int hsh = shift + nb;
  for (long long base = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * 16; base < n;
       base += (long long)gridDim.x * blockDim.x * 16) {
    const long long e = base + 16 < n ? base + 16 : n;
    u32 run_d = 0xffffffffu, run_c = 0;
    for (long long i = base; i < e; i++) {
      const u32 key = to_key<M>(bits[i]);
      if (hsh < 32 && (key >> hsh) != prefix) continue;
      const u32 d = (key >> shift) & ((1u << nb) - 1u);
      if (d != run_d) {
        if (run_c) atomicAdd(&sh[run_d], run_c);
        run_d = d;
        run_c = 0;
      }
      run_c++;
    }
    if (run_c) atomicAdd(&sh[run_d], run_c);
  }
  __syncthreads();
  for (int t = threadIdx.x; t < DSEL_BINS; t += blockDim.x)
    if (sh[t]) atomicAdd(reinterpret_cast<ull*>(&hist[t]), (ull)sh[t]);
}

// After the all-reduce of `hist`: choose the digit holding the sought rank,
// update (prefix, rem), zero the histogram for the next pass.  After the last
// pass (kth key known) count this rank's candidates above / equal to kth into
// gt_eq[0..1] (binary searches over the sorted list), the input of the
// all_gather that decides every rank's contribution.
template <int M>
__global__ void __launch_bounds__(1024) dsel_digit(long long* state, long long* hist, int pass, const u32* bits,
                                                   const long long* cnt, long long* gt_eq) {
  __shared__ long long s_warp[32];
  __shared__ long long s_rem;
  __shared__ int s_d;
  pdl_wait();
  int shift, nb;
  dsel_digit_of(pass, shift, nb);
  const int bins = 1 << nb;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long rem = state[1];
  // suffix sums over the digits = prefix sums over r = bins-1-d; thread t owns r = 2t, 2t+1
  const int r0 = 2 * tid;
  const long long c0 = r0 < bins ? hist[bins - 1 - r0] : 0;
  const long long c1 = r0 + 1 < bins ? hist[bins - 2 - r0] : 0;
  long long x = c0 + c1;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long y = __shfl_up_sync(FULL, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    long long w = s_warp[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(FULL, w, o);
      if (lane >= o) w += y;
    }
    s_warp[lane] = w;
  }
  __syncthreads();
  const long long before = (warp ? s_warp[warp - 1] : 0) + x - c0 - c1;  // at_least of digit bins-1-r0+1
  // the digit holding the sought rank: first r with prefix(r) >= rem
  if (r0 < bins && before < rem && before + c0 >= rem) {
    s_d = bins - 1 - r0;
    s_rem = rem - before;
  } else if (r0 + 1 < bins && before + c0 < rem && before + c0 + c1 >= rem) {
    s_d = bins - 2 - r0;
    s_rem = rem - before - c0;
  }
  __syncthreads();
  for (int t = tid; t < DSEL_BINS; t += blockDim.x) hist[t] = 0;
  if (tid == 0) {
    state[0] = (state[0] << nb) | s_d;
    state[1] = s_rem;
  }
  if (pass != 2) return;
  __syncthreads();
  if (tid >= 32) return;
  const u32 kth = (u32)((state[0]));
  const long long n = *cnt;
  // first position with key < x in a list sorted by key desc, for x = kth + 1 (gt) and kth (ge)
  long long pos[2];
  for (int w = 0; w < 2; w++) {
    const unsigned long long xx = (unsigned long long)kth + (w == 0 ? 1ull : 0ull);
    long long lo = 0, hi = n;
    while (hi > lo) {
      const long long span = hi - lo;
      const long long step = (span + 31) / 32;
      const long long i = lo + (long long)tid * step;
      const bool below = i < hi ? (unsigned long long)to_key<M>(bits[i]) < xx : true;
      const unsigned mm = __ballot_sync(FULL, below);
      const int l = mm ? __ffs(mm) - 1 : 32;
      const long long nlo = l == 0 ? lo : lo + (long long)(l - 1) * step + 1;
      long long nhi = l >= 32 ? hi : lo + (long long)l * step;
      if (nhi > hi) nhi = hi;
      lo = nlo;
      hi = nhi;
      if (step == 1) break;
    }
    pos[w] = lo;
  }
  if (tid == 0) {
    gt_eq[0] = pos[0];
    gt_eq[1] = pos[1] - pos[0];
  }
}

// After the all_gather of every rank's (gt, eq): this rank contributes its first
// gt_r + take_r pairs (ties granted in rank = index order) at offset pre_r of
// the k-slot answer.  Writes the rank's pairs into its slots and zero into all
// others (the all-reduce(SUM) then assembles the answer), plus the segment
// table (offset, length per rank) the merge rounds read.
__global__ void __launch_bounds__(256) dsel_place(const long long* g, const long long* state, int rank, int world,
                                                  long long k, const u32* bits, const long long* idx,
                                                  long long* slots, long long* seg_off, long long* seg_len) {
  __shared__ long long s_pre, s_mine;
  pdl_wait();
  if (threadIdx.x == 0) {
    long long rem = state[1];  // ties still needed at the kth key
    long long pre = 0, eq_before = 0;
    for (int r = 0; r < world; r++) {
      long long take = rem - eq_before;
      if (take < 0) take = 0;
      if (take > g[2 * r + 1]) take = g[2 * r + 1];
      const long long contrib = g[2 * r] + take;
      if (blockIdx.x == 0) {
        seg_off[r] = pre;
        seg_len[r] = contrib;
      }
      if (r == rank) {
        s_pre = pre;
        s_mine = contrib;
      }
      pre += contrib;
      eq_before += g[2 * r + 1];
    }
  }
  __syncthreads();
  const long long pre = s_pre, mine = s_mine;
  for (long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x; s < k; s += (long long)gridDim.x * blockDim.x) {
    const long long o = s - pre;
    const bool own = o >= 0 && o < mine;
    slots[s] = own ? (long long)bits[o] : 0;
    slots[k + s] = own ? idx[o] : 0;
  }
}

}  // namespace dtopk
