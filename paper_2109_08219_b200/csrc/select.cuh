// select.cuh -- radix select (11/11/10-bit MSD digits) for the delegate
// threshold theta = kth(D) and for the exact k-th key of a candidate pool.
//
// Reference: kernels.radix_topk (kernels.py:109-165) -- an in-place MSD radix
// top-k that re-scans its input once per 8-bit digit with the predicate
// (x & mask) == bits.  Here the first pass over D is fused into K1 (delegate
// histogram), the second pass compacts the bucket that holds the k-th key
// into a small buffer, and the third pass runs on that buffer only, so D is
// read exactly once after it is written.  The threshold is always the exact
// kth(D): the reference's skip_last relaxation (kernels.py:161-164) only saves
// a pass on the CPU, while on tie-heavy inputs it can lower theta to min(D)
// and multiply the concatenation work.
#pragma once

#include "common.cuh"

#ifndef DTOPK_K1_CONTIG
#define DTOPK_K1_CONTIG 0
#endif

namespace dtopk {

constexpr int K1_LOG_CHUNK_ = 11;
#ifndef DTOPK_K2R_U
#define DTOPK_K2R_U 4
#endif
constexpr int K2R_U = DTOPK_K2R_U;  // record loads in flight per lane (K2 over records)  // keys per K1 chunk = 2^11 (delegate.cuh K1_LOG_CHUNK)

struct K2Args {
  const u32* D;
  u64 nD;      // beta * S delegates
  u64 k;
  Ctrl* ctrl;
  u32* selbuf;  // region of CTA c: [c * R, c * R + region_cnt[c])
  u32* region_cnt;
  u64 R;        // delegates per CTA region (multiple of 512)
  // candidate superset (delegate path): subranges whose max delegate lies in
  // theta's top-11-bit bucket or above, in subrange order per warp segment
  int beta;
  uint4* sup_sid;  // [S] {sid, d_1, d_2, meta} (beta 2; else {sid, d_1, 0, meta}): segment (cta, warp) from sup_in[seg]
  u32* sup_in;   // [g2 * 8] first slot of each segment
  u32* sup_cnt;  // [g2 * 8] entries of each segment
  u32* sup_off;  // [g2 * 8 + 1] exclusive prefix of sup_cnt (theta resolver)
  const u32* meta;  // [S] K1 meta words, copied into the superset entries
  const uint2* tseg;  // [g2 * 8] (tie lower bound, entries above theta) per segment (pass 3, truncation)
  // filtered delegate pass (K1 fmode): 1 = scan K1's records when ctrl->filt_on,
  // 2 = fallback full scan, only when ctrl->filt_fail
  int fmode;
  const u32* chunk_cnt;  // [nch] (offset << 6) | count of K1 chunk c's records in its warp's stream
  const uint4* frec;     // K1 record streams: chunk c was reduced by warp (c % g1, (c / g1) % 8)
  u64 fcap;              // records per stream
  u32 g1;                // K1 grid
  u64 nch;
  int alpha;
  cudaGraphConditionalHandle fb;  // graph: set when the fallback must run
  int fb_graph;
  int lin;  // first digit family (float32: linear)
};

#ifndef DTOPK_K2_MINB
#define DTOPK_K2_MINB 3  // K2 min CTAs per SM = DTOPK_K2_CPS: all regions of an SM resident (single wave), 80 registers (4: 64, ~6 us slower)
#endif
constexpr int K2_SEG_PER = 24;  // superset segments per thread in the prefix (8 warps x <= 768 K2 CTAs)

// The superset segment counts of thread t: segments [t * K2_SEG_PER, +K2_SEG_PER),
// read as uint4 (sup_cnt is padded to 256 * K2_SEG_PER; nseg = 8 * nregions <=
// 8 * 768 = 256 * K2_SEG_PER).
__device__ __forceinline__ void k2_sup_load(const u32* __restrict__ sup_cnt, uint4 (&x)[K2_SEG_PER / 4]) {
  const uint4* c4 = reinterpret_cast<const uint4*>(sup_cnt) + threadIdx.x * (K2_SEG_PER / 4);
#pragma unroll
  for (int q = 0; q < K2_SEG_PER / 4; q++) x[q] = __ldcg(&c4[q]);
}

// Exclusive prefix of the superset segment counts (loaded by k2_sup_load) ->
// sup_off, sup_total (one CTA).
__device__ __forceinline__ void k2_superset_prefix_regs(Ctrl* ctrl, u32 nregions, const uint4 (&x)[K2_SEG_PER / 4],
                                                        u32* __restrict__ sup_off, ull* scratch) {
  const int tid = threadIdx.x;
  const u32 nseg = nregions * 8;
  u32 c[K2_SEG_PER];
  u32 sum = 0;
#pragma unroll
  for (int q = 0; q < K2_SEG_PER / 4; q++) {
    c[4 * q] = x[q].x;
    c[4 * q + 1] = x[q].y;
    c[4 * q + 2] = x[q].z;
    c[4 * q + 3] = x[q].w;
  }
#pragma unroll
  for (int q = 0; q < K2_SEG_PER; q++) {
    if ((u32)(tid * K2_SEG_PER + q) >= nseg) c[q] = 0u;
    sum += c[q];
  }
  u32* sc = reinterpret_cast<u32*>(scratch);
  const u32 incl = block_incl_scan_256<u32>(sum, sc);
  u32 run = incl - sum;
#pragma unroll
  for (int q = 0; q < K2_SEG_PER; q++) {
    const u32 i = tid * K2_SEG_PER + q;
    if (i < nseg) sup_off[i] = run;
    run += c[q];
  }
  if (tid == 255) {
    sup_off[nseg] = incl;
    ctrl->sup_total = incl;
  }
}

__device__ void k2_superset_prefix(Ctrl* ctrl, u32 nregions, const u32* __restrict__ sup_cnt,
                                   u32* __restrict__ sup_off, ull* scratch) {
  uint4 x[K2_SEG_PER / 4];
  k2_sup_load(sup_cnt, x);
  k2_superset_prefix_regs(ctrl, nregions, x, sup_off, scratch);
}

// theta = kmin + digit 2 + digit 3 from the digit-3 histogram (ctrl->selD.hist3,
// or pass 3's padded shared-memory histogram when `sh3` is set).  One CTA.
__device__ __forceinline__ void k2_theta_from_hist3(Ctrl* ctrl, u32 kmin, const DigitResult& r1,
                                                    const DigitResult& r2, DigitResult* r3, ull* scratch,
                                                    const u32* sh3) {
  if (sh3)
    find_digit_sm<NBD3, true>(sh3, r2.rem, r3, scratch);
  else
    find_digit<NBD3>(ctrl->selD.hist3, r2.rem, r3, scratch);
  if (threadIdx.x == 0) {
    const u32 kth = kmin + (r2.digit << DSH3) + r3->digit;
    ctrl->selD.r3 = *r3;
    ctrl->selD.kth = kth;
    ctrl->res.theta_local = kth;
    ctrl->res.theta_slot = (int64_t)kth;
    ctrl->res.delegate_bucket = r1.cnt;
  }
}

// Resolve theta and publish the exclusive prefix of the superset segment
// counts.  One CTA (256 threads).
__device__ void k2_resolve_theta(Ctrl* ctrl, u32 kmin, const DigitResult& r1, const DigitResult& r2, u32 nregions,
                                 const u32* __restrict__ sup_cnt, u32* __restrict__ sup_off, DigitResult* r3,
                                 ull* scratch, u64 nD, const u32* sh3 = nullptr) {
  k2_theta_from_hist3(ctrl, kmin, r1, r2, r3, scratch, sh3);
  if (sup_cnt == nullptr || r1.cnt * 4 > nD) return;  // deferred: K2b builds and offsets the superset
  k2_superset_prefix(ctrl, nregions, sup_cnt, sup_off, scratch);
}

// K2 over K1's records (filtered pass): warp w of the grid owns a contiguous
// range of K1 chunks; per 32 chunks the lanes read the (offset, count) words, a
// warp scan flattens the counts, and lane l handles records l, l+32, ... (its
// chunk by a 5-step shuffle search over the exclusive prefix).  Chunk c's
// records sit in the stream of the K1 warp that reduced it.  Superset entries
// (d_1 >= kmin) are compacted, in subrange order, into the warp's superset
// segment; bucket members (d_1, d_2 in [kmin, kmax]) feed the digit-2
// histogram and the CTA's selbuf region exactly as in the scan of D.
template <int BETA2>
__device__ __noinline__ void k2_records(const K2Args& a, u32 kmin, u32 span, u32* shist, u32* s_cnt, u32* region,
                                        u64& out0_o, u32& run_o) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const u64 nseg = (u64)gridDim.x * 8;
  const u64 seg = (u64)blockIdx.x * 8 + warp;
  const u64 cpw = (a.nch + nseg - 1) / nseg;
  const u64 c0 = min(a.nch, seg * cpw), c1 = min(a.nch, c0 + cpw);
  const int lspc = K1_LOG_CHUNK_ - a.alpha;
  const u64 out0 = c0 << lspc;
  const u32 lt = lanemask_lt();
  u32 run = 0;
  u32 word = (c0 + lane < c1) ? __ldcg(a.chunk_cnt + c0 + lane) : 0u;
  for (u64 cb = c0; cb < c1; cb += 32) {
    const u64 c = cb + lane;
    // the next 32 chunks' words are in flight while this batch is processed
    const u32 next = (c + 32 < c1) ? __ldcg(a.chunk_cnt + c + 32) : 0u;
    const u32 cnt = word & 63u;
    // start of chunk c's records: its K1 warp's stream + the offset in it
    // (K1 CTA b reduces chunks b + i g1, or [b R, (b+1) R) with DTOPK_K1_CONTIG; warp i % 8)
#if DTOPK_K1_CONTIG
    const u64 R1 = (a.nch + a.g1 - 1) / a.g1;
    const u64 kw = (c / R1) * 8 + (c % R1) % 8;
#else
    const u64 kw = (c % a.g1) * 8 + (c / a.g1) % 8;
#endif
    const u64 src = kw * a.fcap + (word >> 6);
    word = next;
    const u32 incl = warp_incl_scan<u32>(cnt);
    const u32 excl = incl - cnt;
    const u32 tot = __shfl_sync(FULL, incl, 31);
    for (u32 r0 = 0; r0 < tot; r0 += 32 * K2R_U) {
      // up to K2R_U x 32 record loads in flight before any is used
      uint4 e[K2R_U];
#pragma unroll
      for (int u = 0; u < K2R_U; u++) {
        const u32 r = r0 + u * 32 + lane;
        int j = 0;
#pragma unroll
        for (int st = 16; st; st >>= 1) {
          const u32 ex = __shfl_sync(FULL, excl, j + st);
          if (ex <= r) j += st;
        }
        const u32 ej = __shfl_sync(FULL, excl, j);
        const u64 sj = __shfl_sync(FULL, src, j);
        e[u] = r < tot ? __ldcg(&a.frec[sj + (r - ej)]) : make_uint4(0u, 0u, 0u, 0u);
      }
#pragma unroll
      for (int u = 0; u < K2R_U; u++) {
        if (r0 + u * 32 >= tot) break;  // warp-uniform
        const bool v = r0 + u * 32 + lane < tot;
        const bool keep = v && e[u].y >= kmin;
        const u32 qk = __ballot_sync(FULL, keep);
        if (keep) a.sup_sid[out0 + run + __popc(qk & lt)] = e[u];
        run += __popc(qk);
        const bool m1 = v && e[u].y - kmin <= span;
        const bool m2 = BETA2 && v && e[u].z - kmin <= span;
        const u32 nb = (m1 ? 1u : 0u) + (m2 ? 1u : 0u);
        const u32 wnb = __reduce_add_sync(FULL, nb);
        if (wnb == 0) continue;
        const u32 inb = warp_incl_scan<u32>(nb);
        u32 o = 0;
        if (lane == 31) o = atomicAdd(s_cnt, inb);
        o = __shfl_sync(FULL, o, 31) + inb - nb;
        if (m1) {
          atomicAdd(&shist[(e[u].y - kmin) >> DSH3], 1u);
          region[o++] = e[u].y;
        }
        if (m2) {
          atomicAdd(&shist[(e[u].z - kmin) >> DSH3], 1u);
          region[o] = e[u].z;
        }
      }
    }
  }
  out0_o = out0;
  run_o = run;
}

// K2: pass 2 of kth(D) -- one read of D.  CTA c owns the contiguous range
// [c*R, (c+1)*R) of D and each of its warps one eighth of it.  A warp step is
// 512 delegates, 16 consecutive ones per lane (four uint4).  theta's digit-1
// bucket is the key interval [kmin, kmax] (log-scale digit, ddig1):
//   * delegates inside it: digit-2 histogram (shared memory) and compaction
//     into the CTA's region of selbuf (order irrelevant);
//   * max delegates d_1 >= kmin (every subrange that can qualify, whatever
//     theta turns out to be inside the bucket): ordered compaction of their
//     subrange ids into the warp's segment of the superset, the only input
//     K3 reads -- D is not scanned again.
// A lane first tests its 16 keys against kmin through their maximum (for
// beta = 2 the max delegates alone), so most steps cost ~1 op per key.
template <int BETA2>
__global__ void __launch_bounds__(256, DTOPK_K2_MINB) k2_scan_delegates(K2Args a) {
  pdl_trigger();
  pdl_wait();
  __shared__ u32 shist[NBD2];
  __shared__ DigitResult r1;
  __shared__ ull scratch[8];
  __shared__ u32 s_cnt;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (a.fmode == 2 && !ld_volatile_u32(&a.ctrl->filt_fail)) return;  // fallback scan not needed
  const bool records = a.fmode == 1 && ld_volatile_u32(&a.ctrl->filt_on) != 0;
  for (int i = tid; i < NBD2; i += 256) shist[i] = 0;
  if (tid == 0) s_cnt = 0;
  find_digit<NBD1>(a.ctrl->selD.hist1, a.k, &r1, scratch);
  if (blockIdx.x == 0 && tid == 0) a.ctrl->selD.r1 = r1;
  u32 kmin, kmax;
  dbucket(r1.digit, a.lin != 0, kmin, kmax);
  const u32 span = kmax - kmin;
  if (records && (ld_volatile_u32(&a.ctrl->filt_t) > kmin || r1.cnt * 4 > a.nD)) {
    // the sampled floor missed theta's bucket (or the bucket is a large share of
    // D, which pass 3 / K2b resolve from D itself): D was not written, so the
    // full K1 + K2 run again (fmode 2 launches) -- nothing is written here
    if (blockIdx.x == 0 && tid == 0) {
      a.ctrl->filt_fail = 1u;
      a.ctrl->res.filter_fallback = 1u;
      if (a.fb_graph) cudaGraphSetConditional(a.fb, 1u);
    }
    return;
  }
  const u64 lo = (u64)blockIdx.x * a.R;
  const u64 hi = min(a.nD, lo + a.R);
  const u64 wlen = a.R / 8;
  const u64 wlo = min(hi, lo + (u64)warp * wlen), whi = min(hi, wlo + wlen);
  const u64 beta = BETA2 ? 2u : (u64)a.beta;
  u64 out0 = (wlo + beta - 1) / beta;  // first subrange whose d_1 lies in [wlo, whi)
  u32* region = a.selbuf + lo;
  // a bucket holding a large share of D (tie-heavy / narrow range): the bucket
  // floor says little, so the superset is left to K2b, which filters D with
  // the exact theta after pass 3
  const bool sup = a.sup_sid != nullptr && r1.cnt * 4 <= a.nD;
  // a bucket holding a large share of D (tie-heavy or narrow-range inputs): do
  // not copy it into the regions; pass 3 scans D itself (same bytes, no writes)
  const bool compact = r1.cnt * 4 <= a.nD;
  u32 run = 0;
  u32 bmn = 0xffffffffu, bmx = 0u;  // large bucket: value range of its members
  if (records) k2_records<BETA2>(a, kmin, span, shist, &s_cnt, region, out0, run);
  for (u64 base = records ? whi : wlo; base < whi; base += 512) {
    const u64 i0 = base + (u64)lane * 16;
    u32 v[16];
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const u64 i = i0 + 4 * j;
      if (i + 4 <= whi) {
        const uint4 q = *reinterpret_cast<const uint4*>(a.D + i);
        v[4 * j] = q.x;
        v[4 * j + 1] = q.y;
        v[4 * j + 2] = q.z;
        v[4 * j + 3] = q.w;
      } else {
#pragma unroll
        for (int c = 0; c < 4; c++) v[4 * j + c] = i + c < whi ? a.D[i + c] : 0u;
      }
    }
    u32 mx = 0;
    if (BETA2) {  // (d1, d2) pairs, d1 >= d2: the max of the lane is a max delegate
#pragma unroll
      for (int j = 0; j < 16; j += 2) mx = max(mx, v[j]);
    } else {
#pragma unroll
      for (int j = 0; j < 16; j++) mx = max(mx, v[j]);
    }
    const bool any = mx >= kmin;
    if (!__any_sync(FULL, any)) continue;
    // per-lane bit masks over the 16 keys: bucket members and candidate max delegates
    const u32 rem = i0 < whi ? (u32)min((u64)16, whi - i0) : 0u;  // keys of this lane inside the warp range
    u32 mb = 0, mc = 0;
    if (any) {
      u32 r = BETA2 ? 0u : (u32)(i0 % beta);  // ladder slot of element i0 (i0 is even for beta 2)
#pragma unroll
      for (int j = 0; j < 16; j++) {
        const bool in = (u32)j < rem;
        mb |= (in && v[j] - kmin <= span) ? (1u << j) : 0u;
        if (sup) mc |= (in && r == 0 && v[j] >= kmin) ? (1u << j) : 0u;
        r = BETA2 ? (r ^ 1u) : ((r + 1 == (u32)beta) ? 0u : r + 1);
      }
    }
    const u32 nc = __popc(mc), nb = __popc(mb);
    if (sup && __any_sync(FULL, nc)) {
      const u32 incl = warp_incl_scan<u32>(nc);
      u64 o = out0 + run + incl - nc;
      run += __shfl_sync(FULL, incl, 31);
      if (mc) {
#pragma unroll
        for (int j = 0; j < 16; j++) {
          if ((mc >> j) & 1u) {
            // beta 2: (d1, d2) sit in this lane's registers (pairs start at even j)
            const u32 d2 = BETA2 ? v[j | 1] : 0u;
            const u32 sid = (u32)((i0 + j) / beta);
            a.sup_sid[o++] = make_uint4(sid, v[j], d2, __ldg(a.meta + sid));
          }
        }
      }
    }
    const u32 wnb = __reduce_add_sync(FULL, nb);
    if (wnb == 0) continue;
    if (!compact) {
#pragma unroll
      for (int j = 0; j < 16; j++)
        if ((mb >> j) & 1u) {
          bmn = min(bmn, v[j]);
          bmx = max(bmx, v[j]);
        }
    }
    const u32 incl = warp_incl_scan<u32>(nb);
    u32 o = 0;
    if (lane == 31) o = atomicAdd(&s_cnt, incl);
    o = __shfl_sync(FULL, o, 31) + incl - nb;
    if (wnb > 64) {  // many members (tie-heavy / narrow range): warp-aggregated bins
#pragma unroll
      for (int j = 0; j < 16; j++) hist_add_warp(shist, (v[j] - kmin) >> DSH3, (mb >> j) & 1u);
    } else if (mb) {
#pragma unroll
      for (int j = 0; j < 16; j++)
        if ((mb >> j) & 1u) atomicAdd(&shist[(v[j] - kmin) >> DSH3], 1u);
    }
    if (compact && mb) {
#pragma unroll
      for (int j = 0; j < 16; j++)
        if ((mb >> j) & 1u) region[o++] = v[j];
    }
  }
  if (sup && lane == 0) {
    a.sup_in[blockIdx.x * 8 + warp] = (u32)out0;
    a.sup_cnt[blockIdx.x * 8 + warp] = run;
  }
  if (!compact) {
    bmn = __reduce_min_sync(FULL, bmn);
    bmx = __reduce_max_sync(FULL, bmx);
    if (lane == 0 && bmx >= bmn) {
      atomicMax(&a.ctrl->bk_nmin, ~bmn);
      atomicMax(&a.ctrl->bk_max, bmx);
    }
  }
  __syncthreads();
  Ctrl* ctrl = a.ctrl;
  if (tid == 0) a.region_cnt[blockIdx.x] = compact ? s_cnt : 0u;
  for (int i = tid; i < NBD2; i += 256) {
    const u32 c = shist[i];
    if (c) atomicAdd(&ctrl->selD.hist2[i], (ull)c);
  }
}

#ifndef DTOPK_P3_SMALL
#define DTOPK_P3_SMALL 8192
#endif
constexpr int P3_SMALL = DTOPK_P3_SMALL;  // bucket members resolved by one CTA
constexpr int P3_RPT = 3;        // regions per thread in that CTA's prefix
constexpr int P3_REGIONS = 256 * P3_RPT;
constexpr int P3_LPT = 8;           // member loads in flight per thread (8 measured faster than 24)
constexpr int P3_THREAD_MAX = 64;   // larger regions are loaded by whole warps
// padded shared histogram index: thread t's 32 consecutive bins start 33 t
// words apart, so find_digit_sm's per-thread block reads hit 32 banks
__device__ __forceinline__ u32 p3_pad(u32 b) { return b + (b >> 5); }

// Pass 3 of kth(D) over the compacted bucket regions;
// the last CTA resolves theta and the superset record offsets.
// Large single-valued bucket (tie-heavy input), truncation allowed: one pass
// over D with theta known gives, per K2b segment (CTA region g, warp w), a lower
// bound of its ties (d_1 == theta: >= 1, >= 2 when d_2 == theta too) and its
// entries above theta, plus the exact FQ / PQ / candidate counts of the whole
// vector (pipeline.py:104-109: d_beta >= theta / d_1 >= theta > d_beta).  The last
// CTA finds the first segment by which the tie lower bounds reach k: K2b drops
// tie-only entries after it, since the first k ties in index order lie before.
__device__ __noinline__ void p3_tie_bounds(Ctrl* ctrl, const u32* __restrict__ D, u64 nD, u64 R, u32 nregions,
                                           int beta, u64 k, u32 theta, uint2* tseg, ull* scratch, int* am_last) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  ull fq = 0, pq = 0;
  for (u32 g = blockIdx.x; g < nregions; g += gridDim.x) {
    const u64 lo = (u64)g * R, hi = min(nD, lo + R), wlen = R / 8;
    const u64 wlo = min(hi, lo + (u64)warp * wlen), whi = min(hi, wlo + wlen);
    ull lb = 0;
    u32 ngt = 0;
    for (u64 base = wlo; base < whi; base += 512) {
      const u64 i0 = base + (u64)lane * 16;
      u32 v[16];
#pragma unroll
      for (int j = 0; j < 4; j++) {
        const u64 i = i0 + 4 * j;
        if (i + 4 <= whi) {
          const uint4 q = ld_nc_v4(D + i);
          v[4 * j] = q.x;
          v[4 * j + 1] = q.y;
          v[4 * j + 2] = q.z;
          v[4 * j + 3] = q.w;
        } else {
#pragma unroll
          for (int c = 0; c < 4; c++) v[4 * j + c] = i + c < whi ? D[i + c] : 0u;
        }
      }
      const u32 rem = i0 < whi ? (u32)min((u64)16, whi - i0) : 0u;
      if (beta == 2) {  // (d_1, d_2) pairs; i0 is even
#pragma unroll
        for (int j = 0; j < 16; j += 2) {
          if ((u32)j >= rem) break;
          const u32 d1 = v[j], d2 = v[j + 1];
          ngt += d1 > theta;
          lb += d1 == theta ? (d2 == theta ? 2u : 1u) : 0u;
          fq += d2 >= theta;
          pq += d1 >= theta && d2 < theta;
        }
      } else {  // beta 1: d_beta = d_1
#pragma unroll
        for (int j = 0; j < 16; j++) {
          if ((u32)j >= rem) break;
          ngt += v[j] > theta;
          lb += v[j] == theta;
          fq += v[j] >= theta;
        }
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      lb += __shfl_xor_sync(FULL, lb, o);
      ngt += __shfl_xor_sync(FULL, ngt, o);
    }
    if (lane == 0) tseg[g * 8 + warp] = make_uint2((u32)min(lb, (ull)0xffffffffu), ngt);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    fq += __shfl_xor_sync(FULL, fq, o);
    pq += __shfl_xor_sync(FULL, pq, o);
  }
  if (lane == 0) {
    if (fq) atomicAdd((ull*)&ctrl->res.fully_qualified, fq);
    if (pq) atomicAdd((ull*)&ctrl->res.partially_qualified, pq);
    if (fq + pq) atomicAdd((ull*)&ctrl->res.candidate_subranges, fq + pq);
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) *am_last = atomicAdd(&ctrl->tb_done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!*am_last) return;
  __threadfence();
  // first segment whose inclusive tie lower bound reaches k (thread t: segments t*24 ..)
  const u32 nseg = nregions * 8;
  ull c[K2_SEG_PER];
  ull sum = 0;
#pragma unroll
  for (int q = 0; q < K2_SEG_PER; q++) {
    const u32 i = (u32)tid * K2_SEG_PER + q;
    c[q] = i < nseg ? (ull)__ldcg(&tseg[i].x) : 0ull;
    sum += c[q];
  }
  __shared__ u32 s_cut;
  if (tid == 0) s_cut = nseg;
  const ull incl = block_incl_scan_256<ull>(sum, scratch);
  ull run = incl - sum;
#pragma unroll
  for (int q = 0; q < K2_SEG_PER; q++) {
    if (run < k && run + c[q] >= k) s_cut = (u32)tid * K2_SEG_PER + q;
    run += c[q];
  }
  __syncthreads();
  if (tid == 0) {
    ctrl->tie_cut = s_cut;
    ctrl->trunc = 1u;
    if (s_cut + 1 < nseg) atomicAdd((ull*)&ctrl->res.concat_skipped_fq, 1ull);  // |C| not counted past the cut
  }
}

__device__ __forceinline__ void p3_set_theta(Ctrl* ctrl, u32 kth, const DigitResult& r1) {
  ctrl->selD.kth = kth;
  ctrl->res.theta_local = kth;
  ctrl->res.theta_slot = (int64_t)kth;
  ctrl->res.delegate_bucket = r1.cnt;
}

__global__ void __launch_bounds__(256, 1) k2_pass3(Ctrl* ctrl, const u32* __restrict__ selbuf,
                                                const u32* __restrict__ region_cnt, u32 nregions, u64 R,
                                                const u32* __restrict__ sup_cnt, u32* __restrict__ sup_off,
                                                const u32* __restrict__ D, u64 nD, int lin) {
  pdl_trigger();
  pdl_wait();
  __shared__ u32 shist[NBD3 + NBD3 / 32];  // small path: bin b at p3_pad(b) (conflict-free digit scan)
  __shared__ DigitResult r3;
  __shared__ ull scratch[8];
  __shared__ int am_last;
  __shared__ u32 s_big[P3_REGIONS];
  __shared__ u32 s_nbig;
  const int tid = threadIdx.x;
  __shared__ DigitResult r2;
#ifdef DTOPK_P3_PROFILE
  unsigned long long pt[6];
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(pt[0]));
#define P3_MARK(i) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(pt[i]))
#else
#define P3_MARK(i)
#endif
  const DigitResult r1 = ctrl->selD.r1;  // read before the flag: one round trip for both
  if (ld_volatile_u32(&ctrl->small_done)) return;  // fast_tail resolved theta and finished the call
  // a small compacted bucket (small k): one CTA resolves theta from the members
  // directly, without the grid-wide histogram flush and last-CTA hand-off
  const bool small = r1.cnt * 4 <= nD && r1.cnt <= (ull)P3_SMALL && nregions <= (u32)P3_REGIONS;
  if (small && blockIdx.x != 0) return;
  // small path: the region counts and the superset segment counts are loaded
  // before the digit-2 scan, so their round trips overlap it
  u32 c[P3_RPT];
  uint4 supx[K2_SEG_PER / 4];
  const bool sup_now = small && sup_cnt != nullptr;  // (r1.cnt * 4 <= nD holds on the small path)
  if (small) {
#pragma unroll
    for (int q = 0; q < P3_RPT; q++) {
      const u32 g = (u32)tid * P3_RPT + q;
      c[q] = g < nregions ? __ldcg(region_cnt + g) : 0u;
    }
    if (sup_now) k2_sup_load(sup_cnt, supx);
  }
  for (int i = tid; i < NBD3 + NBD3 / 32; i += 256) shist[i] = 0;
  if (tid == 0) s_nbig = 0;
  u32 kmin, kmax;
  dbucket(r1.digit, lin != 0, kmin, kmax);
  P3_MARK(1);
  find_digit<NBD2>(ctrl->selD.hist2, r1.rem, &r2, scratch);
  if (blockIdx.x == 0 && tid == 0) ctrl->selD.r2 = r2;
  const u32 b2 = r2.digit;
  P3_MARK(2);
  if (small) {
    // thread t owns regions t*P3_RPT .. and loads their members itself, P3_LPT
    // loads in flight (a region holds ~members / regions keys: ~7 at k = 2^20);
    // a region above P3_THREAD_MAX members goes to a list that whole warps load.
    // (A flat member loop with a binary search per member over the region
    // prefix took 17 us for 4k members at k = 2^20.)
#pragma unroll
    for (int q = 0; q < P3_RPT; q++) {
      const u32 g = (u32)tid * P3_RPT + q;
      if (c[q] > (u32)P3_THREAD_MAX) {
        s_big[atomicAdd(&s_nbig, 1u)] = g;
        c[q] = 0;
      }
    }
    u32 tot = 0;
#pragma unroll
    for (int q = 0; q < P3_RPT; q++) tot += c[q];
    for (u32 j0 = 0; j0 < tot; j0 += P3_LPT) {
      u32 x[P3_LPT];
#pragma unroll
      for (int u = 0; u < P3_LPT; u++) {
        u32 j = j0 + u;
        x[u] = 0xffffffffu;
        if (j < tot) {
          int q = 0;
#pragma unroll
          for (int r = 0; r < P3_RPT - 1; r++)
            if (q == r && j >= c[r]) {
              j -= c[r];
              q = r + 1;
            }
          x[u] = selbuf[(u64)((u32)tid * P3_RPT + q) * R + j] - kmin;
        }
      }
#pragma unroll
      for (int u = 0; u < P3_LPT; u++)
        if (x[u] != 0xffffffffu && (x[u] >> DSH3) == b2) atomicAdd(&shist[p3_pad(x[u] & ((1u << DSH3) - 1u))], 1u);
    }
    __syncthreads();
    const int lane = tid & 31, warp = tid >> 5;
    for (u32 b = warp; b < s_nbig; b += 8) {
      const u32 g = s_big[b], cnt = region_cnt[g];
      const u32* reg = selbuf + (u64)g * R;
      for (u32 i0 = 0; i0 < cnt; i0 += 32 * P3_LPT) {
        u32 x[P3_LPT];
#pragma unroll
        for (int u = 0; u < P3_LPT; u++) {
          const u32 i = i0 + u * 32 + lane;
          x[u] = i < cnt ? reg[i] - kmin : 0xffffffffu;
        }
#pragma unroll
        for (int u = 0; u < P3_LPT; u++)
          if (x[u] != 0xffffffffu && (x[u] >> DSH3) == b2) atomicAdd(&shist[p3_pad(x[u] & ((1u << DSH3) - 1u))], 1u);
      }
    }
    __syncthreads();
    P3_MARK(3);
    k2_theta_from_hist3(ctrl, kmin, r1, r2, &r3, scratch, shist);
    if (sup_now) k2_superset_prefix_regs(ctrl, nregions, supx, sup_off, scratch);
    P3_MARK(4);
#ifdef DTOPK_P3_PROFILE
    if (tid == 0)
      printf("p3 small: members=%llu regions=%u | r1 %llu find2 %llu loop %llu resolve %llu ns\n", r1.cnt, nregions,
             pt[1] - pt[0], pt[2] - pt[1], pt[3] - pt[2], pt[4] - pt[3]);
#endif
    return;
  }
  if (r1.cnt * 4 > nD) {
    // a large bucket holding one value (all-equal / few-distinct input): theta
    // is that value, no digit-3 pass; with truncation allowed, the pass over D
    // counts ties per K2b segment instead (p3_tie_bounds)
    const u32 bmn = ~ld_volatile_u32(&ctrl->bk_nmin), bmx = ld_volatile_u32(&ctrl->bk_max);
    if (bmn == bmx) {
      if (blockIdx.x == 0 && tid == 0) p3_set_theta(ctrl, bmn, r1);
      return;
    }
    // K2 did not compact this (large) bucket: scan D, four uint4 per thread and step
    const u32 span = kmax - kmin;
    const u64 nq = nD / 4;
    for (u64 q0 = (u64)blockIdx.x * 1024; q0 < nq; q0 += (u64)gridDim.x * 1024) {
      uint4 x[4];
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const u64 q = q0 + u * 256 + tid;
        x[u] = q < nq ? ld_nc_v4(D + 4 * q) : make_uint4(kmin - 1, kmin - 1, kmin - 1, kmin - 1);
      }
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const u32 e[4] = {x[u].x - kmin, x[u].y - kmin, x[u].z - kmin, x[u].w - kmin};
#pragma unroll
        for (int c = 0; c < 4; c++)
          hist_add_warp(shist, e[c] & ((1u << DSH3) - 1u), e[c] <= span && (e[c] >> DSH3) == b2);
      }
    }
    if (blockIdx.x == 0) {  // tail of nD % 4 delegates
      const u64 i = nq * 4 + tid;
      const u32 e = i < nD ? D[i] - kmin : 0xffffffffu;
      if (tid < 32) hist_add_warp(shist, e & ((1u << DSH3) - 1u), e <= span && (e >> DSH3) == b2);
    }
  }
  for (u32 g = blockIdx.x; g < nregions; g += gridDim.x) {
    const u32 cnt = region_cnt[g];
    const u32* reg = selbuf + (u64)g * R;
    for (u32 i0 = 0; i0 < cnt; i0 += 256 * 8) {  // 8 loads in flight per thread
      u32 x[8];
#pragma unroll
      for (int u = 0; u < 8; u++) {
        const u32 i = i0 + u * 256 + tid;
        x[u] = i < cnt ? reg[i] - kmin : 0xffffffffu;
      }
#pragma unroll
      for (int u = 0; u < 8; u++) hist_add_warp(shist, x[u] & ((1u << DSH3) - 1u), x[u] != 0xffffffffu && (x[u] >> DSH3) == b2);
    }
  }
  __syncthreads();
  for (int i = tid; i < NBD3; i += 256) {
    const u32 v = shist[i];
    if (v) atomicAdd(&ctrl->selD.hist3[i], (ull)v);
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) am_last = atomicAdd(&ctrl->selD.done3, 1u) == gridDim.x - 1;
  __syncthreads();
  if (am_last) {
    __threadfence();
    k2_resolve_theta(ctrl, kmin, r1, r2, nregions, sup_cnt, sup_off, &r3, scratch, nD);
  }
}

// K2c: tie bounds for a large-bucket call (tie-heavy input) once theta is
// known; exits at once otherwise (see p3_tie_bounds).
__global__ void __launch_bounds__(256) k2c_tie_bounds(Ctrl* ctrl, const u32* __restrict__ D, u64 nD, u64 R,
                                                      u32 nregions, int beta, u64 k, uint2* tseg) {
  pdl_trigger();
  pdl_wait();
  __shared__ ull scratch[8];
  __shared__ int am_last;
  if (ld_volatile_u32(&ctrl->small_done)) return;
  const DigitResult r1 = ctrl->selD.r1;
  if (r1.cnt * 4 <= nD) return;
  p3_tie_bounds(ctrl, D, nD, R, nregions, beta, k, ctrl->selD.kth, tseg, scratch, &am_last);
}

// K2b: exact candidate superset for calls whose theta bucket held a large share
// of D (K2 deferred it): one more read of D with the exact theta, ordered
// compaction per (CTA, warp) segment as in K2, then the last CTA offsets the
// segments.  Other calls exit at once.
template <int BETA2>
__global__ void __launch_bounds__(256) k2b_superset(K2Args a) {
  pdl_trigger();
  pdl_wait();
  __shared__ ull scratch[8];
  __shared__ int am_last;
  __shared__ uint4 stage[8][BETA2 ? 256 : 1];
  Ctrl* ctrl = a.ctrl;
  if (ld_volatile_u32(&ctrl->small_done)) return;  // finished by fast_tail
  const DigitResult r1 = ctrl->selD.r1;
  if (a.sup_sid == nullptr || r1.cnt * 4 <= a.nD) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const u32 theta = ctrl->selD.kth;  // <= any external theta applied in K3: still a superset
  const u64 lo = (u64)blockIdx.x * a.R;
  const u64 hi = min(a.nD, lo + a.R);
  const u64 wlen = a.R / 8;
  const u64 wlo = min(hi, lo + (u64)warp * wlen), whi = min(hi, wlo + wlen);
  const u64 beta = BETA2 ? 2u : (u64)a.beta;
  const u64 out0 = (wlo + beta - 1) / beta;
  u32 run = 0;
  // truncated (pass 3, p3_tie_bounds): past the cut only entries above theta are
  // kept, and segments without any are not read at all
  const u32 seg = blockIdx.x * 8 + warp;
  const bool trunc = ld_volatile_u32(&ctrl->trunc) != 0;
  const bool ties = !trunc || seg <= ld_volatile_u32(&ctrl->tie_cut);
  const bool skip = !ties && __ldcg(&a.tseg[seg].y) == 0;
  const u32 floor_key = ties ? theta : theta + 1u;  // theta < max key whenever an entry lies above it
  for (u64 base = skip ? whi : wlo; base < whi; base += 512) {
    const u64 i0 = base + (u64)lane * 16;
    u32 v[16];
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const u64 i = i0 + 4 * j;
      if (i + 4 <= whi) {
        const uint4 q = ld_nc_v4(a.D + i);
        v[4 * j] = q.x;
        v[4 * j + 1] = q.y;
        v[4 * j + 2] = q.z;
        v[4 * j + 3] = q.w;
      } else {
#pragma unroll
        for (int c = 0; c < 4; c++) v[4 * j + c] = i + c < whi ? a.D[i + c] : 0u;
      }
    }
    const u32 rem = i0 < whi ? (u32)min((u64)16, whi - i0) : 0u;
    u32 mc = 0, r = BETA2 ? 0u : (u32)(i0 % beta);
#pragma unroll
    for (int j = 0; j < 16; j++) {
      mc |= ((u32)j < rem && r == 0 && v[j] >= floor_key) ? (1u << j) : 0u;
      r = BETA2 ? (r ^ 1u) : ((r + 1 == (u32)beta) ? 0u : r + 1);
    }
    const u32 nc = __popc(mc);
    if (!__any_sync(FULL, nc)) continue;
    const u32 incl = warp_incl_scan<u32>(nc);
    const u32 tot = __shfl_sync(FULL, incl, 31);
    if (BETA2) {
      // stage the warp's (<= 256) entries in shared memory, then store them
      // contiguously: all-candidate inputs (ties) would otherwise store one
      // 16-byte entry per 128-byte line per instruction
      u32 t = incl - nc;
#pragma unroll
      for (int j = 0; j < 16; j += 2)
        if ((mc >> j) & 1u) {
          const u32 sid = (u32)((i0 + j) >> 1);
          stage[warp][t++] = make_uint4(sid, v[j], v[j + 1], __ldg(a.meta + sid));
        }
      __syncwarp();
      for (u32 q = lane; q < tot; q += 32) a.sup_sid[out0 + run + q] = stage[warp][q];
      __syncwarp();
    } else {
      u64 o = out0 + run + incl - nc;
#pragma unroll
      for (int j = 0; j < 16; j++)
        if ((mc >> j) & 1u) {
          const u32 sid = (u32)((i0 + j) / beta);
          a.sup_sid[o++] = make_uint4(sid, v[j], 0u, __ldg(a.meta + sid));
        }
    }
    run += tot;
  }
  if (lane == 0) {
    a.sup_in[blockIdx.x * 8 + warp] = (u32)out0;
    a.sup_cnt[blockIdx.x * 8 + warp] = run;
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) am_last = atomicAdd(&ctrl->k2b_done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  k2_superset_prefix(ctrl, gridDim.x, a.sup_cnt, a.sup_off, scratch);
}

// ---------------------------------------------------------------------------
// Generic select over an arbitrary key array (pool P_gt in key space, or the
// raw input on the direct path).  The k-th key itself is resolved at the start
// of the consumer (scan_emit), so no extra launch is needed.
// ---------------------------------------------------------------------------
struct SelArgs {
  const u32* keys;
  u64 m_host;
  const ull* m_dev;  // element count on device (pool size), or null
  Ctrl* ctrl;
  SelectState* sel;
  u32* selbuf;
  u64 k;
  int check_path;  // run only when ctrl->res.path == PATH_SELECT
  u32* tcnt;       // [ceil(m / 2048)] members of digit-1 bucket per sel_pass2 tile
};

__device__ __forceinline__ bool sel_skip(const SelArgs& a) {
  return a.check_path && ld_volatile_u32(&a.ctrl->big_mode) != BIG_SELECT;
}
__device__ __forceinline__ u64 sel_count(const SelArgs& a) { return a.m_dev ? (u64)*a.m_dev : a.m_host; }

template <int MODE>
__global__ void __launch_bounds__(256) sel_pass1(SelArgs a) {
  if (sel_skip(a)) return;
  __shared__ u32 shist[NB1];
  for (int i = threadIdx.x; i < NB1; i += 256) shist[i] = 0;
  __syncthreads();
  const u64 m = sel_count(a);
  const u64 m4 = m / 4;
  const u64 stride = (u64)gridDim.x * 256;
  const uint4* k4 = reinterpret_cast<const uint4*>(a.keys);
  for (u64 i = (u64)blockIdx.x * 256 + threadIdx.x; i < m4; i += stride) {
    const uint4 v = ld_nc_v4(k4 + i);
    atomicAdd(&shist[dig1(to_key<MODE>(v.x))], 1u);
    atomicAdd(&shist[dig1(to_key<MODE>(v.y))], 1u);
    atomicAdd(&shist[dig1(to_key<MODE>(v.z))], 1u);
    atomicAdd(&shist[dig1(to_key<MODE>(v.w))], 1u);
  }
  for (u64 i = m4 * 4 + (u64)blockIdx.x * 256 + threadIdx.x; i < m; i += stride)
    atomicAdd(&shist[dig1(to_key<MODE>(a.keys[i]))], 1u);
  __syncthreads();
  for (int i = threadIdx.x; i < NB1; i += 256) {
    const u32 v = shist[i];
    if (v) atomicAdd(&a.sel->hist1[i], (ull)v);
  }
}

template <int MODE>
__global__ void __launch_bounds__(256) sel_pass2(SelArgs a) {
  if (sel_skip(a)) return;
  __shared__ u32 shist[NB2];
  __shared__ DigitResult r1;
  __shared__ ull scratch[8];
  __shared__ u32 s_wcnt[8];
  __shared__ ull s_base;
  for (int i = threadIdx.x; i < NB2; i += 256) shist[i] = 0;
  find_digit<NB1>(a.sel->hist1, a.k, &r1, scratch);
  if (blockIdx.x == 0 && threadIdx.x == 0) a.sel->r1 = r1;
  const u32 b1 = r1.digit;
  const u64 m = sel_count(a);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const u32 lt = lanemask_lt();
  // tiles of 256 x 8 keys; one global atomic per tile reserves the slots
  const u64 T = (m + 2047) / 2048;
  for (u64 tile = blockIdx.x; tile < T; tile += gridDim.x) {
    u32 v[8], bl[8], cnt = 0;
#pragma unroll
    for (int j = 0; j < 8; j++) {
      const u64 i = tile * 2048 + (u64)warp * 256 + (u64)j * 32 + lane;
      v[j] = i < m ? to_key<MODE>(a.keys[i]) : 0u;
      const bool p = i < m && dig1(v[j]) == b1;
      bl[j] = __ballot_sync(FULL, p);
      cnt += __popc(bl[j]);
      if (p) atomicAdd(&shist[dig2(v[j])], 1u);
    }
    if (lane == 0) s_wcnt[warp] = cnt;
    __syncthreads();
    // tile-private slots (the tile's own 2048 positions of selbuf): one global
    // atomic counter per tile serialised ~1k tiles on sorted pools
    u64 o = tile * 2048;
    u32 tot = 0;
    for (int w = 0; w < 8; w++) {
      if (w < warp) o += s_wcnt[w];
      tot += s_wcnt[w];
    }
    if (threadIdx.x == 0) a.tcnt[tile] = tot;
#pragma unroll
    for (int j = 0; j < 8; j++) {
      if ((bl[j] >> lane) & 1u) a.selbuf[o + __popc(bl[j] & lt)] = v[j];
      o += __popc(bl[j]);
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < NB2; i += 256) {
    const u32 v = shist[i];
    if (v) atomicAdd(&a.sel->hist2[i], (ull)v);
  }
}

__global__ void __launch_bounds__(256) sel_pass3(SelArgs a) {
  if (sel_skip(a)) return;
  __shared__ u32 shist[NB3];
  __shared__ DigitResult r2;
  __shared__ ull scratch[8];
  for (int i = threadIdx.x; i < NB3; i += 256) shist[i] = 0;
  const DigitResult r1 = a.sel->r1;
  find_digit<NB2>(a.sel->hist2, r1.rem, &r2, scratch);
  if (blockIdx.x == 0 && threadIdx.x == 0) a.sel->r2 = r2;
  const u32 b2 = r2.digit;
  const u64 T = (sel_count(a) + 2047) / 2048;  // sel_pass2 tiles: members at tile * 2048, tcnt[tile] of them
  for (u64 tile = blockIdx.x; tile < T; tile += gridDim.x) {
    const u32 c = a.tcnt[tile];
    for (u32 i = threadIdx.x; i < c; i += 256) {
      const u32 x = a.selbuf[tile * 2048 + i];
      if (dig2(x) == b2) atomicAdd(&shist[dig3(x)], 1u);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < NB3; i += 256) {
    const u32 v = shist[i];
    if (v) atomicAdd(&a.sel->hist3[i], (ull)v);
  }
}

// Resolve the k-th key after sel_pass3 (used by dtopk_kth_largest).
__global__ void __launch_bounds__(256) sel_finalize(SelectState* sel, u32* out_kth) {
  __shared__ DigitResult r3;
  __shared__ ull scratch[8];
  const DigitResult r1 = sel->r1, r2 = sel->r2;
  find_digit<NB3>(sel->hist3, r2.rem, &r3, scratch);
  if (threadIdx.x == 0) {
    const u32 kth = (r1.digit << 21) | (r2.digit << 10) | r3.digit;
    sel->r3 = r3;
    sel->kth = kth;
    *out_kth = kth;
  }
}

}  // namespace dtopk
