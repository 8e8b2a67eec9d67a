// assemble.cuh -- qualification and candidate-pool assembly after theta.
//
// Reference semantics: first_topk qualification (pipeline.py:104-116) and
// concatenate_filtered (pipeline.py:119-159), extended with indices under the
// tie rule of kernels._extract_exact (kernels.py:83-96).
//
// K1 records, per subrange, the offset p1 of (the first occurrence of) its
// maximum and whether the subrange is constant.  With the exact theta every
// qualifying subrange (d_1 >= theta) falls in one class that says what it
// contributes without necessarily re-reading it (d_2 < d_1 means the max is
// unique, so p1 locates the only key >= theta):
//   A  d_1 > theta, d_2 < theta   one element > theta, at p1 (no read)
//   B  d_1 = theta, d_2 < theta   one tie, at p1 (no read)
//   C  d_1 = theta, constant      every key is a tie (no read)
//   T  d_1 = theta otherwise      ties only; K4T counts them, K6 locates the
//                                 ones among the first k ties
//   E  d_1 > theta, d_2 >= theta  (or beta = 1): read by K4.
// For uniform keys almost every candidate is A (the paper's partially
// qualified subranges), so the concatenation re-reads only the fully qualified
// ones; all-equal keys make every candidate C and nothing is re-read.
//
//   K3  classification of K2's candidate superset (subranges whose max
//       delegate reaches theta's first-digit bucket, or >= theta exactly when
//       K2b built it; already in subrange order): one 16-byte record per
//       entry, entries below theta inert.
//   K4  reads the E candidates; each candidate part (<= 8192 keys) writes its
//       elements > theta and its ties, in index order, into a private staging
//       slot -- no global ordering needed.
//   K4T counts the ties of T candidates (ordered early stop on tie-heavy input).
//   K5  ordered scan over the records (k5_count: tile sums, last CTA turns
//       them into prefixes; k5_emit: block scans on top) -> positions in the
//       pool P_gt (index order) and in the tie list (first k, index order).
//   K5b copies the staged keys / ties of E candidates to their places.
//   K6  locates the ties of C / T records that fall among the first k ties.
#pragma once

#include <cub/block/block_radix_sort.cuh>

#include "common.cuh"

namespace dtopk {

enum Cls : u32 { CLS_A = 0, CLS_B = 1, CLS_C = 2, CLS_T = 3, CLS_E = 4, CLS_NONE = 5 };

#ifndef DTOPK_K5E_MINB
#define DTOPK_K5E_MINB 4  // k5_emit min CTAs per SM (register cap: 107 -> 64, one wave; k=2^20: 21 -> 16.5 us)
#endif
#ifndef DTOPK_K3_U
#define DTOPK_K3_U 1
#endif
constexpr int K4_TILE = 8192;   // keys per K4 tile
#ifndef DTOPK_K5_RPT
#define DTOPK_K5_RPT 4
#endif
constexpr int K5_RPT = DTOPK_K5_RPT;  // consecutive records per K5 thread (A/B: 4 beats 2 and 8)
constexpr int K5_TILE = 256 * K5_RPT;  // records per K5 tile
constexpr int SMALL_POOL = 8192;  // pools up to this size are finished by one CTA (8 keys per thread)

// One 16-byte record per qualifying subrange: x = sid, y = d_1,
// z = K1 meta (constant << 31 | p1), w = cls | fq << 3 | (E or T index) << 4.
struct Records {
  uint4* r;
};

struct K3Args {
  const u32* D;
  const u32* meta;
  u64 S;
  u64 n;
  int alpha;
  int beta;
  Ctrl* ctrl;
  const int64_t* theta_override;
  Records rec;          // [sup_total] one record per superset entry, subrange order
  const uint4* sup_sid;  // K2 superset: {sid, d_1, d_2, meta} (beta 2) or {sid, d_1, -, meta}, per segment
  const u32* sup_in;    // [nseg] first superset slot of each segment
  const u32* sup_off;   // [nseg + 1] first record of each segment (K2 pass 3)
  u64 nseg;
  u32* e_sid;  // [nE] subrange of each E candidate
  u32* t_sid;  // [nT] subrange of each T candidate
  u32* t_cnt;  // [nT] ties of each T candidate (zeroed here, filled by K4T)
  u64 cap_e;
  u64* e_epos;  // [nE] tie-list position of each E candidate: set to "beyond k" here, by k5_emit if it places ties
};

__device__ __forceinline__ u64 sub_len(u64 sid, u64 n, int alpha) {
  const u64 W = 1ull << alpha;
  const u64 lo = sid << alpha;
  return min(W, n - lo);
}

// p1 and the constant flag of a K1 meta word (see pack_meta)
__device__ __forceinline__ u32 meta_p1(u32 m) { return m & 0x7fffffffu; }
__device__ __forceinline__ bool meta_const(u32 m) { return (m >> 31) != 0; }

__device__ __forceinline__ u32 classify(u32 d1, u32 d2, u32 m, u32 theta, int beta) {
  const bool single = beta >= 2 && d2 < theta;  // exactly one key >= theta: the unique max at p1
  if (d1 > theta) return single ? CLS_A : CLS_E;
  if (single) return CLS_B;
  return meta_const(m) ? CLS_C : CLS_T;
}

// K3: qualification and classification of the K2 superset (subranges whose
// max delegate reaches theta's digit-1 bucket), warp per superset segment,
// lane per entry.  Entries below theta become inert CLS_NONE records, so the
// record array keeps the superset's subrange order without a second
// compaction; D and meta are gathered only for superset entries.
__global__ void __launch_bounds__(256) k3_classify(K3Args a) {
  pdl_trigger();
  pdl_wait();
  if (ld_volatile_u32(&a.ctrl->small_done)) return;  // finished by fast_tail
  __shared__ ull s_stat[4][8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  Ctrl* ctrl = a.ctrl;
  u32 theta = ctrl->selD.kth;
  if (a.theta_override) {
    const long long o = *a.theta_override;
    const u32 ov = o < 0 ? 0u : (o > 0xffffffffll ? 0xffffffffu : (u32)o);
    theta = max(theta, ov);
  }
  if (blockIdx.x == 0 && tid == 0) ctrl->res.theta = theta;
  const int beta = a.beta;
  const u64 gw = ((u64)blockIdx.x * 256 + tid) >> 5;
  const u64 nw = ((u64)gridDim.x * 256) >> 5;
  const u32 lt = lanemask_lt();
  ull st_cand = 0, st_fq = 0, st_pq = 0, st_a = 0;
  u32 dmax = 0;
  u64 gt_rec = 0;
  for (u64 seg = gw; seg < a.nseg; seg += nw) {
    const u64 in0 = a.sup_in[seg];
    const u64 o0 = a.sup_off[seg];
    const u32 cnt = a.sup_off[seg + 1] - (u32)o0;
    // beta 2: the superset entry alone decides class E (d_1 > theta, d_2 >= theta),
    // so the segment's E slots come from one atomic per segment, counted first
    // (a contended per-group atomic sat on every group's critical path)
    // Likewise the T slots: every entry with d_1 == d_2 == theta is T or C (C =
    // constant subrange, known only from meta); all of them get a slot, C slots
    // become holes (t_sid = ~0) that K4T skips.
    u32 e_next = 0, t_next = 0, t_true = 0;
    const bool seg_e = beta == 2;
    if (seg_e) {
      u32 ne = 0, ntc = 0;
      for (u32 j0 = 0; j0 < cnt; j0 += 32) {
        const u32 j = j0 + lane;
        const uint4 e = j < cnt ? a.sup_sid[in0 + j] : make_uint4(0u, 0u, 0u, 0u);
        ne += __popc(__ballot_sync(FULL, j < cnt && e.y > theta && e.z >= theta));
        ntc += __popc(__ballot_sync(FULL, j < cnt && e.y == theta && e.z == theta));
      }
      if (ne | ntc) {
        if (lane == 0) {
          if (ne) e_next = atomicAdd(&ctrl->nE, ne);
          if (ntc) t_next = atomicAdd(&ctrl->nTslots, ntc);
        }
        e_next = __shfl_sync(FULL, e_next, 0);
        t_next = __shfl_sync(FULL, t_next, 0);
      }
    }
    constexpr int U = DTOPK_K3_U;  // 32-entry groups per warp step (1 measured fastest; 2, 4 slower)
    for (u32 j0 = 0; j0 < cnt; j0 += 32 * U) {
      u32 sid[U], d1[U], d2[U], dl[U], m[U];
#pragma unroll
      for (int u = 0; u < U; u++) {
        const u32 j = j0 + u * 32 + lane;
        const uint4 e = j < cnt ? a.sup_sid[in0 + j] : make_uint4(0u, 0u, 0u, 0u);
        sid[u] = e.x;
        d1[u] = e.y;
        d2[u] = e.z;
        dl[u] = e.z;  // beta 2: d_beta = d_2
        m[u] = e.w;   // K1 meta, copied by K2
      }
#pragma unroll
      for (int u = 0; u < U; u++) {
        const u32 j = j0 + u * 32 + lane;
        if (beta == 1) {  // d_beta = d_1 (D may be unwritten: filtered K1 pass)
          d2[u] = d1[u];
          dl[u] = d1[u];
        } else if (j < cnt && d1[u] >= theta && beta != 2) {  // D gathered for qualifying entries only
          d2[u] = a.D[(u64)sid[u] * beta + 1];
          dl[u] = a.D[(u64)sid[u] * beta + beta - 1];
        }
      }
#pragma unroll
      for (int u = 0; u < U; u++) {
        const u32 j = j0 + u * 32 + lane;
        const bool valid = j < cnt;
        const bool keep = valid && d1[u] >= theta;
        const u32 cls = keep ? classify(d1[u], d2[u], m[u], theta, beta) : CLS_NONE;
        const bool fq = keep && dl[u] >= theta;
        u32 x = cls | (fq ? 8u : 0u);
        // E / T list slots: one atomic per list and 32 entries, only when present
        const u32 be = __ballot_sync(FULL, cls == CLS_E), bt = __ballot_sync(FULL, cls == CLS_T);
        const u32 btc = seg_e ? __ballot_sync(FULL, keep && d1[u] == theta && d2[u] == theta) : 0u;  // T or C
        if (be | bt | btc) {
          u32 e0 = 0, t0 = 0;
          if (lane == 0) {
            if (be) e0 = seg_e ? e_next : atomicAdd(&ctrl->nE, (u32)__popc(be));
            if (bt && !seg_e) t0 = atomicAdd(&ctrl->nT, (u32)__popc(bt));
          }
          e_next += __popc(be);
          e0 = __shfl_sync(FULL, e0, 0);
          t0 = seg_e ? t_next : __shfl_sync(FULL, t0, 0);
          if (cls == CLS_E) {
            const u32 e = e0 + __popc(be & lt);
            if (e < a.cap_e) {
              a.e_sid[e] = sid[u];
              a.e_epos[e] = ~0ull;  // k5_emit may skip this record's tile: then K5b must place nothing
            }
            x |= e << 4;
          } else if (seg_e && ((btc >> lane) & 1u)) {
            const u32 t = t0 + __popc(btc & lt);
            a.t_sid[t] = cls == CLS_T ? sid[u] : 0xffffffffu;  // a C entry leaves a hole
            a.t_cnt[t] = 0;
            if (cls == CLS_T) x |= t << 4;
          } else if (!seg_e && cls == CLS_T) {
            const u32 t = t0 + __popc(bt & lt);
            a.t_sid[t] = sid[u];
            a.t_cnt[t] = 0;
            x |= t << 4;
          }
          if (seg_e) {
            t_next += __popc(btc);
            t_true += __popc(bt);
          }
        }
        if (valid) a.rec.r[o0 + j] = make_uint4(sid[u], d1[u], m[u], x);
        if (!keep) continue;
        st_cand++;
        dmax = max(dmax, d1[u]);
        if (fq) st_fq++; else st_pq++;
        if (cls == CLS_A) st_a++;
        if (cls == CLS_A || cls == CLS_E) gt_rec = max(gt_rec, o0 + j + 1);
      }
    }
    if (t_true && lane == 0) atomicAdd(&ctrl->nT, t_true);
  }
  ull v[4] = {st_cand, st_fq, st_pq, st_a};
#pragma unroll
  for (int i = 0; i < 4; i++) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v[i] += __shfl_xor_sync(FULL, v[i], o);
    if (lane == 0) s_stat[i][warp] = v[i];
  }
  dmax = __reduce_max_sync(FULL, dmax);
#pragma unroll
  for (int o = 16; o; o >>= 1) gt_rec = max(gt_rec, (u64)__shfl_xor_sync(FULL, (ull)gt_rec, o));
  if (lane == 0) {
    if (dmax) atomicMax(&ctrl->maxkey, dmax);
    if (gt_rec) atomicMax(&ctrl->gt_rec_end, (ull)gt_rec);
  }
  __syncthreads();
  if (tid == 0) {
    ull t[4] = {0, 0, 0, 0};
    for (int w = 0; w < 8; w++)
      for (int i = 0; i < 4; i++) t[i] += s_stat[i][w];
    // truncated superset (tie-heavy call): pass 3 counted these over all of D
    const bool counted = ld_volatile_u32(&ctrl->trunc) != 0;
    if (t[0] && !counted) atomicAdd((ull*)&ctrl->res.candidate_subranges, t[0]);
    if (t[1] && !counted) atomicAdd((ull*)&ctrl->res.fully_qualified, t[1]);
    if (t[2] && !counted) atomicAdd((ull*)&ctrl->res.partially_qualified, t[2]);
    if (t[3]) atomicAdd(&ctrl->nA, t[3]);
  }
}

// ---------------------------------------------------------------------------
struct K4Args {
  const u32* keys;
  u64 n;
  int alpha;
  Ctrl* ctrl;
  const u32* e_sid;
  u32* stg_key;  // [nE * W]: per part, keys > theta from the front
  u64* stg_idx;  // [nE * W]: indices > theta from the front, ties from the back
  u32* seg_gt;   // [nE * parts]
  u32* seg_eq;
  u64 cap_e;     // capacity of nE
};

// K4: read the E candidates.  A tile is 8192 keys: 8192 / W whole candidates,
// or one part of a candidate when W > 8192.  Ranks inside each segment come
// from a tile-wide exclusive scan minus the scan value at the segment start.
#ifndef DTOPK_K4_BIG_KEYS
#define DTOPK_K4_BIG_KEYS (1ull << 21)
#endif
// BIG: the instantiation for calls that re-read more than DTOPK_K4_BIG_KEYS keys
// (ascending input: 8.4 M), register-capped for 3 CTAs per SM; the uncapped one
// serves the rest (capping it slowed small k).  Both are launched; each exits
// at once when the other one owns the call.
template <int MODE, int BIG>
__global__ void __launch_bounds__(256, BIG ? 3 : 2) k4_read(K4Args a) {
  pdl_trigger();
  pdl_wait();
  if (ld_volatile_u32(&a.ctrl->small_done)) return;  // finished by fast_tail
  if (((u64)min((u64)ld_volatile_u32(&a.ctrl->nE), a.cap_e) << a.alpha >= DTOPK_K4_BIG_KEYS) != (BIG != 0)) return;
  __shared__ u32 s_wg[8], s_we[8];
  __shared__ u32 s_seg_g[K4_TILE / 4], s_seg_e[K4_TILE / 4];
  __shared__ u32 s_max[8];
  __shared__ ull s_stat[3][8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  Ctrl* ctrl = a.ctrl;
  const u32 theta = ctrl->res.theta;
  // pool floor (K4h): keys above theta but below it cannot reach the answer;
  // they are only counted (|C| stays exact), not staged
  const u32 pf = ld_volatile_u32(&ctrl->pfloor);
  ull st_lo = 0;
  const u64 nE = min((u64)ctrl->nE, a.cap_e);
  const int alpha = a.alpha;
  const u64 W = 1ull << alpha;
  const int lseg = alpha < 13 ? alpha : 13;  // log2 of the segment length
  const u64 seglen = 1ull << lseg;
  const u64 ppc = W >> lseg;  // parts per candidate
  const u64 total = nE * W;
  const u64 T = (total + K4_TILE - 1) / K4_TILE;
  u32 bmax = 0;
  ull st_gt = 0, st_read = 0;
  const u32 lt = lanemask_lt();
  if (alpha < 2) {
    // W == 2: one thread per candidate, both keys in index order
    for (u64 e = (u64)blockIdx.x * 256 + tid; e < nE; e += (u64)gridDim.x * 256) {
      const u64 b = (u64)a.e_sid[e] << 1;
      u32 g = 0, q = 0;
      for (u64 c = 0; c < 2 && b + c < a.n; c++) {
        const u32 key = to_key<MODE>(a.keys[b + c]);
        st_read++;
        if (key > theta && key >= pf) {
          a.stg_key[2 * e + g] = key;
          a.stg_idx[2 * e + g] = b + c;
          g++;
          bmax = max(bmax, key);
        } else if (key == theta) {
          a.stg_idx[2 * e + 1 - q] = b + c;
          q++;
        } else if (key > theta) {
          st_lo++;
        }
      }
      a.seg_gt[e] = g;
      a.seg_eq[e] = q;
      st_gt += g;
    }
  }
  for (u64 tile = blockIdx.x; alpha >= 2 && tile < T; tile += gridDim.x) {
    u32 kv[8][4];
    u32 vm[8];
    u32 cg = 0, ce = 0;
#pragma unroll
    for (int j = 0; j < 8; j++) {
      const u64 v0 = tile * K4_TILE + (u64)warp * 1024 + (u64)j * 128 + (u64)lane * 4;
      u32 valid = 0;
      u32 x[4] = {0u, 0u, 0u, 0u};
      if (v0 < total) {
        const u64 e = v0 >> alpha;
        const u64 phys = ((u64)a.e_sid[e] << alpha) | (v0 & (W - 1));
        if (alpha >= 2 && phys + 4 <= a.n) {
          const uint4 q = ld_nc_v4(a.keys + phys);
          x[0] = to_key<MODE>(q.x);
          x[1] = to_key<MODE>(q.y);
          x[2] = to_key<MODE>(q.z);
          x[3] = to_key<MODE>(q.w);
          valid = 0xfu;
        } else {
#pragma unroll
          for (int c = 0; c < 4; c++) {
            const u64 vc = v0 + c;
            const u64 pc = ((u64)a.e_sid[vc >> alpha] << alpha) | (vc & (W - 1));
            if (vc < total && pc < a.n) {
              x[c] = to_key<MODE>(a.keys[pc]);
              valid |= 1u << c;
            }
          }
        }
      }
#pragma unroll
      for (int c = 0; c < 4; c++) {
        const bool vv = (valid >> c) & 1u;
        const bool g = vv && x[c] > theta && x[c] >= pf;
        st_lo += vv && x[c] > theta && x[c] < pf;
        cg += g;
        ce += vv && x[c] == theta;
        if (g) bmax = max(bmax, x[c]);
        kv[j][c] = x[c];
      }
      vm[j] = valid;
      st_read += __popc(valid);
    }
    const u32 wg = __reduce_add_sync(FULL, cg), we = __reduce_add_sync(FULL, ce);
    if (lane == 0) {
      s_wg[warp] = wg;
      s_we[warp] = we;
    }
    st_gt += cg;
    __syncthreads();
    u32 gbase = 0, ebase = 0;
    for (int w = 0; w < warp; w++) {
      gbase += s_wg[w];
      ebase += s_we[w];
    }
    // pass A: tile-exclusive scan value of every uint4; segment starts to smem
    u32 gx[8], ex[8];
    {
      u32 gr = gbase, er = ebase;
#pragma unroll
      for (int j = 0; j < 8; j++) {
        u32 ng = 0, ne = 0, bg = 0, be = 0;
#pragma unroll
        for (int c = 0; c < 4; c++) {
          const bool vv = (vm[j] >> c) & 1u;
          const u32 b1 = __ballot_sync(FULL, vv && kv[j][c] > theta && kv[j][c] >= pf);
          const u32 b2 = __ballot_sync(FULL, vv && kv[j][c] == theta);
          bg += __popc(b1 & lt);
          be += __popc(b2 & lt);
          ng += __popc(b1);
          ne += __popc(b2);
        }
        gx[j] = gr + bg;
        ex[j] = er + be;
        const u32 local = (u32)warp * 1024 + (u32)j * 128 + (u32)lane * 4;  // tile-local offset
        if ((local & (seglen - 1)) == 0) {
          s_seg_g[local >> lseg] = gx[j];
          s_seg_e[local >> lseg] = ex[j];
        }
        gr += ng;
        er += ne;
      }
    }
    __syncthreads();
    // pass B: write each element at its rank inside its segment
#pragma unroll
    for (int j = 0; j < 8; j++) {
      const u64 v0 = tile * K4_TILE + (u64)warp * 1024 + (u64)j * 128 + (u64)lane * 4;
      if (v0 >= total) continue;
      const u32 local = (u32)warp * 1024 + (u32)j * 128 + (u32)lane * 4;
      const u32 sg = s_seg_g[local >> lseg], se = s_seg_e[local >> lseg];
      u32 rg = gx[j] - sg, re = ex[j] - se;
      const u64 segid = v0 >> lseg;  // global segment = e * ppc + part
      const u64 sbase = segid << lseg;
#pragma unroll
      for (int c = 0; c < 4; c++) {
        if (!((vm[j] >> c) & 1u)) continue;
        const u64 vc = v0 + c;
        const u32 key = kv[j][c];
        if (key > theta && key >= pf) {
          const u64 phys = ((u64)a.e_sid[vc >> alpha] << alpha) | (vc & (W - 1));
          a.stg_key[sbase + rg] = key;
          a.stg_idx[sbase + rg] = phys;
          rg++;
        } else if (key == theta) {
          const u64 phys = ((u64)a.e_sid[vc >> alpha] << alpha) | (vc & (W - 1));
          a.stg_idx[sbase + seglen - 1 - re] = phys;
          re++;
        }
      }
      // the thread holding the segment's last uint4 writes the counts
      if (((local + 4) & (seglen - 1)) == 0) {
        a.seg_gt[segid] = rg;
        a.seg_eq[segid] = re;
      }
    }
    (void)ppc;
    __syncthreads();
  }
  // totals
  bmax = __reduce_max_sync(FULL, bmax);
  if (lane == 0) s_max[warp] = bmax;
  st_gt = __reduce_add_sync(FULL, (u32)min(st_gt, (ull)0xffffffffu));
  ull v[2] = {0, st_read};
#pragma unroll
  for (int i = 0; i < 2; i++) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v[i] += __shfl_xor_sync(FULL, v[i], o);
    if (lane == 0) s_stat[i][warp] = v[i];
  }
  __syncthreads();
  if (tid == 0) {
    u32 m = 0;
    ull rd = 0;
    for (int w = 0; w < 8; w++) {
      m = max(m, s_max[w]);
      rd += s_stat[1][w];
    }
    if (m) atomicMax(&ctrl->maxkey, m);
    if (rd) atomicAdd((ull*)&ctrl->res.elements_reread, rd);
  }
  if (lane == 0 && st_gt) atomicAdd(&ctrl->sumEgt, st_gt);
  st_lo = __reduce_add_sync(FULL, (u32)min(st_lo, (ull)0xffffffffu));
  if (lane == 0 && st_lo) atomicAdd(&ctrl->below_floor, st_lo);
}

// K4T: count the ties of T candidates (d_1 == theta, max not unique,
// subrange not constant).  Few T candidates: count them all in parallel (one
// warp each).  Many (tie-heavy inputs): walk the records in index order, 32
// per warp and 8 warps per ticket, and stop taking tickets once the completed
// chunks already hold k ties -- every later tie lands beyond position k, so
// its count is never needed (it stays 0; concatenated_len is then a lower
// bound, flagged through concat_skipped_fq).
constexpr u32 K4T_PARALLEL_MAX = 65536;  // T candidates counted all at once (truncated tie-heavy calls stay below: <= ~k / 2)
constexpr u32 K4T_CHUNKS_PER_TICKET = 8;  // 32-record chunks (one per warp) per ticket

template <int MODE>
__device__ __forceinline__ u32 count_ties_warp(const u32* __restrict__ keys, u64 n, int alpha, u64 sid, u32 theta) {
  const int lane = threadIdx.x & 31;
  const u64 b = sid << alpha;
  const u64 len = min((u64)(1ull << alpha), (u64)(n - b));
  u32 c = 0;
  for (u64 e = lane; e < len; e += 32) c += to_key<MODE>(keys[b + e]) == theta;
  return __reduce_add_sync(FULL, c);
}

// K4h: the pool floor for calls that re-read many E keys (ascending input:
// 8.4 M keys above theta for k = 2^16).  An exact histogram of the pool's keys
// -- the E candidates' keys above theta plus the A records' single keys -- in
// PF_BINS linear bins over (theta, maxkey]; the last CTA takes the lower edge
// of the bin holding the k-th largest as `pfloor`.  At least k pool keys are
// >= pfloor, so the answer lies above it: K4 stages only those (the rest is
// counted for |C|), and P_gt shrinks to ~k + one bin, skipping the staging /
// copy / select over millions of keys.  Exits at once for small re-reads.
constexpr int PF_BINS = 2048;
#ifndef DTOPK_PF_MIN_KEYS
#define DTOPK_PF_MIN_KEYS (1ull << 21)
#endif

template <int MODE>
__global__ void __launch_bounds__(256) k4h_floor(K4Args a, const uint4* __restrict__ rec, u64 k) {
  pdl_trigger();
  pdl_wait();
  Ctrl* ctrl = a.ctrl;
  if (ld_volatile_u32(&ctrl->small_done)) return;
  const u64 nE = min((u64)ld_volatile_u32(&ctrl->nE), a.cap_e);
  const int alpha = a.alpha;
  const u64 total = nE << alpha;
  if (alpha < 2 || total < max((u64)DTOPK_PF_MIN_KEYS, 8 * k)) return;  // pfloor stays 0
  __shared__ u32 sh[PF_BINS];
  __shared__ ull scratch[8];
  __shared__ int am_last;
  const int tid = threadIdx.x;
  for (int i = tid; i < PF_BINS; i += 256) sh[i] = 0;
  __syncthreads();
  const u32 theta = ctrl->res.theta;
  const u32 mx = ld_volatile_u32(&ctrl->maxkey);
  if (mx <= theta) return;  // nothing above theta
  const u64 range = (u64)(mx - theta);  // keys theta+1 .. mx
  const u64 W = 1ull << alpha;
  // E candidates: 4 uint4 per thread and step, their subrange-id and key loads in
  // flight together (a uint4 never straddles a subrange)
  const u64 nq = total / 4;
  const u64 stride = (u64)gridDim.x * 256;
  for (u64 q0 = (u64)blockIdx.x * 256 + tid; q0 < nq; q0 += 4 * stride) {
    u64 phys[4];
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const u64 v0 = (q0 + u * stride) * 4;
      phys[u] = q0 + u * stride < nq ? (((u64)a.e_sid[v0 >> alpha] << alpha) | (v0 & (W - 1))) : ~0ull;
    }
    u32 xs[4][4];
#pragma unroll
    for (int u = 0; u < 4; u++) {
      if (phys[u] != ~0ull && phys[u] + 4 <= a.n) {
        const uint4 v = ld_nc_v4(a.keys + phys[u]);
        xs[u][0] = to_key<MODE>(v.x);
        xs[u][1] = to_key<MODE>(v.y);
        xs[u][2] = to_key<MODE>(v.z);
        xs[u][3] = to_key<MODE>(v.w);
      } else {
#pragma unroll
        for (int c = 0; c < 4; c++)
          xs[u][c] = phys[u] != ~0ull && phys[u] + c < a.n ? to_key<MODE>(a.keys[phys[u] + c]) : 0u;
      }
    }
#pragma unroll
    for (int u = 0; u < 4; u++) {
      // sorted / narrow inputs put a thread's 4 keys and a warp's 128 in one bin:
      // count runs per thread, then one atomic per warp when its bins agree
      u32 bin = 0xffffffffu, cnt = 0;
#pragma unroll
      for (int c = 0; c < 4; c++) {
        const u32 x = xs[u][c];
        if (x <= theta) continue;
        const u32 bb = (u32)(((u64)(x - theta - 1) * PF_BINS) / range);
        if (bb != bin) {
          if (cnt) atomicAdd(&sh[bin], cnt);
          bin = bb;
          cnt = 0;
        }
        cnt++;
      }
      const u32 act = __activemask();
      const u32 b0 = __shfl_sync(act, bin, __ffs(act) - 1);
      if (__all_sync(act, bin == b0)) {
        const u32 tot = __reduce_add_sync(act, cnt);
        if ((int)(threadIdx.x & 31) == __ffs(act) - 1 && tot && bin != 0xffffffffu) atomicAdd(&sh[bin], tot);
      } else if (cnt) {
        atomicAdd(&sh[bin], cnt);
      }
    }
  }
  // A records: their one key above theta (d_1)
  const u64 nrec = ctrl->sup_total;
  for (u64 r = (u64)blockIdx.x * 256 + tid; r < nrec; r += (u64)gridDim.x * 256) {
    const uint4 rc = rec[r];
    if ((rc.w & 7u) == CLS_A && rc.y > theta) atomicAdd(&sh[(u32)(((u64)(rc.y - theta - 1) * PF_BINS) / range)], 1u);
  }
  __syncthreads();
  for (int i = tid; i < PF_BINS; i += 256)
    if (sh[i]) atomicAdd(&ctrl->pf_hist[i], (ull)sh[i]);
  __threadfence();
  __syncthreads();
  if (tid == 0) am_last = atomicAdd(&ctrl->pf_ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  __shared__ DigitResult res;
  find_digit<PF_BINS>(ctrl->pf_hist, k, &res, scratch);  // the bin holding the k-th largest
  if (tid == 0 && res.valid) {
    const u32 lo = theta + 1u + (u32)(((u64)res.digit * range) / PF_BINS);  // <= its smallest key
    ctrl->pfloor = lo;
  }
}

// Ties of one subrange counted by one lane (16-byte loads, 8 in flight): the
// ticketed K4T path runs 32 T records of a chunk in parallel this way instead
// of one warp-wide count after another (which left a ticket ~32 load
// latencies long).
template <int MODE>
__device__ __forceinline__ u32 count_ties_lane(const u32* __restrict__ keys, u64 n, int alpha, u64 sid, u32 theta) {
  const u64 b = sid << alpha;
  const u64 len = min((u64)(1ull << alpha), (u64)(n - b));
  u32 c = 0;
  if (len == (1ull << alpha)) {  // whole subrange: 16-byte aligned (keys is, and alpha >= 2 here)
    const uint4* p = reinterpret_cast<const uint4*>(keys + b);
    const u32 nq = (u32)(len >> 2);
    for (u32 q = 0; q < nq; q += 8) {
      uint4 v[8];
#pragma unroll
      for (int j = 0; j < 8; j++) v[j] = q + j < nq ? __ldg(p + q + j) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
      for (int j = 0; j < 8; j++)
        if (q + j < nq)
          c += (to_key<MODE>(v[j].x) == theta) + (to_key<MODE>(v[j].y) == theta) + (to_key<MODE>(v[j].z) == theta) +
               (to_key<MODE>(v[j].w) == theta);
    }
  } else {
    for (u64 e = 0; e < len; e++) c += to_key<MODE>(keys[b + e]) == theta;
  }
  return c;
}

struct K4TArgs {
  const u32* keys;
  u64 n;
  u64 S;
  int alpha;
  u64 k;
  Ctrl* ctrl;
  const u32* t_sid;
  u32* t_cnt;
  const uint4* rec;
  const u32* seg_eq;
  int exact;  // DTOPK_FLAG_EXACT_STATS: count every T candidate
};

template <int MODE>
__global__ void __launch_bounds__(256) k4t_count(K4TArgs a) {
  pdl_trigger();
  pdl_wait();
  if (ld_volatile_u32(&a.ctrl->small_done)) return;  // finished by fast_tail
  __shared__ u64 s_chunk;
  __shared__ u32 s_eq[8];
  Ctrl* ctrl = a.ctrl;
  const u32 theta = ctrl->res.theta;
  const u64 nT = ctrl->nT;
  if (nT == 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const u64 gw = ((u64)blockIdx.x * 256 + threadIdx.x) >> 5;
  const u64 nw = ((u64)gridDim.x * 256) >> 5;
  if (nT <= K4T_PARALLEL_MAX || a.exact) {
    const u64 nslots = max(nT, (u64)ctrl->nTslots);  // beta 2: slots include C holes
    for (u64 t = gw; t < nslots; t += nw) {
      const u32 sid = a.t_sid[t];
      if (sid == 0xffffffffu) continue;  // hole left by a C entry (K3)
      const u32 c = count_ties_warp<MODE>(a.keys, a.n, a.alpha, sid, theta);
      if (lane == 0) a.t_cnt[t] = c;
    }
    return;
  }
  const u64 total = ctrl->sup_total;
  const u64 nchunks = (total + 31) / 32;  // 32-record chunks, subrange order
  const int lseg = a.alpha < 13 ? a.alpha : 13;
  const u64 ppc = (1ull << a.alpha) >> lseg;
  // Tickets are handed out at most `window` ahead of the completed ones (about
  // 8 MB of T subranges in flight): with the whole grid grabbing tickets at
  // once, the first wave alone re-read ~37x the subranges the first k ties
  // needed on few-distinct input (161 MB instead of ~4 MB at alpha 8).
  const u32 window = max(4u, 1u << max(0, 13 - a.alpha));
  for (;;) {
    if (threadIdx.x == 0) {
      u64 t = ~0ull;
      for (;;) {
        if (*(volatile ull*)&ctrl->k4t_eq_done >= a.k) break;
        const u32 next = ld_volatile_u32(&ctrl->k4t_ticket);
        if ((u64)next * K4T_CHUNKS_PER_TICKET >= nchunks) {
          t = ~1ull;  // every chunk handed out
          break;
        }
        if (next < ld_volatile_u32(&ctrl->k4t_completed) + window) {
          // claim exactly ticket `next` (a plain atomicAdd let every spinning CTA
          // pass the window test at once)
          if (atomicCAS(&ctrl->k4t_ticket, next, next + 1u) == next) {
            t = next;
            break;
          }
          continue;
        }
        __nanosleep(200);
      }
      s_chunk = t;
    }
    __syncthreads();
    const u64 chunk = s_chunk;
    if (chunk == ~0ull) {  // the first k ties are counted: the rest of the T work is skipped
      if (threadIdx.x == 0 && blockIdx.x == 0) atomicAdd((ull*)&ctrl->res.concat_skipped_fq, 1ull);
      break;
    }
    if (chunk == ~1ull || chunk * K4T_CHUNKS_PER_TICKET >= nchunks) break;
#ifdef DTOPK_K4T_DEBUG
    if (threadIdx.x == 0 && chunk % 64 == 0)
      printf("k4t blk %d chunk %llu completed %u eq_done %llu k %llu nchunks %llu window %u\n", blockIdx.x,
             (unsigned long long)chunk, ctrl->k4t_completed, (unsigned long long)ctrl->k4t_eq_done,
             (unsigned long long)a.k, (unsigned long long)nchunks, window);
#endif
    // one 32-record chunk per warp, lane per record: ties of its B/C/E/T records
    u32 eq = 0;
    const u64 c = chunk * K4T_CHUNKS_PER_TICKET + warp;
    if (c < nchunks) {
      const u64 i = c * 32 + lane;
      const uint4 rc = i < total ? a.rec[i] : make_uint4(0u, 0u, 0u, CLS_NONE);
      const u32 cls = rc.w & 7u;
      u64 e = 0;
      if (cls == CLS_B) {
        e = 1;
      } else if (cls == CLS_C) {
        e = sub_len(rc.x, a.n, a.alpha);
      } else if (cls == CLS_E) {
        const u64 ei = rc.w >> 4;
        for (u64 p = 0; p < ppc; p++) e += a.seg_eq[ei * ppc + p];
      }
      u32 bt = __ballot_sync(FULL, cls == CLS_T);
      if (a.alpha >= 2 && a.alpha <= 9) {  // lane-parallel: every T record of the chunk at once
        if (cls == CLS_T) {
          const u32 cn = count_ties_lane<MODE>(a.keys, a.n, a.alpha, rc.x, theta);
          a.t_cnt[rc.w >> 4] = cn;
          e += cn;
        }
        bt = 0;
      }
      while (bt) {
        const int q = __ffs(bt) - 1;
        bt &= bt - 1;
        const u32 sid = __shfl_sync(FULL, rc.x, q);
        const u32 tix = __shfl_sync(FULL, rc.w >> 4, q);
        const u32 cn = count_ties_warp<MODE>(a.keys, a.n, a.alpha, sid, theta);
        if (lane == 0) a.t_cnt[tix] = cn;
        if (lane == q) e += cn;
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) e += __shfl_xor_sync(FULL, (ull)e, o);
      eq = (u32)min(e, (u64)0x7fffffffu);
    }
    if (lane == 0) s_eq[warp] = eq;
    __syncthreads();
    if (threadIdx.x == 0) {
      u64 tot = 0;
      for (int i = 0; i < 8; i++) tot += s_eq[i];
      if (tot) atomicAdd(&ctrl->k4t_eq_done, (ull)min(tot, (u64)0xffffffffull));
      __threadfence();
      atomicAdd(&ctrl->k4t_completed, 1u);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
struct K5Args {
  Ctrl* ctrl;
  Records rec;     // [sup_total] records, subrange order
  u64 n;
  int alpha;
  u64 k;
  const u32* stg_key;
  const u64* stg_idx;
  const u32* seg_gt;
  const u32* seg_eq;
  const u32* t_cnt;  // ties of each T candidate (K4T)
  u32* gt_keys;      // P_gt, index order
  u64* gt_idx;
  u64* ties;         // first k ties, index order
  u32* d_sid;        // K6 work list: subrange, first tie position, ties needed
  u64* d_pos;
  u32* d_need;
  u64* e_gpos;       // per E candidate: first slot in P_gt / in the tie list (K5b copies)
  u64* e_epos;
  u64* tile_g;   // [tiles] keys > theta per record tile (K5a), then its exclusive prefix
  u64* tile_e;   // [tiles] ties per record tile (K5a), then its exclusive prefix
  int exact;         // DTOPK_FLAG_EXACT_STATS: never skip (exact concatenated_len)
};

__device__ __forceinline__ void rec_counts(const K5Args& a, const uint4 rc, u64& g, u64& e, u32 pf) {
  const u32 x = rc.w;
  const u32 cls = x & 7u;
  g = 0;
  e = 0;
  if (cls == CLS_NONE) {
    return;
  } else if (cls == CLS_A) {
    g = rc.y >= pf;  // its one key above theta, unless below the pool floor
  } else if (cls == CLS_B) {
    e = 1;
  } else if (cls == CLS_C) {
    e = sub_len(rc.x, a.n, a.alpha);
  } else if (cls == CLS_T) {
    e = a.t_cnt[x >> 4];
  } else {
    const int lseg = a.alpha < 13 ? a.alpha : 13;
    const u64 ppc = (1ull << a.alpha) >> lseg;
    const u64 eidx = x >> 4;
    for (u64 p = 0; p < ppc; p++) {
      g += a.seg_gt[eidx * ppc + p];
      e += a.seg_eq[eidx * ppc + p];
    }
  }
}

// K5 runs as two kernels over record tiles (K5_RPT consecutive records per
// thread, K5_TILE per tile) -- no serial look-back chain:
//   k5_count  per-tile (keys > theta, ties) counts; the last CTA turns them
//             into exclusive prefixes and publishes |P_gt|, the path, k_out
//   k5_emit   per tile, block scans on top of the tile prefix -> positions in
//             P_gt (index order) and in the first-k tie list
template <bool EMIT>
__device__ __forceinline__ void k5_tile_counts(const K5Args& a, u64 i0, u64 total, uint4 (&rcs)[K5_RPT],
                                               u64 (&cg)[K5_RPT], u64 (&ce)[K5_RPT], u64& tg, u64& te, u32 pf) {
  tg = te = 0;
#pragma unroll
  for (int r = 0; r < K5_RPT; r++)
    rcs[r] = i0 + r < total ? a.rec.r[i0 + r] : make_uint4(0u, 0u, 0u, CLS_NONE);
#pragma unroll
  for (int r = 0; r < K5_RPT; r++) {
    rec_counts(a, rcs[r], cg[r], ce[r], pf);
    tg += cg[r];
    te += ce[r];
  }
}

__global__ void __launch_bounds__(256) k5_count(K5Args a) {
  pdl_trigger();
  pdl_wait();
  if (ld_volatile_u32(&a.ctrl->small_done)) return;  // finished by fast_tail
  __shared__ u64 scratch_g[8], scratch_e[8];
  __shared__ ull s_cc[8];
  __shared__ int am_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  Ctrl* ctrl = a.ctrl;
  const u64 total = ctrl->sup_total;
  const u64 T = max((u64)1, (total + K5_TILE - 1) / K5_TILE);
  const u32 pf = ld_volatile_u32(&ctrl->pfloor);
  ull st_concat = 0;
  for (u64 tile = blockIdx.x; tile < T; tile += gridDim.x) {
    uint4 rcs[K5_RPT];
    u64 cg[K5_RPT], ce[K5_RPT], tg, te;
    k5_tile_counts<false>(a, tile * K5_TILE + (u64)tid * K5_RPT, total, rcs, cg, ce, tg, te, pf);
#pragma unroll
    for (int r = 0; r < K5_RPT; r++) {
      const u32 x = rcs[r].w, cls = x & 7u;
      if (((x >> 3) & 1u) && (cls == CLS_C || cls == CLS_T || cls == CLS_E)) st_concat += cg[r] + ce[r];
    }
    const u64 ig = block_incl_scan_256<u64>(tg, scratch_g);
    const u64 ie = block_incl_scan_256<u64>(te, scratch_e);
    if (tid == 255) {
      a.tile_g[tile] = ig;
      a.tile_e[tile] = ie;
    }
  }
  for (int o = 16; o; o >>= 1) st_concat += __shfl_xor_sync(FULL, st_concat, o);
  if (lane == 0) s_cc[warp] = st_concat;
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    ull t = 0;
    for (int w = 0; w < 8; w++) t += s_cc[w];
    if (t) atomicAdd((ull*)&ctrl->res.concatenated_len, t);
    am_last = atomicAdd(&ctrl->k5_ticket, 1u) == gridDim.x - 1;
    // E keys above theta left out of the pool by the floor still count in |C|
    // (every E record is fully qualified when the floor is used: beta <= 2)
    if (am_last && ld_volatile_u32(&ctrl->pfloor)) atomicAdd((ull*)&ctrl->res.concatenated_len, ctrl->below_floor);
  }
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  // exclusive prefixes of the tile counts (T <= S / K5_TILE), in place; blocks of
  // 8 tiles per thread and step so the loads of a step are in flight together
  const u64 per = (T + 255) / 256;
  u64 sg = 0, se = 0;
  for (u64 q0 = 0; q0 < per; q0 += 8) {
#pragma unroll
    for (int q = 0; q < 8; q++) {
      const u64 t = (u64)tid * per + q0 + q;
      if (q0 + q < per && t < T) {
        sg += __ldcg(&a.tile_g[t]);
        se += __ldcg(&a.tile_e[t]);
      }
    }
  }
  const u64 xg = block_incl_scan_256<u64>(sg, scratch_g);
  const u64 xe = block_incl_scan_256<u64>(se, scratch_e);
  u64 rg = xg - sg, re = xe - se;
  for (u64 q0 = 0; q0 < per; q0 += 8) {
    u64 g[8], e[8];
#pragma unroll
    for (int q = 0; q < 8; q++) {
      const u64 t = (u64)tid * per + q0 + q;
      const bool in = q0 + q < per && t < T;
      g[q] = in ? __ldcg(&a.tile_g[t]) : 0;
      e[q] = in ? __ldcg(&a.tile_e[t]) : 0;
    }
#pragma unroll
    for (int q = 0; q < 8; q++) {
      const u64 t = (u64)tid * per + q0 + q;
      if (q0 + q < per && t < T) {
        a.tile_g[t] = rg;
        a.tile_e[t] = re;
      }
      rg += g[q];
      re += e[q];
    }
  }
  if (tid == 255) {
    const u64 G = xg, E = xe;
    const u32 theta = ctrl->res.theta;
    ctrl->res.pool_gt = G;
    ctrl->res.pool_eq = min(E, a.k);
    if (G >= a.k) {
      ctrl->res.path = PATH_SELECT;
      ctrl->res.k_out = a.k;
    } else {
      ctrl->res.path = PATH_MERGE;
      ctrl->res.k_out = min(a.k, G + E);
      ctrl->sort_lo = theta;
      atomicMax(&ctrl->maxkey, theta);
    }
  }
}

__global__ void __launch_bounds__(256, DTOPK_K5E_MINB) k5_emit(K5Args a) {
  pdl_trigger();
  pdl_wait();
  if (ld_volatile_u32(&a.ctrl->small_done)) return;  // finished by fast_tail
  __shared__ u64 scratch_g[8], scratch_e[8];
  const int tid = threadIdx.x;
  Ctrl* ctrl = a.ctrl;
  const u64 total = ctrl->sup_total;
  const u64 T = max((u64)1, (total + K5_TILE - 1) / K5_TILE);
  const u64 G = ctrl->res.pool_gt;
  const u32 pf = ld_volatile_u32(&ctrl->pfloor);
  for (u64 tile = blockIdx.x; tile < T; tile += gridDim.x) {
    const u64 gx = a.tile_g[tile], ex = a.tile_e[tile];
    const u64 gnext = tile + 1 < T ? a.tile_g[tile + 1] : G;
    if (gnext == gx && ex >= a.k) continue;  // no key > theta and every tie beyond position k
    uint4 rcs[K5_RPT];
    u64 cg[K5_RPT], ce[K5_RPT], tg, te;
    k5_tile_counts<true>(a, tile * K5_TILE + (u64)tid * K5_RPT, total, rcs, cg, ce, tg, te, pf);
    const u64 ig = block_incl_scan_256<u64>(tg, scratch_g);
    const u64 ie = block_incl_scan_256<u64>(te, scratch_e);
    u64 gpos = gx + ig - tg, epos = ex + ie - te;
#pragma unroll
    for (int r = 0; r < K5_RPT; r++) {
      const uint4 rc = rcs[r];
      const u32 x = rc.w;
      const u32 cls = x & 7u;
      const u64 sid = rc.x;
      const u64 base = sid << a.alpha;
      if (cls == CLS_A && cg[r]) {
        a.gt_keys[gpos] = rc.y;
        a.gt_idx[gpos] = base + meta_p1(rc.z);
      } else if (cls == CLS_B) {
        if (epos < a.k) a.ties[epos] = base + meta_p1(rc.z);
      } else if (cls == CLS_C) {
        if (epos < a.k) {  // a run of ties: K6 writes it (one warp per run)
          const u32 wslot = atomicAdd(&ctrl->k6_count, 1u);
          a.d_sid[wslot] = (u32)sid;
          a.d_pos[wslot] = epos;
          a.d_need[wslot] = (u32)min(ce[r], a.k - epos) | 0x80000000u;
        }
      } else if (cls == CLS_T) {
        if (epos < a.k && ce[r]) {
          const u32 wslot = atomicAdd(&ctrl->k6_count, 1u);
          a.d_sid[wslot] = (u32)sid;
          a.d_pos[wslot] = epos;
          a.d_need[wslot] = (u32)min(ce[r], a.k - epos);
        }
      } else if (cls == CLS_E) {
        // the staged keys of E candidates are copied in parallel by K5b
        const u64 eidx = x >> 4;
        a.e_gpos[eidx] = gpos;
        a.e_epos[eidx] = epos;
      }
      gpos += cg[r];
      epos += ce[r];
    }
  }
}

// K5b: copy the staged keys > theta and ties of every E candidate part to
// its place in P_gt / the tie list (one warp per part).
__global__ void __launch_bounds__(256) k5b_copy(Ctrl* ctrl, int alpha, u64 k, const u32* __restrict__ stg_key,
                                                const u64* __restrict__ stg_idx, const u32* __restrict__ seg_gt,
                                                const u32* __restrict__ seg_eq, const u64* __restrict__ e_gpos,
                                                const u64* __restrict__ e_epos, u64 cap_e, u32* __restrict__ gt_keys,
                                                u64* __restrict__ gt_idx, u64* __restrict__ ties) {
  pdl_trigger();
  pdl_wait();
  if (ld_volatile_u32(&ctrl->small_done)) return;  // finished by fast_tail
  const int lane = threadIdx.x & 31;
  const u64 nE = min((u64)ctrl->nE, cap_e);
  const int lseg = alpha < 13 ? alpha : 13;
  const u64 seglen = 1ull << lseg;
  const u64 ppc = (1ull << alpha) >> lseg;
  if (alpha <= 6) {
    // small subranges (<= 64 keys, a few staged keys each at large k): one E
    // candidate per thread, so the count / offset loads of 32 candidates are in
    // flight per warp instead of one (k = 2^20: 31 k candidates, ~2 keys each).
    // Not for larger subranges: a candidate can stage all of its keys (ascending
    // input at alpha 8: 256 per candidate, 1.09 vs 0.90 ms copied one by one)
    for (u64 e = (u64)blockIdx.x * 256 + threadIdx.x; e < nE; e += (u64)gridDim.x * 256) {
      const u64 eo = e_epos[e];
      if (eo == ~0ull) continue;
      const u64 go = e_gpos[e];
      const u32 ng = seg_gt[e], ne = seg_eq[e];
      const u64 sb = e << lseg;
      for (u32 z = 0; z < ng; z++) {
        gt_keys[go + z] = stg_key[sb + z];
        gt_idx[go + z] = stg_idx[sb + z];
      }
      for (u32 z = 0; z < ne && eo + z < k; z++) ties[eo + z] = stg_idx[sb + seglen - 1 - z];
    }
    return;
  }
  const u64 gw = ((u64)blockIdx.x * 256 + threadIdx.x) >> 5;
  const u64 nw = ((u64)gridDim.x * 256) >> 5;
  for (u64 sg = gw; sg < nE * ppc; sg += nw) {
    const u64 e = sg / ppc, part = sg - e * ppc;
    // e_epos == ~0: k5_emit skipped this record's tile (no key > theta in it, every tie beyond k)
    const u64 eo0 = e_epos[e];
    if (eo0 == ~0ull) continue;
    u64 go = e_gpos[e], eo = eo0;
    for (u64 p = 0; p < part; p++) {
      go += seg_gt[e * ppc + p];
      eo += seg_eq[e * ppc + p];
    }
    const u32 ng = seg_gt[sg], ne = seg_eq[sg];
    const u64 sb = sg << lseg;
    // 8 rounds of loads in flight before their stores (the plain loop kept one)
    for (u32 z0 = 0; z0 < ng; z0 += 256) {
      u32 kk[8];
      u64 ii[8];
#pragma unroll
      for (int u = 0; u < 8; u++) {
        const u32 z = z0 + u * 32 + lane;
        if (z < ng) {
          kk[u] = stg_key[sb + z];
          ii[u] = stg_idx[sb + z];
        }
      }
#pragma unroll
      for (int u = 0; u < 8; u++) {
        const u32 z = z0 + u * 32 + lane;
        if (z < ng) {
          gt_keys[go + z] = kk[u];
          gt_idx[go + z] = ii[u];
        }
      }
    }
    for (u32 z = lane; z < ne && eo + z < k; z += 32) ties[eo + z] = stg_idx[sb + seglen - 1 - z];
  }
}

// K6: locate the ties of class-D records that fall among the first k ties
// (one warp per record; ballot-ordered within the subrange).
template <int MODE>
__global__ void __launch_bounds__(256) k6_ties(Ctrl* ctrl, const u32* __restrict__ keys, u64 n, int alpha,
                                               const u32* __restrict__ d_sid, const u64* __restrict__ d_pos,
                                               const u32* __restrict__ d_need, u64* __restrict__ ties) {
  pdl_trigger();
  pdl_wait();
  if (ld_volatile_u32(&ctrl->small_done)) return;  // finished by fast_tail
  const int lane = threadIdx.x & 31;
  const u32 theta = ctrl->res.theta;
  const u32 cnt = ctrl->k6_count;
  const u64 gw = ((u64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const u64 nw = ((u64)gridDim.x * blockDim.x) >> 5;
  const u32 lt = lanemask_lt();
  for (u64 w = gw; w < cnt; w += nw) {
    const u64 base = (u64)d_sid[w] << alpha;
    const u64 len = sub_len(base >> alpha, n, alpha);
    const u64 pos0 = d_pos[w];
    const u32 need = d_need[w] & 0x7fffffffu;
    if (d_need[w] >> 31) {  // constant subrange: its first `need` positions
      for (u32 z = lane; z < need; z += 32) ties[pos0 + z] = base + z;
      continue;
    }
    u32 found = 0;
    for (u64 off = 0; off < len && found < need; off += 32) {
      const u64 e = off + lane;
      const bool t = e < len && to_key<MODE>(keys[base + e]) == theta;
      const u32 b = __ballot_sync(FULL, t);
      const u32 r = found + __popc(b & lt);
      if (t && r < need) ties[pos0 + r] = base + e;
      found += __popc(b);
    }
  }
}

// Bitonic sort (ascending) of R*T u64 values held by a T-thread block as
// v[j] = element j*T + threadIdx.x: strides < 32 exchange through shuffles,
// strides of 32..T/2 through shared memory, strides >= T stay in the thread.
template <int R, int T>
__device__ __forceinline__ void bitonic_block(unsigned long long (&v)[R], unsigned long long* sm) {
  const u32 tid = threadIdx.x;
  constexpr u32 NP = R * T;
  for (u32 size = 2; size <= NP; size <<= 1) {
    // strides >= T: both elements live in this thread (compile-time slots)
#pragma unroll
    for (int js = R / 2; js >= 1; js >>= 1) {
      if ((u32)js * (u32)T <= (size >> 1)) {
#pragma unroll
        for (int j = 0; j < R; j++) {
          if ((j & js) == 0) {
            const u32 i = (u32)j * (u32)T + tid;
            const bool up = (i & size) == 0;
            const unsigned long long x = v[j], y = v[j | js];
            const bool sw = (x > y) == up;
            v[j] = sw ? y : x;
            v[j | js] = sw ? x : y;
          }
        }
      }
    }
    for (u32 stride = min(size >> 1, (u32)T / 2); stride > 0; stride >>= 1) {
      if (stride >= 32) {
#pragma unroll
        for (int j = 0; j < R; j++) sm[j * T + tid] = v[j];
        __syncthreads();
#pragma unroll
        for (int j = 0; j < R; j++) {
          const u32 i = (u32)j * (u32)T + tid;
          const unsigned long long p = sm[i ^ stride];
          const bool keep_min = ((i & stride) == 0) == ((i & size) == 0);
          v[j] = keep_min ? min(v[j], p) : max(v[j], p);
        }
        __syncthreads();
      } else {
#pragma unroll
        for (int j = 0; j < R; j++) {
          const u32 i = (u32)j * (u32)T + tid;
          const unsigned long long p = __shfl_xor_sync(FULL, v[j], (int)stride);
          const bool keep_min = ((i & stride) == 0) == ((i & size) == 0);
          v[j] = keep_min ? min(v[j], p) : max(v[j], p);
        }
      }
    }
  }
}

template <int R>
__device__ __forceinline__ void bitonic_1024(unsigned long long (&v)[R], unsigned long long* sm) {
  bitonic_block<R, 1024>(v, sm);
}

template <int MODE, int R>
__device__ __forceinline__ void finish_small_r(Ctrl* ctrl, u64 m, u64 ko, u64 G, u32 theta, u32 hi,
                                               const u32* __restrict__ gt_keys, const u64* __restrict__ gt_idx,
                                               const u64* __restrict__ ties, u32* __restrict__ ov,
                                               long long* __restrict__ oi, long long offset,
                                               unsigned long long* sm) {
  unsigned long long v[R];
#pragma unroll
  for (int j = 0; j < R; j++) {
    const u32 i = (u32)j * 1024u + threadIdx.x;
    v[j] = ~0ull;
    if (i < m) {
      const u32 key = i < G ? gt_keys[i] : theta;
      v[j] = ((unsigned long long)(hi - key) << 32) | i;
    }
  }
  bitonic_1024<R>(v, sm);
#pragma unroll
  for (int j = 0; j < R; j++) {
    const u32 i = (u32)j * 1024u + threadIdx.x;
    if (i < ko) {
      const u32 pos = (u32)(v[j] & 0xffffffffu);
      const u32 key = hi - (u32)(v[j] >> 32);
      ov[i] = from_key<MODE>(key);
      oi[i] = (long long)(pos < G ? gt_idx[pos] : ties[pos - G]) + offset;
      if (i == ko - 1) ctrl->res.kth_key = key;
    }
  }
}

// Pools of 2049..SMALL_POOL pairs: one CTA, stable LSD radix sort (CUB block
// primitive, 1024 threads x 8 items in shared memory) of d = hi - key over
// only the bits d can occupy, with the pool position as the value.  The input
// is in position order, so stability yields (key desc, position asc).
// Padding slots (>= m) carry the largest d and come last by stability.
template <int MODE, int ITEMS>
__device__ __forceinline__ void finish_small_radix(Ctrl* ctrl, u64 m, u64 ko, u64 G, u32 theta, u32 hi,
                                                   const u32* __restrict__ gt_keys, const u64* __restrict__ gt_idx,
                                                   const u64* __restrict__ ties, u32* __restrict__ ov,
                                                   long long* __restrict__ oi, long long offset, void* smem) {
  typedef cub::BlockRadixSort<u32, 1024, ITEMS, u32> Sorter;
  static_assert(sizeof(typename Sorter::TempStorage) <= SMALL_POOL * 8, "finish_small shared memory");
  const u32 range = hi - theta;
  const int nbits = range ? 32 - __clz(range) : 0;
  const u32 pad = nbits >= 32 ? 0xffffffffu : ((1u << nbits) - 1u);
  u32 d[ITEMS], pos[ITEMS];
#pragma unroll
  for (int j = 0; j < ITEMS; j++) {
    const u32 i = threadIdx.x * (u32)ITEMS + (u32)j;
    pos[j] = i;
    d[j] = pad;
    if (i < m) d[j] = hi - (i < G ? gt_keys[i] : theta);
  }
  if (nbits) Sorter(*reinterpret_cast<typename Sorter::TempStorage*>(smem)).Sort(d, pos, 0, nbits);
#pragma unroll
  for (int j = 0; j < ITEMS; j++) {
    const u32 r = threadIdx.x * (u32)ITEMS + (u32)j;
    if (r < ko) {
      const u32 key = hi - d[j];
      ov[r] = from_key<MODE>(key);
      oi[r] = (long long)(pos[j] < G ? gt_idx[pos[j]] : ties[pos[j] - G]) + offset;
      if (r == ko - 1) ctrl->res.kth_key = key;
    }
  }
}

// Fused finish for pools of at most SMALL_POOL pairs: one CTA sorts the pool
// (P_gt, plus the ties on the merge path) by (key desc, position asc) and
// writes the first k_out pairs in the input dtype.  Positions follow index
// order, so this is the (key desc, index asc) order of the reference tie rule.
// In a CUDA graph (use_cond != 0) it also sets the conditional that gates the
// large-pool tail, so that tail's kernels are not even launched when unneeded.
template <int MODE>
__global__ void __launch_bounds__(1024) finish_small(Ctrl* ctrl, const u32* __restrict__ gt_keys,
                                                     const u64* __restrict__ gt_idx, const u64* __restrict__ ties,
                                                     u32* __restrict__ ov, long long* __restrict__ oi,
                                                     long long offset, cudaGraphConditionalHandle cond,
                                                     int use_cond) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ unsigned long long sk[];
  if (ld_volatile_u32(&ctrl->small_done)) {  // finished by fast_tail
    if (use_cond && threadIdx.x == 0) cudaGraphSetConditional(cond, 0u);
    return;
  }
  const u32 path = ctrl->res.path;
  const u64 G = ctrl->res.pool_gt;
  const u64 m = path == PATH_SELECT ? G : ctrl->res.k_out;
  if (use_cond && threadIdx.x == 0) cudaGraphSetConditional(cond, m > (u64)SMALL_POOL ? 1u : 0u);
  if (m > (u64)SMALL_POOL || m == 0) return;
  const u64 ko = ctrl->res.k_out;
  const u32 theta = ctrl->res.theta;
  const u32 hi = max(ctrl->maxkey, theta);
  // tiny pools: register/shuffle bitonic; larger: CUB block radix sort over the occupied bits only
  // (the pool of a large-n top-k spans few bits, e.g. ~12 for n = 2^30, k = 1024)
  if (m <= 64)
    finish_small_r<MODE, 1>(ctrl, m, ko, G, theta, hi, gt_keys, gt_idx, ties, ov, oi, offset, sk);
  else if (m <= 1024)
    finish_small_radix<MODE, 1>(ctrl, m, ko, G, theta, hi, gt_keys, gt_idx, ties, ov, oi, offset, sk);
  else if (m <= 2048)
    finish_small_radix<MODE, 2>(ctrl, m, ko, G, theta, hi, gt_keys, gt_idx, ties, ov, oi, offset, sk);
  else if (m <= 4096)
    finish_small_radix<MODE, 4>(ctrl, m, ko, G, theta, hi, gt_keys, gt_idx, ties, ov, oi, offset, sk);
  else
    finish_small_radix<MODE, 8>(ctrl, m, ko, G, theta, hi, gt_keys, gt_idx, ties, ov, oi, offset, sk);
  if (threadIdx.x == 0) ctrl->small_done = 1;
}

}  // namespace dtopk
