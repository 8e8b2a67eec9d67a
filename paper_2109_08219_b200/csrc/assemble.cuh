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
//   K3  ordered compaction of the candidate records (decoupled look-back over
//       tiles of 8192 subranges), class statistics (FQ / PQ).
//   K4  reads the E candidates; each candidate part (<= 8192 keys) writes its
//       elements > theta and its ties, in index order, into a private staging
//       slot -- no global ordering needed.
//   K5  ordered scan over the records (gt, eq counts) -> positions in the pool
//       P_gt (index order) and in the tie list (first k, index order).
//   K6  locates the ties of class-D records that fall among the first k ties.
#pragma once

#include "common.cuh"

namespace dtopk {

enum Cls : u32 { CLS_A = 0, CLS_B = 1, CLS_C = 2, CLS_T = 3, CLS_E = 4 };

constexpr int K3_TILE = 8192;   // subranges per K3 tile (8 warps x 32 steps x 32 lanes)
constexpr int K4_TILE = 8192;   // keys per K4 tile
constexpr int K5_PER = 16;      // records per K5 thread
constexpr int K5_TILE = 256 * K5_PER;
constexpr int SMALL_POOL = 16384;  // pools up to this size are finished by one CTA

struct Records {
  u32* sid;
  u32* d1;
  u32* meta;  // K1 meta: constant << 31 | p1
  u32* x;     // cls | fq << 3 | (E or T list index) << 4
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
  Records rec;
  u32* e_sid;  // [nE] subrange of each E candidate
  u32* t_sid;  // [nT] subrange of each T candidate
  u64 cap_e;
  u64* lb;
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

// K3: qualification + ordered compaction of the candidate records.
__global__ void __launch_bounds__(256) k3_qualify(K3Args a) {
  __shared__ u32 s_wcnt[8];
  __shared__ u64 s_tile, s_prefix;
  __shared__ ull s_stat[5][8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  Ctrl* ctrl = a.ctrl;
  u32 theta = ctrl->selD.kth;
  if (a.theta_override) {
    const long long o = *a.theta_override;
    const u32 ov = o < 0 ? 0u : (o > 0xffffffffll ? 0xffffffffu : (u32)o);
    theta = max(theta, ov);
  }
  if (blockIdx.x == 0 && tid == 0) ctrl->res.theta = theta;
  const u64 T = (a.S + K3_TILE - 1) / K3_TILE;
  const int beta = a.beta;
  ull st_cand = 0, st_fq = 0, st_pq = 0, st_a = 0, st_lastgt = 0;
  u32 dmax = 0;  // largest key of the answer's pool (feeds the sort's key range)
  for (;;) {
    if (tid == 0) s_tile = atomicAdd(&ctrl->k3_ticket, 1u);
    __syncthreads();
    const u64 tile = s_tile;
    if (tile >= T) break;
    const u64 wbase = tile * K3_TILE + (u64)warp * 1024;
    // phase 1: keep masks (lane j of the warp remembers step j's ballot)
    u32 myword = 0, wcnt = 0;
#pragma unroll 8
    for (int j = 0; j < 32; j++) {
      const u64 sid = wbase + (u64)j * 32 + lane;
      const u32 d1 = sid < a.S ? a.D[sid * beta] : 0u;
      const u32 word = __ballot_sync(FULL, sid < a.S && d1 >= theta);
      if (lane == j) myword = word;
      wcnt += __popc(word);
    }
    if (lane == 0) s_wcnt[warp] = wcnt;
    __syncthreads();
    if (warp == 0) {
      u64 agg = 0;
      for (int w = 0; w < 8; w++) agg += s_wcnt[w];
      if (lane == 0) lb_publish_agg(a.lb, tile, agg);
      const u64 excl = lb_warp_prefix(a.lb, tile);
      if (lane == 0) {
        lb_publish_prefix(a.lb, tile, excl + agg);
        s_prefix = excl;
        if (tile == T - 1) ctrl->cand_count = excl + agg;
      }
    }
    __syncthreads();
    u64 pos = s_prefix;
    for (int w = 0; w < warp; w++) pos += s_wcnt[w];
    // phase 2: records of the kept subranges, in subrange order
    for (int j = 0; j < 32; j++) {
      const u32 word = __shfl_sync(FULL, myword, j);
      if (!word) continue;
      const u64 sid = wbase + (u64)j * 32 + lane;
      if ((word >> lane) & 1u) {
        const u32 d1 = a.D[sid * beta];
        const u32 d2 = beta >= 2 ? a.D[sid * beta + 1] : d1;
        const u32 dl = a.D[sid * beta + beta - 1];
        const u32 m = a.meta[sid];
        const u32 cls = classify(d1, d2, m, theta, beta);
        const bool fq = dl >= theta;
        const u64 o = pos + __popc(word & lanemask_lt());
        u32 x = cls | (fq ? 8u : 0u);
        if (cls == CLS_E) {
          const u32 e = atomicAdd(&ctrl->nE, 1u);
          if (e < a.cap_e) a.e_sid[e] = (u32)sid;
          x |= e << 4;
        } else if (cls == CLS_T) {
          const u32 t = atomicAdd(&ctrl->nT, 1u);
          a.t_sid[t] = (u32)sid;
          x |= t << 4;
        }
        a.rec.sid[o] = (u32)sid;
        a.rec.d1[o] = d1;
        a.rec.meta[o] = m;
        a.rec.x[o] = x;
        st_cand++;
        dmax = max(dmax, d1);
        if (fq) st_fq++; else st_pq++;
        if (cls == CLS_A) st_a++;
        if (cls == CLS_A || cls == CLS_E) st_lastgt = max(st_lastgt, (ull)o + 1);
      }
      pos += __popc(word);
    }
  }
  ull v[5] = {st_cand, st_fq, st_pq, st_a, st_lastgt};
#pragma unroll
  for (int i = 0; i < 5; i++) {
    if (i < 4) {
#pragma unroll
      for (int o = 16; o; o >>= 1) v[i] += __shfl_xor_sync(FULL, v[i], o);
    } else {
#pragma unroll
      for (int o = 16; o; o >>= 1) v[i] = max(v[i], __shfl_xor_sync(FULL, v[i], o));
    }
    if (lane == 0) s_stat[i][warp] = v[i];
  }
  dmax = __reduce_max_sync(FULL, dmax);
  if (lane == 0 && dmax) atomicMax(&ctrl->maxkey, dmax);
  __syncthreads();
  if (tid == 0) {
    ull t[5] = {0, 0, 0, 0, 0};
    for (int w = 0; w < 8; w++) {
      for (int i = 0; i < 4; i++) t[i] += s_stat[i][w];
      t[4] = max(t[4], s_stat[4][w]);
    }
    if (t[0]) atomicAdd((ull*)&ctrl->res.candidate_subranges, t[0]);
    if (t[1]) atomicAdd((ull*)&ctrl->res.fully_qualified, t[1]);
    if (t[2]) atomicAdd((ull*)&ctrl->res.partially_qualified, t[2]);
    if (t[3]) atomicAdd(&ctrl->nA, t[3]);
    if (t[4]) atomicMax(&ctrl->gt_rec_end, t[4]);
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
template <int MODE>
__global__ void __launch_bounds__(256) k4_read(K4Args a) {
  __shared__ u32 s_wg[8], s_we[8];
  __shared__ u32 s_seg_g[K4_TILE / 4], s_seg_e[K4_TILE / 4];
  __shared__ u32 s_max[8];
  __shared__ ull s_stat[3][8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  Ctrl* ctrl = a.ctrl;
  const u32 theta = ctrl->res.theta;
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
        if (key > theta) {
          a.stg_key[2 * e + g] = key;
          a.stg_idx[2 * e + g] = b + c;
          g++;
          bmax = max(bmax, key);
        } else if (key == theta) {
          a.stg_idx[2 * e + 1 - q] = b + c;
          q++;
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
        const bool g = vv && x[c] > theta;
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
          const u32 b1 = __ballot_sync(FULL, vv && kv[j][c] > theta);
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
        if (key > theta) {
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
}

// K4T: count the ties of every T candidate (d_1 == theta, max not unique,
// subrange not constant): one warp per candidate (one thread when W < 64).
template <int MODE>
__global__ void __launch_bounds__(256) k4t_count(const u32* __restrict__ keys, u64 n, int alpha, Ctrl* ctrl,
                                                 const u32* __restrict__ t_sid, u32* __restrict__ t_cnt) {
  const u32 theta = ctrl->res.theta;
  const u64 nT = ctrl->nT;
  const u64 W = 1ull << alpha;
  const int lane = threadIdx.x & 31;
  if (W < 64) {
    for (u64 t = (u64)blockIdx.x * 256 + threadIdx.x; t < nT; t += (u64)gridDim.x * 256) {
      const u64 b = (u64)t_sid[t] << alpha;
      u32 c = 0;
      for (u64 e = 0; e < W && b + e < n; e++) c += to_key<MODE>(keys[b + e]) == theta;
      t_cnt[t] = c;
    }
    return;
  }
  const u64 gw = ((u64)blockIdx.x * 256 + threadIdx.x) >> 5;
  const u64 nw = ((u64)gridDim.x * 256) >> 5;
  for (u64 t = gw; t < nT; t += nw) {
    const u64 b = (u64)t_sid[t] << alpha;
    const u64 len = min(W, n - b);
    u32 c = 0;
    for (u64 e = (u64)lane * 2; e < len; e += 64) {
      const u32 k0 = to_key<MODE>(keys[b + e]);
      c += k0 == theta;
      if (e + 1 < len) c += to_key<MODE>(keys[b + e + 1]) == theta;
    }
    c = __reduce_add_sync(FULL, c);
    if (lane == 0) t_cnt[t] = c;
  }
}

// ---------------------------------------------------------------------------
struct K5Args {
  Ctrl* ctrl;
  Records rec;
  u64 n;
  int alpha;
  u64 k;
  const u32* stg_key;
  const u64* stg_idx;
  const u32* seg_gt;
  const u32* seg_eq;
  const u32* t_cnt;  // ties of each T candidate (K4T)
  u32* gt_keys;  // P_gt, index order
  u64* gt_idx;
  u64* ties;     // first k ties, index order
  u32* d_rec;    // K6 work list: record index
  u64* d_pos;    //               tie position and count needed
  u32* d_need;
  u64* lb_gt;
  u64* lb_eq;
};

__device__ __forceinline__ void rec_counts(const K5Args& a, u64 i, u32 theta, u64& g, u64& e) {
  const u32 x = a.rec.x[i];
  const u32 cls = x & 7u;
  g = 0;
  e = 0;
  if (cls == CLS_A) {
    g = 1;
  } else if (cls == CLS_B) {
    e = 1;
  } else if (cls == CLS_C) {
    e = sub_len(a.rec.sid[i], a.n, a.alpha);
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
  (void)theta;
}

// K5: ordered assembly of P_gt and of the first k ties.
__global__ void __launch_bounds__(256) k5_assemble(K5Args a) {
  __shared__ u64 s_tile, s_gx, s_ex;
  __shared__ int s_skip;
  __shared__ u64 scratch_g[8], scratch_e[8];
  __shared__ ull s_cc[8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  Ctrl* ctrl = a.ctrl;
  const u32 theta = ctrl->res.theta;
  const u64 P = ctrl->cand_count;
  const u64 T = (P + K5_TILE - 1) / K5_TILE;
  const u64 gt_end = ctrl->gt_rec_end;
  const u64 W = 1ull << a.alpha;
  const int lseg = a.alpha < 13 ? a.alpha : 13;
  const u64 seglen = 1ull << lseg;
  const u64 ppc = W >> lseg;
  ull st_concat = 0;
  for (;;) {
    if (tid == 0) {
      s_tile = atomicAdd(&ctrl->k5_ticket, 1u);
      s_skip = ld_volatile_u32(&ctrl->ties_full) && s_tile * K5_TILE >= gt_end;
    }
    __syncthreads();
    const u64 tile = s_tile;
    if (tile >= T) break;
    if (s_skip) {
      // nothing > theta from here on and the first k ties are already placed:
      // publish the final prefix without reading anything
      if (tid == 0) {
        const u64 G = ctrl->nA + ctrl->sumEgt;
        st_release(&a.lb_gt[tile], LB_PRE | G);
        st_release(&a.lb_eq[tile], LB_PRE | a.k);
        if (tile == T - 1) {
          ctrl->res.pool_gt = G;
          ctrl->res.pool_eq = a.k;
          ctrl->res.path = G >= a.k ? PATH_SELECT : PATH_MERGE;
          ctrl->res.k_out = a.k;
          if (G < a.k) {
            ctrl->sort_lo = theta;
            atomicMax(&ctrl->maxkey, theta);
          }
        }
      }
      __syncthreads();
      continue;
    }
    const u64 i0 = tile * K5_TILE + (u64)tid * K5_PER;
    u64 tg = 0, te = 0;
    for (int r = 0; r < K5_PER; r++) {
      const u64 i = i0 + r;
      if (i >= P) break;
      u64 g, e;
      rec_counts(a, i, theta, g, e);
      tg += g;
      te += e;
    }
    const u64 ig = block_incl_scan_256<u64>(tg, scratch_g);
    const u64 ie = block_incl_scan_256<u64>(te, scratch_e);
    if (warp == 7) {
      const u64 ag = __shfl_sync(FULL, ig, 31), ae = __shfl_sync(FULL, ie, 31);
      if (lane == 0) {
        lb_publish_agg(a.lb_gt, tile, ag);
        lb_publish_agg(a.lb_eq, tile, ae);
      }
      const u64 xg = lb_warp_prefix(a.lb_gt, tile);
      const u64 xe = lb_warp_prefix(a.lb_eq, tile);
      if (lane == 0) {
        lb_publish_prefix(a.lb_gt, tile, xg + ag);
        lb_publish_prefix(a.lb_eq, tile, xe + ae);
        s_gx = xg;
        s_ex = xe;
        if (xe + ae >= a.k) atomicExch(&ctrl->ties_full, 1u);
        if (tile == T - 1) {
          const u64 G = xg + ag, E = xe + ae;
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
    }
    __syncthreads();
    u64 gpos = s_gx + ig - tg, epos = s_ex + ie - te;
    for (int r = 0; r < K5_PER; r++) {
      const u64 i = i0 + r;
      if (i >= P) break;
      const u32 x = a.rec.x[i];
      const u32 cls = x & 7u;
      const bool fq = (x >> 3) & 1u;
      const u64 sid = a.rec.sid[i];
      const u32 m = a.rec.meta[i];
      const u64 base = sid << a.alpha;
      if (cls == CLS_A) {
        a.gt_keys[gpos] = a.rec.d1[i];
        a.gt_idx[gpos] = base + meta_p1(m);
        gpos++;
      } else if (cls == CLS_B) {
        if (epos < a.k) a.ties[epos] = base + meta_p1(m);
        epos++;
      } else if (cls == CLS_C) {
        const u64 len = sub_len(sid, a.n, a.alpha);
        const u64 take = epos < a.k ? min(len, a.k - epos) : 0;
        for (u64 q = 0; q < take; q++) a.ties[epos + q] = base + q;
        if (fq) st_concat += len;
        epos += len;
      } else if (cls == CLS_T) {
        const u64 c1 = a.t_cnt[x >> 4];
        if (epos < a.k && c1) {
          const u32 slot = atomicAdd(&ctrl->k6_count, 1u);
          a.d_rec[slot] = (u32)i;
          a.d_pos[slot] = epos;
          a.d_need[slot] = (u32)min(c1, a.k - epos);
        }
        if (fq) st_concat += c1;
        epos += c1;
      } else {
        const u64 eidx = x >> 4;
        u64 eg = 0, ee = 0;
        for (u64 p = 0; p < ppc; p++) {
          const u64 sg = eidx * ppc + p;
          const u32 ng = a.seg_gt[sg], ne = a.seg_eq[sg];
          const u64 sb = sg << lseg;
          for (u32 q = 0; q < ng; q++) {
            a.gt_keys[gpos + q] = a.stg_key[sb + q];
            a.gt_idx[gpos + q] = a.stg_idx[sb + q];
          }
          gpos += ng;
          eg += ng;
          for (u32 q = 0; q < ne; q++) {
            if (epos + q < a.k) a.ties[epos + q] = a.stg_idx[sb + seglen - 1 - q];
          }
          epos += ne;
          ee += ne;
        }
        if (fq) st_concat += eg + ee;
      }
    }
    __syncthreads();
  }
  for (int o = 16; o; o >>= 1) st_concat += __shfl_xor_sync(FULL, st_concat, o);
  if (lane == 0) s_cc[warp] = st_concat;
  __syncthreads();
  if (tid == 0) {
    ull t = 0;
    for (int w = 0; w < 8; w++) t += s_cc[w];
    if (t) atomicAdd((ull*)&ctrl->res.concatenated_len, t);
  }
}

// K6: locate the ties of class-D records that fall among the first k ties
// (one warp per record; ballot-ordered within the subrange).
template <int MODE>
__global__ void __launch_bounds__(256) k6_ties(Ctrl* ctrl, const u32* __restrict__ keys, u64 n, int alpha,
                                               const u32* __restrict__ rec_sid, const u32* __restrict__ d_rec,
                                               const u64* __restrict__ d_pos, const u32* __restrict__ d_need,
                                               u64* __restrict__ ties) {
  const int lane = threadIdx.x & 31;
  const u32 theta = ctrl->res.theta;
  const u32 cnt = ctrl->k6_count;
  const u64 gw = ((u64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const u64 nw = ((u64)gridDim.x * blockDim.x) >> 5;
  const u32 lt = lanemask_lt();
  for (u64 w = gw; w < cnt; w += nw) {
    const u64 base = (u64)rec_sid[d_rec[w]] << alpha;
    const u64 len = sub_len(base >> alpha, n, alpha);
    const u64 pos0 = d_pos[w];
    const u32 need = d_need[w];
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

// Fused finish for pools of at most SMALL_POOL pairs: one CTA sorts the pool
// (P_gt, plus the ties on the merge path) by (key desc, position asc) and
// writes the first k_out pairs in the input dtype.  Positions follow index
// order, so this is the (key desc, index asc) order of the reference tie rule.
template <int MODE>
__global__ void __launch_bounds__(1024) finish_small(Ctrl* ctrl, const u32* __restrict__ gt_keys,
                                                     const u64* __restrict__ gt_idx, const u64* __restrict__ ties,
                                                     u32* __restrict__ ov, long long* __restrict__ oi,
                                                     long long offset) {
  extern __shared__ unsigned long long sk[];
  const u32 path = ctrl->res.path;
  const u64 G = ctrl->res.pool_gt;
  const u64 m = path == PATH_SELECT ? G : ctrl->res.k_out;
  if (m > (u64)SMALL_POOL || m == 0) return;
  const u64 ko = ctrl->res.k_out;
  const u32 theta = ctrl->res.theta;
  const u32 hi = max(ctrl->maxkey, theta);
  u32 np = 1;
  while (np < m) np <<= 1;
  for (u32 i = threadIdx.x; i < np; i += 1024) {
    unsigned long long v = ~0ull;
    if (i < m) {
      const u32 key = i < G ? gt_keys[i] : theta;
      v = ((unsigned long long)(hi - key) << 32) | i;
    }
    sk[i] = v;
  }
  __syncthreads();
  for (u32 size = 2; size <= np; size <<= 1) {
    for (u32 stride = size >> 1; stride > 0; stride >>= 1) {
      for (u32 t = threadIdx.x; t < np / 2; t += 1024) {
        const u32 lo = 2 * t - (t & (stride - 1));
        const u32 hi2 = lo + stride;
        const bool up = (lo & size) == 0;
        const unsigned long long x = sk[lo], y = sk[hi2];
        if ((x > y) == up) {
          sk[lo] = y;
          sk[hi2] = x;
        }
      }
      __syncthreads();
    }
  }
  for (u32 i = threadIdx.x; i < ko; i += 1024) {
    const u32 pos = (u32)(sk[i] & 0xffffffffu);
    const u32 key = hi - (u32)(sk[i] >> 32);
    ov[i] = from_key<MODE>(key);
    oi[i] = (long long)(pos < G ? gt_idx[pos] : ties[pos - G]) + offset;
    if (i == ko - 1) ctrl->res.kth_key = key;
  }
  if (threadIdx.x == 0) ctrl->small_done = 1;
}

}  // namespace dtopk
