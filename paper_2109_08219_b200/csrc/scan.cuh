// scan.cuh -- ordered emit of the final top-k over a flat key array, the
// merge copy, the stable radix sort of the answer and its write-out.
//
// Reference: the tie rule of kernels._extract_exact (kernels.py:83-96) --
// every element strictly above the k-th key first, then k-th-key ties in scan
// order until k slots are filled -- and the final np.sort of dr_topk
// (pipeline.py:215-218), here ordered (key desc, index asc).
//
// scan_emit: one tile = 8192 keys = 8 warps x 1024; a warp loads 8 rounds of
// 32 lanes x uint4 (512 contiguous bytes per instruction).  Phase 1 counts
// (gt, eq) per thread; the tile publishes its aggregate on two decoupled
// look-back chains; phase 2 re-derives the predicates from registers and
// writes every selected element at its stable (index-ordered) position using
// ballots, so no per-element atomics and no second read are needed.  It runs
// over the pool P_gt when the pool exceeds k (and SMALL_POOL), and over the
// raw input on the direct path (pipeline.py:184-191).
#pragma once

#include <cub/block/block_radix_sort.cuh>

#include "common.cuh"

namespace dtopk {

constexpr int SC_TILE = 8192;

struct ScanArgs {
  const u32* keys;
  const u64* idx_in;  // explicit indices (null = position)
  u64 m_host;         // element count
  const ull* m_dev;
  Ctrl* ctrl;
  u64 k;
  u32* out_keys;      // answer keys/indices (sort buffer A)
  u64* out_idx;
  u64* lb_gt;
  u64* lb_eq;
  int check_path;
  int direct;
};


template <int MODE>
__global__ void __launch_bounds__(256, DTOPK_TAIL_MINB) scan_emit(ScanArgs a) {
  __shared__ DigitResult r3s;
  __shared__ ull scratch[8];
  __shared__ u32 s_wgt[8], s_weq[8];
  __shared__ u64 s_tile, s_gtx, s_eqx;
  __shared__ u32 s_max[8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  Ctrl* ctrl = a.ctrl;
  if (a.check_path && ld_volatile_u32(&ctrl->big_mode) != BIG_SELECT) return;

  const DigitResult r1 = ctrl->selP.r1, r2 = ctrl->selP.r2;
  find_digit<NB3>(ctrl->selP.hist3, r2.rem, &r3s, scratch);
  const u32 theta = (r1.digit << 21) | (r2.digit << 10) | r3s.digit;
  const u64 eq_cap = r3s.rem;  // ties needed
  const u64 ngt = a.k - eq_cap;
  u32* eqk = a.out_keys + ngt;
  u64* eqi = a.out_idx + ngt;
  if (blockIdx.x == 0 && tid == 0) {
    ctrl->selP.r3 = r3s;
    ctrl->selP.kth = theta;
    ctrl->sort_lo = theta;
    ctrl->sort_m = a.k;
    ctrl->sort_src = a.direct ? 0u : 1u;  // direct: emit into A; pool select: into B
    ctrl->res.k_out = a.k;
    if (a.direct) {
      ctrl->res.path = PATH_DIRECT;
      ctrl->res.theta = theta;
      ctrl->res.pool_gt = ngt;
    }
    atomicMax(&ctrl->maxkey, theta);
  }
  const u64 total = a.m_dev ? (u64)*a.m_dev : a.m_host;
  const u64 T = (total + SC_TILE - 1) / SC_TILE;
  u32 bmax = 0;

  for (;;) {
    if (tid == 0) s_tile = atomicAdd(&ctrl->em_ticket, 1u);
    __syncthreads();
    const u64 tile = s_tile;
    if (tile >= T) break;

    // ---------------- phase 1: load + count
    u32 kv[8][4];
    u32 vm[8];
    u32 cgt = 0, ceq = 0;
#pragma unroll
    for (int j = 0; j < 8; j++) {
      const u64 v0 = tile * SC_TILE + (u64)warp * 1024 + (u64)j * 128 + (u64)lane * 4;
      u32 x[4] = {0u, 0u, 0u, 0u};
      u32 valid = 0;
      if (v0 + 4 <= total) {
        const uint4 q = ld_nc_v4(a.keys + v0);
        x[0] = to_key<MODE>(q.x);
        x[1] = to_key<MODE>(q.y);
        x[2] = to_key<MODE>(q.z);
        x[3] = to_key<MODE>(q.w);
        valid = 0xfu;
      } else {
#pragma unroll
        for (int c = 0; c < 4; c++)
          if (v0 + c < total) {
            x[c] = to_key<MODE>(a.keys[v0 + c]);
            valid |= 1u << c;
          }
      }
#pragma unroll
      for (int c = 0; c < 4; c++) {
        const bool vld = (valid >> c) & 1u;
        const bool g = vld && x[c] > theta;
        cgt += g;
        ceq += vld && x[c] == theta;
        if (g) bmax = max(bmax, x[c]);
        kv[j][c] = x[c];
      }
      vm[j] = valid;
    }
    const u32 wg = __reduce_add_sync(FULL, cgt), we = __reduce_add_sync(FULL, ceq);
    if (lane == 0) {
      s_wgt[warp] = wg;
      s_weq[warp] = we;
    }
    __syncthreads();
    if (warp == 0) {
      u64 ag = 0, ae = 0;
      for (int w = 0; w < 8; w++) {
        ag += s_wgt[w];
        ae += s_weq[w];
      }
      if (lane == 0) {
        lb_publish_agg(a.lb_gt, tile, ag);
        lb_publish_agg(a.lb_eq, tile, ae);
      }
      const u64 xg = lb_warp_prefix(a.lb_gt, tile);
      const u64 xe = lb_warp_prefix(a.lb_eq, tile);
      if (lane == 0) {
        lb_publish_prefix(a.lb_gt, tile, xg + ag);
        lb_publish_prefix(a.lb_eq, tile, xe + ae);
        s_gtx = xg;
        s_eqx = xe;
      }
    }
    __syncthreads();

    // ---------------- phase 2: ordered writes
    u64 gpos = s_gtx, epos = s_eqx;
    for (int w = 0; w < warp; w++) {
      gpos += s_wgt[w];
      epos += s_weq[w];
    }
    const u32 lt = lanemask_lt();
#pragma unroll
    for (int j = 0; j < 8; j++) {
      u32 bg[4], be[4];
      bool g[4], e[4];
#pragma unroll
      for (int c = 0; c < 4; c++) {
        const bool vld = (vm[j] >> c) & 1u;
        g[c] = vld && kv[j][c] > theta;
        e[c] = vld && kv[j][c] == theta;
        bg[c] = __ballot_sync(FULL, g[c]);
        be[c] = __ballot_sync(FULL, e[c]);
      }
      const u32 anyg = bg[0] | bg[1] | bg[2] | bg[3];
      const u32 anye = be[0] | be[1] | be[2] | be[3];
      if (anyg | anye) {
        u64 go = gpos, eo = epos;
#pragma unroll
        for (int c = 0; c < 4; c++) {
          go += __popc(bg[c] & lt);
          eo += __popc(be[c] & lt);
        }
        const u64 v0 = tile * SC_TILE + (u64)warp * 1024 + (u64)j * 128 + (u64)lane * 4;
#pragma unroll
        for (int c = 0; c < 4; c++) {
          if (g[c] || e[c]) {
            const u64 idx = a.idx_in ? a.idx_in[v0 + c] : v0 + c;
            if (g[c]) {
              a.out_keys[go] = kv[j][c];
              a.out_idx[go] = idx;
              go++;
            }
            if (e[c]) {
              if (eo < eq_cap) {
                eqk[eo] = kv[j][c];
                eqi[eo] = idx;
              }
              eo++;
            }
          }
        }
#pragma unroll
        for (int c = 0; c < 4; c++) {
          gpos += __popc(bg[c]);
          epos += __popc(be[c]);
        }
      }
    }
  }
  bmax = __reduce_max_sync(FULL, bmax);
  if (lane == 0) s_max[warp] = bmax;
  __syncthreads();
  if (tid == 0) {
    u32 m = 0;
    for (int w = 0; w < 8; w++) m = max(m, s_max[w]);
    if (m) atomicMax(&ctrl->maxkey, m);
  }
}

// Ordered emit for the pool select (not the direct path), in two kernels
// instead of scan_emit's decoupled look-back: emit_count counts keys above /
// equal to tau per SC_TILE tile and its last CTA turns the counts into
// exclusive prefixes; emit_write re-reads only the tiles that hold something to
// emit.  On sorted pools (ascending input: 8.4 M keys, the answer in the last
// few tiles) scan_emit stalled ~45 us on the look-back chain.
template <int MODE>
__device__ __forceinline__ u32 em_tau(const Ctrl* ctrl, DigitResult* r3s, ull* scratch) {
  const DigitResult r1 = ctrl->selP.r1, r2 = ctrl->selP.r2;
  find_digit<NB3>(ctrl->selP.hist3, r2.rem, r3s, scratch);
  return (r1.digit << 21) | (r2.digit << 10) | r3s->digit;
}

template <int MODE>
__device__ __forceinline__ void em_load(const ScanArgs& a, u64 total, u64 tile, int j, u32 (&x)[4], u32& valid) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const u64 v0 = tile * SC_TILE + (u64)warp * 1024 + (u64)j * 128 + (u64)lane * 4;
  x[0] = x[1] = x[2] = x[3] = 0u;
  valid = 0;
  if (v0 + 4 <= total) {
    const uint4 q = ld_nc_v4(a.keys + v0);
    x[0] = to_key<MODE>(q.x);
    x[1] = to_key<MODE>(q.y);
    x[2] = to_key<MODE>(q.z);
    x[3] = to_key<MODE>(q.w);
    valid = 0xfu;
  } else {
#pragma unroll
    for (int c = 0; c < 4; c++)
      if (v0 + c < total) {
        x[c] = to_key<MODE>(a.keys[v0 + c]);
        valid |= 1u << c;
      }
  }
}

template <int MODE>
__global__ void __launch_bounds__(256) emit_count(ScanArgs a) {
  __shared__ DigitResult r3s;
  __shared__ ull scratch[8];
  __shared__ u32 s_g[8], s_e[8], s_max[8];
  __shared__ int am_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  Ctrl* ctrl = a.ctrl;
  if (a.check_path && ld_volatile_u32(&ctrl->big_mode) != BIG_SELECT) return;
  const u32 tau = em_tau<MODE>(ctrl, &r3s, scratch);
  if (blockIdx.x == 0 && tid == 0) {
    ctrl->selP.r3 = r3s;
    ctrl->selP.kth = tau;
    ctrl->sort_lo = tau;
    ctrl->sort_m = a.k;
    ctrl->sort_src = 1u;  // pool select: the answer goes to sort buffer B
    ctrl->res.k_out = a.k;
    atomicMax(&ctrl->maxkey, tau);
  }
  const u64 total = a.m_dev ? (u64)*a.m_dev : a.m_host;
  const u64 T = (total + SC_TILE - 1) / SC_TILE;
  u32 bmax = 0;
  for (u64 tile = blockIdx.x; tile < T; tile += gridDim.x) {
    u32 cg = 0, ce = 0;
#pragma unroll
    for (int j = 0; j < 8; j++) {
      u32 x[4], valid;
      em_load<MODE>(a, total, tile, j, x, valid);
#pragma unroll
      for (int c = 0; c < 4; c++) {
        const bool v = (valid >> c) & 1u;
        cg += v && x[c] > tau;
        ce += v && x[c] == tau;
        if (v && x[c] > tau) bmax = max(bmax, x[c]);
      }
    }
    cg = __reduce_add_sync(FULL, cg);
    ce = __reduce_add_sync(FULL, ce);
    if (lane == 0) {
      s_g[warp] = cg;
      s_e[warp] = ce;
    }
    __syncthreads();
    if (tid == 0) {
      u64 g = 0, e = 0;
      for (int w = 0; w < 8; w++) {
        g += s_g[w];
        e += s_e[w];
      }
      a.lb_gt[tile] = g;
      a.lb_eq[tile] = e;
    }
    __syncthreads();
  }
  bmax = __reduce_max_sync(FULL, bmax);
  if (lane == 0) s_max[warp] = bmax;
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    u32 m = 0;
    for (int w = 0; w < 8; w++) m = max(m, s_max[w]);
    if (m) atomicMax(&ctrl->maxkey, m);
    am_last = atomicAdd(&ctrl->em_ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  // exclusive prefixes of the tile counts (thread t: tiles [t * per, (t+1) * per))
  const u64 per = (T + 255) / 256;
  const u64 t0 = (u64)tid * per, t1 = min(T, t0 + per);
  ull sg = 0, se = 0;
  for (u64 t = t0; t < t1; t++) {
    sg += __ldcg(&a.lb_gt[t]);
    se += __ldcg(&a.lb_eq[t]);
  }
  const ull ig = block_incl_scan_256<ull>(sg, scratch);
  ull rg = ig - sg;
  const ull ie = block_incl_scan_256<ull>(se, scratch);
  ull re = ie - se;
  for (u64 t = t0; t < t1; t++) {
    const ull g = __ldcg(&a.lb_gt[t]), e = __ldcg(&a.lb_eq[t]);
    a.lb_gt[t] = rg;
    a.lb_eq[t] = re;
    rg += g;
    re += e;
  }
  if (tid == 255) {
    a.lb_gt[T] = ig;  // sentinels: the totals
    a.lb_eq[T] = ie;
  }
}

template <int MODE>
__global__ void __launch_bounds__(256) emit_write(ScanArgs a) {
  __shared__ DigitResult r3s;
  __shared__ ull scratch[8];
  __shared__ u32 s_g[8], s_e[8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  Ctrl* ctrl = a.ctrl;
  if (a.check_path && ld_volatile_u32(&ctrl->big_mode) != BIG_SELECT) return;
  const u32 tau = ld_volatile_u32(&ctrl->selP.kth);
  const u64 eq_cap = ctrl->selP.r3.rem;  // ties needed
  const u64 ngt = a.k - eq_cap;
  u32* eqk = a.out_keys + ngt;
  u64* eqi = a.out_idx + ngt;
  const u64 total = a.m_dev ? (u64)*a.m_dev : a.m_host;
  const u64 T = (total + SC_TILE - 1) / SC_TILE;
  const u32 lt = lanemask_lt();
  for (u64 tile = blockIdx.x; tile < T; tile += gridDim.x) {
    const u64 gx = a.lb_gt[tile], ex = a.lb_eq[tile];
    const u64 ng = a.lb_gt[tile + 1] - gx, ne = a.lb_eq[tile + 1] - ex;
    if (ng == 0 && (ne == 0 || ex >= eq_cap)) continue;  // nothing to emit here (uniform per CTA)
    u32 kv[8][4], vm[8], cg = 0, ce = 0;
#pragma unroll
    for (int j = 0; j < 8; j++) {
      em_load<MODE>(a, total, tile, j, kv[j], vm[j]);
#pragma unroll
      for (int c = 0; c < 4; c++) {
        const bool v = (vm[j] >> c) & 1u;
        cg += v && kv[j][c] > tau;
        ce += v && kv[j][c] == tau;
      }
    }
    cg = __reduce_add_sync(FULL, cg);
    ce = __reduce_add_sync(FULL, ce);
    if (lane == 0) {
      s_g[warp] = cg;
      s_e[warp] = ce;
    }
    __syncthreads();
    u64 gpos = gx, epos = ex;
    for (int w = 0; w < warp; w++) {
      gpos += s_g[w];
      epos += s_e[w];
    }
#pragma unroll
    for (int j = 0; j < 8; j++) {
      u32 bg[4], be[4];
#pragma unroll
      for (int c = 0; c < 4; c++) {
        const bool v = (vm[j] >> c) & 1u;
        bg[c] = __ballot_sync(FULL, v && kv[j][c] > tau);
        be[c] = __ballot_sync(FULL, v && kv[j][c] == tau);
      }
      if ((bg[0] | bg[1] | bg[2] | bg[3] | be[0] | be[1] | be[2] | be[3]) == 0) continue;
      u64 go = gpos, eo = epos;
#pragma unroll
      for (int c = 0; c < 4; c++) {
        go += __popc(bg[c] & lt);
        eo += __popc(be[c] & lt);
      }
      const u64 v0 = tile * SC_TILE + (u64)warp * 1024 + (u64)j * 128 + (u64)lane * 4;
#pragma unroll
      for (int c = 0; c < 4; c++) {
        const bool g = (bg[c] >> lane) & 1u, e = (be[c] >> lane) & 1u;
        if (g || (e && eo < eq_cap)) {
          const u64 idx = a.idx_in ? a.idx_in[v0 + c] : v0 + c;
          if (g) {
            a.out_keys[go] = kv[j][c];
            a.out_idx[go] = idx;
          } else {
            eqk[eo] = kv[j][c];
            eqi[eo] = idx;
          }
        }
        go += g;
        eo += e;
      }
#pragma unroll
      for (int c = 0; c < 4; c++) {
        gpos += __popc(bg[c]);
        epos += __popc(be[c]);
      }
    }
    __syncthreads();
  }
}

constexpr int SMALL_SORT = 8192;  // answers up to this size are sorted by one CTA

// Decide how the pool beyond SMALL_POOL is finished (one thread).
// In a CUDA-graph plan it also sets the conditionals that gate the select
// kernels (BIG_SELECT only; use_cond bit 0) and the multi-CTA bucket sort
// (answers beyond SMALL_SORT; bit 1), so skipped stages are not launched.
__global__ void tail_decide(Ctrl* ctrl, u64 k, cudaGraphConditionalHandle c_sel, cudaGraphConditionalHandle c_bucket,
                            int use_cond) {
  if (ctrl->small_done) {
    ctrl->big_mode = BIG_NONE;
    if (use_cond & 1) cudaGraphSetConditional(c_sel, 0u);
    if (use_cond & 2) cudaGraphSetConditional(c_bucket, 0u);
    return;
  }
  const u64 G = ctrl->res.pool_gt;
  // the pool's keys lie in [max(theta, pool floor), maxkey]: the bucket sort's range
  ctrl->sort_lo = max(ctrl->res.theta, ctrl->pfloor);
  if (ctrl->res.path == PATH_MERGE) {
    ctrl->big_mode = BIG_MERGE;  // pool = P_gt ++ ties, sorted in place
    ctrl->sort_src = 0;
    ctrl->sort_m = ctrl->res.k_out;
  } else if (G <= 4 * k) {
    ctrl->big_mode = BIG_SORT_POOL;  // sort all of P_gt, keep the first k
    ctrl->sort_src = 0;
    ctrl->sort_m = G;
  } else {
    ctrl->big_mode = BIG_SELECT;  // radix select + ordered emit, then sort k
  }
  const bool sel = ctrl->big_mode == BIG_SELECT;
  if (use_cond & 1) cudaGraphSetConditional(c_sel, sel ? 1u : 0u);
  if (use_cond & 2) cudaGraphSetConditional(c_bucket, (sel ? k : (u64)ctrl->sort_m) > (u64)SMALL_SORT ? 1u : 0u);
}

// BIG_MERGE: append the ties (key theta) after P_gt.
__global__ void __launch_bounds__(256) merge_append(Ctrl* ctrl, u32* __restrict__ gk, u64* __restrict__ gi,
                                                    const u64* __restrict__ ties) {
  if (ld_volatile_u32(&ctrl->big_mode) != BIG_MERGE) return;
  const u64 G = ctrl->res.pool_gt, kout = ctrl->res.k_out;
  const u32 theta = ctrl->res.theta;
  for (u64 i = G + (u64)blockIdx.x * 256 + threadIdx.x; i < kout; i += (u64)gridDim.x * 256) {
    gk[i] = theta;
    gi[i] = ties[i - G];
  }
}

// ---------------------------------------------------------------------------
// Stable LSD radix sort of the answer candidates by key descending: digits of
// (maxkey - key), only as many 8-bit passes as maxkey - lo needs.  Input order
// is index order within equal keys, so stability yields (key desc, index asc).
// The number of elements (ctrl->sort_m) and the buffer holding them
// (ctrl->sort_src: 0 = A, 1 = B) are decided on the device.
// ---------------------------------------------------------------------------
constexpr int ST_TILE = 2048;

__device__ __forceinline__ int sort_bits(const Ctrl* c) {
  const u32 lo = c->sort_lo;
  const u32 hi = max(c->maxkey, lo);
  return hi == lo ? 0 : 32 - __clz(hi - lo);
}

__device__ __forceinline__ bool big_sort_skip(const Ctrl* c, int pass) {
  return c->sort_m <= (ull)SMALL_SORT || pass * 8 >= sort_bits(c) || c->small_done || !c->lsd_fallback;
}

struct SortBufs {
  u32* ka;
  u64* ia;
  u32* kb;
  u64* ib;
  u32* counts;     // [256][T] digit-major
  u32* digit_base; // [256]
  u32* digit_tot;  // [256]
};

__device__ __forceinline__ void sort_io(const Ctrl* c, const SortBufs& b, int pass, const u32*& kin, const u64*& iin,
                                        u32*& kout, u64*& iout) {
  const bool from_b = ((c->sort_src + (u32)pass) & 1u) != 0;
  kin = from_b ? b.kb : b.ka;
  iin = from_b ? b.ib : b.ia;
  kout = from_b ? b.ka : b.kb;
  iout = from_b ? b.ia : b.ib;
}

__global__ void __launch_bounds__(256) sort_hist(Ctrl* ctrl, SortBufs b, int pass) {
  if (big_sort_skip(ctrl, pass)) return;
  __shared__ u32 h[256];
  const u32 *keys, *kx;
  const u64 *ix;
  u64* iy;
  u32* ky;
  sort_io(ctrl, b, pass, keys, ix, ky, iy);
  (void)kx;
  const u64 m = ctrl->sort_m;
  const u32 hi = max(ctrl->maxkey, ctrl->sort_lo);
  const u64 T = (m + ST_TILE - 1) / ST_TILE;
  for (u64 tile = blockIdx.x; tile < T; tile += gridDim.x) {
    h[threadIdx.x] = 0;
    __syncthreads();
    for (int r = 0; r < ST_TILE / 256; r++) {
      const u64 e = tile * ST_TILE + (u64)r * 256 + threadIdx.x;
      if (e < m) atomicAdd(&h[((hi - keys[e]) >> (8 * pass)) & 255u], 1u);
    }
    __syncthreads();
    b.counts[(u64)threadIdx.x * T + tile] = h[threadIdx.x];  // digit-major
    __syncthreads();
  }
}

// One warp per digit: exclusive scan of its column over the tiles; the last
// CTA scans the 256 digit totals into digit_base.
__global__ void __launch_bounds__(256) sort_scan(Ctrl* ctrl, SortBufs b, int pass) {
  if (big_sort_skip(ctrl, pass)) return;
  __shared__ int am_last;
  __shared__ u32 scratch[8];
  const int lane = threadIdx.x & 31;
  const u32 d = blockIdx.x * 8 + (threadIdx.x >> 5);  // grid = 32 CTAs
  const u64 T = (ctrl->sort_m + ST_TILE - 1) / ST_TILE;
  u32* col = b.counts + (u64)d * T;
  u32 run = 0;
  for (u64 t0 = 0; t0 < T; t0 += 32) {
    const u64 t = t0 + lane;
    const u32 c = t < T ? col[t] : 0u;
    const u32 incl = warp_incl_scan<u32>(c);
    if (t < T) col[t] = run + incl - c;
    run += __shfl_sync(FULL, incl, 31);
  }
  if (lane == 0) b.digit_tot[d] = run;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) am_last = atomicAdd(&ctrl->sort_done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (am_last) {
    __threadfence();
    const u32 tot = __ldcg(&b.digit_tot[threadIdx.x]);
    const u32 incl = block_incl_scan_256<u32>(tot, scratch);
    b.digit_base[threadIdx.x] = incl - tot;
    if (threadIdx.x == 0) ctrl->sort_done = 0;  // next pass
  }
}

__global__ void __launch_bounds__(256) sort_scatter(Ctrl* ctrl, SortBufs b, int pass) {
  if (big_sort_skip(ctrl, pass)) return;
  __shared__ u32 wc[8][256];
  const u32* kin;
  const u64* iin;
  u32* kout;
  u64* iout;
  sort_io(ctrl, b, pass, kin, iin, kout, iout);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const u64 ko = ctrl->sort_m;
  const u32 hi = max(ctrl->maxkey, ctrl->sort_lo);
  const u64 T = (ko + ST_TILE - 1) / ST_TILE;
  const u32 lt = lanemask_lt();
  for (u64 tile = blockIdx.x; tile < T; tile += gridDim.x) {
    for (int i = tid; i < 8 * 256; i += 256) (&wc[0][0])[i] = 0;
    __syncthreads();
    u32 key[8], dg[8], rk[8];
#pragma unroll
    for (int r = 0; r < 8; r++) {
      const u64 e = tile * ST_TILE + (u64)warp * 256 + (u64)r * 32 + lane;
      key[r] = e < ko ? kin[e] : 0u;
    }
#pragma unroll
    for (int r = 0; r < 8; r++) {
      const u64 e = tile * ST_TILE + (u64)warp * 256 + (u64)r * 32 + lane;
      const bool v = e < ko;
      dg[r] = v ? ((hi - key[r]) >> (8 * pass)) & 255u : 256u;
      const u32 peers = __match_any_sync(FULL, dg[r]);
      const u32 leader = __ffs(peers) - 1;
      rk[r] = v ? wc[warp][dg[r]] + __popc(peers & lt) : 0u;
      __syncwarp();
      if (v && lane == leader) wc[warp][dg[r]] += __popc(peers);
      __syncwarp();
    }
    __syncthreads();
    {
      u32 run = 0;
      for (int w = 0; w < 8; w++) {
        const u32 c = wc[w][tid];
        wc[w][tid] = run;
        run += c;
      }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 8; r++) {
      const u64 e = tile * ST_TILE + (u64)warp * 256 + (u64)r * 32 + lane;
      if (e < ko) {
        const u64 pos = (u64)b.digit_base[dg[r]] + b.counts[(u64)dg[r] * T + tile] + wc[warp][dg[r]] + rk[r];
        kout[pos] = key[r];
        iout[pos] = iin[e];
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Bucket sort of large answers.  Elements go to up to BK_MAX buckets by the
// high bits of d = maxkey - key and carry their input position; (d << 32 |
// position) orders a bucket as (key desc, index asc) whatever order the
// scatter wrote it in.  BK_CHUNKS CTAs own contiguous chunks of the input:
//   bucket_count   per-chunk bucket counts; an atomicAdd on the bucket total
//                  hands each chunk its base inside the bucket
//   bucket_scatter scan of the totals (bucket starts), then composites to
//                  their bucket through shared-memory cursors
//   bucket_sort    CTA per bucket: counting sort on the next BK_SUB_BITS bits
//                  of d in shared memory, then rank inside each sub-bin by
//                  comparison (sub-bins hold ~1 element unless keys repeat),
//                  and write the answer slice directly.
// A bucket above BK_CAP (skewed keys) sends the sort to the LSD radix sort.
// ---------------------------------------------------------------------------
#ifndef DTOPK_BK_CHUNKS
#define DTOPK_BK_CHUNKS 128
#endif
#ifndef DTOPK_BK_TARGET
#define DTOPK_BK_TARGET 2048
#endif
#ifndef DTOPK_BK_SUB_BITS
#define DTOPK_BK_SUB_BITS 10
#endif
constexpr int BK_MAX = 4096;      // buckets
constexpr int BK_CHUNKS = DTOPK_BK_CHUNKS;    // count / scatter CTAs
constexpr int BK_TARGET = DTOPK_BK_TARGET;    // elements per bucket aimed for
constexpr int BK_CAP = 4096;      // largest bucket bucket_sort takes (16 per thread)
constexpr int BK_SUB_BITS = DTOPK_BK_SUB_BITS;  // sub-bins of the in-bucket counting sort
constexpr int BK_SUB = 1 << BK_SUB_BITS;
#ifndef DTOPK_BK_LPT
#define DTOPK_BK_LPT 4
#endif
constexpr int BK_LPT = DTOPK_BK_LPT;  // key loads in flight per thread in bucket_count / bucket_scatter

struct BucketBufs {
  u32* total;   // [BK_MAX] bucket sizes (zeroed per run)
  u32* counts;  // [BK_CHUNKS][BK_MAX] each chunk's base inside its bucket
  u32* start;   // [BK_MAX + 1] bucket starts
  unsigned long long* comp;  // [sort cap] scattered composites
  u32* info;    // [0] shift, [1] buckets, [2] fallback flag
  cudaGraphConditionalHandle c_lsd;  // graph plans: gates the LSD fallback sort
  int use_cond;
};

__device__ __forceinline__ bool bucket_skip(const Ctrl* c) {
  return c->sort_m <= (ull)SMALL_SORT || c->small_done;
}

__device__ __forceinline__ void bucket_geometry(const Ctrl* c, u32& shift, u32& nb) {
  const u64 m = c->sort_m;
  const u32 hi = max(c->maxkey, c->sort_lo);
  const u32 range = hi - c->sort_lo;
  u32 want = 1;
  while (want < BK_MAX && (u64)want * BK_TARGET < m) want <<= 1;
  const int bits = range ? 32 - __clz(range) : 0;  // d < 2^bits
  const int lb = 31 - __clz(want);
  shift = bits > lb ? (u32)(bits - lb) : 0u;
  // range >> shift lies in [want / 2, want): one bit less of shift when that
  // leaves the buckets above 3/4 of BK_CAP on average (k = 2^14: 5 buckets of
  // ~3.3k keys overflowed BK_CAP and sent the sort to the LSD fallback, ~50 us;
  // more, smaller buckets measured ~3 us slower at k = 2^20)
  const u64 nb0 = range ? ((ull)range >> shift) + 1ull : 1ull;
  if (shift > 0 && m > nb0 * (u64)(BK_CAP / 4 * 3) && 2ull * want <= (ull)BK_MAX) shift--;
  nb = (u32)min((ull)BK_MAX, range ? ((ull)range >> shift) + 1ull : 1ull);
}

__device__ __forceinline__ void bucket_chunk(u64 m, u64& lo, u64& hi) {
  const u64 per = (m + BK_CHUNKS - 1) / BK_CHUNKS;
  lo = min(m, (u64)blockIdx.x * per);
  hi = min(m, lo + per);
}

__global__ void __launch_bounds__(512) bucket_count(Ctrl* ctrl, SortBufs b, BucketBufs bb) {
  if (bucket_skip(ctrl)) return;
  __shared__ u32 h[BK_MAX];
  u32 shift, nb;
  bucket_geometry(ctrl, shift, nb);
  for (int i = threadIdx.x; i < (int)nb; i += 512) h[i] = 0;
  __syncthreads();
  const u32* keys = ctrl->sort_src ? b.kb : b.ka;
  const u32 hi = max(ctrl->maxkey, ctrl->sort_lo);
  u64 lo, end;
  bucket_chunk(ctrl->sort_m, lo, end);
  u64 i = lo + threadIdx.x;
  for (; i + (BK_LPT - 1) * 512 < end; i += BK_LPT * 512) {
    u32 d[BK_LPT];
#pragma unroll
    for (int q = 0; q < BK_LPT; q++) d[q] = hi - keys[i + q * 512];
#pragma unroll
    for (int q = 0; q < BK_LPT; q++) atomicAdd(&h[d[q] >> shift], 1u);
  }
  for (; i < end; i += 512) atomicAdd(&h[(hi - keys[i]) >> shift], 1u);
  __syncthreads();
  for (int i = threadIdx.x; i < (int)nb; i += 512)
    bb.counts[(u64)blockIdx.x * BK_MAX + i] = h[i] ? atomicAdd(&bb.total[i], h[i]) : 0u;
}

// Bucket starts = exclusive scan of the bucket totals (every scatter CTA
// does it in shared memory; CTA 0 publishes it).  Decides the fallback.
__device__ __forceinline__ bool bucket_starts(Ctrl* ctrl, const BucketBufs& bb, u32 nb, u32 shift, u32* st) {
  __shared__ u32 wsum[16];
  __shared__ u32 s_max;
  constexpr int PER = BK_MAX / 512;
  if (threadIdx.x == 0) s_max = 0;
  u32 loc[PER], sum = 0, mx = 0;
#pragma unroll
  for (int q = 0; q < PER; q++) {
    const u32 i = threadIdx.x * PER + q;
    loc[q] = i < nb ? bb.total[i] : 0u;
    sum += loc[q];
    mx = max(mx, loc[q]);
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const u32 incl = warp_incl_scan<u32>(sum);
  if (lane == 31) wsum[w] = incl;
  __syncthreads();
  atomicMax(&s_max, mx);
  if (w == 0) {
    const u32 x = lane < 16 ? wsum[lane] : 0u;
    const u32 y = warp_incl_scan<u32>(x);
    if (lane < 16) wsum[lane] = y - x;
  }
  __syncthreads();
  u32 run = wsum[w] + incl - sum;
#pragma unroll
  for (int q = 0; q < PER; q++) {
    const u32 i = threadIdx.x * PER + q;
    if (i < nb) {
      st[i] = run;
      if (blockIdx.x == 0) bb.start[i] = run;
      if (i + 1 == nb) {
        st[nb] = run + loc[q];
        if (blockIdx.x == 0) bb.start[nb] = run + loc[q];
      }
    }
    run += loc[q];
  }
  __syncthreads();
  const bool fb = s_max > (u32)BK_CAP || ctrl->sort_m >= (1ull << 32);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    bb.info[0] = shift;
    bb.info[1] = nb;
    bb.info[2] = fb ? 1u : 0u;
    ctrl->lsd_fallback = fb ? 1u : 0u;
    if (bb.use_cond) cudaGraphSetConditional(bb.c_lsd, fb ? 1u : 0u);
  }
  return fb;
}

__global__ void __launch_bounds__(512) bucket_scatter(Ctrl* ctrl, SortBufs b, BucketBufs bb) {
  if (bucket_skip(ctrl)) return;
  __shared__ u32 cur[BK_MAX + 1];
  u32 shift, nb;
  bucket_geometry(ctrl, shift, nb);
  if (bucket_starts(ctrl, bb, nb, shift, cur)) return;
  for (int i = threadIdx.x; i < (int)nb; i += 512) cur[i] += bb.counts[(u64)blockIdx.x * BK_MAX + i];
  __syncthreads();
  const u32* keys = ctrl->sort_src ? b.kb : b.ka;
  const u32 hi = max(ctrl->maxkey, ctrl->sort_lo);
  u64 lo, end;
  bucket_chunk(ctrl->sort_m, lo, end);
  u64 i = lo + threadIdx.x;
  for (; i + (BK_LPT - 1) * 512 < end; i += BK_LPT * 512) {
    u32 d[BK_LPT];
#pragma unroll
    for (int q = 0; q < BK_LPT; q++) d[q] = hi - keys[i + q * 512];
#pragma unroll
    for (int q = 0; q < BK_LPT; q++) {
      const u32 pos = atomicAdd(&cur[d[q] >> shift], 1u);
      bb.comp[pos] = ((unsigned long long)d[q] << 32) | (u32)(i + q * 512);
    }
  }
  for (; i < end; i += 512) {
    const u32 d = hi - keys[i];
    const u32 pos = atomicAdd(&cur[d >> shift], 1u);
    bb.comp[pos] = ((unsigned long long)d << 32) | (u32)i;
  }
}

template <int MODE>
__global__ void __launch_bounds__(256, 4) bucket_sort(Ctrl* ctrl, SortBufs b, BucketBufs bb, u32* __restrict__ ov,
                                                      long long* __restrict__ oi, long long offset) {
  if (bucket_skip(ctrl) || bb.info[2]) return;
  constexpr int PER = BK_CAP / 256;
  __shared__ unsigned long long tmp[BK_CAP];
  __shared__ u32 hs[BK_SUB + 1];
  __shared__ u32 scr[8];
  const u32 shift = bb.info[0], nb = bb.info[1];
  const u32 s2 = shift > (u32)BK_SUB_BITS ? shift - BK_SUB_BITS : 0u;
  const u64 ko = ctrl->res.k_out;
  const u32 hi = max(ctrl->maxkey, ctrl->sort_lo);
  const u64* idx = ctrl->sort_src ? b.ib : b.ia;
  for (u32 bk = blockIdx.x; bk < nb; bk += gridDim.x) {
    const u32 lo = bb.start[bk], cnt = bb.start[bk + 1] - lo;
    if ((u64)lo >= ko || cnt == 0) continue;  // uniform across the CTA
    for (int i = threadIdx.x; i < BK_SUB; i += 256) hs[i] = 0;
    __syncthreads();
    u32 ss[PER];  // sub << 16 | slot in the sub-bin, then sub << 16 | place in tmp
    unsigned long long ce[PER];  // the bucket's composites, loaded once (all in flight together)
#pragma unroll
    for (int r = 0; r < PER; r++) {
      const u32 i = r * 256 + threadIdx.x;
      ce[r] = i < cnt ? bb.comp[lo + i] : 0ull;
    }
#pragma unroll
    for (int r = 0; r < PER; r++) {
      const u32 i = r * 256 + threadIdx.x;
      if (i < cnt) {
        const u32 sub = ((u32)(ce[r] >> 32) >> s2) & (BK_SUB - 1);
        ss[r] = sub << 16 | atomicAdd(&hs[sub], 1u);
      }
    }
    __syncthreads();
    u32 loc[BK_SUB / 256], sum = 0;
#pragma unroll
    for (int q = 0; q < BK_SUB / 256; q++) {
      loc[q] = hs[threadIdx.x * (BK_SUB / 256) + q];
      sum += loc[q];
    }
    u32 run = block_incl_scan_256<u32>(sum, scr) - sum;
#pragma unroll
    for (int q = 0; q < BK_SUB / 256; q++) {
      hs[threadIdx.x * (BK_SUB / 256) + q] = run;
      run += loc[q];
    }
    if (threadIdx.x == 255) hs[BK_SUB] = run;
    __syncthreads();
#pragma unroll
    for (int r = 0; r < PER; r++) {
      const u32 i = r * 256 + threadIdx.x;
      if (i < cnt) {
        const u32 sub = ss[r] >> 16;
        const u32 place = hs[sub] + (ss[r] & 0xffffu);
        tmp[place] = ce[r];
        ss[r] = sub << 16 | place;
      }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < PER; r++) {
      const u32 i = r * 256 + threadIdx.x;
      if (i < cnt) {
        const u32 sub = ss[r] >> 16;
        const unsigned long long e = tmp[ss[r] & 0xffffu];
        const u32 b0 = hs[sub], b1 = hs[sub + 1];
        u32 rank = b0;
        if (b1 - b0 > 1)
          for (u32 q = b0; q < b1; q++) rank += tmp[q] < e ? 1u : 0u;
        const u64 pos = (u64)lo + rank;
        if (pos < ko) {
          const u32 key = hi - (u32)(e >> 32);
          ov[pos] = from_key<MODE>(key);
          oi[pos] = (long long)idx[(u32)e] + offset;
          if (pos == ko - 1) ctrl->res.kth_key = key;
        }
      }
    }
    __syncthreads();
  }
}

// Write the first k_out sorted pairs in the input dtype (big sorts only).
template <int MODE>
__global__ void __launch_bounds__(256) writeout(Ctrl* ctrl, SortBufs b, u32* __restrict__ ov,
                                                long long* __restrict__ oi, long long offset) {
  if (ctrl->sort_m <= (ull)SMALL_SORT || ctrl->small_done || !ctrl->lsd_fallback) return;
  const int passes = (sort_bits(ctrl) + 7) / 8;
  const bool in_b = ((ctrl->sort_src + (u32)passes) & 1u) != 0;
  const u32* ks = in_b ? b.kb : b.ka;
  const u64* is = in_b ? b.ib : b.ia;
  const u64 ko = ctrl->res.k_out;
  for (u64 i = (u64)blockIdx.x * 256 + threadIdx.x; i < ko; i += (u64)gridDim.x * 256) {
    const u32 key = ks[i];
    ov[i] = from_key<MODE>(key);
    oi[i] = (long long)is[i] + offset;
    if (i == ko - 1) ctrl->res.kth_key = key;
  }
}

// One CTA sorts up to SMALL_SORT pairs in shared memory and writes the first
// k_out: bitonic sort of (maxkey - key) << 32 | position, so equal keys keep
// their (index-ordered) input positions -- a stable descending sort.
template <int MODE>
__global__ void __launch_bounds__(1024) sort_small(Ctrl* ctrl, SortBufs b, u32* __restrict__ ov,
                                                   long long* __restrict__ oi, long long offset) {
  extern __shared__ unsigned long long sk[];  // SMALL_SORT entries (64 KiB, dynamic)
  const u64 m = ctrl->sort_m;
  if (m > (u64)SMALL_SORT || m == 0 || ctrl->small_done) return;
  const u64 ko = ctrl->res.k_out;
  const u32* kA = ctrl->sort_src ? b.kb : b.ka;
  const u64* iA = ctrl->sort_src ? b.ib : b.ia;
  // stable LSD radix sort of d = hi - key over the bits d can occupy (CUB
  // block primitive, 1024 threads x 8 items); input order is index order
  // within equal keys, so the result is (key desc, index asc)
  typedef cub::BlockRadixSort<u32, 1024, 8, u32> Sorter;
  static_assert(sizeof(typename Sorter::TempStorage) <= SMALL_SORT * 8, "sort_small shared memory");
  __shared__ u32 s_lo[32], s_hi[32];
  u32 key_in[8], lo = 0xffffffffu, hi = 0;
#pragma unroll
  for (int j = 0; j < 8; j++) {
    const u32 i = threadIdx.x * 8u + (u32)j;
    key_in[j] = i < m ? kA[i] : kA[0];
    lo = min(lo, key_in[j]);
    hi = max(hi, key_in[j]);
  }
  lo = __reduce_min_sync(FULL, lo);
  hi = __reduce_max_sync(FULL, hi);
  if ((threadIdx.x & 31) == 0) {
    s_lo[threadIdx.x >> 5] = lo;
    s_hi[threadIdx.x >> 5] = hi;
  }
  __syncthreads();
  lo = __reduce_min_sync(FULL, s_lo[threadIdx.x & 31]);
  hi = __reduce_max_sync(FULL, s_hi[threadIdx.x & 31]);
  const u32 dmax = hi - lo;  // every key lies in [lo, hi]
  const int nbits = dmax ? 32 - __clz(dmax) : 0;
  const u32 pad = nbits >= 32 ? 0xffffffffu : ((1u << nbits) - 1u);
  u32 d[8], pos[8];
#pragma unroll
  for (int j = 0; j < 8; j++) {
    const u32 i = threadIdx.x * 8u + (u32)j;
    pos[j] = i;
    d[j] = i < m ? hi - key_in[j] : pad;
  }
  __syncthreads();  // s_lo reads done before the sort reuses shared memory
  if (nbits) Sorter(*reinterpret_cast<typename Sorter::TempStorage*>(sk)).Sort(d, pos, 0, nbits);
#pragma unroll
  for (int j = 0; j < 8; j++) {
    const u32 r = threadIdx.x * 8u + (u32)j;
    if (r < ko) {
      const u32 key = hi - d[j];
      ov[r] = from_key<MODE>(key);
      oi[r] = (long long)iA[pos[j]] + offset;
      if (r == ko - 1) ctrl->res.kth_key = key;
    }
  }
}

}  // namespace dtopk
