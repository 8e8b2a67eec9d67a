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

namespace dtopk {

constexpr int K2_TILE = 2048;  // subranges per tile of the delegate scan
constexpr int K3_TILE = 2048;  // bitmap words (65536 subranges) per qualification tile

struct K2Args {
  const u32* D;
  u64 S;
  int beta;
  u64 k;
  Ctrl* ctrl;
  u32* selbuf;
  u32* bitmap;  // one bit per subrange: max delegate can still reach theta
};

// Warp-aggregated append of `x` (where pred) to buf[*counter++].
__device__ __forceinline__ void warp_append(u32* buf, ull* counter, u32 x, bool pred) {
  const u32 b = __ballot_sync(FULL, pred);
  if (!b) return;
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(b) - 1;
  ull base = 0;
  if (lane == leader) base = atomicAdd(counter, (ull)__popc(b));
  base = __shfl_sync(FULL, base, leader);
  if (pred) buf[base + __popc(b & lanemask_lt())] = x;
}

// K2: one pass over D.
//  * pass 2 of kth(D): histogram of digit 2 for delegates in theta's digit-1
//    bucket, and compaction of that bucket into selbuf;
//  * a bitmap of the subranges whose max delegate can still reach theta
//    (digit1(d_1) >= digit1(theta)), consumed by K3 once theta is exact.
__global__ void __launch_bounds__(256) k2_scan_delegates(K2Args a) {
  __shared__ u32 shist[NB2];
  __shared__ DigitResult r1;
  __shared__ ull scratch[8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < NB2; i += 256) shist[i] = 0;
  find_digit<NB1>(a.ctrl->selD.hist1, a.k, &r1, scratch);
  if (blockIdx.x == 0 && tid == 0) a.ctrl->selD.r1 = r1;
  const u32 b1 = r1.digit;
  const u64 T = (a.S + K2_TILE - 1) / K2_TILE;
  const int beta = a.beta;

  for (u64 tile = blockIdx.x; tile < T; tile += gridDim.x) {
    const u64 base = tile * K2_TILE + (u64)warp * 256;
#pragma unroll 2
    for (int j = 0; j < 8; j++) {
      const u64 sid = base + (u64)j * 32 + lane;
      const bool ok = sid < a.S;
      u32 d1 = 0;
      if (beta == 2) {
        u32 dl = 0;
        if (ok) {
          const uint2 v = *reinterpret_cast<const uint2*>(a.D + sid * 2);
          d1 = v.x;
          dl = v.y;
        }
        const bool p1 = ok && dig1(d1) == b1, p2 = ok && dig1(dl) == b1;
        if (p1) atomicAdd(&shist[dig2(d1)], 1u);
        if (p2) atomicAdd(&shist[dig2(dl)], 1u);
        warp_append(a.selbuf, &a.ctrl->selD.buf_count, d1, p1);
        warp_append(a.selbuf, &a.ctrl->selD.buf_count, dl, p2);
      } else {
        for (int i = 0; i < beta; i++) {
          const u32 d = ok ? a.D[sid * beta + i] : 0u;
          if (i == 0) d1 = d;
          const bool p = ok && dig1(d) == b1;
          if (p) atomicAdd(&shist[dig2(d)], 1u);
          warp_append(a.selbuf, &a.ctrl->selD.buf_count, d, p);
        }
      }
      const u32 word = __ballot_sync(FULL, ok && dig1(d1) >= b1);
      if (lane == 0 && base + (u64)j * 32 < a.S) a.bitmap[(base >> 5) + j] = word;
    }
  }
  __syncthreads();
  for (int i = tid; i < NB2; i += 256) {
    const u32 v = shist[i];
    if (v) atomicAdd(&a.ctrl->selD.hist2[i], (ull)v);
  }
}

struct K3Args {
  const u32* D;
  u64 S;
  int beta;
  const u32* bitmap;
  Ctrl* ctrl;
  const int64_t* theta_override;
  u32* q_sid;
  u32* q_d1;
  u32* q_dl;
  u64* lb;
};

// K3 (qualification, pipeline.py:104-116 without bincount): with the exact
// theta, keep the subranges whose max delegate d_1 >= theta, in subrange order
// (ordered compaction with decoupled look-back); count fully qualified
// (d_beta >= theta) and partially qualified (d_1 >= theta > d_beta) ones.
__global__ void __launch_bounds__(256) k3_qualify(K3Args a) {
  __shared__ u32 s_wcnt[8];
  __shared__ u64 s_tile, s_prefix;
  __shared__ ull s_stat[3][8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  Ctrl* ctrl = a.ctrl;
  u32 theta = ctrl->selD.kth;
  if (a.theta_override) {
    const long long o = *a.theta_override;
    const u32 ov = o < 0 ? 0u : (o > 0xffffffffll ? 0xffffffffu : (u32)o);
    theta = max(theta, ov);
  }
  if (blockIdx.x == 0 && tid == 0) ctrl->res.theta = theta;
  const u64 nwords = (a.S + 31) / 32;
  const u64 T = (nwords + K3_TILE - 1) / K3_TILE;
  const int beta = a.beta;
  ull st_cand = 0, st_fq = 0, st_pq = 0;
  for (;;) {
    if (tid == 0) s_tile = atomicAdd(&ctrl->k3_ticket, 1u);
    __syncthreads();
    const u64 tile = s_tile;
    if (tile >= T) break;
    const u64 wbase = tile * K3_TILE + (u64)warp * 256;
    u32 q[8];
    u32 cnt = 0;
#pragma unroll
    for (int j = 0; j < 8; j++) {
      const u64 w = wbase + (u64)j * 32 + lane;
      u32 bits = w < nwords ? a.bitmap[w] : 0u;
      u32 keep = 0;
      while (bits) {
        const int b = __ffs(bits) - 1;
        bits &= bits - 1;
        const u64 sid = w * 32 + b;
        const u32 d1 = a.D[sid * beta];
        if (d1 >= theta) {
          keep |= 1u << b;
          const u32 dl = a.D[sid * beta + beta - 1];
          st_cand++;
          if (dl >= theta) st_fq++; else st_pq++;
        }
      }
      q[j] = keep;
      cnt += __popc(keep);
    }
    const u32 wsum = __reduce_add_sync(FULL, cnt);
    if (lane == 0) s_wcnt[warp] = wsum;
    __syncthreads();
    if (warp == 0) {
      u64 agg = 0;
      for (int w2 = 0; w2 < 8; w2++) agg += s_wcnt[w2];
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
    for (int w2 = 0; w2 < warp; w2++) pos += s_wcnt[w2];
    // order inside the warp: round j, then lane, then bit
#pragma unroll
    for (int j = 0; j < 8; j++) {
      const u32 c = __popc(q[j]);
      const u32 incl = warp_incl_scan<u32>(c);
      u64 o = pos + incl - c;
      u32 bits = q[j];
      const u64 w = wbase + (u64)j * 32 + lane;
      while (bits) {
        const int b = __ffs(bits) - 1;
        bits &= bits - 1;
        const u64 sid = w * 32 + b;
        a.q_sid[o] = (u32)sid;
        a.q_d1[o] = a.D[sid * beta];
        a.q_dl[o] = a.D[sid * beta + beta - 1];
        o++;
      }
      pos += __shfl_sync(FULL, incl, 31);
    }
  }
  ull v[3] = {st_cand, st_fq, st_pq};
#pragma unroll
  for (int i = 0; i < 3; i++) {
    v[i] = __reduce_add_sync(FULL, (u32)v[i]);
    if (lane == 0) s_stat[i][warp] = v[i];
  }
  __syncthreads();
  if (tid == 0) {
    ull t[3] = {0, 0, 0};
    for (int i = 0; i < 3; i++)
      for (int w2 = 0; w2 < 8; w2++) t[i] += s_stat[i][w2];
    if (t[0]) atomicAdd((ull*)&ctrl->res.candidate_subranges, t[0]);
    if (t[1]) atomicAdd((ull*)&ctrl->res.fully_qualified, t[1]);
    if (t[2]) atomicAdd((ull*)&ctrl->res.partially_qualified, t[2]);
  }
}

// Pass 3 of kth(D) over the compacted bucket; the last CTA resolves theta.
__global__ void __launch_bounds__(256) k2_pass3(Ctrl* ctrl, const u32* __restrict__ selbuf) {
  __shared__ u32 shist[NB3];
  __shared__ DigitResult r2, r3;
  __shared__ ull scratch[8];
  __shared__ int am_last;
  const int tid = threadIdx.x;
  for (int i = tid; i < NB3; i += 256) shist[i] = 0;
  const DigitResult r1 = ctrl->selD.r1;
  find_digit<NB2>(ctrl->selD.hist2, r1.rem, &r2, scratch);
  if (blockIdx.x == 0 && tid == 0) ctrl->selD.r2 = r2;
  const u32 b2 = r2.digit;
  const u64 m = r1.cnt;
  for (u64 i = (u64)blockIdx.x * 256 + tid; i < m; i += (u64)gridDim.x * 256) {
    const u32 x = selbuf[i];
    if (dig2(x) == b2) atomicAdd(&shist[dig3(x)], 1u);
  }
  __syncthreads();
  for (int i = tid; i < NB3; i += 256) {
    const u32 v = shist[i];
    if (v) atomicAdd(&ctrl->selD.hist3[i], (ull)v);
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) am_last = atomicAdd(&ctrl->selD.done3, 1u) == gridDim.x - 1;
  __syncthreads();
  if (am_last) {
    __threadfence();
    find_digit<NB3>(ctrl->selD.hist3, r2.rem, &r3, scratch);
    if (tid == 0) {
      const u32 kth = (r1.digit << 21) | (b2 << 10) | r3.digit;
      ctrl->selD.r3 = r3;
      ctrl->selD.kth = kth;
      ctrl->res.theta_local = kth;
      ctrl->res.theta_slot = (int64_t)kth;
      ctrl->res.delegate_bucket = r1.cnt;
    }
  }
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
};

__device__ __forceinline__ bool sel_skip(const SelArgs& a) {
  return a.check_path && ld_volatile_u32(&a.ctrl->res.path) != PATH_SELECT;
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
  for (int i = threadIdx.x; i < NB2; i += 256) shist[i] = 0;
  find_digit<NB1>(a.sel->hist1, a.k, &r1, scratch);
  if (blockIdx.x == 0 && threadIdx.x == 0) a.sel->r1 = r1;
  const u32 b1 = r1.digit;
  const u64 m = sel_count(a);
  const u64 stride = (u64)gridDim.x * 256;
  const u64 m_pad = (m + 31) & ~31ull;  // whole warps for warp_append
  for (u64 i = (u64)blockIdx.x * 256 + threadIdx.x; i < m_pad; i += stride) {
    const u32 x = i < m ? to_key<MODE>(a.keys[i]) : 0u;
    const bool p = i < m && dig1(x) == b1;
    if (p) atomicAdd(&shist[dig2(x)], 1u);
    warp_append(a.selbuf, &a.sel->buf_count, x, p);
  }
  __syncthreads();
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
  const u64 m = r1.cnt;
  for (u64 i = (u64)blockIdx.x * 256 + threadIdx.x; i < m; i += (u64)gridDim.x * 256) {
    const u32 x = a.selbuf[i];
    if (dig2(x) == b2) atomicAdd(&shist[dig3(x)], 1u);
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
