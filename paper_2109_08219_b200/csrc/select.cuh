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

struct K2Args {
  const u32* D;
  u64 nD;      // beta * S delegates
  u64 k;
  Ctrl* ctrl;
  u32* selbuf;  // region of CTA c: [c * R, c * R + region_cnt[c])
  u32* region_cnt;
  u64 R;        // delegates per CTA region (multiple of 512)
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

// K2: pass 2 of kth(D) -- one read of D.  CTA c owns the contiguous range
// [c*R, (c+1)*R) of D; its warps histogram digit 2 of the delegates in
// theta's digit-1 bucket and compact them into the CTA's own region of selbuf
// through a shared-memory counter (no global atomics, no barriers in the loop).
__global__ void __launch_bounds__(256) k2_scan_delegates(K2Args a) {
  __shared__ u32 shist[NB2];
  __shared__ DigitResult r1;
  __shared__ ull scratch[8];
  __shared__ u32 s_cnt;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < NB2; i += 256) shist[i] = 0;
  if (tid == 0) s_cnt = 0;
  find_digit<NB1>(a.ctrl->selD.hist1, a.k, &r1, scratch);
  if (blockIdx.x == 0 && tid == 0) a.ctrl->selD.r1 = r1;
  const u32 b1 = r1.digit;
  const u64 lo = (u64)blockIdx.x * a.R;
  const u64 hi = min(a.nD, lo + a.R);
  u32* region = a.selbuf + lo;
  const u32 lt = lanemask_lt();
  for (u64 base = lo + (u64)warp * 512; base < hi; base += 8 * 512) {
    u32 v[16];
    u32 bl[16];
    u32 cnt = 0;
#pragma unroll
    for (int j = 0; j < 16; j++) {
      const u64 i = base + (u64)j * 32 + lane;
      v[j] = i < hi ? a.D[i] : 0u;
    }
#pragma unroll
    for (int j = 0; j < 16; j++) {
      const u64 i = base + (u64)j * 32 + lane;
      const bool p = i < hi && dig1(v[j]) == b1;
      bl[j] = __ballot_sync(FULL, p);
      cnt += __popc(bl[j]);
      if (p) atomicAdd(&shist[dig2(v[j])], 1u);
    }
    if (cnt) {
      u32 o = 0;
      if (lane == 0) o = atomicAdd(&s_cnt, cnt);
      o = __shfl_sync(FULL, o, 0);
#pragma unroll
      for (int j = 0; j < 16; j++) {
        if ((bl[j] >> lane) & 1u) region[o + __popc(bl[j] & lt)] = v[j];
        o += __popc(bl[j]);
      }
    }
  }
  __syncthreads();
  if (tid == 0) a.region_cnt[blockIdx.x] = s_cnt;
  for (int i = tid; i < NB2; i += 256) {
    const u32 c = shist[i];
    if (c) atomicAdd(&a.ctrl->selD.hist2[i], (ull)c);
  }
}

// Pass 3 of kth(D) over the compacted bucket regions; the last CTA resolves theta.
__global__ void __launch_bounds__(256) k2_pass3(Ctrl* ctrl, const u32* __restrict__ selbuf,
                                                const u32* __restrict__ region_cnt, u32 nregions, u64 R) {
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
  for (u32 g = blockIdx.x; g < nregions; g += gridDim.x) {
    const u32 cnt = region_cnt[g];
    const u32* reg = selbuf + (u64)g * R;
    for (u32 i = tid; i < cnt; i += 256) {
      const u32 x = reg[i];
      if (dig2(x) == b2) atomicAdd(&shist[dig3(x)], 1u);
    }
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
    if (threadIdx.x == 0) {
      u32 tot = 0;
      for (int w = 0; w < 8; w++) tot += s_wcnt[w];
      s_base = tot ? atomicAdd(&a.sel->buf_count, (ull)tot) : 0ull;
    }
    __syncthreads();
    u64 o = s_base;
    for (int w = 0; w < warp; w++) o += s_wcnt[w];
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
