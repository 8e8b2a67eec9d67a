// fast.cuh -- one-CTA finish of small calls: theta resolution, qualification,
// concatenation and the second top-k in a single kernel after K2.
//
// Reference semantics are those of select.cuh / assemble.cuh (the exact
// theta = kth(D) of radix_topk kernels.py:109-165, first_topk qualification
// pipeline.py:104-116, concatenate_filtered pipeline.py:119-159, the exact
// second top-k kernels.py:83-96 + np.sort, pipeline.py:212-220), restated for
// the case where everything after K2 fits in one CTA's shared memory:
//   * theta's first-digit bucket holds <= FT_BUCKET delegates, compacted by K2
//     (only when `resolve`: otherwise K2 pass 3 has resolved theta already);
//   * the candidate superset (K2, subrange order) has <= FT_SUP entries and at
//     most FT_CAND of them reach theta;
//   * the E / T candidates (the only ones whose keys are re-read) hold at most
//     FT_REREAD keys;
//   * the pool (keys > theta, plus the first k - |P_gt| ties on the merge
//     path) has at most SMALL_POOL pairs, and no FT_RUN + 1 of its keys > theta
//     fall into one of the 8192 buckets of its sort.
// That is every small-k call on ordinary data: at N = 2^30, k = 1024 the bucket
// holds ~1.5k delegates, there are ~1.04k superset entries, one fully qualified
// candidate (2048 keys re-read) and a ~1.03k-pair pool.  The kernel replaces
// K2 pass 3, K2b, K3, K4, K4T, K5 (count, emit), K5b, K6 and finish_small --
// ten dependent launches, mostly of idle CTAs -- with one launch whose critical
// path is four rounds of global loads.  When a condition fails it writes
// nothing the general chain depends on and leaves the call to that chain (in
// a CUDA-graph plan through a conditional node, so the chain is not even
// launched when the fast path succeeded; eagerly, every chain kernel returns at
// once when ctrl->small_done is set).
#pragma once

#include "assemble.cuh"
#include "common.cuh"
#include "select.cuh"

namespace dtopk {

constexpr int FT_THREADS = 1024;
constexpr int FT_CAND = 4096;         // qualifying candidates held in shared memory
constexpr u32 FT_SUP = 16384;         // superset entries scanned
constexpr u64 FT_REREAD = 1u << 16;   // keys of E / T candidates re-read
constexpr int FT_SEG_CAP = 6208;      // superset segments (<= 768 K2 CTAs x 8 warps) + 1
constexpr int FT_MAX_ALPHA = 18;      // pool sources pack (candidate << alpha | offset) in 32 bits
constexpr int FT_ET = 1024;           // E / T candidates (one per thread in their prefix)
constexpr int FT_RPT = 4;             // superset records per thread and step
constexpr int FT_KPT = 8;             // re-read keys per thread and step
constexpr int FT_BUCKET = 8192;       // theta bucket members resolved here (8 per thread)
constexpr int FT_SORT_BINS = 8192;    // bucket sort of the pool
constexpr int FT_RUN = 32;            // longest equal-bucket run the bucket sort fixes up serially
static_assert(P3_REGIONS <= SMALL_POOL, "region prefix aliases the pool keys");

// dynamic shared memory layout (bytes).  Front part (offsets, segment inputs,
// candidate fields) is reused: by the delegate digit-3 histogram before the
// candidates exist, and by the pool sort after they are consumed.
constexpr size_t FT_OFF = 0;                           // u32 [FT_SEG_CAP] superset segment offsets
constexpr size_t FT_IN = FT_OFF + FT_SEG_CAP * 4;      // u32 [FT_SEG_CAP] superset segment first slots
constexpr size_t FT_CKEY = FT_IN + FT_SEG_CAP * 4;     // u32 [FT_CAND] d_1
constexpr size_t FT_CP1 = FT_CKEY + FT_CAND * 4;       // u32 [FT_CAND] K1 meta
constexpr size_t FT_CG = FT_CP1 + FT_CAND * 4;         // u32 [FT_CAND] keys > theta, then position
constexpr size_t FT_CE = FT_CG + FT_CAND * 4;          // u32 [FT_CAND] ties, then tie position
constexpr size_t FT_CCLS = FT_CE + FT_CAND * 4;        // u8  [FT_CAND] class
constexpr size_t FT_FRONT = FT_CCLS + FT_CAND;
constexpr size_t FT_CSID = FT_FRONT;                   // u32 [FT_CAND] subrange
constexpr size_t FT_PKEY = FT_CSID + FT_CAND * 4;      // u32 [SMALL_POOL] pool keys
constexpr size_t FT_PSRC = FT_PKEY + SMALL_POOL * 4;   // u32 [SMALL_POOL] pool sources
constexpr size_t FT_ETC = FT_PSRC + SMALL_POOL * 4;    // u32 [FT_ET]
constexpr size_t FT_ETG = FT_ETC + FT_ET * 4;
constexpr size_t FT_ETE = FT_ETG + FT_ET * 4;
constexpr size_t FT_SMEM = FT_ETE + FT_ET * 4;
constexpr size_t FT_H3 = FT_CKEY;                      // u32 [NBD3] digit-3 histogram (resolve)
constexpr size_t FT_SHIST = 0;                         // u32 [FT_SORT_BINS] pool sort
constexpr size_t FT_SD = FT_SHIST + FT_SORT_BINS * 4;  // u32 [SMALL_POOL] sorted d
constexpr size_t FT_SP = FT_SD + SMALL_POOL * 4;       // u32 [SMALL_POOL] sorted positions
static_assert(FT_SMEM <= 227 * 1024, "fast_tail shared memory");
static_assert(FT_H3 + NBD3 * 4 <= FT_CCLS, "digit-3 histogram alias");
static_assert(FT_SP + SMALL_POOL * 4 <= FT_FRONT, "pool sort alias");

struct FTArgs {
  Ctrl* ctrl;
  const u32* keys;
  u64 n;
  int alpha;
  int beta;
  u64 k;
  u64 nD;
  const u32* D;
  const uint4* sup_sid;
  const u32* sup_in;
  const u32* sup_cnt;  // resolve: K2's per-segment counts
  const u32* sup_off;  // !resolve: pass 3's segment offsets
  u32 nseg;
  // theta resolution (resolve != 0): K2's compacted bucket members
  int resolve;
  const u32* selbuf;
  const u32* region_cnt;
  u32 nregions;
  u64 R;
  const int64_t* theta_override;
  u32* ov;
  long long* oi;
  long long offset;
  cudaGraphConditionalHandle cond;  // "run the general chain" (graph plans)
  int use_cond;
};

// Inclusive scan over a 1024-thread block; all threads call. scratch >= 32 T.
template <typename T>
__device__ __forceinline__ T block_incl_scan_1024(T v, T* scratch) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  v = warp_incl_scan(v);
  if (lane == 31) scratch[w] = v;
  __syncthreads();
  if (w == 0) {
    T x = scratch[lane];
    x = warp_incl_scan(x);
    scratch[lane] = x;
  }
  __syncthreads();
  const T add = w ? scratch[w - 1] : (T)0;
  __syncthreads();
  return v + add;
}

// Digit finder for a 1024-thread block over per-thread bin counts: thread t
// holds bins NB-1-t*PER .. NB-PER-t*PER (descending, loc[0] the highest).
template <int PER>
__device__ __forceinline__ void ft_find_digit(const ull (&loc)[PER], int NB, ull k_rem, DigitResult* out, ull* scratch) {
  ull sum = 0;
#pragma unroll
  for (int i = 0; i < PER; i++) sum += loc[i];
  if (threadIdx.x == 0) out->valid = 0;
  const ull incl = block_incl_scan_1024<ull>(sum, scratch);
  ull run = incl - sum;
#pragma unroll
  for (int i = 0; i < PER; i++) {
    const int b = NB - 1 - ((int)threadIdx.x * PER + i);
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

// Pool order: positions [0, G) hold keys > theta in index order, [G, m) ties in
// index order.  The answer is the keys > theta by (key desc, position asc), then
// the ties.  Keys > theta: bucket sort on the top bits of d = hi - key (8192
// buckets; pools of <= 8192 spread over the key range leave buckets nearly
// empty), then each multi-entry bucket ordered by (d, position) serially.
// Returns false (nothing written) if some bucket run is longer than FT_RUN.
template <int MODE>
__device__ bool ft_bucket_sort_write(const FTArgs& a, u32 G, u32 m, u32 ko, u32 theta, u32 hi, const u32* pkey,
                                     const u32* psrc, const u32* csid, unsigned char* sm, ull* scratch) {
  u32* hist = reinterpret_cast<u32*>(sm + FT_SHIST);
  u32* sd = reinterpret_cast<u32*>(sm + FT_SD);
  u32* sp = reinterpret_cast<u32*>(sm + FT_SP);
  const int tid = threadIdx.x;
  const u32 range = hi - theta;
  const int nbits = range ? 32 - __clz(range) : 0;
  const int shift = nbits > 13 ? nbits - 13 : 0;
  const u32 ng = min(G, m);
  __syncthreads();  // the sort storage aliases dead candidate fields
  for (int i = tid; i < FT_SORT_BINS; i += FT_THREADS) hist[i] = 0;
  __syncthreads();
  constexpr int PT = SMALL_POOL / FT_THREADS;
  u32 d[PT], b[PT], slot[PT];
#pragma unroll
  for (int j = 0; j < PT; j++) {
    const u32 i = (u32)j * FT_THREADS + tid;
    d[j] = i < ng ? hi - pkey[i] : 0u;
    b[j] = d[j] >> shift;
    slot[j] = i < ng ? atomicAdd(&hist[b[j]], 1u) : 0u;
  }
  __syncthreads();
  // exclusive bucket starts (8 bins per thread), longest run
  constexpr int BPT = FT_SORT_BINS / FT_THREADS;
  u32 c[BPT], sum = 0, mx = 0;
#pragma unroll
  for (int q = 0; q < BPT; q++) {
    c[q] = hist[tid * BPT + q];
    sum += c[q];
    mx = max(mx, c[q]);
  }
  const u32 incl = block_incl_scan_1024<u32>(sum, reinterpret_cast<u32*>(scratch));
  mx = __reduce_max_sync(FULL, mx);
  __shared__ u32 s_mx;
  if (tid == 0) s_mx = 0;
  __syncthreads();
  if ((tid & 31) == 0) atomicMax(&s_mx, mx);
  u32 run = incl - sum;
#pragma unroll
  for (int q = 0; q < BPT; q++) {
    hist[tid * BPT + q] = run;
    run += c[q];
  }
  __syncthreads();
  if (s_mx > (u32)FT_RUN) return false;
#pragma unroll
  for (int j = 0; j < PT; j++) {
    const u32 i = (u32)j * FT_THREADS + tid;
    if (i < ng) {
      const u32 p = hist[b[j]] + slot[j];
      sd[p] = d[j];
      sp[p] = i;
    }
  }
  __syncthreads();
  // order each run of equal buckets by (d, position)
#pragma unroll
  for (int q = 0; q < BPT; q++) {
    const u32 cnt = c[q];
    if (cnt < 2) continue;
    const u32 s0 = hist[tid * BPT + q];
    for (u32 x = s0 + 1; x < s0 + cnt; x++) {
      const u32 kd = sd[x], kp = sp[x];
      u32 y = x;
      while (y > s0 && (sd[y - 1] > kd || (sd[y - 1] == kd && sp[y - 1] > kp))) {
        sd[y] = sd[y - 1];
        sp[y] = sp[y - 1];
        y--;
      }
      sd[y] = kd;
      sp[y] = kp;
    }
  }
  __syncthreads();
  const u32 wmask = (1u << a.alpha) - 1u;
  for (u32 r = tid; r < ko; r += FT_THREADS) {
    u32 key, pos;
    if (r < ng) {
      key = hi - sd[r];
      pos = sp[r];
    } else {
      key = theta;
      pos = r;  // ties keep their pool order
    }
    const u32 src = psrc[pos];
    const u64 idx = ((u64)csid[src >> a.alpha] << a.alpha) | (src & wmask);
    a.ov[r] = from_key<MODE>(key);
    a.oi[r] = (long long)idx + a.offset;
    if (r == ko - 1) a.ctrl->res.kth_key = key;
  }
  return true;
}

#ifdef DTOPK_FT_PROFILE
#define FT_MARK(i)                             \
  do {                                         \
    __syncthreads();                           \
    if (threadIdx.x == 0) ft_t[i] = clock64(); \
  } while (0)
#else
#define FT_MARK(i) \
  do {             \
  } while (0)
#endif

template <int MODE>
__global__ void __launch_bounds__(FT_THREADS, 1) fast_tail(FTArgs a) {
  pdl_trigger();
  pdl_wait();
#ifdef DTOPK_FT_PROFILE
  __shared__ long long ft_t[12];
#endif
  FT_MARK(0);
  extern __shared__ __align__(16) unsigned char ft_sm[];
  u32* s_off = reinterpret_cast<u32*>(ft_sm + FT_OFF);
  u32* s_in = reinterpret_cast<u32*>(ft_sm + FT_IN);
  u32* c_key = reinterpret_cast<u32*>(ft_sm + FT_CKEY);
  u32* c_p1 = reinterpret_cast<u32*>(ft_sm + FT_CP1);
  u32* c_g = reinterpret_cast<u32*>(ft_sm + FT_CG);
  u32* c_e = reinterpret_cast<u32*>(ft_sm + FT_CE);
  unsigned char* c_cls = ft_sm + FT_CCLS;
  u32* c_sid = reinterpret_cast<u32*>(ft_sm + FT_CSID);
  u32* p_key = reinterpret_cast<u32*>(ft_sm + FT_PKEY);
  u32* p_src = reinterpret_cast<u32*>(ft_sm + FT_PSRC);
  u32* et_c = reinterpret_cast<u32*>(ft_sm + FT_ETC);  // candidate of the j-th E/T candidate
  u32* et_g = reinterpret_cast<u32*>(ft_sm + FT_ETG);  // its keys > theta, then their flat prefix
  u32* et_e = reinterpret_cast<u32*>(ft_sm + FT_ETE);  // its ties, then their flat prefix
  __shared__ ull scratch[32];
  __shared__ u32 s_ncand, s_bail, s_hi, s_nre, s_total, s_G, s_E, s_chunk;
  __shared__ ull s_stat[4];  // fq, pq, concat, reread
  __shared__ DigitResult s_r2, s_r3;
  const int tid = threadIdx.x, lane = tid & 31;
  Ctrl* ctrl = a.ctrl;
  u32* scr = reinterpret_cast<u32*>(scratch);
  const int alpha = a.alpha, beta = a.beta;
  const u64 W = 1ull << alpha;
  const u32 nseg = a.nseg;
  bool ok = nseg + 1 <= (u32)FT_SEG_CAP && alpha <= FT_MAX_ALPHA && alpha >= 1 && a.sup_sid != nullptr;
  if (tid == 0) {
    s_ncand = 0;
    s_bail = 0;
  }
  if (tid < 4) s_stat[tid] = 0;
  constexpr int SPT = (FT_SEG_CAP + FT_THREADS - 1) / FT_THREADS;  // segments per thread
  u32 theta;
  if (a.resolve) {
    // ---- R: theta = kth(D) from K2's compacted bucket (round 1: digit-1 result,
    // digit-2 histogram, region and segment counts, segment first slots)
    const DigitResult r1 = ctrl->selD.r1;
    ull h2[NBD2 / FT_THREADS];
    {
      const ulonglong2* p = reinterpret_cast<const ulonglong2*>(ctrl->selD.hist2 + NBD2 - 4 - tid * 4);
      const ulonglong2 q0 = __ldcg(p), q1 = __ldcg(p + 1);
      h2[3] = q0.x;
      h2[2] = q0.y;
      h2[1] = q1.x;
      h2[0] = q1.y;
    }
    const u32 rc = (u32)tid < a.nregions ? a.region_cnt[tid] : 0u;
    u32 sc[SPT];
#pragma unroll
    for (int q = 0; q < SPT; q++) {
      const u32 g = (u32)tid * SPT + q;
      sc[q] = (ok && g < nseg) ? a.sup_cnt[g] : 0u;
      if (ok && g < nseg) s_in[g] = a.sup_in[g];
    }
    ok = ok && r1.cnt * 4 <= a.nD && r1.cnt <= (ull)FT_BUCKET && a.nregions <= (u32)FT_THREADS && r1.valid;
    if (!ok) {  // uniform: every thread read the same r1
      if (tid == 0 && a.use_cond) cudaGraphSetConditional(a.cond, 1u);
      return;
    }
    u32 kmin, kmax;
    dbucket(r1.digit, MODE >= 2, kmin, kmax);
    ft_find_digit<NBD2 / FT_THREADS>(h2, NBD2, r1.rem, &s_r2, scratch);
    const u32 b2 = s_r2.digit;
    // region prefix (aliases the pool keys, unused until phase D), digit-3 histogram
    u32* s_rpre = p_key;
    u32* h3 = reinterpret_cast<u32*>(ft_sm + FT_H3);
    const u32 ri = block_incl_scan_1024<u32>(rc, scr);
    if ((u32)tid < a.nregions) s_rpre[tid] = ri - rc;
    for (int i = tid; i < NBD3; i += FT_THREADS) h3[i] = 0;
    // superset segment offsets
    u32 ssum = 0;
#pragma unroll
    for (int q = 0; q < SPT; q++) ssum += sc[q];
    const u32 si = block_incl_scan_1024<u32>(ssum, scr);
    {
      u32 run = si - ssum;
#pragma unroll
      for (int q = 0; q < SPT; q++) {
        const u32 g = (u32)tid * SPT + q;
        if (g <= nseg) s_off[g] = run;
        run += sc[q];
      }
    }
    if (tid == FT_THREADS - 1) s_total = si;
    __syncthreads();
    // round 2: the bucket members; digit 3 of those in digit-2 bucket b2
    const u32 nm = (u32)r1.cnt;
    constexpr int MPT = FT_BUCKET / FT_THREADS;
    u32 x[MPT];
#pragma unroll
    for (int j = 0; j < MPT; j++) {
      const u32 i = (u32)j * FT_THREADS + tid;
      x[j] = 0xffffffffu;
      if (i < nm) {
        u32 lo = 0, hi = a.nregions;  // last region whose prefix is <= i
        while (hi - lo > 1) {
          const u32 mid = (lo + hi) >> 1;
          if (s_rpre[mid] <= i) lo = mid; else hi = mid;
        }
        x[j] = a.selbuf[(u64)lo * a.R + (i - s_rpre[lo])] - kmin;
      }
    }
#pragma unroll
    for (int j = 0; j < MPT; j++)
      if (x[j] != 0xffffffffu && (x[j] >> DSH3) == b2) atomicAdd(&h3[x[j] & ((1u << DSH3) - 1u)], 1u);
    __syncthreads();
    ull h3l[NBD3 / FT_THREADS];
#pragma unroll
    for (int i = 0; i < NBD3 / FT_THREADS; i++) h3l[i] = h3[NBD3 - 1 - (tid * (NBD3 / FT_THREADS) + i)];
    ft_find_digit<NBD3 / FT_THREADS>(h3l, NBD3, s_r2.rem, &s_r3, scratch);
    const u32 kth = kmin + (b2 << DSH3) + s_r3.digit;
    if (tid == 0) {
      ctrl->selD.r2 = s_r2;
      ctrl->selD.r3 = s_r3;
      ctrl->selD.kth = kth;
      ctrl->res.theta_local = kth;
      ctrl->res.theta_slot = (int64_t)kth;
      ctrl->res.delegate_bucket = r1.cnt;
      ctrl->sup_total = s_total;
    }
    theta = kth;
  } else {
    theta = ctrl->selD.kth;
    if (ok) {
      for (u32 i = tid; i <= nseg; i += FT_THREADS) {
        s_off[i] = a.sup_off[i];
        if (i < nseg) s_in[i] = a.sup_in[i];
      }
    }
    if (tid == 0) s_total = ctrl->sup_total;
  }
  if (a.theta_override) {
    const long long o = *a.theta_override;
    const u32 ovr = o < 0 ? 0u : (o > 0xffffffffll ? 0xffffffffu : (u32)o);
    theta = max(theta, ovr);
  }
  if (tid == 0) s_hi = theta;
  __syncthreads();
  const u32 total = s_total;
  ok = ok && total <= FT_SUP;
  FT_MARK(1);
  // ---- A: qualification of the superset (FT_RPT consecutive records per thread,
  // their loads in flight together), ordered compaction of the candidates
  ull st_fq = 0, st_pq = 0;
  for (u32 r0 = 0; ok && r0 < total; r0 += FT_THREADS * FT_RPT) {
    u32 sid[FT_RPT], d1[FT_RPT], d2[FT_RPT], dl[FT_RPT], m[FT_RPT];
    bool keep[FT_RPT];
    u32 seg = 0;
    {
      const u32 r = r0 + (u32)tid * FT_RPT;
      u32 lo = 0, hi = nseg;  // last segment whose first record is <= r
      while (hi - lo > 1) {
        const u32 mid = (lo + hi) >> 1;
        if (s_off[mid] <= r) lo = mid; else hi = mid;
      }
      seg = lo;
    }
#pragma unroll
    for (int q = 0; q < FT_RPT; q++) {
      const u32 r = r0 + (u32)tid * FT_RPT + q;
      keep[q] = false;
      sid[q] = d1[q] = d2[q] = dl[q] = m[q] = 0;
      if (r < total) {
        while (seg + 1 < nseg && s_off[seg + 1] <= r) seg++;
        const uint4 e = a.sup_sid[(u64)s_in[seg] + (r - s_off[seg])];
        sid[q] = e.x;
        d1[q] = e.y;
        d2[q] = e.z;
        dl[q] = e.z;
        m[q] = e.w;
        keep[q] = e.y >= theta;
      }
    }
    u32 nk = 0;
#pragma unroll
    for (int q = 0; q < FT_RPT; q++) {
      if (keep[q]) {
        if (beta == 1) {  // d_beta = d_1 (D may be unwritten: filtered K1 pass)
          d2[q] = d1[q];
          dl[q] = d1[q];
        } else if (beta != 2) {
          d2[q] = a.D[(u64)sid[q] * beta + 1];
          dl[q] = a.D[(u64)sid[q] * beta + beta - 1];
        }
        nk++;
      }
    }
    const u32 incl = block_incl_scan_1024<u32>(nk, scr);
    const u32 base = s_ncand;
    u32 c = base + incl - nk;
#pragma unroll
    for (int q = 0; q < FT_RPT; q++) {
      if (!keep[q]) continue;
      if (dl[q] >= theta) st_fq++; else st_pq++;
      if (c < (u32)FT_CAND) {
        c_sid[c] = sid[q];
        c_key[c] = d1[q];
        c_p1[c] = m[q];
        c_cls[c] = (unsigned char)classify(d1[q], d2[q], m[q], theta, beta);
      }
      c++;
    }
    __syncthreads();
    if (tid == FT_THREADS - 1) {
      s_ncand = base + incl;
      if (base + incl > (u32)FT_CAND) s_bail = 1;
    }
    __syncthreads();
    ok = !s_bail;
  }
  FT_MARK(2);
  const u32 nc = min(s_ncand, (u32)FT_CAND);
  // ---- B: counts of A / B / C candidates; ordered list of the E / T candidates
  // (the only ones whose keys are re-read)
  constexpr int CPT = FT_CAND / FT_THREADS;
  u32 nre = 0;
  if (ok) {
    u32 ne = 0;
#pragma unroll
    for (int q = 0; q < CPT; q++) {
      const u32 c = (u32)tid * CPT + q;
      if (c >= nc) continue;
      const u32 cls = c_cls[c];
      u32 g = 0, e = 0;
      if (cls == CLS_A) g = 1;
      else if (cls == CLS_B) e = 1;
      else if (cls == CLS_C) e = (u32)sub_len(c_sid[c], a.n, alpha);
      else ne++;
      c_g[c] = g;
      c_e[c] = e;
    }
    const u32 incl = block_incl_scan_1024<u32>(ne, scr);
    if (tid == FT_THREADS - 1) s_nre = incl;
    u32 j = incl - ne;
#pragma unroll
    for (int q = 0; q < CPT; q++) {
      const u32 c = (u32)tid * CPT + q;
      if (c < nc && c_cls[c] >= CLS_T && c_cls[c] <= CLS_E) {
        if (j < (u32)FT_ET) {
          et_c[j] = c;
          et_g[j] = 0;
          et_e[j] = 0;
        }
        j++;
      }
    }
    __syncthreads();
    nre = s_nre;
    ok = nre <= (u32)FT_ET && (u64)nre * W <= FT_REREAD;
  }
  if (!ok) {
    if (tid == 0 && a.use_cond) cudaGraphSetConditional(a.cond, 1u);
    return;
  }
  FT_MARK(3);
  // E / T keys as one flat range: flat index i -> (E/T candidate i >> alpha,
  // offset i & (W - 1)); every thread takes FT_KPT consecutive keys per chunk
  const u64 flat = (u64)nre * W;
  const bool vec = alpha >= 3;  // 8 consecutive keys share a candidate, 32-byte aligned
  auto load8 = [&](u64 i0, u32 (&x)[FT_KPT], u32& valid, u32& jj) {
    valid = 0;
    jj = (u32)(i0 >> alpha);
    if (i0 >= flat) return;
    const u64 b = (u64)c_sid[et_c[jj]] << alpha;
    const u64 len = min(W, a.n - b);
    const u64 off = i0 & (W - 1);
    if (vec && off + FT_KPT <= len) {
      const uint4* p = reinterpret_cast<const uint4*>(a.keys + b + off);
      const uint4 q0 = ld_nc_v4(p), q1 = ld_nc_v4(p + 1);
      x[0] = q0.x; x[1] = q0.y; x[2] = q0.z; x[3] = q0.w;
      x[4] = q1.x; x[5] = q1.y; x[6] = q1.z; x[7] = q1.w;
      valid = 0xffu;
    } else {
#pragma unroll
      for (int q = 0; q < FT_KPT; q++) {
        const u64 i = i0 + q;
        const u32 j = (u32)(i >> alpha);
        x[q] = 0;
        if (i < flat) {
          const u64 bq = (u64)c_sid[et_c[j]] << alpha;
          const u64 oq = i & (W - 1);
          if (oq < min(W, a.n - bq)) {
            x[q] = a.keys[bq + oq];
            valid |= 1u << q;
          }
        }
      }
    }
#pragma unroll
    for (int q = 0; q < FT_KPT; q++) x[q] = to_key<MODE>(x[q]);
  };
  ull st_reread = 0;
  for (u64 i0 = 0; i0 < flat; i0 += (u64)FT_THREADS * FT_KPT) {
    u32 x[FT_KPT], valid, j0;
    load8(i0 + (u64)tid * FT_KPT, x, valid, j0);
    st_reread += __popc(valid);
    if (vec) {  // the 8 keys share candidate j0; whole warps usually share it too
      u32 ng = 0, ne = 0;
#pragma unroll
      for (int q = 0; q < FT_KPT; q++) {
        const bool v = (valid >> q) & 1u;
        ng += v && x[q] > theta;
        ne += v && x[q] == theta;
      }
      const u32 jl = __shfl_sync(FULL, j0, 0);
      if (__all_sync(FULL, valid == 0u || j0 == jl)) {
        ng = __reduce_add_sync(FULL, ng);
        ne = __reduce_add_sync(FULL, ne);
        if (lane == 0) {
          if (ng) atomicAdd(&et_g[jl], ng);
          if (ne) atomicAdd(&et_e[jl], ne);
        }
      } else {
        if (ng) atomicAdd(&et_g[j0], ng);
        if (ne) atomicAdd(&et_e[j0], ne);
      }
    } else {
#pragma unroll
      for (int q = 0; q < FT_KPT; q++) {
        const u32 j = (u32)((i0 + (u64)tid * FT_KPT + q) >> alpha);
        const bool v = (valid >> q) & 1u;
        if (v && x[q] > theta) atomicAdd(&et_g[j], 1u);
        if (v && x[q] == theta) atomicAdd(&et_e[j], 1u);
      }
    }
  }
  __syncthreads();
  for (u32 j = tid; j < nre; j += FT_THREADS) {
    c_g[et_c[j]] = et_g[j];
    c_e[et_c[j]] = et_e[j];
  }
  __syncthreads();
  FT_MARK(4);
  // ---- C: exclusive positions (candidate order = index order), pool shape;
  // (keys > theta, ties) scanned together as one u64 (g << 32 | e)
  ull lge[CPT], sge = 0;
#pragma unroll
  for (int q = 0; q < CPT; q++) {
    const u32 c = (u32)tid * CPT + q;
    lge[q] = c < nc ? (((ull)c_g[c] << 32) | c_e[c]) : 0ull;
    sge += lge[q];
  }
  const ull ige = block_incl_scan_1024<ull>(sge, scratch);
  if (tid == FT_THREADS - 1) {
    s_G = (u32)(ige >> 32);
    s_E = (u32)ige;
  }
  {
    ull rge = ige - sge;
#pragma unroll
    for (int q = 0; q < CPT; q++) {
      const u32 c = (u32)tid * CPT + q;
      if (c < nc) {
        c_g[c] = (u32)(rge >> 32);  // c_g / c_e now hold exclusive positions
        c_e[c] = (u32)rge;
      }
      rge += lge[q];
    }
  }
  // flat prefixes of the E / T candidates' counts (nre <= FT_ET = FT_THREADS)
  {
    const ull v = (u32)tid < nre ? (((ull)et_g[tid] << 32) | et_e[tid]) : 0ull;
    const ull xv = block_incl_scan_1024<ull>(v, scratch) - v;
    if ((u32)tid < nre) {
      et_g[tid] = (u32)(xv >> 32);
      et_e[tid] = (u32)xv;
    }
  }
  __syncthreads();
  const u64 G = s_G, E = s_E;
  const u64 k = a.k;
  const bool sel = G >= k;
  const u64 ko = sel ? k : min(k, G + E);
  const u64 m = sel ? G : ko;
  if (m > (u64)SMALL_POOL || m == 0) {
    if (tid == 0 && a.use_cond) cudaGraphSetConditional(a.cond, 1u);
    return;
  }
  FT_MARK(5);
  // ---- D: fill the pool (positions: keys > theta at [0, G), ties at G + tie rank)
  const u32 wmask = (u32)(W - 1);
  u32 hi = theta;
  for (u32 c = tid; c < nc; c += FT_THREADS) {
    const u32 cls = c_cls[c];
    const u32 p1 = meta_p1(c_p1[c]) & wmask;
    if (cls == CLS_A) {
      p_key[c_g[c]] = c_key[c];
      p_src[c_g[c]] = (c << alpha) | p1;
      hi = max(hi, c_key[c]);
    } else if (cls == CLS_B) {
      const u64 p = G + c_e[c];
      if (p < m) {
        p_key[p] = theta;
        p_src[p] = (c << alpha) | p1;
      }
    } else if (cls == CLS_C) {
      const u64 p0 = G + c_e[c];
      const u64 len = sub_len(c_sid[c], a.n, alpha);
      for (u64 z = 0; z < len && p0 + z < m; z++) {
        p_key[p0 + z] = theta;
        p_src[p0 + z] = (c << alpha) | (u32)z;
      }
    }
  }
  FT_MARK(6);
  // E / T keys: a block scan per chunk of the (> theta, == theta) flags in flat
  // order gives every key its rank inside its candidate
  u32 fg = 0, fe = 0;  // flat counts of the chunks before this one
  for (u64 i0 = 0; i0 < flat; i0 += (u64)FT_THREADS * FT_KPT) {
    u32 x[FT_KPT], valid, j0;
    const u64 ib = i0 + (u64)tid * FT_KPT;
    load8(ib, x, valid, j0);
    u32 ng = 0, ne = 0;
#pragma unroll
    for (int q = 0; q < FT_KPT; q++) {
      const bool v = (valid >> q) & 1u;
      ng += v && x[q] > theta;
      ne += v && x[q] == theta;
    }
    const u32 packed = ng | (ne << 16);
    const u32 incl = block_incl_scan_1024<u32>(packed, scr);
    if (tid == FT_THREADS - 1) s_chunk = incl;
    u32 rg = fg + ((incl - packed) & 0xffffu), re = fe + ((incl - packed) >> 16);
#pragma unroll
    for (int q = 0; q < FT_KPT; q++) {
      if (!((valid >> q) & 1u)) continue;
      const u32 j = vec ? j0 : (u32)((ib + q) >> alpha);
      const u32 c = et_c[j];
      const u32 o = (u32)((ib + q) & (W - 1));
      if (x[q] > theta) {
        const u32 p = c_g[c] + (rg - et_g[j]);
        p_key[p] = x[q];
        p_src[p] = (c << alpha) | o;
        hi = max(hi, x[q]);
        rg++;
      } else if (x[q] == theta) {
        const u64 p = G + c_e[c] + (re - et_e[j]);
        if (p < m) {
          p_key[p] = theta;
          p_src[p] = (c << alpha) | o;
        }
        re++;
      }
    }
    __syncthreads();
    fg += s_chunk & 0xffffu;
    fe += s_chunk >> 16;
  }
  FT_MARK(7);
  hi = __reduce_max_sync(FULL, hi);
  if (lane == 0) atomicMax(&s_hi, hi);
  // the reference counters (core.py:69-74): concatenated_len = keys >= theta of
  // the fully qualified subranges (classes C / T / E with d_beta >= theta)
  ull st_concat = 0;
  for (u32 c = tid; c < nc; c += FT_THREADS) {
    const u32 cls = c_cls[c];
    if (cls == CLS_C || cls == CLS_T || cls == CLS_E) {
      // beta <= 2: every C / T / E candidate has d_beta >= theta
      const bool fq = beta <= 2 || a.D[(u64)c_sid[c] * beta + beta - 1] >= theta;
      if (fq) {
        const u64 cnt = (cls == CLS_C) ? sub_len(c_sid[c], a.n, alpha)
                                       : (u64)(((c + 1 < nc) ? c_g[c + 1] : (u32)G) - c_g[c]) +
                                             (u64)(((c + 1 < nc) ? c_e[c + 1] : (u32)E) - c_e[c]);
        st_concat += cnt;
      }
    }
  }
  {
    ull v[4] = {st_fq, st_pq, st_concat, st_reread};
#pragma unroll
    for (int i = 0; i < 4; i++) {
#pragma unroll
      for (int o = 16; o; o >>= 1) v[i] += __shfl_xor_sync(FULL, v[i], o);
      if (lane == 0 && v[i]) atomicAdd(&s_stat[i], v[i]);
    }
  }
  __syncthreads();
  FT_MARK(8);
  // ---- E: sort the pool by (key desc, position asc) and write the answer
  const u32 hk = s_hi;
  if (!ft_bucket_sort_write<MODE>(a, (u32)G, (u32)m, (u32)ko, theta, hk, p_key, p_src, c_sid, ft_sm, scratch)) {
    // long runs of equal keys > theta (few distinct values): nothing was written;
    // the general chain (finish_small's radix sort) takes the call
    if (tid == 0 && a.use_cond) cudaGraphSetConditional(a.cond, 1u);
    return;
  }
  FT_MARK(9);
#ifdef DTOPK_FT_PROFILE
  if (tid == 0)
    printf("fast_tail m=%llu nc=%u nre=%u total=%u | R %lld A %lld B %lld cnt %lld C %lld Dabc %lld Det %lld stat %lld sort %lld\n",
           (unsigned long long)m, nc, nre, total, ft_t[1] - ft_t[0], ft_t[2] - ft_t[1], ft_t[3] - ft_t[2],
           ft_t[4] - ft_t[3], ft_t[5] - ft_t[4], ft_t[6] - ft_t[5], ft_t[7] - ft_t[6], ft_t[8] - ft_t[7],
           ft_t[9] - ft_t[8]);
#endif
  if (tid == 0) {
    dtopk_result& res = ctrl->res;
    res.theta = theta;
    res.candidate_subranges = nc;
    res.fully_qualified = s_stat[0];
    res.partially_qualified = s_stat[1];
    res.concatenated_len = s_stat[2];
    res.elements_reread = s_stat[3];
    res.pool_gt = G;
    res.pool_eq = min(E, k);
    res.path = sel ? PATH_SELECT : PATH_MERGE;
    res.k_out = ko;
    ctrl->maxkey = hk;
    ctrl->small_done = 1;
    if (a.use_cond) cudaGraphSetConditional(a.cond, 0u);
  }
}

}  // namespace dtopk
