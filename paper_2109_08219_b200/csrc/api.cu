// api.cu -- workspace layout, stream-ordered launch sequence and the C ABI
// (include/dtopk.h) of the B200 Dr. Top-k pipeline.
//
// Stage map (paper Eq. 1; pipeline.py:172-220):
//   Delegate : K1 k1_delegates (+ k1_merge when 2^alpha > 8192)
//   FirstK   : K2 k2_scan_delegates, k2_pass3          -> theta = kth(D)
//   Concat   : K4 scan_emit<CAND>                       -> P_gt, first ties
//   SecondK  : sel_pass1..3 + scan_emit<FLAT> (pool > k) or merge_copy,
//              then sort_{hist,scan,scatter} x passes, writeout
// No host synchronisation happens inside a call; data-dependent sizes live in
// the device control block and every kernel sizes its own loop from it.
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <set>
#include <utility>

#include <nvtx3/nvToolsExt.h>

#include "common.cuh"
#include "assemble.cuh"
#include "delegate.cuh"
#include "fast.cuh"
#include "generate.cuh"
#include "merge.cuh"
#include "scan.cuh"
#include "select.cuh"
#include "stage.cuh"

#ifndef DTOPK_K2_CPS
#define DTOPK_K2_CPS 3  // K2 CTAs (regions) per SM (A/B: 3 beats 2, 4, 5 at k = 2^14..2^20)
#endif

using namespace dtopk;

namespace {

// NVTX ranges (header-only NVTX3; inert unless a profiler is attached): every
// C entry point, and the reference's stages (core.STAGES) inside a call, so
// an nsys timeline groups the kernel launches as Delegate / FirstK / Concat /
// SecondK.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
#define DTOPK_RANGE(name) NvtxRange nvtx_range_(name)

std::atomic<unsigned long long> g_launches{0};  // kernels launched by this library
thread_local unsigned long long t_launches = 0;  // kernels launched (or captured) by this thread
inline void counted(int n = 1) {
  g_launches.fetch_add((unsigned long long)n, std::memory_order_relaxed);
  t_launches += (unsigned long long)n;
}
inline unsigned long long dtopk_launch_count_internal() { return t_launches; }

constexpr size_t ALIGN = 256;
inline size_t align_up(size_t x) { return (x + ALIGN - 1) / ALIGN * ALIGN; }

int num_sms();

struct Layout {
  size_t ctrl, lb_emg, lb_eme, zero_bytes, k5_tg, k5_te;
  size_t D, meta, partial, pmeta, selbuf, region_cnt, sup_sid, sup_in, sup_cnt, sup_off, rec, e_sid, t_sid, t_cnt,
      stg_key, stg_idx, seg_gt, seg_eq, d_sid, d_pos, d_need, e_gpos, e_epos, gt_keys, gt_idx, ties, sak, sai, sbk, sbi, counts,
      digit_base, digit_tot, bk_total, bk_count, bk_start, bk_comp, bk_info, chunk_cnt, tseg, sel_tcnt, total;
  u64 fcap, S, nch, W, cap_gt, cap_e, cap_d, m_emit, k4_tiles, k5_tiles, em_tiles, sort_tiles, D_len, nseg, words, R2,
      sort_cap;
  u32 g2;
};

// fast_tail holds <= FT_CAND qualifying subranges.  At least k / beta
// subranges qualify, and about k on inputs without many equal keys (nearly every
// candidate holds one key above theta), so above FT_CAND it would mostly bail
// out (~18 us: k = 8192 at beta 2).
#ifndef DTOPK_FT_KMAX_BETA
#define DTOPK_FT_KMAX_BETA 0  // 1: admit k <= beta * FT_CAND (the bound for inputs with many equal keys)
#endif
inline bool ft_enabled(int alpha, int beta, u64 k) {
  return alpha <= FT_MAX_ALPHA && k <= (u64)(DTOPK_FT_KMAX_BETA ? beta : 1) * FT_CAND;
}

// Filtered delegate pass (K0 sample -> K1 records -> K2 over records): where
// K1's D + meta writes are a measurable share of the stream (alpha 6..8: 12 B
// per 256..1024 B read) and the records carry everything the rest of the
// pipeline reads (beta <= 2).
inline bool filt_possible(u64 S, int alpha, int beta, int direct) {
#ifdef DTOPK_NO_FILTER
  return false;
#endif
  return !direct && alpha >= 6 && alpha <= 8 && beta <= 2 && S >= (1ull << 16);
}

inline int grid_for(u64 work_items, int cap);
inline u32 k1_grid(u64 nch) { return (u32)grid_for(nch, num_sms() * K1_CPS); }

Layout make_layout(u64 n, u64 k, int alpha, int beta, int direct) {
  Layout L{};
  size_t off = 0;
  auto take = [&](u64 bytes) {
    const size_t o = off;
    off = align_up(off + (size_t)bytes);
    return o;
  };
  const u64 W = direct ? 1ull : (1ull << alpha);
  L.W = W;
  L.nch = (n + K1_CHUNK - 1) / K1_CHUNK;
  L.S = direct ? 0 : (n + W - 1) / W;
  L.D_len = direct ? 0 : (u64)beta * L.S;
  // Elements strictly above theta live in the < k subranges whose max delegate
  // exceeds theta = kth(D): the pool and the K4 staging hold <= (k-1) * 2^alpha.
  const u64 kg = std::max<u64>(1, k - 1);
  L.cap_gt = direct ? 0 : std::min<u64>(n, kg * W);
  L.cap_e = direct ? 0 : std::min<u64>(L.S, kg);
  L.cap_d = direct ? 0 : std::min<u64>(L.S, k);
  const int lseg = alpha < 13 ? alpha : 13;
  L.nseg = direct ? 0 : L.cap_e * (W >> lseg);
  L.m_emit = direct ? n : L.cap_gt;
  L.words = (L.S + 31) / 32;
  // K2 regions: one contiguous range of D per CTA
  // <= 768 CTAs: the superset prefix holds K2_SEG_PER (24) segments per thread
  const u64 g2 = std::max<u64>(1, std::min<u64>(std::min<u64>((u64)num_sms() * DTOPK_K2_CPS, 768), (L.D_len + 4095) / 4096));
  L.g2 = (u32)g2;
  L.R2 = ((L.D_len + g2 - 1) / g2 + 511) / 512 * 512;
  const bool filt = filt_possible(L.S, alpha, beta, direct);
  if (filt) {  // K2 over records: a CTA owns 8 warps x ceil(nch / (8 g2)) chunks of 2048 >> alpha subranges
    const u64 cpw = (L.nch + 8 * g2 - 1) / (8 * g2);
    L.R2 = std::max<u64>(L.R2, (8 * cpw * (2048ull >> alpha) * (u64)beta + 511) / 512 * 512);
  }
  L.k4_tiles = (L.cap_e * W + K4_TILE - 1) / K4_TILE;
  L.k5_tiles = std::max<u64>(1, (L.S + K5_TILE - 1) / K5_TILE);  // records <= S
  L.em_tiles = (L.m_emit + SC_TILE - 1) / SC_TILE;
  // largest sort: the answer (k), or a pool of up to 4k kept whole (BIG_SORT_POOL)
  L.sort_cap = direct ? k : std::max<u64>(k, std::min<u64>(4 * k, L.cap_gt));
  L.sort_tiles = (L.sort_cap + ST_TILE - 1) / ST_TILE;
  L.ctrl = take(sizeof(Ctrl));
  L.bk_total = take(L.sort_cap > (u64)SMALL_SORT ? BK_MAX * 4 : 0);
  L.lb_emg = take((L.em_tiles + 1) * 8);  // + 1: emit_count's total sentinel
  L.lb_eme = take((L.em_tiles + 1) * 8);
  L.zero_bytes = off;
  L.D = take(L.D_len * 4);
  L.meta = take(L.S * 4);
  const bool parts = !direct && alpha > K1_LOG_CHUNK;
  L.partial = take(parts ? (u64)beta * L.nch * 4 : 0);
  L.pmeta = take(parts ? 2 * L.nch * 4 : 0);
  L.selbuf = take(std::max<u64>((u64)L.g2 * L.R2, L.m_emit) * 4);
  L.region_cnt = take((u64)L.g2 * 4);
  L.sup_sid = take(L.S * 16);
  L.sup_in = take((u64)L.g2 * 8 * 4);
  L.sup_cnt = take(std::max<u64>((u64)L.g2 * 8, 256 * K2_SEG_PER) * 4);  // padded: read as uint4 by thread
  L.sup_off = take(((u64)L.g2 * 8 + 1) * 4);
  // K3 records; in a filtered call first K1's per-warp record streams (K1 grid x 8 warps x fcap)
  // (a CTA reduces <= ceil(nch / grid) chunks, a warp <= ceil(that / 8))
  L.fcap = filt ? ((L.nch + k1_grid(L.nch) - 1) / k1_grid(L.nch) + 7) / 8 * (2048ull >> alpha) : 0;
  L.rec = take(std::max<u64>(L.S, (u64)k1_grid(L.nch) * 8 * L.fcap) * 16);
  L.k5_tg = take(L.k5_tiles * 8);
  L.k5_te = take(L.k5_tiles * 8);
  L.e_sid = take(L.cap_e * 4);
  L.t_sid = take(L.S * 4);
  L.t_cnt = take(L.S * 4);
  L.stg_key = take(L.cap_e * W * 4);
  L.stg_idx = take(L.cap_e * W * 8);
  L.seg_gt = take(L.nseg * 4);
  L.seg_eq = take(L.nseg * 4);
  L.d_sid = take(L.cap_d * 4);
  L.e_gpos = take(L.cap_e * 8);
  L.e_epos = take(L.cap_e * 8);
  L.d_pos = take(L.cap_d * 8);
  L.d_need = take(L.cap_d * 4);
  L.gt_keys = take(L.cap_gt * 4);
  L.gt_idx = take(L.cap_gt * 8);
  L.ties = take(direct ? 0 : k * 8);
  L.sak = take(direct ? k * 4 : 0);
  L.sai = take(direct ? k * 8 : 0);
  L.sbk = take(L.sort_cap * 4);
  L.sbi = take(L.sort_cap * 8);
  L.counts = take(L.sort_tiles * 256 * 4);
  L.digit_base = take(256 * 4);
  L.digit_tot = take(256 * 4);
  const bool bk = L.sort_cap > (u64)SMALL_SORT;
  L.bk_count = take(bk ? (u64)BK_CHUNKS * BK_MAX * 4 : 0);
  L.bk_start = take(bk ? (BK_MAX + 1) * 4 : 0);
  L.bk_info = take(4 * 4);
  L.bk_comp = take(bk ? L.sort_cap * 8 : 0);
  L.chunk_cnt = take(filt ? L.nch * 4 : 0);
  L.tseg = take(direct ? 0 : (u64)L.g2 * 8 * 8);
  L.sel_tcnt = take((L.m_emit / 2048 + 1) * 4);
  L.total = off;
  return L;
}


// Opt a kernel into `bytes` of dynamic shared memory on the current device.
// The attribute is per (function, device context): a process that runs on
// cuda:0 and then cuda:1 must set it once on each, so the guard is keyed by
// both and taken under a lock (run_distributed lanes launch concurrently).
template <typename F>
void ensure_smem(F* fn, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  cudaGetDevice(&dev);
  const std::pair<const void*, int> key{reinterpret_cast<const void*>(fn), dev};
  std::lock_guard<std::mutex> g(mu);
  if (done.count(key)) return;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) == cudaSuccess) done.insert(key);
}

int num_sms() {
  static std::atomic<int> cache[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  int c = cache[dev].load(std::memory_order_relaxed);
  if (!c) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    c = v > 0 ? v : 148;
    cache[dev].store(c, std::memory_order_relaxed);
  }
  return c;
}

// Launch with programmatic stream serialization (PDL, see common.cuh): the
// kernel's CTAs may be scheduled while its predecessor in the stream runs;
// the kernel itself waits (griddepcontrol.wait) before touching its inputs.
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

#ifndef DTOPK_K5B_GRID
#define DTOPK_K5B_GRID 8  // K5b: latency-bound, one warp per part; 8 CTAs per SM keep more parts in flight
#endif

inline int grid_for(u64 work_items, int cap) {
  if (work_items == 0) return 1;
  return (int)std::max<u64>(1, std::min<u64>(work_items, (u64)cap));
}

inline dtopk_status cuda_status() {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    fprintf(stderr, "dtopk: CUDA error %s\n", cudaGetErrorString(e));
    return DTOPK_CUDA_ERROR;
  }
  return DTOPK_OK;
}

inline void rec(void* const* ev, int i, cudaStream_t s) {
  if (ev && ev[i]) cudaEventRecord(reinterpret_cast<cudaEvent_t>(ev[i]), s);
}

inline int key_mode(int dtype, int largest) { return (dtype == DTOPK_F32 ? 2 : 0) + (largest ? 0 : 1); }

// ---------------------------------------------------------------------------
template <int MODE, int B>
void launch_k1(const K1Args& a, cudaStream_t s, int nsm, u64 nch, int merge = 1) {
  ensure_smem(k1_delegates<MODE, B>, (int)K1_SMEM);
  if (a.c_end > a.c_begin) {
    // the full-range launch keeps the grid the record streams were sized for (k1_grid)
    k1_delegates<MODE, B><<<grid_for(a.c_begin == 0 && a.c_end == nch ? nch : a.c_end - a.c_begin, nsm * K1_CPS),
                            k1_threads<B>(), K1_SMEM, s>>>(a);
    counted();
  }
  if (merge && a.alpha > K1_LOG_CHUNK) {
    k1_merge<B><<<grid_for((a.S + 255) / 256, nsm * 4), 256, 0, s>>>(a.partial, a.pmeta, nch, a.alpha, a.S, a.D,
                                                                       a.meta, a.hist1, a.lin);
    counted();
  }
}

// K1 over chunks [c0, c1) (all by default); `merge` 0 skips k1_merge (alpha >
// 11: run once after the last range), `k1` 0 runs only k1_merge.
template <int MODE>
void stage_delegates(const u32* keys, u64 n, int alpha, int beta, u32* D, char* ws, const Layout& L, cudaStream_t s,
                     int nsm, int fmode = 0, u64 c0 = 0, u64 c1 = ~0ull, int merge = 1, int k1 = 1) {
  Ctrl* ctrl = reinterpret_cast<Ctrl*>(ws + L.ctrl);
  K1Args a{keys,
           n,
           alpha,
           L.S,
           D,
           reinterpret_cast<u32*>(ws + L.partial),
           ctrl->selD.hist1,
           // the fallback pass keeps the filtered pass's (complete) histogram
           (alpha <= K1_LOG_CHUNK && fmode != 2) ? 1 : 0,
           reinterpret_cast<u32*>(ws + L.meta),
           reinterpret_cast<u32*>(ws + L.pmeta),
           ctrl,
           fmode,
           reinterpret_cast<uint4*>(ws + L.rec),
           reinterpret_cast<u32*>(ws + L.chunk_cnt),
           L.fcap,
           k1 ? c0 : 0,
           k1 ? std::min<u64>(c1, L.nch) : 0,
           MODE >= 2 ? 1 : 0};
  switch (beta) {
    case 1: launch_k1<MODE, 1>(a, s, nsm, L.nch, merge); break;
    case 2: launch_k1<MODE, 2>(a, s, nsm, L.nch, merge); break;
    case 3: launch_k1<MODE, 3>(a, s, nsm, L.nch, merge); break;
    case 4: launch_k1<MODE, 4>(a, s, nsm, L.nch, merge); break;
    case 5: launch_k1<MODE, 5>(a, s, nsm, L.nch, merge); break;
    case 6: launch_k1<MODE, 6>(a, s, nsm, L.nch, merge); break;
    case 7: launch_k1<MODE, 7>(a, s, nsm, L.nch, merge); break;
    case 8: launch_k1<MODE, 8>(a, s, nsm, L.nch, merge); break;
    default:
      if (beta <= 32) {
        k1_generic<MODE><<<grid_for((L.S + 7) / 8, nsm * 8), 256, 0, s>>>(
            keys, n, alpha, beta, L.S, D, reinterpret_cast<u32*>(ws + L.meta), ctrl->selD.hist1);
      } else {  // any beta < 2^alpha for subranges of <= 8192 keys: block sort per subrange
        k1_bigbeta<MODE><<<grid_for(L.S, nsm * 4), K1B_THREADS, 0, s>>>(
            keys, n, alpha, beta, L.S, D, reinterpret_cast<u32*>(ws + L.meta), ctrl->selD.hist1);
      }
      counted();
  }
}

K2Args k2_args(char* ws, const Layout& L, u64 k, int beta, int lin, int alpha = 0, int fmode = 0,
               cudaGraphConditionalHandle fb = {}, int fb_graph = 0) {
  return K2Args{reinterpret_cast<u32*>(ws + L.D),
                L.D_len,
                k,
                reinterpret_cast<Ctrl*>(ws + L.ctrl),
                reinterpret_cast<u32*>(ws + L.selbuf),
                reinterpret_cast<u32*>(ws + L.region_cnt),
                L.R2,
                beta,
                reinterpret_cast<uint4*>(ws + L.sup_sid),
                reinterpret_cast<u32*>(ws + L.sup_in),
                reinterpret_cast<u32*>(ws + L.sup_cnt),
                reinterpret_cast<u32*>(ws + L.sup_off),
                reinterpret_cast<const u32*>(ws + L.meta),
                reinterpret_cast<const uint2*>(ws + L.tseg),
                fmode,
                reinterpret_cast<const u32*>(ws + L.chunk_cnt),
                reinterpret_cast<const uint4*>(ws + L.rec),
                L.fcap,
                k1_grid(L.nch),
                L.nch,
                alpha,
                fb,
                fb_graph,
                lin};
}

// Graph capture context: when `graph` is set, run_finish ends the main
// capture after finish_small, adds a conditional IF node set by finish_small
// and captures the large-pool tail into its body; inside the tail, nested IF
// nodes (captured on s2 / s3) gate the select kernels, the bucket sort and the
// LSD fallback sort, so only the stages a run needs are launched.
struct GraphCtx {
  cudaGraph_t graph = nullptr;
  cudaGraphConditionalHandle cond{};  // large-pool tail (set by finish_small)
  cudaGraphConditionalHandle gen{};   // general chain K3..finish_small (set by fast_tail)
  cudaGraphConditionalHandle fb{};    // full K1 + K2 rerun after a failed filtered pass (set by K2)
  cudaStream_t s2 = nullptr, s3 = nullptr, s4 = nullptr, s5 = nullptr, s6 = nullptr;
  unsigned long long main_kernels = 0, body_kernels = 0;
  bool ok = true;
};

inline bool cap_ok(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return true;
  fprintf(stderr, "dtopk: graph capture step %s failed: %s\n", what, cudaGetErrorString(e));
  return false;
}

// Conditional handle for a node anywhere in the plan's graph (handles belong
// to the root graph; the node may sit in a nested conditional body).
bool cond_handle(cudaGraph_t root, cudaGraphConditionalHandle* h) {
  return cap_ok(cudaGraphConditionalHandleCreate(h, root, 0, cudaGraphCondAssignDefault), "handle create");
}

// Append an IF node on handle h at the capture point of s; capture its body on `inner`.
bool cond_begin(cudaStream_t s, cudaGraphConditionalHandle h, cudaStream_t inner) {
  cudaStreamCaptureStatus cst;
  const cudaGraphNode_t* deps = nullptr;
  size_t ndeps = 0;
  cudaGraph_t g = nullptr;
  if (!cap_ok(cudaStreamGetCaptureInfo(s, &cst, nullptr, &g, &deps, &ndeps), "capture info")) return false;
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeIf;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  return cap_ok(cudaGraphAddNode(&node, g, deps, ndeps, &cp), "add conditional node") &&
         cap_ok(cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies), "update deps") &&
         cap_ok(cudaStreamBeginCaptureToGraph(inner, cp.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                              cudaStreamCaptureModeRelaxed), "begin body capture");
}

bool cond_end(cudaStream_t inner) {
  cudaGraph_t g = nullptr;
  return cap_ok(cudaStreamEndCapture(inner, &g), "end body capture");
}

// K2 pass 3 (theta from the bucket members) and K2b (the exact superset of a
// large-bucket call).
void theta_resolve(char* ws, const Layout& L, u64 k, int beta, int lin, cudaStream_t s, int nsm,
                   bool trunc_ok = false) {
  const K2Args k2 = k2_args(ws, L, k, beta, lin);
  launch_pdl(k2_pass3, dim3(grid_for(L.g2, nsm)), dim3(256), 0, s, k2.ctrl, k2.selbuf, k2.region_cnt, L.g2, L.R2,
             k2.sup_cnt, k2.sup_off, k2.D, L.D_len, lin);
  counted();
#ifndef DTOPK_NOOPT_EXP
#define DTOPK_NOOPT_EXP 0  // experiment: 1 = leave out the call-dependent optional kernels (K2c, K4h, big K4)
#endif
  if (trunc_ok && beta <= 2 && !DTOPK_NOOPT_EXP) {
    launch_pdl(k2c_tie_bounds, dim3(grid_for(L.g2, nsm)), dim3(256), 0, s, k2.ctrl, k2.D, L.D_len, L.R2, L.g2, beta,
               k, reinterpret_cast<uint2*>(ws + L.tseg));
    counted();
  }
  if (beta == 2)
    launch_pdl(k2b_superset<1>, dim3(L.g2), dim3(256), 0, s, k2);
  else
    launch_pdl(k2b_superset<0>, dim3(L.g2), dim3(256), 0, s, k2);
  counted();
}

// Delegates (K1) and the delegate scan (K2).  `fused` (a whole dtopk_select or
// plan): theta is resolved by fast_tail, or by K2 pass 3 inside the general
// chain when fast_tail declines.  Otherwise (dtopk_select_begin) pass 3 and K2b
// run here, so that theta_slot holds theta when the call returns.
template <int MODE>
void run_begin(const u32* keys, u64 n, u64 k, int alpha, int beta, char* ws, const Layout& L, cudaStream_t s, int nsm,
               void* const* ev, bool fused = false, GraphCtx* gc = nullptr, bool delegates_done = false) {
  u32* D = reinterpret_cast<u32*>(ws + L.D);
  Ctrl* ctrl = reinterpret_cast<Ctrl*>(ws + L.ctrl);
  if (delegates_done) {  // K1 already ran range by range (dtopk_delegates_range, streamed host input)
    rec(ev, 0, s);
    if (alpha > K1_LOG_CHUNK) stage_delegates<MODE>(keys, n, alpha, beta, D, ws, L, s, nsm, 0, 0, 0, 1, 0);
    rec(ev, 1, s);
    const K2Args k2 = k2_args(ws, L, k, beta, MODE >= 2, alpha, 0);
    if (beta == 2)
      launch_pdl(k2_scan_delegates<1>, dim3(L.g2), dim3(256), 0, s, k2);
    else
      launch_pdl(k2_scan_delegates<0>, dim3(L.g2), dim3(256), 0, s, k2);
    counted();
    if (!fused) theta_resolve(ws, L, k, beta, MODE >= 2, s, nsm);
    rec(ev, 2, s);
    return;
  }
  cudaMemsetAsync(ws, 0, L.zero_bytes, s);
  rec(ev, 0, s);
  nvtxRangePushA("Delegate");
  const bool filt = filt_possible(L.S, alpha, beta, 0);
  if (filt) {
    const u64 nch_full = n >> K1_LOG_CHUNK;
    const int g0 = grid_for((K0_REGIONS * k0_run(nch_full) + 7) / 8, nsm * 4);
    if (beta == 2)
      k0_sample<MODE, 2><<<g0, 256, 0, s>>>(keys, alpha, L.S, k, L.D_len, ctrl, nch_full);
    else
      k0_sample<MODE, 1><<<g0, 256, 0, s>>>(keys, alpha, L.S, k, L.D_len, ctrl, nch_full);
    counted();
  }
  stage_delegates<MODE>(keys, n, alpha, beta, D, ws, L, s, nsm, filt ? 1 : 0);
  nvtxRangePop();
  rec(ev, 1, s);
  DTOPK_RANGE("FirstK");
  const bool g = gc != nullptr && filt;
  const K2Args k2 =
      k2_args(ws, L, k, beta, MODE >= 2, alpha, filt ? 1 : 0, g ? gc->fb : cudaGraphConditionalHandle{}, g ? 1 : 0);
  if (beta == 2)
    launch_pdl(k2_scan_delegates<1>, dim3(L.g2), dim3(256), 0, s, k2);
  else
    launch_pdl(k2_scan_delegates<0>, dim3(L.g2), dim3(256), 0, s, k2);
  counted();
  if (filt) {
    // the sampled floor missed theta's bucket: full K1 (D + meta) and K2 again.
    // Graph: the body of a conditional node K2 sets; eager: both exit at once
    // unless ctrl->filt_fail is set.
    cudaStream_t fs = s;
    if (g) {
      gc->ok = gc->ok && cond_begin(s, gc->fb, gc->s6);
      fs = gc->s6;
    }
    stage_delegates<MODE>(keys, n, alpha, beta, D, ws, L, fs, nsm, 2);
    const K2Args k2f = k2_args(ws, L, k, beta, MODE >= 2, alpha, 2);
    if (beta == 2)
      launch_pdl(k2_scan_delegates<1>, dim3(L.g2), dim3(256), 0, fs, k2f);
    else
      launch_pdl(k2_scan_delegates<0>, dim3(L.g2), dim3(256), 0, fs, k2f);
    counted();
    if (g) gc->ok = gc->ok && cond_end(gc->s6);
  }
  if (!fused) theta_resolve(ws, L, k, beta, MODE >= 2, s, nsm);
  rec(ev, 2, s);
}

SortBufs sort_bufs(char* ws, const Layout& L, bool direct) {
  SortBufs b;
  b.ka = reinterpret_cast<u32*>(ws + (direct ? L.sak : L.gt_keys));
  b.ia = reinterpret_cast<u64*>(ws + (direct ? L.sai : L.gt_idx));
  b.kb = reinterpret_cast<u32*>(ws + L.sbk);
  b.ib = reinterpret_cast<u64*>(ws + L.sbi);
  b.counts = reinterpret_cast<u32*>(ws + L.counts);
  b.digit_base = reinterpret_cast<u32*>(ws + L.digit_base);
  b.digit_tot = reinterpret_cast<u32*>(ws + L.digit_tot);
  return b;
}

void run_sort(Ctrl* ctrl, const SortBufs& b, const Layout& L, cudaStream_t s, int nsm) {
  const int g = grid_for(L.sort_tiles, nsm * 4);
  for (int p = 0; p < 4; p++) {
    sort_hist<<<g, 256, 0, s>>>(ctrl, b, p);
    counted();
    sort_scan<<<32, 256, 0, s>>>(ctrl, b, p);
    counted();
    sort_scatter<<<g, 256, 0, s>>>(ctrl, b, p);
    counted();
  }
}

template <int MODE>
void big_tail(u64 k, const u32* keys_for_emit, const u64* idx_for_emit, const ull* m_dev, u64 m_host, int direct,
              void* out_values, int64_t* out_indices, int64_t offset, char* ws, const Layout& L, cudaStream_t s,
              int nsm, GraphCtx* gc = nullptr) {
  // SecondK beyond SMALL_POOL (or the direct path): merge / sort the pool /
  // exact radix select + ordered emit, then the stable sort and write-out.
  Ctrl* ctrl = reinterpret_cast<Ctrl*>(ws + L.ctrl);
  const SortBufs sb = sort_bufs(ws, L, direct != 0);
  u32* selbuf = reinterpret_cast<u32*>(ws + L.selbuf);
  const bool g = gc != nullptr && !direct;
  cudaGraphConditionalHandle h_sel{}, h_bucket{}, h_lsd{};
  // a handle must belong to a conditional node: h_bucket only when the bucket stage exists
  const bool bucket_stage = L.sort_cap > (u64)SMALL_SORT;
  if (g) gc->ok = gc->ok && cond_handle(gc->graph, &h_sel) && (!bucket_stage || cond_handle(gc->graph, &h_bucket));
  if (!direct) {
    tail_decide<<<1, 1, 0, s>>>(ctrl, k, h_sel, h_bucket, g ? (bucket_stage ? 3 : 1) : 0);
    counted();
    merge_append<<<grid_for((k + 255) / 256, nsm * 4), 256, 0, s>>>(ctrl, sb.ka, sb.ia,
                                                                     reinterpret_cast<u64*>(ws + L.ties));
    counted();
  }
  cudaStream_t cs = s;  // stream of the current (possibly conditional) body
  if (g) {
    gc->ok = gc->ok && cond_begin(s, h_sel, gc->s2);
    cs = gc->s2;
  }
  const u64 mcap = m_dev ? L.cap_gt : m_host;
  const int gs = grid_for((mcap + 2047) / 2048, nsm * 4);
  SelArgs sp{keys_for_emit, m_host, m_dev, ctrl, &ctrl->selP, selbuf, k, direct ? 0 : 1,
             reinterpret_cast<u32*>(ws + L.sel_tcnt)};
  if (direct) {
    sel_pass1<MODE><<<gs, 256, 0, cs>>>(sp);
    counted();
    sel_pass2<MODE><<<gs, 256, 0, cs>>>(sp);
    counted();
  } else {
    sel_pass1<KM_KEY><<<gs, 256, 0, cs>>>(sp);
    counted();
    sel_pass2<KM_KEY><<<grid_for((mcap + 2047) / 2048, nsm * 8), 256, 0, cs>>>(sp);  // latency-bound: 8 CTAs / SM
    counted();
  }
  sel_pass3<<<gs, 256, 0, cs>>>(sp);
  counted();
  ScanArgs em{};
  em.keys = keys_for_emit;
  em.idx_in = idx_for_emit;
  em.m_host = m_host;
  em.m_dev = m_dev;
  em.ctrl = ctrl;
  em.k = k;
  em.out_keys = direct ? sb.ka : sb.kb;
  em.out_idx = direct ? sb.ia : sb.ib;
  em.lb_gt = reinterpret_cast<u64*>(ws + L.lb_emg);
  em.lb_eq = reinterpret_cast<u64*>(ws + L.lb_eme);
  em.check_path = direct ? 0 : 1;
  em.direct = direct;
  if (direct) {
    scan_emit<MODE><<<grid_for(L.em_tiles, nsm * 4), 256, 0, cs>>>(em);
    counted();
  } else {  // pool select: count + scan, then write only the tiles that emit
    emit_count<KM_KEY><<<grid_for(L.em_tiles, nsm * 8), 256, 0, cs>>>(em);
    emit_write<KM_KEY><<<grid_for(L.em_tiles, nsm * 4), 256, 0, cs>>>(em);
    counted(2);
  }
  if (g) {
    gc->ok = gc->ok && cond_end(gc->s2);
    cs = s;
  }
  ensure_smem(sort_small<MODE>, SMALL_SORT * 8);
  sort_small<MODE><<<1, 1024, SMALL_SORT * 8, s>>>(ctrl, sb, reinterpret_cast<u32*>(out_values),
                                                   reinterpret_cast<long long*>(out_indices), (long long)offset);
  counted();
  if (bucket_stage) {
    if (g) {
      gc->ok = gc->ok && cond_begin(s, h_bucket, gc->s2) && cond_handle(gc->graph, &h_lsd);
      cs = gc->s2;
    }
    BucketBufs bb{reinterpret_cast<u32*>(ws + L.bk_total), reinterpret_cast<u32*>(ws + L.bk_count), reinterpret_cast<u32*>(ws + L.bk_start),
                  reinterpret_cast<unsigned long long*>(ws + L.bk_comp), reinterpret_cast<u32*>(ws + L.bk_info),
                  h_lsd, g ? 1 : 0};
    bucket_count<<<BK_CHUNKS, 512, 0, cs>>>(ctrl, sb, bb);
    counted();
    bucket_scatter<<<BK_CHUNKS, 512, 0, cs>>>(ctrl, sb, bb);
    counted();
    bucket_sort<MODE><<<grid_for(BK_MAX, nsm * 6), 256, 0, cs>>>(
        ctrl, sb, bb, reinterpret_cast<u32*>(out_values), reinterpret_cast<long long*>(out_indices),
        (long long)offset);
    counted();
    cudaStream_t ls = cs;
    if (g) {
      gc->ok = gc->ok && cond_begin(cs, h_lsd, gc->s3);
      ls = gc->s3;
    }
    run_sort(ctrl, sb, L, ls, nsm);
    writeout<MODE><<<grid_for((k + 255) / 256, nsm * 4), 256, 0, ls>>>(
        ctrl, sb, reinterpret_cast<u32*>(out_values), reinterpret_cast<long long*>(out_indices), (long long)offset);
    counted();
    if (g) gc->ok = gc->ok && cond_end(gc->s3) && cond_end(gc->s2);
  }
}


template <int MODE>
void run_finish(const u32* keys, u64 n, u64 k, int alpha, int beta, u32 flags, const int64_t* theta_override,
                void* out_values, int64_t* out_indices, int64_t offset, char* ws, const Layout& L, cudaStream_t s,
                int nsm, void* const* ev, GraphCtx* gc = nullptr, bool fused = false) {
  Ctrl* ctrl = reinterpret_cast<Ctrl*>(ws + L.ctrl);
  // fast_tail: the whole post-theta work of a small call in one CTA (fast.cuh);
  // the general chain below runs only when it declines (graph: conditional node,
  // eager: every chain kernel returns when ctrl->small_done is set)
  const bool fast = ft_enabled(alpha, beta, k);
  const bool g = gc != nullptr;
  if (fast) {
    ensure_smem(fast_tail<MODE>, (int)FT_SMEM);
    FTArgs fa{ctrl,
              keys,
              n,
              alpha,
              beta,
              k,
              L.D_len,
              reinterpret_cast<const u32*>(ws + L.D),
              reinterpret_cast<const uint4*>(ws + L.sup_sid),
              reinterpret_cast<const u32*>(ws + L.sup_in),
              reinterpret_cast<const u32*>(ws + L.sup_cnt),
              reinterpret_cast<const u32*>(ws + L.sup_off),
              (u32)(L.g2 * 8),
              fused ? 1 : 0,
              reinterpret_cast<const u32*>(ws + L.selbuf),
              reinterpret_cast<const u32*>(ws + L.region_cnt),
              L.g2,
              L.R2,
              theta_override,
              reinterpret_cast<u32*>(out_values),
              reinterpret_cast<long long*>(out_indices),
              (long long)offset,
              g ? gc->gen : cudaGraphConditionalHandle{},
              g ? 1 : 0};
    launch_pdl(fast_tail<MODE>, dim3(1), dim3(FT_THREADS), FT_SMEM, s, fa);
    counted();
    if (g) {
      gc->main_kernels = dtopk_launch_count_internal();  // always executed: K1 .. fast_tail
      gc->ok = gc->ok && cond_begin(s, gc->gen, gc->s4);
    }
  }
  cudaStream_t s_outer = s;
  if (g && fast) s = gc->s4;  // the general chain is the body of the conditional node
  // fused call: theta was left to fast_tail; the general chain resolves it itself.
  // No external theta here, so a tie-heavy call may drop tie-only superset
  // entries past the first k ties (not with exact stats: |C| counts every one)
  if (fused) theta_resolve(ws, L, k, beta, MODE >= 2, s, nsm, (flags & DTOPK_FLAG_EXACT_STATS) == 0);
  nvtxRangePushA("Concat");
  Records rc{reinterpret_cast<uint4*>(ws + L.rec)};
  u32* e_sid = reinterpret_cast<u32*>(ws + L.e_sid);
  u32* t_sid = reinterpret_cast<u32*>(ws + L.t_sid);
  u32* t_cnt = reinterpret_cast<u32*>(ws + L.t_cnt);
  const u64 nseg = (u64)L.g2 * 8;
  K3Args k3{reinterpret_cast<const u32*>(ws + L.D),
            reinterpret_cast<const u32*>(ws + L.meta),
            L.S,
            n,
            alpha,
            beta,
            ctrl,
            theta_override,
            rc,
            reinterpret_cast<const uint4*>(ws + L.sup_sid),
            reinterpret_cast<const u32*>(ws + L.sup_in),
            reinterpret_cast<const u32*>(ws + L.sup_off),
            nseg,
            e_sid,
            t_sid,
            t_cnt,
            L.cap_e,
            reinterpret_cast<u64*>(ws + L.e_epos)};
  launch_pdl(k3_classify, dim3(grid_for((nseg + 7) / 8, nsm * 8)), dim3(256), 0, s, k3);
  counted();
  K4Args k4{keys, n, alpha, ctrl, e_sid, reinterpret_cast<u32*>(ws + L.stg_key),
            reinterpret_cast<u64*>(ws + L.stg_idx), reinterpret_cast<u32*>(ws + L.seg_gt),
            reinterpret_cast<u32*>(ws + L.seg_eq), L.cap_e};
  if (beta <= 2 && (L.cap_e << alpha) >= DTOPK_PF_MIN_KEYS && !DTOPK_NOOPT_EXP) {  // pool floor (every E record is then fully qualified)
    launch_pdl(k4h_floor<MODE>, dim3(nsm * 4), dim3(256), 0, s, k4, static_cast<const uint4*>(rc.r), k);
    counted();
  }
  launch_pdl(k4_read<MODE, 0>, dim3(grid_for(std::max<u64>(L.k4_tiles, (L.cap_e + 255) / 256), nsm * 4)), dim3(256), 0, s,
             k4);
  if (L.cap_e << alpha >= DTOPK_K4_BIG_KEYS && !DTOPK_NOOPT_EXP) {
    launch_pdl(k4_read<MODE, 1>, dim3(grid_for(std::max<u64>(L.k4_tiles, (L.cap_e + 255) / 256), nsm * 3)), dim3(256),
               0, s, k4);
    counted();
  }
  counted();
  const int exact = (flags & DTOPK_FLAG_EXACT_STATS) ? 1 : 0;
  K4TArgs k4t{keys, n,  L.S,   alpha, k, ctrl, t_sid, t_cnt, rc.r, reinterpret_cast<const u32*>(ws + L.seg_eq),
              exact};
  launch_pdl(k4t_count<MODE>, dim3(grid_for((L.S + 7) / 8, nsm * 4)), dim3(256), 0, s, k4t);
  counted();
  K5Args k5{ctrl,
            rc,
            n,
            alpha,
            k,
            reinterpret_cast<const u32*>(ws + L.stg_key),
            reinterpret_cast<const u64*>(ws + L.stg_idx),
            reinterpret_cast<const u32*>(ws + L.seg_gt),
            reinterpret_cast<const u32*>(ws + L.seg_eq),
            t_cnt,
            reinterpret_cast<u32*>(ws + L.gt_keys),
            reinterpret_cast<u64*>(ws + L.gt_idx),
            reinterpret_cast<u64*>(ws + L.ties),
            reinterpret_cast<u32*>(ws + L.d_sid),
            reinterpret_cast<u64*>(ws + L.d_pos),
            reinterpret_cast<u32*>(ws + L.d_need),
            reinterpret_cast<u64*>(ws + L.e_gpos),
            reinterpret_cast<u64*>(ws + L.e_epos),
            reinterpret_cast<u64*>(ws + L.k5_tg),
            reinterpret_cast<u64*>(ws + L.k5_te),
            exact};
  launch_pdl(k5_count, dim3(grid_for(L.k5_tiles, nsm * 4)), dim3(256), 0, s, k5);
  counted();
  launch_pdl(k5_emit, dim3(grid_for(L.k5_tiles, nsm * 4)), dim3(256), 0, s, k5);
  counted();
  launch_pdl(k5b_copy, dim3(grid_for((L.nseg + 7) / 8, nsm * DTOPK_K5B_GRID)), dim3(256), 0, s, ctrl, alpha, k, k5.stg_key, k5.stg_idx, k5.seg_gt,
                                                               k5.seg_eq, k5.e_gpos, k5.e_epos, L.cap_e,
                                                               k5.gt_keys, k5.gt_idx, k5.ties);
  counted();
  launch_pdl(k6_ties<MODE>, dim3(grid_for((L.cap_d + 7) / 8, nsm * 4)), dim3(256), 0, s, ctrl, keys, n, alpha, k5.d_sid, k5.d_pos,
                                                                      k5.d_need, k5.ties);
  counted();
  rec(ev, 3, s_outer);
  nvtxRangePop();
  DTOPK_RANGE("SecondK");
  ensure_smem(finish_small<MODE>, SMALL_POOL * 8);
  const bool need_tail = std::max<u64>(L.cap_gt, k) > (u64)SMALL_POOL;  // pools beyond SMALL_POOL possible
  const bool cond = g && need_tail;
  launch_pdl(finish_small<MODE>, dim3(1), dim3(1024), SMALL_POOL * 8, s, ctrl, k5.gt_keys, k5.gt_idx, k5.ties,
                                                     reinterpret_cast<u32*>(out_values),
                                                     reinterpret_cast<long long*>(out_indices), (long long)offset,
                                                     cond ? gc->cond : cudaGraphConditionalHandle{}, cond ? 1 : 0);
  counted();
  if (need_tail) {
    if (!g) {
      big_tail<MODE>(k, k5.gt_keys, k5.gt_idx, (const ull*)&ctrl->res.pool_gt, 0, 0, out_values, out_indices,
                     offset, ws, L, s, nsm);
    } else {
      // graph mode: the large-pool tail is the body of a conditional node set by finish_small
      gc->ok = gc->ok && cond_begin(s, gc->cond, gc->s5);
      big_tail<MODE>(k, k5.gt_keys, k5.gt_idx, (const ull*)&ctrl->res.pool_gt, 0, 0, out_values, out_indices,
                     offset, ws, L, gc->s5, nsm, gc);
      gc->ok = gc->ok && cond_end(gc->s5);
    }
  }
  if (g && fast) {
    gc->ok = gc->ok && cond_end(gc->s4);
    gc->body_kernels = dtopk_launch_count_internal() - gc->main_kernels;  // the general chain (conditional)
  }
  rec(ev, 4, s_outer);
}

template <int MODE>
void run_direct(const u32* keys, u64 n, u64 k, void* out_values, int64_t* out_indices, int64_t offset, char* ws,
                const Layout& L, cudaStream_t s, int nsm, void* const* ev) {
  cudaMemsetAsync(ws, 0, L.zero_bytes, s);
  for (int i = 0; i < 4; i++) rec(ev, i, s);  // pipeline.py:185-186: only SecondK runs
  big_tail<MODE>(k, keys, nullptr, nullptr, n, 1, out_values, out_indices, offset, ws, L, s, nsm);
  rec(ev, 4, s);
}

dtopk_status check_common(const void* keys, u64 n, int dtype, u64 k) {
  if (n == 0) return DTOPK_EMPTY_INPUT;
  if (k < 1 || k > n || k > 0xffffffffull) return DTOPK_INVALID_K;
  if (dtype != DTOPK_U32 && dtype != DTOPK_F32) return DTOPK_INVALID_ARG;
  if (keys == nullptr || (reinterpret_cast<uintptr_t>(keys) & 15u) != 0) return DTOPK_INVALID_ARG;
  return DTOPK_OK;
}

dtopk_status check_delegate(u64 n, int alpha, int beta) {
  if (alpha < 1 || alpha > 40 || (1ull << alpha) > n) return DTOPK_INVALID_ARG;
  if (beta < 1 || (u64)beta >= (1ull << alpha)) return DTOPK_INVALID_BETA;
  if (beta > 32 && alpha > 13) return DTOPK_UNSUPPORTED;  // beta > 32: subranges of <= 8192 keys (k1_bigbeta)
  if (((n + (1ull << alpha) - 1) >> alpha) > 0xffffffffull) return DTOPK_INVALID_ARG;
  return DTOPK_OK;
}


// ---------------------------------------------------------------------------
// Multi-GPU candidate merge (merge.cuh): ShardedTopK's device-side glue.
// ---------------------------------------------------------------------------
template <int M>
void run_merge_lists(const uint32_t* in_val, int vmul, int vstride, const int64_t* in_idx, const int64_t* in_off,
                     int64_t in_stride, const int64_t* in_len, int64_t len_stride, int n_lists, int64_t cap,
                     uint32_t* out_val,
                     int64_t* out_idx, uint32_t* tmp_val, int64_t* tmp_idx, int64_t* tmp_len, cudaStream_t s) {
  // tmp_* hold two ping-pong levels of ceil(n_lists / 2) lists of `cap` pairs
  const int half = (n_lists + 1) / 2;
  const int64_t level = (int64_t)half * cap;
  MergeArgs a{};
  a.in_val = in_val;
  a.vmul = vmul;
  a.vstride = vstride;
  a.in_idx = reinterpret_cast<const long long*>(in_idx);
  a.in_off = reinterpret_cast<const long long*>(in_off);
  a.in_stride = in_stride;
  a.in_len = reinterpret_cast<const long long*>(in_len);
  a.len_stride = len_stride;
  a.n_lists = n_lists;
  a.cap = cap;
  int lvl = 0;
  const unsigned gx = (unsigned)std::max<int64_t>(1, (cap + MG_TILE - 1) / MG_TILE);
  for (;;) {
    const int pairs = (a.n_lists + 1) / 2;
    const bool last = pairs == 1;
    a.out_val = last ? out_val : tmp_val + lvl * level;
    a.out_idx = reinterpret_cast<long long*>(last ? out_idx : tmp_idx + lvl * level);
    a.out_stride = last ? 0 : cap;
    a.out_len = reinterpret_cast<long long*>(tmp_len + lvl * half);
    launch_pdl(merge_round<M>, dim3(gx, pairs), dim3(MG_THREADS), 0, s, a);
    counted();
    if (last) break;
    a.in_val = a.out_val;
    a.vmul = 1;
    a.vstride = 1;
    a.in_idx = a.out_idx;
    a.in_off = nullptr;
    a.in_stride = cap;
    a.in_len = a.out_len;
    a.len_stride = 1;
    a.n_lists = pairs;
    lvl ^= 1;
  }
}
template <int M>
void run_dsel_hist(const uint32_t* bits, const int64_t* cnt, const int64_t* state, int pass, int64_t* hist,
                   uint64_t cap, cudaStream_t s) {
  const int g = grid_for((cap + 256 * 16 - 1) / (256 * 16), num_sms() * 4);
  launch_pdl(dsel_hist<M>, dim3(g), dim3(256), 0, s, bits, reinterpret_cast<const long long*>(cnt),
             reinterpret_cast<const long long*>(state), pass, reinterpret_cast<long long*>(hist));
  counted();
}

template <int M>
void run_dsel_digit(int64_t* state, int64_t* hist, int pass, const uint32_t* bits, const int64_t* cnt,
                    int64_t* gt_eq, cudaStream_t s) {
  launch_pdl(dsel_digit<M>, dim3(1), dim3(1024), 0, s, reinterpret_cast<long long*>(state),
             reinterpret_cast<long long*>(hist), pass, bits, reinterpret_cast<const long long*>(cnt),
             reinterpret_cast<long long*>(gt_eq));
  counted();
}


template <int MODE>
void run_concat(const u32* raw, u64 n, int alpha, const u32* fq, u64 nfq, u32 theta, u32* out, int64_t* out_count,
                u32* tc, cudaStream_t s) {
  const u64 nv = nfq << alpha;
  const u64 tiles = std::max<u64>(1, (nv + STG_TILE - 1) / STG_TILE);
  concat_count<MODE><<<(unsigned)tiles, STG_THREADS, 0, s>>>(raw, n, alpha, fq, nv, theta, tc);
  stg_scan<<<1, STG_THREADS, 0, s>>>(tc, tiles, 1, out_count);
  concat_emit<MODE><<<(unsigned)tiles, STG_THREADS, 0, s>>>(raw, n, alpha, fq, nv, theta, tc, out);
  counted(3);
}



#define DISPATCH_MODE(mode, FN, ...)  \
  switch (mode) {                     \
    case 0: FN<0>(__VA_ARGS__); break; \
    case 1: FN<1>(__VA_ARGS__); break; \
    case 2: FN<2>(__VA_ARGS__); break; \
    default: FN<3>(__VA_ARGS__); break; \
  }

}  // namespace

extern "C" {

size_t dtopk_stage_workspace_bytes(uint64_t n_elements);

size_t dtopk_workspace_bytes(uint64_t n, uint64_t k, int alpha, int beta, int direct) {
  if (k < 1) k = 1;
  return make_layout(n, k, alpha, beta, direct).total;
}

size_t dtopk_result_offset(void) { return 0; }

struct dtopk_plan_s {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaStream_t cap = nullptr;
  unsigned long long main_kernels = 0, body_kernels = 0;
};

dtopk_status dtopk_plan_create(const void* keys, uint64_t n, int dtype, uint64_t k, int largest, int alpha, int beta,
                               int direct, uint32_t flags, void* out_values, int64_t* out_indices,
                               int64_t index_offset, void* ws, size_t ws_bytes, dtopk_plan* out_plan) {
  DTOPK_RANGE("dtopk_plan_create");
  if (out_plan == nullptr) return DTOPK_INVALID_ARG;
  *out_plan = nullptr;
  dtopk_status st = check_common(keys, n, dtype, k);
  if (st != DTOPK_OK) return st;
  if (out_values == nullptr || out_indices == nullptr) return DTOPK_INVALID_ARG;
  if (!direct) {
    if ((st = check_delegate(n, alpha, beta)) != DTOPK_OK) return st;
    if ((u64)beta * ((n + (1ull << alpha) - 1) >> alpha) < k) return DTOPK_INVALID_K;
  }
  const Layout L = direct ? make_layout(n, k, 0, 1, 1) : make_layout(n, k, alpha, beta, 0);
  if (ws == nullptr || ws_bytes < L.total) return DTOPK_WORKSPACE_TOO_SMALL;
  // Run once eagerly: sets kernel attributes and validates the configuration.
  // The warm-up writes the workspace and reads the keys, so it must not race
  // work the caller queued on its own (possibly non-blocking) streams, e.g. a
  // replay of another plan sharing this workspace: drain the device first.
  if (cudaDeviceSynchronize() != cudaSuccess) return cuda_status();
  st = dtopk_select(keys, n, dtype, k, largest, alpha, beta, direct, flags, out_values, out_indices, index_offset, ws,
                    ws_bytes, nullptr, nullptr);
  if (st != DTOPK_OK) return st;
  if (cudaDeviceSynchronize() != cudaSuccess) return cuda_status();
  dtopk_plan_s* p = new dtopk_plan_s();
  GraphCtx gc;
  bool ok = cudaStreamCreateWithFlags(&p->cap, cudaStreamNonBlocking) == cudaSuccess &&
            cudaStreamCreateWithFlags(&gc.s2, cudaStreamNonBlocking) == cudaSuccess &&
            cudaStreamCreateWithFlags(&gc.s3, cudaStreamNonBlocking) == cudaSuccess &&
            cudaStreamCreateWithFlags(&gc.s4, cudaStreamNonBlocking) == cudaSuccess &&
            cudaStreamCreateWithFlags(&gc.s5, cudaStreamNonBlocking) == cudaSuccess &&
            cudaStreamCreateWithFlags(&gc.s6, cudaStreamNonBlocking) == cudaSuccess &&
            cudaGraphCreate(&p->graph, 0) == cudaSuccess &&
            cudaGraphConditionalHandleCreate(&gc.cond, p->graph, 0, cudaGraphCondAssignDefault) == cudaSuccess &&
            (direct || !ft_enabled(alpha, beta, k) ||
             cudaGraphConditionalHandleCreate(&gc.gen, p->graph, 1, cudaGraphCondAssignDefault) == cudaSuccess) &&
            (!filt_possible(L.S, alpha, beta, direct) ||
             cudaGraphConditionalHandleCreate(&gc.fb, p->graph, 0, cudaGraphCondAssignDefault) == cudaSuccess) &&
            cudaStreamBeginCaptureToGraph(p->cap, p->graph, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed) ==
                cudaSuccess;
  if (ok) {
    gc.graph = p->graph;
    t_launches = 0;
    const int nsm = num_sms();
    const u32* kp = reinterpret_cast<const u32*>(keys);
    char* w = reinterpret_cast<char*>(ws);
    cudaStream_t s = p->cap;
    if (direct) {
      DISPATCH_MODE(key_mode(dtype, largest), run_direct, kp, n, k, out_values, out_indices, index_offset, w, L, s,
                    nsm, nullptr);
    } else {
      const bool fused = alpha <= FT_MAX_ALPHA;
      DISPATCH_MODE(key_mode(dtype, largest), run_begin, kp, n, k, alpha, beta, w, L, s, nsm, nullptr, fused, &gc);
      DISPATCH_MODE(key_mode(dtype, largest), run_finish, kp, n, k, alpha, beta, flags, nullptr, out_values,
                    out_indices, index_offset, w, L, s, nsm, nullptr, &gc, fused);
    }
    cudaGraph_t g = nullptr;
    ok = cudaStreamEndCapture(s, &g) == cudaSuccess;
    if (gc.main_kernels == 0) gc.main_kernels = t_launches;
    ok = ok && gc.ok && cap_ok(cudaGraphInstantiate(&p->exec, p->graph, 0), "instantiate");
    p->main_kernels = gc.main_kernels;
    p->body_kernels = gc.body_kernels;
  }
  for (cudaStream_t x : {gc.s2, gc.s3, gc.s4, gc.s5, gc.s6})
    if (x) cudaStreamDestroy(x);
  if (!ok) {
    cudaGetLastError();
    dtopk_plan_destroy(p);
    return DTOPK_CUDA_ERROR;
  }
  *out_plan = p;
  return DTOPK_OK;
}

dtopk_status dtopk_plan_launch(dtopk_plan plan, void* stream) {
  DTOPK_RANGE("dtopk_plan_launch");
  if (plan == nullptr || plan->exec == nullptr) return DTOPK_INVALID_ARG;
  if (cudaGraphLaunch(plan->exec, reinterpret_cast<cudaStream_t>(stream)) != cudaSuccess) return cuda_status();
  counted((int)plan->main_kernels);
  return DTOPK_OK;
}

void dtopk_plan_kernels(dtopk_plan plan, unsigned long long* main_kernels, unsigned long long* tail_kernels) {
  if (plan == nullptr) return;
  if (main_kernels) *main_kernels = plan->main_kernels;
  if (tail_kernels) *tail_kernels = plan->body_kernels;
}

void dtopk_plan_destroy(dtopk_plan plan) {
  if (plan == nullptr) return;
  if (plan->exec) cudaGraphExecDestroy(plan->exec);
  if (plan->graph) cudaGraphDestroy(plan->graph);
  if (plan->cap) cudaStreamDestroy(plan->cap);
  delete plan;
}

int dtopk_num_sms(void) { return num_sms(); }

dtopk_status dtopk_generate(void* out, uint64_t n, int dist, uint64_t seed, uint64_t param, void* stream) {
  if (out == nullptr) return DTOPK_INVALID_ARG;
  if (n == 0) return DTOPK_OK;
  gen_kernel<<<grid_for((n + 255) / 256, num_sms() * 8), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<u32*>(out), n, dist, seed, param);
  counted();
  return cuda_status();
}

void* dtopk_event_create(void) {
  cudaEvent_t e = nullptr;
  if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
  return reinterpret_cast<void*>(e);
}

void dtopk_event_destroy(void* ev) {
  if (ev) cudaEventDestroy(reinterpret_cast<cudaEvent_t>(ev));
}

float dtopk_event_elapsed_ms(void* start, void* end) {
  float ms = -1.0f;
  if (!start || !end) return ms;
  if (cudaEventSynchronize(reinterpret_cast<cudaEvent_t>(end)) != cudaSuccess) return ms;
  if (cudaEventElapsedTime(&ms, reinterpret_cast<cudaEvent_t>(start), reinterpret_cast<cudaEvent_t>(end)) !=
      cudaSuccess)
    return -1.0f;
  return ms;
}

unsigned long long dtopk_launch_count(void) { return g_launches.load(); }

const char* dtopk_version(void) { return "dtopk-b200 0.1.0 (sm_100a)"; }

dtopk_status dtopk_select_begin(const void* keys, uint64_t n, int dtype, uint64_t k, int largest, int alpha, int beta,
                                uint32_t flags, void* ws, size_t ws_bytes, void* stream, void* const* stage_events) {
  DTOPK_RANGE("dtopk_select_begin");
  (void)flags;
  dtopk_status st = check_common(keys, n, dtype, k);
  if (st != DTOPK_OK) return st;
  if ((st = check_delegate(n, alpha, beta)) != DTOPK_OK) return st;
  if ((u64)beta * ((n + (1ull << alpha) - 1) >> alpha) < k) return DTOPK_INVALID_K;
  const Layout L = make_layout(n, k, alpha, beta, 0);
  if (ws == nullptr || ws_bytes < L.total) return DTOPK_WORKSPACE_TOO_SMALL;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int nsm = num_sms();
  const u32* kp = reinterpret_cast<const u32*>(keys);
  char* w = reinterpret_cast<char*>(ws);
  DISPATCH_MODE(key_mode(dtype, largest), run_begin, kp, n, k, alpha, beta, w, L, s, nsm, stage_events);
  return cuda_status();
}

dtopk_status dtopk_select_finish(const void* keys, uint64_t n, int dtype, uint64_t k, int largest, int alpha, int beta,
                                 uint32_t flags, const int64_t* theta_override, void* out_values,
                                 int64_t* out_indices, int64_t index_offset, void* ws, size_t ws_bytes,
                                 void* stream, void* const* stage_events) {
  DTOPK_RANGE("dtopk_select_finish");
  dtopk_status st = check_common(keys, n, dtype, k);
  if (st != DTOPK_OK) return st;
  if ((st = check_delegate(n, alpha, beta)) != DTOPK_OK) return st;
  if (out_values == nullptr || out_indices == nullptr) return DTOPK_INVALID_ARG;
  const Layout L = make_layout(n, k, alpha, beta, 0);
  if (ws == nullptr || ws_bytes < L.total) return DTOPK_WORKSPACE_TOO_SMALL;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int nsm = num_sms();
  const u32* kp = reinterpret_cast<const u32*>(keys);
  char* w = reinterpret_cast<char*>(ws);
  DISPATCH_MODE(key_mode(dtype, largest), run_finish, kp, n, k, alpha, beta, flags, theta_override, out_values,
                out_indices,
                index_offset, w, L, s, nsm, stage_events);
  return cuda_status();
}

dtopk_status dtopk_select(const void* keys, uint64_t n, int dtype, uint64_t k, int largest, int alpha, int beta,
                          int direct, uint32_t flags, void* out_values, int64_t* out_indices, int64_t index_offset,
                          void* ws, size_t ws_bytes, void* stream, void* const* stage_events) {
  DTOPK_RANGE("dtopk_select");
  dtopk_status st = check_common(keys, n, dtype, k);
  if (st != DTOPK_OK) return st;
  if (out_values == nullptr || out_indices == nullptr) return DTOPK_INVALID_ARG;
  if (direct) {
    const Layout L = make_layout(n, k, 0, 1, 1);
    if (ws == nullptr || ws_bytes < L.total) return DTOPK_WORKSPACE_TOO_SMALL;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int nsm = num_sms();
    const u32* kp = reinterpret_cast<const u32*>(keys);
    char* w = reinterpret_cast<char*>(ws);
    DISPATCH_MODE(key_mode(dtype, largest), run_direct, kp, n, k, out_values, out_indices, index_offset, w, L, s, nsm,
                  stage_events);
    return cuda_status();
  }
  if ((st = check_delegate(n, alpha, beta)) != DTOPK_OK) return st;
  if ((u64)beta * ((n + (1ull << alpha) - 1) >> alpha) < k) return DTOPK_INVALID_K;
  const Layout L = make_layout(n, k, alpha, beta, 0);
  if (ws == nullptr || ws_bytes < L.total) return DTOPK_WORKSPACE_TOO_SMALL;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int nsm = num_sms();
  const u32* kp = reinterpret_cast<const u32*>(keys);
  char* w = reinterpret_cast<char*>(ws);
  const bool fused = alpha <= FT_MAX_ALPHA;
  const bool done = (flags & DTOPK_FLAG_DELEGATES_DONE) != 0;
  if (done && beta > 8) return DTOPK_INVALID_ARG;  // streamed delegates: the K1 ladder kernels only
  DISPATCH_MODE(key_mode(dtype, largest), run_begin, kp, n, k, alpha, beta, w, L, s, nsm, stage_events, fused, nullptr,
                done);
  DISPATCH_MODE(key_mode(dtype, largest), run_finish, kp, n, k, alpha, beta, flags, nullptr, out_values, out_indices,
                index_offset, w, L, s, nsm, stage_events, nullptr, fused);
  return cuda_status();
}

dtopk_status dtopk_delegates_range(const void* keys, uint64_t n, int dtype, uint64_t k, int largest, int alpha,
                                   int beta, uint64_t chunk_begin, uint64_t chunk_end, void* ws, size_t ws_bytes,
                                   void* stream) {
  DTOPK_RANGE("dtopk_delegates_range");
  dtopk_status st = check_common(keys, n, dtype, k);
  if (st != DTOPK_OK) return st;
  if ((st = check_delegate(n, alpha, beta)) != DTOPK_OK) return st;
  if (beta > 8) return DTOPK_INVALID_ARG;
  const Layout L = make_layout(n, k, alpha, beta, 0);
  if (ws == nullptr || ws_bytes < L.total) return DTOPK_WORKSPACE_TOO_SMALL;
  if (chunk_begin > chunk_end || chunk_end > L.nch) return DTOPK_INVALID_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  char* w = reinterpret_cast<char*>(ws);
  if (chunk_begin == 0) cudaMemsetAsync(w, 0, L.zero_bytes, s);
  const u32* kp = reinterpret_cast<const u32*>(keys);
  DISPATCH_MODE(key_mode(dtype, largest), stage_delegates, kp, n, alpha, beta, reinterpret_cast<u32*>(w + L.D), w, L,
                s, num_sms(), 0, chunk_begin, chunk_end, 0, 1);
  return cuda_status();
}

dtopk_status dtopk_extract_delegates(const void* keys, uint64_t n, int dtype, int largest, int alpha, int beta,
                                     uint32_t* out_delegates, void* ws, size_t ws_bytes, void* stream) {
  DTOPK_RANGE("dtopk_extract_delegates");
  dtopk_status st = check_common(keys, n, dtype, 1);
  if (st != DTOPK_OK) return st;
  if ((st = check_delegate(n, alpha, beta)) != DTOPK_OK) return st;
  if (out_delegates == nullptr) return DTOPK_INVALID_ARG;
  const Layout L = make_layout(n, 1, alpha, beta, 0);
  if (ws == nullptr || ws_bytes < L.total) return DTOPK_WORKSPACE_TOO_SMALL;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  char* w = reinterpret_cast<char*>(ws);
  cudaMemsetAsync(w, 0, L.zero_bytes, s);
  const u32* kp = reinterpret_cast<const u32*>(keys);
  DISPATCH_MODE(key_mode(dtype, largest), stage_delegates, kp, n, alpha, beta, out_delegates, w, L, s, num_sms());
  return cuda_status();
}

dtopk_status dtopk_kth_largest(const uint32_t* keys, uint64_t n, uint64_t k, uint32_t* out_kth, void* ws,
                               size_t ws_bytes, void* stream) {
  DTOPK_RANGE("dtopk_kth_largest");
  dtopk_status st = check_common(keys, n, DTOPK_U32, k);
  if (st != DTOPK_OK) return st;
  if (out_kth == nullptr) return DTOPK_INVALID_ARG;
  const Layout L = make_layout(n, k, 0, 1, 1);
  if (ws == nullptr || ws_bytes < L.total) return DTOPK_WORKSPACE_TOO_SMALL;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  char* w = reinterpret_cast<char*>(ws);
  Ctrl* ctrl = reinterpret_cast<Ctrl*>(w + L.ctrl);
  cudaMemsetAsync(w, 0, L.zero_bytes, s);
  const int nsm = num_sms();
  const int gs = grid_for((n + 2047) / 2048, nsm * 4);
  SelArgs sd{keys, n, nullptr, ctrl, &ctrl->selP, reinterpret_cast<u32*>(w + L.selbuf), k, 0,
             reinterpret_cast<u32*>(w + L.sel_tcnt)};
  sel_pass1<KM_KEY><<<gs, 256, 0, s>>>(sd);
  counted();
  sel_pass2<KM_KEY><<<gs, 256, 0, s>>>(sd);
  counted();
  sel_pass3<<<gs, 256, 0, s>>>(sd);
  counted();
  sel_finalize<<<1, 256, 0, s>>>(&ctrl->selP, out_kth);
  counted();
  return cuda_status();
}

size_t dtopk_merge_tmp_pairs(int n_lists, uint64_t cap) { return 2ull * (uint64_t)((n_lists + 1) / 2) * cap; }

dtopk_status dtopk_merge_lists(int dtype, int largest, const uint32_t* in_val, int vmul, int vstride,
                               const int64_t* in_idx,
                               const int64_t* in_off, int64_t in_stride, const int64_t* in_len,
                               int64_t len_stride, int n_lists, uint64_t cap, uint32_t* out_val, int64_t* out_idx, uint32_t* tmp_val, int64_t* tmp_idx,
                               int64_t* tmp_len, void* stream) {
  DTOPK_RANGE("dtopk_merge_lists");
  if (dtype != DTOPK_U32 && dtype != DTOPK_F32) return DTOPK_INVALID_ARG;
  if (n_lists < 1 || cap < 1 || (vstride != 1 && vstride != 2) || vmul < 1) return DTOPK_INVALID_ARG;
  if (!in_val || !in_idx || !in_len || !out_val || !out_idx || !tmp_len) return DTOPK_INVALID_ARG;
  if (n_lists > 1 && (!tmp_val || !tmp_idx)) return DTOPK_INVALID_ARG;
  if ((!in_off && in_stride < 0) || len_stride < 1) return DTOPK_INVALID_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  DISPATCH_MODE(key_mode(dtype, largest), run_merge_lists, in_val, vmul, vstride, in_idx, in_off, in_stride, in_len, len_stride,
                n_lists, (int64_t)cap, out_val, out_idx, tmp_val, tmp_idx, tmp_len, s);
  return cuda_status();
}

dtopk_status dtopk_dsel_init(int64_t* state, int64_t* hist, uint64_t k, void* stream) {
  if (!state || !hist || k < 1) return DTOPK_INVALID_ARG;
  launch_pdl(dsel_init, dim3(1), dim3(256), 0, reinterpret_cast<cudaStream_t>(stream),
             reinterpret_cast<long long*>(state), reinterpret_cast<long long*>(hist), (long long)k);
  counted();
  return cuda_status();
}

dtopk_status dtopk_dsel_hist(int dtype, int largest, const uint32_t* bits, const int64_t* cnt, uint64_t cap,
                             const int64_t* state, int pass, int64_t* hist, void* stream) {
  DTOPK_RANGE("dtopk_dsel_hist");
  if (dtype != DTOPK_U32 && dtype != DTOPK_F32) return DTOPK_INVALID_ARG;
  if (!bits || !cnt || !state || !hist || pass < 0 || pass > 2) return DTOPK_INVALID_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  DISPATCH_MODE(key_mode(dtype, largest), run_dsel_hist, bits, cnt, state, pass, hist, cap, s);
  return cuda_status();
}

dtopk_status dtopk_dsel_digit(int dtype, int largest, int64_t* state, int64_t* hist, int pass, const uint32_t* bits,
                              const int64_t* cnt, int64_t* gt_eq, void* stream) {
  DTOPK_RANGE("dtopk_dsel_digit");
  if (dtype != DTOPK_U32 && dtype != DTOPK_F32) return DTOPK_INVALID_ARG;
  if (!state || !hist || !bits || !cnt || !gt_eq || pass < 0 || pass > 2) return DTOPK_INVALID_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  DISPATCH_MODE(key_mode(dtype, largest), run_dsel_digit, state, hist, pass, bits, cnt, gt_eq, s);
  return cuda_status();
}

dtopk_status dtopk_dsel_place(const int64_t* gathered, const int64_t* state, int rank, int world, uint64_t k,
                              const uint32_t* bits, const int64_t* idx, int64_t* slots, int64_t* seg_off,
                              int64_t* seg_len, void* stream) {
  DTOPK_RANGE("dtopk_dsel_place");
  if (!gathered || !state || !bits || !idx || !slots || !seg_off || !seg_len) return DTOPK_INVALID_ARG;
  if (world < 1 || rank < 0 || rank >= world || k < 1) return DTOPK_INVALID_ARG;
  const int g = grid_for((k + 255) / 256, num_sms() * 4);
  launch_pdl(dsel_place, dim3(g), dim3(256), 0, reinterpret_cast<cudaStream_t>(stream),
             reinterpret_cast<const long long*>(gathered), reinterpret_cast<const long long*>(state), rank, world,
             (long long)k, bits, reinterpret_cast<const long long*>(idx), reinterpret_cast<long long*>(slots),
             reinterpret_cast<long long*>(seg_off), reinterpret_cast<long long*>(seg_len));
  counted();
  return cuda_status();
}

dtopk_status dtopk_qualify(const uint32_t* delegates, uint64_t n_delegates, int beta, uint32_t theta,
                           uint32_t* sel_values, uint32_t* sel_tags, uint32_t* part_values, uint32_t* part_tags,
                           uint32_t* fq_sids, int64_t* out_counts, void* ws, size_t ws_bytes, void* stream) {
  DTOPK_RANGE("dtopk_qualify");
  if (!delegates || !out_counts || beta < 1 || n_delegates == 0 || n_delegates % (uint64_t)beta) return DTOPK_INVALID_ARG;
  if (!sel_values || !sel_tags || !part_values || !part_tags || !fq_sids) return DTOPK_INVALID_ARG;
  const u64 tiles = (n_delegates + STG_TILE - 1) / STG_TILE;
  if (ws == nullptr || ws_bytes < dtopk_stage_workspace_bytes(n_delegates)) return DTOPK_WORKSPACE_TOO_SMALL;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  u32* tc = reinterpret_cast<u32*>(ws);
  qual_count<<<(unsigned)tiles, STG_THREADS, 0, s>>>(delegates, n_delegates, beta, theta, tc);
  stg_scan<<<1, STG_THREADS, 0, s>>>(tc, tiles, STG_STREAMS, reinterpret_cast<int64_t*>(out_counts));
  qual_emit<<<(unsigned)tiles, STG_THREADS, 0, s>>>(delegates, n_delegates, beta, theta, tc, sel_values, sel_tags,
                                                    part_values, part_tags, fq_sids);
  counted(3);
  return cuda_status();
}

size_t dtopk_stage_workspace_bytes(uint64_t n_elements) {
  return (size_t)((n_elements + STG_TILE - 1) / STG_TILE) * STG_STREAMS * 4 + 256;
}

dtopk_status dtopk_concat(const void* keys, uint64_t n, int dtype, int largest, int alpha, const uint32_t* fq_sids,
                          uint64_t n_fq, uint32_t theta, void* out_values, int64_t* out_count, void* ws,
                          size_t ws_bytes, void* stream) {
  DTOPK_RANGE("dtopk_concat");
  dtopk_status st = check_common(keys, n, dtype, 1);
  if (st != DTOPK_OK) return st;
  if (alpha < 0 || alpha > 40 || !out_values || !out_count || (n_fq && !fq_sids)) return DTOPK_INVALID_ARG;
  if (ws == nullptr || ws_bytes < dtopk_stage_workspace_bytes(std::max<u64>(1, n_fq << alpha)))
    return DTOPK_WORKSPACE_TOO_SMALL;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  DISPATCH_MODE(key_mode(dtype, largest), run_concat, reinterpret_cast<const u32*>(keys), n, alpha, fq_sids, n_fq,
                theta, reinterpret_cast<u32*>(out_values), out_count, reinterpret_cast<u32*>(ws), s);
  return cuda_status();
}

dtopk_status dtopk_min_at_least(const uint32_t* keys, uint64_t n, uint32_t edge, uint32_t* out_min, void* stream) {
  if (!keys || !out_min) return DTOPK_INVALID_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  cudaMemsetAsync(out_min, 0xff, 4, s);
  if (n) {
    min_at_least<<<grid_for((n + STG_THREADS - 1) / STG_THREADS, num_sms() * 8), STG_THREADS, 0, s>>>(keys, n, edge,
                                                                                                  out_min);
    counted();
  }
  return cuda_status();
}

}  // extern "C"
