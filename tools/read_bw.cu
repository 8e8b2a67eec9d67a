// read_bw.cu -- pure-read HBM ceiling on this B200 (tooling, not the product).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/read_bw tools/read_bw.cu && /tmp/read_bw
//
// Streams 4 GiB (2^30 u32, the BASELINE config-2 input) through variants of a
// trivially cheap reduction and prints GB/s for each: the upper bound K1
// (k1_delegates, one read of V) can reach.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

typedef unsigned int u32;
typedef unsigned long long u64;

__device__ __forceinline__ uint4 ldnc(const u32* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}

template <int U>
__global__ void ldg_max(const u32* __restrict__ x, u64 n, u32* out) {
  u32 m = 0;
  const u64 stride = (u64)gridDim.x * blockDim.x * 4 * U;
  for (u64 b = ((u64)blockIdx.x * blockDim.x + threadIdx.x) * 4; b < n; b += stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const u64 o = b + (u64)u * gridDim.x * blockDim.x * 4;
      v[u] = o < n ? ldnc(x + o) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; u++) m = max(m, max(max(v[u].x, v[u].y), max(v[u].z, v[u].w)));
  }
  if (m == 0x12345678u) out[0] = m;
}

// contiguous per-CTA chunks (like K1's chunk ownership)
template <int U>
__global__ void ldg_chunk(const u32* __restrict__ x, u64 n, u32* out) {
  u32 m = 0;
  const u64 chunk = (u64)blockDim.x * 4 * U;
  const u64 nch = n / chunk;
  for (u64 c = blockIdx.x; c < nch; c += gridDim.x) {
    const u32* p = x + c * chunk + threadIdx.x * 4;
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; u++) v[u] = ldnc(p + (u64)u * blockDim.x * 4);
#pragma unroll
    for (int u = 0; u < U; u++) m = max(m, max(max(v[u].x, v[u].y), max(v[u].z, v[u].w)));
  }
  if (m == 0x12345678u) out[0] = m;
}

// TMA 1-D bulk ring: one producer lane, NW consumer warps, STAGES x CH bytes
template <int STAGES, int CH, int NW>
__global__ void __launch_bounds__((NW + 1) * 32, 1) tma_ring(const u32* __restrict__ x, u64 n, u32* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  u64* full = reinterpret_cast<u64*>(smem + (size_t)STAGES * CH);
  u64* empty = full + STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; s++) {
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"((u32)__cvta_generic_to_shared(full + s)));
      asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"((u32)__cvta_generic_to_shared(empty + s)), "r"(1));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const u64 nch = n * 4 / CH;
  const u64 my = nch > blockIdx.x ? (nch - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  if (warp == NW) {
    if (lane == 0) {
      for (u64 i = 0; i < my; i++) {
        const int s = i % STAGES;
        const u32 ph = (i / STAGES) & 1;
        if (i >= STAGES) {
          asm volatile(
              "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(
                  (u32)__cvta_generic_to_shared(empty + s)),
              "r"(ph ^ 1));
        }
        const u32 fb = (u32)__cvta_generic_to_shared(full + s);
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(fb), "r"(CH));
        const unsigned char* src = reinterpret_cast<const unsigned char*>(x) + (blockIdx.x + i * gridDim.x) * (u64)CH;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                (u32)__cvta_generic_to_shared(smem + (size_t)s * CH)),
            "l"(src), "r"(CH), "r"(fb)
            : "memory");
      }
    }
    return;
  }
  u32 m = 0;
  for (u64 i = warp; i < my; i += NW) {
    const int s = i % STAGES;
    const u32 ph = (i / STAGES) & 1;
    asm volatile(
        "{\n .reg .pred p;\n W2: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra W2;\n}\n" ::"r"(
            (u32)__cvta_generic_to_shared(full + s)),
        "r"(ph));
    const uint4* b = reinterpret_cast<const uint4*>(smem + (size_t)s * CH);
#pragma unroll 4
    for (int j = lane; j < CH / 16; j += 32) {
      const uint4 v = b[j];
      m = max(m, max(max(v.x, v.y), max(v.z, v.w)));
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"((u32)__cvta_generic_to_shared(empty + s)));
  }
  if (m == 0x12345678u) out[0] = m;
}

template <typename F>
float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; i++) f();
  float best = 1e9;
  for (int r = 0; r < 10; r++) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    if (cudaEventSynchronize(b) != cudaSuccess) { printf("err %s\n", cudaGetErrorString(cudaGetLastError())); return -1; }
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    best = ms < best ? ms : best;
  }
  return best;
}

int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  const u64 n = 1ull << 30;
  u32 *x, *out;
  if (cudaMalloc(&x, n * 4) != cudaSuccess || cudaMalloc(&out, 64) != cudaSuccess) { printf("malloc failed\n"); return 1; }
  printf("alloc ok\n");
  cudaMemset(x, 1, n * 4);
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  auto rep = [&](const char* name, float ms) { printf("%-40s %8.3f ms  %7.1f GB/s\n", name, ms, n * 4 / (ms * 1e-3) / 1e9); };
  for (int bpsm : {1, 2, 4, 8}) {
    char nm[64];
    snprintf(nm, 64, "ldg_max<4> 1024t x %d/SM", bpsm);
    rep(nm, timeit([&] { ldg_max<4><<<nsm * bpsm, 1024>>>(x, n, out); }));
    snprintf(nm, 64, "ldg_max<8> 512t x %d/SM", bpsm);
    rep(nm, timeit([&] { ldg_max<8><<<nsm * bpsm, 512>>>(x, n, out); }));
    snprintf(nm, 64, "ldg_chunk<8> 256t x %d/SM", bpsm);
    rep(nm, timeit([&] { ldg_chunk<8><<<nsm * bpsm, 256>>>(x, n, out); }));
    snprintf(nm, 64, "ldg_chunk<16> 256t x %d/SM", bpsm);
    rep(nm, timeit([&] { ldg_chunk<16><<<nsm * bpsm, 256>>>(x, n, out); }));
  }
#define TMA(ST, CH, NW, BPS)                                                                          \
  {                                                                                                   \
    auto k = tma_ring<ST, CH, NW>;                                                                    \
    size_t sm = (size_t)ST * CH + 2 * ST * 8;                                                         \
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);                    \
    rep("tma_ring<" #ST "," #CH "," #NW "> x" #BPS, timeit([&] { k<<<nsm * BPS, (NW + 1) * 32, sm>>>(x, n, out); })); \
  }
  TMA(16, 8192, 8, 1)
  TMA(24, 8192, 8, 1)
  TMA(8, 16384, 8, 1)
  TMA(12, 16384, 4, 1)
  TMA(6, 32768, 6, 1)
  TMA(8, 8192, 8, 2)
  TMA(6, 16384, 6, 2)
  TMA(4, 16384, 4, 3)
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
