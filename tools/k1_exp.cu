// k1_exp.cu -- times k1_delegates alone on 2^30 random u32 keys (tooling).
//   nvcc ... -DDTOPK_K1_EXP=<0|1|2> tools/k1_exp.cu
#include <cstdio>
#ifndef DTOPK_GEN_DIST
#define DTOPK_GEN_DIST 0
#endif
#include "../paper_2109_08219_b200/csrc/delegate.cuh"
#include "../paper_2109_08219_b200/csrc/generate.cuh"
using namespace dtopk;

int main(int argc, char** argv) {
  setvbuf(stdout, NULL, _IONBF, 0);
  const u64 n = 1ull << 30;
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  u32 *x, *D, *meta;
  ull* hist;
  cudaMalloc(&x, n * 4);
  cudaMalloc(&D, (n / 32) * 4);
  cudaMalloc(&meta, (n / 64) * 4);
  cudaMalloc(&hist, NB1 * 8);
  gen_kernel<<<nsm * 8, 256>>>(x, n, DTOPK_GEN_DIST, 1234, 0x5A5A5A5A);
  for (int alpha : {6, 8, 11, 16}) {
    if (alpha > K1_LOG_CHUNK && alpha != 16) continue;
    const u64 S = n >> alpha;
    K1Args a{x, n, alpha, S, D, nullptr, hist, 1, meta, nullptr};
    if (alpha > K1_LOG_CHUNK) { cudaMalloc(&a.partial, (n / K1_CHUNK) * 8); cudaMalloc(&a.pmeta, (n / K1_CHUNK) * 8); }
    cudaFuncSetAttribute(k1_delegates<0, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K1_SMEM);
    const u64 nch = n / K1_CHUNK;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e9;
    for (int r = 0; r < 13; r++) {
      cudaEventRecord(e0);
      k1_delegates<0, 2><<<(int)std::min<u64>(nch, (u64)nsm * K1_CPS), K1_THREADS, K1_SMEM>>>(a);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r >= 3) best = ms < best ? ms : best;
    }
    printf("EXP=%d alpha=%d k1 %.4f ms  %.1f GB/s  (%s)\n", DTOPK_K1_EXP, alpha, best, n * 4 / (best * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
