// generate.cuh -- counter-based synthetic inputs (value i depends only on
// (seed, i)), the device twin of paper_2109_08219_b200/data.py.  Mirrors the
// reference datasets (data.py:58-113): uniform u32 (UD), rint(N(1e8, 10))
// (ND), plus the BASELINE configs' float32 normal / Pareto(1.5) and the
// adversarial ascending / all-equal / few-distinct vectors.  Not on the hot path.
#pragma once

#include "common.cuh"

namespace dtopk {

enum GenDist : int {
  GEN_UNIFORM = 0,
  GEN_ASCENDING = 1,
  GEN_CONSTANT = 2,
  GEN_FEW_DISTINCT = 3,
  GEN_NORMAL_F32 = 4,
  GEN_PARETO_F32 = 5,
  GEN_ND_U32 = 6,
  GEN_DESCENDING = 7,
};

__device__ __forceinline__ u64 splitmix64(u64 x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// uniform double in (0, 1) from 53 random bits
__device__ __forceinline__ double u01(u64 h) { return ((double)(h >> 11) + 0.5) * (1.0 / 9007199254740992.0); }

__global__ void __launch_bounds__(256) gen_kernel(u32* __restrict__ out, u64 n, int dist, u64 seed, u64 param) {
  const u64 key = splitmix64(seed ^ 0xD1B54A32D192ED03ull);
  for (u64 i = (u64)blockIdx.x * 256 + threadIdx.x; i < n; i += (u64)gridDim.x * 256) {
    const u64 h = splitmix64(key + i);
    u32 v;
    switch (dist) {
      case GEN_UNIFORM: v = (u32)(h >> 32); break;
      case GEN_ASCENDING: v = (u32)(i + param); break;
      case GEN_DESCENDING: v = (u32)(param - i); break;
      case GEN_CONSTANT: v = (u32)param; break;
      case GEN_FEW_DISTINCT: v = (u32)((h >> 32) % (param ? param : 1)); break;
      case GEN_NORMAL_F32:
      case GEN_ND_U32: {
        const u64 h2 = splitmix64(h ^ 0x632BE59BD9B4E019ull);
        const double r = sqrt(-2.0 * log(u01(h))) * cospi(2.0 * u01(h2));
        if (dist == GEN_NORMAL_F32) {
          v = __float_as_uint((float)r);
        } else {
          double x = rint(1e8 + 10.0 * r);
          x = x < 0 ? 0 : (x > 4294967295.0 ? 4294967295.0 : x);
          v = (u32)x;
        }
        break;
      }
      case GEN_PARETO_F32: {
        // numpy's pareto(a): (1 - U)^(-1/a) - 1, a = param / 1000 (1.5 -> 1500)
        const double a = param ? (double)param / 1000.0 : 1.5;
        v = __float_as_uint((float)(pow(u01(h), -1.0 / a) - 1.0));
        break;
      }
      default: v = 0;
    }
    out[i] = v;
  }
}

}  // namespace dtopk
