// Replication summaries on the device (output part):
// the quartiles of every time-series metric across replications
// (runner.py:195-207 `summarize`: np.percentile(stacked, [25, 50, 75],
// axis=1), numpy's default "linear" method), straight from the device
// records of an ensemble, so a 1,024-replica sweep never copies its
// [R, horizon, 24] records to the host.
//
// One block per (metric, step): the R values are sorted in shared memory
// (bitonic, R <= 4096) and interpolated exactly as numpy does:
//   v = (n - 1) q, i = floor(v), g = v - i,  a = x[i], b = x[min(i + 1, n - 1)]
//   lerp = g < 0.5 ? a + (b - a) g : b - (b - a)(1 - g)        (numpy _lerp)
// with the int64 -> float64 conversions numpy applies, so the result is
// bitwise np.percentile's (tests/test_gpu_series.py, golden fixtures from the
// reference's own `summarize`).
#pragma once

#include <cstdint>

namespace epi {

constexpr int SUMMARY_MAX_R = 4096;

__device__ __forceinline__ double np_lerp(int64_t a, int64_t b, double g) {
  const double d = (double)(b - a);
  return g >= 0.5 ? (double)b - d * (1.0 - g) : (double)a + d * g;
}

// data [R][H][C] int64, cols[n_cols] = record columns, out [n_cols][H][3]
__global__ void __launch_bounds__(1024) k_quartiles(const int64_t* __restrict__ data, int R, int H, int C,
                                                    const int32_t* __restrict__ cols, double* __restrict__ out) {
  __shared__ int64_t x[SUMMARY_MAX_R];
  const int step = blockIdx.x, mi = blockIdx.y;
  const int col = cols[mi];
  int P = 1;
  while (P < R) P <<= 1;
  for (int i = threadIdx.x; i < P; i += blockDim.x)
    x[i] = i < R ? data[((int64_t)i * H + step) * C + col] : INT64_MAX;
  __syncthreads();
  for (int k = 2; k <= P; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < P; i += blockDim.x) {
        const int l = i ^ j;
        if (l > i) {
          const bool up = (i & k) == 0;
          const int64_t a = x[i], b = x[l];
          if ((a > b) == up) { x[i] = b; x[l] = a; }
        }
      }
      __syncthreads();
    }
  if (threadIdx.x < 3) {
    const double q = 0.25 * (threadIdx.x + 1);
    const double v = (double)(R - 1) * q;     // numpy "linear": (n - 1) * q
    const double fi = floor(v);
    const double g = v - fi;
    int i = (int)fi;
    i = i < 0 ? 0 : (i > R - 1 ? R - 1 : i);
    const int i1 = i + 1 > R - 1 ? R - 1 : i + 1;
    out[((int64_t)mi * H + step) * 3 + threadIdx.x] = np_lerp(x[i], x[i1], g);
  }
}

}  // namespace epi
