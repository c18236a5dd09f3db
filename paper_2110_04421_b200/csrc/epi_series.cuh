// Replication summaries on the device (output part):
// the quartiles of every time-series metric across replications
// (runner.py:195-207 `summarize`: np.percentile(stacked, [25, 50, 75],
// axis=1), numpy's default "linear" method), straight from the device
// records of an ensemble, so a 1,024-replica sweep never copies its
// [R, horizon, 24] records to the host.
//
// One block per (metric, step): the R values are sorted in shared memory
// (bitonic, R <= 4096; more replications: k_quartiles_large) and
// interpolated exactly as numpy does:
//   v = (n - 1) q, i = floor(v), g = v - i,  a = x[i], b = x[min(i + 1, n - 1)]
//   lerp = g < 0.5 ? a + (b - a) g : b - (b - a)(1 - g)        (numpy _lerp)
// with the int64 -> float64 conversions numpy applies, so the result is
// bitwise np.percentile's (tests/test_gpu_series.py, golden fixtures from the
// reference's own `summarize`).
#pragma once

#include <climits>
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

// More than SUMMARY_MAX_R replications: the six order statistics the three
// quartiles need (x[i], x[i + 1] per quantile) by bisection on the value:
// the k-th smallest is the least v with #{x <= v} > k, each count a block
// reduction over the R values in global memory (64 rounds per statistic at
// most, int64 values).  Same interpolation as k_quartiles.
__device__ __forceinline__ long long block_sum_ll(long long v, long long* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xFFFFFFFFu, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  long long t = 0;
  for (int w = 0; w < nw; ++w) t += red[w];
  return t;
}
__global__ void __launch_bounds__(1024) k_quartiles_large(const int64_t* __restrict__ data, int64_t R, int H, int C,
                                                          const int32_t* __restrict__ cols, double* __restrict__ out) {
  __shared__ long long red[32];
  __shared__ long long lo_s, hi_s;
  const int step = blockIdx.x, mi = blockIdx.y;
  const int col = cols[mi];
  auto at = [&](int64_t r) { return data[(r * H + step) * C + col]; };
  long long mn = LLONG_MAX, mx = LLONG_MIN;
  for (int64_t r = threadIdx.x; r < R; r += blockDim.x) {
    const long long v = at(r);
    mn = v < mn ? v : mn;
    mx = v > mx ? v : mx;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const long long a = __shfl_down_sync(0xFFFFFFFFu, mn, o), b = __shfl_down_sync(0xFFFFFFFFu, mx, o);
    mn = a < mn ? a : mn;
    mx = b > mx ? b : mx;
  }
  if (threadIdx.x == 0) { lo_s = LLONG_MAX; hi_s = LLONG_MIN; }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) { atomicMin(&lo_s, mn); atomicMax(&hi_s, mx); }
  __syncthreads();
  const long long vmin = lo_s, vmax = hi_s;
  double res[3];
  for (int qi = 0; qi < 3; ++qi) {
    const double q = 0.25 * (qi + 1);
    const double v = (double)(R - 1) * q;
    const double fi = floor(v);
    const double g = v - fi;
    int64_t i = (int64_t)fi;
    i = i < 0 ? 0 : (i > R - 1 ? R - 1 : i);
    const int64_t i1 = i + 1 > R - 1 ? R - 1 : i + 1;
    long long xs[2];
    for (int w = 0; w < 2; ++w) {
      const int64_t k = w == 0 ? i : i1;          // rank wanted (0-based)
      long long lo = vmin, hi = vmax;              // invariant: answer in [lo, hi]
      while (lo < hi) {
        const long long mid = lo + (long long)(((unsigned long long)(hi - lo)) >> 1);
        long long c = 0;
        for (int64_t r = threadIdx.x; r < R; r += blockDim.x) c += at(r) <= mid ? 1 : 0;
        c = block_sum_ll(c, red);
        if (c > k) hi = mid;
        else lo = mid + 1;
      }
      xs[w] = lo;
    }
    res[qi] = np_lerp(xs[0], xs[1], g);
  }
  if (threadIdx.x == 0)
    for (int qi = 0; qi < 3; ++qi) out[((int64_t)mi * H + step) * 3 + qi] = res[qi];
}

}  // namespace epi
