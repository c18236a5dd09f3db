// Config-population synthesis on the device.
//
// Bitwise the same population as the host restatement
// paper_2110_04421_b200/confignet.py::synthesize (ages, contiguous
// households, keyed workplace shuffle, seed infections), built from the same
// keyed hashes (purposes 76-79) with CUB scans, selects and radix sorts
// instead of host loops: 10M agents in milliseconds instead of ~7 s of numpy.
//
//   age       : #(cum_age <= u) clipped, u = keyed_u(POP_AGE, a);
//   households: size_k = sizes[#(cum_hh <= u_k)] for household k = 0, 1, ...
//               (u_k = keyed_u(POP_HOUSEHOLD, k)); ends = inclusive scan; the
//               household of agent a is the first k with ends[k] > a, the
//               last one truncated at N;
//   workplaces: workers (age in the worker bands) stably sorted by
//               hash(POP_WORKPLACE, worker) (ties: ascending id), cut into
//               blocks of wp_min + floor(u_w * span), u_w = keyed_u(
//               POP_WORKPLACE, w, k=1), the last block truncated;
//   seeds     : the `n_seeds` agents with the smallest hash(POP_SEEDS, a)
//               (ties: ascending id), in ascending id order.
#pragma once

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include "epi_common.cuh"

namespace epi {

enum PopPurpose : int { P_POP_AGE = 76, P_POP_HOUSEHOLD = 77, P_POP_WORKPLACE = 78, P_POP_SEEDS = 79 };

struct PopTables {
  double cum_age[9];
  double cum_hh[32];
  int32_t hh_sizes[32];
  int32_t n_sizes;
  uint32_t worker_mask;   // bit b: age band b is a worker band
};

__device__ __forceinline__ uint64_t keyed_h(uint64_t prefix, uint64_t i, uint64_t k = 0) {
  return fold(fold(prefix, i), k);
}

// Per agent: age, worker flag, seed key; per household index k = a: its size.
__global__ void k_pop_agents(PopTables T, int64_t n, uint64_t p_age, uint64_t p_hh, uint64_t p_seed,
                             int8_t* __restrict__ age, uint8_t* __restrict__ worker,
                             int64_t* __restrict__ hh_size_k, uint64_t* __restrict__ seed_key,
                             int32_t* __restrict__ ids) {
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < n; a += (int64_t)gridDim.x * blockDim.x) {
    const double u = unit(keyed_h(p_age, (uint64_t)a));
    int b = 0;
#pragma unroll
    for (int i = 0; i < 9; ++i) b += (T.cum_age[i] <= u) ? 1 : 0;
    b = b < 8 ? b : 8;
    age[a] = (int8_t)b;
    worker[a] = (uint8_t)((T.worker_mask >> b) & 1u);
    const double uh = unit(keyed_h(p_hh, (uint64_t)a));
    int j = 0;
    for (int i = 0; i < T.n_sizes; ++i) j += (T.cum_hh[i] <= uh) ? 1 : 0;
    j = j < T.n_sizes - 1 ? j : T.n_sizes - 1;
    hh_size_k[a] = T.hh_sizes[j];
    seed_key[a] = keyed_h(p_seed, (uint64_t)a);
    ids[a] = (int32_t)a;
  }
}

// first k in [0, len) with ends[k] > x (ends non-decreasing; len if none)
__device__ __forceinline__ int64_t first_above(const int64_t* __restrict__ ends, int64_t len, int64_t x) {
  int64_t lo = 0, hi = len;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (ends[mid] > x) hi = mid; else lo = mid + 1;
  }
  return lo;
}

__global__ void k_pop_households(int64_t n, const int64_t* __restrict__ ends, const int64_t* __restrict__ size_k,
                                 int32_t* __restrict__ household_id, uint8_t* __restrict__ hh_off,
                                 uint8_t* __restrict__ hh_size) {
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < n; a += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = first_above(ends, n, a);
    const int64_t start = ends[k] - size_k[k];
    const int64_t sz = ends[k] <= n ? size_k[k] : n - start;   // the last household is truncated
    household_id[a] = (int32_t)k;
    hh_off[a] = (uint8_t)(a - start);
    hh_size[a] = (uint8_t)sz;
  }
}

// Workplace keys of the compacted workers; the block sizes of w < max_w.
__global__ void k_pop_worker_keys(const int32_t* __restrict__ workers, const int64_t* __restrict__ n_workers,
                                  uint64_t p_wp, uint64_t* __restrict__ keys, int64_t max_w, int wp_min,
                                  int span, int64_t* __restrict__ wsz) {
  const int64_t W = *n_workers;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < W; i += stride)
    keys[i] = keyed_h(p_wp, (uint64_t)workers[i]);
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < max_w; w += stride)
    wsz[w] = wp_min + (int64_t)(unit(keyed_h(p_wp, (uint64_t)w, 1)) * (double)span);
}

// Member position p -> its workplace (first w with wend[w] > p) and local
// slot; per workplace its base and (truncated) size; the counts out.
__global__ void k_pop_workplaces(const int32_t* __restrict__ members, const int64_t* __restrict__ n_workers,
                                 const int64_t* __restrict__ wend, const int64_t* __restrict__ wsz, int64_t max_w,
                                 int32_t* __restrict__ wp_id, uint8_t* __restrict__ wp_local,
                                 int32_t* __restrict__ wp_base, int32_t* __restrict__ wp_size,
                                 int64_t* __restrict__ counts) {
  const int64_t W = *n_workers;
  const int64_t n_w = W > 0 ? first_above(wend, max_w, W - 1) + 1 : 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t0 == 0) {
    counts[0] = n_w;
    counts[1] = W;
  }
  for (int64_t p = t0; p < W; p += stride) {
    const int64_t w = first_above(wend, n_w, p);
    const int64_t base = wend[w] - wsz[w];
    wp_id[members[p]] = (int32_t)w;
    wp_local[members[p]] = (uint8_t)(p - base);
  }
  for (int64_t w = t0; w < n_w; w += stride) {
    const int64_t base = wend[w] - wsz[w];
    wp_base[w] = (int32_t)base;
    wp_size[w] = (int32_t)(wend[w] <= W ? wsz[w] : W - base);
  }
}

__global__ void k_widen(const int32_t* __restrict__ a, int64_t n, int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = a[i];
}

__global__ void k_fill_i32(int32_t* __restrict__ p, int64_t n, int32_t v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

}  // namespace epi
