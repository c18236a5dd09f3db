// Device-side building blocks shared by every kernel of libepib200.
//
//  * keyed splitmix64 draws — bit-identical to the reference chain
//    (pkg/src/epivec/rng.py:60-100): u = (h >> 11) * 2^-53 on the 2^-53 grid;
//  * progression lookups: cumulative branch tables (progression.py:117-123)
//    and the exact delay step functions (threshold tables, see
//    paper_2110_04421_b200/progression.py) replacing scipy's ppf + rint
//    (progression.py:48-62, 85-87);
//  * the 16-bit per-agent source code used by every message pass.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/epi_b200.h"

namespace epi {

constexpr int8_t NEVER8 = -1;
constexpr int32_t NEVER = -1;

enum StageId : int {
  S_SUS = 0, S_ASYM = 1, S_PMILD = 2, S_PSEV = 3, S_MILD = 4, S_SEV = 5,
  S_HOSP = 6, S_ICU = 7, S_REC = 8, S_VAC = 9, S_DEAD = 10
};

// Purpose tags (rng.py:37-57 + config-network tags of keyed.py).
enum PurposeId : int {
  P_INFECTION = 1, P_INFECTION_EDGE = 2, P_ENTRY = 3, P_BRANCH = 4, P_DELAY = 5, P_TEST_POS = 6,
  P_TEST_TURN = 7, P_QDROP = 8, P_DEN = 9, P_APP = 10, P_VAX = 11,
  P_NET_RCOUNT = 72, P_NET_RPERM = 73, P_NET_WPERM = 74, P_NET_WSHIFT = 75
};

__host__ __device__ __forceinline__ bool infectious_stage(int s) { return s >= 1 && s <= 5; }
__host__ __device__ __forceinline__ bool asym_like_stage(int s) { return s >= 1 && s <= 3; }
__host__ __device__ __forceinline__ bool active_stage(int s) { return s >= 1 && s <= 7; }

// ---- keyed hash ---------------------------------------------------------
constexpr uint64_t K_GOLDEN = 0x9E3779B97F4A7C15ull;
constexpr uint64_t K_MIX1 = 0xBF58476D1CE4E5B9ull;
constexpr uint64_t K_MIX2 = 0x94D049BB133111EBull;
constexpr uint64_t K_INIT = 0x243F6A8885A308D3ull;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * K_MIX1;
  z = (z ^ (z >> 27)) * K_MIX2;
  return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t fold(uint64_t h, uint64_t v) {
  return mix64(h ^ (K_GOLDEN * (v + 1)));
}
__host__ __device__ __forceinline__ uint64_t key_prefix(uint64_t seed, int64_t step, int purpose) {
  return fold(fold(mix64(K_INIT ^ seed), (uint64_t)step), (uint64_t)purpose);
}
__host__ __device__ __forceinline__ double unit(uint64_t h) {
  return (double)(h >> 11) * 0x1p-53;
}
__device__ __forceinline__ double keyed_u(uint64_t prefix, uint64_t agent, uint64_t k = 0) {
  return unit(fold(fold(prefix, agent), k));
}

// Prefixes of one step for every purpose the step phases draw from.
struct StepKeys {
  uint64_t p[12];       // indexed by purpose 1..11
};
inline StepKeys make_step_keys(uint64_t seed, int step) {
  StepKeys k;
  for (int i = 0; i < 12; ++i) k.p[i] = key_prefix(seed, step, i);
  return k;
}

// Optional injected draws (tests): per purpose a device double[N] or null.
struct Injected {
  const double* u[12];
};

__device__ __forceinline__ double draw(const StepKeys& K, const Injected* inj, int purpose,
                                       int64_t agent, int k = 0) {
  if (inj != nullptr && inj->u[purpose] != nullptr) return inj->u[purpose][agent];
  return keyed_u(K.p[purpose], (uint64_t)agent, (uint64_t)k);
}

// ---- progression ----------------------------------------------------------
// j = #(u >= cum[stage][age][:]) clipped to n-1 (progression.py:117-123)
__device__ __forceinline__ int pick_branch(const epi_params* __restrict__ P, int stage, int age,
                                           double u) {
  const int n = P->n_targets[stage];
  int j = 0;
  for (int i = 0; i < n; ++i) j += (u >= P->cum[stage][age][i]) ? 1 : 0;
  return j < n - 1 ? j : n - 1;
}

// delay = 1 + #(tau <= u): exact encoding of max(rint(ppf(u)), 1)
//
// With `lut` (TAU_LUT entries per spec: lut[k] = #(tau < k / TAU_LUT)) the
// count starts at the bucket of u and steps over the few thresholds inside
// the bucket: two dependent loads instead of a log2(len)-deep binary search.
// Both give the same count: #(tau < floor(u*L)/L) <= #(tau <= u).
constexpr int TAU_LUT = 1024;
__device__ __forceinline__ int delay_steps(const epi_params* __restrict__ P, int spec, double u,
                                           const uint16_t* __restrict__ lut = nullptr) {
  const double* tau = P->tau[spec];
  const int len = P->tau_len[spec];
  if (lut != nullptr) {
    int lo = lut[spec * TAU_LUT + (int)(u * TAU_LUT)];
    while (lo < len && tau[lo] <= u) ++lo;
    return 1 + lo;
  }
  int lo = 0, hi = len;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (tau[mid] <= u) lo = mid + 1; else hi = mid;
  }
  return 1 + lo;
}

// (next_stage, delay) out of `stage`; absorbing / entry stages give
// (NEVER, NEVER) like progression.py:137-162.
__device__ __forceinline__ void schedule(const epi_params* __restrict__ P, int stage, int age,
                                         double ub, double ud, int& next, int& delay,
                                         const uint16_t* __restrict__ lut = nullptr) {
  if (stage == S_SUS || stage > 10 || stage < 0 || P->n_targets[stage] == 0) {
    next = NEVER; delay = NEVER; return;
  }
  const int j = pick_branch(P, stage, age, ub);
  next = P->targets[stage][j];
  delay = delay_steps(P, P->spec_of[stage][j], ud, lut);
}

// Host: the bucket table of delay_steps (spec-major, TAU_LUT per spec).
inline void fill_tau_lut(uint16_t* lut, const epi_params& p) {
  for (int s = 0; s < EPI_MAX_SPECS; ++s) {
    int c = 0;
    for (int k = 0; k < TAU_LUT; ++k) {
      const double edge = (double)k / TAU_LUT;
      while (s < p.n_specs && c < p.tau_len[s] && p.tau[s][c] < edge) ++c;
      lut[s * TAU_LUT + k] = (uint16_t)c;
    }
  }
}

// ---- source codes ---------------------------------------------------------
// bits 0-6: days since infection t (0 = not a valid source), bit 7:
// asymptomatic-like, bits 8-13: random-slot count, bit 15: dead.
constexpr uint16_t CODE_T_MASK = 0x7F;
constexpr uint16_t CODE_ASYM = 0x80;
constexpr uint16_t CODE_DEAD = 0x8000;
__device__ __forceinline__ int code_count(uint16_t c) { return (c >> 8) & 0x3F; }
__device__ __forceinline__ bool code_dead(uint16_t c) { return (c & CODE_DEAD) != 0; }

// validity of a source at `step` (engine.py:89-94)
__device__ __forceinline__ uint16_t source_code(const epi_params* __restrict__ P, int stage,
                                                int32_t infected_at, int32_t q_until, int step) {
  if (!infectious_stage(stage) || q_until > step) return 0;
  const int64_t t = (int64_t)step - (int64_t)infected_at;
  if (t < 1 || t > P->t_max) return 0;
  return (uint16_t)t | (asym_like_stage(stage) ? CODE_ASYM : 0);
}

// ---- programmatic dependent launch ------------------------------------------
// The per-day kernels are launched with programmatic stream serialization so
// the next kernel's launch and shared-memory prologue overlap the current
// kernel's tail.  Rule: a kernel's prologue reads only data finished at least
// two launches earlier and writes nothing global; pdl_wait() (all prior grids
// complete and visible) precedes every dependent read and every global write;
// pdl_trigger() is issued only after pdl_wait(), which keeps the chain
// transitive.  Without a programmatic predecessor both are no-ops.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" :::); }

// ---- warp helpers -----------------------------------------------------------
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

template <int N>
struct BlockCounters {
  unsigned long long v[N];
};

}  // namespace epi
