// Step kernels: message pass (gather), fused transmission/progression update,
// intervention phases, per-step record.  Host wrappers live in epi_b200.cu.
#pragma once

#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "epi_common.cuh"
#include "epi_confignet.cuh"

namespace epi {

constexpr int NUM_BUCKETS = 54;      // 3 groups x 9 age bands x 2 dose ranks
constexpr uint8_t FL_SYMPTOMATIC = 1, FL_NOTIFIER = 2, FL_NOTIFIED = 4;
constexpr uint8_t NO_BUCKET = 0xFF;

// ---------------------------------------------------------------------------
// Per-block accumulation of the EPI_REC_* record.  Every warp owns a row of
// 32-bit counters that only its own lanes update, with plain shared-memory
// adds (no atomics, no contention between warps); rec_flush sums the rows
// and adds the block total to the global record with integer atomics, so
// the totals are deterministic.
constexpr int REC_MAX_WARPS = 32;
struct RecAcc {
  unsigned v[REC_MAX_WARPS][EPI_REC_LEN];
};

__device__ __forceinline__ void rec_init(RecAcc& s) {
  for (int i = threadIdx.x; i < REC_MAX_WARPS * EPI_REC_LEN; i += blockDim.x) (&s.v[0][0])[i] = 0u;
}
// warp-aggregated add of `x` (all 32 lanes must call)
__device__ __forceinline__ void rec_add(RecAcc& s, int slot, unsigned x) {
  const unsigned t = __reduce_add_sync(0xFFFFFFFFu, x);
  if (lane_id() == 0) s.v[threadIdx.x >> 5][slot] += t;
}
__device__ __forceinline__ void rec_or(RecAcc& s, int slot, unsigned x) {
  const unsigned t = __reduce_or_sync(0xFFFFFFFFu, x);
  if (lane_id() == 0) s.v[threadIdx.x >> 5][slot] |= t;
}
// all threads of the block must call
__device__ __forceinline__ void rec_flush(const RecAcc& s, long long* rec, int step = -1) {
  __syncthreads();
  if (step >= 0 && blockIdx.x == 0 && threadIdx.x == 0) rec[EPI_REC_STEP] = step;
  const int nw = (blockDim.x + 31) >> 5;
  for (int i = threadIdx.x; i < EPI_REC_LEN; i += blockDim.x) {
    unsigned long long t = 0;
    if (i == EPI_REC_FLAGS) {
      for (int w = 0; w < nw; ++w) t |= s.v[w][i];
      if (t) atomicOr((unsigned long long*)&rec[i], t);
    } else {
      for (int w = 0; w < nw; ++w) t += s.v[w][i];
      if (t) atomicAdd((unsigned long long*)&rec[i], t);
    }
  }
}

// Stage histogram + derived time-series columns (runner.py:101-116) and the
// structural invariants of state.py:90-102, for one agent per lane.  The
// histogram is one match per warp: the lowest lane of each stage group adds
// the group's size (distinct groups, distinct counters).
__device__ __forceinline__ void rec_agent(RecAcc& s, bool valid, int stage, int32_t infected_at) {
  const bool in_range = stage >= 0 && stage <= 10;
  const unsigned grp = __match_any_sync(0xFFFFFFFFu, valid && in_range ? stage : -1);
  if (valid && in_range && lane_id() == __ffs(grp) - 1)
    s.v[threadIdx.x >> 5][EPI_REC_STAGE0 + stage] += __popc(grp);
  rec_add(s, EPI_REC_CUM_INF, valid && infected_at != NEVER);
  rec_add(s, EPI_REC_CUM_DEATHS, valid && stage == S_DEAD);
  rec_add(s, EPI_REC_IN_CARE, valid && (stage == S_HOSP || stage == S_ICU));
  unsigned fl = 0;
  if (valid && !in_range) fl |= EPI_FLAG_STAGE_RANGE;
  if (valid && stage != S_SUS && stage != S_VAC && infected_at == NEVER) fl |= EPI_FLAG_NO_TIMESTAMP;
  rec_or(s, EPI_REC_FLAGS, fl);
  __syncwarp();
}

// ---------------------------------------------------------------------------
// Debug export of the hazard every step kernel feeds its Bernoulli
// (epi_set_lambda_probe): out[(t - first) * n + agent] = the fp32 lambda of
// day t, 0 for non-targets, for days first <= t < first + days.  It exists so
// the timed kernels are checked against the oracle's gather_exposure
// (engine.py:77-117) on the very values they consume.
struct LamProbe {
  float* out;
  int64_t n;
  int first, days;
};
__device__ __forceinline__ void probe_lambda(const LamProbe& p, int t, int64_t b, double lam) {
  if (p.out != nullptr && (unsigned)(t - p.first) < (unsigned)p.days)
    p.out[(size_t)(t - p.first) * (size_t)p.n + (size_t)b] = (float)lam;
}

// Kernel arguments shared by the step kernels.
struct StepArgs {
  const epi_params* __restrict__ P;
  epi_state st;
  int step;
  StepKeys K;
  const Injected* inj;        // device pointer or null
  long long* rec;             // EPI_REC_LEN
  uint8_t* flags;             // per agent scratch
  int64_t lo, hi;             // owned agent rows [lo, hi) (partitioned runs)
  int indep;                  // independent-edges infection (oracle.py:185-192)
  const uint16_t* tau_lut;    // bucket table of delay_steps (or null: binary search)
  LamProbe probe;             // debug export of the per-agent hazard (epi_set_lambda_probe)
};

// Shared tables for the fp32 message: factor[t | asym<<7] = rate*A*w[t],
// sfac[age] = S[age] / Ibar, bfac[kind] = B[kind].
struct MsgTables {
  float factor[256];
  float sfac[16];
  float bfac[4];
};
// Weight of a pre-joined message (k_msg_pass): rate*A*w[t]*B[kind] (computed
// in fp64, stored fp32) at [idx << 2 | kind], idx = source code & 0xFF; the
// message itself is the byte offset of its weight, (idx << 2 | kind) << 2.
// Message 0 (a non-infectious household source) weighs 0: it pads rows.
struct MsgComb {
  float w[4 * 256];
};
inline void fill_msg_tables(MsgTables& T, const epi_params& P, double rate) {
  for (int i = 0; i < 256; ++i) {
    const int t = i & 0x7F;
    float f = 0.f;
    if (t >= 1 && t <= P.t_max)
      f = (float)(rate * ((i & 0x80) ? P.asymptomatic_factor : 1.0) * P.day_weights[t]);
    T.factor[i] = f;
  }
  for (int i = 0; i < 16; ++i)
    T.sfac[i] = i < 9 ? (float)(P.age_susceptibility[i] / P.mean_daily_interactions) : 0.f;
  for (int i = 0; i < 4; ++i) T.bfac[i] = i < 3 ? (float)P.network_scale[i] : 0.f;
}
inline void fill_msg_comb(MsgComb& C, const epi_params& P, double rate) {
  for (int i = 0; i < 256; ++i) {
    const int t = i & 0x7F;
    for (int k = 0; k < 4; ++k) {
      double w = 0.0;
      if (t >= 1 && t <= P.t_max && k < 3)
        w = ((rate * ((i & 0x80) ? P.asymptomatic_factor : 1.0)) * P.network_scale[k]) * P.day_weights[t];
      C.w[(i << 2) | k] = (float)w;
    }
  }
}
__device__ __forceinline__ void load_msg_tables(MsgTables& S, const MsgTables* __restrict__ G) {
  const uint32_t* src = (const uint32_t*)G;
  uint32_t* dst = (uint32_t*)&S;
  for (int i = threadIdx.x; i < (int)(sizeof(MsgTables) / 4); i += blockDim.x) dst[i] = src[i];
}
__device__ __forceinline__ void build_msg_tables(MsgTables& T, const epi_params* __restrict__ P,
                                                 double rate) {
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    const int t = i & 0x7F;
    float f = 0.f;
    if (t >= 1 && t <= P->t_max)
      f = (float)(rate * ((i & 0x80) ? P->asymptomatic_factor : 1.0) * P->day_weights[t]);
    T.factor[i] = f;
  }
  for (int i = threadIdx.x; i < 9; i += blockDim.x)
    T.sfac[i] = (float)(P->age_susceptibility[i] / P->mean_daily_interactions);
  for (int i = threadIdx.x; i < 3; i += blockDim.x) T.bfac[i] = (float)P->network_scale[i];
}

// fp64 term with the reference's pinned factor order (engine.py:100-107,
// transmission.py:131-134): ((((rate*S[age_d])*A)*B[k])/Ibar)*w[t].
__device__ __forceinline__ double term_f64(const epi_params* __restrict__ P, double rate_s,
                                           uint16_t code, int kind) {
  double x = __dmul_rn(rate_s, (code & CODE_ASYM) ? P->asymptomatic_factor : 1.0);
  x = __dmul_rn(x, P->network_scale[kind]);
  x = __ddiv_rn(x, P->mean_daily_interactions);
  return __dmul_rn(x, P->day_weights[code & CODE_T_MASK]);
}

__device__ __forceinline__ bool is_target(const epi_params* __restrict__ P, const epi_state& st,
                                          int64_t a) {
  return st.stage[a] == S_SUS && !(P->sterilizing && st.immune[a]);
}

// ---------------------------------------------------------------------------
// Phases 1-2 for one agent (engine.py:153-200).  Returns event bits:
// 1 new infection, 2 death, 4 hospitalisation, 8 newly symptomatic.
// The state fields of one agent that phases 1-2 and the next code read,
// loaded once (the fused day kernel issues these loads before its gather).
struct AgentHot {
  int stage, immune, age, next_stage;
  int32_t nta, infected_at, q_until;
};
// The same fields read once per day as a stream (evict-first in L2: at 10 M
// agents the random gathers' tables -- codes, colleague positions and codes --
// should keep L2, not the agents' own columns).
__device__ __forceinline__ AgentHot load_hot_stream(const epi_state& st, int64_t a) {
  AgentHot h;
  h.stage = __ldcs(st.stage + a);
  h.immune = __ldcs(st.immune + a);
  h.age = __ldcs(st.age_band + a);
  h.next_stage = __ldcs(st.next_stage + a);
  h.nta = __ldcs(st.next_transition_at + a);
  h.infected_at = __ldcs(st.infected_at + a);
  h.q_until = __ldcs(st.quarantine_until + a);
  return h;
}
__device__ __forceinline__ AgentHot load_hot(const epi_state& st, int64_t a) {
  AgentHot h;
  h.stage = st.stage[a];
  h.immune = st.immune[a];
  h.age = st.age_band[a];
  h.next_stage = st.next_stage[a];
  h.nta = st.next_transition_at[a];
  h.infected_at = st.infected_at[a];
  h.q_until = st.quarantine_until[a];
  return h;
}

// Phases 1-2 on preloaded state (updated in place, and written through).
// `forced` >= 0: the infection decision was already drawn per edge
// (independent-edges mode) and replaces the aggregate draw.
// The core takes the step's key prefixes explicitly (kernel parameter or, in
// the persistent run, shared memory).
__device__ __forceinline__ unsigned transmit_progress_core(const epi_params* __restrict__ P, const epi_state& st,
                                                           const StepKeys& K, const Injected* inj, int step,
                                                           const uint16_t* __restrict__ tau_lut, int64_t a,
                                                           double lam, int forced, AgentHot& h) {
  unsigned ev = 0;
  if (h.stage == S_SUS && !(P->sterilizing && h.immune)) {
    // lam == 0 gives p == 0 and u < p never holds: skip the draw
    bool infect = false;
    if (forced >= 0) {
      infect = forced != 0;
    } else {
      // p = 0 never infects: no exp, no draw for the (many) zero hazards
      if (lam > 0.0) infect = draw(K, inj, P_INFECTION, a) < 1.0 - exp(-lam);
    }
    if (infect) {
      int entry = P->targets[S_SUS][pick_branch(P, S_SUS, h.age, draw(K, inj, P_ENTRY, a))];
      if (!P->sterilizing && h.immune) entry = S_ASYM;
      int nxt, delay;
      schedule(P, entry, h.age, draw(K, inj, P_BRANCH, a), draw(K, inj, P_DELAY, a), nxt, delay,
               tau_lut);
      h.stage = entry;
      h.infected_at = step;
      h.next_stage = nxt;
      h.nta = step + delay;
      st.stage[a] = (int8_t)entry;
      st.infected_at[a] = step;
      st.next_stage[a] = (int8_t)nxt;
      st.next_transition_at[a] = h.nta;
      ev |= 1u;
    }
  }
  if (h.nta == step) {
    const int dest = h.next_stage;
    h.stage = dest;
    st.stage[a] = (int8_t)dest;
    if (dest == S_DEAD) ev |= 2u;
    if (dest == S_HOSP) ev |= 4u;
    if (dest == S_MILD || dest == S_SEV) ev |= 8u;
    if (dest == S_REC || dest == S_DEAD) {
      h.next_stage = NEVER8;
      h.nta = NEVER;
    } else {
      int nxt, delay;
      schedule(P, dest, h.age, draw(K, inj, P_BRANCH, a), draw(K, inj, P_DELAY, a), nxt, delay,
               tau_lut);
      h.next_stage = nxt;
      h.nta = step + delay;
    }
    st.next_stage[a] = (int8_t)h.next_stage;
    st.next_transition_at[a] = h.nta;
  }
  return ev;
}

// transmit_progress_core split in two for the persistent runs: the day's
// decisions now (infection + entry stage, due transition + destination:
// everything the day's record and tomorrow's code need), the scheduling of
// the next transition (branch + delay draws, threshold tables: the longest
// dependent chain) later, between the day's barrier arrive and wait — it
// only feeds tomorrow's transition check.  Same draws, same results.
// `pend` = the stage to schedule from, -1 if none.
__device__ __forceinline__ unsigned transmit_progress_now(const epi_params* __restrict__ P, const epi_state& st,
                                                          const StepKeys& K, int step, int64_t a, double lam,
                                                          AgentHot& h, int& pend) {
  unsigned ev = 0;
  pend = -1;
  bool infected = false;
  if (h.stage == S_SUS && !(P->sterilizing && h.immune)) {
    if (lam > 0.0) infected = draw(K, nullptr, P_INFECTION, a) < 1.0 - exp(-lam);
    if (infected) {
      int entry = P->targets[S_SUS][pick_branch(P, S_SUS, h.age, draw(K, nullptr, P_ENTRY, a))];
      if (!P->sterilizing && h.immune) entry = S_ASYM;
      h.stage = entry;
      h.infected_at = step;
      st.stage[a] = (int8_t)entry;
      st.infected_at[a] = step;
      pend = entry;
      ev |= 1u;
    }
  }
  // (after an infection the next transition is >= 1 day away)
  if (!infected && h.nta == step) {
    const int dest = h.next_stage;
    h.stage = dest;
    st.stage[a] = (int8_t)dest;
    if (dest == S_DEAD) ev |= 2u;
    if (dest == S_HOSP) ev |= 4u;
    if (dest == S_MILD || dest == S_SEV) ev |= 8u;
    if (dest == S_REC || dest == S_DEAD) {
      h.next_stage = NEVER8;
      h.nta = NEVER;
      st.next_stage[a] = (int8_t)h.next_stage;
      st.next_transition_at[a] = h.nta;
    } else {
      pend = dest;
    }
  }
  return ev;
}
__device__ __forceinline__ void schedule_pending(const epi_params* __restrict__ P, const epi_state& st,
                                                 const StepKeys& K, int step, const uint16_t* __restrict__ tau_lut,
                                                 int64_t a, int pend, AgentHot& h) {
  int nxt, delay;
  schedule(P, pend, h.age, draw(K, nullptr, P_BRANCH, a), draw(K, nullptr, P_DELAY, a), nxt, delay, tau_lut);
  h.next_stage = nxt;
  h.nta = step + delay;
  st.next_stage[a] = (int8_t)nxt;
  st.next_transition_at[a] = h.nta;
}

__device__ __forceinline__ unsigned transmit_progress_hot(const StepArgs& A, int64_t a, double lam, int forced,
                                                          AgentHot& h) {
  return transmit_progress_core(A.P, A.st, A.K, A.inj, A.step, A.tau_lut, a, lam, forced, h);
}

__device__ __forceinline__ unsigned transmit_progress(const StepArgs& A, int64_t a, double lam,
                                                      int forced = -1) {
  AgentHot h = load_hot(A.st, a);
  return transmit_progress_hot(A, a, lam, forced, h);
}

__device__ __forceinline__ void rec_events(RecAcc& s, unsigned ev) {
  rec_add(s, EPI_REC_NEW_INF, ev & 1u);
  rec_add(s, EPI_REC_DEATHS, (ev >> 1) & 1u);
  rec_add(s, EPI_REC_HOSP, (ev >> 2) & 1u);
}

// Next-step source code from preloaded (post-update) state.
__device__ __forceinline__ uint16_t next_code_hot(const epi_params* __restrict__ P, const AgentHot& h, int64_t a,
                                                  int next_step, const epi_net* net, uint64_t rcount_prefix) {
  uint16_t c = source_code(P, h.stage, h.infected_at, h.q_until, next_step);
  if (h.stage == S_DEAD) {
    c |= CODE_DEAD;
  } else if (net != nullptr) {
    c |= (uint16_t)(random_count(*net, rcount_prefix, a) << 8);
  }
  return c;
}

// Next-step source code of agent a (after every phase of `step`).
__device__ __forceinline__ uint16_t next_code(const epi_params* __restrict__ P, const epi_state& st,
                                              int64_t a, int next_step, const epi_net* net,
                                              uint64_t rcount_prefix) {
  const int stage = st.stage[a];
  uint16_t c = source_code(P, stage, st.infected_at[a], st.quarantine_until[a], next_step);
  if (stage == S_DEAD) {
    c |= CODE_DEAD;
  } else if (net != nullptr) {
    c |= (uint16_t)(random_count(*net, rcount_prefix, a) << 8);
  }
  return c;
}

// ---------------------------------------------------------------------------
// Codes from state (graph-in gather, and step 0 of a config simulation).
// (With `died_at`: every agent's death step restarts — -1 if already dead.)
__global__ void k_codes(const epi_params* __restrict__ P, epi_state st, int step, const epi_net* net,
                        uint64_t rcount_prefix, uint16_t* __restrict__ codes, int64_t lo, int64_t hi,
                        int32_t* __restrict__ died_at = nullptr, int64_t n_all = 0) {
  pdl_wait();
  pdl_trigger();
  const int64_t n = hi;
  for (int64_t a = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < n;
       a += (int64_t)gridDim.x * blockDim.x)
    codes[a] = next_code(P, st, a, step, net, rcount_prefix);
  if (died_at)
    for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < n_all; a += (int64_t)gridDim.x * blockDim.x)
      died_at[a] = st.stage[a] == S_DEAD ? -1 : INT32_MAX;
}

// ---------------------------------------------------------------------------
// Graph-in: COO -> sort keys (dst << 32 | src << 2 | kind) + validation.

// Row bounds of the sorted keys; entries = low 32 bits (src << 2 | kind).
// Canonical CSR by counting sort (graph load): edges counted per
// destination, rows placed by an exclusive scan, entries scattered, then each
// row sorted by (src, kind) — the (dst, src, kind) order of np.lexsort
// (engine.py:98) without a full radix sort of the edge keys.  Equal entries
// are identical values, so the result does not depend on the scatter order.
__global__ void k_coo_count(const int32_t* __restrict__ src, const int32_t* __restrict__ dst,
                            const int8_t* __restrict__ kind, int64_t E, int64_t n,
                            int32_t* __restrict__ row_len, long long* flag_word,
                            const unsigned long long* __restrict__ count) {
  unsigned fl = 0;
  const int64_t live = count ? (int64_t)(*count < (unsigned long long)E ? *count : (unsigned long long)E) : E;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < live;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t s = src[i], d = dst[i];
    const int k = kind[i];
    const bool bad = s < 0 || d < 0 || s >= n || d >= n;
    if (bad) fl |= EPI_FLAG_INDEX;
    if (s == d) fl |= EPI_FLAG_SELFLOOP;
    if (k < 0 || k > 2) fl |= EPI_FLAG_KIND;
    if (!bad) atomicAdd(&row_len[d], 1);
  }
  if (fl) atomicOr((unsigned long long*)flag_word, (unsigned long long)fl);
}
__global__ void k_coo_scatter(const int32_t* __restrict__ src, const int32_t* __restrict__ dst,
                              const int8_t* __restrict__ kind, int64_t E, int64_t n,
                              const int64_t* __restrict__ row_begin, int32_t* __restrict__ fill,
                              uint32_t* __restrict__ entries, const unsigned long long* __restrict__ count,
                              unsigned* __restrict__ long_count) {
  pdl_wait();
  pdl_trigger();
  if (blockIdx.x == 0 && threadIdx.x == 0) *long_count = 0u;   // k_rows_sort lists this load's long rows
  const int64_t live = count ? (int64_t)(*count < (unsigned long long)E ? *count : (unsigned long long)E) : E;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // 4 edges per thread in flight: loads, then cursors, then stores
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < live; i0 += 4 * stride) {
    int32_t s[4], d[4];
    int8_t k[4];
    bool ok[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t i = i0 + q * stride;
      const bool in = i < live;
      s[q] = in ? src[i] : -1;
      d[q] = in ? dst[i] : -1;
      k[q] = in ? kind[i] : 0;
    }
    int64_t pos[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      ok[q] = !(s[q] < 0 || d[q] < 0 || s[q] >= n || d[q] >= n);
      pos[q] = ok[q] ? row_begin[d[q]] + atomicAdd(&fill[d[q]], 1) : 0;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (ok[q]) entries[pos[q]] = ((uint32_t)s[q] << 2) | (uint32_t)(k[q] & 3);
  }
}
// Canonical row order: ascending (src << 2 | kind).  One thread per row; a
// row of <= 32 entries is sorted in registers by a bitonic network (padding
// ~0u sorts last; a real entry is at most (2^30 - 1) << 2 | 2), longer rows
// (none on the reference networks at its defaults) by insertion in place.
template <int W>
__device__ __forceinline__ void bitonic_regs(uint32_t (&v)[W]) {
#pragma unroll
  for (int k = 2; k <= W; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
#pragma unroll
      for (int i = 0; i < W; ++i) {
        const int l = i ^ j;
        if (l > i) {
          const uint32_t a = v[i], b = v[l];
          const bool up = (i & k) == 0;
          const uint32_t lo = a < b ? a : b, hi = a < b ? b : a;
          v[i] = up ? lo : hi;
          v[l] = up ? hi : lo;
        }
      }
    }
  }
}
template <int W>
__device__ __forceinline__ void sort_row_regs(uint32_t* row, int len) {
  uint32_t v[W];
#pragma unroll
  for (int i = 0; i < W; ++i) v[i] = i < len ? row[i] : ~0u;
  bitonic_regs<W>(v);
#pragma unroll
  for (int i = 0; i < W; ++i)
    if (i < len) row[i] = v[i];
}
// (also re-zeroes the scatter's fill cursors, so they are zero at the next
// load).  Rows of <= 32 entries are sorted in registers by their thread;
// longer rows (hubs: a graph-in StepGraph may give one destination 1e5
// in-edges) are listed for k_rows_sort_long, one block per row.
__global__ void k_rows_sort(int64_t n, const int64_t* __restrict__ row_begin, const int32_t* __restrict__ row_len,
                            uint32_t* __restrict__ entries, int32_t* __restrict__ fill,
                            int32_t* __restrict__ long_rows, unsigned* __restrict__ long_count) {
  pdl_wait();
  pdl_trigger();
  for (int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; d < n; d += (int64_t)gridDim.x * blockDim.x) {
    fill[d] = 0;
    uint32_t* row = entries + row_begin[d];
    const int len = row_len[d];
    if (len <= 1) continue;
    if (len <= 8) {
      sort_row_regs<8>(row, len);
    } else if (len <= 16) {
      sort_row_regs<16>(row, len);
    } else if (len <= 32) {
      sort_row_regs<32>(row, len);
    } else {
      long_rows[atomicAdd(long_count, 1u)] = (int32_t)d;
    }
  }
}

// Long rows: one 1024-thread block per row.  Tiles of LONG_TILE entries are
// bitonic-sorted in shared memory, then merged pairwise (merge path: every
// thread merges a contiguous slice of the output) between the row and a
// scratch copy, log2(len / LONG_TILE) passes.  O(len log len) per row.
constexpr int LONG_TILE = 8192;
__device__ __forceinline__ int merge_path(const uint32_t* a, int la, const uint32_t* b, int lb, int diag) {
  int lo = diag - lb > 0 ? diag - lb : 0, hi = diag < la ? diag : la;
  while (lo < hi) {
    const int i = (lo + hi) >> 1;
    if (a[i] <= b[diag - 1 - i]) lo = i + 1;
    else hi = i;
  }
  return lo;
}
__device__ __forceinline__ void merge_block(const uint32_t* a, int la, const uint32_t* b, int lb, uint32_t* out) {
  const int total = la + lb;
  const int chunk = (total + (int)blockDim.x - 1) / (int)blockDim.x;
  const int d0 = threadIdx.x * chunk;
  if (d0 >= total) return;
  const int d1 = d0 + chunk < total ? d0 + chunk : total;
  int ia = merge_path(a, la, b, lb, d0), ib = d0 - ia;
  for (int k = d0; k < d1; ++k) {
    if (ia < la && (ib >= lb || a[ia] <= b[ib])) out[k] = a[ia++];
    else out[k] = b[ib++];
  }
}
__global__ void __launch_bounds__(1024) k_rows_sort_long(const int64_t* __restrict__ row_begin,
                                                         const int32_t* __restrict__ row_len,
                                                         uint32_t* __restrict__ entries, uint32_t* __restrict__ tmp,
                                                         const int32_t* __restrict__ long_rows,
                                                         const unsigned* __restrict__ long_count) {
  __shared__ uint32_t sm[LONG_TILE];
  pdl_wait();
  pdl_trigger();
  const unsigned nl = *long_count;
  for (unsigned r = blockIdx.x; r < nl; r += gridDim.x) {
    const int32_t d = long_rows[r];
    uint32_t* row = entries + row_begin[d];
    uint32_t* aux = tmp + row_begin[d];
    const int len = row_len[d];
    for (int t0 = 0; t0 < len; t0 += LONG_TILE) {
      const int tl = len - t0 < LONG_TILE ? len - t0 : LONG_TILE;
      int p2 = 64;
      while (p2 < tl) p2 <<= 1;
      for (int i = threadIdx.x; i < p2; i += blockDim.x) sm[i] = i < tl ? row[t0 + i] : ~0u;
      __syncthreads();
      for (int k = 2; k <= p2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
          for (int i = threadIdx.x; i < p2; i += blockDim.x) {
            const int l = i ^ j;
            if (l > i) {
              const uint32_t x = sm[i], y = sm[l];
              if ((x > y) == ((i & k) == 0)) { sm[i] = y; sm[l] = x; }
            }
          }
          __syncthreads();
        }
      }
      for (int i = threadIdx.x; i < tl; i += blockDim.x) row[t0 + i] = sm[i];
      __syncthreads();
    }
    uint32_t* a = row;
    uint32_t* b = aux;
    for (int w = LONG_TILE; w < len; w <<= 1) {
      for (int m0 = 0; m0 < len; m0 += 2 * w) {
        const int la = len - m0 < w ? len - m0 : w;
        const int rest = len - m0 - la;
        const int lb = rest < w ? rest : w;
        merge_block(a + m0, la, a + m0 + la, lb, b + m0);
      }
      __syncthreads();
      uint32_t* t = a; a = b; b = t;
    }
    if (a != row)
      for (int i = threadIdx.x; i < len; i += blockDim.x) row[i] = a[i];
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Gather / fused gather + update over a CSR given either by explicit
// row_begin (graph-in) or implicitly by row * cap (padded config CSR).
// Row capacity of the tile-packed message blocks (rows padded to 8).
__host__ __device__ __forceinline__ int msg_cap(int cap) { return (cap + 7) & ~7; }

struct CsrView {
  const uint32_t* __restrict__ entries;
  const int32_t* __restrict__ row_len;
  const int64_t* __restrict__ row_begin;   // null: padded rows of `cap`
  int cap;
  // Optional pre-joined messages, tile-packed: msg = (source code & 0xFF) << 4
  // | kind << 2 (a byte offset into the MsgComb table), written by the
  // generator, so the fp32 message pass (k_msg_pass, epi_msgpass.cuh) streams
  // 2 B per edge with no gathers.  Tile k (32 rows from lo) owns the block
  // msgs[k*32*msg_cap(cap) ...]; its rows are packed back to back, each
  // padded to whole 4-message half-groups, and tile_off[k*33 + r] = row r's
  // first half-group | pad << 12 (tile_off[k*33 + 32] = half-groups in the tile).
  const uint16_t* __restrict__ msgs;
  const uint16_t* __restrict__ tile_off;
  __device__ __forceinline__ int64_t begin(int64_t r) const {
    return row_begin ? row_begin[r] : r * (int64_t)cap;
  }
};

// MODE 0: write hazard (gather_exposure); MODE 1: fused update (+ record if
// `final_pass`, + next codes).
template <bool F64, int MODE>
__global__ void __launch_bounds__(256) k_pass(StepArgs A, CsrView g, const uint16_t* __restrict__ codes,
                                              void* __restrict__ lam_out, double rate,
                                              int final_pass, uint16_t* __restrict__ codes_next,
                                              const epi_net* net, uint64_t rcount_next,
                                              const MsgTables* __restrict__ mt) {
  __shared__ MsgTables T;
  __shared__ float lam_tile[8][32];
  __shared__ RecAcc racc;
  if (!F64) {
    if (mt) load_msg_tables(T, mt);
    else build_msg_tables(T, A.P, rate);
  }
  rec_init(racc);
  __syncthreads();
  pdl_wait();
  pdl_trigger();
  const epi_params* __restrict__ P = A.P;
  const int64_t n = A.hi;
  const int warp = threadIdx.x >> 5, lane = lane_id();
  const int64_t n_tiles = (n - A.lo + 31) / 32;
  const int64_t warps_total = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t tile = blockIdx.x * (int64_t)(blockDim.x >> 5) + warp; tile < n_tiles;
       tile += warps_total) {
    const int64_t base = A.lo + tile * 32;
    const int64_t a = base + lane;
    const bool valid = a < n;
    double lam = 0.0;
    unsigned edges = 0;
    int forced = -1;
    if (F64) {
      // one lane per row, sequential in canonical order
      if (valid) {
        const int len = g.row_len[a];
        edges = (unsigned)len;
        if (is_target(P, A.st, a)) {
          const double rate_s = __dmul_rn(rate, P->age_susceptibility[A.st.age_band[a]]);
          const uint32_t* e = g.entries + g.begin(a);
          if (MODE == 1 && A.indep) {
            // independent edges: contribution j (nonzero, canonical order) infects
            // with u(INFECTION_EDGE, a, k=j) < 1 - exp(-h_j)
            int j = 0;
            forced = 0;
            for (int i = 0; i < len; ++i) {
              const uint32_t x = e[i];
              const uint16_t c = codes[x >> 2];
              if (!(c & CODE_T_MASK)) continue;
              const double h = term_f64(P, rate_s, c, (int)(x & 3));
              if (h == 0.0) continue;
              if (keyed_u(A.K.p[P_INFECTION_EDGE], (uint64_t)a, (uint64_t)j) < 1.0 - exp(-h)) forced = 1;
              ++j;
            }
          } else {
            // entries and their code gathers 4 at a time (memory-level
            // parallelism); the sum itself stays sequential in canonical order
            double h = 0.0;
            for (int i0 = 0; i0 < len; i0 += 4) {
              uint32_t x[4];
              uint16_t c[4];
#pragma unroll
              for (int q = 0; q < 4; ++q) x[q] = i0 + q < len ? __ldg(e + i0 + q) : 0u;
#pragma unroll
              for (int q = 0; q < 4; ++q) c[q] = i0 + q < len ? codes[x[q] >> 2] : (uint16_t)0;
#pragma unroll
              for (int q = 0; q < 4; ++q)
                if (c[q] & CODE_T_MASK) h = __dadd_rn(h, term_f64(P, rate_s, c[q], (int)(x[q] & 3)));
            }
            lam = h;
          }
        }
      }
    } else {
      // 8 lanes per row, 4 rows per pass, tree sum in fp32
      const int grp = lane >> 3, gl = lane & 7;
#pragma unroll 1
      for (int r4 = 0; r4 < 8; ++r4) {
        const int64_t row = base + r4 * 4 + grp;
        float acc = 0.f;
        if (row < n) {
          const int len = g.row_len[row];
          const uint32_t* e = g.entries + g.begin(row);
          // 8 lanes x 4 entries in flight per pass, then their 4 code gathers
          for (int i0 = gl; i0 < len; i0 += 32) {
            uint32_t x[4];
            uint16_t c[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) x[q] = (i0 + 8 * q < len) ? __ldg(e + i0 + 8 * q) : 0xFFFFFFFFu;
#pragma unroll
            for (int q = 0; q < 4; ++q) c[q] = (x[q] != 0xFFFFFFFFu) ? codes[x[q] >> 2] : (uint16_t)0;
#pragma unroll
            for (int q = 0; q < 4; ++q) acc += T.factor[c[q] & 0xFF] * T.bfac[x[q] & 3];
          }
        }
        acc += __shfl_xor_sync(0xFFFFFFFFu, acc, 4);
        acc += __shfl_xor_sync(0xFFFFFFFFu, acc, 2);
        acc += __shfl_xor_sync(0xFFFFFFFFu, acc, 1);
        if (gl == 0) lam_tile[warp][r4 * 4 + grp] = acc;
      }
      __syncwarp();
      if (valid) {
        edges = (unsigned)g.row_len[a];
        lam = is_target(P, A.st, a)
                  ? (double)(lam_tile[warp][lane] * T.sfac[A.st.age_band[a]])
                  : 0.0;
      }
      __syncwarp();
    }
    if (MODE == 0) {
      if (valid) {
        if (F64) ((double*)lam_out)[a] = lam;
        else ((float*)lam_out)[a] = (float)lam;
      }
      rec_add(racc, EPI_REC_EDGES, edges);
      continue;
    }
    // MODE 1: fused update for this lane's agent
    unsigned ev = 0;
    if (valid) ev = transmit_progress(A, a, lam, forced);
    if (valid && (ev & 8u) && A.flags) A.flags[a] = FL_SYMPTOMATIC;
    rec_events(racc, ev);
    rec_add(racc, EPI_REC_EDGES, edges);
    if (final_pass) {
      int stage = valid ? A.st.stage[a] : 0;
      rec_agent(racc, valid, stage, valid ? A.st.infected_at[a] : 0);
      if (valid && codes_next) codes_next[a] = next_code(P, A.st, a, A.step + 1, net, rcount_next);
    }
  }
  __syncthreads();
  rec_flush(racc, A.rec, A.step);
}

// Update from an externally supplied fp64 hazard (injected-draw parity).
__global__ void k_update_from_hazard(StepArgs A, const double* __restrict__ hazard, int final_pass) {
  __shared__ RecAcc racc;
  rec_init(racc);
  __syncthreads();
  const int64_t n = A.hi;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = A.lo + blockIdx.x * (int64_t)blockDim.x; base < n; base += stride) {
    const int64_t a = base + threadIdx.x;
    const bool valid = a < n;
    unsigned ev = 0;
    if (valid) {
      const double lam = is_target(A.P, A.st, a) ? hazard[a] : 0.0;
      if (lam < 0) atomicOr((unsigned long long*)&A.rec[EPI_REC_FLAGS], EPI_FLAG_NEG_HAZARD);
      ev = transmit_progress(A, a, lam);
      if ((ev & 8u) && A.flags) A.flags[a] = FL_SYMPTOMATIC;
    }
    rec_events(racc, ev);
    if (final_pass) rec_agent(racc, valid, valid ? A.st.stage[a] : 0, valid ? A.st.infected_at[a] : 0);
  }
  __syncthreads();
  rec_flush(racc, A.rec, A.step);
}

// Day-0 keys (every later day's keys are written by the previous day's
// k_day_tables).
__global__ void k_day_keys(NetTables* __restrict__ NT, uint64_t rperm, long long* rec) {
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x < EPI_MAX_SLOTS) NT->rk[threadIdx.x] = random_slot_keys(rperm, threadIdx.x);
  if (rec && threadIdx.x < EPI_REC_LEN) rec[threadIdx.x] = 0;   // the day's record
}

__device__ __forceinline__ void clear_rin_row(const WorkTables* wt, int64_t b) {
  if (wt != nullptr && wt->rin != nullptr) {
    uint4* row = (uint4*)(wt->rin + (size_t)b * RT_SLOTS);
    row[0] = make_uint4(0, 0, 0, 0);
    row[1] = make_uint4(0, 0, 0, 0);
  }
}

// ---------------------------------------------------------------------------
// Config CSR generation (mode 0): one lane per destination row; each row is
// staged in shared memory (odd stride: conflict-free), optionally sorted into
// canonical (src, kind) order, and the warp's 32 rows are written out
// coalesced: id rows one warp-wide store per row, message tiles as 16-byte
// groups (one 16-byte group = two 4-message half-groups per lane and store).  With PUSH (message-only
// runs over the whole population) the random in-edges come from the day's
// push tables (rin/rout, built by k_day_tables) instead of the random-slot
// bijections, and the rin rows consumed are cleared.
template <bool SORT, bool BATCH, bool PUSH = false>
__global__ void __launch_bounds__(128, (BATCH && !PUSH) ? 5 : 6) k_net_realize(epi_net net, NetKeys nk, const uint16_t* __restrict__ codes,
                                                     uint32_t* __restrict__ entries,
                                                     uint16_t* __restrict__ msgs,
                                                     uint16_t* __restrict__ tile_off,
                                                     int32_t* __restrict__ row_len, long long* rec,
                                                     const WorkTables* wt, int64_t lo, int64_t hi,
                                                     const NetTables* __restrict__ NTp) {
  extern __shared__ uint32_t stage_buf[];
  __shared__ NetTables NT;
  __shared__ RecAcc racc;
  __shared__ int goff_s[4][33], len_s[4][32];   // message tiles: group offsets, row lengths
  load_net_tables(NT, NTp);
  rec_init(racc);
  __syncthreads();
  pdl_wait();
  pdl_trigger();
  const int cap = net.row_cap;
  const int stride_w = cap | 1;
  const int warp = threadIdx.x >> 5, lane = lane_id();
  uint32_t* mine = stage_buf + (size_t)(warp * 32 + lane) * stride_w;
  uint32_t* wbuf = stage_buf + (size_t)warp * 32 * stride_w;
  const int64_t n = hi;
  const int64_t n_tiles = (n - lo + 31) / 32;
  const int64_t warps_total = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t tile = blockIdx.x * (int64_t)(blockDim.x >> 5) + warp; tile < n_tiles;
       tile += warps_total) {
    const int64_t base = lo + tile * 32;
    const int64_t b = base + lane;
    int cnt = 0;
    if (b < n) {
      const uint16_t cb = codes[b];
      if (!code_dead(cb)) {
        // the staging row holds either ids (src<<2|kind) or messages
        // ((code & 0xFF) << 4 | kind << 2: the byte offset of the weight in
        // MsgComb) when only messages are requested; one enumeration loop per
        // form, so the per-edge store carries no test
        auto run = [&](auto&& put) {
          if (PUSH)
            for_each_in_code(net, nk, NT.rk, NT.wrad, NT.dn, wt, codes, b, cb,
                             [&](int kind, uint16_t cc) { put(0, kind, cc); });
          else if (BATCH) for_each_in_edge_batched<16, 8>(net, nk, NT.rk, NT.wrad, wt, codes, b, cb, put);
          else for_each_in_edge(net, nk, NT.rk, NT.wrad, codes, b, cb, 0, 1, put);
        };
        if (entries)
          run([&](int64_t c, int kind, uint16_t) { mine[cnt++] = ((uint32_t)c << 2) | (uint32_t)kind; });
        else
          run([&](int64_t, int kind, uint16_t cc) {
            mine[cnt++] = ((uint32_t)(cc & 0xFF) << 4) | ((uint32_t)kind << 2);
          });
      }
      if (PUSH || BATCH) clear_rin_row(wt, b);    // consumed push rows (if any) start empty
      if (SORT) {
        for (int i = 1; i < cnt; ++i) {
          const uint32_t x = mine[i];
          int j = i - 1;
          while (j >= 0 && mine[j] > x) { mine[j + 1] = mine[j]; --j; }
          mine[j + 1] = x;
        }
      }
      if (entries) row_len[b] = cnt;
    }
    rec_add(racc, EPI_REC_EDGES, (unsigned)cnt);
    __syncwarp();
    const int rows = (n - base) < 32 ? (int)(n - base) : 32;
    if (entries) {
      for (int r = 0; r < rows; ++r) {
        const int len = __shfl_sync(0xFFFFFFFFu, cnt, r);
        const uint32_t* srcrow = wbuf + r * stride_w;
        uint32_t* dst = entries + (base + r) * (int64_t)cap;
        for (int i = lane; i < len; i += 32) dst[i] = srcrow[i];
      }
    } else {
      // tile-packed messages: rows back to back, each padded with weight-0
      // messages to whole 4-message half-groups (8 B; a 16-byte group holds
      // two, possibly of two rows); per row its first half-group and its pad
      // count (toff = half | pad << 12), toff[32] = the tile's half-groups
      const int nh = (cnt + 3) >> 2;
      int incl = nh;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += v;
      }
      const int excl = incl - nh;
      uint16_t* toff = tile_off + tile * 33;
      toff[lane] = (uint16_t)(excl | ((nh * 4 - cnt) << 12));
      if (lane == 31) toff[32] = (uint16_t)incl;
      goff_s[warp][lane] = excl;
      len_s[warp][lane] = cnt;
      if (lane == 31) goff_s[warp][32] = incl;
      __syncwarp();
      // one 16-byte group (two half-groups) per lane: the row of a half is the
      // last row starting at or before it (rows without messages share their
      // successor's start)
      uint4* blk = (uint4*)(msgs + tile * (int64_t)(32 * msg_cap(cap)));
      const int halves = __shfl_sync(0xFFFFFFFFu, incl, 31);
      for (int gi = lane; gi < (halves + 1) >> 1; gi += 32) {
        uint32_t w[4];
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int h = 2 * gi + hh;
          w[2 * hh] = w[2 * hh + 1] = 0u;
          if (h < halves) {
            int r = 0;
#pragma unroll
            for (int st = 16; st >= 1; st >>= 1)
              if (goff_s[warp][r + st] <= h) r += st;
            const int k = (h - goff_s[warp][r]) << 2;
            const int len = len_s[warp][r];
            const uint32_t* src = wbuf + r * stride_w + k;
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const uint32_t m0 = k + 2 * q < len ? src[2 * q] : 0u;
              const uint32_t m1 = k + 2 * q + 1 < len ? src[2 * q + 1] : 0u;
              w[2 * hh + q] = (m0 & 0xFFFFu) | (m1 << 16);
            }
          }
        }
        blk[gi] = make_uint4(w[0], w[1], w[2], w[3]);
      }
    }
    __syncwarp();
  }
  __syncthreads();
  if (rec) rec_flush(racc, rec);
}

// Fused generate + gather + update (mode 1): the in-edges are enumerated and
// their source codes consumed on the fly, so no CSR ever reaches memory.  One
// lane per agent; with the day's push tables the random and workplace codes
// come from contiguous rows (for_each_in_code).
// Tomorrow's push tables built in the epilogue of today's fused kernel
// ("merged" mode: one kernel per simulated day).  Everything written here is
// tomorrow's buffers; each agent scatters only its own next-day code.
struct NextTables {
  const WorkTables* wt;          // parity (t+1) buffers (device struct)
  const NetTables* keys;         // day t+1 random-slot keys (read after pdl_wait)
  NetTables* keys_out;           // day t+2 keys, written by block 0
  uint64_t rperm_t2;             // NET_RANDOM_PERM prefix of day t+2
  NetKeys nk;                    // prefixes of day t+1
};

// Phase 3 + 4a for agent a (engine.py:202-242): test sampling, then
// delivery.  `fl` is the agent's flags byte (in/out); returns 1 if sampled.
__device__ __forceinline__ unsigned test_agent(const StepArgs& A, int64_t a, int stage, uint8_t& fl,
                                               int32_t* __restrict__ notif, int* n_notif) {
  const epi_params* __restrict__ P = A.P;
  const epi_state& st = A.st;
  const int step = A.step;
  unsigned tested = 0;
  bool cand = (fl & FL_SYMPTOMATIC) != 0;
  if (st.den_test_due_at[a] == step) {
    st.den_test_due_at[a] = NEVER;
    cand = true;
  }
  if (cand && st.test_result_at[a] == NEVER && stage != S_DEAD) {
    const double up = draw(A.K, A.inj, P_TEST_POS, a);
    const bool pos = active_stage(stage) ? (up < P->detection_prob) : (up < P->false_positive_prob);
    const int span = P->turnaround_max - P->turnaround_min + 1;
    const int turn = P->turnaround_min + (int)(draw(A.K, A.inj, P_TEST_TURN, a) * span);
    st.test_sample_at[a] = step;
    st.test_result_at[a] = step + turn;
    st.test_positive[a] = pos;
    tested = 1;
  }
  // delivery
  if (st.test_result_at[a] == step) {
    const bool pos = st.test_positive[a] != 0;
    st.test_result_at[a] = NEVER;
    st.test_positive[a] = 0;
    if (pos) {
      if (P->quarantine_enabled) {
        st.quarantine_until[a] = step + P->quarantine_duration;
        st.quarantine_started_at[a] = step;
      }
      if (P->den_enabled && st.has_den_app[a]) {
        fl |= FL_NOTIFIER;
        if (notif) notif[atomicAdd(n_notif, 1)] = (int32_t)a;
      }
    }
  }
  return tested;
}

// Tomorrow's push tables from agent b's next-day code cn.  All 32 lanes of
// the warp call; the warp's lanes hold consecutive agents from wbase_agent.
//   workplace: the worker's next-day position q, wcode[q] = cn, the shifts;
//   random   : the warp's (agent, slot < n) items flattened 32 at a time:
//              rout[a][j] = pi_j(a), rin[pi_j(a)][j] = cn | PRESENT.
__device__ __forceinline__ void push_next_day(const epi_net& net, const NextTables& nx, bool valid, int64_t b,
                                              uint16_t cn, const PermKeys* rk_next, const Radix& dn,
                                              int* excl_w, uint16_t* cn_w, uint8_t* own_w, int64_t wbase_agent,
                                              int lane) {
  const WorkTables& W = *nx.wt;
  const int w = valid ? net.wp_id[b] : -1;
  if (w >= 0) {
    const int m = net.wp_size[w];
    if (m >= 2) {
      const int wbase = net.wp_base[w];
      const int loc = net.wp_local[b];
      const uint32_t q = walk_inv((uint32_t)loc, work_keys(nx.nk.wperm, w), make_radix((uint32_t)m));
      W.pos_of[wbase + loc] = (uint8_t)q;
      W.wcode[wbase + q] = cn;
      for (int j = loc; j < net.colleague_draws; j += m)
        W.shift[(size_t)w * net.colleague_draws + j] = (uint8_t)work_shift(nx.nk.wshift, w, j, m);
    }
  }
  int na = valid ? code_count(cn) : 0;
  na = na < RT_SLOTS ? na : RT_SLOTS;
  int incl = na;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= o) incl += v;
  }
  const int total = __shfl_sync(0xFFFFFFFFu, incl, 31);
  const int excl = incl - na;
  excl_w[lane] = excl;
  cn_w[lane] = cn;
  for (int i = 0; i < na; ++i) own_w[excl + i] = (uint8_t)lane;   // item -> its agent's lane
  __syncwarp();
  for (int k = lane; k < total; k += 32) {
    const int l = own_w[k];
    const int j = k - excl_w[l];
    const uint32_t src = (uint32_t)(wbase_agent + l);
    const uint32_t y = walk_fwd(src, rk_next[j], dn);
    W.rout[(size_t)src * RT_SLOTS + j] = y;
    if (y != src) W.rin[(size_t)y * RT_SLOTS + j] = cn_w[l] | CODE_PRESENT;
  }
  __syncwarp();
}

// Tomorrow's SPARSE push rows (sparse_kind_sums): only agents whose
// next-day code is infectious (code byte != 0) scatter rin[pi_j(b)][j] =
// cn | PRESENT for their slots j < n; the warp's items flattened 32 at a
// time.  No out-rows (the day kernel walks the out-partners itself).
__device__ __forceinline__ void push_next_sparse(const NextTables& nx, bool valid, uint16_t cn,
                                                 const PermKeys* rk_next, const Radix& dn, int* excl_w,
                                                 uint16_t* cn_w, uint8_t* own_w, int64_t wbase_agent, int lane) {
  const WorkTables& W = *nx.wt;
  int na = (valid && (cn & 0xFF) != 0) ? code_count(cn) : 0;
  na = na < RT_SLOTS ? na : RT_SLOTS;
  int incl = na;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= o) incl += v;
  }
  const int total = __shfl_sync(0xFFFFFFFFu, incl, 31);
  if (total == 0) return;                        // (warp-uniform)
  const int excl = incl - na;
  excl_w[lane] = excl;
  cn_w[lane] = cn;
  for (int i = 0; i < na; ++i) own_w[excl + i] = (uint8_t)lane;
  __syncwarp();
  for (int k = lane; k < total; k += 32) {
    const int l = own_w[k];
    const int j = k - excl_w[l];
    const uint32_t src = (uint32_t)(wbase_agent + l);
    const uint32_t y = walk_fwd(src, rk_next[j], dn);
    if (y != src) __stcs(W.rin + (size_t)y * RT_SLOTS + j, (unsigned short)(cn_w[l] | CODE_PRESENT));
  }
  __syncwarp();
}

// Today's sparse rows from today's codes: the first day of a whole-population
// chain (later days come from the previous day's epilogue), and every day of
// a partitioned rank, whose in-partners may live on any rank: all n sources
// are scanned (the day's code vector is complete after the all-gather) and
// only pushes into the rank's own rows [lo, hi) are kept.
__global__ void __launch_bounds__(256) k_sparse_seed(const uint16_t* __restrict__ codes, int64_t n, int64_t lo,
                                                     int64_t hi, const NetTables* __restrict__ NTp,
                                                     uint16_t* __restrict__ rin) {
  __shared__ PermKeys rk[RT_SLOTS];
  if (threadIdx.x < RT_SLOTS) rk[threadIdx.x] = NTp->rk[threadIdx.x];
  __syncthreads();
  const Radix dn = NTp->dn;
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < n; b += (int64_t)gridDim.x * blockDim.x) {
    const uint16_t c = codes[b];
    if ((c & 0xFF) == 0) continue;
    int na = code_count(c);
    na = na < RT_SLOTS ? na : RT_SLOTS;
    for (int j = 0; j < na; ++j) {
      const uint32_t y = walk_fwd((uint32_t)b, rk[j], dn);
      if (y != (uint32_t)b && (int64_t)y >= lo && (int64_t)y < hi) rin[(size_t)y * RT_SLOTS + j] = c | CODE_PRESENT;
    }
  }
}

// tomorrow's random-slot keys into shared memory; block 0 writes those of
// the day after into the ring unless another kernel does (all threads call;
// ends with a bar.sync)
__device__ __forceinline__ void load_next_keys(const NextTables& nx, PermKeys* rk_next) {
  for (int j = threadIdx.x; j < EPI_MAX_SLOTS; j += blockDim.x) rk_next[j] = nx.keys->rk[j];
  if (blockIdx.x == 0 && threadIdx.x < EPI_MAX_SLOTS && nx.keys_out != nullptr)
    nx.keys_out->rk[threadIdx.x] = random_slot_keys(nx.rperm_t2, threadIdx.x);
  __syncthreads();
}

// Testing fused into the day kernel (intervention days on the whole
// population): the notifier work list of the DEN scan.
struct DayTests {
  int on;
  int32_t* notif;
  int* n_notif;
};

// PUSH (the `push` argument, fixed per instantiation so each variant is a
// smaller kernel: the three-way kernel's instruction-cache misses were 19 %
// of its stall samples at 10 M agents)
template <int PUSH>
__global__ void __launch_bounds__(128, 8) k_fused_step(StepArgs A, epi_net net, NetKeys nk,
                                                    const uint16_t* __restrict__ codes, double rate,
                                                    uint16_t* __restrict__ codes_next,
                                                    const epi_net* net_dev, uint64_t rcount_next,
                                                    int final_pass, const WorkTables* wt,
                                                    const MsgTables* __restrict__ mt,
                                                    const NetTables* __restrict__ NTp, NextTables nx,
                                                    int push_arg, DayTests tests) {
  constexpr int push = PUSH;
  (void)push_arg;
  __shared__ MsgTables T;
  __shared__ NetTables NT;
  __shared__ RecAcc racc;
  __shared__ PermKeys rk_next[EPI_MAX_SLOTS];
  __shared__ int excl_s[4][32];
  __shared__ uint16_t cn_s[4][32];
  __shared__ uint8_t own_s[4][32 * RT_SLOTS];
  load_msg_tables(T, mt);
  // with the day's push tables (random rows + workplace codes) only the agent
  // domain is needed; the epilogue derives workplace domains on the fly.
  // push: 0 none (inverse slot walks), 1 push tables, 2 sparse push rows
  if (push == 1) {
    if (threadIdx.x < (int)(sizeof(Radix) / 4))
      ((uint32_t*)&NT.dn)[threadIdx.x] = ((const uint32_t*)&NTp->dn)[threadIdx.x];
  } else {
    load_net_tables(NT, NTp);
  }
  rec_init(racc);
  __syncthreads();
  pdl_wait();
  pdl_trigger();
  const bool merge = nx.wt != nullptr;
  if (merge) load_next_keys(nx, rk_next);
  const Radix dn = NT.dn;
  const int warp = threadIdx.x >> 5, lane = lane_id();
  // one contiguous chunk per block; the grid is a multiple of the SM count,
  // so every SM carries the same number of agents
  const int64_t chunk = (A.hi - A.lo + gridDim.x - 1) / gridDim.x;
  const int64_t c_lo = A.lo + blockIdx.x * chunk;
  const int64_t n = c_lo + chunk < A.hi ? c_lo + chunk : A.hi;
  for (int64_t base = c_lo; base < n; base += blockDim.x) {
    const int64_t b = base + threadIdx.x;
    const bool valid = b < n;
    unsigned edges = 0;
    double lam = 0.0;
    AgentHot h{};
    if (valid) h = push == 2 ? load_hot_stream(A.st, b) : load_hot(A.st, b);   // before the gather's loads
    if (valid) {
      const uint16_t cb = codes[b];
      bool row_used = true;                // (sparse rows: cleared only when non-empty)
      if (!code_dead(cb)) {
        // one sum per network kind (the kind is a constant at every visit),
        // scaled by B[kind] once
        float acc[3] = {0.f, 0.f, 0.f};
        if (push == 1)
          push_kind_sums(net, wt, codes, b, cb, T.factor, acc, edges);
        else if (push == 2)
          sparse_kind_sums(net, NT.rk, dn, wt, codes, b, cb, T.factor, acc, edges, row_used);
        else
          code_kind_sums(net, NT.rk, dn, wt, codes, b, cb, T.factor, acc, edges);
        const float tot = acc[0] * T.bfac[0] + acc[1] * T.bfac[1] + acc[2] * T.bfac[2];
        if (h.stage == S_SUS && !(A.P->sterilizing && h.immune)) lam = (double)(tot * T.sfac[h.age]);
      }
      if (push == 2) {                     // (sparse rows: streamed, evict-first)
        uint4* row = (uint4*)(wt->rin + (size_t)b * RT_SLOTS);
        if (row_used) {
          __stcs(row, make_uint4(0, 0, 0, 0));
          __stcs(row + 1, make_uint4(0, 0, 0, 0));
        }
      } else {
        clear_rin_row(wt, b);
      }
    }
    unsigned ev = 0;
    if (valid) probe_lambda(A.probe, A.step, b, lam);
    if (valid) ev = transmit_progress_hot(A, b, lam, -1, h);
    if (tests.on) {
      // phase 3 + 4a on the agent's own state (k_iv_tests, fused)
      unsigned tested = 0;
      if (valid) {
        uint8_t fl = (ev & 8u) ? FL_SYMPTOMATIC : A.flags[b];
        tested = test_agent(A, b, h.stage, fl, tests.notif, tests.n_notif);
        A.flags[b] = fl;
      }
      rec_add(racc, EPI_REC_TESTS, tested);
    } else if (valid && (ev & 8u) && A.flags) {
      A.flags[b] = FL_SYMPTOMATIC;
    }
    rec_events(racc, ev);
    rec_add(racc, EPI_REC_EDGES, edges);
    if (final_pass) {
      rec_agent(racc, valid, valid ? h.stage : 0, valid ? h.infected_at : 0);
      uint16_t cn = 0;
      if (valid) {
        cn = next_code_hot(A.P, h, b, A.step + 1, net_dev, rcount_next);
        codes_next[b] = cn;
      }
      if (merge && push == 2)
        push_next_sparse(nx, valid, cn, rk_next, dn, excl_s[warp], cn_s[warp], own_s[warp],
                         base + (threadIdx.x & ~31), lane);
      else if (merge)
        push_next_day(net, nx, valid, b, cn, rk_next, dn, excl_s[warp], cn_s[warp], own_s[warp],
                      base + (threadIdx.x & ~31), lane);
    }
  }
  __syncthreads();
  rec_flush(racc, A.rec, A.step);
}

// The workplace codes of a day whose sigma tables were built ahead (without
// codes): wcode[slot] = code of the worker at that position, once the day's
// code vector is complete (after a partitioned run's all-gather).
__global__ void __launch_bounds__(256) k_wcode(int64_t n_slots, const int32_t* __restrict__ member_at_pos,
                                               const uint16_t* __restrict__ codes, uint16_t* __restrict__ wcode) {
  pdl_wait();
  pdl_trigger();
  // four slots per thread per pass, every load of a level issued before any
  // use (the code gather is one dependent level after member_at_pos)
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < n_slots; i0 += 4 * stride) {
    int32_t who[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) who[u] = i0 + u * stride < n_slots ? member_at_pos[i0 + u * stride] : -1;
    uint16_t cw[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) cw[u] = who[u] >= 0 ? codes[who[u]] : (uint16_t)0;
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (who[u] >= 0) wcode[i0 + u * stride] = cw[u];
  }
}

// Per-day tables.  Blocks [0, wblocks) own the workplace member slots (one
// thread each: member_at_pos / pos_of / shift, and wcode in fused mode);
// the remaining blocks own agent rows [lo, hi) for the random push tables:
// each warp takes 32 agents, flattens their (agent, slot j < n_a) work items
// with a warp prefix sum and evaluates them 32 at a time (no idle lanes),
// writing rout[a][j] = code(pi_j(a)) and scattering rin[pi_j(a)][j] = code(a)
// (conflict-free: pi_j is a bijection).
__global__ void __launch_bounds__(256) k_day_tables(epi_net net, NetKeys nk, WorkTables wt,
                                                    const uint16_t* __restrict__ codes, int64_t lo,
                                                    int64_t hi, int wblocks, const NetTables* __restrict__ NTp,
                                                    NetTables* __restrict__ NTnext, uint64_t rperm_next,
                                                    long long* rec) {
  __shared__ NetTables NT;
  __shared__ int excl_s[8][32];
  load_net_tables(NT, NTp);
  __syncthreads();
  pdl_wait();
  pdl_trigger();
  // tomorrow's random-slot keys (the other buffer: yesterday's kernels, its
  // last readers, are complete after pdl_wait) and today's zeroed record
  if (blockIdx.x == 0 && threadIdx.x < EPI_MAX_SLOTS)
    NTnext->rk[threadIdx.x] = random_slot_keys(rperm_next, threadIdx.x);
  if (blockIdx.x == 0 && rec && threadIdx.x < EPI_REC_LEN) rec[threadIdx.x] = 0;
  const int draws = net.colleague_draws;
  if ((int)blockIdx.x < wblocks) {
    // one warp per workplace (m <= 255 members, lanes over its positions):
    // the workplace's size, base and permutation keys once, then per position
    // q the member at sigma(q) -- two dependent loads instead of four per slot
    if (draws <= 0) return;
    const int warp = threadIdx.x >> 5, lane = lane_id();
    const int64_t wwarps = (int64_t)wblocks * (blockDim.x >> 5);
    for (int64_t w = blockIdx.x * (int64_t)(blockDim.x >> 5) + warp; w < net.n_workplaces; w += wwarps) {
      const int base = net.wp_base[w];
      const int m = net.wp_size[w];
      if (m < 2) {
        if (lane < m) {
          const int32_t c = net.wp_members[base + lane];
          wt.pos_of[base + lane] = 0;
          wt.member_at_pos[base + lane] = c;
          if (wt.wcode) wt.wcode[base + lane] = codes[c];
        }
        continue;
      }
      const PermKeys K = work_keys(nk.wperm, (int)w);
      const Radix d = NT.wrad[m];
      for (int q = lane; q < m; q += 32) {
        const uint32_t loc = walk_fwd((uint32_t)q, K, d);
        const int32_t who = net.wp_members[base + loc];
        wt.pos_of[base + loc] = (uint8_t)q;
        for (int j = q; j < draws; j += m)
          wt.shift[(size_t)w * draws + j] = (uint8_t)work_shift(nk.wshift, (int)w, j, m);
        wt.member_at_pos[base + q] = who;
        if (wt.wcode) wt.wcode[base + q] = codes[who];
      }
    }
    return;
  }
  if (wt.rin == nullptr || net.n_agents < 2) return;
  const Radix dn = NT.dn;
  const int warp = threadIdx.x >> 5, lane = lane_id();
  const int64_t n_tiles = (hi - lo + 31) / 32;
  const int64_t warps_total = (int64_t)(gridDim.x - wblocks) * (blockDim.x >> 5);
  for (int64_t tile = (blockIdx.x - wblocks) * (int64_t)(blockDim.x >> 5) + warp; tile < n_tiles;
       tile += warps_total) {
    const int64_t base = lo + tile * 32;
    const int64_t a = base + lane;
    uint16_t ca = 0;
    int na = 0;
    if (a < hi) {
      ca = codes[a];
      na = code_count(ca);
      na = na < RT_SLOTS ? na : RT_SLOTS;
    }
    int incl = na;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if (lane >= o) incl += v;
    }
    const int total = __shfl_sync(0xFFFFFFFFu, incl, 31);
    excl_s[warp][lane] = incl - na;
    __syncwarp();
    for (int k = lane; k < total; k += 32) {
      int l = 0;                                    // owner: last lane with excl <= k
#pragma unroll
      for (int step = 16; step >= 1; step >>= 1)
        if (l + step < 32 && excl_s[warp][l + step] <= k) l += step;
      const int j = k - excl_s[warp][l];
      const uint32_t src = (uint32_t)(base + l);
      const uint32_t y = walk_fwd(src, NT.rk[j], dn);
      wt.rout[(size_t)src * RT_SLOTS + j] = y;
      if (y != src) wt.rin[(size_t)y * RT_SLOTS + j] = codes[src] | CODE_PRESENT;
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// Intervention phases (engine.py:202-347).

// Phase 3 + 4a: test sampling, then delivery (engine.py:202-242).
// Notifiers are also appended to `notif` (count in *n_notif) when given:
// the work list of the DEN regeneration scan.
// Notifiers are also appended to `notif` (count in *n_notif) when given:
// the work list of the DEN regeneration scan.
__global__ void k_iv_tests(StepArgs A, int32_t* __restrict__ notif = nullptr, int* n_notif = nullptr) {
  __shared__ RecAcc racc;
  rec_init(racc);
  __syncthreads();
  const int64_t n = A.hi;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = A.lo + blockIdx.x * (int64_t)blockDim.x; base < n; base += stride) {
    const int64_t a = base + threadIdx.x;
    unsigned tested = 0;
    if (a < n) {
      uint8_t fl = A.flags[a];
      tested = test_agent(A, a, A.st.stage[a], fl, notif, n_notif);
      A.flags[a] = fl;
    }
    rec_add(racc, EPI_REC_TESTS, tested);
  }
  __syncthreads();
  rec_flush(racc, A.rec, A.step);
}

// Contact scan over a COO ring slot: notified[dst] if src is a notifier
// (ContactLog.contacts_of, interventions.py:160-178).
__global__ void k_den_scan_coo(const int32_t* __restrict__ src, const int32_t* __restrict__ dst,
                               int64_t E, uint8_t* __restrict__ flags) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < E;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (flags[src[i]] & FL_NOTIFIER) {
      const int32_t d = dst[i];
      if (!(flags[d] & FL_NOTIFIED)) atomicOr((unsigned*)(flags + (d & ~3)), (unsigned)FL_NOTIFIED << (8 * (d & 3)));
    }
  }
}
// ---------------------------------------------------------------------------
// Exposure notification without a contact log (config networks).  Every
// day's graph is a pure function of (seed, day, who is dead that day), so a
// notifier's contacts of the last `lookback` days are enumerated again
// instead of being stored: for day s an agent is in the networks iff it had
// not died before s (died_at[c] >= s), and its random-slot count is the keyed
// draw of day s.  One warp per (notifier, day) of the day's notifier list
// (lanes split the household, colleague draws and random slots), contacts
// marked NOTIFIED.  The marks
// equal those of a scan over the stored edges of those days (ContactLog,
// interventions.py:145-178), without the 4 B/edge/day log.
constexpr int DEN_MAX_DAYS = 16;
struct DenRegen {
  NetKeys nk[DEN_MAX_DAYS];     // prefixes of days step - n_days .. step - 1
  int first_day, n_days;
};

// died_at[c] = the step during which c died (-1: dead at the start), from
// the day's (complete) code vector: dead in day t's codes and not yet known.
__global__ void k_died_update(const uint16_t* __restrict__ codes, int64_t n, int step,
                              int32_t* __restrict__ died_at) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x)
    if (code_dead(codes[c]) && died_at[c] == INT32_MAX) died_at[c] = step - 1;
}

// One (notifier, past day) item of the DEN regeneration, one warp: the
// notifier's in-edges of that day enumerated again (who was dead that day:
// died_at) and their sources marked notified.  The in-edges of
// for_each_in_edge_f, with each lane on ONE kind so that its load and walk
// chain is one network's, not three in a row: lanes 0-7 household members,
// 8-15 colleague draws, 16-31 random slots (the marks are an OR: the order of
// the visits is free).  `rk_w` is unused (each random lane derives its slot's
// keys).
__device__ __forceinline__ void den_regen_item(const epi_net& net, const NetKeys& nk, int day, int64_t an,
                                               PermKeys* rk_w, const Radix* wrad,
                                               const int32_t* __restrict__ died_at, uint8_t* mark, int lane) {
  (void)rk_w;
  auto code_of = [&](int64_t c) -> uint16_t {
    if (died_at[c] < day) return CODE_DEAD;
    return (uint16_t)(random_count(net, nk.rcount, c) << 8);
  };
  auto mark_c = [&](int64_t c) {
    if (!(mark[c] & FL_NOTIFIED)) atomicOr((unsigned*)(mark + (c & ~3ll)), (unsigned)FL_NOTIFIED << (8 * (c & 3)));
  };
  if (lane < 8) {
    // household: contiguous range
    const int off = net.hh_off[an];
    const int sz = net.hh_size[an];
    const int64_t start = an - off;
    for (int i = lane; i < sz; i += 8) {
      const int64_t c = start + i;
      if (c != an && !code_dead(code_of(c))) mark_c(c);
    }
  } else if (lane < 16) {
    const int li = lane - 8;
    const int w = li < net.colleague_draws ? net.wp_id[an] : -1;
    if (w >= 0) {
      const int m = net.wp_size[w];
      if (m >= 2) {
        const Radix d = wrad[m];
        const PermKeys K = work_keys(nk.wperm, w);
        const int base = net.wp_base[w];
        const uint32_t p = walk_inv(net.wp_local[an], K, d);
        const uint64_t hw = fold(nk.wshift, (uint64_t)w);
        for (int j = li; j < net.colleague_draws; j += 8) {
          const uint64_t hq = fold(hw, (uint64_t)(j >> 2));
          const uint32_t v = (uint32_t)((hq >> (16 * (j & 3))) & 0xFFFF);
          const uint32_t r = 1u + ((v * (uint32_t)(m - 1)) >> 16);
          const int32_t co = net.wp_members[base + walk_fwd(add_mod(p, r, (uint32_t)m), K, d)];
          const int32_t ci = net.wp_members[base + walk_fwd(sub_mod(p, r, (uint32_t)m), K, d)];
          if (!code_dead(code_of(co))) mark_c(co);
          if (!code_dead(code_of(ci))) mark_c(ci);
        }
      }
    }
  } else {
    const uint32_t n = (uint32_t)net.n_agents;
    if (n >= 2) {
      const Radix d = make_radix(n);
      const int nb = code_count(code_of(an));
      for (int j = lane - 16; j < net.random_slots; j += 16) {
        const PermKeys K = random_slot_keys(nk.rperm, j);
        const uint32_t ci = walk_inv((uint32_t)an, K, d);
        if (j < nb) {
          const uint32_t c = walk_fwd((uint32_t)an, K, d);
          if (c != (uint32_t)an && !code_dead(code_of(c))) mark_c(c);
        }
        if (ci != (uint32_t)an && j < code_count(code_of(ci))) mark_c(ci);
      }
    }
  }
  __syncwarp();
}

__global__ void __launch_bounds__(256) k_den_regen(epi_net net, DenRegen D, const int32_t* __restrict__ died_at,
                                                   const int32_t* __restrict__ notif, const int* n_notif,
                                                   uint8_t* __restrict__ mark, const Radix* __restrict__ wrad_g) {
  __shared__ Radix wrad[256];
  __shared__ PermKeys rk[8][EPI_MAX_SLOTS];
  for (int m = threadIdx.x; m < 256; m += blockDim.x) wrad[m] = wrad_g[m];     // static workplace domains
  __syncthreads();
  pdl_wait();
  pdl_trigger();
  const int warp = threadIdx.x >> 5, lane = lane_id();
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  // one warp per (notifier, day)
  const int64_t items = (int64_t)(*n_notif) * D.n_days;
  for (int64_t it = blockIdx.x * (int64_t)(blockDim.x >> 5) + warp; it < items; it += warps) {
    const int d = (int)(it % D.n_days);
    den_regen_item(net, D.nk[d], D.first_day + d, notif[it / D.n_days], rk[warp], wrad, died_at, mark, lane);
  }
}

// Partitioned runs: the notifications pushed by every rank (OR-reduced into
// `mark`) for the owned rows.
__global__ void k_den_merge(const uint8_t* __restrict__ mark, int64_t lo, int64_t hi, uint8_t* __restrict__ flags) {
  for (int64_t a = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < hi; a += (int64_t)gridDim.x * blockDim.x)
    if (mark[a] & FL_NOTIFIED) flags[a] |= FL_NOTIFIED;
}

__device__ __forceinline__ void realize_immunity(const StepArgs& A, int64_t a, int dose) {
  const epi_state& st = A.st;
  const double u = draw(A.K, A.inj, P_VAX, a, dose);
  if (u < st.immunity_check_prob[a] && st.stage[a] == S_SUS) {
    st.immune[a] = 1;
    if (A.P->sterilizing) st.stage[a] = S_VAC;
  }
  st.immunity_check_at[a] = NEVER;
  st.immunity_check_prob[a] = 0.0;
  st.immunity_check_dose[a] = 0;
}

// Phase 4b (DEN follow-ups), 5 (dropout), 6a (due immunity checks,
// eligibility buckets, active count).  engine.py:244-310.
__device__ __forceinline__ void iv_post_agent(const StepArgs& A, int64_t a, uint8_t* __restrict__ bucket,
                                              unsigned* h, unsigned& notified, unsigned& active) {
  const epi_params* __restrict__ P = A.P;
  const epi_state& st = A.st;
  const int step = A.step;
  const uint8_t fl = A.flags[a];
  if (P->den_enabled && (fl & FL_NOTIFIED) && st.has_den_app[a] &&
      st.quarantine_until[a] <= step && st.stage[a] != S_DEAD) {
    notified = 1;
    if (draw(A.K, A.inj, P_DEN, a) < P->den_compliance) st.den_test_due_at[a] = step + 1;
  }
  if (P->quarantine_enabled && st.quarantine_until[a] > step && st.quarantine_started_at[a] < step) {
    if (draw(A.K, A.inj, P_QDROP, a) < P->quarantine_dropout) st.quarantine_until[a] = step;
  }
  if (P->vaccination_enabled) {
    if (st.immunity_check_at[a] == step) {
      const int dose = st.immunity_check_dose[a];
      if (dose == 1 || dose == 2) realize_immunity(A, a, dose);
    }
    const int stage = st.stage[a];
    active = active_stage(stage);
    const bool blocked = stage == S_DEAD || stage == S_HOSP || stage == S_ICU;
    const int vs = st.vaccine_status[a];
    const bool d1 = vs == 0 && !blocked;
    const int32_t d1at = st.dose1_at[a];
    const bool d2 = vs == 1 && d1at != NEVER && step >= d1at + P->dose_gap && !blocked;
    uint8_t bk = NO_BUCKET;
    if (d1 || d2) {
      const int age = st.age_band[a];
      int group;
      if (P->strategy == 0) group = d2 ? 0 : 1;
      else if (P->strategy == 1) group = d2 ? 1 : 0;
      else group = (age >= P->elderly_band) ? 0 : (d2 ? 2 : 1);
      bk = (uint8_t)((group * 9 + (8 - age)) * 2 + (d2 ? 1 : 0));
      atomicAdd(&h[bk], 1u);
    }
    bucket[a] = bk;
  }
}

// iv_post_agent in two parts for k_iv_run, which takes the eligibility into
// the day's first phase (see there): the vaccination bucket + active count,
// and the rest (DEN follow-up, dropout, due immunity checks) in order.
__device__ __forceinline__ uint8_t iv_elig_agent(const StepArgs& A, int64_t a, unsigned* h, unsigned& active) {
  const epi_params* __restrict__ P = A.P;
  const epi_state& st = A.st;
  const int stage = st.stage[a];
  active = active_stage(stage);
  const bool blocked = stage == S_DEAD || stage == S_HOSP || stage == S_ICU;
  const int vs = st.vaccine_status[a];
  const bool d1 = vs == 0 && !blocked;
  const int32_t d1at = st.dose1_at[a];
  const bool d2 = vs == 1 && d1at != NEVER && A.step >= d1at + P->dose_gap && !blocked;
  uint8_t bk = NO_BUCKET;
  if (d1 || d2) {
    const int age = st.age_band[a];
    int group;
    if (P->strategy == 0) group = d2 ? 0 : 1;
    else if (P->strategy == 1) group = d2 ? 1 : 0;
    else group = (age >= P->elderly_band) ? 0 : (d2 ? 2 : 1);
    bk = (uint8_t)((group * 9 + (8 - age)) * 2 + (d2 ? 1 : 0));
    atomicAdd(&h[bk], 1u);
  }
  return bk;
}
// (k_iv_run applies the DEN follow-up itself, the next morning: den = false)
__device__ __forceinline__ void iv_post_rest_agent(const StepArgs& A, int64_t a, bool den) {
  const epi_params* __restrict__ P = A.P;
  const epi_state& st = A.st;
  const int step = A.step;
  if (den) {
    const uint8_t fl = A.flags[a];
    if (P->den_enabled && (fl & FL_NOTIFIED) && st.has_den_app[a] &&
        st.quarantine_until[a] <= step && st.stage[a] != S_DEAD) {
      if (draw(A.K, A.inj, P_DEN, a) < P->den_compliance) st.den_test_due_at[a] = step + 1;
    }
  }
  if (P->quarantine_enabled && st.quarantine_until[a] > step && st.quarantine_started_at[a] < step) {
    if (draw(A.K, A.inj, P_QDROP, a) < P->quarantine_dropout) st.quarantine_until[a] = step;
  }
  if (P->vaccination_enabled && st.immunity_check_at[a] == step) {
    const int dose = st.immunity_check_dose[a];
    if (dose == 1 || dose == 2) realize_immunity(A, a, dose);
  }
}

__global__ void k_iv_post(StepArgs A, uint8_t* __restrict__ bucket, unsigned long long* __restrict__ hist) {
  __shared__ RecAcc racc;
  __shared__ unsigned h[NUM_BUCKETS];
  rec_init(racc);
  for (int i = threadIdx.x; i < NUM_BUCKETS; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const int64_t n = A.hi;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = A.lo + blockIdx.x * (int64_t)blockDim.x; base < n; base += stride) {
    const int64_t a = base + threadIdx.x;
    unsigned notified = 0, active = 0;
    if (a < n) iv_post_agent(A, a, bucket, h, notified, active);
    rec_add(racc, EPI_REC_NOTIFY, notified);
    rec_add(racc, EPI_REC_ACTIVE, active);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < NUM_BUCKETS; i += blockDim.x)
    if (h[i]) atomicAdd(&hist[i], (unsigned long long)h[i]);
  rec_flush(racc, A.rec, A.step);
}

// plan[0] = cut bucket (-1: nobody), plan[1] = remaining slots in the cut
// bucket.  Trigger latch + budget (engine.py:286-310).  `hist` is the
// population's eligibility histogram; hist[NUM_BUCKETS] the population's
// active count when `global_active` (partitioned runs: summed over ranks),
// else the active count is this record's.  Only `write_doses` ranks record
// the doses given (rank 0 of a partitioned run).
__device__ __forceinline__ void vax_plan(const epi_params* __restrict__ P, const unsigned long long* hist,
                                         long long* rec, int32_t* vax_open, long long* plan, int global_active,
                                         int write_doses) {
  int open = *vax_open;
  const double active = global_active ? (double)__ldcg(hist + NUM_BUCKETS) : (double)__ldcg(rec + EPI_REC_ACTIVE);
  if (!open && active >= P->start_trigger_count) open = 1;
  *vax_open = open;
  plan[0] = -1;
  plan[1] = 0;
  const long long budget = P->dose_budget;
  if (!open || budget <= 0) return;
  long long cum = 0;
  for (int b = 0; b < NUM_BUCKETS; ++b) {
    const long long c = (long long)__ldcg(hist + b);
    if (cum + c >= budget) {
      plan[0] = b;
      plan[1] = budget - cum;
      if (write_doses) rec[EPI_REC_DOSES] = budget;
      return;
    }
    cum += c;
  }
  plan[0] = NUM_BUCKETS;       // everyone eligible gets a dose
  plan[1] = 0;
  if (write_doses) rec[EPI_REC_DOSES] = cum;
}

__global__ void k_vax_plan(const epi_params* __restrict__ P, const unsigned long long* __restrict__ hist,
                           long long* rec, int32_t* vax_open, long long* plan, int global_active,
                           int write_doses) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  vax_plan(P, hist, rec, vax_open, plan, global_active, write_doses);
}

// Phase 6b for one selected agent (engine.py:306-335): bucket bit 0 = dose rank.
__device__ __forceinline__ void give_dose(const StepArgs& A, int64_t a, uint8_t bk) {
  const epi_params* __restrict__ P = A.P;
  const epi_state& st = A.st;
  const int step = A.step;
  if ((bk & 1) == 0) {       // first dose
    st.vaccine_status[a] = 1;
    st.dose1_at[a] = step;
    st.immunity_check_at[a] = step + P->dose1_latency;
    st.immunity_check_prob[a] = P->dose1_efficacy;
    st.immunity_check_dose[a] = 1;
    if (P->dose1_latency == 0) realize_immunity(A, a, 1);
  } else {                   // second dose
    st.vaccine_status[a] = 2;
    st.dose2_at[a] = step;
    double prob = (st.immunity_check_at[a] != NEVER) ? P->dose2_efficacy : P->dose2_topup;
    if (st.immune[a]) prob = 0.0;
    st.immunity_check_at[a] = step + P->dose2_latency;
    st.immunity_check_prob[a] = prob;
    st.immunity_check_dose[a] = 2;
    if (P->dose2_latency == 0) realize_immunity(A, a, 2);
  }
}

constexpr int VAX_TILE = 1024;

// Tiles of VAX_TILE agents over the owned rows [lo, n).
__global__ void k_vax_tilecount(const uint8_t* __restrict__ bucket, int64_t lo, int64_t n, const long long* plan,
                                int* __restrict__ tile_count) {
  const long long cut = plan[0];
  __shared__ int cnt;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  const int64_t a = lo + blockIdx.x * (int64_t)VAX_TILE + threadIdx.x;
  const int hit = (cut >= 0 && cut < NUM_BUCKETS && a < n && bucket[a] == (uint8_t)cut) ? 1 : 0;
  const int w = __reduce_add_sync(0xFFFFFFFFu, hit);
  if (lane_id() == 0 && w) atomicAdd(&cnt, w);
  __syncthreads();
  if (threadIdx.x == 0) tile_count[blockIdx.x] = cnt;
}

// Exclusive scan of the tile counts; the total (this range's agents in the
// cut bucket) goes to *total.
__global__ void k_vax_tilescan(int* __restrict__ tile_count, int64_t tiles, long long* total) {
  // single block exclusive scan (tiles <= a few 10k)
  typedef cub::BlockScan<int, 1024> Scan;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < tiles; base += 1024) {
    const int64_t i = base + threadIdx.x;
    const int v = i < tiles ? tile_count[i] : 0;
    int ex, total;
    Scan(tmp).ExclusiveSum(v, ex, total);
    if (i < tiles) tile_count[i] = ex + carry;
    __syncthreads();
    if (threadIdx.x == 0) carry += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = carry;
}

// Phase 6b: administer doses to the selected agents (engine.py:306-335).
// The cut bucket is served in id order: `offset` (nullable) = its agents on
// lower-ranked (lower-id) partitions.
__global__ void __launch_bounds__(1024) k_vax_apply(StepArgs A, const uint8_t* __restrict__ bucket,
                                                    const long long* plan, const int* __restrict__ tile_off,
                                                    const long long* offset) {
  typedef cub::BlockScan<int, 1024> Scan;
  __shared__ typename Scan::TempStorage tmp;
  const long long cut = plan[0], rem = plan[1] - (offset ? *offset : 0);
  const int64_t n = A.hi;
  const int64_t a = A.lo + blockIdx.x * (int64_t)VAX_TILE + threadIdx.x;
  const uint8_t bk = a < n ? bucket[a] : NO_BUCKET;
  const int in_cut = (cut >= 0 && cut < NUM_BUCKETS && bk == (uint8_t)cut) ? 1 : 0;
  int rank;
  Scan(tmp).ExclusiveSum(in_cut, rank);
  if (cut < 0 || bk == NO_BUCKET) return;
  const bool take = (long long)bk < cut || (in_cut && (long long)(tile_off[blockIdx.x] + rank) < rem);
  if (take) give_dose(A, a, bk);
}

// Last kernel of an intervention step: record + next codes + clear flags.
__global__ void k_finish(StepArgs A, uint16_t* __restrict__ codes_next, const epi_net* net,
                         uint64_t rcount_next) {
  __shared__ RecAcc racc;
  rec_init(racc);
  __syncthreads();
  const int64_t n = A.hi;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = A.lo + blockIdx.x * (int64_t)blockDim.x; base < n; base += stride) {
    const int64_t a = base + threadIdx.x;
    const bool valid = a < n;
    rec_agent(racc, valid, valid ? A.st.stage[a] : 0, valid ? A.st.infected_at[a] : 0);
    if (valid) {
      if (codes_next) codes_next[a] = next_code(A.P, A.st, a, A.step + 1, net, rcount_next);
      if (A.flags) A.flags[a] = 0;
    }
  }
  __syncthreads();
  rec_flush(racc, A.rec, A.step);
}

// ---------------------------------------------------------------------------
// Intervention day on the whole population in three launches after the fused
// day kernel (which also runs the testing phase): [k_den_regen] ->
// k_iv_post_chunks -> k_finish_iv.  Both walk the same contiguous chunks (one
// per block, a multiple of 256 agents), so a chunk is the vaccination tile:
//   k_iv_post_chunks: phases 4b/5/6a per agent; the chunk's 54-bucket
//     eligibility histogram to tile_hist[block] and into the day's histogram;
//   k_finish_iv: every block derives the vaccination plan (trigger latch, cut
//     bucket, remaining budget: k_vax_plan) from the day's histogram and its
//     chunk's offset in the cut bucket from the earlier chunks' counts
//     (k_vax_tilecount + k_vax_tilescan), gives the doses in id order
//     (k_vax_apply), records the day each agent died (k_died_update, one day
//     early), the record, next codes, cleared flags, and tomorrow's push
//     tables (the merged fused epilogue) — so no k_day_tables.
// The day's histogram is parity-buffered: k_finish_iv zeroes tomorrow's.
// Same per-agent operations as the per-phase kernels: bitwise the same run.
struct IvPlan {
  unsigned long long* hist;     // [2][NUM_BUCKETS] by day parity
  unsigned* tile_hist;          // [blocks][NUM_BUCKETS]
  int32_t* vax_open;
  int64_t chunk;
  int vax;
};

__global__ void __launch_bounds__(256) k_iv_post_chunks(StepArgs A, uint8_t* __restrict__ bucket, IvPlan V) {
  __shared__ RecAcc racc;
  __shared__ unsigned h[NUM_BUCKETS];
  rec_init(racc);
  for (int i = threadIdx.x; i < NUM_BUCKETS; i += blockDim.x) h[i] = 0;
  __syncthreads();
  pdl_wait();
  pdl_trigger();
  const int64_t lo = A.lo + blockIdx.x * V.chunk;
  const int64_t hi = lo + V.chunk < A.hi ? lo + V.chunk : A.hi;
  for (int64_t base = lo; base < hi; base += blockDim.x) {
    const int64_t a = base + threadIdx.x;
    unsigned notified = 0, active = 0;
    if (a < hi) iv_post_agent(A, a, bucket, h, notified, active);
    rec_add(racc, EPI_REC_NOTIFY, notified);
    rec_add(racc, EPI_REC_ACTIVE, active);
  }
  __syncthreads();
  if (V.vax) {
    unsigned long long* hist = V.hist + (A.step & 1) * NUM_BUCKETS;
    for (int i = threadIdx.x; i < NUM_BUCKETS; i += blockDim.x) {
      V.tile_hist[(size_t)blockIdx.x * NUM_BUCKETS + i] = h[i];
      if (h[i]) atomicAdd(&hist[i], (unsigned long long)h[i]);
    }
  }
  rec_flush(racc, A.rec, A.step);
}

__global__ void __launch_bounds__(256) k_finish_iv(StepArgs A, uint16_t* __restrict__ codes_next,
                                                   const epi_net* net_dev, uint64_t rcount_next,
                                                   const uint8_t* __restrict__ bucket, IvPlan V,
                                                   int32_t* __restrict__ died_at, int* den_count, epi_net net,
                                                   NextTables nx, Radix dn) {
  typedef cub::BlockScan<int, 256> Scan;
  typedef cub::BlockReduce<int, 256> Reduce;
  __shared__ union {
    typename Scan::TempStorage scan;
    typename Reduce::TempStorage reduce;
  } tmp;
  __shared__ RecAcc racc;
  __shared__ PermKeys rk_next[EPI_MAX_SLOTS];
  __shared__ int excl_s[8][32];
  __shared__ uint16_t cn_s[8][32];
  __shared__ uint8_t own_s[8][32 * RT_SLOTS];
  __shared__ unsigned long long h_s[NUM_BUCKETS];
  __shared__ long long plan_s[2];
  __shared__ int off_s;
  rec_init(racc);
  // prologue (overlaps the previous kernel): tomorrow's random-slot keys
  // (written by yesterday's k_finish_iv)
  for (int j = threadIdx.x; j < EPI_MAX_SLOTS; j += blockDim.x) rk_next[j] = nx.keys->rk[j];
  pdl_wait();
  pdl_trigger();
  if (blockIdx.x == 0 && threadIdx.x < EPI_MAX_SLOTS)
    nx.keys_out->rk[threadIdx.x] = random_slot_keys(nx.rperm_t2, threadIdx.x);
  const int warp = threadIdx.x >> 5, lane = lane_id();
  long long cut = -1, rem = 0;
  int carry = 0;
  if (V.vax) {
    // the day's plan, derived by every block from the complete histogram
    const unsigned long long* hist = V.hist + (A.step & 1) * NUM_BUCKETS;
    for (int i = threadIdx.x; i < NUM_BUCKETS; i += blockDim.x) h_s[i] = hist[i];
    if (blockIdx.x == 0)     // tomorrow's histogram starts empty
      for (int i = threadIdx.x; i < NUM_BUCKETS; i += blockDim.x) V.hist[((A.step + 1) & 1) * NUM_BUCKETS + i] = 0;
    __syncthreads();
    if (threadIdx.x == 0) {
      const epi_params* __restrict__ P = A.P;
      int open = *V.vax_open;
      if (!open && (double)A.rec[EPI_REC_ACTIVE] >= P->start_trigger_count) open = 1;
      long long c = -1, r = 0, doses = -1;
      if (open && P->dose_budget > 0) {
        long long cum = 0;
        c = NUM_BUCKETS;                // everyone eligible gets a dose
        doses = -2;
        for (int b = 0; b < NUM_BUCKETS; ++b) {
          const long long hb = (long long)h_s[b];
          if (cum + hb >= P->dose_budget) { c = b; r = P->dose_budget - cum; doses = P->dose_budget; break; }
          cum += hb;
        }
        if (doses == -2) doses = cum;
      }
      if (blockIdx.x == 0) {     // the latch only ever closes -> opens: a late reader derives the same
        *V.vax_open = open;
        if (doses >= 0) A.rec[EPI_REC_DOSES] = doses;
      }
      plan_s[0] = c;
      plan_s[1] = r;
    }
    __syncthreads();
    cut = plan_s[0];
    rem = plan_s[1];
    // this chunk's offset in the cut bucket: the earlier chunks' counts
    int part = 0;
    if (cut >= 0 && cut < NUM_BUCKETS)
      for (int t = threadIdx.x; t < (int)blockIdx.x; t += blockDim.x)
        part += (int)V.tile_hist[(size_t)t * NUM_BUCKETS + cut];
    const int tot = Reduce(tmp.reduce).Sum(part);
    if (threadIdx.x == 0) off_s = tot;
    __syncthreads();
    carry = off_s;
  }
  __syncthreads();
  if (den_count && blockIdx.x == 0 && threadIdx.x == 0) *den_count = 0;   // tomorrow's notifier list
  const bool in_scan = cut >= 0 && cut < NUM_BUCKETS;
  const int64_t lo = A.lo + blockIdx.x * V.chunk;
  const int64_t hi = lo + V.chunk < A.hi ? lo + V.chunk : A.hi;
  for (int64_t base = lo; base < hi; base += blockDim.x) {
    const int64_t a = base + threadIdx.x;
    const bool valid = a < hi;
    if (V.vax) {
      const uint8_t bk = valid ? bucket[a] : NO_BUCKET;
      const int in_cut = (in_scan && bk == (uint8_t)cut) ? 1 : 0;
      int rank, total;
      Scan(tmp.scan).ExclusiveSum(in_cut, rank, total);
      if (cut >= 0 && bk != NO_BUCKET &&
          ((long long)bk < cut || (in_cut && (long long)(carry + rank) < rem)))
        give_dose(A, a, bk);
      carry += total;
      __syncthreads();
    }
    int stage = 0;
    int32_t inf = 0;
    uint16_t cn = 0;
    if (valid) {
      stage = A.st.stage[a];
      inf = A.st.infected_at[a];
      if (died_at && stage == S_DEAD && died_at[a] == INT32_MAX) died_at[a] = A.step;
      cn = next_code(A.P, A.st, a, A.step + 1, net_dev, rcount_next);
      codes_next[a] = cn;
      A.flags[a] = 0;
    }
    rec_agent(racc, valid, stage, inf);
    push_next_day(net, nx, valid, a, cn, rk_next, dn, excl_s[warp], cn_s[warp], own_s[warp],
                  base + (threadIdx.x & ~31), lane);
  }
  __syncthreads();
  rec_flush(racc, A.rec, A.step);
}

// ---------------------------------------------------------------------------
__global__ void k_uniforms(uint64_t prefix, const int64_t* __restrict__ ids, int64_t n, int k,
                           double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = keyed_u(prefix, (uint64_t)(ids ? ids[i] : i), (uint64_t)k);
}

// Seeding at step 0 (population.py:151-177 after the choice of ids).
__global__ void k_seed(const epi_params* __restrict__ P, epi_state st, StepKeys K,
                       const int64_t* __restrict__ ids, int64_t m) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = ids[i];
    const int age = st.age_band[a];
    const int entry = P->targets[S_SUS][pick_branch(P, S_SUS, age, keyed_u(K.p[P_ENTRY], a))];
    int nxt, delay;
    schedule(P, entry, age, keyed_u(K.p[P_BRANCH], a), keyed_u(K.p[P_DELAY], a), nxt, delay);
    st.stage[a] = (int8_t)entry;
    st.infected_at[a] = 0;
    st.next_stage[a] = (int8_t)nxt;
    st.next_transition_at[a] = delay;
  }
}

__global__ void k_assign_app(epi_state st, uint64_t prefix, double adoption) {
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < st.n_agents;
       a += (int64_t)gridDim.x * blockDim.x)
    st.has_den_app[a] = keyed_u(prefix, (uint64_t)a) < adoption;
}

}  // namespace epi
