// Persistent fused run: every day of a config-network simulation in ONE
// launch (epi_sim_run, merged fused mode: no interventions, whole population,
// push tables).  One block per SM, one thread per agent for the whole run and
// a grid barrier between days, so what the per-day kernel (k_fused_step)
// reloads every day stays in registers:
//   - the agent's static network data (household range, workplace id, slot,
//     size, base) and its state (AgentHot), written through on change only;
//   - its own code and its workplace position of the day (computed by itself
//     in the previous day's epilogue), which removes the two deepest levels
//     of the per-day load chain (wp_id -> wp_size/base -> pos_of -> wcode);
//   - the message tables.
// A service warp per block computes the next day's key prefixes and flushes
// the previous day's record while the agent warps work, so nothing sits
// between the barrier's arrive and wait.
// Arithmetic, visit order and sums are those of k_fused_step with
// push_kind_sums, so results are bitwise identical to the per-day path
// (tests/test_gpu_persistent.py).
//
// Data written inside the kernel (codes, push tables) is read with plain
// coherent loads, never through the read-only (.nc) path; the colleague
// shifts are hashed in registers instead of read from the shift table.
#pragma once

#include "epi_kernels.cuh"

namespace epi {

struct DayKeys {
  StepKeys K;                     // purposes of day t
  uint64_t wshift;                // P_NET_WSHIFT of day t (the colleague shifts, computed)
  uint64_t rcount_next;           // P_NET_RCOUNT of t + 1 (tomorrow's codes)
  uint64_t wperm_next, wshift_next;
  PermKeys rk_next[RT_SLOTS];     // random-slot keys of t + 1 (tomorrow's push rows)
};

// one warp fills the keys of day t
__device__ __forceinline__ void day_keys(DayKeys& D, uint64_t seed, int t, int lane) {
  if (lane < 12) D.K.p[lane] = key_prefix(seed, t, lane);
  else if (lane == 12) D.rcount_next = key_prefix(seed, t + 1, P_NET_RCOUNT);
  else if (lane == 13) D.wperm_next = key_prefix(seed, t + 1, P_NET_WPERM);
  else if (lane == 14) D.wshift_next = key_prefix(seed, t + 1, P_NET_WSHIFT);
  else if (lane == 15) D.wshift = key_prefix(seed, t, P_NET_WSHIFT);
  else if (lane >= 16) D.rk_next[lane - 16] = random_slot_keys(key_prefix(seed, t + 1, P_NET_RPERM), lane - 16);
}

struct RunArgs {
  const epi_params* P;
  epi_state st;
  uint64_t seed;
  int first_step, n_days;
  long long* records;             // [n_days][EPI_REC_LEN], zeroed
  uint16_t* codes[2];             // by day parity
  WorkTables wt[2];               // push tables by day parity
  NetTables* ring_t2;             // rk of day first+n_days+1 (keeps the merged chain resumable)
  const MsgTables* mt;
  const uint16_t* tau_lut;
  Radix dn;
  unsigned* barrier;              // zeroed arrival counter
  LamProbe probe;
  uint4* wtab;                    // [3][n_workplaces][2]: per-workplace window values by run day mod 3 (a slow block may still read day d's while a fast one writes day d + 1's)
  // colleague rows (k_fused_run<RUN_MAX_THREADS>), by workplace position:
  // crow[par][(base_W + q) * 16 + s] = the code of the colleague in slot s
  // (2j: out-partner of draw j, 2j + 1: in-partner) of the worker at position
  // q on the days of that parity, written only by infectious or dead
  // colleagues (0 otherwise) and cleared by its reader; all zero between
  // launches
  uint16_t* crow[2];
};

// Grid barrier between days: one arrival per block (release reduction on one
// counter) after a bar.sync, so every store of the block's day precedes it;
// thread 0 polls with acquire loads and the closing bar.sync extends the
// order to the block.  The last block to arrive releases the grid at once
// (measured 1.3 us from its arrival).  One block per SM keeps the arrivals at
// 148 (1.2 us per barrier, tools/micro/grid_barrier.cu; cg::grid.sync with 6
// blocks per SM: 1.9 us).
// Arrival: a release reduction (the block's stores of the day, ordered
// before it by the bar.sync, precede it; no value comes back).
__device__ __forceinline__ void grid_arrive(unsigned* bar) {
  asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
}
// Wait: acquire loads until every block has arrived `target` times in all.
__device__ __forceinline__ void grid_wait(const unsigned* bar, unsigned target) {
  unsigned v;
  do {
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
  } while (v < target);
}
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    grid_arrive(bar);
    grid_wait(bar, target);
  }
  __syncthreads();
}

// The record rows of a finished day (all warps past a bar.sync) into the
// day's record, by one warp: lane c sums column c over the warps' rows and
// zeroes them (their next adds come two days later).
__device__ __forceinline__ void rec_flush_warp(RecAcc& s, long long* rec, int step, int nw, int lane) {
  if (blockIdx.x == 0 && lane == 0) rec[EPI_REC_STEP] = step;
  if (lane >= EPI_REC_LEN || lane == EPI_REC_STEP) return;
  unsigned long long t = 0;
  for (int w = 0; w < nw; ++w) {
    const unsigned v = s.v[w][lane];
    s.v[w][lane] = 0u;
    t = lane == EPI_REC_FLAGS ? (t | v) : (t + v);
  }
  if (!t) return;
  if (lane == EPI_REC_FLAGS) atomicOr((unsigned long long*)&rec[lane], t);
  else atomicAdd((unsigned long long*)&rec[lane], t);
}

constexpr int RUN_MAX_DAYS = 1 << 20;      // days per launch (no per-day state)

// one block per SM: up to 704 agent threads (one agent each) + one service
// warp that flushes yesterday's record and computes tomorrow's keys while
// the agent warps work
constexpr int RUN_MAX_AGENTS = 704;
constexpr int RUN_MAX_THREADS = RUN_MAX_AGENTS + 32;
// The block's out-rows (rout: each agent's random out-partners of the day)
// live in dynamic shared memory for the whole run: the block writes them
// itself (its own push items) and only it reads them, so the global table
// is written on the last day only (for the per-day path).  Row stride 20
// words: a quarter warp's 16-byte row reads hit distinct banks.
constexpr int RUN_OUT_STRIDE = RT_SLOTS + 4;
constexpr size_t RUN_DYN_SMEM = (size_t)RUN_MAX_AGENTS * RUN_OUT_STRIDE * sizeof(uint32_t);
// k_fused_run also comes as a 1024-thread block (992 agents per SM, at most 64
// registers) for populations between 104 k and 147 k agents
constexpr int RUN_BIG_THREADS = 1024;
constexpr int RUN_BIG_AGENTS = RUN_BIG_THREADS - 32;
template <int MAXT> constexpr size_t run_dyn_smem() { return (size_t)(MAXT - 32) * RUN_OUT_STRIDE * sizeof(uint32_t); }
// loads of data written during the run: plain (coherent) global loads; the
// grid barrier orders them after the writers' stores
template <class T> __device__ __forceinline__ T LDM(const T* p) { return *p; }

// A colleague row (16 slots of codes, two uint4, low half of each word
// first = the visit order out, in per draw): the slot-ordered factor adds
// when some slot holds an infectious colleague (the others add +0.0f: bitwise
// add_src_group over the gathered codes), and `present` minus the dead
// colleagues as edges.
__device__ __forceinline__ void add_crow(float& acc, unsigned& edges, const float* __restrict__ factor, uint4 c0,
                                         uint4 c1, unsigned present) {
  const uint32_t w[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
  uint32_t any = 0, dead = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    any |= w[i];
    dead += (w[i] >> 15) & 0x00010001u;
  }
  if (any & 0x00FF00FFu) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      acc += factor[w[i] & 0xFF];
      acc += factor[(w[i] >> 16) & 0xFF];
    }
  }
  edges += present - ((dead & 0xFFFFu) + (dead >> 16));
}
// Code `c` of the worker at position `q` of a workplace window (base, m) into
// the colleague rows `crn` (by position) of the day the shifts `sh` belong
// to: it is the out-partner of draw j of the worker at q - r_j and the
// in-partner of the one at q + r_j (stores only).
template <int DR>
__device__ __forceinline__ void push_colleague_rows(uint16_t* crn, int base, uint32_t q, uint32_t m, uint2 sh,
                                                    int draws, uint16_t c) {
#pragma unroll
  for (int j = 0; j < DR; ++j) {
    if (j < draws) {
      const uint32_t r = ((j < 4 ? sh.x : sh.y) >> (8 * (j & 3))) & 0xFFu;
      crn[(size_t)(base + sub_mod(q, r, m)) * 16 + 2 * j] = c;
      crn[(size_t)(base + add_mod(q, r, m)) * 16 + 2 * j + 1] = c;
    }
  }
}

// The day's 8 colleague shifts r_j of workplace w (work_shift: four 16-bit
// fields per hash), packed one byte each (r_j <= m - 1 <= 254).
__device__ __forceinline__ uint2 day_shifts(uint64_t wshift_prefix, int w, int m) {
  const uint64_t hw = fold(wshift_prefix, (uint64_t)w);
  const uint64_t h0 = fold(hw, 0), h1 = fold(hw, 1);
  uint32_t lo = 0, hi = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    lo |= (1u + ((((uint32_t)(h0 >> (16 * q))) & 0xFFFFu) * (uint32_t)(m - 1) >> 16)) << (8 * q);
    hi |= (1u + ((((uint32_t)(h1 >> (16 * q))) & 0xFFFFu) * (uint32_t)(m - 1) >> 16)) << (8 * q);
  }
  return make_uint2(lo, hi);
}

// The per-workplace values of the barrier window after a day (the colleague
// shifts of the coming day, the permutation keys of the day after), computed
// once per workplace by the service warps a day ahead instead of by every
// member: entry = {fold(fold(wperm, w), 0) (64 bits), fold(fold(wperm, w), 1)
// low 32 bits, 0}, {shifts.x, shifts.y}.
__device__ __forceinline__ PermKeys work_keys_from(uint64_t ha, uint32_t hb) {
  PermKeys K;
  K.k1[0] = (uint32_t)(ha & 0xFFFF);
  K.k2[0] = (uint32_t)((ha >> 16) & 0xFFFF) | 1u;
  K.k1[1] = (uint32_t)((ha >> 32) & 0xFFFF);
  K.k2[1] = (uint32_t)((ha >> 48) & 0xFFFF) | 1u;
  K.k1[2] = hb & 0xFFFF;
  K.k2[2] = ((hb >> 16) & 0xFFFF) | 1u;
  return K;
}

template <int MAXT>
__global__ void __launch_bounds__(MAXT, 1) k_fused_run(RunArgs R, epi_net net) {
  constexpr int HH = 8, DR = 8;
  __shared__ MsgTables T;
  __shared__ RecAcc racc[2];               // record rows by day parity
  __shared__ int excl_s[MAXT / 32][32];
  __shared__ uint16_t cn_s[MAXT / 32][32];
  __shared__ uint8_t own_s[MAXT / 32][32 * RT_SLOTS];
  __shared__ DayKeys dk[2];                // keys by day parity
  __shared__ uint16_t hcode_s[2][MAXT - 32];     // the block's codes by day parity
  __shared__ double cdf_s[EPI_MAX_SLOTS];         // the random-slot count CDF (per-lane indexed)
  extern __shared__ uint4 run_dyn_s[];
  uint32_t* const out_s = (uint32_t*)run_dyn_s;    // [agent][RUN_OUT_STRIDE]
  load_msg_tables(T, R.mt);
  if (threadIdx.x < EPI_MAX_SLOTS) cdf_s[threadIdx.x] = net.poisson_cdf[threadIdx.x];
  rec_init(racc[0]);
  rec_init(racc[1]);
  const int warp = threadIdx.x >> 5, lane = lane_id();
  const int nwa = (int)(blockDim.x >> 5) - 1;     // agent warps; warp nwa is the service warp
  const bool service = warp == nwa;
  if (warp == 0) day_keys(dk[0], R.seed, R.first_step, lane);
  const int64_t n = net.n_agents;
  // equal contiguous agent ranges per block (one block per SM)
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t blo = blockIdx.x * per;
  const int64_t bhi = blo + per < n ? blo + per : n;
  const int64_t b = blo + threadIdx.x;
  const bool valid = !service && b < bhi;
  const uint32_t self = (uint32_t)b;
  const int draws = net.colleague_draws;
  // static network data and the agent's state, once
  int off = 0, sz = 0, w = -1, loc = 0, m = 0, base = 0;
  AgentHot h{};
  uint16_t cb = CODE_DEAD;
  uint32_t p = 0;
  if (valid) {
    off = net.hh_off[b];
    sz = net.hh_size[b];
    w = net.wp_id[b];
    loc = net.wp_local[b];
    h = load_hot(R.st, b);
    cb = LDM(R.codes[R.first_step & 1] + b);
    if (w >= 0) {
      m = net.wp_size[w];
      base = net.wp_base[w];
      if (m >= 2) p = LDM(R.wt[R.first_step & 1].pos_of + base + loc);
    }
    hcode_s[R.first_step & 1][threadIdx.x] = cb;
    const uint4* ro = (const uint4*)(R.wt[R.first_step & 1].rout + (size_t)b * RT_SLOTS);
    uint4* os = (uint4*)(out_s + threadIdx.x * RUN_OUT_STRIDE);
#pragma unroll
    for (int q = 0; q < RT_SLOTS / 4; ++q) os[q] = LDM(ro + q);
  }
  // household members inside the block's range are read from hcode_s
  const int hl0 = (int)threadIdx.x - off;
  const int nloc = (int)(bhi - blo);
  const bool works = w >= 0 && m >= 2;
  const int64_t start = b - off;
  // the whole household in the block: its codes come from hcode_s
  const bool hin = hl0 >= 0 && hl0 + sz <= nloc;
  const unsigned hmask = household_mask(HH, sz, off);
  const Radix rm = make_radix(works ? (uint32_t)m : 1u);
  __syncthreads();
  // state-independent values of the coming day, computed ahead (here, then
  // between each barrier's arrive and wait): today's shifts, the slot count
  // of tomorrow's code and tomorrow's workplace position
  uint2 shp = works ? day_shifts(dk[0].wshift, w, m) : make_uint2(0, 0);
  int cnt_nx = valid ? random_count_cdf(cdf_s, net.random_slots, dk[0].rcount_next, b) : 0;
  uint32_t q_nx = works ? walk_inv((uint32_t)loc, work_keys(dk[0].wperm_next, w), rm) : 0u;
  // colleague rows (the 736-thread variant): infectious and dead workers push
  // their code of day t + 1 into the rows, by position, of their colleagues of
  // t + 1, so a worker reads one 32-byte row instead of gathering 16 codes;
  // the launch's first day is pushed before the loop
  constexpr bool CROW = MAXT <= RUN_MAX_THREADS;
  unsigned bar0 = 0;                       // grid barriers before the first day's
  uint2 shq = make_uint2(0, 0);            // the shifts of the rows being pushed (t + 1)
  auto push_rows = [&](uint16_t c, uint32_t q, uint2 sh, uint16_t* crn) {
    push_colleague_rows<DR>(crn, base, q, (uint32_t)m, sh, draws, c);
  };
  if (CROW) {
    // the rows of the launch's first day from today's codes
    if (works && (cb & 0x80FFu) != 0u) push_rows(cb, p, shp, R.crow[R.first_step & 1]);
    if (works && R.n_days > 1) shq = day_shifts(key_prefix(R.seed, R.first_step + 1, P_NET_WSHIFT), w, m);
    grid_barrier(R.barrier, gridDim.x);
    bar0 = 1;
  }
  for (int d = 0; d < R.n_days; ++d) {
    const int t = R.first_step + d;
    const int par = t & 1;
    const DayKeys& D = dk[d & 1];
    RecAcc& rc = racc[d & 1];
    int pend = -1;                         // the day's deferred transition scheduling
    if (service) {
      // yesterday's record rows (complete since the barrier); tomorrow's keys
      if (d > 0) rec_flush_warp(racc[(d - 1) & 1], R.records + (size_t)(d - 1) * EPI_REC_LEN, t - 1, nwa, lane);
      if (d + 1 < R.n_days) day_keys(dk[(d + 1) & 1], R.seed, t + 1, lane);
      if (d + 2 < R.n_days) {
        // the workplace values of the window after day d + 1: shifts of
        // t + 2, permutation keys of t + 3 (this block's share of the workplaces)
        const uint64_t wsh = key_prefix(R.seed, t + 2, P_NET_WSHIFT);
        const uint64_t wpm = key_prefix(R.seed, t + 3, P_NET_WPERM);
        const int nW = net.n_workplaces;
        const int per_w = (nW + (int)gridDim.x - 1) / (int)gridDim.x;
        const int w_lo = (int)blockIdx.x * per_w, w_hi = w_lo + per_w < nW ? w_lo + per_w : nW;
        uint4* tab = R.wtab + (size_t)((d + 1) % 3) * 2 * nW;
        for (int ww = w_lo + lane; ww < w_hi; ww += 32) {
          const int mm = net.wp_size[ww];
          if (mm < 2) continue;
          const uint64_t hw = fold(wpm, (uint64_t)ww);
          const uint64_t ha = fold(hw, 0), hb = fold(hw, 1);
          const uint2 sh = day_shifts(wsh, ww, mm);
          tab[2 * ww] = make_uint4((uint32_t)ha, (uint32_t)(ha >> 32), (uint32_t)hb, 0u);
          tab[2 * ww + 1] = make_uint4(sh.x, sh.y, 0u, 0u);
        }
      }
    } else {
    const uint16_t* codes = R.codes[par];
    uint16_t* codes_next = R.codes[par ^ 1];
    const WorkTables& W = R.wt[par];
    const WorkTables& Wn = R.wt[par ^ 1];
    unsigned edges = 0;
    double lam = 0.0;
    if (valid) {
      // rows of the day (level 1)
      const uint4* ri = (const uint4*)(W.rin + (size_t)b * RT_SLOTS);
      const uint4 in0 = LDM(ri), in1 = LDM(ri + 1);
      const bool rows = CROW && works;
      bool row_used = false;
      if (!code_dead(cb)) {
        const uint4* ro = (const uint4*)(out_s + threadIdx.x * RUN_OUT_STRIDE);
        const int nb = code_count(cb);
        const int nbe = nb < RT_SLOTS ? nb : RT_SLOTS;
        const uint4 o0 = nbe > 0 ? ro[0] : make_uint4(self, self, self, self);
        // level 2: every load of the day's sources before any sum
        uint16_t hc[HH], wio[2 * DR];
        if constexpr (CROW) {
          load_household<HH>(hc, hin ? hcode_s[par] + hl0 : codes + start, hmask);
          (void)wio;
        } else {
          // the 64-register variant: per-member in-block tests and per-draw
          // modular indices spill less (measured 2.44 vs 2.69 ms at 120 k agents)
          const uint16_t* hcs = hcode_s[par];
#pragma unroll
          for (int i = 0; i < HH; ++i)
            hc[i] = (i < sz && start + i != b)
                        ? ((unsigned)(hl0 + i) < (unsigned)nloc ? hcs[hl0 + i] : LDM(codes + start + i))
                        : (uint16_t)CODE_DEAD;
#pragma unroll
          for (int j = 0; j < DR; ++j) {
            wio[2 * j] = wio[2 * j + 1] = (uint16_t)CODE_DEAD;
            if (works && j < draws) {
              const uint32_t r = ((j < 4 ? shp.x : shp.y) >> (8 * (j & 3))) & 0xFFu;
              wio[2 * j] = LDM(W.wcode + base + add_mod(p, r, (uint32_t)m));
              wio[2 * j + 1] = LDM(W.wcode + base + sub_mod(p, r, (uint32_t)m));
            }
          }
        }
        const uint32_t po0[4] = {o0.x, o0.y, o0.z, o0.w};
        uint16_t co0[4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
          co0[q] = (q < nbe && po0[q] != self) ? LDM(codes + po0[q]) : (uint16_t)CODE_DEAD;
        // per-kind sums in the visit order of for_each_in_code
        float acc[3] = {0.f, 0.f, 0.f};
        add_src_group<HH>(acc[0], edges, T.factor, hc);
        for (int i = HH; i < sz; ++i) {
          if (i == off) continue;
          add_src(acc[0], edges, T.factor, LDM((hin ? hcode_s[par] + hl0 : codes + start) + i));
        }
        if (CROW) {
          if (works) {
            const uint4* cr = (const uint4*)(R.crow[par] + (size_t)(base + p) * 16);
            const uint4 cr0 = LDM(cr), cr1 = LDM(cr + 1);
            row_used = (cr0.x | cr0.y | cr0.z | cr0.w | cr1.x | cr1.y | cr1.z | cr1.w) != 0u;
            add_crow(acc[1], edges, T.factor, cr0, cr1, 2u * (unsigned)draws);
          }
        } else {
          add_src_group<2 * DR>(acc[1], edges, T.factor, wio);
        }
        if (n >= 2) {
          unsigned eo = 0;
          add_src_group<4>(acc[2], eo, T.factor, co0);
          for (int j0 = 4; j0 < nbe; j0 += 4) {
            const uint4 o = ro[j0 >> 2];
            const uint32_t po[4] = {o.x, o.y, o.z, o.w};
            uint16_t co[4];
#pragma unroll
            for (int q = 0; q < 4; ++q)
              co[q] = (j0 + q < nbe && po[q] != self) ? LDM(codes + po[q]) : (uint16_t)CODE_DEAD;
            add_src_group<4>(acc[2], eo, T.factor, co);
          }
          // random in-edges between alive agents total the random out-edges
          // (each is one (source, slot) pair seen from either end): counted as
          // twice the out-partners, so the rows may be sparse (infectious only)
          edges += 2u * eo;
          add_rin_row_sparse(acc[2], T.factor, in0, in1);
        }
        const float tot = acc[0] * T.bfac[0] + acc[1] * T.bfac[1] + acc[2] * T.bfac[2];
        if (h.stage == S_SUS && !(R.P->sterilizing && h.immune)) lam = (double)(tot * T.sfac[h.age]);
      }
      // the consumed row starts empty (it is written again two days on)
      // (only infectious in-partners write it: most rows are already empty)
      if ((in0.x | in0.y | in0.z | in0.w | in1.x | in1.y | in1.z | in1.w) != 0u) {
        uint4* rw = (uint4*)(W.rin + (size_t)b * RT_SLOTS);
        rw[0] = make_uint4(0, 0, 0, 0);
        rw[1] = make_uint4(0, 0, 0, 0);
      }
      // (so is the colleague row, also a dead agent's)
      if (rows && code_dead(cb)) {         // (a dead agent's row is read only to be cleared)
        const uint4* cr = (const uint4*)(R.crow[par] + (size_t)(base + p) * 16);
        const uint4 cr0 = LDM(cr), cr1 = LDM(cr + 1);
        row_used = (cr0.x | cr0.y | cr0.z | cr0.w | cr1.x | cr1.y | cr1.z | cr1.w) != 0u;
      }
      if (row_used) {
        uint4* cw = (uint4*)(R.crow[par] + (size_t)(base + p) * 16);
        cw[0] = make_uint4(0, 0, 0, 0);
        cw[1] = make_uint4(0, 0, 0, 0);
      }
    }
    unsigned ev = 0;
    if (valid) probe_lambda(R.probe, t, b, lam);
    if (valid) ev = transmit_progress_now(R.P, R.st, D.K, t, b, lam, h, pend);
    rec_events(rc, ev);
    rec_add(rc, EPI_REC_EDGES, edges);
    rec_agent(rc, valid, valid ? h.stage : 0, valid ? h.infected_at : 0);
    // tomorrow's code
    uint16_t cn = 0;
    if (valid) {
      cn = source_code(R.P, h.stage, h.infected_at, h.q_until, t + 1);
      if (h.stage == S_DEAD) cn |= CODE_DEAD;
      else cn |= (uint16_t)(cnt_nx << 8);
      codes_next[b] = cn;
      hcode_s[par ^ 1][threadIdx.x] = cn;
    }
    // tomorrow's push tables: the worker's position and its code there
    if (valid && works) {
      const uint32_t q = q_nx;
      Wn.wcode[base + q] = cn;
      p = q;
      if (d + 1 == R.n_days) {         // position and shift tables for the per-day path
        Wn.pos_of[base + loc] = (uint8_t)q;
        for (int j = loc; j < draws; j += m)
          Wn.shift[(size_t)w * draws + j] = (uint8_t)work_shift(D.wshift_next, w, j, m);
      } else if (CROW && (cn & 0x80FFu) != 0u) {
        push_rows(cn, q, shq, R.crow[par ^ 1]);   // tomorrow's colleague rows
      }
    }
    // random: flatten the warp's (agent, slot < n) items, 32 at a time
    {
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
      excl_s[warp][lane] = excl;
      cn_s[warp][lane] = cn;
      for (int i = 0; i < na; ++i) own_s[warp][excl + i] = (uint8_t)lane;   // item -> its agent's lane
      __syncwarp();
      const int64_t wbase_agent = b - lane;
      for (int k = lane; k < total; k += 32) {
        const int l = own_s[warp][k];
        const int j = k - excl_s[warp][l];
        const uint32_t src = (uint32_t)(wbase_agent + l);
        const uint32_t y = walk_fwd(src, D.rk_next[j], R.dn);
        out_s[(warp * 32 + l) * RUN_OUT_STRIDE + j] = y;
        if (d + 1 == R.n_days) Wn.rout[(size_t)src * RT_SLOTS + j] = y;
        // only infectious sources (code byte != 0) feed a lambda; the last
        // day's rows are complete (the per-day path counts their present bits)
        if (y != src && ((cn_s[warp][l] & 0xFF) != 0 || d + 1 == R.n_days))
          Wn.rin[(size_t)y * RT_SLOTS + j] = cn_s[warp][l] | CODE_PRESENT;
      }
    }
    cb = cn;
    }
    if (d + 1 < R.n_days) {
      // grid barrier, split: tomorrow's shifts (keys ready since the
      // service warp's day) are hashed between arrive and wait
      __syncthreads();
      if (threadIdx.x == 0) grid_arrive(R.barrier);
      if (pend >= 0) schedule_pending(R.P, R.st, D.K, t, R.tau_lut, b, pend, h);   // feeds tomorrow's check
      if (works) {
        if (d >= 1) {                      // computed by a service warp during day d - 1
          const uint4* e = R.wtab + (size_t)(d % 3) * 2 * net.n_workplaces + 2 * w;
          const uint4 e0 = LDM(e);
          if (!CROW) {
            const uint4 e1 = LDM(e + 1);
            shp = make_uint2(e1.x, e1.y);
          }
          q_nx = walk_inv((uint32_t)loc, work_keys_from(((uint64_t)e0.y << 32) | e0.x, e0.z), rm);
        } else {
          if (!CROW) shp = day_shifts(dk[(d + 1) & 1].wshift, w, m);
          q_nx = walk_inv((uint32_t)loc, work_keys(dk[(d + 1) & 1].wperm_next, w), rm);
        }
      }
      if (valid) cnt_nx = random_count_cdf(cdf_s, net.random_slots, dk[(d + 1) & 1].rcount_next, b);
      if (threadIdx.x == 0) grid_wait(R.barrier, (unsigned)(d + 1 + bar0) * gridDim.x);
      __syncthreads();
      if (CROW && works && d + 2 < R.n_days) {
        // the pushes of day d + 1 (rows of t + 2): the shifts of t + 2, written
        // during day d by the service warp of whichever block owns workplace w,
        // so read only after the barrier's wait (in the window, before it, a
        // slow block's entry could still be missing: an intermittent race)
        const uint4 e1 = LDM(R.wtab + (size_t)((d + 1) % 3) * 2 * net.n_workplaces + 2 * w + 1);
        shq = make_uint2(e1.x, e1.y);
      }
    } else if (pend >= 0) {
      schedule_pending(R.P, R.st, D.K, t, R.tau_lut, b, pend, h);
    }
  }
  __syncthreads();
  if (service)
    rec_flush_warp(racc[(R.n_days - 1) & 1], R.records + (size_t)(R.n_days - 1) * EPI_REC_LEN,
                   R.first_step + R.n_days - 1, nwa, lane);
  // the merged chain resumes at first + n_days: its kernel reads the
  // random-slot keys of the day after from the ring
  if (blockIdx.x == 0 && threadIdx.x < RT_SLOTS && R.ring_t2 != nullptr)
    R.ring_t2->rk[threadIdx.x] =
        random_slot_keys(key_prefix(R.seed, R.first_step + R.n_days + 1, P_NET_RPERM), threadIdx.x);
}

}  // namespace epi
