// Persistent intervention run: the fused intervention days of a config
// network (epi_sim_run, fused mode, whole population, push tables) in ONE
// launch, like k_fused_run for the days without interventions.  One block
// per SM, one thread per agent for the whole run, a service warp; the day's
// phases are separated by grid barriers instead of kernel boundaries:
//   0  the DEN follow-ups of yesterday's notifications (engine.py:244-262)
//   A  gather + transmission/progression + testing (k_fused_step + tests),
//      the vaccination eligibility (per-warp histograms -> the day's
//      histogram), dropout and due immunity checks, death days, tomorrow's
//      codes and push tables
//        | barrier 1 (notifier list, histogram, codes complete) [DEN or vaccination]
//   B  DEN regeneration: one warp per (notifier, past day) (k_den_regen)
//   C  vaccination plan (every warp derives it) + doses in id order, record
//        | barrier (end of day: the DEN marks are complete)
// The agent's static network data, own code and workplace position stay in
// registers; its state is reloaded at the start of each day (the later
// phases change it through the shared per-phase functions).  The same
// per-agent functions in the same order as the per-phase kernels: bitwise
// the same run (tests/test_gpu_persistent.py).
#pragma once

#include "epi_persistent.cuh"

namespace epi {

struct IvRunArgs {
  StepArgs A0;                    // P, st, flags, tau_lut (K and step are per day)
  uint64_t seed;
  int first_step, n_days;
  long long* records;             // [n_days][EPI_REC_LEN], zeroed
  uint16_t* codes[2];
  WorkTables wt[2];
  NetTables* ring_t2;
  const MsgTables* mt;
  const Radix* wrad;              // static workplace domains (DEN regeneration)
  Radix dn;
  unsigned* barrier;
  uint8_t* bucket;
  unsigned long long* hist;       // [3][NUM_BUCKETS + 1] by run day mod 3 (+ active count), zeroed
  unsigned* tile_hist;            // [2][blocks][NUM_BUCKETS] by run day parity
  int32_t* vax_open;
  int32_t* den_list;              // [2][den_stride] by day parity
  int* den_count;                 // [3] by run day mod 3 (day d's list length; zeroed at launch)
  int64_t den_stride;
  int32_t* died_at;
  int den_lookback;
  int den, tests, post, vax;      // phases present
  uint4* wtab;                    // [3][n_workplaces][2]: per-workplace keys, domain, shifts by run day mod 3
};

// Phase timeline (a build with -DEPI_IV_TRACE only, tools/iv_timeline.py):
// %globaltimer of thread 0 of every block at the day's phase boundaries.
#ifdef EPI_IV_TRACE
constexpr int IV_TRACE_DAYS = 200, IV_TRACE_BLOCKS = 160, IV_TRACE_PTS = 6;
__device__ unsigned long long g_iv_trace[IV_TRACE_DAYS][IV_TRACE_BLOCKS][IV_TRACE_PTS];
__device__ __forceinline__ void iv_mark(int d, int k) {
  if (threadIdx.x == 0 && d < IV_TRACE_DAYS && blockIdx.x < IV_TRACE_BLOCKS) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_iv_trace[d][blockIdx.x][k] = t;
  }
}
#else
__device__ __forceinline__ void iv_mark(int, int) {}
#endif

constexpr int IV_HIST = NUM_BUCKETS + 1;
constexpr int IV_HW_ROW = NUM_BUCKETS + 1;           // + the warp's active count
constexpr int IV_HW_WORDS = 2 * (RUN_MAX_THREADS / 32) * IV_HW_ROW;
constexpr size_t IV_DYN_SMEM = RUN_DYN_SMEM + IV_HW_WORDS * sizeof(unsigned);

// Phase 4b of day t - 1 for agent b, applied at the start of day t:
// notified (marked by a notifier's contact regeneration) and eligible then
// -> den_test_due_at = t with the compliance draw of day t - 1
// (engine.py:244-262); counted in day t - 1's record; the day's flags cleared.
__device__ __forceinline__ void den_follow_up(const IvRunArgs& R, int64_t b, bool valid, bool den_ok,
                                              uint64_t den_pref, int t, RecAcc& rc_prev) {
  unsigned notified = 0;
  if (valid) {
    const uint8_t fl = R.A0.flags[b];
    if (den_ok && (fl & FL_NOTIFIED)) {
      notified = 1;
      if (keyed_u(den_pref, (uint64_t)b, 0) < R.A0.P->den_compliance) R.A0.st.den_test_due_at[b] = t;
    }
    R.A0.flags[b] = 0;
  }
  rec_add(rc_prev, EPI_REC_NOTIFY, notified);
}

__global__ void __launch_bounds__(RUN_MAX_THREADS, 1) k_iv_run(IvRunArgs R, epi_net net) {
  constexpr int HH = 8, DR = 8;
  __shared__ MsgTables T;
  // record rows, keys and step arguments by run day mod 3: without DEN a day
  // has one grid barrier, and a warp still dosing day d must not see day d + 2's
  __shared__ RecAcc racc[3];
  __shared__ DayKeys dk[3];
  __shared__ StepArgs As[3];
  __shared__ Radix wrad[256];
  __shared__ PermKeys rk_w[RUN_MAX_THREADS / 32][RT_SLOTS];
  __shared__ int excl_s[RUN_MAX_THREADS / 32][32];
  __shared__ uint16_t cn_s[RUN_MAX_THREADS / 32][32];
  __shared__ uint8_t own_s[RUN_MAX_THREADS / 32][32 * RT_SLOTS];
  __shared__ uint16_t hcode_s[2][RUN_MAX_AGENTS];   // the block's codes by day parity
  __shared__ double cdf_s[EPI_MAX_SLOTS];           // the random-slot count CDF (per-lane indexed)
  extern __shared__ uint4 run_dyn_s[];
  uint32_t* const out_s = (uint32_t*)run_dyn_s;    // out-rows [agent][RUN_OUT_STRIDE] (as k_fused_run)
  // per-warp eligibility histograms by day parity [2][warps][NUM_BUCKETS + 1]:
  // the block's histogram is their sum, and a warp's rank offset in the cut
  // bucket is the sum over the warps before it (no block barrier for either)
  unsigned* const hw_s = (unsigned*)(out_s + (size_t)RUN_MAX_AGENTS * RUN_OUT_STRIDE);
  load_msg_tables(T, R.mt);
  if (threadIdx.x < EPI_MAX_SLOTS) cdf_s[threadIdx.x] = net.poisson_cdf[threadIdx.x];
  rec_init(racc[0]);
  rec_init(racc[1]);
  rec_init(racc[2]);
  for (int m = threadIdx.x; m < 256; m += blockDim.x) wrad[m] = R.wrad[m];
  for (int i = threadIdx.x; i < IV_HW_WORDS; i += blockDim.x) hw_s[i] = 0u;
  const int warp = threadIdx.x >> 5, lane = lane_id();
  const int nwa = (int)(blockDim.x >> 5) - 1;
  const bool service = warp == nwa;
  if (warp == 0) {
    day_keys(dk[0], R.seed, R.first_step, lane);
    __syncwarp();
    if (lane == 0) {
      As[0] = R.A0;
      As[0].K = dk[0].K;
      As[0].step = R.first_step;
    }
  }
  const int64_t n = net.n_agents;
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t blo = blockIdx.x * per;
  const int64_t bhi = blo + per < n ? blo + per : n;
  const int64_t b = blo + threadIdx.x;
  const bool valid = !service && b < bhi;
  const uint32_t self = (uint32_t)b;
  const int draws = net.colleague_draws;
  const epi_state& st = R.A0.st;
  int off = 0, sz = 0, w = -1, loc = 0, m = 0, base = 0;
  uint16_t cb = CODE_DEAD;
  uint32_t p = 0;
  if (valid) {
    off = net.hh_off[b];
    sz = net.hh_size[b];
    w = net.wp_id[b];
    loc = net.wp_local[b];
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
  const int hl0 = (int)threadIdx.x - off;  // household members inside the block: from hcode_s
  const int nloc = (int)(bhi - blo);
  const bool works = w >= 0 && m >= 2;
  const int64_t start = b - off;
  unsigned bar = 0;                        // barriers passed
  // DEN: whether the agent could be notified today (engine.py:253-256:
  // has the app, not quarantined, alive -- after today's test delivery,
  // before dropout) and today's compliance-draw key; the notification itself
  // is applied at the start of tomorrow, once every block's marks are in
  bool den_ok = false;
  uint64_t den_pref = 0;
  __syncthreads();
  uint2 shp = works ? day_shifts(dk[0].wshift, w, m) : make_uint2(0, 0);   // the day's colleague shifts
  // the agent's hot state for the coming day: only its own thread writes it,
  // so it is reloaded once the day's last write (doses, transition
  // scheduling) is done -- between the end barrier's arrive and wait
  AgentHot hp{};
  if (valid) hp = load_hot(st, b);
  for (int d = 0; d < R.n_days; ++d) {
    const int t = R.first_step + d;
    const int par = t & 1;
    const int d3 = d % 3, d3p = (d + 2) % 3, d3n = (d + 1) % 3;   // today, yesterday, tomorrow
    const DayKeys& D = dk[d3];
    const StepArgs& A = As[d3];
    RecAcc& rc = racc[d3];
    int pend = -1;                         // the day's deferred transition scheduling
    int age = 0;
    uint8_t bk = NO_BUCKET;                // the agent's vaccination bucket of the day
    unsigned long long* hist = R.hist + (size_t)d3 * IV_HIST;
    unsigned* tile_hist = R.tile_hist + (size_t)(d & 1) * gridDim.x * NUM_BUCKETS;
    const uint16_t* codes = R.codes[par];
    uint16_t* codes_next = R.codes[par ^ 1];
    const WorkTables& W = R.wt[par];
    const WorkTables& Wn = R.wt[par ^ 1];
    const int first_day = t - R.den_lookback > 0 ? t - R.den_lookback : 0;
    const int n_back = t - first_day;
    const bool phase_b = R.den && R.tests && n_back > 0;
    const bool bar1 = phase_b || R.vax;    // a grid barrier after phase A
    // tomorrow's code and push tables, at the end of phase A: final once the
    // agent's dropout has run; the later phases (DEN marks, doses) do not
    // change a code (a dose only turns code-0 susceptibles into code-0
    // vaccinated agents), so they are complete at barrier 1 and the DEN
    // regeneration after it overlaps nothing but the plan and the doses
    auto next_day = [&]() {
      uint16_t cn = 0;
      if (valid) {
        const int stage = st.stage[b];
        if (R.died_at && stage == S_DEAD && R.died_at[b] == INT32_MAX) R.died_at[b] = t;
        cn = source_code(A.P, stage, st.infected_at[b], st.quarantine_until[b], t + 1);
        if (stage == S_DEAD) cn |= CODE_DEAD;
        else cn |= (uint16_t)(random_count_cdf(cdf_s, net.random_slots, D.rcount_next, b) << 8);
        codes_next[b] = cn;
        hcode_s[par ^ 1][threadIdx.x] = cn;
      }
      if (valid && works) {
        uint32_t q;
        if (d >= 1) {                      // keys + domain by a service warp during day d - 1
          const uint4* e = R.wtab + (size_t)(d % 3) * 2 * net.n_workplaces + 2 * w;
          const uint4 e0 = LDM(e), e1 = LDM(e + 1);
          q = walk_inv((uint32_t)loc, work_keys_from(((uint64_t)e0.y << 32) | e0.x, e0.z),
                       Radix{e1.x & 0xFFu, (e1.x >> 8) & 0xFFu, (e1.x >> 16) & 0xFFu, e1.y});
        } else {
          q = walk_inv((uint32_t)loc, work_keys(D.wperm_next, w), make_radix((uint32_t)m));
        }
        Wn.wcode[base + q] = cn;
        p = q;
        if (d + 1 == R.n_days) {
          Wn.pos_of[base + loc] = (uint8_t)q;
          for (int j = loc; j < draws; j += m)
            Wn.shift[(size_t)w * draws + j] = (uint8_t)work_shift(D.wshift_next, w, j, m);
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
      excl_s[warp][lane] = excl;
      cn_s[warp][lane] = cn;
      for (int i = 0; i < na; ++i) own_s[warp][excl + i] = (uint8_t)lane;
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
      cb = cn;
    };
    if (R.den && d > 0) {
      // yesterday's exposure notifications (phase 4b of t - 1): the marks of
      // every block are complete since the barrier; counted in yesterday's
      // record, which the service warp flushes after barrier 1 (or after this)
      if (!service) den_follow_up(R, b, valid, den_ok, den_pref, t, racc[d3p]);
      if (!bar1) __syncthreads();
    }
    // ---- phase A ----------------------------------------------------------
    iv_mark(d, 0);
    // tomorrow's list length starts at 0: its last readers (day d - 2's phase
    // B) are done since barrier 1 of d - 1, and tomorrow's appends come after
    // today's barrier 1
    if (blockIdx.x == 0 && threadIdx.x == 0 && R.den_count) R.den_count[d3n] = 0;
    if (service) {
      if (d > 0 && !bar1)
        rec_flush_warp(racc[d3p], R.records + (size_t)(d - 1) * EPI_REC_LEN, t - 1, nwa, lane);
      if (d + 1 < R.n_days) {
        day_keys(dk[d3n], R.seed, t + 1, lane);
        __syncwarp();
        if (lane == 0) {
          As[d3n] = R.A0;
          As[d3n].K = dk[d3n].K;
          As[d3n].step = t + 1;
        }
        // tomorrow's per-workplace permutation keys (of t + 2) and domains,
        // and the colleague shifts of t + 2 (read in tomorrow's end-of-day
        // window), this block's share of the workplaces
        const uint64_t wpm = key_prefix(R.seed, t + 2, P_NET_WPERM);
        const uint64_t wsh = key_prefix(R.seed, t + 2, P_NET_WSHIFT);
        const int nW = net.n_workplaces;
        const int per_w = (nW + (int)gridDim.x - 1) / (int)gridDim.x;
        const int w_lo = (int)blockIdx.x * per_w, w_hi = w_lo + per_w < nW ? w_lo + per_w : nW;
        uint4* tab = R.wtab + (size_t)((d + 1) % 3) * 2 * nW;
        for (int ww = w_lo + lane; ww < w_hi; ww += 32) {
          const int mm = net.wp_size[ww];
          if (mm < 2) continue;
          const uint64_t hw = fold(wpm, (uint64_t)ww);
          const uint64_t ha = fold(hw, 0), hb = fold(hw, 1);
          const Radix rr = make_radix((uint32_t)mm);
          const uint2 sh = day_shifts(wsh, ww, mm);
          tab[2 * ww] = make_uint4((uint32_t)ha, (uint32_t)(ha >> 32), (uint32_t)hb, 0u);
          tab[2 * ww + 1] = make_uint4(rr.n | rr.a << 8 | rr.b << 16, rr.magic, sh.x, sh.y);   // (m <= 255)
        }
      }
    } else {
      AgentHot h = hp;
      age = h.age;
      unsigned edges = 0;
      double lam = 0.0;
      if (valid) {
        const uint4* ri = (const uint4*)(W.rin + (size_t)b * RT_SLOTS);
        const uint4 in0 = LDM(ri), in1 = LDM(ri + 1);
        if (!code_dead(cb)) {
          const uint4* ro = (const uint4*)(out_s + threadIdx.x * RUN_OUT_STRIDE);
          const int nb = code_count(cb);
          const int nbe = nb < RT_SLOTS ? nb : RT_SLOTS;
          const uint4 o0 = nbe > 0 ? ro[0] : make_uint4(self, self, self, self);
          const uint16_t* hcs = hcode_s[par];
          auto hh_code = [&](int i) -> uint16_t {
            return (unsigned)(hl0 + i) < (unsigned)nloc ? hcs[hl0 + i] : LDM(codes + start + i);
          };
          uint16_t hc[HH];
#pragma unroll
          for (int i = 0; i < HH; ++i)
            hc[i] = (i < sz && start + i != b) ? hh_code(i) : (uint16_t)CODE_DEAD;
          uint32_t sh[DR];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            sh[q] = (shp.x >> (8 * q)) & 0xFFu;
            sh[4 + q] = (shp.y >> (8 * q)) & 0xFFu;
          }
          const uint32_t po0[4] = {o0.x, o0.y, o0.z, o0.w};
          uint16_t co0[4];
#pragma unroll
          for (int q = 0; q < 4; ++q)
            co0[q] = (q < nbe && po0[q] != self) ? LDM(codes + po0[q]) : (uint16_t)CODE_DEAD;
          uint16_t wo[DR], wi[DR];
#pragma unroll
          for (int j = 0; j < DR; ++j) {
            wo[j] = wi[j] = (uint16_t)CODE_DEAD;
            if (works && j < draws) {
              const uint32_t r = sh[j];
              wo[j] = LDM(W.wcode + base + add_mod(p, r, (uint32_t)m));
              wi[j] = LDM(W.wcode + base + sub_mod(p, r, (uint32_t)m));
            }
          }
          float acc[3] = {0.f, 0.f, 0.f};
          add_src_group<HH>(acc[0], edges, T.factor, hc);
          for (int i = HH; i < sz; ++i) {
            if (start + i == b) continue;
            add_src(acc[0], edges, T.factor, hh_code(i));
          }
          uint16_t wio[2 * DR];                 // visit order: out, in per draw
#pragma unroll
          for (int j = 0; j < DR; ++j) {
            wio[2 * j] = wo[j];
            wio[2 * j + 1] = wi[j];
          }
          add_src_group<2 * DR>(acc[1], edges, T.factor, wio);
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
          if (h.stage == S_SUS && !(A.P->sterilizing && h.immune)) lam = (double)(tot * T.sfac[h.age]);
        }
        // (only infectious in-partners write it: most rows are already empty)
        if ((in0.x | in0.y | in0.z | in0.w | in1.x | in1.y | in1.z | in1.w) != 0u) {
          uint4* rw = (uint4*)(W.rin + (size_t)b * RT_SLOTS);
          rw[0] = make_uint4(0, 0, 0, 0);
          rw[1] = make_uint4(0, 0, 0, 0);
        }
      }
      unsigned ev = 0;
      if (valid) probe_lambda(R.A0.probe, t, b, lam);
      if (valid) ev = transmit_progress_now(A.P, st, A.K, t, b, lam, h, pend);
      unsigned tested = 0;
      if (R.tests) {
        if (valid) {
          uint8_t fl = (ev & 8u) ? FL_SYMPTOMATIC : A.flags[b];
          tested = test_agent(A, b, h.stage, fl, R.den ? R.den_list + (size_t)par * R.den_stride : nullptr,
                              R.den_count ? R.den_count + d3 : nullptr);
          A.flags[b] = fl;
        }
        if (R.den) {
          den_ok = valid && st.has_den_app[b] && st.quarantine_until[b] <= t && h.stage != S_DEAD;
          den_pref = A.K.p[P_DEN];
        }
        rec_add(rc, EPI_REC_TESTS, tested);
      } else if (valid && (ev & 8u)) {
        A.flags[b] = FL_SYMPTOMATIC;
      }
      rec_events(rc, ev);
      rec_add(rc, EPI_REC_EDGES, edges);
      // the vaccination eligibility of the day (bucket + active count,
      // engine.py:286-302), here in phase A: none of the phases between
      // (test delivery, DEN follow-ups, dropout, immunity realisation) changes
      // a stage's active / blocked class, a vaccine status or a dose date, so
      // the histogram is complete at the first barrier of the day
      if (R.vax) {
        unsigned active = 0;
        if (valid) bk = iv_elig_agent(A, b, hw_s + ((size_t)par * (RUN_MAX_THREADS / 32) + warp) * IV_HW_ROW, active);
        rec_add(rc, EPI_REC_ACTIVE, active);
        const unsigned wa = __reduce_add_sync(0xFFFFFFFFu, active);
        if (lane == 0) hw_s[((size_t)par * (RUN_MAX_THREADS / 32) + warp) * IV_HW_ROW + NUM_BUCKETS] = wa;
      }
      // dropout and due immunity checks (independent of the plan), then
      // tomorrow's code and push tables
      if (R.post && valid) iv_post_rest_agent(A, b, false);
      next_day();
    }
    iv_mark(d, 1);
    if (R.vax) {
      // the block's histogram to the day's histogram and to its tile row
      __syncthreads();
      // (and the block's active count: one atomic per block)
      const unsigned* hw = hw_s + (size_t)par * (RUN_MAX_THREADS / 32) * IV_HW_ROW;
      unsigned* hw_next = hw_s + (size_t)(par ^ 1) * (RUN_MAX_THREADS / 32) * IV_HW_ROW;
      // (one warp per bucket: lane w holds warp w's row entry, one warp sum)
      for (int i = warp; i < IV_HW_ROW; i += nwa + 1) {
        unsigned v = 0;
        for (int ww = lane; ww < nwa; ww += 32) v += hw[ww * IV_HW_ROW + i];
        v = __reduce_add_sync(0xFFFFFFFFu, v);
        if (lane == 0) {
          if (i < NUM_BUCKETS) tile_hist[(size_t)blockIdx.x * NUM_BUCKETS + i] = v;
          if (v) atomicAdd(&hist[i], (unsigned long long)v);
        }
      }
      // tomorrow's rows start empty (yesterday's doses, their last reader, are done)
      for (int i = threadIdx.x; i < (RUN_MAX_THREADS / 32) * IV_HW_ROW; i += blockDim.x) hw_next[i] = 0u;
    }
    // ---- phase B: DEN regeneration ----------------------------------------
    // barrier 1: the notifier list and the eligibility histogram are complete
    if (bar1) {
      grid_barrier(R.barrier, ++bar * gridDim.x);
      iv_mark(d, 2);
      if (service && d > 0)               // yesterday's record (incl. this morning's follow-ups)
        rec_flush_warp(racc[d3p], R.records + (size_t)(d - 1) * EPI_REC_LEN, t - 1, nwa, lane);
    }
    // the day's notifier count (complete at barrier 1, the same in every block):
    // a day without notifiers makes no DEN marks and needs no end barrier
    const int den_items = phase_b ? LDM(R.den_count + d3) : 0;
    if (den_items > 0) {
      if (!service) {
        const int64_t items = (int64_t)den_items * n_back;
        const int32_t* list = R.den_list + (size_t)par * R.den_stride;
        // items spread over the blocks first (a few hundred items: one per
        // block and warp, so no block carries more than its share)
        const int64_t gw = (int64_t)warp * gridDim.x + blockIdx.x, warps = (int64_t)gridDim.x * nwa;
        for (int64_t it = gw; it < items; it += warps) {
          const int dd = (int)(it % n_back);
          const int day = first_day + dd;
          den_regen_item(net, make_net_keys(R.seed, day), day, LDM(list + it / n_back), rk_w[warp], wrad,
                         R.died_at, A.flags, lane);
        }
      }
      // no barrier: nothing until tomorrow reads the marks (see den_ok)
    }
    iv_mark(d, 3);
    // ---- phase C: the vaccination plan (every warp derives it from the
    // complete histogram) and the doses in id order -------------------------
    // the vaccination plan (every warp derives it from the complete
    // histogram, barrier 1) and the doses in id order; the day's record rows.
    // Thread-local writes only: with DEN in the end barrier's window, else
    // right after barrier 1
    auto finish_day = [&]() {
      // the record's stage and infection day: loaded first, so their latency
      // overlaps the plan's (reloaded after a dose, whose immunity may be
      // realised at once with a zero latency)
      bool dosed = false;
      int stage = 0;
      int32_t inf = 0;
      if (valid) {
        stage = st.stage[b];
        inf = st.infected_at[b];
      }
      if (R.vax) {
        // the plan (k_vax_plan), derived by every warp from the complete
        // histogram (no block barrier): lane l holds buckets 2l, 2l+1; the cut
        // bucket is the first whose inclusive prefix reaches the budget
        const epi_params* __restrict__ P = A.P;
        const long long c0 = lane < NUM_BUCKETS / 2 ? (long long)LDM(hist + 2 * lane) : 0;
        const long long c1 = lane < NUM_BUCKETS / 2 ? (long long)LDM(hist + 2 * lane + 1) : 0;
        int open = *R.vax_open;
        if (!open && (double)LDM(hist + NUM_BUCKETS) >= P->start_trigger_count) open = 1;
        long long cut = -1, rem = 0, doses = -1;
        const long long budget = P->dose_budget;
        if (open && budget > 0) {
          const long long pair = c0 + c1;
          long long S = pair;
  #pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const long long v = __shfl_up_sync(0xFFFFFFFFu, S, o);
            if (lane >= o) S += v;
          }
          const unsigned ball = __ballot_sync(0xFFFFFFFFu, S >= budget);
          if (ball) {
            const int L = __ffs(ball) - 1;
            const long long E = __shfl_sync(0xFFFFFFFFu, S - pair, L);
            const long long cA = __shfl_sync(0xFFFFFFFFu, c0, L);
            if (E + cA >= budget) { cut = 2 * L; rem = budget - E; }
            else { cut = 2 * L + 1; rem = budget - E - cA; }
            doses = budget;
          } else {
            cut = NUM_BUCKETS;                // everyone eligible gets a dose
            doses = __shfl_sync(0xFFFFFFFFu, S, 31);
          }
        }
        if (blockIdx.x == 0 && warp == 0 && lane == 0) {
          *R.vax_open = open;                 // the latch only opens: a late reader derives the same
          if (doses > 0) rc.v[0][EPI_REC_DOSES] += (unsigned)doses;
        }
        // cut-bucket rank of each agent in id order: the blocks before (their
        // tile rows), the warps before (their histogram rows), the lanes before
        const bool in_cut = cut >= 0 && cut < NUM_BUCKETS && bk == (uint8_t)cut;
        if (cut >= 0 && cut < NUM_BUCKETS && !service) {
          const unsigned ball = __ballot_sync(0xFFFFFFFFu, in_cut);
          // (the blocks' tile rows: every load issued before the first add)
          unsigned part = 0;
          if (blockIdx.x <= 256) {
            unsigned v[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const int bb = lane + 32 * k;
              v[k] = bb < (int)blockIdx.x ? LDM(tile_hist + (size_t)bb * NUM_BUCKETS + cut) : 0u;
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) part += v[k];
          } else {
            for (int bb = lane; bb < (int)blockIdx.x; bb += 32) part += LDM(tile_hist + (size_t)bb * NUM_BUCKETS + cut);
          }
          if (lane < warp) part += hw_s[((size_t)par * (RUN_MAX_THREADS / 32) + lane) * IV_HW_ROW + cut];
          const long long rank = (long long)__reduce_add_sync(0xFFFFFFFFu, part) + __popc(ball & ((1u << lane) - 1u));
          if (valid && bk != NO_BUCKET && ((long long)bk < cut || (in_cut && rank < rem))) { give_dose(A, b, bk); dosed = true; }
        } else if (valid && cut >= 0 && bk != NO_BUCKET) {
          give_dose(A, b, bk);                // cut == NUM_BUCKETS: every eligible agent
          dosed = true;
        }
        if (dosed) {
          stage = st.stage[b];
          inf = st.infected_at[b];
        }
      }
      if (valid && !R.den) A.flags[b] = 0;   // (with DEN: cleared by tomorrow's follow-up)
      rec_agent(rc, valid, stage, inf);
    };
    if (R.vax && blockIdx.x == 0)           // the histogram of day d + 2 starts empty
      for (int i = threadIdx.x; i < IV_HIST; i += blockDim.x) R.hist[(size_t)d3p * IV_HIST + i] = 0;
    // end of day: a grid barrier when DEN marks were made today (tomorrow's
    // follow-ups read them) or when there was no barrier 1 (tomorrow's codes)
    const bool end_bar = d + 1 < R.n_days && (den_items > 0 || !bar1);
    if (end_bar) {
      // end of day, split: the plan, the doses and tomorrow's shifts between
      // arrive and wait
      __syncthreads();
      if (threadIdx.x == 0) grid_arrive(R.barrier);
      if (!service) finish_day();
      if (pend >= 0) {                     // feeds tomorrow's transition check
        AgentHot hs{};
        hs.age = age;
        schedule_pending(A.P, st, A.K, t, A.tau_lut, b, pend, hs);
      }
      if (works) {
        if (d >= 1) {                      // (written during day d - 1 with the keys)
          const uint4 e1 = LDM(R.wtab + (size_t)(d % 3) * 2 * net.n_workplaces + 2 * w + 1);
          shp = make_uint2(e1.z, e1.w);
        } else {
          shp = day_shifts(dk[d3n].wshift, w, m);
        }
      }
      if (valid) hp = load_hot(st, b);
      iv_mark(d, 4);
      ++bar;
      if (threadIdx.x == 0) grid_wait(R.barrier, bar * gridDim.x);
      __syncthreads();
      iv_mark(d, 5);
    } else {
      if (!service) finish_day();
      if (pend >= 0) {
        AgentHot hs{};
        hs.age = age;
        schedule_pending(A.P, st, A.K, t, A.tau_lut, b, pend, hs);
      }
      if (d + 1 < R.n_days && works) {
        if (d >= 1) {
          const uint4 e1 = LDM(R.wtab + (size_t)(d % 3) * 2 * net.n_workplaces + 2 * w + 1);
          shp = make_uint2(e1.z, e1.w);
        } else {
          shp = day_shifts(dk[d3n].wshift, w, m);
        }
      }
      if (d + 1 < R.n_days && valid) hp = load_hot(st, b);
      iv_mark(d, 4);
    }
  }
  if (R.den) {
    // the last day's notifications, once every block's marks are in
    grid_barrier(R.barrier, ++bar * gridDim.x);
    if (!service)
      den_follow_up(R, b, valid, den_ok, den_pref, R.first_step + R.n_days, racc[(R.n_days - 1) % 3]);
    if (blockIdx.x == 0 && threadIdx.x == 0 && R.den_count) R.den_count[0] = R.den_count[1] = R.den_count[2] = 0;
  }
  __syncthreads();
  if (service)
    rec_flush_warp(racc[(R.n_days - 1) % 3], R.records + (size_t)(R.n_days - 1) * EPI_REC_LEN,
                   R.first_step + R.n_days - 1, nwa, lane);
  if (blockIdx.x == 0 && threadIdx.x < RT_SLOTS && R.ring_t2 != nullptr)
    R.ring_t2->rk[threadIdx.x] =
        random_slot_keys(key_prefix(R.seed, R.first_step + R.n_days + 1, P_NET_RPERM), threadIdx.x);
}

}  // namespace epi
