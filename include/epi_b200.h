/*
 * epi_b200.h — C ABI of the B200-native DeepABM-COVID step (libepib200.so).
 *
 * Plain pointers and sizes only (no torch / C++ types).  Every device pointer
 * is caller-owned CUDA memory; a context owns parameter tables and scratch.
 * Calls are asynchronous on the given stream (`void*` = cudaStream_t, NULL =
 * legacy default stream) unless documented otherwise.
 *
 * The reference has no FFI: its interface for this path is the Python object
 * API.  Each entry point below names the reference function it replaces
 * (paths relative to /root/reference/pkg/src/epivec/):
 *
 *   epi_uniforms          rng.uniforms                     rng.py:92-100
 *   epi_graph_load        Engine.step validation + the
 *                         canonical lexsort of gather      engine.py:124-133, 98
 *   epi_gather            Engine.gather_exposure           engine.py:77-117
 *   epi_step              Engine.step (all phases)         engine.py:121-347
 *   epi_net_realize       GraphRealizer.realize            graphs.py:200-240
 *   epi_sim_step          runner loop body realize+step    runner.py:145-152
 *   epi_read_flags        check_invariants / errors        state.py:90-102
 *
 * Return codes: 0 ok; -1 bad argument (ConfigError); -2 invariant
 * (InvariantViolation); -3 CUDA/NCCL error.  epi_last_error() gives the text.
 */
#ifndef EPI_B200_H
#define EPI_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EPI_OK 0
#define EPI_EARG (-1)
#define EPI_EINVARIANT (-2)
#define EPI_ECUDA (-3)

#define EPI_MAX_T 127          /* day-weight table length - 1 (7-bit code)   */
#define EPI_MAX_SPECS 16       /* distinct duration distributions            */
#define EPI_MAX_TAUS 512       /* delay thresholds per distribution          */
#define EPI_MAX_SLOTS 32       /* random-network slots / colleague draws     */

/* Per-step record written by the device (int64 each), see DESIGN.md §4. */
#define EPI_REC_STEP 0
#define EPI_REC_STAGE0 1        /* 11 stage counts: 1..11                     */
#define EPI_REC_CUM_INF 12
#define EPI_REC_CUM_DEATHS 13
#define EPI_REC_IN_CARE 14
#define EPI_REC_NEW_INF 15
#define EPI_REC_TESTS 16
#define EPI_REC_DOSES 17
#define EPI_REC_NOTIFY 18
#define EPI_REC_EDGES 19
#define EPI_REC_DEATHS 20
#define EPI_REC_HOSP 21
#define EPI_REC_ACTIVE 22
#define EPI_REC_FLAGS 23        /* invariant bits, see EPI_FLAG_*            */
#define EPI_REC_LEN 24

#define EPI_FLAG_INDEX 1        /* graph references agent >= n_agents        */
#define EPI_FLAG_SELFLOOP 2
#define EPI_FLAG_KIND 4
#define EPI_FLAG_STAGE_RANGE 8
#define EPI_FLAG_NO_TIMESTAMP 16
#define EPI_FLAG_NEG_HAZARD 32

/* Precision of the message pass. */
#define EPI_F32 0               /* factored per-source message, fp32 sums    */
#define EPI_F64_CANONICAL 1     /* bitwise reference order (dst, src, kind)  */

/* Model parameters, flattened from DiseaseParams / ProgressionTable /
 * InterventionConfig (transmission.py:71-104, progression.py:99-216,
 * interventions.py:84-204). */
typedef struct epi_params {
    double rate_scale;
    double asymptomatic_factor;
    double mean_daily_interactions;
    double age_susceptibility[9];
    double network_scale[3];
    int32_t t_max;
    int32_t sterilizing;
    double day_weights[EPI_MAX_T + 1];
    /* progression: per stage, up to 3 branches */
    int32_t n_targets[11];
    int32_t targets[11][3];
    int32_t spec_of[11][3];
    double cum[11][9][3];
    int32_t n_specs;
    int32_t tau_len[EPI_MAX_SPECS];
    double tau[EPI_MAX_SPECS][EPI_MAX_TAUS];
    /* interventions */
    int32_t quarantine_enabled;
    int32_t quarantine_duration;
    double quarantine_dropout;
    int32_t testing_enabled;
    int32_t turnaround_min;
    int32_t turnaround_max;
    int32_t den_enabled;
    double detection_prob;
    double false_positive_prob;
    double den_compliance;
    int32_t den_lookback;
    int32_t vaccination_enabled;
    int32_t strategy;
    int32_t elderly_band;
    double dose1_efficacy;
    double dose2_efficacy;
    double dose2_topup;
    int32_t dose1_latency;
    int32_t dose2_latency;
    int32_t dose_gap;
    int32_t _pad0;
    int64_t dose_budget;          /* rint(daily_rate * N)                  */
    double start_trigger_count;   /* start_trigger * N (float64, as ref)   */
} epi_params;

/* Device SoA columns, same dtypes as AgentColumns (state.py:21-75). */
typedef struct epi_state {
    int64_t n_agents;
    int8_t *age_band;
    int8_t *stage;
    int32_t *infected_at;
    int32_t *next_transition_at;
    int8_t *next_stage;
    int32_t *quarantine_until;
    int32_t *quarantine_started_at;
    uint8_t *has_den_app;
    int8_t *vaccine_status;
    int32_t *dose1_at;
    int32_t *dose2_at;
    uint8_t *immune;
    int32_t *immunity_check_at;
    double *immunity_check_prob;
    int8_t *immunity_check_dose;
    int32_t *test_sample_at;
    int32_t *test_result_at;
    uint8_t *test_positive;
    int32_t *den_test_due_at;
} epi_state;

/* Static config-network layout (paper_2110_04421_b200/confignet.py). */
typedef struct epi_net {
    int64_t n_agents;
    const uint8_t *hh_off;
    const uint8_t *hh_size;
    const int32_t *wp_id;
    const uint8_t *wp_local;
    const int32_t *wp_base;
    const int32_t *wp_size;
    const int32_t *wp_members;
    int32_t n_workplaces;
    int32_t colleague_draws;
    int32_t random_slots;
    int32_t row_cap;              /* padded CSR row capacity              */
    int64_t n_member_slots;       /* length of wp_members                 */
    double poisson_cdf[EPI_MAX_SLOTS];
} epi_net;

/* Config-population synthesis on the device (row f3; host restatement:
 * paper_2110_04421_b200/confignet.py::synthesize).  Cumulative tables are
 * computed by the caller in fp64 (np.cumsum) so both sides compare against
 * the same doubles. */
typedef struct epi_pop_spec {
    int64_t n_agents;
    double age_cum[9];
    int32_t n_sizes;              /* household size classes (<= 32)       */
    int32_t hh_sizes[32];
    double hh_cum[32];
    uint32_t worker_mask;         /* bit b: age band b works (0: no workplaces) */
    int32_t wp_min, wp_max;
    int64_t n_seeds;
} epi_pop_spec;

/* Caller-owned device outputs.  wp_members/wp_base/wp_size hold the first
 * counts[1] / counts[0] entries; capacities: N, N / wp_min + 2. */
typedef struct epi_pop_out {
    int8_t *age_band;
    int32_t *household_id;
    uint8_t *hh_off, *hh_size;
    int32_t *wp_id;
    uint8_t *wp_local;
    int32_t *wp_members;
    int32_t *wp_base, *wp_size;
    int64_t *seeds;               /* [n_seeds], ascending ids             */
    int64_t *counts;              /* device [2]: workplaces, members      */
} epi_pop_out;

int epi_pop_synthesize(const epi_pop_spec *spec, uint64_t seed, const epi_pop_out *out, void *stream);

typedef struct epi_ctx epi_ctx;

/* Context: parameters + scratch for `n_agents` agents. */
int epi_create(const epi_params *params, int64_t n_agents, epi_ctx **out);
int epi_destroy(epi_ctx *ctx);
int epi_set_params(epi_ctx *ctx, const epi_params *params);
/* Restrict the config-simulation kernels to the owned agent rows [lo, hi)
 * (agent-range partition; state/code buffers stay globally indexed). */
int epi_set_rows(epi_ctx *ctx, int64_t lo, int64_t hi);
const char *epi_last_error(void);
int epi_version(void);
/* sizeof of the ABI structs (0 params, 1 state, 2 net) for binding checks */
int64_t epi_struct_size(int32_t which);

/* Keyed uniforms u(seed, step, purpose, ids[i], k) -> out[i] (device).
 * ids == NULL means ids[i] = i.  Replaces rng.uniforms (rng.py:92-100). */
int epi_uniforms(uint64_t seed, int32_t step, int32_t purpose, const int64_t *ids,
                 int64_t n, int32_t k, double *out, void *stream);

/* Graph-in mode: COO (src, dst, kind) device arrays -> canonical CSR kept in
 * the context.  Index range / self-loop / kind are checked on the device and
 * reported through epi_read_flags (engine.py:124-133). */
int epi_graph_load(epi_ctx *ctx, const int32_t *src, const int32_t *dst,
                   const int8_t *kind, int64_t n_edges, void *stream);

/* epi_graph_load for a device-side producer: the first *count (device
 * uint64) of the `capacity` entries are the edges; no host synchronisation
 * (the rest of the buffer is ignored).  Not with exposure notification (the
 * contact log needs the host count). */
int epi_graph_load_counted(epi_ctx *ctx, const int32_t *src, const int32_t *dst,
                           const int8_t *kind, const uint64_t *count, int64_t capacity,
                           void *stream);

/* Hazard per agent over the loaded graph at `step` (engine.py:77-117).
 * precision EPI_F64_CANONICAL writes double[N] bitwise equal to the
 * reference; EPI_F32 writes float[N]. */
int epi_gather(epi_ctx *ctx, const epi_state *st, int32_t step, int32_t precision,
               void *lambda_out, void *stream);

/* One full Engine.step over the loaded graph (engine.py:121-151): gather
 * (fp64 canonical), transmission, progression, enabled intervention phases,
 * contact-log push, invariant flags.  `record` = device int64[EPI_REC_LEN],
 * zeroed and filled.  `vax_open` = device int32 latch (engine.vaccination_open).
 * `injected` = NULL or 12 nullable device double[N] arrays indexed by
 * Purpose (1..11) that replace the keyed draws. */
int epi_step(epi_ctx *ctx, const epi_state *st, int32_t step, uint64_t seed,
             int64_t *record, int32_t *vax_open, const double *const *injected,
             int32_t check_invariants, void *stream);

/* Apply update phases (transmission..vaccination) with an externally supplied
 * hazard (double[N]) — for injected-draw parity tests. */
int epi_step_with_hazard(epi_ctx *ctx, const epi_state *st, int32_t step, uint64_t seed,
                         const double *hazard, int64_t *record, int32_t *vax_open,
                         const double *const *injected, void *stream);

/* Host read of the invariant bits accumulated by the last graph_load/step
 * (synchronises the stream), then clears them. */
int epi_read_flags(epi_ctx *ctx, int32_t *flags_out, void *stream);

/* ---- config networks (BASELINE.json configs 0-4) ---------------------- */

/* Per-agent 16-bit source code for `step` from the state: days since
 * infection (7 bits) | asymptomatic-like << 7 | random-slot count << 8 |
 * dead << 15 (count uses `net`, may be NULL).  Output uint16[N]. */
int epi_codes(epi_ctx *ctx, const epi_state *st, const epi_net *net, uint64_t graph_seed,
              int32_t step, uint16_t *codes_out, void *stream);

/* Materialise step `step`'s in-edges as a padded dst-major CSR:
 * entries[b*row_cap + i] = src << 2 | kind, i < row_len[b].  sort_rows = 1
 * puts every row in canonical (src, kind) order.  Replaces
 * GraphRealizer.realize (graphs.py:200-240) for the config networks. */
int epi_net_realize(const epi_net *net, uint64_t graph_seed, int32_t step,
                    const uint16_t *codes, uint32_t *entries, int32_t *row_len,
                    int32_t sort_rows, void *stream);

/* L2 residency for the day's random gathers (no reference counterpart:
 * device tuning).  `base`/`bytes` = the source-code buffers of a simulation;
 * the step kernels launch with a persisting L2 access-policy window over it
 * (hit ratio = persisting carve-out / window).  bytes = 0 clears it. */
int epi_set_hot_window(epi_ctx *ctx, const void *base, int64_t bytes);

/* Infection decision of epi_step (graph-in, fp64 canonical): one aggregate
 * draw against 1 - exp(-sum of hazards) (Engine, engine.py:153-175), or one
 * Bernoulli per incident edge with keyed INFECTION_EDGE draws k = j over the
 * nonzero contributions in (src, kind) order (the reference oracle's
 * independent-edges mode, oracle.py:185-192; validation only). */
#define EPI_INFECT_AGGREGATE 0
#define EPI_INFECT_INDEPENDENT 1
int epi_set_infection_mode(epi_ctx *ctx, int32_t mode);

/* Cross-rank exchange of a partitioned run (agent ranges, SURVEY §8(e) and
 * §8(f) row f2), called synchronously from inside epi_sim_step on `stream`;
 * returns 0 on success.  Kinds:
 *   EPI_X_GATHER_U8  all-gather: every rank's owned range [lo, hi) of the
 *                    global-indexed byte array `buf` (count = N) to all
 *                    ranks (the DEN notifier flags);
 *   EPI_X_SUM_U64    all-reduce sum of `count` uint64 (the vaccination
 *                    eligibility histogram + active count);
 *   EPI_X_EXSCAN_I64 exclusive prefix sum over the ranks, in rank (= id)
 *                    order, of `count` int64, in place (the cut-bucket offset);
 *   EPI_X_OR_U8      all-reduce bitwise OR of `count` bytes (the DEN
 *                    notifications each rank pushed to anyone's contacts). */
#define EPI_X_GATHER_U8 1
#define EPI_X_SUM_U64 2
#define EPI_X_EXSCAN_I64 3
#define EPI_X_OR_U8 4
#define EPI_X_GATHER_U16 5   /* the per-day code all-gather (epi_set_code_exchange mode 1):
                                buf = the uint16 code vector (world * count entries), every
                                rank's chunk [rank * count, (rank + 1) * count) to every rank */
typedef int (*epi_exchange_fn)(void *user, int32_t kind, void *buf, int64_t count, void *stream);
int epi_set_exchange(epi_ctx *ctx, epi_exchange_fn fn, void *user);

/* Whole-population runs build the random-slot push tables (96 B/agent) only
 * up to `max_agents` agents (-1 = while they fit in L2). */
int epi_set_push_max(epi_ctx *ctx, int64_t max_agents);

/* Beyond the push tables, whole-population fused days without interventions
 * push only infectious sources into sparse in-rows (32 B/agent, in HBM)
 * instead of evaluating the 16 inverse slot bijections per agent (default
 * on; bitwise the same records either way). */
int epi_set_sparse_push(epi_ctx *ctx, int32_t on);

/* ---- Agent-range partitions over NCCL (SURVEY §8(b) abm_allgather_codes,
 * §8(e)).  No reference counterpart: the reference runs one process per
 * replication (runner.py:164-190) and never partitions a population.
 *
 * Rank 0 calls epi_comm_unique_id, ships the 128 bytes to its peers (any
 * channel: torch.distributed here), every rank calls epi_comm_create with its
 * rank on its current CUDA device (ncclCommInitRank; NCCL is opened at run
 * time from libnccl.so.2, the one torch already loaded when present).
 * epi_set_code_exchange(ctx, comm, 2, chunk) makes every day of
 * epi_sim_step / epi_sim_run end with an in-place all-gather of the code
 * vector (chunk codes per rank, ranks own rows [rank * chunk, ...)); mode 1
 * routes the same exchange through the epi_set_exchange callback
 * (EPI_X_GATHER_U16; emulated ranks in tests), mode 0 leaves it to the
 * caller.  With NCCL the whole partitioned run can be captured in a CUDA
 * graph.  epi_allgather_codes runs the exchange once (the day-0 codes). */
typedef struct epi_comm epi_comm;
int epi_comm_unique_id(uint8_t *out128);
int epi_comm_create(const uint8_t *id128, int32_t world, int32_t rank, epi_comm **out);
int epi_comm_destroy(epi_comm *comm);
int epi_set_code_exchange(epi_ctx *ctx, epi_comm *comm, int32_t mode, int64_t chunk);
int epi_allgather_codes(epi_ctx *ctx, uint16_t *codes, void *stream);

/* Fused days without push tables (partitioned ranks, populations above the
 * push-table cut-off): build tomorrow's code-independent workplace tables on a
 * side stream while today's day kernel and the code exchange run (default on;
 * results are identical either way). */
int epi_set_sigma_ahead(epi_ctx *ctx, int32_t on);

/* Debug export of the hazard the step kernels consume (test hook for the
 * timed fp32 paths: k_fused_step, k_fused_run, k_iv_run, k_msg_pass<1>).
 * While set, every step kernel of day t in [first_step, first_step + n_days)
 * writes its agents' fp32 lambda -- the value fed to p = 1 - exp(-lambda),
 * engine.py:157-161 -- to out[(t - first_step) * n_agents + agent]; 0 for
 * non-targets (engine.py:109, 112-117).  `out` is a caller-owned device buffer
 * of n_days * n_agents floats.  n_days = 0 turns the export off. */
int epi_set_lambda_probe(epi_ctx *ctx, float *out, int32_t first_step, int32_t n_days);

/* Bind a config network to the context and allocate its per-step padded CSR
 * (a ring of den_lookback slots when exposure notification is enabled). */
int epi_net_attach(epi_ctx *ctx, const epi_net *net);

/* Fast path: one simulated day on the attached network, state resident on
 * the device.  mode 0 = generate the CSR, then the fused message-pass+update
 * kernel; mode 1 = fused generate+gather+update (no CSR in memory; no DEN).
 * codes_cur holds this step's codes (see epi_codes), codes_next receives the
 * next step's.  `record` as epi_step. */
int epi_sim_step(epi_ctx *ctx, const epi_state *st, int32_t step, uint64_t seed,
                 int32_t mode, int32_t precision, const uint16_t *codes_cur,
                 uint16_t *codes_next, int64_t *record, int32_t *vax_open, void *stream);

/* Days [first_step, first_step + n_days) in one call: codes0 / codes1 are
 * the codes of even / odd days, records is int64[n_days][EPI_REC_LEN]
 * (zeroed here).  Same kernels as epi_sim_step. */
int epi_sim_run(epi_ctx *ctx, const epi_state *st, int32_t first_step, int32_t n_days,
                uint64_t seed, int32_t mode, int32_t precision, uint16_t *codes0,
                uint16_t *codes1, int64_t *records, int32_t *vax_open, void *stream);

/* epi_sim_run sends the days after the first of a fused run (mode 1, fp32,
 * whole population, push tables, N <= 148 x 704) to one persistent launch:
 * k_fused_run without interventions, k_iv_run with them (one resident thread
 * per agent, grid barriers between a day's phases; intervention days need
 * epi_set_iv_fusion on); bitwise the same results as the per-day kernels.
 * on = 0 forces the per-day kernels. */
int epi_set_persistent(epi_ctx *ctx, int32_t on);
/* Replication summary (runner.py:195-207 `summarize`): quartiles q25/q50/q75
 * across n_rep replications (any count), bitwise np.percentile (linear method).
 * data: device int64 [n_rep][horizon][rec_len] (stacked records), cols:
 * device int32[n_cols] record columns, out: device double
 * [n_cols][horizon][3]. */
int epi_quartiles(const int64_t *data, int64_t n_rep, int32_t horizon, int32_t rec_len,
                  const int32_t *cols, int32_t n_cols, double *out, void *stream);

/* Fused-mode intervention days on the whole population in 4 launches
 * (testing inside the day kernel; plan + doses + tomorrow's push tables in
 * k_iv_post_chunks / k_finish_iv); bitwise the same as the per-phase kernels
 * (on = 0). */
int epi_set_iv_fusion(epi_ctx *ctx, int32_t on);
/* Grid of the per-day fused kernel: at most blocks_per_sm blocks per SM
 * (0 = default 16).  Replicas run concurrently on several streams fill the
 * GPU better with 1 (config 4). */
int epi_set_day_grid(epi_ctx *ctx, int32_t blocks_per_sm);
/* 1 if epi_sim_run(mode, precision) of >= 2 days would use k_fused_run. */
int epi_run_persistent(epi_ctx *ctx, int32_t mode, int32_t precision);

/* epi_sim_step that also records 4 caller-created cudaEvent_t: before the
 * generator, before the message pass, after it, after the intervention
 * phases — per-kernel device times for the roofline (bench.py). */
int epi_sim_step_timed(epi_ctx *ctx, const epi_state *st, int32_t step, uint64_t seed,
                       int32_t mode, int32_t precision, const uint16_t *codes_cur,
                       uint16_t *codes_next, int64_t *record, int32_t *vax_open,
                       void *const *events4, void *stream);

/* The north-star decomposition of one day, as separate launches:
 *   (c) epi_net_generate: day tables + generator writing the pre-joined
 *       16-bit message CSR of day `step` (ctx-owned, padded rows);
 *   (a) epi_net_gather: the message pass alone, hazard float[N] out
 *       (engine.py:77-117 on the config networks, fp32 fast mode);
 *       `record` (nullable) receives the edge count. */
int epi_net_generate(epi_ctx *ctx, int32_t step, uint64_t seed, const uint16_t *codes_cur,
                     void *stream);
int epi_net_gather(epi_ctx *ctx, const epi_state *st, int32_t step, const uint16_t *codes_cur,
                   float *lambda_out, int64_t *record, void *stream);

/* Device pointers of the CSR slot written for `step` (mode 0), for export. */
int epi_net_csr(epi_ctx *ctx, int32_t step, uint32_t **entries, int32_t **row_len);

/* Seed infections at step 0: entry stage + first transition for ids[0..n)
 * (population.py:151-177 after the choice of ids). */
int epi_seed_infections(epi_ctx *ctx, const epi_state *st, uint64_t seed,
                        const int64_t *ids, int64_t n, void *stream);

/* DEN app adoption u(seed, 0, DEN_APP, a) < adoption (runner.py:86-89). */
int epi_assign_app(const epi_state *st, uint64_t seed, double adoption, void *stream);

/* ---- reference-native networks ------------------
 * Households from an arbitrary household_id, per-occupation Watts-Strogatz and
 * configuration-model stub pairing as keyed parallel algorithms (specification
 * in csrc/epi_refnet.cuh); replaces GraphRealizer (graphs.py:176-240). */
typedef struct epi_refnet_desc {
    int64_t n_agents;
    const int32_t *hh_members;    /* agents grouped by household            */
    const int32_t *hh_start;      /* per agent: first slot of its household */
    const int32_t *hh_size;       /* per agent                              */
    int32_t n_occ;
    int32_t _pad;
    const int32_t *occ_members;   /* agents grouped by occupation, ids asc  */
    const int32_t *occ_start;     /* [n_occ + 1]                            */
    const int32_t *occ_k;         /* round_to_even(mean interactions)       */
    int64_t n_member_slots;
    double rewire_beta;
    const double *random_degree;  /* [N] target random degree               */
    int64_t table_slots;          /* power of two >= 2 * (rewired + pairs)  */
} epi_refnet_desc;

typedef struct epi_refnet_t epi_refnet_t;

int epi_refnet_create(const epi_refnet_desc *desc, epi_refnet_t **out);
int epi_refnet_destroy(epi_refnet_t *net);
/* Edges of step `step` given dead[N] (u8): writes COO into src/dst/kind
 * (capacity entries) and *n_edges (host; synchronises the stream). */
int epi_refnet_realize(epi_refnet_t *net, uint64_t seed, int32_t step, const uint8_t *dead,
                       int32_t *src, int32_t *dst, int8_t *kind, int64_t capacity,
                       int64_t *n_edges, void *stream);
/* The same without synchronising: count[0] = edges, count[1] = error bits
 * (1 capacity, 2 dedupe table, 4 stub overflow), both device uint64. */
int epi_refnet_realize_counted(epi_refnet_t *net, uint64_t seed, int32_t step, const uint8_t *dead,
                               int32_t *src, int32_t *dst, int8_t *kind, int64_t capacity,
                               uint64_t *count, void *stream);

/* The replication loop of the reference (runner.py:138-150, bench
 * runner.py:282-287) for steps [first, last), issued natively with no host
 * synchronisation (graph_seed: the realizer's, seed: the engine's): per step
 * realize into src/dst/kind (capacity entries; the dead agents read from
 * st->stage), load, epi_step.  counts = device uint64[last-first][2] (edges,
 * realizer error bits as epi_refnet_realize_counted), records = device
 * int64[last-first][EPI_REC_LEN]; both are zeroed and filled.  Not with
 * exposure notification (its contact log needs host-known edge counts). */
int epi_refnet_run(epi_refnet_t *net, epi_ctx *ctx, const epi_state *st, uint64_t graph_seed,
                   uint64_t seed, int32_t first, int32_t last, int32_t *src, int32_t *dst,
                   int8_t *kind, int64_t capacity, uint64_t *counts, int64_t *records,
                   int32_t *vax_open, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* EPI_B200_H */
