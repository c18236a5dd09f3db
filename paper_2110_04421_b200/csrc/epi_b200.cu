// libepib200 — host side of the C ABI declared in include/epi_b200.h.
//
// A context owns: the device copy of epi_params, per-agent scratch (codes,
// flags, vaccination buckets), the graph-in CSR (counting sort by destination
// + per-row sorts into (dst, src, kind) order), the contact ring for exposure
// notification, the per-step padded CSR ring and day tables of an attached
// config network, and (partitioned runs) the code-exchange settings.
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include <cub/device/device_scan.cuh>
#include <cuda/std/functional>
#include <dlfcn.h>
#include <nccl.h>

#include "epi_kernels.cuh"
#include "epi_msgpass.cuh"
#include "epi_persistent.cuh"
#include "epi_persistent_iv.cuh"
#include "epi_population.cuh"
#include "epi_refnet.cuh"
#include "epi_series.cuh"

using namespace epi;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CK(call)                                                                         \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return fail(EPI_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));        \
  } while (0)

#define CKL()                                                                            \
  do {                                                                                   \
    cudaError_t e_ = cudaGetLastError();                                                 \
    if (e_ != cudaSuccess)                                                               \
      return fail(EPI_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(e_));   \
  } while (0)

inline cudaStream_t S(void* s) { return (cudaStream_t)s; }

int g_sms = 0;
int sm_count() {
  if (!g_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_sms <= 0) g_sms = 148;
  }
  return g_sms;
}
inline int grid_for(int64_t n, int threads, int per_sm = 8) {
  int64_t g = (n + threads - 1) / threads;
  int64_t cap = (int64_t)sm_count() * per_sm;
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

// L2 residency window for the random gathers of a day (the source-code
// buffers): lines inside it are persisting, so the streamed tables and
// messages of a 10M-agent day cannot evict them (epi_set_hot_window).
struct HotWindow {
  const void* base = nullptr;
  size_t bytes = 0;
  float hit_ratio = 0.f;
};

// Launch with programmatic stream serialization (see pdl_wait/pdl_trigger)
// and, if given, the L2 access-policy window (kept by graph capture).
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl_w(const HotWindow* w, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                         cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.numAttrs = 1;
  if (w != nullptr && w->bytes > 0) {
    attr[1].id = cudaLaunchAttributeAccessPolicyWindow;
    attr[1].val.accessPolicyWindow.base_ptr = const_cast<void*>(w->base);
    attr[1].val.accessPolicyWindow.num_bytes = w->bytes;
    attr[1].val.accessPolicyWindow.hitRatio = w->hit_ratio;
    attr[1].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr[1].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    cfg.numAttrs = 2;
  }
  cfg.attrs = attr;
  return cudaLaunchKernelEx(&cfg, kernel, ((KArgs)args)...);
}
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args... args) {
  return launch_pdl_w(nullptr, kernel, grid, block, smem, s, args...);
}

// Device buffers of contexts come from a process-wide cache: epi_destroy
// synchronises the device once and returns its buffers to the cache, and the
// next context asking for the same (256-byte rounded) size reuses them.  A
// caller building many short-lived engines (the reference's own test suite
// builds ~20 000) otherwise pays a cudaFree per buffer -- each a device
// synchronisation and an unmap, ~100 ms for a garbage-collection pass that
// finalises a few hundred engines at once.  At most 1 GiB stays cached.
namespace {
struct DevCache {
  std::mutex m;
  std::unordered_map<void*, size_t> live;              // cache-managed pointer -> bytes
  std::unordered_multimap<size_t, void*> idle;
  size_t idle_bytes = 0;
};
DevCache& dcache() {
  static DevCache* c = new DevCache;                    // never destroyed: used until process exit
  return *c;
}
constexpr size_t DCACHE_CAP = (size_t)1 << 30;
}  // namespace

cudaError_t dmalloc(void** p, size_t bytes) {
  bytes = ((bytes ? bytes : 1) + 255) & ~(size_t)255;
  DevCache& c = dcache();
  {
    std::lock_guard<std::mutex> g(c.m);
    auto it = c.idle.find(bytes);
    if (it != c.idle.end()) {
      *p = it->second;
      c.idle.erase(it);
      c.idle_bytes -= bytes;
      c.live[*p] = bytes;
      return cudaSuccess;
    }
  }
  cudaError_t e = cudaMalloc(p, bytes);
  if (e == cudaErrorMemoryAllocation) {                 // give the cached buffers back and retry
    cudaGetLastError();
    std::lock_guard<std::mutex> g(c.m);
    for (auto& kv : c.idle) cudaFree(kv.second);
    c.idle.clear();
    c.idle_bytes = 0;
    e = cudaMalloc(p, bytes);
  }
  if (e == cudaSuccess) {
    std::lock_guard<std::mutex> g(c.m);
    c.live[*p] = bytes;
  }
  return e;
}
// Free now (cudaFree: synchronous), cache-managed or not.
void dfree_now(void* p) {
  if (!p) return;
  {
    DevCache& c = dcache();
    std::lock_guard<std::mutex> g(c.m);
    c.live.erase(p);
  }
  cudaFree(p);
}
// Return to the cache; only after the device has been synchronised (no
// kernel may still use the buffer when the next context receives it).
void dput(void* p) {
  if (!p) return;
  DevCache& c = dcache();
  {
    std::lock_guard<std::mutex> g(c.m);
    auto it = c.live.find(p);
    if (it != c.live.end()) {
      const size_t b = it->second;
      c.live.erase(it);
      if (c.idle_bytes + b <= DCACHE_CAP) {
        c.idle.emplace(b, p);
        c.idle_bytes += b;
        return;
      }
    }
  }
  cudaFree(p);
}

template <class T>
int dalloc(T** p, size_t count) {
  if (*p) dfree_now(*p);
  *p = nullptr;
  if (count == 0) count = 1;
  CK(dmalloc((void**)p, count * sizeof(T)));
  return 0;
}

// NCCL, opened at run time (the process's libnccl.so.2 -- torch's when torch
// is loaded -- so one NCCL serves both), for the per-day code all-gather of
// agent-range partitioned runs.
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};
const NcclApi* nccl_api() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.get_unique_id = (decltype(api.get_unique_id))dlsym(h, "ncclGetUniqueId");
      api.comm_init_rank = (decltype(api.comm_init_rank))dlsym(h, "ncclCommInitRank");
      api.comm_destroy = (decltype(api.comm_destroy))dlsym(h, "ncclCommDestroy");
      api.all_gather = (decltype(api.all_gather))dlsym(h, "ncclAllGather");
      api.error_string = (decltype(api.error_string))dlsym(h, "ncclGetErrorString");
      if (api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.all_gather && api.error_string)
        api.h = h;
    }
  }
  return api.h ? &api : nullptr;
}

}  // namespace

struct epi_comm {
  ncclComm_t comm = nullptr;
  int world = 1, rank = 0;
};

struct epi_ctx {
  HotWindow hot;                     // L2-persisting window (source codes)
  epi_exchange_fn xfn = nullptr;     // cross-rank exchange of a partitioned run
  void* xuser = nullptr;
  int push_max = -1;                 // push tables up to this many agents (-1: by L2 size)
  int indep = 0;                     // graph-in fp64: independent-edges infection draws
  int32_t* died_at = nullptr;        // DEN on config networks: death step per agent
  uint8_t* den_mark = nullptr;       // DEN, partitioned: notifications pushed by this rank
  int32_t* den_list = nullptr;       // DEN: the day's notifiers (work list of k_den_regen)
  int* den_count = nullptr;
  epi_params host{};
  epi_params* P = nullptr;           // device copy
  int64_t n = 0;
  int64_t lo = 0, hi = 0;            // owned rows (agent-range partition)
  uint8_t* flags = nullptr;          // n rounded up to 4
  uint8_t* bucket = nullptr;
  unsigned long long* hist = nullptr;
  long long* plan = nullptr;
  int* tile_off = nullptr;
  long long* scratch_rec = nullptr;  // record when the caller passes none
  long long* gflags = nullptr;       // graph validation bits (epi_graph_load)
  uint16_t* codes = nullptr;         // graph-in codes
  uint16_t* codes_alt = nullptr;     // epi_refnet_run: the other buffer of the codes ping-pong
  // graph-in CSR
  int64_t edge_cap = 0, n_edges = 0;
  uint32_t* entries = nullptr;
  int64_t* row_begin = nullptr;
  int32_t* row_len = nullptr;
  int32_t* row_fill = nullptr;       // graph load: per-row scatter cursors
  uint32_t* entries_tmp = nullptr;   // graph load: merge scratch of the long-row sort
  int32_t* long_rows = nullptr;      // graph load: rows of > 32 in-edges (k_rows_sort_long)
  unsigned* long_count = nullptr;
  void* cub_tmp = nullptr;
  size_t cub_bytes = 0;
  const int32_t *g_src = nullptr, *g_dst = nullptr;   // current graph (device, caller-owned)
  // contact ring (graph-in)
  struct Slot { int32_t *src = nullptr, *dst = nullptr; int64_t cap = 0, n = 0; };
  std::vector<Slot> ring;
  int ring_head = 0, ring_count = 0;
  // attached config network
  bool has_net = false;
  epi_net net{};
  epi_net* net_dev = nullptr;
  int net_slots = 0;
  std::vector<uint32_t*> net_entries;
  uint16_t* net_msgs = nullptr;      // fp32 csr mode: tile-packed pre-joined messages
  uint16_t* net_toff = nullptr;      // per-tile row offsets (33 per tile of 32 rows)
  std::vector<int32_t*> net_rowlen;
  std::vector<int32_t> net_slot_step;
  MsgTables* msg_dev = nullptr;      // fp32 message tables (rate_scale baked in)
  MsgComb* comb_dev = nullptr;       // weights of the pre-joined messages
  uint16_t* tau_lut = nullptr;       // bucket table of delay_steps
  NetTables ntab{};                  // host copy (static radix tables)
  NetTables* ntab_dev[3] = {nullptr, nullptr, nullptr};   // per-day keys, by step % 3
  WorkTables wt_host[2]{};           // day tables by step parity
  WorkTables* wt_dev[2][4] = {};     // device structs per parity x variant (0 member tables,
                                     // 1 + wcode, 2 + rin/rout, 3 + rin)
                                     //   0 csr (ids), 1 fused partitioned, 2 fused whole,
                                     //   3 fused whole beyond the push tables (sparse rows)
  int merged_ready = -1;             // day whose tables the previous merged kernel built
  int sparse_push = 1;               // sparse push rows beyond the push tables (epi_set_sparse_push)
  int sparse_ready = -1;             // day whose sparse rows the previous day kernel pushed
  int sparse_clean = -1;             // day whose sparse rows are all zero (the chain goes on)
  Injected* inj_dev = nullptr;
  int persistent = 1;                // epi_sim_run: one launch for the merged days
  int iv_fusion = 1;                 // intervention days in 4 launches (k_iv_post_chunks, k_finish_iv)
  int day_blocks_per_sm = 16;        // k_fused_step grid cap (concurrent replicas: 1)
  unsigned* iv_tile_hist = nullptr;  // [chunks][NUM_BUCKETS]
  unsigned long long* iv_hist = nullptr;   // [2][NUM_BUCKETS] eligibility histogram by day parity
  unsigned long long* ivr_hist = nullptr;  // k_iv_run: [3][NUM_BUCKETS + 1] (+ active count)
  unsigned* ivr_tile_hist = nullptr;       // k_iv_run: [2][SMs][NUM_BUCKETS]
  unsigned* run_barrier = nullptr;   // arrival counter of k_fused_run's grid barrier
  uint4* run_wtab = nullptr;         // per-workplace window values of the persistent runs [3][W][2]
  uint16_t* run_crow = nullptr;      // k_fused_run's colleague rows [2][member slots][16] (all zero between launches)
  LamProbe probe{};                  // debug hazard export (epi_set_lambda_probe)
  // days of a fused run without push tables (partitioned ranks, populations
  // above the L2 cut-off): tomorrow's sigma tables are built on a side
  // stream while today's kernel and the code exchange run
  cudaStream_t side = nullptr;
  cudaEvent_t fork_ev = nullptr, sigma_ev = nullptr;
  int sigma_day = -1;                // the day whose sigma tables are (being) built ahead
  uint64_t sigma_seed = 0;
  int sigma_ahead = 1;               // epi_set_sigma_ahead
  // the per-day code exchange of a partitioned run (epi_set_comm / callback)
  int gather_mode = 0;               // 0: the caller exchanges; 1: xfn EPI_X_GATHER_U16; 2: NCCL
  epi_comm* comm = nullptr;
  int64_t gather_chunk = 0;          // codes per rank (the buffer holds world * chunk)
};

namespace {

int upload_params(epi_ctx* c, const epi_params* p) {
  if (p->t_max < 1 || p->t_max > EPI_MAX_T) return fail(EPI_EARG, "t_max outside [1, 127]");
  if (p->n_specs < 0 || p->n_specs > EPI_MAX_SPECS) return fail(EPI_EARG, "too many duration specs");
  for (int i = 0; i < p->n_specs; ++i)
    if (p->tau_len[i] < 0 || p->tau_len[i] > EPI_MAX_TAUS) return fail(EPI_EARG, "tau table too long");
  c->host = *p;
  if (!c->P) CK(dmalloc((void**)&c->P, sizeof(epi_params)));
  CK(cudaMemcpy(c->P, p, sizeof(epi_params), cudaMemcpyHostToDevice));
  MsgTables mt;
  fill_msg_tables(mt, *p, p->rate_scale);
  if (!c->msg_dev) CK(dmalloc((void**)&c->msg_dev, sizeof(MsgTables)));
  CK(cudaMemcpy(c->msg_dev, &mt, sizeof(MsgTables), cudaMemcpyHostToDevice));
  static MsgComb mc;   // 4 KB: not on the stack
  fill_msg_comb(mc, *p, p->rate_scale);
  if (!c->comb_dev) CK(dmalloc((void**)&c->comb_dev, sizeof(MsgComb)));
  CK(cudaMemcpy(c->comb_dev, &mc, sizeof(MsgComb), cudaMemcpyHostToDevice));
  std::vector<uint16_t> lut((size_t)EPI_MAX_SPECS * TAU_LUT);
  fill_tau_lut(lut.data(), *p);
  if (!c->tau_lut) CK(dmalloc((void**)&c->tau_lut, lut.size() * sizeof(uint16_t)));
  CK(cudaMemcpy(c->tau_lut, lut.data(), lut.size() * sizeof(uint16_t), cudaMemcpyHostToDevice));
  return 0;
}

StepArgs make_args(epi_ctx* c, const epi_state* st, int step, uint64_t seed, long long* rec,
                   const Injected* inj, bool with_flags) {
  StepArgs A;
  A.P = c->P;
  A.st = *st;
  A.step = step;
  A.K = make_step_keys(seed, step);
  A.inj = inj;
  A.rec = rec;
  A.flags = with_flags ? c->flags : nullptr;
  A.lo = c->lo;
  A.hi = c->hi;
  A.indep = c->indep;
  A.tau_lut = c->tau_lut;
  A.probe = c->probe;
  return A;
}

int upload_injected(epi_ctx* c, const double* const* injected, const Injected** out, cudaStream_t s) {
  *out = nullptr;
  if (!injected) return 0;
  Injected h;
  for (int i = 0; i < 12; ++i) h.u[i] = injected[i];
  if (!c->inj_dev) CK(dmalloc((void**)&c->inj_dev, sizeof(Injected)));
  CK(cudaMemcpyAsync(c->inj_dev, &h, sizeof(Injected), cudaMemcpyHostToDevice, s));
  *out = c->inj_dev;
  return 0;
}

bool interventions_on(const epi_params& p) {
  return p.testing_enabled || p.quarantine_enabled || p.den_enabled || p.vaccination_enabled;
}

// Phases 3-6 + finish, shared by the graph-in step and the config sim step.
// `den_scan` launches the contact scan for this step (may be empty).
static bool partitioned(const epi_ctx* c) { return c->lo != 0 || c->hi != c->n; }

static int exchange(epi_ctx* c, int32_t kind, void* buf, int64_t count, cudaStream_t s) {
  if (!c->xfn) return fail(EPI_EARG, "partitioned run without an exchange (epi_set_exchange)");
  const int rc = c->xfn(c->xuser, kind, buf, count, (void*)s);
  return rc ? fail(EPI_ECUDA, "exchange callback failed") : 0;
}

// `den_scan(partitioned)` marks this step's notified contacts (may be empty).
template <class DenScan>
int run_interventions(epi_ctx* c, const StepArgs& A, uint16_t* codes_next, const epi_net* net_dev,
                      uint64_t rcount_next, int32_t* vax_open, cudaStream_t s, DenScan&& den_scan) {
  const epi_params& p = c->host;
  const int64_t n = c->n;
  const bool part = partitioned(c);
  const int threads = 256;
  const int grid = grid_for(n, threads);
  if (p.testing_enabled) {
    // config networks with DEN: the day's notifiers as a work list
    const bool listed = p.den_enabled && c->den_list != nullptr && c->has_net;
    if (listed) CK(cudaMemsetAsync(c->den_count, 0, sizeof(int), s));
    k_iv_tests<<<grid, threads, 0, s>>>(A, listed ? c->den_list : nullptr, listed ? c->den_count : nullptr);
    CKL();
  }
  if (p.den_enabled) {
    int rc = den_scan(part);
    if (rc) return rc;
  }
  if (p.vaccination_enabled)
    CK(cudaMemsetAsync(c->hist, 0, (NUM_BUCKETS + 2) * sizeof(unsigned long long), s));
  if (p.den_enabled || p.quarantine_enabled || p.vaccination_enabled) {
    k_iv_post<<<grid, threads, 0, s>>>(A, c->bucket, c->hist);
    CKL();
  }
  if (p.vaccination_enabled) {
    if (!vax_open) return fail(EPI_EARG, "vaccination enabled but no vax_open latch given");
    if (part) {
      // population histogram and active count: summed over the ranks
      CK(cudaMemcpyAsync(c->hist + NUM_BUCKETS, A.rec + EPI_REC_ACTIVE, sizeof(long long),
                         cudaMemcpyDeviceToDevice, s));
      int rc = exchange(c, EPI_X_SUM_U64, c->hist, NUM_BUCKETS + 1, s);
      if (rc) return rc;
    }
    k_vax_plan<<<1, 32, 0, s>>>(c->P, c->hist, A.rec, vax_open, c->plan, part ? 1 : 0, c->lo == 0 ? 1 : 0);
    CKL();
    const int64_t tiles = (c->hi - c->lo + VAX_TILE - 1) / VAX_TILE;
    if (tiles > 0) {
      k_vax_tilecount<<<(unsigned)tiles, VAX_TILE, 0, s>>>(c->bucket, c->lo, c->hi, c->plan, c->tile_off);
      CKL();
      k_vax_tilescan<<<1, 1024, 0, s>>>(c->tile_off, tiles, c->plan + 2);
      CKL();
    } else {
      CK(cudaMemsetAsync(c->plan + 2, 0, sizeof(long long), s));
    }
    // the cut bucket is served in id order across the ranks' contiguous ranges
    if (part) {
      int rc = exchange(c, EPI_X_EXSCAN_I64, c->plan + 2, 1, s);
      if (rc) return rc;
    }
    if (tiles > 0) {
      k_vax_apply<<<(unsigned)tiles, VAX_TILE, 0, s>>>(A, c->bucket, c->plan, c->tile_off,
                                                       part ? (const long long*)(c->plan + 2) : nullptr);
      CKL();
    }
  }
  k_finish<<<grid, threads, 0, s>>>(A, codes_next, net_dev, rcount_next);
  CKL();
  return 0;
}

}  // namespace

// Push tables (rin/rout: 96 B per agent, scattered to by random rows) pay
// off while they stay in L2; beyond that the scatter goes to DRAM as
// partial-sector writes and evaluating the bijections is cheaper.
static bool push_fits(const epi_ctx* c) {
  if (c->push_max >= 0) return c->n <= c->push_max;
  int dev = 0, l2 = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
  return (double)c->n * 96.0 <= (double)l2;
}

// Could the days of a run go to the persistent kernels (one co-resident
// thread per agent, epi_set_persistent on)?  (persistent_ok adds the rest.)
static bool run_fits(const epi_ctx* c) {
  const int64_t sms = sm_count();
  const int64_t threads = ((c->n + sms - 1) / sms + 31) / 32 * 32;     // (run_threads)
  return c->persistent && c->net.colleague_draws <= 8 && threads <= RUN_BIG_AGENTS;
}

// k_msg_pass: per-warp segment scratch
static int msg_pass_smem(int) { return MP_SMEM; }

// persistent grid: as many k_msg_pass blocks as fit on every SM at once
template <int MODE>
static int msg_pass_grid(int cap, int64_t rows) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_msg_pass<MODE>, MP_WARPS * 32,
                                                    msg_pass_smem(cap)) != cudaSuccess || per_sm < 1)
    per_sm = 1;
  int64_t tiles = (rows + 31) / 32;
  int64_t g = (int64_t)sm_count() * per_sm;
  const int64_t need = (tiles + MP_WARPS - 1) / MP_WARPS;
  if (g > need) g = need;
  return (int)(g < 1 ? 1 : g);
}

extern "C" {

const char* epi_last_error(void) { return g_err.c_str(); }
int epi_version(void) { return 1; }

int64_t epi_struct_size(int32_t which) {
  switch (which) {
    case 0: return (int64_t)sizeof(epi_params);
    case 1: return (int64_t)sizeof(epi_state);
    case 2: return (int64_t)sizeof(epi_net);
    case 3: return (int64_t)sizeof(epi_refnet_desc);
    default: return -1;
  }
}

int epi_create(const epi_params* params, int64_t n_agents, epi_ctx** out) {
  if (!params || !out) return fail(EPI_EARG, "null argument");
  if (n_agents < 1 || n_agents >= (1ll << 30)) return fail(EPI_EARG, "n_agents must be in [1, 2^30)");
  epi_ctx* c = new epi_ctx();
  c->n = n_agents;
  c->lo = 0;
  c->hi = n_agents;
  int rc = upload_params(c, params);
  const int64_t n4 = (n_agents + 3) / 4 * 4;
  const int64_t tiles = (n_agents + VAX_TILE - 1) / VAX_TILE;
  if (!rc) rc = dalloc(&c->flags, n4);
  if (!rc) rc = dalloc(&c->bucket, n_agents);
  if (!rc) rc = dalloc(&c->hist, NUM_BUCKETS + 2);   // + population active count
  if (!rc) rc = dalloc(&c->plan, 4);
  if (!rc) rc = dalloc(&c->tile_off, tiles);
  if (!rc) rc = dalloc(&c->scratch_rec, EPI_REC_LEN);
  if (!rc) rc = dalloc(&c->gflags, 1);
  if (!rc) rc = dalloc(&c->codes, n_agents);
  if (!rc) rc = dalloc(&c->row_begin, n_agents);
  if (!rc) rc = dalloc(&c->row_len, n_agents);
  if (!rc) {
    if (cudaMemset(c->flags, 0, n4) != cudaSuccess || cudaMemset(c->gflags, 0, 8) != cudaSuccess)
      rc = fail(EPI_ECUDA, "memset scratch");
  }
  if (rc) {
    epi_destroy(c);
    return rc;
  }
  *out = c;
  return 0;
}

int epi_destroy(epi_ctx* c) {
  if (!c) return 0;
  cudaDeviceSynchronize();             // no kernel of this context may still use its buffers
  dput(c->P);
  dput(c->flags);
  dput(c->bucket);
  dput(c->hist);
  dput(c->plan);
  dput(c->tile_off);
  dput(c->scratch_rec);
  dput(c->gflags);
  dput(c->codes);
  dput(c->codes_alt);
  dput(c->entries);
  dput(c->row_begin);
  dput(c->row_len);
  dput(c->row_fill);
  dput(c->entries_tmp);
  dput(c->long_rows);
  dput(c->long_count);
  dput(c->cub_tmp);
  dput(c->net_dev);
  dput(c->inj_dev);
  dput(c->msg_dev);
  dput(c->comb_dev);
  dput(c->tau_lut);
  dput(c->died_at);
  dput(c->den_mark);
  dput(c->den_list);
  dput(c->den_count);
  dput(c->run_barrier);
  dput(c->run_wtab);
  dput(c->run_crow);
  dput(c->iv_tile_hist);
  dput(c->iv_hist);
  dput(c->ivr_hist);
  dput(c->ivr_tile_hist);
  for (auto* p : c->ntab_dev) dput(p);
  dput(c->wt_host[0].member_at_pos);
  dput(c->wt_host[1].member_at_pos);
  if (c->side) cudaStreamDestroy(c->side);
  if (c->fork_ev) cudaEventDestroy(c->fork_ev);
  if (c->sigma_ev) cudaEventDestroy(c->sigma_ev);
  for (auto& w : c->wt_host) {
    dput(w.pos_of);
    dput(w.shift);
    dput(w.wcode);
    dput(w.rout);
    dput(w.rin);
  }
  for (auto& row : c->wt_dev)
    for (auto* p : row) dput(p);
  for (auto& s : c->ring) { dput(s.src); dput(s.dst); }
  for (auto* p : c->net_entries) dput(p);
  for (auto* p : c->net_rowlen) dput(p);
  dput(c->net_msgs);
  dput(c->net_toff);
  delete c;
  return 0;
}

int epi_set_rows(epi_ctx* c, int64_t lo, int64_t hi) {
  if (!c || lo < 0 || hi > c->n || lo >= hi) return fail(EPI_EARG, "row range outside [0, n_agents)");
  c->lo = lo;
  c->hi = hi;
  return 0;
}

int epi_set_params(epi_ctx* c, const epi_params* p) {
  if (!c || !p) return fail(EPI_EARG, "null argument");
  return upload_params(c, p);
}

int epi_uniforms(uint64_t seed, int32_t step, int32_t purpose, const int64_t* ids, int64_t n,
                 int32_t k, double* out, void* stream) {
  if (n < 0 || (!out && n)) return fail(EPI_EARG, "bad output");
  if (!n) return 0;
  k_uniforms<<<grid_for(n, 256), 256, 0, S(stream)>>>(key_prefix(seed, step, purpose), ids, n, k, out);
  CKL();
  return 0;
}

static int graph_load_impl(epi_ctx* c, const int32_t* src, const int32_t* dst, const int8_t* kind, int64_t E,
                           const unsigned long long* count, void* stream, bool rows_counted = false);

int epi_graph_load(epi_ctx* c, const int32_t* src, const int32_t* dst, const int8_t* kind,
                   int64_t E, void* stream) {
  return graph_load_impl(c, src, dst, kind, E, nullptr, stream);
}

int epi_graph_load_counted(epi_ctx* c, const int32_t* src, const int32_t* dst, const int8_t* kind,
                           const uint64_t* count, int64_t capacity, void* stream) {
  if (!count) return fail(EPI_EARG, "null count");
  if (c && c->host.den_enabled)
    return fail(EPI_EARG, "a device-counted graph cannot feed the exposure-notification contact log");
  return graph_load_impl(c, src, dst, kind, capacity, (const unsigned long long*)count, stream);
}

// rows_counted: row_len already holds the in-edges per destination of the
// first min(*count, E) edges, all valid (a device generator wrote them).
static int graph_load_impl(epi_ctx* c, const int32_t* src, const int32_t* dst, const int8_t* kind, int64_t E,
                           const unsigned long long* count, void* stream, bool rows_counted) {
  if (!c || E < 0) return fail(EPI_EARG, "bad argument");
  cudaStream_t s = S(stream);
  c->n_edges = E;
  c->g_src = src;
  c->g_dst = dst;
  if (!rows_counted) CK(cudaMemsetAsync(c->row_len, 0, c->n * sizeof(int32_t), s));
  if (E == 0) {
    CK(cudaMemsetAsync(c->row_len, 0, c->n * sizeof(int32_t), s));
    CK(cudaMemsetAsync(c->row_begin, 0, c->n * sizeof(int64_t), s));
    return 0;
  }
  if (E > c->edge_cap) {
    int64_t cap = E + E / 4;
    int rc = dalloc(&c->entries, cap);
    if (!rc) rc = dalloc(&c->entries_tmp, cap);
    if (rc) return rc;
    c->edge_cap = cap;
  }
  if (!c->long_rows) {
    int rc = dalloc(&c->long_rows, (size_t)c->n);
    if (!rc) rc = dalloc(&c->long_count, 1);
    if (rc) return rc;
  }
  // counting sort by destination + per-row sorts (canonical order)
  if (!c->row_fill) {   // zero here, and again after every load (k_rows_sort)
    int rc = dalloc(&c->row_fill, (size_t)c->n);
    if (rc) return rc;
    CK(cudaMemsetAsync(c->row_fill, 0, c->n * sizeof(int32_t), s));
  }
  if (!rows_counted) {
    k_coo_count<<<grid_for(E, 256), 256, 0, s>>>(src, dst, kind, E, c->n, c->row_len, c->gflags, count);
    CKL();
  }
  size_t need = 0;
  // int32 lengths, int64 offsets: the scan accumulates in int64 (init value type)
  CK(cub::DeviceScan::ExclusiveScan(nullptr, need, c->row_len, c->row_begin, cuda::std::plus<>{}, (int64_t)0,
                                    (int)c->n, s));
  if (need > c->cub_bytes) {
    dfree_now(c->cub_tmp);
    c->cub_tmp = nullptr;
    CK(dmalloc(&c->cub_tmp, need));
    c->cub_bytes = need;
  }
  CK(cub::DeviceScan::ExclusiveScan(c->cub_tmp, need, c->row_len, c->row_begin, cuda::std::plus<>{}, (int64_t)0,
                                    (int)c->n, s));
  CK(launch_pdl(k_coo_scatter, dim3(grid_for(E, 256)), dim3(256), 0, s, src, dst, kind, E, c->n,
                (const int64_t*)c->row_begin, c->row_fill, c->entries, count, c->long_count));
  CK(launch_pdl(k_rows_sort, dim3(grid_for(c->n, 128)), dim3(128), 0, s, c->n, (const int64_t*)c->row_begin,
                (const int32_t*)c->row_len, c->entries, c->row_fill, c->long_rows, c->long_count));
  // rows of more than 32 in-edges: one block each (usually none: the blocks exit at once)
  CK(launch_pdl(k_rows_sort_long, dim3(sm_count()), dim3(1024), 0, s, (const int64_t*)c->row_begin,
                (const int32_t*)c->row_len, c->entries, c->entries_tmp, (const int32_t*)c->long_rows,
                (const unsigned*)c->long_count));
  return 0;
}

int epi_read_flags(epi_ctx* c, int32_t* flags_out, void* stream) {
  if (!c || !flags_out) return fail(EPI_EARG, "null argument");
  long long f = 0;
  CK(cudaMemcpyAsync(&f, c->gflags, sizeof(long long), cudaMemcpyDeviceToHost, S(stream)));
  CK(cudaStreamSynchronize(S(stream)));
  CK(cudaMemsetAsync(c->gflags, 0, sizeof(long long), S(stream)));
  *flags_out = (int32_t)f;
  return 0;
}

int epi_gather(epi_ctx* c, const epi_state* st, int32_t step, int32_t precision, void* lam_out,
               void* stream) {
  if (!c || !st || !lam_out) return fail(EPI_EARG, "null argument");
  if (st->n_agents != c->n) return fail(EPI_EARG, "state size differs from context");
  cudaStream_t s = S(stream);
  k_codes<<<grid_for(c->n, 256), 256, 0, s>>>(c->P, *st, step, nullptr, 0, c->codes, 0, c->n);
  CKL();
  StepArgs A = make_args(c, st, step, 0, c->scratch_rec, nullptr, false);
  CsrView g{c->entries, c->row_len, c->row_begin, 0, nullptr, nullptr};
  const int grid = grid_for(c->n, 256);
  if (precision == EPI_F64_CANONICAL)
    k_pass<true, 0><<<grid, 256, 0, s>>>(A, g, c->codes, lam_out, c->host.rate_scale, 0, nullptr, nullptr, 0,
                                         c->msg_dev);
  else
    k_pass<false, 0><<<grid, 256, 0, s>>>(A, g, c->codes, lam_out, c->host.rate_scale, 0, nullptr, nullptr, 0,
                                          c->msg_dev);
  CKL();
  return 0;
}

static int push_ring(epi_ctx* c, cudaStream_t s) {
  const int L = c->host.den_lookback;
  if ((int)c->ring.size() != L) {
    for (auto& sl : c->ring) { dfree_now(sl.src); dfree_now(sl.dst); }
    c->ring.assign(L, epi_ctx::Slot{});
    c->ring_head = 0;
    c->ring_count = 0;
  }
  epi_ctx::Slot& sl = c->ring[c->ring_head];
  if (c->n_edges > sl.cap) {
    int rc = dalloc(&sl.src, c->n_edges);
    if (!rc) rc = dalloc(&sl.dst, c->n_edges);
    if (rc) return rc;
    sl.cap = c->n_edges;
  }
  sl.n = c->n_edges;
  if (sl.n) {
    CK(cudaMemcpyAsync(sl.src, c->g_src, sl.n * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(sl.dst, c->g_dst, sl.n * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
  }
  c->ring_head = (c->ring_head + 1) % L;
  if (c->ring_count < L) ++c->ring_count;
  return 0;
}

// codes_in: the step's codes already computed (k_codes skipped); codes_out:
// the update writes the next step's codes there (only without interventions:
// their phases change the state after the update).
static int step_impl(epi_ctx* c, const epi_state* st, int32_t step, uint64_t seed,
                     const double* hazard, int64_t* record, int32_t* vax_open,
                     const double* const* injected, void* stream, bool rec_zeroed = false,
                     const uint16_t* codes_in = nullptr, uint16_t* codes_out = nullptr) {
  if (!c || !st) return fail(EPI_EARG, "null argument");
  if (st->n_agents != c->n) return fail(EPI_EARG, "state size differs from context");
  cudaStream_t s = S(stream);
  long long* rec = record ? (long long*)record : c->scratch_rec;
  if (!(rec_zeroed && record)) CK(cudaMemsetAsync(rec, 0, EPI_REC_LEN * sizeof(long long), s));
  const Injected* inj = nullptr;
  int rc = upload_injected(c, injected, &inj, s);
  if (rc) return rc;
  const bool iv = interventions_on(c->host);
  StepArgs A = make_args(c, st, step, seed, rec, inj, iv);
  const int grid = grid_for(c->n, 256);
  if (hazard) {
    k_update_from_hazard<<<grid, 256, 0, s>>>(A, hazard, iv ? 0 : 1);
  } else {
    if (!codes_in)
      CK(launch_pdl(k_codes, dim3(grid), dim3(256), 0, s, c->P, *st, step, (const epi_net*)nullptr, (uint64_t)0,
                    c->codes, (int64_t)0, c->n, (int32_t*)nullptr, (int64_t)0));
    if (iv) codes_out = nullptr;
    CsrView g{c->entries, c->row_len, c->row_begin, 0, nullptr, nullptr};
    CK(launch_pdl(k_pass<true, 1>, dim3(grid), dim3(256), 0, s, A, g, codes_in ? codes_in : (const uint16_t*)c->codes,
                  (void*)nullptr, c->host.rate_scale, iv ? 0 : 1, codes_out, (const epi_net*)nullptr, (uint64_t)0,
                  (const MsgTables*)c->msg_dev));
  }
  CKL();
  if (iv) {
    rc = run_interventions(c, A, nullptr, nullptr, 0, vax_open, s, [&](bool) -> int {
      for (int i = 0; i < c->ring_count; ++i) {
        const epi_ctx::Slot& sl = c->ring[i];
        if (!sl.n) continue;
        k_den_scan_coo<<<grid_for(sl.n, 256), 256, 0, s>>>(sl.src, sl.dst, sl.n, c->flags);
        CKL();
      }
      return 0;
    });
    if (rc) return rc;
  }
  if (c->host.den_enabled && !hazard) {
    rc = push_ring(c, s);
    if (rc) return rc;
  }
  return 0;
}

int epi_step(epi_ctx* c, const epi_state* st, int32_t step, uint64_t seed, int64_t* record,
             int32_t* vax_open, const double* const* injected, int32_t check_invariants,
             void* stream) {
  (void)check_invariants;   // flags are always accumulated; the caller decides to read them
  return step_impl(c, st, step, seed, nullptr, record, vax_open, injected, stream);
}

int epi_step_with_hazard(epi_ctx* c, const epi_state* st, int32_t step, uint64_t seed,
                         const double* hazard, int64_t* record, int32_t* vax_open,
                         const double* const* injected, void* stream) {
  if (!hazard) return fail(EPI_EARG, "hazard is null");
  return step_impl(c, st, step, seed, hazard, record, vax_open, injected, stream);
}

int epi_codes(epi_ctx* c, const epi_state* st, const epi_net* net, uint64_t graph_seed, int32_t step,
              uint16_t* codes_out, void* stream) {
  if (!c || !st || !codes_out) return fail(EPI_EARG, "null argument");
  const epi_net* nd = nullptr;
  if (net) {
    if (!c->has_net) return fail(EPI_EARG, "epi_codes with a network needs epi_net_attach first");
    nd = c->net_dev;
  }
  // a config simulation starting over: death steps restart from the state
  int32_t* died = (net && step == 0) ? c->died_at : nullptr;
  k_codes<<<grid_for(c->n, 256), 256, 0, S(stream)>>>(
      c->P, *st, step, nd, key_prefix(graph_seed, step, P_NET_RCOUNT), codes_out, c->lo, c->hi, died, c->n);
  CKL();
  return 0;
}

static int check_net(const epi_net* net) {
  if (!net) return fail(EPI_EARG, "null network");
  if (net->random_slots < 0 || net->random_slots > EPI_MAX_SLOTS) return fail(EPI_EARG, "random_slots > 32");
  if (net->colleague_draws < 0 || net->colleague_draws > EPI_MAX_SLOTS) return fail(EPI_EARG, "colleague_draws > 32");
  if (net->row_cap < 1 || net->row_cap > 4096) return fail(EPI_EARG, "bad row_cap");
  return 0;
}

static size_t realize_smem(const epi_net* net) {
  return (size_t)128 * (net->row_cap | 1) * sizeof(uint32_t);
}

// the register-batched enumerator covers <= 16 random slots and <= 8 draws
static bool batched(const epi_net* net) { return net->random_slots <= 16 && net->colleague_draws <= 8; }

static size_t g_realize_smem_set = 0;
static int prepare_realize(const epi_net* net) {
  const size_t smem = realize_smem(net);
  if (smem > g_realize_smem_set) {
    CK(cudaFuncSetAttribute(k_net_realize<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CK(cudaFuncSetAttribute(k_net_realize<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CK(cudaFuncSetAttribute(k_net_realize<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CK(cudaFuncSetAttribute(k_net_realize<false, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)smem));
    CK(cudaFuncSetAttribute(k_net_realize<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int psmem = msg_pass_smem(net->row_cap);
    CK(cudaFuncSetAttribute(k_msg_pass<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, psmem));
    CK(cudaFuncSetAttribute(k_msg_pass<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, psmem));
    g_realize_smem_set = smem;
  }
  return 0;
}

static int launch_realize(const epi_net* net, uint64_t g, int32_t step, const uint16_t* codes,
                          uint32_t* entries, uint16_t* msgs, uint16_t* toff, int32_t* row_len, int sort_rows,
                          long long* rec,
                          const WorkTables* wt, int64_t lo, int64_t hi, cudaStream_t s,
                          const NetTables* ntab_dev = nullptr, bool push = false,
                          const HotWindow* hot = nullptr) {
  const size_t smem = realize_smem(net);
  if (smem > g_realize_smem_set) return fail(EPI_EARG, "realize smem not prepared");
  NetKeys nk = make_net_keys(g, step);
  static NetTables* scratch = nullptr;           // standalone epi_net_realize only
  if (!ntab_dev) {
    NetTables local;
    fill_net_tables(local, *net, nk.rperm);
    if (!scratch) CK(cudaMalloc((void**)&scratch, sizeof(NetTables)));
    CK(cudaMemcpyAsync(scratch, &local, sizeof(NetTables), cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
    ntab_dev = scratch;
  }
  const int grid = grid_for(hi - lo, 128, 16);
  const bool batch = batched(net);
  // push: messages from the day's push tables (wt must hold rin/rout)
  auto kern = push ? k_net_realize<false, true, true>
              : sort_rows ? (batch ? k_net_realize<true, true> : k_net_realize<true, false>)
                          : (batch ? k_net_realize<false, true> : k_net_realize<false, false>);
  CK(launch_pdl_w(hot, kern, dim3(grid), dim3(128), smem, s, *net, nk, codes, entries, msgs, toff, row_len, rec,
                wt, lo, hi, ntab_dev));
  CKL();
  return 0;
}

int epi_net_realize(const epi_net* net, uint64_t graph_seed, int32_t step, const uint16_t* codes,
                    uint32_t* entries, int32_t* row_len, int32_t sort_rows, void* stream) {
  int rc = check_net(net);
  if (rc) return rc;
  if (!codes || !entries || !row_len) return fail(EPI_EARG, "null buffer");
  rc = prepare_realize(net);
  if (rc) return rc;
  return launch_realize(net, graph_seed, step, codes, entries, nullptr, nullptr, row_len, sort_rows, nullptr,
                        nullptr,
                        0, net->n_agents, S(stream));
}

int epi_pop_synthesize(const epi_pop_spec* sp, uint64_t seed, const epi_pop_out* o, void* stream) {
  if (!sp || !o) return fail(EPI_EARG, "null argument");
  const int64_t n = sp->n_agents;
  if (n < 1 || n >= (1ll << 30)) return fail(EPI_EARG, "n_agents outside [1, 2^30)");
  if (sp->n_sizes < 1 || sp->n_sizes > 32) return fail(EPI_EARG, "household size classes outside [1, 32]");
  if (sp->wp_min < 2 || sp->wp_max < sp->wp_min || sp->wp_max > 255) return fail(EPI_EARG, "bad workplace sizes");
  if (sp->n_seeds < 0 || sp->n_seeds > n) return fail(EPI_EARG, "n_seeds outside [0, n_agents]");
  cudaStream_t s = S(stream);
  PopTables T{};
  for (int i = 0; i < 9; ++i) T.cum_age[i] = sp->age_cum[i];
  for (int i = 0; i < sp->n_sizes; ++i) {
    T.cum_hh[i] = sp->hh_cum[i];
    T.hh_sizes[i] = sp->hh_sizes[i];
  }
  T.n_sizes = sp->n_sizes;
  T.worker_mask = sp->worker_mask;
  const int64_t max_w = n / sp->wp_min + 2;
  // scratch (one-time setup: plain allocations, freed at the end)
  uint8_t* worker = nullptr;
  int64_t *size_k = nullptr, *ends = nullptr, *nW = nullptr, *wsz = nullptr, *wend = nullptr;
  uint64_t *seed_key = nullptr, *key_sorted = nullptr, *wkey = nullptr, *wkey_sorted = nullptr;
  int32_t *ids = nullptr, *ids_sorted = nullptr, *workers = nullptr, *seed32 = nullptr;
  void* tmp = nullptr;
  auto cleanup = [&]() {
    for (void* p : {(void*)worker, (void*)size_k, (void*)ends, (void*)nW, (void*)wsz, (void*)wend,
                    (void*)seed_key, (void*)key_sorted, (void*)wkey, (void*)wkey_sorted, (void*)ids,
                    (void*)ids_sorted, (void*)workers, (void*)seed32, tmp})
      if (p) dfree_now(p);
  };
  int rc = 0;
  rc = rc ? rc : dalloc(&worker, n);
  rc = rc ? rc : dalloc(&size_k, n);
  rc = rc ? rc : dalloc(&ends, n);
  rc = rc ? rc : dalloc(&nW, 1);
  rc = rc ? rc : dalloc(&wsz, max_w);
  rc = rc ? rc : dalloc(&wend, max_w);
  rc = rc ? rc : dalloc(&seed_key, n);
  rc = rc ? rc : dalloc(&key_sorted, n);
  rc = rc ? rc : dalloc(&wkey, n);
  rc = rc ? rc : dalloc(&wkey_sorted, n);
  rc = rc ? rc : dalloc(&ids, n);
  rc = rc ? rc : dalloc(&ids_sorted, n);
  rc = rc ? rc : dalloc(&workers, n);
  rc = rc ? rc : dalloc(&seed32, sp->n_seeds > 0 ? sp->n_seeds : 1);
  if (rc) { cleanup(); return rc; }
  size_t tb = 0, t1 = 0;
  cub::DeviceScan::InclusiveSum(nullptr, t1, size_k, ends, (int)n, s); tb = t1 > tb ? t1 : tb;
  cub::DeviceScan::InclusiveSum(nullptr, t1, wsz, wend, (int)max_w, s); tb = t1 > tb ? t1 : tb;
  cub::DeviceSelect::Flagged(nullptr, t1, ids, worker, workers, nW, (int)n, s); tb = t1 > tb ? t1 : tb;
  cub::DeviceRadixSort::SortPairs(nullptr, t1, seed_key, key_sorted, ids, ids_sorted, (int)n, 0, 64, s);
  tb = t1 > tb ? t1 : tb;
  cub::DeviceRadixSort::SortKeys(nullptr, t1, ids_sorted, seed32, (int)(sp->n_seeds > 0 ? sp->n_seeds : 1), 0, 32,
                                 s);
  tb = t1 > tb ? t1 : tb;
  if (cudaMalloc(&tmp, tb > 0 ? tb : 1) != cudaSuccess) { cleanup(); return fail(EPI_ECUDA, "temp alloc"); }
  const int g = grid_for(n, 256);
#define PCK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { cleanup(); return fail(EPI_ECUDA, cudaGetErrorString(e_)); } } while (0)
  k_pop_agents<<<g, 256, 0, s>>>(T, n, key_prefix(seed, 0, P_POP_AGE), key_prefix(seed, 0, P_POP_HOUSEHOLD),
                                 key_prefix(seed, 0, P_POP_SEEDS), o->age_band, worker, size_k, seed_key, ids);
  PCK(cudaGetLastError());
  PCK(cub::DeviceScan::InclusiveSum(tmp, tb, size_k, ends, (int)n, s));
  k_pop_households<<<g, 256, 0, s>>>(n, ends, size_k, o->household_id, o->hh_off, o->hh_size);
  PCK(cudaGetLastError());
  // workplaces: stable sort of the workers by key (ties keep ascending ids)
  PCK(cub::DeviceSelect::Flagged(tmp, tb, ids, worker, workers, nW, (int)n, s));
  int64_t W = 0;
  PCK(cudaMemcpyAsync(&W, nW, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  PCK(cudaStreamSynchronize(s));
  k_pop_worker_keys<<<g, 256, 0, s>>>(workers, nW, key_prefix(seed, 0, P_POP_WORKPLACE), wkey, max_w, sp->wp_min,
                                      sp->wp_max - sp->wp_min + 1, wsz);
  PCK(cudaGetLastError());
  if (W > 0) PCK(cub::DeviceRadixSort::SortPairs(tmp, tb, wkey, wkey_sorted, workers, o->wp_members, (int)W, 0, 64, s));
  PCK(cub::DeviceScan::InclusiveSum(tmp, tb, wsz, wend, (int)max_w, s));
  k_fill_i32<<<g, 256, 0, s>>>(o->wp_id, n, -1);
  PCK(cudaMemsetAsync(o->wp_local, 0, (size_t)n, s));
  k_pop_workplaces<<<g, 256, 0, s>>>(o->wp_members, nW, wend, wsz, max_w, o->wp_id, o->wp_local, o->wp_base,
                                     o->wp_size, o->counts);
  PCK(cudaGetLastError());
  // seeds: the n_seeds smallest keys (ties: ascending id), then by id
  if (sp->n_seeds > 0) {
    PCK(cub::DeviceRadixSort::SortPairs(tmp, tb, seed_key, key_sorted, ids, ids_sorted, (int)n, 0, 64, s));
    PCK(cub::DeviceRadixSort::SortKeys(tmp, tb, ids_sorted, seed32, (int)sp->n_seeds, 0, 32, s));
    k_widen<<<grid_for(sp->n_seeds, 256), 256, 0, s>>>(seed32, sp->n_seeds, o->seeds);
    PCK(cudaGetLastError());
  }
#undef PCK
  const cudaError_t e = cudaStreamSynchronize(s);
  cleanup();
  if (e != cudaSuccess) return fail(EPI_ECUDA, cudaGetErrorString(e));
  return 0;
}

int epi_set_hot_window(epi_ctx* c, const void* base, int64_t bytes) {
  if (!c || bytes < 0 || (bytes > 0 && !base)) return fail(EPI_EARG, "bad hot window");
  c->hot = HotWindow{};
  if (bytes == 0) return 0;
  int dev = 0, maxp = 0, maxw = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev));
  CK(cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, dev));
  if (maxp <= 0 || maxw <= 0) return 0;               // no persisting L2: plain caching
  const size_t win = (size_t)bytes < (size_t)maxw ? (size_t)bytes : (size_t)maxw;
  size_t cur = 0;
  CK(cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize));
  const size_t want = win < (size_t)maxp ? win : (size_t)maxp;
  if (cur < want) CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want));
  c->hot.base = base;
  c->hot.bytes = win;
  c->hot.hit_ratio = (float)((double)want / (double)win);
  return 0;
}

int epi_set_infection_mode(epi_ctx* c, int32_t mode) {
  if (!c || (mode != EPI_INFECT_AGGREGATE && mode != EPI_INFECT_INDEPENDENT))
    return fail(EPI_EARG, "infection mode must be EPI_INFECT_AGGREGATE or EPI_INFECT_INDEPENDENT");
  c->indep = mode == EPI_INFECT_INDEPENDENT;
  return 0;
}

int epi_set_exchange(epi_ctx* c, epi_exchange_fn fn, void* user) {
  if (!c) return fail(EPI_EARG, "null ctx");
  c->xfn = fn;
  c->xuser = user;
  return 0;
}

int epi_set_push_max(epi_ctx* c, int64_t max_agents) {
  if (!c) return fail(EPI_EARG, "null ctx");
  c->push_max = max_agents < 0 ? -1 : (int)(max_agents > 0x7FFFFFFF ? 0x7FFFFFFF : max_agents);
  c->merged_ready = -1;
  c->sparse_ready = -1;
  c->sparse_clean = -1;
  return 0;
}

int epi_net_attach(epi_ctx* c, const epi_net* net) {
  if (!c) return fail(EPI_EARG, "null ctx");
  int rc = check_net(net);
  if (rc) return rc;
  if (net->n_agents != c->n) return fail(EPI_EARG, "network size differs from context");
  rc = prepare_realize(net);
  if (rc) return rc;
  c->net = *net;
  fill_net_tables(c->ntab, *net, 0);
  for (int i = 0; i < 3; ++i) {
    if (!c->ntab_dev[i]) CK(dmalloc((void**)&c->ntab_dev[i], sizeof(NetTables)));
    CK(cudaMemcpy(c->ntab_dev[i], &c->ntab, sizeof(NetTables), cudaMemcpyHostToDevice));
  }
  c->has_net = true;
  if (!c->net_dev) CK(dmalloc((void**)&c->net_dev, sizeof(epi_net)));
  CK(cudaMemcpy(c->net_dev, net, sizeof(epi_net), cudaMemcpyHostToDevice));
  // one CSR slot (id rows for fp64 order / export); DEN regenerates past
  // days' contacts instead of keeping a contact log
  const int slots = 1;
  if (c->host.den_enabled) {
    if (c->host.den_lookback > DEN_MAX_DAYS) return fail(EPI_EARG, "den.lookback > 16 on config networks");
    rc = dalloc(&c->died_at, (size_t)c->n);
    if (!rc) rc = dalloc(&c->den_mark, (size_t)c->n + 4);
    if (!rc) rc = dalloc(&c->den_list, 2 * (size_t)c->n);     // [2][n]: k_iv_run uses both day parities
    if (!rc) rc = dalloc(&c->den_count, 3);      // k_iv_run: [3] by run day mod 3
    if (rc) return rc;
    k_fill_i32<<<grid_for(c->n, 256), 256>>>(c->died_at, c->n, INT32_MAX);
    CKL();
  }
  for (auto* p : c->net_entries) dfree_now(p);
  for (auto* p : c->net_rowlen) dfree_now(p);
  c->net_entries.assign(slots, nullptr);
  c->net_rowlen.assign(slots, nullptr);
  c->net_slot_step.assign(slots, -1);
  c->net_slots = slots;
  for (int i = 0; i < slots; ++i) {
    rc = dalloc(&c->net_entries[i], (size_t)c->n * net->row_cap);
    if (!rc) rc = dalloc(&c->net_rowlen[i], (size_t)c->n);
    if (rc) return rc;
  }
  // zero-filled: every u16 of the buffer is always a valid weight-table offset
  const size_t n_msgs = (size_t)((c->n + 31) / 32) * 32 * msg_cap(net->row_cap) + 16;
  rc = dalloc(&c->net_msgs, n_msgs);
  if (!rc) rc = dalloc(&c->net_toff, (size_t)((c->n + 31) / 32) * 33);
  if (rc) return rc;
  CK(cudaMemset(c->net_msgs, 0, n_msgs * sizeof(uint16_t)));
  for (int par = 0; par < 2; ++par) {
    WorkTables& w = c->wt_host[par];
    rc = dalloc(&w.member_at_pos, (size_t)net->n_member_slots);
    if (!rc) rc = dalloc(&w.pos_of, (size_t)net->n_member_slots);
    if (!rc) rc = dalloc(&w.shift, (size_t)net->n_workplaces * (net->colleague_draws + 1));
    if (!rc) rc = dalloc(&w.wcode, (size_t)net->n_member_slots);
    if (!rc) rc = dalloc(&w.rout, (size_t)c->n * RT_SLOTS);
    if (!rc) rc = dalloc(&w.rin, (size_t)c->n * RT_SLOTS);
    if (rc) return rc;
    CK(cudaMemset(w.rin, 0, (size_t)c->n * RT_SLOTS * sizeof(uint16_t)));
    for (int var = 0; var < 4; ++var) {
      WorkTables v = w;
      if (var == 0) v.wcode = nullptr;
      if (var < 2) { v.rin = nullptr; v.rout = nullptr; }
      if (var == 3) v.rout = nullptr;
      if (!c->wt_dev[par][var]) CK(dmalloc((void**)&c->wt_dev[par][var], sizeof(WorkTables)));
      CK(cudaMemcpy(c->wt_dev[par][var], &v, sizeof(WorkTables), cudaMemcpyHostToDevice));
    }
  }
  c->merged_ready = -1;
  c->sparse_ready = -1;
  c->sparse_clean = -1;
  c->sigma_day = -1;
  return 0;
}

int epi_net_csr(epi_ctx* c, int32_t step, uint32_t** entries, int32_t** row_len) {
  if (!c || !c->has_net || !entries || !row_len) return fail(EPI_EARG, "no attached network");
  const int slot = step % c->net_slots;
  if (c->net_slot_step[slot] != step) return fail(EPI_EARG, "CSR for that step is not resident");
  *entries = c->net_entries[slot];
  *row_len = c->net_rowlen[slot];
  return 0;
}

// Balanced grids: a multiple of the SM count, the agents split into equal
// contiguous chunks (<= `threads` agents per block up to `per_sm` blocks per
// SM, longer chunks beyond), so no SM carries an extra block.
static int balanced_grid(int64_t n, int threads, int per_sm) {
  const int64_t sms = sm_count();
  int64_t k = (n + sms * threads - 1) / (sms * threads);
  k = k < 1 ? 1 : (k > per_sm ? per_sm : k);
  return (int)(sms * k);
}

// Chunks of k_iv_post_chunks / k_finish_iv (the vaccination tiles).
static void iv_chunks(int64_t n, int64_t* chunk, int* blocks) {
  *blocks = balanced_grid(n, 256, 1 << 20);
  *chunk = (n + *blocks - 1) / *blocks;
  if (*chunk < 1) *chunk = 1;
  *blocks = (int)((n + *chunk - 1) / *chunk);
}

// One intervention day on the whole population with the push tables:
// k_fused_step (+ testing) -> [k_den_regen] -> [k_iv_post_chunks] ->
// k_finish_iv (+ doses, death days, tomorrow's push tables).  The day's
// tables come from yesterday's k_finish_iv (merged_ready) or are built here.
static int iv_fused_day(epi_ctx* c, const StepArgs& A, int32_t step, uint64_t seed, const uint16_t* codes_cur,
                        uint16_t* codes_next, long long* rec, bool zero_record, int32_t* vax_open, void* const* ev,
                        cudaStream_t s) {
  const epi_params& p = c->host;
  if (p.vaccination_enabled && !vax_open) return fail(EPI_EARG, "vaccination enabled but no vax_open latch given");
  const NetKeys nk = make_net_keys(seed, step);
  NetTables* nt_today = c->ntab_dev[step % 3];
  NetTables* nt_next = c->ntab_dev[(step + 1) % 3];
  const int par = step & 1;
  const uint64_t rcount_next = key_prefix(seed, step + 1, P_NET_RCOUNT);
  int64_t chunk;
  int blocks;
  iv_chunks(c->n, &chunk, &blocks);
  int rc = 0;
  if (!c->iv_hist) {
    rc = dalloc(&c->iv_hist, (size_t)2 * NUM_BUCKETS);
    if (!rc) CK(cudaMemsetAsync(c->iv_hist, 0, (size_t)2 * NUM_BUCKETS * sizeof(unsigned long long), s));
  }
  if (!rc && !c->iv_tile_hist) rc = dalloc(&c->iv_tile_hist, (size_t)blocks * NUM_BUCKETS);
  if (rc) return rc;
  const bool listed = p.den_enabled && p.testing_enabled && c->den_list != nullptr;
  const bool first = c->merged_ready != step;
  if (ev) CK(cudaEventRecord((cudaEvent_t)ev[0], s));
  if (first) {
    // the day's tables from scratch; the day-to-day counters to zero
    k_day_keys<<<1, 32, 0, s>>>(nt_today, nk.rperm, nullptr);
    CKL();
    // both parities: tomorrow's may hold the scatter of a run that stopped
    // before consuming it (then reset to an earlier day)
    CK(cudaMemsetAsync(c->wt_host[par].rin, 0, (size_t)c->n * RT_SLOTS * sizeof(uint16_t), s));
    CK(cudaMemsetAsync(c->wt_host[par ^ 1].rin, 0, (size_t)c->n * RT_SLOTS * sizeof(uint16_t), s));
    const bool has_work = c->net.n_member_slots > 0 && c->net.colleague_draws > 0;
    const int wblocks = has_work ? grid_for(c->net.n_member_slots, 256, 8) : 0;
    const int rblocks = grid_for(c->n, 256, 8);
    CK(launch_pdl_w(&c->hot, k_day_tables, dim3(wblocks + rblocks), dim3(256), 0, s, c->net, nk, c->wt_host[par],
                    codes_cur, (int64_t)0, c->n, wblocks, (const NetTables*)nt_today, nt_next,
                    key_prefix(seed, step + 1, P_NET_RPERM), zero_record ? rec : (long long*)nullptr));
    CK(cudaMemsetAsync(c->iv_hist, 0, (size_t)2 * NUM_BUCKETS * sizeof(unsigned long long), s));
    if (listed) CK(cudaMemsetAsync(c->den_count, 0, sizeof(int), s));
    if (p.den_enabled) {
      // deaths of yesterday (later days: recorded by k_finish_iv)
      k_died_update<<<grid_for(c->n, 256), 256, 0, s>>>(codes_cur, c->n, step, c->died_at);
      CKL();
    }
  } else if (zero_record) {
    CK(cudaMemsetAsync(rec, 0, EPI_REC_LEN * sizeof(long long), s));
  }
  if (ev) CK(cudaEventRecord((cudaEvent_t)ev[1], s));
  const int fgrid = balanced_grid(c->n, 128, c->day_blocks_per_sm);
  DayTests tests{p.testing_enabled ? 1 : 0, listed ? c->den_list : nullptr, listed ? c->den_count : nullptr};
  CK(launch_pdl_w(&c->hot, k_fused_step<1>, dim3(fgrid), dim3(128), 0, s, A, c->net, nk, codes_cur,
                  c->host.rate_scale, codes_next, (const epi_net*)c->net_dev, rcount_next, 0,
                  (const WorkTables*)c->wt_dev[par][2], (const MsgTables*)c->msg_dev, (const NetTables*)nt_today,
                  NextTables{}, 1, tests));
  if (ev) CK(cudaEventRecord((cudaEvent_t)ev[2], s));
  if (p.den_enabled && p.testing_enabled) {
    // contacts of the notifiers over steps step-L .. step-1, regenerated
    DenRegen D{};
    D.first_day = step - p.den_lookback > 0 ? step - p.den_lookback : 0;
    D.n_days = step - D.first_day;
    if (D.n_days > 0) {
      for (int d = 0; d < D.n_days; ++d) D.nk[d] = make_net_keys(seed, D.first_day + d);
      // one warp per (notifier, day) item, read on the device: one block per SM
      CK(launch_pdl_w(&c->hot, k_den_regen, dim3(sm_count()), dim3(256), 0, s, c->net, D, (const int32_t*)c->died_at,
                      (const int32_t*)c->den_list, (const int*)c->den_count, c->flags,
                      (const Radix*)c->ntab_dev[0]->wrad));
    }
  }
  IvPlan V{c->iv_hist, c->iv_tile_hist, vax_open, chunk, p.vaccination_enabled ? 1 : 0};
  if (p.den_enabled || p.quarantine_enabled || p.vaccination_enabled) {
    CK(launch_pdl_w(&c->hot, k_iv_post_chunks, dim3(blocks), dim3(256), 0, s, A, c->bucket, V));
  }
  NextTables nx{};
  nx.wt = c->wt_dev[par ^ 1][2];
  nx.keys = nt_next;
  nx.keys_out = c->ntab_dev[(step + 2) % 3];
  nx.rperm_t2 = key_prefix(seed, step + 2, P_NET_RPERM);
  nx.nk = make_net_keys(seed, step + 1);
  CK(launch_pdl_w(&c->hot, k_finish_iv, dim3(blocks), dim3(256), 0, s, A, codes_next, (const epi_net*)c->net_dev,
                  rcount_next, (const uint8_t*)c->bucket, V, p.den_enabled ? c->died_at : (int32_t*)nullptr,
                  listed ? c->den_count : (int*)nullptr, c->net, nx, c->ntab.dn));
  c->merged_ready = step + 1;
  c->sparse_ready = -1;
  c->sparse_clean = -1;
  if (ev) CK(cudaEventRecord((cudaEvent_t)ev[3], s));
  return 0;
}

// Day tables of a fused day without push tables (partitioned ranks,
// populations above the push-table cut-off), split so the code-independent
// part overlaps: the sigma tables (member_at_pos / pos_of / shift of every
// workplace, tomorrow's random-slot keys) depend on (seed, day) only and are
// built one day ahead on a side stream, concurrently with today's day kernel
// and the code exchange; only the workplace codes (k_wcode) wait for the
// day's complete code vector.  Tomorrow's tables go to the other parity,
// whose last readers (yesterday's kernels) precede the fork in stream order.
static int sigma_day_tables(epi_ctx* c, int32_t step, uint64_t seed, const uint16_t* codes_cur, long long* rec_zero,
                            cudaStream_t s) {
  const int par = step & 1;
  const int wblocks = grid_for(c->net.n_member_slots, 256, 8);
  auto sigma_only = [&](int p) {
    WorkTables w = c->wt_host[p];
    w.wcode = nullptr;
    w.rin = nullptr;
    w.rout = nullptr;
    return w;
  };
  if (c->sigma_day == step && c->sigma_seed == seed) {
    CK(cudaStreamWaitEvent(s, c->sigma_ev, 0));
    if (rec_zero) CK(cudaMemsetAsync(rec_zero, 0, EPI_REC_LEN * sizeof(long long), s));
  } else {
    CK(launch_pdl_w(&c->hot, k_day_tables, dim3(wblocks), dim3(256), 0, s, c->net, make_net_keys(seed, step),
                    sigma_only(par), codes_cur, c->lo, c->hi, wblocks, (const NetTables*)c->ntab_dev[step % 3],
                    c->ntab_dev[(step + 1) % 3], key_prefix(seed, step + 1, P_NET_RPERM), rec_zero));
  }
  CK(launch_pdl_w(&c->hot, k_wcode, dim3(grid_for(c->net.n_member_slots, 256 * 4, 8)), dim3(256), 0, s,
                  (int64_t)c->net.n_member_slots, (const int32_t*)c->wt_host[par].member_at_pos, codes_cur,
                  c->wt_host[par].wcode));
  if (!c->side) {
    CK(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&c->fork_ev, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->sigma_ev, cudaEventDisableTiming));
  }
  CK(cudaEventRecord(c->fork_ev, s));
  CK(cudaStreamWaitEvent(c->side, c->fork_ev, 0));
  CK(launch_pdl(k_day_tables, dim3(wblocks), dim3(256), 0, c->side, c->net, make_net_keys(seed, step + 1),
                sigma_only(par ^ 1), codes_cur, c->lo, c->hi, wblocks, (const NetTables*)c->ntab_dev[(step + 1) % 3],
                c->ntab_dev[(step + 2) % 3], key_prefix(seed, step + 2, P_NET_RPERM), (long long*)nullptr));
  CK(cudaEventRecord(c->sigma_ev, c->side));
  c->sigma_day = step + 1;
  c->sigma_seed = seed;
  return 0;
}

// Join the side stream into `s` (nothing may be left unjoined at the end of
// a call: CUDA-graph capture, and callers timing the stream).
static int join_side(epi_ctx* c, cudaStream_t s) {
  if (c->side && c->sigma_day >= 0) CK(cudaStreamWaitEvent(s, c->sigma_ev, 0));
  return 0;
}

// The per-day code exchange of a partitioned run: every rank's chunk of the
// code vector it just wrote, to every rank, in place.
static int gather_codes(epi_ctx* c, uint16_t* codes, cudaStream_t s) {
  if (c->gather_mode == 2) {
    const NcclApi* api = nccl_api();
    const epi_comm* m = c->comm;
    const size_t bytes = (size_t)c->gather_chunk * sizeof(uint16_t);
    const ncclResult_t r = api->all_gather((const void*)(codes + (size_t)m->rank * c->gather_chunk), (void*)codes,
                                           bytes, ncclUint8, m->comm, s);
    if (r != ncclSuccess) return fail(EPI_ECUDA, std::string("ncclAllGather: ") + api->error_string(r));
    return 0;
  }
  if (c->gather_mode == 1) return exchange(c, EPI_X_GATHER_U16, codes, c->gather_chunk, s);
  return 0;
}

static int sim_step_impl(epi_ctx* c, const epi_state* st, int32_t step, uint64_t seed, int32_t mode,
                         int32_t precision, const uint16_t* codes_cur, uint16_t* codes_next,
                         int64_t* record, int32_t* vax_open, void* const* ev, void* stream,
                         bool zero_record = true) {
  if (!c || !st || !codes_cur || !codes_next) return fail(EPI_EARG, "null argument");
  if (!c->has_net) return fail(EPI_EARG, "epi_sim_step needs epi_net_attach first");
  if (st->n_agents != c->n) return fail(EPI_EARG, "state size differs from context");
  const bool iv = interventions_on(c->host);
  if (partitioned(c) && (c->host.den_enabled || c->host.vaccination_enabled) && !c->xfn)
    return fail(EPI_EARG, "exposure notification and vaccination in a partitioned run need a "
                          "cross-rank exchange (epi_set_exchange)");
  if (mode == 1 && precision != EPI_F32) return fail(EPI_EARG, "fused mode is fp32 only");
  cudaStream_t s = S(stream);
  long long* rec = record ? (long long*)record : c->scratch_rec;
  StepArgs A = make_args(c, st, step, seed, rec, nullptr, iv);
  const uint64_t rcount_next = key_prefix(seed, step + 1, P_NET_RCOUNT);
  const int grid = grid_for(c->hi - c->lo, 256);
  const int slot = step % c->net_slots;
  if (ev) CK(cudaEventRecord((cudaEvent_t)ev[0], s));
  const NetKeys nk = make_net_keys(seed, step);
  NetTables* nt_today = c->ntab_dev[step % 3];
  NetTables* nt_next = c->ntab_dev[(step + 1) % 3];
  const int par = step & 1;
  // day tables: workplace sigma cache (all modes); in fused mode also the
  // push tables (workplace codes; random-slot codes for whole-population runs
  // — a partitioned rank cannot scatter into its peers' rows).  Fused runs
  // without interventions are "merged": today's kernel builds tomorrow's
  // tables in its epilogue, so after the first day there is one kernel per day.
  const bool has_work = c->net.n_member_slots > 0 && c->net.colleague_draws > 0;
  // csr mode writes messages only in fp32 without a contact log
  const bool msg_only = mode == 0 && precision == EPI_F32 && c->net.row_cap <= MP_MAX_CAP;
  // Fused days without interventions use the full push tables only where a
  // persistent run (k_fused_run) can follow, which needs them: elsewhere the
  // sparse rows measured faster at every size (tools/push_vs_sparse.py:
  // 200 k agents 6.1 vs 7.1 ms per simulation, 1 M 21.7 vs 35.0 ms).
  const bool prefer_sparse = mode == 1 && !iv && c->sparse_push && !run_fits(c);
  const bool push_rand = (mode == 1 || msg_only) && c->lo == 0 && c->hi == c->n && c->net.n_agents >= 2 &&
                         c->net.random_slots == RT_SLOTS && batched(&c->net) && push_fits(c) && !prefer_sparse;
  const bool merged = mode == 1 && push_rand && !iv;
  // beyond the push tables (and on partitioned ranks), fused days without
  // interventions push only infectious sources into sparse in-rows
  // (sparse_kind_sums): a whole population's tomorrow in today's epilogue, a
  // chain's first rows and every day of a partitioned rank seeded here
  const bool whole = c->lo == 0 && c->hi == c->n;
  const bool sparse = mode == 1 && !push_rand && !iv && c->sparse_push && c->net.n_agents >= 2 &&
                      c->net.random_slots == RT_SLOTS && batched(&c->net);
  if (mode == 1 && push_rand && iv && c->iv_fusion)
    return iv_fused_day(c, A, step, seed, codes_cur, codes_next, rec, zero_record, vax_open, ev, s);
  const bool use_wt = (mode == 0 && (push_rand || (has_work && batched(&c->net)))) || mode == 1;
  const int variant = push_rand ? 2 : (mode == 0 ? 0 : 1);
  long long* rec_zero = zero_record ? rec : nullptr;
  if (merged && c->merged_ready == step) {
    if (rec_zero) CK(cudaMemsetAsync(rec, 0, EPI_REC_LEN * sizeof(long long), s));
  } else {
    if (step == 0 || merged) {
      k_day_keys<<<1, 32, 0, s>>>(nt_today, nk.rperm, nullptr);
      CKL();
    }
    if (use_wt) {
      if (push_rand && (step == 0 || merged)) {
        // a new chain: today's scatter target, and (merged) tomorrow's, which
        // may hold the scatter of a run that stopped before consuming it
        CK(cudaMemsetAsync(c->wt_host[par].rin, 0, (size_t)c->n * RT_SLOTS * sizeof(uint16_t), s));
        if (merged) CK(cudaMemsetAsync(c->wt_host[par ^ 1].rin, 0, (size_t)c->n * RT_SLOTS * sizeof(uint16_t), s));
      }
      const int wblocks = has_work ? grid_for(c->net.n_member_slots, 256, 8) : 0;
      const int rblocks = push_rand ? grid_for(c->hi - c->lo, 256, 8) : 0;
      WorkTables w = c->wt_host[par];
      if (variant == 0) w.wcode = nullptr;
      if (variant < 2) { w.rin = nullptr; w.rout = nullptr; }
      if (mode == 1 && !push_rand && !iv && has_work && c->sigma_ahead) {
        int rc = sigma_day_tables(c, step, seed, codes_cur, rec_zero, s);
        if (rc) return rc;
      } else {
        CK(launch_pdl_w(&c->hot, k_day_tables, dim3(wblocks + rblocks > 0 ? wblocks + rblocks : 1), dim3(256), 0, s,
                      c->net, nk, w, codes_cur, c->lo, c->hi, wblocks, (const NetTables*)nt_today, nt_next,
                      key_prefix(seed, step + 1, P_NET_RPERM), rec_zero));
        c->sigma_day = -1;
      }
    } else {
      CK(launch_pdl(k_day_keys, dim3(1), dim3(32), 0, s, nt_next, key_prefix(seed, step + 1, P_NET_RPERM),
                    rec_zero));
    }
  }
  if (sparse && c->sparse_ready != step) {
    if (c->sparse_clean != step) {        // a new chain: both parities start empty
      CK(cudaMemsetAsync(c->wt_host[par].rin, 0, (size_t)c->n * RT_SLOTS * sizeof(uint16_t), s));
      CK(cudaMemsetAsync(c->wt_host[par ^ 1].rin, 0, (size_t)c->n * RT_SLOTS * sizeof(uint16_t), s));
    }
    k_sparse_seed<<<grid_for(c->n, 256, 8), 256, 0, s>>>(codes_cur, c->n, c->lo, c->hi, (const NetTables*)nt_today,
                                                           c->wt_host[par].rin);
    CKL();
  }
  const WorkTables* wt = use_wt ? c->wt_dev[par][sparse ? 3 : variant] : nullptr;
  if (mode == 0) {
    // fp32 without contact log: the generator writes pre-joined messages and
    // the message pass streams them; otherwise ids (export, DEN, fp64 order)
    uint32_t* entries = msg_only ? nullptr : c->net_entries[slot];
    uint16_t* msgs = msg_only ? c->net_msgs : nullptr;
    int32_t* row_len = c->net_rowlen[slot];
    int rc = launch_realize(&c->net, seed, step, codes_cur, entries, msgs, c->net_toff, row_len,
                            precision == EPI_F64_CANONICAL, nullptr, wt, c->lo, c->hi, s, nt_today,
                            msg_only && push_rand, &c->hot);
    if (rc) return rc;
    c->net_slot_step[slot] = msg_only ? -1 : step;
    c->merged_ready = -1;
    c->sparse_ready = -1;
    c->sparse_clean = -1;
    if (ev) CK(cudaEventRecord((cudaEvent_t)ev[1], s));
    CsrView g{entries, row_len, nullptr, c->net.row_cap, msgs, c->net_toff};
    if (precision == EPI_F64_CANONICAL)
      k_pass<true, 1><<<grid, 256, 0, s>>>(A, g, codes_cur, nullptr, c->host.rate_scale, iv ? 0 : 1,
                                           codes_next, c->net_dev, rcount_next, c->msg_dev);
    else if (msgs)
      CK(launch_pdl_w(&c->hot, k_msg_pass<1>, dim3(msg_pass_grid<1>(c->net.row_cap, c->hi - c->lo)),
                    dim3(MP_WARPS * 32), (size_t)msg_pass_smem(c->net.row_cap), s, A, g, (float*)nullptr,
                    iv ? 0 : 1, codes_next, (const epi_net*)c->net_dev, rcount_next,
                    (const MsgTables*)c->msg_dev, (const MsgComb*)c->comb_dev));
    else
      CK(launch_pdl(k_pass<false, 1>, dim3(grid), dim3(256), (size_t)0, s, A, g, codes_cur, (void*)nullptr,
                    c->host.rate_scale, iv ? 0 : 1, codes_next, (const epi_net*)c->net_dev, rcount_next,
                    (const MsgTables*)c->msg_dev));
    CKL();
  } else {
    if (ev) CK(cudaEventRecord((cudaEvent_t)ev[1], s));
    const int fgrid = balanced_grid(c->hi - c->lo, 128, c->day_blocks_per_sm);
    NextTables nx{};
    if (merged) {
      nx.wt = c->wt_dev[par ^ 1][2];
      nx.keys = nt_next;
      nx.keys_out = c->ntab_dev[(step + 2) % 3];
      nx.rperm_t2 = key_prefix(seed, step + 2, P_NET_RPERM);
      nx.nk = make_net_keys(seed, step + 1);
    } else if (sparse && whole) {
      nx.wt = c->wt_dev[par ^ 1][3];
      nx.keys = nt_next;                  // (written by today's day tables; the day after's too)
      nx.keys_out = nullptr;
    }
    const int push = push_rand ? 1 : (sparse ? 2 : 0);
    CK(launch_pdl_w(&c->hot, push == 1 ? k_fused_step<1> : push == 2 ? k_fused_step<2> : k_fused_step<0>,
                    dim3(fgrid), dim3(128), 0, s, A, c->net, nk, codes_cur,
                    c->host.rate_scale, codes_next, (const epi_net*)c->net_dev, rcount_next, iv ? 0 : 1, wt,
                    (const MsgTables*)c->msg_dev, (const NetTables*)nt_today, nx, push, DayTests{}));
    c->merged_ready = merged ? step + 1 : -1;
    c->sparse_ready = sparse && whole ? step + 1 : -1;
    c->sparse_clean = sparse ? step + 1 : -1;   // (the day's consumed rows were cleared)
  }
  if (ev) CK(cudaEventRecord((cudaEvent_t)ev[2], s));
  if (iv) {
    if (c->host.den_enabled) {
      // who died yesterday (the day's code vector is complete here)
      k_died_update<<<grid_for(c->n, 256), 256, 0, s>>>(codes_cur, c->n, step, c->died_at);
      CKL();
    }
    int rc = run_interventions(c, A, codes_next, c->net_dev, rcount_next, vax_open, s, [&](bool part) -> int {
      // contacts of the notifiers over steps step-L .. step-1, regenerated
      DenRegen D{};
      D.first_day = step - c->host.den_lookback > 0 ? step - c->host.den_lookback : 0;
      D.n_days = step - D.first_day;
      if (D.n_days <= 0) return 0;
      for (int d = 0; d < D.n_days; ++d) D.nk[d] = make_net_keys(seed, D.first_day + d);
      if (!c->host.testing_enabled) return 0;           // no test results, no notifiers
      const int g = sm_count() * 8;                    // persistent: items read on the device
      if (!part) {
        k_den_regen<<<g, 256, 0, s>>>(c->net, D, c->died_at, c->den_list, c->den_count, c->flags,
                                      (const Radix*)c->ntab_dev[0]->wrad);
        CKL();
        return 0;
      }
      // partitioned: contacts may be anyone's; OR the ranks' marks together
      CK(cudaMemsetAsync(c->den_mark, 0, (size_t)c->n, s));
      k_den_regen<<<g, 256, 0, s>>>(c->net, D, c->died_at, c->den_list, c->den_count, c->den_mark,
                                    (const Radix*)c->ntab_dev[0]->wrad);
      CKL();
      int rc2 = exchange(c, EPI_X_OR_U8, c->den_mark, c->n, s);
      if (rc2) return rc2;
      k_den_merge<<<grid_for(c->hi - c->lo, 256), 256, 0, s>>>(c->den_mark, c->lo, c->hi, c->flags);
      CKL();
      return 0;
    });
    if (rc) return rc;
  }
  if (ev) CK(cudaEventRecord((cudaEvent_t)ev[3], s));
  return 0;
}

int epi_sim_step(epi_ctx* c, const epi_state* st, int32_t step, uint64_t seed, int32_t mode,
                 int32_t precision, const uint16_t* codes_cur, uint16_t* codes_next, int64_t* record,
                 int32_t* vax_open, void* stream) {
  int rc = sim_step_impl(c, st, step, seed, mode, precision, codes_cur, codes_next, record, vax_open,
                         nullptr, stream);
  if (!rc) rc = gather_codes(c, codes_next, S(stream));
  if (!rc) rc = join_side(c, S(stream));
  return rc;
}

// k_fused_run: one block per SM, threads = the SM's agents rounded up to a warp
static int64_t run_threads(int64_t n) {
  const int64_t sms = sm_count();
  const int64_t per = (n + sms - 1) / sms;
  return (per + 31) / 32 * 32;
}

// Can the merged days of a run go to k_fused_run (one co-resident thread per
// agent)?  Same conditions as the merged per-day path plus residency.
static bool persistent_ok(epi_ctx* c, int32_t mode, int32_t precision) {
  if (!c->persistent || mode != 1 || precision != EPI_F32 || interventions_on(c->host)) return false;
  if (partitioned(c) || c->net.n_agents < 2 || c->net.random_slots != RT_SLOTS || !batched(&c->net) ||
      !push_fits(c) || c->net.colleague_draws > 8)
    return false;
  const int64_t threads = run_threads(c->n);
  if (threads > RUN_BIG_AGENTS) return false;
  const bool big = threads > RUN_MAX_AGENTS;
  static int per_sm[2] = {-1, -1};
  int& ps = per_sm[big ? 1 : 0];
  if (ps < 0) {
    cudaError_t e;
    if (big) {
      e = cudaFuncSetAttribute(k_fused_run<RUN_BIG_THREADS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)run_dyn_smem<RUN_BIG_THREADS>());
      if (e == cudaSuccess)
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps, k_fused_run<RUN_BIG_THREADS>, RUN_BIG_THREADS,
                                                          run_dyn_smem<RUN_BIG_THREADS>());
    } else {
      e = cudaFuncSetAttribute(k_fused_run<RUN_MAX_THREADS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)run_dyn_smem<RUN_MAX_THREADS>());
      if (e == cudaSuccess)
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps, k_fused_run<RUN_MAX_THREADS>, RUN_MAX_THREADS,
                                                          run_dyn_smem<RUN_MAX_THREADS>());
    }
    if (e != cudaSuccess) {
      cudaGetLastError();
      ps = 0;
    }
  }
  return ps >= 1;
}

// The persistent kernels' colleague rows, [2][member slots][16] codes, zeroed
// once (every launch leaves them zero).
static int run_crow(epi_ctx* c, cudaStream_t s, uint16_t* out[2]) {
  const size_t len = (size_t)16 * (size_t)(c->net.n_member_slots > 0 ? c->net.n_member_slots : 1);
  if (!c->run_crow) {
    int rc = dalloc(&c->run_crow, 2 * len);
    if (rc) return rc;
    CK(cudaMemsetAsync(c->run_crow, 0, 2 * len * sizeof(uint16_t), s));
  }
  out[0] = c->run_crow;
  out[1] = c->run_crow + len;
  return 0;
}

static int launch_run(epi_ctx* c, const epi_state* st, int32_t first, int32_t n_days, uint64_t seed,
                      uint16_t* codes0, uint16_t* codes1, int64_t* records, cudaStream_t s) {
  if (!c->run_barrier) CK(dmalloc((void**)&c->run_barrier, sizeof(unsigned)));
  if (!c->run_wtab) {
    int rc = dalloc(&c->run_wtab, (size_t)6 * (c->net.n_workplaces > 0 ? c->net.n_workplaces : 1));
    if (rc) return rc;
  }
  const bool big = run_threads(c->n) > RUN_MAX_AGENTS;      // (the 1024-thread variant)
  uint16_t* crow[2] = {nullptr, nullptr};
  if (!big) {
    int rc = run_crow(c, s, crow);
    if (rc) return rc;
  }
  CK(cudaMemsetAsync(c->run_barrier, 0, sizeof(unsigned), s));
  RunArgs R{};
  R.P = c->P;
  R.st = *st;
  R.seed = seed;
  R.first_step = first;
  R.n_days = n_days;
  R.records = (long long*)records;
  R.codes[0] = codes0;
  R.codes[1] = codes1;
  R.wt[0] = c->wt_host[0];
  R.wt[1] = c->wt_host[1];
  R.ring_t2 = c->ntab_dev[(first + n_days + 1) % 3];
  R.mt = (const MsgTables*)c->msg_dev;
  R.tau_lut = c->tau_lut;
  R.dn = c->ntab.dn;
  R.barrier = c->run_barrier;
  R.probe = c->probe;
  R.wtab = c->run_wtab;
  R.crow[0] = crow[0];
  R.crow[1] = crow[1];
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)sm_count());
  cfg.blockDim = dim3((unsigned)run_threads(c->n) + 32);     // + the service warp
  cfg.dynamicSmemBytes = big ? run_dyn_smem<RUN_BIG_THREADS>() : run_dyn_smem<RUN_MAX_THREADS>();
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;     // every block resident: the grid barrier is safe
  attr[0].val.cooperative = 1;
  cfg.numAttrs = 1;
  if (c->hot.bytes > 0) {
    attr[1].id = cudaLaunchAttributeAccessPolicyWindow;
    attr[1].val.accessPolicyWindow.base_ptr = const_cast<void*>(c->hot.base);
    attr[1].val.accessPolicyWindow.num_bytes = c->hot.bytes;
    attr[1].val.accessPolicyWindow.hitRatio = c->hot.hit_ratio;
    attr[1].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr[1].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    cfg.numAttrs = 2;
  }
  cfg.attrs = attr;
  if (big) CK(cudaLaunchKernelEx(&cfg, k_fused_run<RUN_BIG_THREADS>, R, c->net));
  else CK(cudaLaunchKernelEx(&cfg, k_fused_run<RUN_MAX_THREADS>, R, c->net));
  c->merged_ready = first + n_days;
  c->sparse_ready = -1;
  c->sparse_clean = -1;
  return 0;
}

// Intervention days in one persistent launch (k_iv_run): the fused
// intervention day's conditions + one resident thread per agent.
static bool persistent_iv_ok(epi_ctx* c, int32_t mode, int32_t precision) {
  if (!c->persistent || !c->iv_fusion || mode != 1 || precision != EPI_F32 || !interventions_on(c->host))
    return false;
  if (partitioned(c) || c->net.n_agents < 2 || c->net.random_slots != RT_SLOTS || !batched(&c->net) ||
      !push_fits(c) || c->net.colleague_draws > 8)
    return false;
  static int per_sm = -1;
  if (per_sm < 0 &&
      (cudaFuncSetAttribute(k_iv_run, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)IV_DYN_SMEM) !=
           cudaSuccess ||
       cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_iv_run, RUN_MAX_THREADS, IV_DYN_SMEM) !=
           cudaSuccess))
    per_sm = 0;
  return per_sm >= 1 && run_threads(c->n) <= RUN_MAX_AGENTS;
}

static int launch_iv_run(epi_ctx* c, const epi_state* st, int32_t first, int32_t n_days, uint64_t seed,
                         uint16_t* codes0, uint16_t* codes1, int64_t* records, int32_t* vax_open, cudaStream_t s) {
  const epi_params& p = c->host;
  if (p.vaccination_enabled && !vax_open) return fail(EPI_EARG, "vaccination enabled but no vax_open latch given");
  int rc = 0;
  if (!c->ivr_hist) rc = dalloc(&c->ivr_hist, (size_t)3 * IV_HIST);
  if (!rc && !c->ivr_tile_hist) rc = dalloc(&c->ivr_tile_hist, (size_t)2 * sm_count() * NUM_BUCKETS);
  if (rc) return rc;
  if (!c->run_barrier) CK(dmalloc((void**)&c->run_barrier, sizeof(unsigned)));
  CK(cudaMemsetAsync(c->run_barrier, 0, sizeof(unsigned), s));
  CK(cudaMemsetAsync(c->ivr_hist, 0, (size_t)3 * IV_HIST * sizeof(unsigned long long), s));
  IvRunArgs R{};
  R.A0 = make_args(c, st, first, seed, nullptr, nullptr, true);
  R.seed = seed;
  R.first_step = first;
  R.n_days = n_days;
  R.records = (long long*)records;
  R.codes[0] = codes0;
  R.codes[1] = codes1;
  R.wt[0] = c->wt_host[0];
  R.wt[1] = c->wt_host[1];
  R.ring_t2 = c->ntab_dev[(first + n_days + 1) % 3];
  R.mt = (const MsgTables*)c->msg_dev;
  R.wrad = (const Radix*)c->ntab_dev[0]->wrad;
  R.dn = c->ntab.dn;
  R.barrier = c->run_barrier;
  R.bucket = c->bucket;
  R.hist = c->ivr_hist;
  R.tile_hist = c->ivr_tile_hist;
  R.vax_open = vax_open;
  const bool listed = p.den_enabled && p.testing_enabled && c->den_list != nullptr;
  R.den_list = listed ? c->den_list : nullptr;
  R.den_count = listed ? c->den_count : nullptr;
  R.den_stride = c->n;
  R.died_at = p.den_enabled ? c->died_at : nullptr;
  R.den_lookback = p.den_lookback;
  R.den = listed ? 1 : 0;
  R.tests = p.testing_enabled ? 1 : 0;
  R.post = (p.den_enabled || p.quarantine_enabled || p.vaccination_enabled) ? 1 : 0;
  R.vax = p.vaccination_enabled ? 1 : 0;
  if (!c->run_wtab) {
    int rc2 = dalloc(&c->run_wtab, (size_t)6 * (c->net.n_workplaces > 0 ? c->net.n_workplaces : 1));
    if (rc2) return rc2;
  }
  R.wtab = c->run_wtab;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)sm_count());
  cfg.blockDim = dim3((unsigned)run_threads(c->n) + 32);
  cfg.dynamicSmemBytes = IV_DYN_SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.numAttrs = 1;
  if (c->hot.bytes > 0) {
    attr[1].id = cudaLaunchAttributeAccessPolicyWindow;
    attr[1].val.accessPolicyWindow.base_ptr = const_cast<void*>(c->hot.base);
    attr[1].val.accessPolicyWindow.num_bytes = c->hot.bytes;
    attr[1].val.accessPolicyWindow.hitRatio = c->hot.hit_ratio;
    attr[1].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr[1].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    cfg.numAttrs = 2;
  }
  cfg.attrs = attr;
  CK(cudaLaunchKernelEx(&cfg, k_iv_run, R, c->net));
  c->merged_ready = first + n_days;
  c->sparse_ready = -1;
  c->sparse_clean = -1;
  // the per-day path resumes with an empty histogram (k_iv_run used its own)
  if (c->iv_hist) CK(cudaMemsetAsync(c->iv_hist, 0, (size_t)2 * NUM_BUCKETS * sizeof(unsigned long long), s));
  return 0;
}

int epi_run_persistent(epi_ctx* c, int32_t mode, int32_t precision) {
  if (!c) return fail(EPI_EARG, "null ctx");
  return c->has_net && (persistent_ok(c, mode, precision) || persistent_iv_ok(c, mode, precision)) ? 1 : 0;
}

int epi_quartiles(const int64_t* data, int64_t n_rep, int32_t horizon, int32_t rec_len, const int32_t* cols,
                  int32_t n_cols, double* out, void* stream) {
  if (!data || !cols || !out || n_rep < 1 || horizon < 0 || rec_len < 1 || n_cols < 0)
    return fail(EPI_EARG, "bad argument");
  if (horizon == 0 || n_cols == 0) return 0;
  if (n_rep > SUMMARY_MAX_R) {
    k_quartiles_large<<<dim3((unsigned)horizon, (unsigned)n_cols), 1024, 0, S(stream)>>>(data, n_rep, horizon,
                                                                                        rec_len, cols, out);
    CKL();
    return 0;
  }
  k_quartiles<<<dim3((unsigned)horizon, (unsigned)n_cols), 1024, 0, S(stream)>>>(data, (int)n_rep, horizon, rec_len,
                                                                                  cols, out);
  CKL();
  return 0;
}

int epi_set_day_grid(epi_ctx* c, int32_t blocks_per_sm) {
  if (!c || blocks_per_sm < 0) return fail(EPI_EARG, "bad argument");
  c->day_blocks_per_sm = blocks_per_sm == 0 ? 16 : blocks_per_sm;
  return 0;
}

int epi_set_sparse_push(epi_ctx* c, int32_t on) {
  if (!c) return fail(EPI_EARG, "null ctx");
  c->sparse_push = on != 0;
  c->sparse_ready = -1;
  c->sparse_clean = -1;
  return 0;
}

int epi_set_iv_fusion(epi_ctx* c, int32_t on) {
  if (!c) return fail(EPI_EARG, "null ctx");
  c->iv_fusion = on != 0;
  c->merged_ready = -1;
  c->sparse_ready = -1;
  c->sparse_clean = -1;
  return 0;
}

int epi_comm_unique_id(uint8_t* out) {
  const NcclApi* api = nccl_api();
  if (!api) return fail(EPI_ECUDA, "libnccl.so.2 not found");
  if (!out) return fail(EPI_EARG, "null argument");
  ncclUniqueId id;
  const ncclResult_t r = api->get_unique_id(&id);
  if (r != ncclSuccess) return fail(EPI_ECUDA, std::string("ncclGetUniqueId: ") + api->error_string(r));
  std::memcpy(out, id.internal, NCCL_UNIQUE_ID_BYTES);
  return 0;
}

int epi_comm_create(const uint8_t* id, int32_t world, int32_t rank, epi_comm** out) {
  const NcclApi* api = nccl_api();
  if (!api) return fail(EPI_ECUDA, "libnccl.so.2 not found");
  if (!id || !out || world < 1 || rank < 0 || rank >= world) return fail(EPI_EARG, "bad argument");
  ncclUniqueId uid;
  std::memcpy(uid.internal, id, NCCL_UNIQUE_ID_BYTES);
  epi_comm* m = new epi_comm();
  m->world = world;
  m->rank = rank;
  const ncclResult_t r = api->comm_init_rank(&m->comm, world, uid, rank);
  if (r != ncclSuccess) {
    delete m;
    return fail(EPI_ECUDA, std::string("ncclCommInitRank: ") + api->error_string(r));
  }
  *out = m;
  return 0;
}

int epi_comm_destroy(epi_comm* m) {
  if (!m) return 0;
  const NcclApi* api = nccl_api();
  if (api && m->comm) api->comm_destroy(m->comm);
  delete m;
  return 0;
}

int epi_set_code_exchange(epi_ctx* c, epi_comm* comm, int32_t mode, int64_t chunk) {
  if (!c || mode < 0 || mode > 2 || (mode > 0 && chunk < 1)) return fail(EPI_EARG, "bad argument");
  if (mode == 2) {
    if (!comm) return fail(EPI_EARG, "NCCL code exchange without a communicator");
    if ((int64_t)comm->world * chunk < c->n) return fail(EPI_EARG, "world * chunk does not cover the agents");
    if (c->lo != (int64_t)comm->rank * chunk) return fail(EPI_EARG, "owned rows do not start at rank * chunk");
  }
  if (mode == 1 && !c->xfn) return fail(EPI_EARG, "callback code exchange without epi_set_exchange");
  c->gather_mode = mode;
  c->comm = mode == 2 ? comm : nullptr;
  c->gather_chunk = chunk;
  return 0;
}

int epi_allgather_codes(epi_ctx* c, uint16_t* codes, void* stream) {
  if (!c || !codes) return fail(EPI_EARG, "null argument");
  return gather_codes(c, codes, S(stream));
}

int epi_set_sigma_ahead(epi_ctx* c, int32_t on) {
  if (!c) return fail(EPI_EARG, "null ctx");
  c->sigma_ahead = on != 0;
  c->sigma_day = -1;
  return 0;
}

int epi_set_lambda_probe(epi_ctx* c, float* out, int32_t first_step, int32_t n_days) {
  if (!c || n_days < 0 || (n_days > 0 && !out)) return fail(EPI_EARG, "bad argument");
  c->probe.out = n_days > 0 ? out : nullptr;
  c->probe.n = c->n;
  c->probe.first = first_step;
  c->probe.days = n_days;
  return 0;
}

int epi_set_persistent(epi_ctx* c, int32_t on) {
  if (!c) return fail(EPI_EARG, "null ctx");
  c->persistent = on != 0;
  return 0;
}

int epi_sim_run(epi_ctx* c, const epi_state* st, int32_t first_step, int32_t n_days, uint64_t seed,
                int32_t mode, int32_t precision, uint16_t* codes0, uint16_t* codes1, int64_t* records,
                int32_t* vax_open, void* stream) {
  if (!c || !records || !codes0 || !codes1 || n_days < 0) return fail(EPI_EARG, "bad argument");
  CK(cudaMemsetAsync(records, 0, (size_t)n_days * EPI_REC_LEN * sizeof(int64_t), S(stream)));
  const bool iv_run = n_days >= 2 && c->has_net && st && st->n_agents == c->n && persistent_iv_ok(c, mode, precision);
  if (iv_run) {
    // day 0 of the chain on the per-day path (tables, death days, counters);
    // every later day in one launch
    int d0 = 0;
    if (c->merged_ready != first_step) {
      const int t = first_step;
      int rc = sim_step_impl(c, st, t, seed, mode, precision, (t & 1) ? codes1 : codes0, (t & 1) ? codes0 : codes1,
                             records, vax_open, nullptr, stream, false);
      if (rc) return rc;
      d0 = 1;
    }
    if (n_days - d0 >= 1) {
      // the per-day path's notifier list / histogram state is not carried over
      if (c->den_count) CK(cudaMemsetAsync(c->den_count, 0, 3 * sizeof(int), S(stream)));
      return launch_iv_run(c, st, first_step + d0, n_days - d0, seed, codes0, codes1,
                           records + (size_t)d0 * EPI_REC_LEN, vax_open, S(stream));
    }
    return 0;
  }
  if (n_days >= 2 && c->has_net && st && st->n_agents == c->n && persistent_ok(c, mode, precision)) {
    // the first day on the per-day path builds the day's tables (unless a
    // previous merged day already did); every later day in one launch
    int d0 = 0;
    if (c->merged_ready != first_step) {
      const int t = first_step;
      int rc = sim_step_impl(c, st, t, seed, mode, precision, (t & 1) ? codes1 : codes0, (t & 1) ? codes0 : codes1,
                             records, vax_open, nullptr, stream, false);
      if (rc) return rc;
      d0 = 1;
    }
    // launches of <= RUN_MAX_DAYS days
    for (int d = d0; d < n_days; d += RUN_MAX_DAYS) {
      const int nd = n_days - d < RUN_MAX_DAYS ? n_days - d : RUN_MAX_DAYS;
      if (nd == 1) {
        const int t = first_step + d;
        int rc = sim_step_impl(c, st, t, seed, mode, precision, (t & 1) ? codes1 : codes0,
                               (t & 1) ? codes0 : codes1, records + (size_t)d * EPI_REC_LEN, vax_open, nullptr,
                               stream, false);
        if (rc) return rc;
        continue;
      }
      int rc = launch_run(c, st, first_step + d, nd, seed, codes0, codes1, records + (size_t)d * EPI_REC_LEN,
                          S(stream));
      if (rc) return rc;
    }
    return 0;
  }
  // one day at a time (partitioned ranks: the day's code exchange between
  // days; tomorrow's sigma tables on the side stream meanwhile)
  for (int d = 0; d < n_days; ++d) {
    const int t = first_step + d;
    uint16_t* cur = (t & 1) ? codes1 : codes0;
    uint16_t* nxt = (t & 1) ? codes0 : codes1;
    int rc = sim_step_impl(c, st, t, seed, mode, precision, cur, nxt, records + (size_t)d * EPI_REC_LEN,
                           vax_open, nullptr, stream, false);
    if (!rc) rc = gather_codes(c, nxt, S(stream));
    if (rc) return rc;
  }
  return join_side(c, S(stream));
}

int epi_sim_step_timed(epi_ctx* c, const epi_state* st, int32_t step, uint64_t seed, int32_t mode,
                       int32_t precision, const uint16_t* codes_cur, uint16_t* codes_next,
                       int64_t* record, int32_t* vax_open, void* const* events4, void* stream) {
  if (!events4) return fail(EPI_EARG, "events4 is null");
  return sim_step_impl(c, st, step, seed, mode, precision, codes_cur, codes_next, record, vax_open,
                       events4, stream);
}

int epi_net_generate(epi_ctx* c, int32_t step, uint64_t seed, const uint16_t* codes_cur, void* stream) {
  if (!c || !c->has_net || !codes_cur) return fail(EPI_EARG, "needs an attached network and codes");
  if (!batched(&c->net)) return fail(EPI_EARG, "epi_net_generate needs <= 16 slots and <= 8 draws");
  if (c->net.row_cap > MP_MAX_CAP) return fail(EPI_EARG, "epi_net_generate needs row_cap <= 128");
  cudaStream_t s = S(stream);
  const NetKeys nk = make_net_keys(seed, step);
  NetTables* nt = c->ntab_dev[step % 3];
  k_day_keys<<<1, 32, 0, s>>>(nt, nk.rperm, nullptr);
  CKL();
  const bool has_work = c->net.n_member_slots > 0 && c->net.colleague_draws > 0;
  WorkTables w = c->wt_host[step & 1];
  w.wcode = nullptr;
  w.rin = nullptr;
  w.rout = nullptr;
  c->merged_ready = -1;
  c->sparse_ready = -1;
  c->sparse_clean = -1;
  if (has_work) {
    k_day_tables<<<grid_for(c->net.n_member_slots, 256, 4), 256, 0, s>>>(
        c->net, nk, w, codes_cur, c->lo, c->hi, grid_for(c->net.n_member_slots, 256, 4), nt,
        c->ntab_dev[(step + 1) % 3], key_prefix(seed, step + 1, P_NET_RPERM), nullptr);
    CKL();
  }
  return launch_realize(&c->net, seed, step, codes_cur, nullptr, c->net_msgs, c->net_toff,
                        c->net_rowlen[0], 0, nullptr, has_work ? c->wt_dev[step & 1][0] : nullptr, c->lo,
                        c->hi, s, nt);
}

int epi_net_gather(epi_ctx* c, const epi_state* st, int32_t step, const uint16_t* codes_cur,
                   float* lambda_out, int64_t* record, void* stream) {
  if (!c || !c->has_net || !st || !lambda_out) return fail(EPI_EARG, "null argument");
  long long* rec = record ? (long long*)record : c->scratch_rec;
  if (record) CK(cudaMemsetAsync(rec, 0, EPI_REC_LEN * sizeof(long long), S(stream)));
  StepArgs A = make_args(c, st, step, 0, rec, nullptr, false);
  CsrView g{nullptr, c->net_rowlen[0], nullptr, c->net.row_cap, c->net_msgs, c->net_toff};
  k_msg_pass<0><<<msg_pass_grid<0>(c->net.row_cap, c->hi - c->lo), MP_WARPS * 32,
                  msg_pass_smem(c->net.row_cap), S(stream)>>>(A, g, lambda_out, 0, nullptr, nullptr, 0,
                                                              (const MsgTables*)c->msg_dev,
                                                              (const MsgComb*)c->comb_dev);
  CKL();
  return 0;
}

int epi_seed_infections(epi_ctx* c, const epi_state* st, uint64_t seed, const int64_t* ids, int64_t n,
                        void* stream) {
  if (!c || !st) return fail(EPI_EARG, "null argument");
  if (n <= 0) return 0;
  k_seed<<<grid_for(n, 256), 256, 0, S(stream)>>>(c->P, *st, make_step_keys(seed, 0), ids, n);
  CKL();
  return 0;
}

int epi_assign_app(const epi_state* st, uint64_t seed, double adoption, void* stream) {
  if (!st) return fail(EPI_EARG, "null argument");
  k_assign_app<<<grid_for(st->n_agents, 256), 256, 0, S(stream)>>>(*st, key_prefix(seed, 0, P_APP), adoption);
  CKL();
  return 0;
}

struct epi_refnet_t {
  RefNet net{};
  RefScratch sc{};
  int64_t n_member_slots = 0;
  int ws_blocks = 1;            // blocks per occupation: the largest lattice / 256
  void* scan_tmp = nullptr;
  size_t scan_bytes = 0;
};

int epi_refnet_create(const epi_refnet_desc* d, epi_refnet_t** out) {
  if (!d || !out || d->n_agents < 1 || d->n_agents >= (1ll << 30) || d->n_occ < 0)
    return fail(EPI_EARG, "bad reference-network descriptor");
  if (d->table_slots < 2 || (d->table_slots & (d->table_slots - 1)))
    return fail(EPI_EARG, "table_slots must be a power of two");
  epi_refnet_t* r = new epi_refnet_t();
  RefNet& n = r->net;
  n.n_agents = d->n_agents;
  n.hh_members = d->hh_members;
  n.hh_start = d->hh_start;
  n.hh_size = d->hh_size;
  n.n_occ = d->n_occ;
  n.occ_members = d->occ_members;
  n.occ_start = d->occ_start;
  n.occ_k = d->occ_k;
  n.beta = d->rewire_beta;
  n.random_degree = d->random_degree;
  RefScratch& S = r->sc;
  int rc = dalloc(&S.live_members, (size_t)d->n_member_slots + 1);
  if (!rc) rc = dalloc(&S.occ_live, (size_t)d->n_occ + 1);
  if (!rc) rc = dalloc(&S.stub_count, (size_t)d->n_agents + 1);
  if (!rc) rc = dalloc(&S.stub_off, (size_t)d->n_agents + 1);
  if (!rc) rc = dalloc(&S.table, (size_t)d->table_slots * 2);
  if (!rc) rc = dalloc(&S.counter, 2);
  S.table_slots = d->table_slots;
  r->n_member_slots = d->n_member_slots;
  if (!rc) {   // one-time host reads: the stub bound and the largest lattice
    std::vector<double> deg((size_t)d->n_agents);
    std::vector<int32_t> occ_start((size_t)d->n_occ + 1), occ_k((size_t)d->n_occ + 1);
    if (cudaMemcpy(deg.data(), d->random_degree, deg.size() * sizeof(double), cudaMemcpyDeviceToHost) !=
            cudaSuccess ||
        (d->n_occ > 0 &&
         (cudaMemcpy(occ_start.data(), d->occ_start, ((size_t)d->n_occ + 1) * sizeof(int32_t),
                     cudaMemcpyDeviceToHost) != cudaSuccess ||
          cudaMemcpy(occ_k.data(), d->occ_k, (size_t)d->n_occ * sizeof(int32_t), cudaMemcpyDeviceToHost) !=
              cudaSuccess))) {
      rc = fail(EPI_ECUDA, "descriptor read");
    } else {
      int64_t stubs = 0;
      for (double x : deg) stubs += (int64_t)std::ceil(x > 0 ? x : 0.0);
      S.max_stubs = stubs;
      int64_t most = 0, lattice = 0;
      for (int j = 0; j < d->n_occ; ++j) {
        const int64_t e = (int64_t)(occ_start[j + 1] - occ_start[j]) * std::max(occ_k[j] / 2, 0);
        most = std::max(most, e);
        lattice += e;
      }
      S.loser_cap = lattice;
      if (!rc) rc = dalloc(&S.ws_losers, (size_t)lattice + 1);
      if (!rc) rc = dalloc(&S.n_losers, 1);
      if (!rc) rc = dalloc(&S.links_done, 1);
      if (!rc && cudaMemset(S.links_done, 0, sizeof(unsigned)) != cudaSuccess) rc = fail(EPI_ECUDA, "memset");
      r->ws_blocks = (int)std::min<int64_t>(std::max<int64_t>((most + 255) / 256, 1), 1024);
      if (!rc) rc = dalloc(&S.stub_owner, (size_t)stubs + 1);
      if (!rc) rc = dalloc(&S.pair_uv, (size_t)(stubs / 2) + 1);
    }
  }
  if (!rc) {
    size_t need = 0;
    if (cub::DeviceScan::ExclusiveSum(nullptr, need, S.stub_count, S.stub_off, (int)(d->n_agents + 1)) !=
        cudaSuccess)
      rc = fail(EPI_ECUDA, "scan sizing");
    else if (cudaMalloc(&r->scan_tmp, need + 16) != cudaSuccess)
      rc = fail(EPI_ECUDA, "scan scratch");
    r->scan_bytes = need + 16;
  }
  if (rc) {
    epi_refnet_destroy(r);
    return rc;
  }
  *out = r;
  return 0;
}

int epi_refnet_destroy(epi_refnet_t* r) {
  if (!r) return 0;
  dfree_now(r->sc.live_members);
  dfree_now(r->sc.occ_live);
  dfree_now(r->sc.stub_count);
  dfree_now(r->sc.stub_off);
  dfree_now(r->sc.table);
  dfree_now(r->sc.counter);
  dfree_now(r->sc.stub_owner);
  dfree_now(r->sc.pair_uv);
  dfree_now(r->sc.ws_losers);
  dfree_now(r->sc.n_losers);
  dfree_now(r->sc.links_done);
  dfree_now(r->scan_tmp);
  delete r;
  return 0;
}

static int refnet_realize_impl(epi_refnet_t* r, uint64_t seed, int32_t step, DeadView dead, int32_t* src,
                               int32_t* dst, int8_t* kind, int64_t capacity, int64_t* n_edges, uint64_t* count_dev,
                               void* stream, int32_t* row_len = nullptr, bool counter_zeroed = false);

int epi_refnet_realize(epi_refnet_t* r, uint64_t seed, int32_t step, const uint8_t* dead, int32_t* src,
                       int32_t* dst, int8_t* kind, int64_t capacity, int64_t* n_edges, void* stream) {
  if (!n_edges) return fail(EPI_EARG, "null argument");
  return refnet_realize_impl(r, seed, step, DeadView{(const int8_t*)dead, 1}, src, dst, kind, capacity, n_edges,
                             nullptr, stream);
}

int epi_refnet_realize_counted(epi_refnet_t* r, uint64_t seed, int32_t step, const uint8_t* dead, int32_t* src,
                               int32_t* dst, int8_t* kind, int64_t capacity, uint64_t* count, void* stream) {
  if (!count) return fail(EPI_EARG, "null argument");
  return refnet_realize_impl(r, seed, step, DeadView{(const int8_t*)dead, 1}, src, dst, kind, capacity, nullptr,
                             count, stream);
}

static int refnet_realize_impl(epi_refnet_t* r, uint64_t seed, int32_t step, DeadView dead, int32_t* src,
                               int32_t* dst, int8_t* kind, int64_t capacity, int64_t* n_edges, uint64_t* count_dev,
                               void* stream, int32_t* row_len, bool counter_zeroed) {
  if (!r || !dead.p || !src || !dst || !kind) return fail(EPI_EARG, "null argument");
  cudaStream_t s = S(stream);
  RefScratch S = r->sc;
  S.out_src = src;
  S.out_dst = dst;
  S.out_kind = kind;
  S.capacity = capacity;
  S.row_len = row_len;
  const int64_t n = r->net.n_agents;
  if (count_dev) S.counter = (unsigned long long*)count_dev;   // counted mode: the caller's words are the counter
  if (!counter_zeroed) CK(cudaMemsetAsync(S.counter, 0, 2 * sizeof(unsigned long long), s));
  // 1: households + stub counts (+ table clear)
  CK(launch_pdl(k_ref_agents, dim3(grid_for(std::max<int64_t>(n, S.table_slots), 256)), dim3(256), 0, s, r->net,
                dead, S, key_prefix(seed, step, P_REF_STUB)));
  size_t bytes = r->scan_bytes;
  CK(cub::DeviceScan::ExclusiveSum(r->scan_tmp, bytes, S.stub_count, S.stub_off, (int)(n + 1), s));
  // 2: alive members per occupation + stub owners
  CK(launch_pdl(k_ref_occ_stubs, dim3(r->net.n_occ + grid_for(n, kOccLiveThreads, 2)), dim3(kOccLiveThreads), 0, s,
                r->net, dead, S));
  // 3, 4: lattices + stub pairs, inserts then winners
  const uint64_t ws = key_prefix(seed, step, P_REF_WS);
  const PermKeys K = random_slot_keys(key_prefix(seed, step, P_REF_PERM), 0);
  const int ws_blocks = r->net.n_occ > 0 ? r->ws_blocks : 0;
  const int links = ws_blocks * r->net.n_occ + grid_for(S.max_stubs / 2, 256);
  CK(launch_pdl(k_ref_links<0>, dim3(links), dim3(256), 0, s, r->net, S, ws, K, ws_blocks));
  CK(launch_pdl(k_ref_links<1>, dim3(links), dim3(256), 0, s, r->net, S, ws, K, ws_blocks));
  // (the rewired lattice edges whose pair was taken draw again in launch 4's
  // last block: the edge count is preserved)
  if (count_dev) return 0;                  // no synchronisation: count + error bits stay on the device
  unsigned long long h[2] = {0, 0};
  CK(cudaMemcpyAsync(h, S.counter, sizeof(h), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  *n_edges = (int64_t)h[0];
  if (h[1] & 1ull) return fail(EPI_EARG, "edge output capacity exceeded");
  if (h[1] & 2ull) return fail(EPI_EARG, "dedupe hash table full");
  if (h[1] & 4ull) return fail(EPI_EARG, "more than 2^31 random-network stubs");
  if (h[1] & 8ull) return fail(EPI_EARG, "rewiring collision list overflow");
  return 0;
}

// The reference's replication loop (runner.py:138-150) for steps
// [first, last) with every step issued from here: dead mask from the stage,
// (graph_seed = the GraphRealizer's seed, seed = the Engine's),
// realize (counted), graph load (counted), Engine.step.  No host
// synchronisation; counts[(t - first) * 2 + {0, 1}] = edges / realizer error
// bits, records[(t - first) * EPI_REC_LEN ...] = the step's record.
int epi_refnet_run(epi_refnet_t* r, epi_ctx* c, const epi_state* st, uint64_t graph_seed, uint64_t seed,
                   int32_t first, int32_t last, int32_t* src, int32_t* dst, int8_t* kind, int64_t capacity,
                   uint64_t* counts, int64_t* records, int32_t* vax_open, void* stream) {
  if (!r || !c || !st || !counts || !records) return fail(EPI_EARG, "null argument");
  if (st->n_agents != c->n || r->net.n_agents != c->n) return fail(EPI_EARG, "state size differs from context");
  if (c->host.den_enabled)
    return fail(EPI_EARG, "a device-counted graph cannot feed the exposure-notification contact log");
  if (first < 0 || last < first) return fail(EPI_EARG, "bad step range");
  if (last == first) return 0;
  cudaStream_t s = S(stream);
  const int64_t steps = last - first;
  CK(cudaMemsetAsync(counts, 0, (size_t)steps * 2 * sizeof(uint64_t), s));
  CK(cudaMemsetAsync(records, 0, (size_t)steps * EPI_REC_LEN * sizeof(int64_t), s));
  const DeadView dead{st->stage, (int8_t)S_DEAD};   // the realizer reads the stage column in place
  // Without interventions the update of step t writes the codes of step t+1
  // (ping-pong between c->codes and c->codes_alt): no k_codes launch after
  // the first step.
  const bool chain = !interventions_on(c->host);
  if (chain && !c->codes_alt) {
    int rc = dalloc(&c->codes_alt, (size_t)c->n);
    if (rc) return rc;
  }
  uint16_t* cbuf[2] = {c->codes, c->codes_alt};
  for (int32_t t = first; t < last; ++t) {
    uint64_t* cnt = counts + 2 * (int64_t)(t - first);
    // the realizer counts the in-edges it writes per destination straight into
    // the graph load's row lengths (its edges are valid by construction)
    int rc = refnet_realize_impl(r, graph_seed, t, dead, src, dst, kind, capacity, nullptr, cnt, stream, c->row_len,
                                 true);
    if (!rc) rc = graph_load_impl(c, src, dst, kind, capacity, (const unsigned long long*)cnt, stream, true);
    const int k = (t - first) & 1;
    if (!rc) rc = step_impl(c, st, t, seed, nullptr, records + (int64_t)(t - first) * EPI_REC_LEN, vax_open, nullptr,
                            stream, true, (chain && t > first) ? cbuf[k] : nullptr,
                            chain ? cbuf[k ^ 1] : nullptr);
    if (rc) return rc;
  }
  return 0;
}

#ifdef EPI_IV_TRACE
// k_iv_run's phase timeline of the last launch (a -DEPI_IV_TRACE build only)
int epi_debug_iv_trace(unsigned long long* out, long long n) {
  const size_t bytes = sizeof(epi::g_iv_trace);
  if ((size_t)n * sizeof(unsigned long long) < bytes) return -1;
  return cudaMemcpyFromSymbol(out, epi::g_iv_trace, bytes) == cudaSuccess ? 0 : -3;
}
#endif
}  // extern "C"
