// Reference-native networks on the device:
// households from an arbitrary household_id, one Watts-Strogatz small-world
// graph per occupation, and configuration-model stub pairing — the three
// families of GraphRealizer.realize (graphs.py:54-75, 86-129, 138-168,
// 200-240), re-defined as keyed parallel algorithms:
//
//  * households: complete graph on the alive members (exact, no randomness);
//  * occupation j: ring lattice over its alive members in id order, k =
//    min(round_to_even(mean_j), 2*floor((m-1)/2)); lattice edge e = (p, p+i),
//    index e = (i-1)*m + p, is rewired iff u(e) < beta, to the position
//    p + k/2 + 1 + floor(u_1(e) * (m-k-1)) (uniform over p's non-neighbours);
//    like the reference (graphs.py:116-128: "rewiring replaces edges
//    one-for-one, so the undirected edge count is always n*k/2"), a rewired
//    pair that collides with another is drawn again, never dropped: the
//    lowest edge index keeps a contested pair, every other contender draws
//    again from u_{1+r}(e) in round r (ws_resolve_block, run by the last block of
//    launch 4), and a pair placed
//    in an earlier round is never taken over.  An edge still unplaced after
//    WS_ROUNDS draws keeps its lattice pair (the reference's "no free target:
//    keep v"; free, since rewired targets are never lattice neighbours);
//  * stub pairing: agent a gets floor(d_a) + [u(a) < frac(d_a)] stubs; stub q
//    sits at position pi^{-1}(q) of a keyed Feistel permutation of [0, S);
//    positions (2i, 2i+1) pair up; self pairs are dropped.
// Duplicate undirected stub pairs are resolved deterministically: a pair
// survives only for its lowest pair index (atomicMin into an open-addressing
// hash table), matching the reference's "keep first" rule
// (graphs.py:161-167).
#pragma once

#include "epi_confignet.cuh"

namespace epi {

enum RefPurpose : int { P_REF_WS = 81, P_REF_STUB = 82, P_REF_PERM = 83 };

struct RefNet {
  int64_t n_agents;
  const int32_t* hh_members;    // agents grouped by household
  const int32_t* hh_start;      // per agent: first slot of its household
  const int32_t* hh_size;       // per agent
  int32_t n_occ;                // occupations 1..n_occ
  const int32_t* occ_members;   // agents grouped by occupation, ascending ids
  const int32_t* occ_start;     // [n_occ + 1]
  const int32_t* occ_k;         // [n_occ] round_to_even(mean) (clipped per step)
  double beta;
  const double* random_degree;  // [N]
};

struct RefScratch {
  int32_t* live_members;        // per occupation: its alive members, compacted
  int32_t* occ_live;            // [n_occ]: alive count
  int64_t* stub_count;          // [N + 1] (last = 0)
  int64_t* stub_off;            // [N + 1] exclusive scan (device scan writes it)
  unsigned long long* table;    // hash: (key, lowest index) per slot; all-ones = empty
  int64_t table_slots;          // power of two
  int32_t* out_src;
  int32_t* out_dst;
  int8_t* out_kind;
  unsigned long long* counter;  // [0] = edges written, [1] = flags
  int64_t capacity;
  int32_t* stub_owner;          // [max_stubs]: agent of every stub (stub_off order)
  int64_t max_stubs;            // sum of ceil(random_degree): bound on the stubs of a step
  int2* pair_uv;                // [max_stubs / 2]: owners of stub pair i (pass 0 -> pass 1)
  int32_t* row_len;             // nullable: in-edges per destination of the edges written
                                // (the graph load's row lengths; the households kernel
                                // initialises every row)
  unsigned long long* ws_losers;  // rewired lattice edges that lost their first pair (edge
                                  // index; ~0 once placed), appended by launch 4
  unsigned* n_losers;             // zeroed by launch 1
  int64_t loser_cap;              // the lattice edges of all occupations
  unsigned* links_done;           // blocks of launch 4 finished (the last one resolves; reset by it)
};

__device__ __forceinline__ double ref_u(uint64_t prefix, uint64_t idx, uint64_t k) {
  return unit(fold(fold(prefix, idx), k));
}

// Block-aggregated reservation of `n` output slots (n may differ per
// thread, 0 for threads with nothing to write): one atomic per block on the
// single output counter.  Must be called by every thread
// of the block (block-uniform loop trip counts); blockDim <= 1024.
__device__ __forceinline__ int64_t reserve_block(unsigned long long* counter, int n) {
  __shared__ int warp_tot[32];
  __shared__ unsigned long long block_base;
  int incl = n;
  const int lane = lane_id(), warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int t = lane < nw ? warp_tot[lane] : 0;
    int x = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xFFFFFFFFu, x, o);
      if (lane >= o) x += v;
    }
    if (lane < nw) warp_tot[lane] = x - t;                      // exclusive warp offsets
    const int total = __shfl_sync(0xFFFFFFFFu, x, 31);
    if (lane == 0) block_base = total ? atomicAdd(counter, (unsigned long long)total) : 0ull;
  }
  __syncthreads();
  const int64_t at = (int64_t)block_base + warp_tot[warp] + incl - n;
  __syncthreads();                                              // smem reusable by the next call
  return at;
}

__device__ __forceinline__ void emit2(const RefScratch& S, int64_t at, int32_t u, int32_t v, int8_t kind) {
  if (at + 2 <= S.capacity) {
    S.out_src[at] = u; S.out_dst[at] = v; S.out_kind[at] = kind;
    S.out_src[at + 1] = v; S.out_dst[at + 1] = u; S.out_kind[at + 1] = kind;
    if (S.row_len) {
      atomicAdd(&S.row_len[u], 1);
      atomicAdd(&S.row_len[v], 1);
    }
  } else {
    atomicOr(&S.counter[1], 1ull);   // overflow flag
  }
}

// Who is dead: a u8 mask (code 1) or the engine's stage column read in place
// (code S_DEAD) — both one byte per agent.
struct DeadView {
  const int8_t* __restrict__ p;
  int8_t code;
  __device__ __forceinline__ bool operator[](int64_t i) const { return p[i] == code; }
};

// Launch 1 (per agent): households — each alive agent b emits c -> b for its
// alive co-members — and the agent's random-network stub count; the dedupe
// table is cleared on the side (first used by launch 3).
__global__ void k_ref_agents(RefNet net, DeadView dead, RefScratch S, uint64_t stub_prefix) {
  pdl_wait();     // launched programmatically after the previous step kernel
  pdl_trigger();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  ulonglong2* tab = reinterpret_cast<ulonglong2*>(S.table);
  for (int64_t i = tid; i < S.table_slots; i += stride) tab[i] = make_ulonglong2(~0ull, ~0ull);
  if (tid == 0) {
    S.stub_count[net.n_agents] = 0;
    *S.n_losers = 0u;
  }
  for (int64_t b0 = (int64_t)blockIdx.x * blockDim.x; b0 < net.n_agents; b0 += stride) {
    const int64_t b = b0 + threadIdx.x;
    const bool in = b < net.n_agents;
    const bool alive = in && !dead[b];
    const int st = alive ? net.hh_start[b] : 0, sz = alive ? net.hh_size[b] : 0;
    int cnt = 0;
    for (int i = 0; i < sz; ++i) {
      const int32_t c = net.hh_members[st + i];
      cnt += (c != b && !dead[c]) ? 1 : 0;
    }
    const int64_t at = reserve_block(S.counter, cnt);
    int o = 0;
    for (int i = 0; i < sz; ++i) {
      const int32_t c = net.hh_members[st + i];
      if (c != b && !dead[c]) {
        if (at + o < S.capacity) {
          S.out_src[at + o] = c; S.out_dst[at + o] = (int32_t)b; S.out_kind[at + o] = 0;
        } else {
          atomicOr(&S.counter[1], 1ull);
        }
        ++o;
      }
    }
    if (in) {
      if (S.row_len) {   // edges written into row b (all of them unless the output overflowed)
        const int64_t room = S.capacity - at;
        S.row_len[b] = (int32_t)(room >= cnt ? cnt : (room > 0 ? room : 0));
      }
      int c = 0;
      if (alive) {
        const double d = net.random_degree[b];
        const double fl = floor(d);
        c = (int)fl + (ref_u(stub_prefix, (uint64_t)b, 0) < d - fl ? 1 : 0);
      }
      S.stub_count[b] = c;
    }
  }
}

// Launch 2: blocks [0, n_occ) compact the alive members of occupation j (ids
// ascending); the remaining blocks write the owner of every stub (agent a owns
// stubs [stub_off[a], stub_off[a+1]); stub_off is launch 1's scan).
constexpr int kOccLiveThreads = 1024;
__global__ void __launch_bounds__(kOccLiveThreads) k_ref_occ_stubs(RefNet net, DeadView dead, RefScratch S) {
  pdl_wait();     // launched programmatically after the previous step kernel
  pdl_trigger();
  if ((int)blockIdx.x >= net.n_occ) {
    if (S.stub_off[net.n_agents] > S.max_stubs) return;   // launch 3 flags it
    const int64_t nb = gridDim.x - net.n_occ;
    for (int64_t a = (blockIdx.x - net.n_occ) * (int64_t)blockDim.x + threadIdx.x; a < net.n_agents;
         a += nb * blockDim.x) {
      const int64_t b = S.stub_off[a], e = S.stub_off[a + 1];
      for (int64_t q = b; q < e; ++q) S.stub_owner[q] = (int32_t)a;
    }
    return;
  }
  typedef cub::BlockScan<int, kOccLiveThreads> Scan;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int carry;
  const int j = blockIdx.x;
  const int lo = net.occ_start[j], hi = net.occ_start[j + 1];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int b0 = lo; b0 < hi; b0 += kOccLiveThreads) {
    const int i = b0 + threadIdx.x;
    const int32_t a = i < hi ? net.occ_members[i] : 0;
    const int alive = (i < hi && !dead[a]) ? 1 : 0;
    int ex, total;
    Scan(tmp).ExclusiveSum(alive, ex, total);
    if (alive) S.live_members[lo + carry + ex] = a;
    __syncthreads();
    if (threadIdx.x == 0) carry += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) S.occ_live[j] = carry;
}

__device__ __forceinline__ uint64_t hash_slot(uint64_t key, int64_t slots) {
  return mix64(key ^ 0x5851F42D4C957F2Dull) & (uint64_t)(slots - 1);
}
// undirected pair + network kind (pairs only collide within one family)
__device__ __forceinline__ uint64_t pair_key(uint32_t u, uint32_t v, int kind) {
  const uint32_t a = u < v ? u : v, b = u < v ? v : u;
  return ((uint64_t)kind << 62) | ((uint64_t)a << 31) | b;
}
__device__ __forceinline__ bool table_is_winner(const RefScratch& S, uint64_t key, uint64_t idx) {
  uint64_t h = hash_slot(key, S.table_slots);
  for (int64_t probe = 0; probe < S.table_slots; ++probe) {
    const unsigned long long kk = S.table[2 * h];
    if (kk == key) return S.table[2 * h + 1] == idx;
    if (kk == ~0ull) return false;
    h = (h + 1) & (uint64_t)(S.table_slots - 1);
  }
  return false;
}
// Insert key; keep the minimum index for it.  Returns the slot.
__device__ __forceinline__ int64_t table_insert(const RefScratch& S, uint64_t key, uint64_t idx) {
  uint64_t h = hash_slot(key, S.table_slots);
  for (int64_t probe = 0; probe < S.table_slots; ++probe) {
    unsigned long long* k = S.table + 2 * h;
    const unsigned long long prev = atomicCAS(k, ~0ull, key);       // ~0 = empty
    if (prev == ~0ull || prev == key) {
      atomicMin(k + 1, (unsigned long long)idx);
      return (int64_t)h;
    }
    h = (h + 1) & (uint64_t)(S.table_slots - 1);
  }
  atomicOr(&S.counter[1], 2ull);     // table full
  return -1;
}

// Watts-Strogatz lattice edges of occupation j, chunk `bx` of `nbx` (threads
// over edge indices).  Pass 0 inserts rewired pairs, pass 1 emits.
template <int PASS>
__device__ __forceinline__ void ws_block(const RefNet& net, const RefScratch& S, uint64_t ws_prefix, int j, int bx,
                                         int nbx) {
  const int lo = net.occ_start[j];
  const int m = S.occ_live[j];
  const int kmax = 2 * ((m - 1) / 2);
  const int k = net.occ_k[j] < kmax ? net.occ_k[j] : kmax;
  if (m < 3 || k < 2) return;
  const int half = k / 2;
  const int64_t n_edges = (int64_t)half * m;
  const int span = m - k - 1;                   // non-neighbours of a node
  const int64_t stride = (int64_t)nbx * blockDim.x;
  for (int64_t e0 = (int64_t)bx * blockDim.x; e0 < n_edges; e0 += stride) {
    const int64_t e = e0 + threadIdx.x;
    bool emit = false;
    int32_t u = 0, v = 0;
    if (e < n_edges) {
      const int i = (int)(e / m) + 1, p = (int)(e % m);
      const uint64_t idx = ((uint64_t)(j + 1) << 40) | (uint64_t)e;
      const bool rewired = span > 0 && ref_u(ws_prefix, idx, 0) < net.beta;
      int q = (p + i) % m;
      if (rewired) q = (int)((p + half + 1 + (int)(ref_u(ws_prefix, idx, 1) * span)) % m);
      u = S.live_members[lo + p];
      v = S.live_members[lo + q];
      if (!rewired) {
        emit = PASS == 1;
      } else {
        const uint64_t key = pair_key((uint32_t)u, (uint32_t)v, 1);
        if (PASS == 0) {
          table_insert(S, key, idx);
        } else {
          emit = table_is_winner(S, key, idx);
          if (!emit) {                   // drawn again by ws_resolve_block
            const unsigned at = atomicAdd(S.n_losers, 1u);
            if (at < S.loser_cap) S.ws_losers[at] = idx;
            else atomicOr(&S.counter[1], 8ull);
          }
        }
      }
    }
    if (PASS == 1) {
      const int64_t at = reserve_block(S.counter, emit ? 2 : 0);
      if (emit) emit2(S, at, u, v, 1);
    }
  }
}

// Launch 4's last block: the rewired lattice edges whose first pair was taken draw
// again, in rounds r = 1, 2, ... (one block; a handful of edges per step).
// Round r: every unplaced edge proposes the pair of draw u_{1+r} and inserts
// it with value r << 56 | edge index, so a pair placed in an earlier round
// (smaller value) is never taken over and the lowest index wins among the
// round's contenders; the winners are emitted.  Phases of a round are
// separated by bar.sync; table words written in this launch are read with
// ld.cg (the atomics are performed in L2).
constexpr int WS_ROUNDS = 64;
__device__ __forceinline__ void ws_resolve_block(const RefNet& net, const RefScratch& S, uint64_t ws_prefix) {
  const unsigned nl0 = __ldcg(S.n_losers);
  const unsigned nl = nl0 < S.loser_cap ? nl0 : (unsigned)S.loser_cap;
  if (nl == 0) return;
  // the proposal of loser li in round r (u, v, key, value)
  auto propose = [&](unsigned li, int r, int32_t& u, int32_t& v, uint64_t& key, uint64_t& val) {
    const uint64_t idx = __ldcg(S.ws_losers + li);
    const int j = (int)(idx >> 40) - 1;
    const int64_t e = (int64_t)(idx & ((1ull << 40) - 1));
    const int lo = net.occ_start[j];
    const int m = S.occ_live[j];
    const int kmax = 2 * ((m - 1) / 2);
    const int k = net.occ_k[j] < kmax ? net.occ_k[j] : kmax;
    const int half = k / 2, span = m - k - 1;
    const int i = (int)(e / m) + 1, p = (int)(e % m);
    int q = (p + i) % m;                                        // r < 0: the lattice pair
    if (r >= 0) q = (int)((p + half + 1 + (int)(ref_u(ws_prefix, idx, 1 + (uint64_t)r) * span)) % m);
    u = S.live_members[lo + p];
    v = S.live_members[lo + q];
    key = pair_key((uint32_t)u, (uint32_t)v, 1);
    val = ((uint64_t)(r < 0 ? 0 : r) << 56) | idx;
  };
  for (int r = 1; r <= WS_ROUNDS; ++r) {
    for (unsigned li = threadIdx.x; li < nl; li += blockDim.x) {
      if (__ldcg(S.ws_losers + li) == ~0ull) continue;
      int32_t u, v; uint64_t key, val;
      propose(li, r, u, v, key, val);
      table_insert(S, key, val);
    }
    __syncthreads();
    int left = 0;
    for (unsigned b0 = 0; b0 < nl; b0 += blockDim.x) {          // block-uniform trips
      const unsigned li = b0 + threadIdx.x;
      bool won = false;
      int32_t u = 0, v = 0;
      if (li < nl && __ldcg(S.ws_losers + li) != ~0ull) {
        uint64_t key, val;
        propose(li, r, u, v, key, val);
        uint64_t h = hash_slot(key, S.table_slots);
        for (int64_t probe = 0; probe < S.table_slots; ++probe) {
          const unsigned long long kk = __ldcg(S.table + 2 * h);
          if (kk == key) { won = __ldcg(S.table + 2 * h + 1) == val; break; }
          if (kk == ~0ull) break;
          h = (h + 1) & (uint64_t)(S.table_slots - 1);
        }
        left += won ? 0 : 1;
      }
      const int64_t at = reserve_block(S.counter, won ? 2 : 0);
      if (won) {
        emit2(S, at, u, v, 1);
        S.ws_losers[li] = ~0ull;
      }
    }
    if (!__syncthreads_or(left)) return;
  }
  // no free pair in WS_ROUNDS draws: the lattice pair (never proposed by a
  // rewired edge, so never taken)
  for (unsigned b0 = 0; b0 < nl; b0 += blockDim.x) {
    const unsigned li = b0 + threadIdx.x;
    const bool keep = li < nl && __ldcg(S.ws_losers + li) != ~0ull;
    int32_t u = 0, v = 0;
    if (keep) {
      uint64_t key, val;
      propose(li, -1, u, v, key, val);
    }
    const int64_t at = reserve_block(S.counter, keep ? 2 : 0);
    if (keep) emit2(S, at, u, v, 1);
  }
}

// Stub pairs: positions (2i, 2i+1) of the keyed permutation of [0, S);
// pass 0 resolves the owners (kept for pass 1) and inserts, pass 1 emits.
template <int PASS>
__device__ __forceinline__ void pairs_block(const RefNet& net, const RefScratch& S, const PermKeys& K, int64_t bx,
                                            int64_t nbx) {
  const int64_t n_stubs = S.stub_off[net.n_agents];
  if (n_stubs >= (1ll << 31) || n_stubs > S.max_stubs) {
    if (PASS == 0 && bx == 0 && threadIdx.x == 0) atomicOr(&S.counter[1], 4ull);
    return;
  }
  if (n_stubs < 2) return;
  const Radix d = make_radix((uint32_t)n_stubs);
  const int64_t n_pairs = n_stubs / 2;
  const int64_t stride = nbx * blockDim.x;
  for (int64_t i0 = bx * blockDim.x; i0 < n_pairs; i0 += stride) {
    const int64_t i = i0 + threadIdx.x;
    bool emit = false;
    int32_t u = 0, v = 0;
    if (i < n_pairs) {
      if (PASS == 0) {
        u = S.stub_owner[walk_fwd((uint32_t)(2 * i), K, d)];
        v = S.stub_owner[walk_fwd((uint32_t)(2 * i + 1), K, d)];
        S.pair_uv[i] = make_int2(u, v);
      } else {
        const int2 uv = S.pair_uv[i];
        u = uv.x;
        v = uv.y;
      }
      if (u != v) {
        const uint64_t key = pair_key((uint32_t)u, (uint32_t)v, 2);
        if (PASS == 0) table_insert(S, key, (uint64_t)i);
        else emit = table_is_winner(S, key, (uint64_t)i);
      }
    }
    if (PASS == 1) {
      const int64_t at = reserve_block(S.counter, emit ? 2 : 0);
      if (emit) emit2(S, at, u, v, 2);
    }
  }
}

// Launches 3 (PASS 0: inserts) and 4 (PASS 1: winners emitted): blocks
// [0, ws_blocks * n_occ) walk the occupations' lattices (ws_blocks chunks per
// occupation), the remaining blocks the stub pairs.
template <int PASS>
__global__ void k_ref_links(RefNet net, RefScratch S, uint64_t ws_prefix, PermKeys K, int ws_blocks) {
  pdl_wait();     // launched programmatically after the previous step kernel
  pdl_trigger();
  const int nws = ws_blocks * net.n_occ;
  if ((int)blockIdx.x < nws)
    ws_block<PASS>(net, S, ws_prefix, blockIdx.x / ws_blocks, blockIdx.x % ws_blocks, ws_blocks);
  else
    pairs_block<PASS>(net, S, K, blockIdx.x - nws, gridDim.x - nws);
  if (PASS == 1 && net.n_occ > 0) {
    // the last block to finish places the rewired edges whose pair was
    // taken (no launch of its own: threadFence-reduction pattern)
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(S.links_done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (last) {
      __threadfence();
      ws_resolve_block(net, S, ws_prefix);
      if (threadIdx.x == 0) *S.links_done = 0u;
    }
  }
}

}  // namespace epi
