// Config-network generator on the device (BASELINE.json configs 0-4).
//
// Specification: paper_2110_04421_b200/confignet.py (module docstring); CPU
// restatement: oracle/confignet_np.py.  Replaces, for these networks, the
// reference's per-step GraphRealizer.realize (graphs.py:200-240), whose
// Watts-Strogatz rewiring loop and stub-pairing sort are 81 % of reference
// wall time.
//
// Every in-edge of a destination b is enumerated by b's owner alone:
//   household : contiguous id range [b - hh_off, b - hh_off + hh_size);
//   workplace : sigma^{-1}(local) then sigma(p +- r_j) on a <= 8-bit domain;
//   random    : pi_j(b) (own draw, if j < n_b) and pi_j^{-1}(b) (the agent
//               whose draw lands on b, if j < its n) for every slot j.
// No sort, no atomics, no cross-GPU exchange: a rank owning rows [lo, hi)
// needs only the all-gathered 16-bit codes (dead bit + slot count).
#pragma once

#include "epi_common.cuh"

namespace epi {

// Keyed bijection of [0, n): a 3-round Feistel network on the mixed-radix
// domain [0, a*b), b = ceil(sqrt(n)), a = ceil(n / b), so a*b - n < b and the
// cycle walk back into [0, n) almost never iterates (probability < 1/sqrt(n)
// per evaluation) — no warp divergence from rejection loops.
//   x = L*b + R;  L += F(R,k0) mod a;  R += F(L,k1) mod b;  L += F(R,k2) mod a
// F(v, k) = mulhi(mix(v ^ k.x, k.y), radix): uniform in [0, radix).
struct PermKeys {
  uint32_t k1[3], k2[3];
};
struct Radix {
  uint32_t n, a, b, magic;   // magic = floor((2^32 - 1) / b)
};

__host__ __device__ __forceinline__ uint32_t isqrt_ceil(uint32_t n) {
  // smallest b with b*b >= n (n >= 1)
  uint32_t b = (uint32_t)sqrt((double)n);
  while ((uint64_t)b * b < n) ++b;
  while (b > 1 && (uint64_t)(b - 1) * (b - 1) >= n) --b;
  return b;
}
__host__ __device__ __forceinline__ Radix make_radix(uint32_t n) {
  Radix r;
  r.n = n;
  r.b = isqrt_ceil(n < 1 ? 1 : n);
  r.a = (n + r.b - 1) / r.b;
  r.magic = 0xFFFFFFFFu / r.b;
  return r;
}
// Round function: keyed multiply, then one xorshift-multiply-xorshift stage.
// The plain multiplicative hash is nearly linear in v, which made pi(x+1) -
// pi(x) take only a few thousand distinct values (adjacent agents got
// partners that were adjacent too); the extra stage gives random-like spacing.
__device__ __forceinline__ uint32_t feistel_f(uint32_t v, uint32_t k1, uint32_t k2, uint32_t radix) {
  uint32_t h = (v ^ k1) * k2;
  h = (h ^ (h >> 16)) * 0x7FEB352Du;
  return __umulhi(h ^ (h >> 15), radix);
}
__device__ __forceinline__ void split(uint32_t x, const Radix& d, uint32_t& L, uint32_t& R) {
  L = __umulhi(x, d.magic);          // floor(x/b) or one less (x < 2^31)
  R = x - L * d.b;
  if (R >= d.b) { R -= d.b; ++L; }
}
__device__ __forceinline__ uint32_t add_mod(uint32_t x, uint32_t y, uint32_t m) {
  const uint32_t z = x + y;
  return z >= m ? z - m : z;
}
__device__ __forceinline__ uint32_t sub_mod(uint32_t x, uint32_t y, uint32_t m) {
  return x >= y ? x - y : x + m - y;
}
__device__ __forceinline__ uint32_t perm_fwd(uint32_t x, const PermKeys& K, const Radix& d) {
  uint32_t L, R;
  split(x, d, L, R);
  L = add_mod(L, feistel_f(R, K.k1[0], K.k2[0], d.a), d.a);
  R = add_mod(R, feistel_f(L, K.k1[1], K.k2[1], d.b), d.b);
  L = add_mod(L, feistel_f(R, K.k1[2], K.k2[2], d.a), d.a);
  return L * d.b + R;
}
__device__ __forceinline__ uint32_t perm_inv(uint32_t y, const PermKeys& K, const Radix& d) {
  uint32_t L, R;
  split(y, d, L, R);
  L = sub_mod(L, feistel_f(R, K.k1[2], K.k2[2], d.a), d.a);
  R = sub_mod(R, feistel_f(L, K.k1[1], K.k2[1], d.b), d.b);
  L = sub_mod(L, feistel_f(R, K.k1[0], K.k2[0], d.a), d.a);
  return L * d.b + R;
}
// Cycle walking restricts the bijection of [0, a*b) to [0, n).
__device__ __forceinline__ uint32_t walk_fwd(uint32_t x, const PermKeys& K, const Radix& d) {
  do { x = perm_fwd(x, K, d); } while (x >= d.n);
  return x;
}
__device__ __forceinline__ uint32_t walk_inv(uint32_t y, const PermKeys& K, const Radix& d) {
  do { y = perm_inv(y, K, d); } while (y >= d.n);
  return y;
}

// Hash prefixes of one generated step (purposes 72-75 at (graph_seed, step)).
struct NetKeys {
  uint64_t rcount, rperm, wperm, wshift;
};
__host__ __device__ inline NetKeys make_net_keys(uint64_t g, int step) {
  return NetKeys{key_prefix(g, step, P_NET_RCOUNT), key_prefix(g, step, P_NET_RPERM),
                 key_prefix(g, step, P_NET_WPERM), key_prefix(g, step, P_NET_WSHIFT)};
}

__host__ __device__ __forceinline__ PermKeys random_slot_keys(uint64_t rperm_prefix, int slot) {
  PermKeys K;
  const uint64_t hs = fold(rperm_prefix, (uint64_t)slot);
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    const uint64_t h = fold(hs, (uint64_t)r);
    K.k1[r] = (uint32_t)h;
    K.k2[r] = (uint32_t)(h >> 32) | 1u;
  }
  return K;
}

__device__ __forceinline__ PermKeys work_keys(uint64_t wperm_prefix, int w) {
  PermKeys K;
  const uint64_t hw = fold(wperm_prefix, (uint64_t)w);
  const uint64_t ha = fold(hw, 0), hb = fold(hw, 1);
  K.k1[0] = (uint32_t)(ha & 0xFFFF);
  K.k2[0] = (uint32_t)((ha >> 16) & 0xFFFF) | 1u;
  K.k1[1] = (uint32_t)((ha >> 32) & 0xFFFF);
  K.k2[1] = (uint32_t)((ha >> 48) & 0xFFFF) | 1u;
  K.k1[2] = (uint32_t)(hb & 0xFFFF);
  K.k2[2] = (uint32_t)((hb >> 16) & 0xFFFF) | 1u;
  return K;
}

// Per-day key/domain tables, computed once on the host per simulated day and
// passed by value (kernel parameter); blocks copy them to shared memory.
struct NetTables {
  PermKeys rk[EPI_MAX_SLOTS];   // random-slot Feistel keys of the day
  Radix wrad[256];              // workplace domains, m <= 255 (static)
  Radix dn;                     // agent domain [0, N)
};
inline void fill_net_tables(NetTables& T, const epi_net& net, uint64_t rperm) {
  for (int j = 0; j < EPI_MAX_SLOTS; ++j) T.rk[j] = random_slot_keys(rperm, j);
  for (int m = 0; m < 256; ++m) T.wrad[m] = make_radix(m < 1 ? 1u : (uint32_t)m);
  T.dn = make_radix(net.n_agents < 1 ? 1u : (uint32_t)net.n_agents);
}
__device__ __forceinline__ void load_net_tables(NetTables& S, const NetTables* __restrict__ P) {
  const uint32_t* src = (const uint32_t*)P;
  uint32_t* dst = (uint32_t*)&S;
  for (int i = threadIdx.x; i < (int)(sizeof(NetTables) / 4); i += blockDim.x) dst[i] = src[i];
}

// Per-day workplace tables (a cache of sigma_{t,W} and the shifts): built by
// k_day_tables with one bijection evaluation per member slot, then read by
// every worker instead of 1 + 2*draws evaluations each.
//   member_at_pos[base_W + q] = wp_members[base_W + sigma(q)]
//   pos_of[base_W + l]        = sigma^{-1}(l)
//   shift[W * draws + j]      = r_{t,W,j}
struct WorkTables {
  int32_t* member_at_pos;
  uint8_t* pos_of;
  uint8_t* shift;
  // Fused mode only ("push" tables: the consumer reads contiguous rows
  // instead of evaluating bijections / gathering random 2-byte codes):
  //   wcode[base_W + q] = code of the worker at position q
  //   rout[a*16 + j] = pi_{t,j}(a) for j < n_{t,a}   (own out-partners)
  //   rin [b*16 + j] = code(c) | PRESENT where pi_{t,j}(c) = b, j < n_{t,c}, c != b
  // (whole-population runs only; the scatter into rin is conflict-free because
  // pi is a bijection, and rin rows are cleared by their consumer).
  uint16_t* wcode;
  uint32_t* rout;
  uint16_t* rin;
};
constexpr int RT_SLOTS = 16;
constexpr uint16_t CODE_PRESENT = 0x4000;

__device__ __forceinline__ uint32_t work_shift(uint64_t wshift_prefix, int w, int j, int m) {
  const uint64_t hq = fold(fold(wshift_prefix, (uint64_t)w), (uint64_t)(j >> 2));
  const uint32_t v = (uint32_t)((hq >> (16 * (j & 3))) & 0xFFFF);
  return 1u + ((v * (uint32_t)(m - 1)) >> 16);
}

// Random-slot count n_{t,a} ~ Poisson(mean) truncated at `slots`.
// (cdf: the network's Poisson CDF, from wherever the caller keeps it -- a
// kernel parameter's array indexed per lane is a serialised constant load)
__device__ __forceinline__ int random_count_cdf(const double* cdf, int slots, uint64_t rcount_prefix, int64_t a) {
  const double u = keyed_u(rcount_prefix, (uint64_t)a, 0);
  // #{k < slots : u >= cdf[k]} for the non-decreasing cdf: a branch-free
  // binary search (6 compares instead of up to 32)
  int c = 0;
#pragma unroll
  for (int step = EPI_MAX_SLOTS / 2; step >= 1; step >>= 1) {
    const int k = c + step - 1;
    c += (k < slots && u >= cdf[k]) ? step : 0;
  }
  c += (c < slots && u >= cdf[c < EPI_MAX_SLOTS ? c : EPI_MAX_SLOTS - 1]) ? 1 : 0;
  return c;
}
__device__ __forceinline__ int random_count(const epi_net& net, uint64_t rcount_prefix, int64_t a) {
  return random_count_cdf(net.poisson_cdf, net.random_slots, rcount_prefix, a);
}

// Enumerate the in-edges of destination b (alive); visit(src, kind, code_src).
// The work of one row is split over `nl` cooperating lanes; lane `li` takes
// household members i, colleague draws j and random slots j with
// index % nl == li.  With nl == 1 the order is: household members ascending,
// workplace slots (out, in), random slots (out, in).  `rk` holds the
// random-slot keys of this step (shared memory).  `code_of(c)` gives agent
// c's 16-bit code of the step (dead bit + random-slot count are all the
// enumeration reads): the day's code vector, or a code rebuilt for a past
// day (k_den_regen).
template <class CodeOf, class Visit>
__device__ __forceinline__ void for_each_in_edge_f(const epi_net& net, const NetKeys& nk,
                                                   const PermKeys* __restrict__ rk,
                                                   const Radix* __restrict__ wrad, CodeOf&& codes,
                                                   int64_t b, uint16_t code_b, int li, int nl, Visit&& visit) {
  // household: contiguous range
  {
    const int off = net.hh_off[b];
    const int sz = net.hh_size[b];
    const int64_t start = b - off;
    for (int i = li; i < sz; i += nl) {
      const int64_t c = start + i;
      if (c == b) continue;
      const uint16_t cc = codes(c);
      if (!code_dead(cc)) visit(c, 0, cc);
    }
  }
  // workplace
  const int w = li < net.colleague_draws ? net.wp_id[b] : -1;
  if (w >= 0) {
    const int m = net.wp_size[w];
    if (m >= 2) {
      const Radix d = wrad[m];
      const PermKeys K = work_keys(nk.wperm, w);
      const int base = net.wp_base[w];
      const uint32_t p = walk_inv(net.wp_local[b], K, d);
      const uint64_t hw = fold(nk.wshift, (uint64_t)w);
      uint64_t hq = 0;
      int q_have = -1;
      for (int j = li; j < net.colleague_draws; j += nl) {
        if ((j >> 2) != q_have) { q_have = j >> 2; hq = fold(hw, (uint64_t)q_have); }
        const uint32_t v = (uint32_t)((hq >> (16 * (j & 3))) & 0xFFFF);
        const uint32_t r = 1u + ((v * (uint32_t)(m - 1)) >> 16);
        const int32_t co = net.wp_members[base + walk_fwd(add_mod(p, r, (uint32_t)m), K, d)];
        const int32_t ci = net.wp_members[base + walk_fwd(sub_mod(p, r, (uint32_t)m), K, d)];
        const uint16_t cco = codes(co);
        const uint16_t cci = codes(ci);
        if (!code_dead(cco)) visit((int64_t)co, 1, cco);
        if (!code_dead(cci)) visit((int64_t)ci, 1, cci);
      }
    }
  }
  // random slots
  const uint32_t n = (uint32_t)net.n_agents;
  if (n >= 2) {
    const Radix d = make_radix(n);
    const int nb = code_count(code_b);
    for (int j = li; j < net.random_slots; j += nl) {
      const PermKeys& K = rk[j];
      const uint32_t ci = walk_inv((uint32_t)b, K, d);
      if (j < nb) {
        const uint32_t c = walk_fwd((uint32_t)b, K, d);
        if (c != (uint32_t)b) {
          const uint16_t cc = codes(c);
          if (!code_dead(cc)) visit((int64_t)c, 2, cc);
        }
      }
      if (ci != (uint32_t)b) {
        const uint16_t cc = codes(ci);
        if (j < code_count(cc)) visit((int64_t)ci, 2, cc);
      }
    }
  }
}

template <class Visit>
__device__ __forceinline__ void for_each_in_edge(const epi_net& net, const NetKeys& nk,
                                                 const PermKeys* __restrict__ rk,
                                                 const Radix* __restrict__ wrad,
                                                 const uint16_t* __restrict__ codes, int64_t b,
                                                 uint16_t code_b, int li, int nl, Visit&& visit) {
  for_each_in_edge_f(net, nk, rk, wrad, [&](int64_t c) { return codes[c]; }, b, code_b, li, nl, visit);
}

// Batched single-lane enumeration: every partner id of a section is computed
// first (pure ALU: keyed bijections), then all their codes are loaded at once
// (up to JMAX independent gathers in flight per lane), then visited.  Visit
// order: household, workplace (out, in per draw), random out-partners, random
// in-partners (the edge multiset equals for_each_in_edge's).  Requires
// random_slots <= JMAX and colleague_draws <= DMAX.
template <int JMAX, int DMAX, class Visit>
__device__ __forceinline__ void for_each_in_edge_batched(const epi_net& net, const NetKeys& nk,
                                                         const PermKeys* __restrict__ rk,
                                                         const Radix* __restrict__ wrad,
                                                         const WorkTables* wt,
                                                         const uint16_t* __restrict__ codes,
                                                         int64_t b, uint16_t code_b, Visit&& visit) {
  // household: contiguous range, one cache line in practice
  {
    const int off = net.hh_off[b];
    const int sz = net.hh_size[b];
    const int64_t start = b - off;
    for (int i = 0; i < sz; ++i) {
      const int64_t c = start + i;
      if (c == b) continue;
      const uint16_t cc = codes[c];
      if (!code_dead(cc)) visit(c, 0, cc);
    }
  }
  // workplace
  const int w = net.wp_id[b];
  if (w >= 0) {
    const int m = net.wp_size[w];
    if (m >= 2) {
      const int base = net.wp_base[w];
      const int draws = net.colleague_draws;
      int32_t mo[DMAX], mi[DMAX];
      if (wt != nullptr) {
        const uint32_t p = wt->pos_of[base + net.wp_local[b]];
        const uint8_t* sh = wt->shift + (size_t)w * draws;
#pragma unroll
        for (int j = 0; j < DMAX; ++j) {
          if (j < draws) {
            const uint32_t r = sh[j];
            mo[j] = wt->member_at_pos[base + add_mod(p, r, (uint32_t)m)];
            mi[j] = wt->member_at_pos[base + sub_mod(p, r, (uint32_t)m)];
          }
        }
      } else {
        const Radix d = wrad[m];
        const PermKeys K = work_keys(nk.wperm, w);
        const uint32_t p = walk_inv(net.wp_local[b], K, d);
#pragma unroll
        for (int j = 0; j < DMAX; ++j) {
          if (j < draws) {
            const uint32_t r = work_shift(nk.wshift, w, j, m);
            mo[j] = base + (int32_t)walk_fwd(add_mod(p, r, (uint32_t)m), K, d);
            mi[j] = base + (int32_t)walk_fwd(sub_mod(p, r, (uint32_t)m), K, d);
          }
        }
#pragma unroll
        for (int j = 0; j < DMAX; ++j) {
          if (j < draws) {
            mo[j] = net.wp_members[mo[j]];
            mi[j] = net.wp_members[mi[j]];
          }
        }
      }
      uint16_t co[DMAX], ci[DMAX];
#pragma unroll
      for (int j = 0; j < DMAX; ++j) {
        if (j < draws) {
          co[j] = codes[mo[j]];
          ci[j] = codes[mi[j]];
        }
      }
#pragma unroll
      for (int j = 0; j < DMAX; ++j) {
        if (j < draws) {
          if (!code_dead(co[j])) visit((int64_t)mo[j], 1, co[j]);
          if (!code_dead(ci[j])) visit((int64_t)mi[j], 1, ci[j]);
        }
      }
    }
  }
  // random slots
  const uint32_t n = (uint32_t)net.n_agents;
  if (n >= 2) {
    const Radix d = make_radix(n);
    const int nb = code_count(code_b);
    const int slots = net.random_slots;
    const uint32_t self = (uint32_t)b;
    // in-partners: one inverse evaluation per slot, all lanes busy
    uint32_t pin[JMAX];
    // straight-line first application for every slot (16 independent chains
    // the scheduler can interleave), then the rare cycle-walk fix-ups
#pragma unroll
    for (int j = 0; j < JMAX; ++j) pin[j] = (j < slots) ? perm_inv(self, rk[j], d) : self;
#pragma unroll
    for (int j = 0; j < JMAX; ++j)
      if (pin[j] >= d.n) pin[j] = walk_inv(pin[j], rk[j], d);
    uint16_t cin[JMAX];
#pragma unroll
    for (int j = 0; j < JMAX; ++j) cin[j] = pin[j] != self ? codes[pin[j]] : (uint16_t)0;
    // out-partners: only the nb activated slots, in chunks of 4 (per-lane trip count)
    const int nbe = nb < slots ? nb : slots;
    for (int j0 = 0; j0 < nbe; j0 += 4) {
      uint32_t po[4];
      uint16_t co[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) po[q] = (j0 + q < nbe) ? perm_fwd(self, rk[j0 + q], d) : self;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (po[q] >= d.n) po[q] = walk_fwd(po[q], rk[j0 + q], d);
#pragma unroll
      for (int q = 0; q < 4; ++q) co[q] = po[q] != self ? codes[po[q]] : (uint16_t)CODE_DEAD;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (!code_dead(co[q])) visit((int64_t)po[q], 2, co[q]);
    }
#pragma unroll
    for (int j = 0; j < JMAX; ++j)
      if (j < code_count(cin[j])) visit((int64_t)pin[j], 2, cin[j]);
  }
}

// Code-only enumeration for the fused kernel: visit(kind, code_src) for every
// in-edge of alive b, reading the day's push tables (wt != null) where they
// exist, else evaluating the bijections (partitioned ranks).  Same edge
// multiset and the same visit order as for_each_in_edge_batched.
template <class Visit>
__device__ __forceinline__ void for_each_in_code(const epi_net& net, const NetKeys& nk,
                                                 const PermKeys* __restrict__ rk,
                                                 const Radix* __restrict__ wrad, const Radix& dn,
                                                 const WorkTables* wt,
                                                 const uint16_t* __restrict__ codes, int64_t b,
                                                 uint16_t code_b, Visit&& visit) {
  // household: contiguous ids -> contiguous codes
  {
    const int off = net.hh_off[b];
    const int sz = net.hh_size[b];
    const int64_t start = b - off;
    for (int i = 0; i < sz; ++i) {
      const int64_t c = start + i;
      if (c == b) continue;
      const uint16_t cc = codes[c];
      if (!code_dead(cc)) visit(0, cc);
    }
  }
  const int w = net.wp_id[b];
  if (w >= 0) {
    const int m = net.wp_size[w];
    if (m >= 2) {
      const int base = net.wp_base[w];
      const int draws = net.colleague_draws;
      if (wt != nullptr && wt->wcode != nullptr) {
        const uint32_t p = wt->pos_of[base + net.wp_local[b]];
        const uint8_t* sh = wt->shift + (size_t)w * draws;
        const uint16_t* wc = wt->wcode + base;
        for (int j = 0; j < draws; ++j) {
          const uint32_t r = sh[j];
          const uint16_t co = wc[add_mod(p, r, (uint32_t)m)];
          const uint16_t ci = wc[sub_mod(p, r, (uint32_t)m)];
          if (!code_dead(co)) visit(1, co);
          if (!code_dead(ci)) visit(1, ci);
        }
      } else {
        const Radix d = wrad[m];
        const PermKeys K = work_keys(nk.wperm, w);
        const uint32_t p = walk_inv(net.wp_local[b], K, d);
        for (int j = 0; j < draws; ++j) {
          const uint32_t r = work_shift(nk.wshift, w, j, m);
          const uint16_t co = codes[net.wp_members[base + walk_fwd(add_mod(p, r, (uint32_t)m), K, d)]];
          const uint16_t ci = codes[net.wp_members[base + walk_fwd(sub_mod(p, r, (uint32_t)m), K, d)]];
          if (!code_dead(co)) visit(1, co);
          if (!code_dead(ci)) visit(1, ci);
        }
      }
    }
  }
  if (net.n_agents < 2) return;
  if (wt != nullptr && wt->rin != nullptr) {
    const uint32_t self = (uint32_t)b;
    const int nb = code_count(code_b);
    const int nbe = nb < RT_SLOTS ? nb : RT_SLOTS;
    const uint4* ri = (const uint4*)(wt->rin + (size_t)b * RT_SLOTS);
    const uint4 in[2] = {ri[0], ri[1]};
    const uint4* ro = (const uint4*)(wt->rout + (size_t)b * RT_SLOTS);
    for (int j0 = 0; j0 < nbe; j0 += 4) {
      const uint4 o = ro[j0 >> 2];
      const uint32_t po[4] = {o.x, o.y, o.z, o.w};
      uint16_t co[4];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        co[q] = (j0 + q < nbe && po[q] != self) ? codes[po[q]] : (uint16_t)CODE_DEAD;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (!code_dead(co[q])) visit(2, co[q]);
    }
    const uint16_t* iv = (const uint16_t*)in;
#pragma unroll
    for (int j = 0; j < RT_SLOTS; ++j)
      if (iv[j] & CODE_PRESENT) visit(2, (uint16_t)(iv[j] & ~CODE_PRESENT));
    return;
  }
  // random section evaluated on the fly (no tables)
  const uint32_t self = (uint32_t)b;
  const int nb = code_count(code_b);
  const int slots = net.random_slots;
  const int nbe = nb < slots ? nb : slots;
  for (int j0 = 0; j0 < nbe; j0 += 4) {
    uint32_t po[4];
    uint16_t co[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) po[q] = (j0 + q < nbe) ? walk_fwd(self, rk[j0 + q], dn) : self;
#pragma unroll
    for (int q = 0; q < 4; ++q) co[q] = po[q] != self ? codes[po[q]] : (uint16_t)CODE_DEAD;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (!code_dead(co[q])) visit(2, co[q]);
  }
  for (int j0 = 0; j0 < slots; j0 += 8) {
    uint32_t pi[8];
    uint16_t ci[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) pi[q] = (j0 + q < slots) ? perm_inv(self, rk[j0 + q], dn) : self;
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (pi[q] >= dn.n) pi[q] = walk_inv(pi[q], rk[j0 + q], dn);
#pragma unroll
    for (int q = 0; q < 8; ++q) ci[q] = pi[q] != self ? codes[pi[q]] : (uint16_t)0;
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (j0 + q < code_count(ci[q])) visit(2, ci[q]);
  }
}

// One source of a per-kind sum, branch-free: acc += factor[c & 0xFF] for every
// slot.  A dead or absent source has code byte 0 and factor[0] = 0, and
// acc + 0.0f == acc (acc >= +0), so the sums are bitwise those of skipping
// it; `edges` counts the alive (resp. present) ones.
// (`1 - dead bit` lets the unrolled callers fold the constant ones and add
// two slots' dead bits per IADD3.)
__device__ __forceinline__ void add_src(float& acc, unsigned& edges, const float* __restrict__ factor, uint16_t c) {
  acc += factor[c & 0xFF];
  edges += 1u - ((unsigned)c >> 15);
}
// A group of K sources in visit order: the edge count branch-free, the factor
// adds only when some source of the group is infectious (code byte != 0).
// Skipped adds are all +0.0f on a sum >= +0, so the result is bitwise that
// of K add_src calls; most groups of most days have no infectious source.
template <int K>
__device__ __forceinline__ void add_src_group(float& acc, unsigned& edges, const float* __restrict__ factor,
                                              const uint16_t* c) {
  // the dead bits summed in place (bit 15 of each code; K <= 16 cannot carry
  // out of 32 bits): one LOP3 + half an IADD3 per code, where `1 - (c >> 15)`
  // compiles to a sign-extend, a compare and a predicated increment
  unsigned any = 0, dead = 0;
#pragma unroll
  for (int i = 0; i < K; ++i) {
    any |= c[i];
    dead += (unsigned)c[i] & 0x8000u;
  }
  edges += (unsigned)K - (dead >> 15);
  if (any & 0xFFu) {
#pragma unroll
    for (int i = 0; i < K; ++i) acc += factor[c[i] & 0xFF];
  }
}
// The household in-edge sources of an agent in visit order (members
// ascending, the agent itself skipped).  `hp` points at the first member's
// code of the day: the block's shared-memory copy when the whole household
// lies in the block, else the global code vector (a generic pointer either
// way); bit i of the static `hmask` is set for the members i < HH other than
// the agent.  Absent slots read as CODE_DEAD (no edge, factor 0).
template <int HH>
__device__ __forceinline__ void load_household(uint16_t (&hc)[HH], const uint16_t* hp, unsigned hmask) {
#pragma unroll
  for (int i = 0; i < HH; ++i) hc[i] = ((hmask >> i) & 1u) ? hp[i] : (uint16_t)CODE_DEAD;
}
__host__ __device__ __forceinline__ unsigned household_mask(int hh, int sz, int off) {
  return (sz >= hh ? (1u << hh) - 1u : (1u << sz) - 1u) & (off < hh ? ~(1u << off) : ~0u);
}
// The colleague in-edge sources of a worker at position p of its workplace
// window (m >= 2 members, codes at wc[base .. base + m)): per draw j the
// partners at p + r_j and p - r_j (mod m), visit order out, in; the day's
// shifts r_j (1 <= r_j <= m - 1) packed one byte each in `shp`.  Non-workers
// and draws >= `draws` read as CODE_DEAD.  32-bit table indices, the window
// wrap as a select between two precomputed bases; the full-draw case (every
// config network) has no per-draw test.
template <int DR>
__device__ __forceinline__ void load_colleagues(uint16_t (&wio)[2 * DR], bool works, const uint16_t* wc, uint32_t base,
                                                uint32_t p, uint32_t m, uint2 shp, int draws) {
#pragma unroll
  for (int j = 0; j < 2 * DR; ++j) wio[j] = (uint16_t)CODE_DEAD;
  const uint32_t bp = base + p, mp = m - p;          // out: p + r wraps iff r >= m - p
  const uint32_t bpo = bp - m, bpi = bp + m;         // in: p - r wraps iff r > p
  auto load = [&](int j) {
    const uint32_t r = ((j < 4 ? shp.x : shp.y) >> (8 * (j & 3))) & 0xFFu;
    wio[2 * j] = wc[(r >= mp ? bpo : bp) + r];
    wio[2 * j + 1] = wc[(r > p ? bpi : bp) - r];
  };
  if (works && draws == DR) {
#pragma unroll
    for (int j = 0; j < DR; ++j) load(j);
  } else if (works) {
#pragma unroll
    for (int j = 0; j < DR; ++j)
      if (j < draws) load(j);
  }
}

// A push row (RT_SLOTS codes as two uint4, low half of each word first): the
// same adds in slot order; the present bits (14) of both halves of a word are
// counted together in 16-bit lanes of one register.
__device__ __forceinline__ void add_rin_row(float& acc, unsigned& edges, const float* __restrict__ factor,
                                            uint4 in0, uint4 in1) {
  const uint32_t w[8] = {in0.x, in0.y, in0.z, in0.w, in1.x, in1.y, in1.z, in1.w};
  uint32_t pres = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    acc += factor[w[i] & 0xFF];
    acc += factor[(w[i] >> 16) & 0xFF];
    pres += (w[i] >> 14) & 0x00010001u;
  }
  edges += (pres & 0xFFFFu) + (pres >> 16);
}
// A sparse in-row (infectious in-partners only, the rest 0): the same
// slot-ordered adds, skipped when the row is empty -- sixteen additions of
// +0.0f leave a sum >= +0 unchanged, so the result is bitwise add_rin_row's.
__device__ __forceinline__ void add_rin_row_sparse(float& acc, const float* __restrict__ factor, uint4 in0,
                                                   uint4 in1) {
  if ((in0.x | in0.y | in0.z | in0.w | in1.x | in1.y | in1.z | in1.w) == 0u) return;
  unsigned present = 0;
  add_rin_row(acc, present, factor, in0, in1);
}

// Branch-free per-kind sums of for_each_in_code without push rows (the
// fused day kernel of partitioned ranks and of runs too large for the push
// tables): the same visit order, every slot added (absent ones as code 0).
// Needs the day's workplace code table (wt->wcode).
__device__ __forceinline__ void code_kind_sums(const epi_net& net, const PermKeys* __restrict__ rk,
                                               const Radix& dn, const WorkTables* __restrict__ wt,
                                               const uint16_t* __restrict__ codes, int64_t b, uint16_t code_b,
                                               const float* __restrict__ factor, float acc[3], unsigned& edges) {
  {
    const int off = net.hh_off[b];
    const int sz = net.hh_size[b];
    const int64_t start = b - off;
    for (int i = 0; i < sz; ++i) {
      const int64_t c = start + i;
      add_src(acc[0], edges, factor, c == b ? (uint16_t)CODE_DEAD : codes[c]);
    }
  }
  const int w = net.wp_id[b];
  if (w >= 0) {
    const int m = net.wp_size[w];
    if (m >= 2) {
      const int base = net.wp_base[w];
      const int draws = net.colleague_draws;
      const uint32_t p = wt->pos_of[base + net.wp_local[b]];
      const uint8_t* sh = wt->shift + (size_t)w * draws;
      const uint16_t* wc = wt->wcode + base;
      for (int j = 0; j < draws; ++j) {
        const uint32_t r = sh[j];
        add_src(acc[1], edges, factor, wc[add_mod(p, r, (uint32_t)m)]);
        add_src(acc[1], edges, factor, wc[sub_mod(p, r, (uint32_t)m)]);
      }
    }
  }
  if (net.n_agents < 2) return;
  const uint32_t self = (uint32_t)b;
  const int nb = code_count(code_b);
  const int slots = net.random_slots;
  const int nbe = nb < slots ? nb : slots;
  for (int j0 = 0; j0 < nbe; j0 += 4) {
    uint32_t po[4];
    uint16_t co[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) po[q] = (j0 + q < nbe) ? walk_fwd(self, rk[j0 + q], dn) : self;
#pragma unroll
    for (int q = 0; q < 4; ++q) co[q] = po[q] != self ? codes[po[q]] : (uint16_t)CODE_DEAD;
#pragma unroll
    for (int q = 0; q < 4; ++q) add_src(acc[2], edges, factor, co[q]);
  }
  for (int j0 = 0; j0 < slots; j0 += 8) {
    uint32_t pi[8];
    uint16_t ci[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) pi[q] = (j0 + q < slots) ? perm_inv(self, rk[j0 + q], dn) : self;
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (pi[q] >= dn.n) pi[q] = walk_inv(pi[q], rk[j0 + q], dn);
#pragma unroll
    for (int q = 0; q < 8; ++q) ci[q] = pi[q] != self ? codes[pi[q]] : (uint16_t)0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const bool in = j0 + q < code_count(ci[q]);
      acc[2] += in ? factor[ci[q] & 0xFF] : 0.f;
      edges += in ? 1u : 0u;
    }
  }
}

// code_kind_sums with the random in-partners from a SPARSE push row instead
// of 16 inverse slot walks (whole-population runs too large for the full
// push tables): rin[b][j] holds the code of the in-partner of slot j only if
// that source is infectious (code byte != 0); every other slot is 0, and
// factor[0] = 0, so the slot-ordered sum is bitwise that of code_kind_sums.
// The in-edge count cannot come from the row: summed over the population the
// random in-edges between alive agents equal the random out-edges between
// alive agents (each is one (source, slot) pair seen from either end), so
// each alive agent counts its alive out-partners twice.  Only the record's
// population total uses `edges`.
__device__ __forceinline__ void sparse_kind_sums(const epi_net& net, const PermKeys* __restrict__ rk,
                                                 const Radix& dn, const WorkTables* __restrict__ wt,
                                                 const uint16_t* __restrict__ codes, int64_t b, uint16_t code_b,
                                                 const float* __restrict__ factor, float acc[3],
                                                 unsigned& edges, bool& row_used) {
  // the rows stream through L2 once a day (640 MB at 10 M agents): evict-first,
  // so they do not push the codes and the state out
  const uint4* ri = (const uint4*)(wt->rin + (size_t)b * RT_SLOTS);
  const uint4 in0 = __ldcs(ri), in1 = __ldcs(ri + 1);   // issued first: the row's latency under the rest
  {
    // (the agent itself skipped: its slot would add +0.0f and no edge)
    const int off = net.hh_off[b];
    const int sz = net.hh_size[b];
    const uint16_t* hp = codes + (b - off);
    for (int i = 0; i < sz; ++i)
      if (i != off) add_src(acc[0], edges, factor, hp[i]);
  }
  const int w = net.wp_id[b];
  if (w >= 0) {
    const int m = net.wp_size[w];
    if (m >= 2) {
      const int base = net.wp_base[w];
      const int draws = net.colleague_draws;
      const uint32_t p = wt->pos_of[base + net.wp_local[b]];
      if (draws == 8) {                    // every config network: the 8 shifts in one load
        const uint2 shp = *(const uint2*)(wt->shift + (size_t)w * 8);
        uint16_t wio[16];
        load_colleagues<8>(wio, true, wt->wcode, (uint32_t)base, p, (uint32_t)m, shp, 8);
#pragma unroll
        for (int k = 0; k < 16; ++k) add_src(acc[1], edges, factor, wio[k]);
      } else {
        const uint8_t* sh = wt->shift + (size_t)w * draws;
        const uint16_t* wc = wt->wcode + base;
        for (int j = 0; j < draws; ++j) {
          const uint32_t r = sh[j];
          add_src(acc[1], edges, factor, wc[add_mod(p, r, (uint32_t)m)]);
          add_src(acc[1], edges, factor, wc[sub_mod(p, r, (uint32_t)m)]);
        }
      }
    }
  }
  if (net.n_agents < 2) return;
  const uint32_t self = (uint32_t)b;
  const int nb = code_count(code_b);
  const int nbe = nb < RT_SLOTS ? nb : RT_SLOTS;
  unsigned eo = 0;
  for (int j0 = 0; j0 < nbe; j0 += 4) {
    uint32_t po[4];
    uint16_t co[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) po[q] = (j0 + q < nbe) ? walk_fwd(self, rk[j0 + q], dn) : self;
#pragma unroll
    for (int q = 0; q < 4; ++q) co[q] = po[q] != self ? codes[po[q]] : (uint16_t)CODE_DEAD;
#pragma unroll
    for (int q = 0; q < 4; ++q) add_src(acc[2], eo, factor, co[q]);
  }
  edges += 2u * eo;
  row_used = (in0.x | in0.y | in0.z | in0.w | in1.x | in1.y | in1.z | in1.w) != 0u;
  add_rin_row_sparse(acc[2], factor, in0, in1);
}

// Push-table form of for_each_in_code for the fused day kernel, written so
// that every load of a level is issued before any of them is consumed
// (memory-level parallelism for the ~21 warps per SM of a 100k-agent day):
//   level 1: household range, workplace id/slot, rin row, first rout row;
//   level 2: household codes, workplace size/base/shifts, out-partner codes;
//   level 3: the worker's position; level 4: the colleagues' codes.
// The sums are accumulated per kind in exactly the visit order of
// for_each_in_code (household, workplace out/in per draw, random out, random
// in), so results are bitwise those of the generic enumerator.
// Requires the day's push tables (wt->wcode, wt->rin) and <= 8 draws.
__device__ __forceinline__ void push_kind_sums(const epi_net& net, const WorkTables* __restrict__ wt,
                                               const uint16_t* __restrict__ codes, int64_t b, uint16_t code_b,
                                               const float* __restrict__ factor, float acc[3],
                                               unsigned& edges) {
  constexpr int HH = 8, DR = 8;
  // level 1
  const int off = net.hh_off[b];
  const int sz = net.hh_size[b];
  const int w = net.wp_id[b];
  const int loc = net.wp_local[b];
  const uint4* ri = (const uint4*)(wt->rin + (size_t)b * RT_SLOTS);
  const uint4 in0 = ri[0], in1 = ri[1];
  const uint4* ro = (const uint4*)(wt->rout + (size_t)b * RT_SLOTS);
  const uint32_t self = (uint32_t)b;
  const int nb = code_count(code_b);
  const int nbe = nb < RT_SLOTS ? nb : RT_SLOTS;
  const uint4 o0 = nbe > 0 ? ro[0] : make_uint4(self, self, self, self);
  // level 2
  const int64_t start = b - off;
  uint16_t hc[HH];
#pragma unroll
  for (int i = 0; i < HH; ++i) hc[i] = (i < sz && start + i != b) ? codes[start + i] : (uint16_t)CODE_DEAD;
  const int draws = net.colleague_draws;
  int m = 0, base = 0;
  uint8_t sh[DR];
  if (w >= 0) {
    m = net.wp_size[w];
    base = net.wp_base[w];
    const uint8_t* shp = wt->shift + (size_t)w * draws;
#pragma unroll
    for (int j = 0; j < DR; ++j) sh[j] = j < draws ? shp[j] : (uint8_t)0;
  }
  const uint32_t po0[4] = {o0.x, o0.y, o0.z, o0.w};
  uint16_t co0[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) co0[q] = (q < nbe && po0[q] != self) ? codes[po0[q]] : (uint16_t)CODE_DEAD;
  // level 3
  uint32_t p = 0;
  if (w >= 0 && m >= 2) p = wt->pos_of[base + loc];
  // level 4
  uint16_t wo[DR], wi[DR];
#pragma unroll
  for (int j = 0; j < DR; ++j) {
    wo[j] = wi[j] = (uint16_t)CODE_DEAD;
    if (w >= 0 && m >= 2 && j < draws) {
      const uint32_t r = sh[j];
      wo[j] = wt->wcode[base + add_mod(p, r, (uint32_t)m)];
      wi[j] = wt->wcode[base + sub_mod(p, r, (uint32_t)m)];
    }
  }
  // accumulate in visit order
#pragma unroll
  for (int i = 0; i < HH; ++i) add_src(acc[0], edges, factor, hc[i]);
  for (int i = HH; i < sz; ++i) {            // households larger than HH (rare)
    if (start + i == b) continue;
    add_src(acc[0], edges, factor, codes[start + i]);
  }
#pragma unroll
  for (int j = 0; j < DR; ++j) {
    add_src(acc[1], edges, factor, wo[j]);
    add_src(acc[1], edges, factor, wi[j]);
  }
  if (net.n_agents < 2) return;
#pragma unroll
  for (int q = 0; q < 4; ++q) add_src(acc[2], edges, factor, co0[q]);
  for (int j0 = 4; j0 < nbe; j0 += 4) {       // more than 4 out-partners
    const uint4 o = ro[j0 >> 2];
    const uint32_t po[4] = {o.x, o.y, o.z, o.w};
    uint16_t co[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) co[q] = (j0 + q < nbe && po[q] != self) ? codes[po[q]] : (uint16_t)CODE_DEAD;
#pragma unroll
    for (int q = 0; q < 4; ++q) add_src(acc[2], edges, factor, co[q]);
  }
  static_assert(RT_SLOTS == 16, "push rows are two uint4");
  add_rin_row(acc[2], edges, factor, in0, in1);
}

}  // namespace epi
