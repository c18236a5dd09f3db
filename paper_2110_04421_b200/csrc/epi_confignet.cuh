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

struct PermKeys {
  uint32_t mult[3], inv[3], key[3];
};

__host__ __device__ __forceinline__ uint32_t inv_odd32(uint32_t m) {
  uint32_t x = m;                 // correct to 3 bits for odd m
  x *= 2u - m * x;                // 6
  x *= 2u - m * x;                // 12
  x *= 2u - m * x;                // 24
  x *= 2u - m * x;                // 48
  return x;
}

__host__ __device__ __forceinline__ int domain_bits(uint32_t n) {
  // smallest k >= 1 with 2^k >= n
  uint32_t v = n > 1 ? n - 1 : 1;
  int k = 0;
  while (v) { ++k; v >>= 1; }
  return k < 1 ? 1 : k;
}

// One application of the 3-round multiply / xorshift bijection of [0, 2^k).
__device__ __forceinline__ uint32_t perm_fwd(uint32_t x, const PermKeys& K, uint32_t mask, int s) {
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    x = ((x ^ (K.key[r] & mask)) * K.mult[r]) & mask;
    x ^= x >> s;
  }
  return x;
}
__device__ __forceinline__ uint32_t perm_inv(uint32_t y, const PermKeys& K, uint32_t mask, int s) {
#pragma unroll
  for (int r = 2; r >= 0; --r) {
    y ^= y >> s;
    y = ((y * K.inv[r]) & mask) ^ (K.key[r] & mask);
  }
  return y;
}
// Cycle walking restricts the bijection of [0, 2^k) to [0, n).
__device__ __forceinline__ uint32_t walk_fwd(uint32_t x, const PermKeys& K, uint32_t n,
                                             uint32_t mask, int s) {
  do { x = perm_fwd(x, K, mask, s); } while (x >= n);
  return x;
}
__device__ __forceinline__ uint32_t walk_inv(uint32_t y, const PermKeys& K, uint32_t n,
                                             uint32_t mask, int s) {
  do { y = perm_inv(y, K, mask, s); } while (y >= n);
  return y;
}

// Hash prefixes of one generated step (purposes 72-75 at (graph_seed, step)).
struct NetKeys {
  uint64_t rcount, rperm, wperm, wshift;
};
inline NetKeys make_net_keys(uint64_t g, int step) {
  return NetKeys{key_prefix(g, step, P_NET_RCOUNT), key_prefix(g, step, P_NET_RPERM),
                 key_prefix(g, step, P_NET_WPERM), key_prefix(g, step, P_NET_WSHIFT)};
}

__device__ __forceinline__ PermKeys random_slot_keys(uint64_t rperm_prefix, int slot) {
  PermKeys K;
  const uint64_t hs = fold(rperm_prefix, (uint64_t)slot);
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    const uint64_t h = fold(hs, (uint64_t)r);
    K.mult[r] = (uint32_t)h | 1u;
    K.inv[r] = inv_odd32(K.mult[r]);
    K.key[r] = (uint32_t)(h >> 32);
  }
  return K;
}

__device__ __forceinline__ PermKeys work_keys(uint64_t wperm_prefix, int w) {
  PermKeys K;
  const uint64_t h = fold(fold(wperm_prefix, (uint64_t)w), 0);
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    K.mult[r] = (uint32_t)((h >> (16 * r)) & 0xFF) | 1u;
    K.inv[r] = inv_odd32(K.mult[r]);
    K.key[r] = (uint32_t)((h >> (16 * r + 8)) & 0xFF);
  }
  return K;
}

// Random-slot count n_{t,a} ~ Poisson(mean) truncated at `slots`.
__device__ __forceinline__ int random_count(const epi_net& net, uint64_t rcount_prefix, int64_t a) {
  const double u = keyed_u(rcount_prefix, (uint64_t)a, 0);
  int c = 0;
  for (int k = 0; k < net.random_slots; ++k) c += (u >= net.poisson_cdf[k]) ? 1 : 0;
  return c;
}

// Enumerate the in-edges of destination b (alive); visit(src, kind, code_src).
// Order: household members ascending, workplace slots (out, in), random slots
// (out, in).  `rk` holds the random-slot keys of this step (shared memory).
template <class Visit>
__device__ __forceinline__ void for_each_in_edge(const epi_net& net, const NetKeys& nk,
                                                 const PermKeys* __restrict__ rk,
                                                 const uint16_t* __restrict__ codes, int64_t b,
                                                 uint16_t code_b, Visit&& visit) {
  // household: contiguous range
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
      const int kb = domain_bits((uint32_t)m);
      const uint32_t mask = (1u << kb) - 1u;
      const int s = (kb + 1) >> 1;
      const PermKeys K = work_keys(nk.wperm, w);
      const int base = net.wp_base[w];
      const uint32_t p = walk_inv(net.wp_local[b], K, (uint32_t)m, mask, s);
      uint64_t hq = 0;
      for (int j = 0; j < net.colleague_draws; ++j) {
        if ((j & 3) == 0) hq = fold(fold(nk.wshift, (uint64_t)w), (uint64_t)(j >> 2));
        const uint32_t v = (uint32_t)((hq >> (16 * (j & 3))) & 0xFFFF);
        const uint32_t r = 1u + ((v * (uint32_t)(m - 1)) >> 16);
        const uint32_t po = (p + r) % (uint32_t)m;
        const uint32_t pi = (p + (uint32_t)m - r) % (uint32_t)m;
        const int32_t co = net.wp_members[base + walk_fwd(po, K, (uint32_t)m, mask, s)];
        const uint16_t cco = codes[co];
        if (!code_dead(cco)) visit((int64_t)co, 1, cco);
        const int32_t ci = net.wp_members[base + walk_fwd(pi, K, (uint32_t)m, mask, s)];
        const uint16_t cci = codes[ci];
        if (!code_dead(cci)) visit((int64_t)ci, 1, cci);
      }
    }
  }
  // random slots
  const uint32_t n = (uint32_t)net.n_agents;
  if (n >= 2 && net.random_slots > 0) {
    const int kb = domain_bits(n);
    const uint32_t mask = (kb >= 32) ? 0xFFFFFFFFu : ((1u << kb) - 1u);
    const int s = (kb + 1) >> 1;
    const int nb = code_count(code_b);
    for (int j = 0; j < net.random_slots; ++j) {
      const PermKeys& K = rk[j];
      if (j < nb) {
        const uint32_t c = walk_fwd((uint32_t)b, K, n, mask, s);
        if (c != (uint32_t)b) {
          const uint16_t cc = codes[c];
          if (!code_dead(cc)) visit((int64_t)c, 2, cc);
        }
      }
      const uint32_t c = walk_inv((uint32_t)b, K, n, mask, s);
      if (c != (uint32_t)b) {
        const uint16_t cc = codes[c];
        if (j < code_count(cc)) visit((int64_t)c, 2, cc);
      }
    }
  }
}

}  // namespace epi
