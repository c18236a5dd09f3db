// The fp32 message pass over tile-packed pre-joined messages (north-star part
// (a); replaces Engine.gather_exposure, engine.py:77-117, in csr mode).
//
// Input, per tile of 32 destination rows (written by k_net_realize):
//   msgs[tile * 32 * msg_cap ...]  the rows' 16-bit messages back to back, each
//                               a byte offset into the fp32 weight table
//                               MsgComb ((source code & 0xFF) << 4 | kind << 2),
//                               every row padded with 0 (weight 0) to whole
//                               4-message half-groups (a 16-byte group holds
//                               two, possibly of two rows);
//   tile_off[tile * 33 + r]     row r's first half-group | pad count << 12;
//   tile_off[tile * 33 + 32]    half-groups in the tile.
//
// Design (B200): see k_msg_pass.  The path is HBM-bound integer/byte work
// plus one fp32 add per message: no tensor cores.
#pragma once

#include "epi_kernels.cuh"

namespace epi {

constexpr int MP_MAX_CAP = 128;           // row capacity of the message path
constexpr int MP_MAX_HALVES = 8 * MP_MAX_CAP;   // 4-message half-groups per tile
constexpr int MP_STEPS = 4;               // groups per lane held in registers
constexpr int MP_WARPS = 8;               // warps per block
constexpr int MP_SMEM = MP_WARPS * MP_MAX_HALVES * 4 + (int)sizeof(MsgComb);

struct MsgTile {
  uint4 v[MP_STEPS];   // 16-byte groups lane, lane + 32, ... of the tile
  int off, groups;     // lane's row: first half-group | pad << 12; half-groups in the tile
  int st, im, ag;      // MODE 0: stage, immune, age band of the lane's row
};

// the two 4-message half sums of a 16-byte group (its halves may belong to
// two rows)
__device__ __forceinline__ float2 group_sums(const uint4& v, const char* __restrict__ comb) {
  const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
  float w[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint32_t m = (j & 1) ? (wv[j >> 1] >> 16) : (wv[j >> 1] & 0xFFFFu);
    w[j] = *(const float*)(comb + m);
  }
  return make_float2((w[0] + w[1]) + (w[2] + w[3]), (w[4] + w[5]) + (w[6] + w[7]));
}

// MODE 0: hazard out (float[N], gather_exposure); MODE 1: fused
// transmission / progression update (+ record and next codes if final_pass).
// Persistent grid, one warp per 32-row tile.  Every row is padded to whole
// 4-message half-groups by the generator, so a half belongs to exactly one row:
// lane l sums groups l, l + 32, ... (one 16-byte load and eight table
// lookups each, no per-message branching) into two half sums in gsum[],
// then the owner of row r adds its half-groups' sums in order.  The next tile's offsets, first
// MP_STEPS groups and state bytes are loaded into registers while the
// current tile is summed (two register sets, alternating).
// MODE 0 at 4 blocks per SM (64 registers, no spills): 0.131 -> 0.123 ms at
// 10 M agents; MODE 1 (with the update) spills at 64 and stays at 3.
template <int MODE>
__global__ void __launch_bounds__(MP_WARPS * 32, MODE == 0 ? 4 : 3) k_msg_pass(StepArgs A, CsrView g, float* __restrict__ lam_out,
                                                            int final_pass, uint16_t* __restrict__ codes_next,
                                                            const epi_net* net, uint64_t rcount_next,
                                                            const MsgTables* __restrict__ mt,
                                                            const MsgComb* __restrict__ mc) {
  __shared__ MsgTables T;
  __shared__ RecAcc racc;
  extern __shared__ __align__(16) float mp_smem[];
  const int warp = threadIdx.x >> 5, lane = lane_id();
  MsgComb* C = (MsgComb*)mp_smem;
  float* gsum = mp_smem + sizeof(MsgComb) / 4 + warp * MP_MAX_HALVES;
  for (int i = threadIdx.x; i < 4 * 256; i += blockDim.x) C->w[i] = mc->w[i];
  load_msg_tables(T, mt);
  rec_init(racc);
  __syncthreads();
  pdl_wait();
  pdl_trigger();
  const epi_params* __restrict__ P = A.P;
  const char* __restrict__ comb = (const char*)C->w;
  const int lo_row = (int)A.lo, n = (int)A.hi;
  const int n_tiles = (n - lo_row + 31) >> 5;
  const int wstride = gridDim.x * MP_WARPS;
  const int t0 = blockIdx.x * MP_WARPS + warp;
  const uint16_t* __restrict__ toff = g.tile_off;
  const int tile_words = 4 * msg_cap(g.cap);        // 16-byte words (groups) per tile block
  const uint4* __restrict__ msgs = (const uint4*)g.msgs;
  auto load_offsets = [&](MsgTile& X, int t) {
    X.off = X.groups = 0;
    if (t < n_tiles) {
      X.off = __ldg(toff + t * 33 + lane);
      X.groups = __ldg(toff + t * 33 + 32);
    }
  };
  auto load_rest = [&](MsgTile& X, int t) {
    X.st = S_DEAD;
    X.im = X.ag = 0;
    const uint4* blk = msgs + (size_t)t * tile_words;
    const int g16 = (X.groups + 1) >> 1;                     // 16-byte groups
#pragma unroll
    for (int q = 0; q < MP_STEPS; ++q)
      X.v[q] = (t < n_tiles && q * 32 + lane < g16) ? __ldg(blk + q * 32 + lane) : make_uint4(0, 0, 0, 0);
    const int a = lo_row + t * 32 + lane;
    if (MODE == 0 && t < n_tiles && a < n) {
      X.st = A.st.stage[a];
      X.im = A.st.immune[a];
      X.ag = A.st.age_band[a];
    }
  };
  unsigned edges = 0;
  int off2, grp2;
  // one tile: load tile t1 into Xn (its offsets are already there) and tile
  // t2's offsets, then sum tile `tile` from Xc
  auto body = [&](MsgTile& Xc, MsgTile& Xn, int tile) {
    const int t1 = tile + wstride, t2 = tile + 2 * wstride;
    load_rest(Xn, t1);
    off2 = grp2 = 0;
    if (t2 < n_tiles) {
      off2 = __ldg(toff + t2 * 33 + lane);
      grp2 = __ldg(toff + t2 * 33 + 32);
    }
    const int a = lo_row + tile * 32 + lane;
    const bool valid = a < n;
    const uint4* blk = msgs + (size_t)tile * tile_words;
    // MODE 1: the row's state, loaded before the sums so the loads overlap them
    AgentHot h{};
    if (MODE == 1 && valid) h = load_hot(A.st, a);
    // group sums
    const int g16 = (Xc.groups + 1) >> 1;
    float2* gsum2 = (float2*)gsum;
#pragma unroll
    for (int q = 0; q < MP_STEPS; ++q)
      if (q * 32 < g16) {
        const int gi = q * 32 + lane;
        if (gi < g16) gsum2[gi] = group_sums(Xc.v[q], comb);
      }
    for (int gi = MP_STEPS * 32 + lane; gi < g16; gi += 32) gsum2[gi] = group_sums(__ldg(blk + gi), comb);
    __syncwarp();
    // row sums: half-groups [h0, h1) of the lane's row, in order
    const int h0 = Xc.off & 0xFFF;
    const int hn = __shfl_down_sync(0xFFFFFFFFu, h0, 1);
    const int h1 = lane < 31 ? hn : Xc.groups;
    float acc = 0.f;
#pragma unroll 4
    for (int hi = h0; hi < h1; ++hi) acc += gsum[hi];
    __syncwarp();
    if (valid) edges += (unsigned)(4 * (h1 - h0) - (Xc.off >> 12));
    if (MODE == 0) {
      if (valid) {
        const bool target = Xc.st == S_SUS && !(P->sterilizing && Xc.im);
        lam_out[a] = target ? acc * T.sfac[Xc.ag] : 0.f;
      }
    } else {
      double lam = 0.0;
      if (valid && h.stage == S_SUS && !(P->sterilizing && h.immune)) lam = (double)(acc * T.sfac[h.age]);
      unsigned ev = 0;
      if (valid) probe_lambda(A.probe, A.step, a, lam);
      if (valid) ev = transmit_progress_hot(A, a, lam, -1, h);
      if (valid && (ev & 8u) && A.flags) A.flags[a] = FL_SYMPTOMATIC;
      rec_events(racc, ev);
      if (final_pass) {
        rec_agent(racc, valid, valid ? h.stage : 0, valid ? h.infected_at : 0);
        if (valid && codes_next) codes_next[a] = next_code_hot(P, h, a, A.step + 1, net, rcount_next);
      }
    }
  };
  MsgTile X0, X1;
  load_offsets(X0, t0);
  load_rest(X0, t0);
  load_offsets(X1, t0 + wstride);
  for (int tile = t0; tile < n_tiles; tile += 2 * wstride) {
    body(X0, X1, tile);
    X0.off = off2;
    X0.groups = grp2;
    if (tile + wstride >= n_tiles) break;
    body(X1, X0, tile + wstride);
    X1.off = off2;
    X1.groups = grp2;
  }
  rec_add(racc, EPI_REC_EDGES, edges);
  __syncthreads();
  rec_flush(racc, A.rec, A.step);
}

}  // namespace epi
