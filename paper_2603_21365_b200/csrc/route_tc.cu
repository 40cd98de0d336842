// K1 (+K2 fused): fused RMSNorm + router + exit mask + stable compaction on
// tcgen05 tensor cores.
//
// Restates, for a block of rows at once:
//   ee/router_ops.py:68-87   fused_layernorm_route  (score per row)
//   ee/runtime.py:149,171    mask = score > f32(theta)       (strict)
//   ee/router_ops.py:116-134 _compact_prefix_sum    (stable partition indices)
//   ee/runtime.py:175-178    exited_at / exit_layers / remaining (row_idx mode)
//
// Layout: h [rows, d] (bf16 | f16) row-major, W_down [b, d] same dtype
// (K-major for the MMA), w_up [b] f32.  Accumulator D = h_tile . W^T lives in
// TMEM (128 lanes = 128 tokens, N = b columns, f32).
//
// CTA roles (352 threads, one CTA per SM, persistent over row groups of up
// to 4 token tiles of 128 rows):
//   warp 0      TMA producer: W k-chunks into the W ring, A k-chunks into the
//               A ring (128-row boxes, 64/32/16-row boxes for the ragged
//               tail, tile::gather4 rows when peeling by row_idx).
//   warp 1      TMEM allocator + MMA issuer (one elected lane).  Phase 1,
//               K-outer / M-inner: each W k-chunk in smem feeds every tile of
//               the group, whose accumulators all live in TMEM (4 x 128 cols),
//               so W is read from L2 once per group.  Phase 2, tile-major over
//               the last nw k-chunks (their W slots stay resident): tiles
//               complete one after another and their epilogues overlap the
//               stream of later tiles.
//   warps 2-9   two sets of 4 (set 0: tiles 0 and 2, set 1: tiles 1 and 3):
//               sum of squares of their tiles' A slots from smem while the
//               MMAs run (FHFMA), then each tile's epilogue as soon as its
//               accumulator is complete: tcgen05.ld (two in flight), scale,
//               SiLU (tanh form), dot w_up, f64 sigmoid, strict threshold,
//               ballots.
//   warp 10     compaction: per-group popc scan + flat look-back over all
//               predecessors' tagged aggregates, int64 exit / continuing
//               indices.
// Launched with programmatic dependent launch (see route_tc_launch).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "internal.h"

namespace tide {

constexpr int kThreadsTC = 352;  // 11 warps: producer, MMA, 2 x 4 epilogue, compaction
constexpr int kMaxNA = 16;
constexpr int kMaxNW = 4;
constexpr int kASlotBytes = 128 * 128;  // 128 rows x 64 cols x 2 B
constexpr int kMaxMC = 24;              // checkpoints of one K1m launch

struct TcParams {
  int64_t n_host;
  const int64_t* n_dev;
  int64_t rows_total;
  int32_t d, b, npad, bp, tpg, nk, na, nw, nx, gran;
  int32_t pair;  // 1: an A slot holds two tiles (one 256-row TMA box, 32 KB, one barrier cycle)
  uint32_t idesc, tmem_cols, wslot;
  uint32_t off_a, off_wup, off_bar, off_words, off_ids, off_tmem;
  const int64_t* row_idx;
  int32_t ids_from_rows;
  const float* w_up;
  float eps, inv_d, theta;
  int64_t layer;
  int32_t inputs_ready;  // TIDE_ROUTE_INPUTS_READY
  float* scores;
  float* logits;
  uint8_t* mask;
  int64_t* exit_idx;
  int64_t* cont_idx;
  int64_t* exit_layers;
  int64_t* counts;
  Workspace* ws;
  unsigned long long* dbg;  // optional per-CTA timeline (globaltimer ns), 8 slots per CTA
  // K1m (NC > 1): nc checkpoints in one launch; checkpoint c reads its rows
  // through MultiMaps::h[c], its router through MultiMaps::w[c] / wups[c] and
  // writes scores[c * cap + position]; gathered launches route only when
  // n_min <= *n_dev <= n_limit
  int32_t nc;
  int64_t cap, n_min, n_limit;
  const float* wups[kMaxMC];
  int64_t layers[kMaxMC];  // exit layer of checkpoint c (ascending)
};

// exit_layers[row] = min(current, layer) where NO_EXIT (-1) counts as +inf:
// the first firing checkpoint of a row scored by several CTAs at once
// (deterministic: the result is a minimum, whatever the arrival order)
__device__ __forceinline__ void exit_min(int64_t* slot, int64_t layer) {
  unsigned long long* a = reinterpret_cast<unsigned long long*>(slot);
  long long cur = *reinterpret_cast<volatile long long*>(slot);
  while (cur < 0 || cur > layer) {
    const long long prev = (long long)atomicCAS(a, (unsigned long long)cur, (unsigned long long)layer);
    if (prev == cur) break;
    cur = prev;
  }
}

// Per-checkpoint tensor maps of a K1m launch (kernel parameters): h[c] is the
// 128-row box map of capture c (dense) or its 1-row gather4 map (gathered).
template <int NC>
struct MultiMaps {
  CUtensorMap h[NC];
  CUtensorMap w[NC];
  CUtensorMap p[NC];  // dense pair slots: the 256-row box map of capture c
};
template <>
struct MultiMaps<1> {
  int unused;
};
template <int NC>
__device__ __forceinline__ const CUtensorMap* mm_h(const MultiMaps<NC>& m, int c) {
  if constexpr (NC > 1) return &m.h[c];
  else return nullptr;
}
template <int NC>
__device__ __forceinline__ const CUtensorMap* mm_p(const MultiMaps<NC>& m, int c) {
  if constexpr (NC > 1) return &m.p[c];
  else return nullptr;
}
template <int NC>
__device__ __forceinline__ const CUtensorMap* mm_w(const MultiMaps<NC>& m, int c) {
  if constexpr (NC > 1) return &m.w[c];
  else return nullptr;
}

// The groups of rows one CTA walks, in the same order in every role.
//  NC == 1: groups g = blockIdx.x, + gridDim.x, ... of NG balanced groups of
//           whole gran-row units (group_range).
//  NC > 1:  CTA b owns virtual tiles [b TT / G, (b + 1) TT / G) of the
//           checkpoint-major tile space (TT = nc x Tc, Tc = tiles per
//           checkpoint); a group is up to tpg consecutive tiles of ONE
//           checkpoint (its W chunk feeds all of them).
struct GroupIter {
  int64_t g, NG, G, n, n32;
  int gran;
  int64_t v, vend, Tc;
  int tpg;
};

// Cycle counters inside the streaming loops only in profiling builds
// (-DTIDE_K1_PROFILE=1, tools/timeline.py): CS2R reads in the hot loops cost
// issue slots the MMA warp shares.
#ifndef TIDE_K1_PROFILE
#define TIDE_K1_PROFILE 0
#endif
__device__ __forceinline__ long long pclk() {
#if TIDE_K1_PROFILE
  return clock64();
#else
  return 0;
#endif
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Groups are balanced in units of p.gran rows: 16 (the smallest TMA box of
// the ragged tail; per-CTA work differs by at most 16 rows) or, once every
// CTA holds at least two tiles, 128 — whole tiles per CTA: no MMA on padding
// rows (a balanced split of 65,536 rows gives every CTA a 59-row fourth tile,
// 15% of the tensor work on padding) at the price of a one-tile imbalance;
// measured faster both in the timed region and power-capped.
constexpr int kGran = 16;
constexpr int kBox = 16;  // smallest TMA box of the ragged tail
__device__ __forceinline__ void group_range(int64_t g, int64_t n, int64_t nu, int64_t ng,
                                            int gran, int64_t& r0, int64_t& r1) {
  r0 = (g * nu / ng) * gran;
  r1 = ((g + 1) * nu / ng) * gran;
  if (r1 > n) r1 = n;
}

template <int NC>
__device__ __forceinline__ bool next_group(GroupIter& it, int& c, int64_t& g, int64_t& r0,
                                           int64_t& r1) {
  if constexpr (NC == 1) {
    if (it.g >= it.NG) return false;
    c = 0;
    g = it.g;
    group_range(it.g, it.n, it.n32, it.NG, it.gran, r0, r1);
    it.g += it.G;
    return true;
  } else {
    if (it.v >= it.vend) return false;
    c = (int)(it.v / it.Tc);
    const int64_t t0 = it.v - (int64_t)c * it.Tc;
    int64_t t1 = t0 + it.tpg;
    if (t1 > it.Tc) t1 = it.Tc;
    if (t1 - t0 > it.vend - it.v) t1 = t0 + (it.vend - it.v);
    g = it.v;
    r0 = t0 * 128;
    r1 = t1 * 128 < it.n ? t1 * 128 : it.n;
    it.v += t1 - t0;
    return true;
  }
}

template <bool kBF16, int NC>
__global__ void __launch_bounds__(kThreadsTC, 1)
    route_tc_kernel(const __grid_constant__ CUtensorMap tm_h128,
                    const __grid_constant__ CUtensorMap tm_h64,
                    const __grid_constant__ CUtensorMap tm_h32b,
                    const __grid_constant__ CUtensorMap tm_h32,
                    const __grid_constant__ CUtensorMap tm_w,
                    const __grid_constant__ CUtensorMap tm_g4,
                    const __grid_constant__ CUtensorMap tm_h256,
                    const __grid_constant__ MultiMaps<NC> mm, const __grid_constant__ TcParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sW = smem;
  // pair mode: slot = two tiles' 64-column chunk (rows 0-127: tile 2j, rows
  // 128-255: tile 2j+1); every RMS warp of both sets reads it
  const uint32_t slot_bytes = p.pair ? 2u * kASlotBytes : (uint32_t)kASlotBytes;
  uint8_t* sA = smem + p.off_a;
  float* sWup = reinterpret_cast<float*>(smem + p.off_wup);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.off_bar);
  uint64_t* w_full = bars;
  uint64_t* w_empty = bars + kMaxNW;
  uint64_t* a_full = bars + 2 * kMaxNW;
  uint64_t* a_empty = a_full + kMaxNA;
  uint64_t* t_full = a_empty + kMaxNA;
  uint64_t* t_empty = t_full + 4;
  uint64_t* m_full = t_empty + 4;
  uint64_t* m_empty = m_full + 2;
  uint32_t* words = reinterpret_cast<uint32_t*>(smem + p.off_words);
  uint32_t* ids = reinterpret_cast<uint32_t*>(smem + p.off_ids);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + p.off_tmem);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // PDL: inputs written by the previous launch (the peeled chain's live count
  // and row index) are read only after it completed; otherwise this grid
  // streams its rows while the previous one finishes its tail, and waits only
  // before its first global write / look-back (epilogue and compaction warps).
  // PDL: this grid may be resident before the previous kernel on the stream
  // has finished; griddepcontrol.wait is what makes that kernel's writes
  // visible.  Wait before the first read of any input (h, W_down, w_up, the
  // previous link's live count / row index) unless the caller asserted that
  // the kernel in flight writes none of them (TIDE_ROUTE_INPUTS_READY and no
  // row index: back-to-back routing of a resident buffer) — then the stream
  // starts while the previous grid drains and only the writes wait.
  const bool dep_inputs = p.n_dev != nullptr || p.row_idx != nullptr || !p.inputs_ready;
  if (dep_inputs) griddep_wait();
  if (threadIdx.x == 0) griddep_launch_dependents();
  int64_t n = p.n_dev ? *p.n_dev : p.n_host;
  if (NC > 1 && p.n_dev && (n < p.n_min || n > p.n_limit)) n = 0;  // K1m tail gate
  const int64_t n32 = (n + p.gran - 1) / p.gran;  // number of gran-row units
  const int64_t G = gridDim.x;
  const int64_t cpg = (int64_t)p.tpg * (128 / p.gran);
  int64_t NG = n32 < G ? n32 : G;
  if ((n32 + cpg - 1) / cpg > NG) NG = (n32 + cpg - 1) / cpg;
  const bool gathered = p.row_idx != nullptr;
  const bool need_scan = NC == 1 && (p.exit_idx || p.cont_idx || p.counts);
  auto make_iter = [&]() {
    GroupIter it;
    it.g = blockIdx.x;
    it.NG = NG;
    it.G = G;
    it.n = n;
    it.n32 = n32;
    it.gran = p.gran;
    it.tpg = p.tpg;
    it.Tc = (n + 127) / 128;
    const int64_t TT = (int64_t)p.nc * it.Tc;
    it.v = (int64_t)blockIdx.x * TT / G;
    it.vend = ((int64_t)blockIdx.x + 1) * TT / G;
    return it;
  };

  if (warp == 0 && lane == 0) {
    if constexpr (NC > 1) {
      for (int c = 0; c < p.nc; ++c) {
        prefetch_tmap(mm_w<NC>(mm, c));
        prefetch_tmap(p.pair ? mm_p<NC>(mm, c) : mm_h<NC>(mm, c));
      }
    } else {
      prefetch_tmap(&tm_w);
      prefetch_tmap(gathered ? &tm_g4 : &tm_h128);
      if (!gathered) prefetch_tmap(p.pair ? &tm_h256 : &tm_h32);
    }
    for (int i = 0; i < p.nw; ++i) {
      mbar_init(&w_full[i], 1);
      mbar_init(&w_empty[i], 1);
    }
    for (int i = 0; i < p.na; ++i) {
      mbar_init(&a_full[i], 1);
      // MMA commit + all 8 RMS warps (each waits every slot, reads its own tile's)
      mbar_init(&a_empty[i], 1 + 8);
    }
    for (int i = 0; i < 4; ++i) {
      mbar_init(&t_full[i], 1);
      mbar_init(&t_empty[i], 4);  // the 4 epilogue warps owning the tile
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&m_full[i], 8);
      mbar_init(&m_empty[i], 1);
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    tmem_alloc(tmem_slot, p.tmem_cols);
    tmem_relinquish();
  }
  if (NC == 1)
    for (int i = threadIdx.x; i < p.b; i += blockDim.x) sWup[i] = p.w_up[i];
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  unsigned long long* dbg = p.dbg ? p.dbg + 24 * blockIdx.x : nullptr;
  if (dbg && threadIdx.x == 0) dbg[0] = gtimer();

  if (warp == 0) {
    // ----------------------------------------------------------- producer
    const uint64_t pol_h = policy_evict_first();
    const uint64_t pol_w = policy_evict_last();
    int as = 0, aph = 0, wsl = 0, wph = 0;
    long long pw_cyc = 0, p_begin = pclk();
    GroupIter it = make_iter();
    int c;
    int64_t g, r0, r1;
    while (next_group<NC>(it, c, g, r0, r1)) {
      const int T = (int)((r1 - r0 + 127) / 128);
      const CUtensorMap* const tw = NC > 1 ? mm_w<NC>(mm, c) : &tm_w;
      const CUtensorMap* const th = NC > 1 ? mm_h<NC>(mm, c) : (gathered ? &tm_g4 : &tm_h128);
      if (gathered) {
        __syncwarp();
        for (int64_t i = r0 + lane; i < r0 + (int64_t)T * 128; i += 32)
          ids[i - r0] = i < r1 ? (uint32_t)p.row_idx[i] : (uint32_t)p.rows_total;
        __syncwarp();
      }
      if (lane == 0) {
        auto load_w = [&](int kc) {
          mbar_wait(&w_empty[wsl], wph ^ 1);
          mbar_arrive_expect_tx(&w_full[wsl], p.wslot);
          tma_load_2d(sW + (size_t)wsl * p.wslot, tw, &w_full[wsl], kc * 64, 0, pol_w);
          if (++wsl == p.nw) { wsl = 0; wph ^= 1; }
        };
        auto load_pair = [&](int kc, int pt) {
          mbar_wait(&a_empty[as], aph ^ 1);
          uint8_t* dst = sA + (size_t)as * slot_bytes;
          const int64_t rb = r0 + (int64_t)pt * 256;
          const bool two = 2 * pt + 1 < T;
          mbar_arrive_expect_tx(&a_full[as], two ? 2u * kASlotBytes : (uint32_t)kASlotBytes);
          const CUtensorMap* const tp =
              NC > 1 ? (two ? mm_p<NC>(mm, c) : th) : (two ? &tm_h256 : &tm_h128);
          tma_load_2d(dst, tp, &a_full[as], kc * 64, (int)rb, pol_h);
          if (++as == p.na) { as = 0; aph ^= 1; }
        };
        auto load_a = [&](int kc, int t) {
          const long long q0 = pclk();
          mbar_wait(&a_empty[as], aph ^ 1);
          pw_cyc += pclk() - q0;
          uint8_t* dst = sA + (size_t)as * slot_bytes;
          const int64_t rb = r0 + (int64_t)t * 128;
          const int rows_in = (int)((r1 - rb) < 128 ? (r1 - rb) : 128);
          if (!gathered) {
            if (rows_in == 128 || NC > 1) {
              // K1m groups are whole tiles: a ragged tile is the capture's
              // last one, its out-of-range rows are zero-filled (no reads)
              mbar_arrive_expect_tx(&a_full[as], kASlotBytes);
              tma_load_2d(dst, th, &a_full[as], kc * 64, (int)rb, pol_h);
            } else {
              // ragged tail: greedy 64/32/16-row boxes (16-row boxes stream poorly)
              const int rr = (rows_in + kBox - 1) / kBox * kBox;
              mbar_arrive_expect_tx(&a_full[as], (uint32_t)(rr * 128));
              int off = 0;
              if (rr - off >= 64) {
                tma_load_2d(dst, &tm_h64, &a_full[as], kc * 64, (int)rb, pol_h);
                off += 64;
              }
              if (rr - off >= 32) {
                tma_load_2d(dst + off * 128, &tm_h32b, &a_full[as], kc * 64, (int)(rb + off), pol_h);
                off += 32;
              }
              if (rr - off >= 16) {
                tma_load_2d(dst + off * 128, &tm_h32, &a_full[as], kc * 64, (int)(rb + off), pol_h);
                off += 16;
              }
            }
          } else {
            const int ng4 = (rows_in + 3) / 4;
            mbar_arrive_expect_tx(&a_full[as], ng4 * 512);
            const uint32_t* id = ids + t * 128;
            for (int q = 0; q < ng4; ++q)
              tma_gather4(dst + q * 512, th, &a_full[as], kc * 64, (int)id[4 * q],
                          (int)id[4 * q + 1], (int)id[4 * q + 2], (int)id[4 * q + 3], pol_h);
          }
          if (++as == p.na) { as = 0; aph ^= 1; }
        };
        // phase 1 (K-outer): chunk kc's W slot feeds all T tiles
        const int P1 = p.nk - p.nx;
        const int NP = (T + 1) / 2;
        for (int kc = 0; kc < P1; ++kc) {
          load_w(kc);
          if (p.pair)
            for (int pt = 0; pt < NP; ++pt) load_pair(kc, pt);
          else
            for (int t = 0; t < T; ++t) load_a(kc, t);
        }
        // phase 2 (tile-major over the last nx chunks, whose W slots stay
        // resident): tile t's accumulator completes while later tiles still
        // stream, so its epilogue overlaps the tail of the stream (pair mode:
        // pair-major, tiles 2j and 2j+1 complete together)
        if (p.pair) {
          for (int pt = 0; pt < NP; ++pt)
            for (int j = 0; j < p.nx; ++j) {
              if (pt == 0) load_w(P1 + j);
              load_pair(P1 + j, pt);
            }
        } else {
          for (int t = 0; t < T; ++t)
            for (int j = 0; j < p.nx; ++j) {
              if (t == 0) load_w(P1 + j);
              load_a(P1 + j, t);
            }
        }
      }
    }
    if (dbg && lane == 0) { dbg[1] = gtimer(); dbg[18] = pw_cyc; dbg[19] = pclk() - p_begin; }
  } else if (warp == 1) {
    // ----------------------------------------------------------- MMA issuer
    // The whole warp walks the loop (warp-uniform state -> uniform registers);
    // one elected lane issues.  Descriptors are built once per slot and
    // advanced by +2 (32 bytes >> 4) per K=16 step.
    int as = 0, aph = 0, wsl = 0, wph = 0;
    uint32_t accph = 0;
    long long wait_cyc = 0, t_begin = pclk();
    const uint64_t desc_hi = sw128_kmajor_desc(0);
    GroupIter it = make_iter();
    int c;
    int64_t g, r0, r1;
    while (next_group<NC>(it, c, g, r0, r1)) {
      const int T = (int)((r1 - r0 + 127) / 128);
      for (int t = 0; t < T; ++t) mbar_wait(&t_empty[t], ((accph >> t) & 1u) ^ 1u);
      tc_fence_after();
      auto mma_slot = [&](int kc, int t, uint64_t bdesc) {
        const long long w1 = pclk();
        mbar_wait(&a_full[as], aph);
        wait_cyc += pclk() - w1;
        tc_fence_after();
        if (elect_one()) {
          const uint64_t adesc =
              desc_hi | (uint64_t)((smem_u32(sA + (size_t)as * slot_bytes) & 0x3FFFFu) >> 4);
          const uint32_t dt = tmem_base + (uint32_t)(t * p.bp);
#pragma unroll
          for (int k = 0; k < 4; ++k)
            tc_mma_f16(dt, adesc + 2 * k, bdesc + 2 * k, p.idesc, (kc | k) != 0);
          // the slot is released as soon as ITS 4 MMAs retire
          tc_commit(&a_empty[as]);
          if (kc == p.nk - 1) tc_commit(&t_full[t]);
        }
        __syncwarp();
        if (++as == p.na) { as = 0; aph ^= 1; }
      };
      auto wdesc = [&](int slot) {
        return desc_hi | (uint64_t)((smem_u32(sW + (size_t)slot * p.wslot) & 0x3FFFFu) >> 4);
      };
      // pair slot: tile 2pt from rows 0-127, tile 2pt+1 from rows 128-255
      auto mma_pair = [&](int kc, int pt, uint64_t bdesc) {
        mbar_wait(&a_full[as], aph);
        tc_fence_after();
        if (elect_one()) {
          const uint64_t adesc =
              desc_hi | (uint64_t)((smem_u32(sA + (size_t)as * slot_bytes) & 0x3FFFFu) >> 4);
          const int nt = (2 * pt + 1 < T) ? 2 : 1;
          for (int u = 0; u < nt; ++u) {
            const int t = 2 * pt + u;
            const uint64_t ad = adesc + (uint64_t)((u * kASlotBytes) >> 4);
            const uint32_t dt = tmem_base + (uint32_t)(t * p.bp);
#pragma unroll
            for (int k = 0; k < 4; ++k)
              tc_mma_f16(dt, ad + 2 * k, bdesc + 2 * k, p.idesc, (kc | k) != 0);
            if (kc == p.nk - 1) tc_commit(&t_full[t]);
          }
          tc_commit(&a_empty[as]);
        }
        __syncwarp();
        if (++as == p.na) { as = 0; aph ^= 1; }
      };
      const int NP = (T + 1) / 2;
      // phase 1: K-outer
      const int P1 = p.nk - p.nx;
      for (int kc = 0; kc < P1; ++kc) {
        const long long w0 = pclk();
        mbar_wait(&w_full[wsl], wph);
        wait_cyc += pclk() - w0;
        const uint64_t bdesc = wdesc(wsl);
        if (p.pair)
          for (int pt = 0; pt < NP; ++pt) mma_pair(kc, pt, bdesc);
        else
          for (int t = 0; t < T; ++t) mma_slot(kc, t, bdesc);
        if (elect_one()) tc_commit(&w_empty[wsl]);
        __syncwarp();
        if (++wsl == p.nw) { wsl = 0; wph ^= 1; }
      }
      // phase 2: tile-major over the last nx chunks (W slots wsl .. wsl+nx-1)
      if (p.pair) {
        for (int pt = 0; pt < NP; ++pt) {
          int sl = wsl, ph = wph;
          for (int j = 0; j < p.nx; ++j) {
            if (pt == 0) mbar_wait(&w_full[sl], ph);
            mma_pair(P1 + j, pt, wdesc(sl));
            if (pt == NP - 1) {
              if (elect_one()) tc_commit(&w_empty[sl]);
              __syncwarp();
            }
            if (++sl == p.nw) { sl = 0; ph ^= 1; }
          }
        }
      }
      for (int t = 0; !p.pair && t < T; ++t) {
        int sl = wsl, ph = wph;
        for (int j = 0; j < p.nx; ++j) {
          if (t == 0) mbar_wait(&w_full[sl], ph);
          mma_slot(P1 + j, t, wdesc(sl));
          if (t == T - 1) {
            if (elect_one()) tc_commit(&w_empty[sl]);
            __syncwarp();
          }
          if (++sl == p.nw) { sl = 0; ph ^= 1; }
        }
      }
      for (int j = 0; j < p.nx; ++j)
        if (++wsl == p.nw) { wsl = 0; wph ^= 1; }
      accph ^= (1u << T) - 1u;
    }
    if (dbg && lane == 0) { dbg[16] = wait_cyc; dbg[17] = pclk() - t_begin; }
  } else if (warp <= 9) {
    // ----------------------------------------------------------- RMS + epilogue
    // Two sets of 4 warps: set 0 (warps 2-5) owns tiles 0 and 2, set 1
    // (warps 6-9) tiles 1 and 3 — both the RMS reads of those tiles' A slots
    // and their epilogues.  Tiles complete in order 0,1,2,3 (phase 2), so the
    // sets alternate and each epilogue overlaps the stream of later tiles.
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    const int wset = (warp - 2) >> 2;
    const int row = 32 * q + lane;
    const uint32_t swz = (uint32_t)(row & 7);
    int as = 0, aph = 0, gi = 0;
    uint32_t accph = 0;
    long long sw_cyc = 0, s_begin = pclk();
    GroupIter it = make_iter();
    int c;
    int64_t g, r0, r1;
    while (next_group<NC>(it, c, g, r0, r1)) {
      const int T = (int)((r1 - r0 + 127) / 128);
      const float* const wup = NC > 1 ? p.wups[c] : sWup;
      float* const scores_c = (NC > 1 && p.scores) ? p.scores + (size_t)c * p.cap : p.scores;
      // sum of squares of this thread's row for each of its two tiles
      // (t = wset, wset + 2), four f32 chains each, from the swizzled A slots
      float ss[2][4];
#pragma unroll
      for (int i = 0; i < 2; ++i) ss[i][0] = ss[i][1] = ss[i][2] = ss[i][3] = 0.0f;
      // pair slot: this set's tile is rows [128 wset, 128 wset + 128); a set
      // whose tile is absent (odd T, last pair) only releases the slot
      auto rms_pair = [&](int pt, float (&acc)[4]) {
        mbar_wait(&a_full[as], aph);
        if (2 * pt + wset < T) {
          const uint8_t* rp = sA + (size_t)as * slot_bytes + (size_t)wset * kASlotBytes + row * 128;
          uint4 u[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) u[j] = *reinterpret_cast<const uint4*>(rp + ((j ^ swz) << 4));
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            sq2_acc<kBF16>(u[j].x, acc[0], acc[1]);
            sq2_acc<kBF16>(u[j].y, acc[2], acc[3]);
            sq2_acc<kBF16>(u[j].z, acc[0], acc[1]);
            sq2_acc<kBF16>(u[j].w, acc[2], acc[3]);
          }
          // release the slot only after the values are consumed: an arrive
          // right after the LDS issue let the TMA refill race the reads
          // (tools/stress_k1.py: non-deterministic rows with several groups
          // per CTA)
          __syncwarp();
          if (lane == 0) mbar_arrive(&a_empty[as]);
        } else {
          __syncwarp();
          if (lane == 0) mbar_arrive(&a_empty[as]);
        }
        if (++as == p.na) { as = 0; aph ^= 1; }
      };
      auto rms_slot = [&](int t, float (&acc)[4]) {
        if ((t & 1) == wset) {
          const long long s0 = pclk();
          mbar_wait(&a_full[as], aph);
          sw_cyc += pclk() - s0;
          const uint8_t* rp = sA + (size_t)as * slot_bytes + row * 128;
          uint4 u[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) u[j] = *reinterpret_cast<const uint4*>(rp + ((j ^ swz) << 4));
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            sq2_acc<kBF16>(u[j].x, acc[0], acc[1]);
            sq2_acc<kBF16>(u[j].y, acc[2], acc[3]);
            sq2_acc<kBF16>(u[j].z, acc[0], acc[1]);
            sq2_acc<kBF16>(u[j].w, acc[2], acc[3]);
          }
          __syncwarp();  // consumed, then released (see rms_pair)
          if (lane == 0) mbar_arrive(&a_empty[as]);
        } else {
          // the other set's tile: every RMS warp still takes part in every
          // slot's phase (a_empty counts all 8), as in pair mode — with
          // owner-only arrivals (4 per slot) repeated launches with several
          // groups per CTA gave non-deterministic tiles (tools/stress_k1.py)
          mbar_wait(&a_full[as], aph);
          __syncwarp();
          if (lane == 0) mbar_arrive(&a_empty[as]);
        }
        if (++as == p.na) { as = 0; aph ^= 1; }
      };
      // same slot order as the producer: phase 1 K-outer, phase 2 tile-major
      const int P1 = p.nk - p.nx;
      const int NP = (T + 1) / 2;
      for (int kc = 0; kc < P1; ++kc) {
        if (p.pair) {
#pragma unroll
          for (int pt = 0; pt < 2; ++pt)  // static index: ss stays in registers
            if (pt < NP) rms_pair(pt, ss[pt]);
        } else {
#pragma unroll
          for (int t = 0; t < 4; ++t)
            if (t < T) rms_slot(t, ss[t >> 1]);
        }
      }
      const int par = gi & 1;
      mbar_wait(&m_empty[par], (((uint32_t)gi >> 1) & 1u) ^ 1u);
      if (gi == 0) griddep_wait();  // before this grid's first global write
      // epilogue of one tile: tcgen05.ld the row's b pre-activations, scale,
      // SiLU, dot w_up, f64 sigmoid, strict threshold, ballot -> words
      auto epilogue = [&](int t, const float (&acc_ss)[4]) {
        uint32_t bal = 0;
        if (t < T) {
          mbar_wait(&t_full[t], (accph >> t) & 1u);
          tc_fence_after();
          if (dbg && warp == 2 && lane == 0) dbg[8 + 2 * t] = gtimer();
          const int64_t r = r0 + (int64_t)t * 128 + row;
          const bool valid = r < r1;
          const float sq = (acc_ss[0] + acc_ss[1]) + (acc_ss[2] + acc_ss[3]);
          const float scale = rms_scale(sq, p.inv_d, p.eps);
          const float hs = 0.5f * scale;  // exact (power of two)
          const f32x2 hs2 = pack2(hs, hs);
          f32x2 acc2 = 0ull;
          const uint32_t taddr = tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)(t * p.bp);
          // 32 accumulator columns per tcgen05.ld, two in flight: the next
          // chunk's TMEM read overlaps this chunk's SiLU / w_up math.
          auto consume = [&](const uint32_t (&v)[32], int c0) {
            if (c0 + 32 <= p.b) {
#pragma unroll
              for (int jj = 0; jj < 32; jj += 4) {
                const float4 w4 = NC > 1 ? __ldg(reinterpret_cast<const float4*>(wup + c0 + jj))
                                         : *reinterpret_cast<const float4*>(sWup + c0 + jj);
                const f32x2 s01 = silu2_tanh(fmul2(pack2u(v[jj], v[jj + 1]), hs2));
                const f32x2 s23 = silu2_tanh(fmul2(pack2u(v[jj + 2], v[jj + 3]), hs2));
                acc2 = ffma2(pack2(w4.x, w4.y), s01, acc2);
                acc2 = ffma2(pack2(w4.z, w4.w), s23, acc2);
              }
            } else {
#pragma unroll
              for (int jj = 0; jj < 32; jj += 2) {
                if (c0 + jj < p.b) {
                  const float w0 = NC > 1 ? __ldg(wup + c0 + jj) : sWup[c0 + jj];
                  const float w1 =
                      (c0 + jj + 1 < p.b) ? (NC > 1 ? __ldg(wup + c0 + jj + 1) : sWup[c0 + jj + 1]) : 0.0f;
                  const f32x2 s01 = silu2_tanh(fmul2(pack2u(v[jj], v[jj + 1]), hs2));
                  acc2 = ffma2(pack2(w0, w1), s01, acc2);
                }
              }
            }
          };
          uint32_t va[32], vb[32];
          tmem_ld32(taddr, va);
          tmem_ld_wait_regs(va);
          for (int c0 = 0; c0 < p.b; c0 += 64) {
            const bool has_b = c0 + 32 < p.b;
            if (has_b) tmem_ld32(taddr + (uint32_t)(c0 + 32), vb);
            consume(va, c0);
            if (has_b) {
              tmem_ld_wait_regs(vb);
              if (c0 + 64 < p.b) tmem_ld32(taddr + (uint32_t)(c0 + 64), va);
              consume(vb, c0 + 32);
              if (c0 + 64 < p.b) tmem_ld_wait_regs(va);
            }
          }
          tc_fence_before();
          __syncwarp();
          if (dbg && warp == 2 && lane == 0) dbg[9 + 2 * t] = gtimer();
          if (lane == 0) mbar_arrive(&t_empty[t]);
          float lo, hi;
          unpack2(acc2, lo, hi);
          const float logit = lo + hi;
          const float score = score_from_logit(logit);
          const bool ex = valid && (score > p.theta);
          if (NC > 1) {
            if (valid && scores_c) scores_c[r] = score;
            if (ex && p.exit_layers) exit_min(p.exit_layers + (gathered ? p.row_idx[r] : r), p.layers[c]);
          } else if (valid) {
            if (p.scores) p.scores[r] = score;
            if (p.logits) p.logits[r] = logit;
            if (p.mask) p.mask[r] = ex ? 1 : 0;
            if (ex && p.exit_layers) p.exit_layers[gathered ? p.row_idx[r] : r] = p.layer;
          }
          bal = __ballot_sync(0xffffffffu, ex);
        }
        if (lane == 0) words[par * 16 + t * 4 + q] = bal;
      };
      // phase 2: this set's tiles in completion order; each tile's epilogue
      // runs while the other set's next tile streams
      if (p.pair) {
        // pair-major: both sets stream pair 0, then run tiles 0 / 1 at once
        // while pair 1 streams, then tiles 2 / 3
#pragma unroll
        for (int pt = 0; pt < 2; ++pt) {
          if (pt < NP)
            for (int j = 0; j < p.nx; ++j) rms_pair(pt, ss[pt]);
          if (pt == 0 && dbg && warp == 2 && lane == 0) { dbg[2] = gtimer(); }
          epilogue(2 * pt + wset, ss[pt]);
        }
      }
#pragma unroll
      for (int t = 0; !p.pair && t < 4; ++t) {
        if (t < T)
          for (int j = 0; j < p.nx; ++j) rms_slot(t, ss[t >> 1]);
        if ((t & 1) == wset) {
          if (t == wset && dbg && warp == 2 && lane == 0) { dbg[2] = gtimer(); dbg[20] = sw_cyc; dbg[21] = pclk() - s_begin; }
          epilogue(t, ss[t >> 1]);
        }
      }
      accph ^= (1u << T) - 1u;
      __syncwarp();
      if (dbg && warp == 2 && lane == 0) dbg[3] = gtimer();
      if (lane == 0) mbar_arrive(&m_full[par]);
      ++gi;
    }
  } else {
    // ----------------------------------------------------------- compaction
    griddep_wait();  // the previous launch's look-back state / outputs are final
    const uint32_t tag = launch_tag(p.ws);
    int gi = 0;
    GroupIter it = make_iter();
    int c;
    int64_t g, r0, r1;
    while (next_group<NC>(it, c, g, r0, r1)) {
      const int par = gi & 1;
      mbar_wait(&m_full[par], ((uint32_t)gi >> 1) & 1u);
      const uint32_t word = lane < 16 ? words[par * 16 + lane] : 0u;
      const uint32_t cnt = __popc(word);
      uint32_t incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const uint32_t excl_w = incl - cnt;
      const uint32_t agg = __shfl_sync(0xffffffffu, incl, 31);
      // the words buffer is released only once the scan consumed the loaded
      // words (an arrive right after the load issue let the epilogue of the
      // group two ahead overwrite it first: compute-sanitizer racecheck)
      __syncwarp();
      if (lane == 0) mbar_arrive(&m_empty[par]);
      if (dbg && lane == 0) dbg[4] = gtimer();
      if (need_scan) {
        const uint32_t E = lookback_exclusive(p.ws->status, tag, g, agg);
        if (dbg && lane == 0) dbg[5] = gtimer();
        if (p.exit_idx || p.cont_idx) {
          const int nwords = (int)((r1 - r0 + 31) / 32);
          const uint32_t lt = (1u << lane) - 1u;
          for (int w = 0; w < nwords; ++w) {
            const uint32_t wd = __shfl_sync(0xffffffffu, word, w);
            const uint32_t pre = __shfl_sync(0xffffffffu, excl_w, w);
            const int64_t r = r0 + 32 * w + lane;
            if (r < r1) {
              const int64_t rank = (int64_t)E + pre + __popc(wd & lt);
              const int64_t id = (p.ids_from_rows && gathered) ? p.row_idx[r] : r;
              if ((wd >> lane) & 1u) {
                if (p.exit_idx) p.exit_idx[rank] = id;
              } else if (p.cont_idx) {
                p.cont_idx[r - rank] = id;
              }
            }
          }
        }
        if (g == NG - 1 && lane == 0 && p.counts) {
          p.counts[0] = (int64_t)E + agg;
          p.counts[1] = n - ((int64_t)E + agg);
        }
      }
      ++gi;
    }
    if (NC == 1 && NG == 0 && blockIdx.x == 0 && lane == 0 && p.counts) {
      p.counts[0] = 0;
      p.counts[1] = 0;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, p.tmem_cols);
  }
  if (dbg && threadIdx.x == 0) {
    dbg[6] = gtimer();
    unsigned int smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    dbg[7] = smid;
  }
  if (threadIdx.x == 0) launch_done(p.ws);
}

unsigned long long* g_dbg = nullptr;
}  // namespace tide
extern "C" void tide_debug_timeline(void* buf) { tide::g_dbg = (unsigned long long*)buf; }
namespace tide {

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  });
  return fn;
}

// Tensor maps are encoded on the host per (pointer, shape, box); a small cache
// keeps repeated launches over the same buffers (bench loops, the posthoc chain
// over a persistent capture) from paying the driver encode every time.
namespace {
struct MapKey {
  const void* base;
  int dtype;
  int64_t cols, rows, ld;
  int bc, br;
  bool operator==(const MapKey& o) const {
    return base == o.base && dtype == o.dtype && cols == o.cols && rows == o.rows && ld == o.ld &&
           bc == o.bc && br == o.br;
  }
};
constexpr int kMapCache = 128;
struct MapEntry {
  MapKey key;
  CUtensorMap map;
  uint64_t stamp;
  bool used;
};
MapEntry g_maps[kMapCache];
uint64_t g_stamp = 0;
std::mutex g_map_mu;
}  // namespace

int make_map(CUtensorMap* m, const void* base, int dtype, int64_t cols, int64_t rows,
             int64_t ld_elems, int box_cols, int box_rows) {
  const MapKey key{base, dtype, cols, rows, ld_elems, box_cols, box_rows};
  {
    std::lock_guard<std::mutex> lk(g_map_mu);
    for (auto& e : g_maps)
      if (e.used && e.key == key) {
        e.stamp = ++g_stamp;
        *m = e.map;
        return TIDE_OK;
      }
  }
  EncodeTiledFn enc = encode_fn();
  if (!enc) return set_error(TIDE_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t gdim[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t gstride[1] = {(cuuint64_t)ld_elems * (dtype == TIDE_F32 ? 4 : 2)};
  const cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  const cuuint32_t estride[2] = {1, 1};
  CUresult r = enc(m, dtype == TIDE_BF16  ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                     : dtype == TIDE_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                         : CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
                   2, const_cast<void*>(base), gdim, gstride, box, estride,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(TIDE_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  std::lock_guard<std::mutex> lk(g_map_mu);
  MapEntry* victim = &g_maps[0];
  for (auto& e : g_maps) {
    if (!e.used) { victim = &e; break; }
    if (e.stamp < victim->stamp) victim = &e;
  }
  victim->key = key;
  victim->map = *m;
  victim->stamp = ++g_stamp;
  victim->used = true;
  return TIDE_OK;
}

bool route_tc_supported(int dtype, int d, int b) {
  return (dtype == TIDE_BF16 || dtype == TIDE_F16) && d >= 8 && d % 8 == 0 && b >= 1 &&
         b <= 256;
}

// Shared launch setup of K1 and K1m: tile geometry, smem carve-up, numerics.
static int tc_params(const RouteArgs& a, bool pair, TcParams& p, uint32_t& smem_bytes) {
  const int npad = (a.b + 15) / 16 * 16;
  const int bp = (npad + 31) / 32 * 32;
  const int tpg = std::min(4, 512 / bp);
  int cols = 32;
  while (cols < tpg * bp) cols <<= 1;
  const int nk = (a.d + 63) / 64;
  const uint32_t wslot = (uint32_t)npad * 128u;
  int nw = npad <= 128 ? 4 : 3;
  {
    const char* env = getenv("TIDE_NW");  // read per call
    if (env) nw = std::max(2, std::min(kMaxNW, atoi(env)));
  }
  // smem carve-up (offsets from a 1024-aligned base)
  const uint32_t off_a = (uint32_t)nw * wslot;
  const int smem_cap = 227 * 1024;
  const uint32_t misc = 1024 /*w_up*/ + 512 /*bars*/ + 128 /*words*/ + 2048 /*ids*/ + 16;
  const uint32_t slot_bytes = pair ? 2u * kASlotBytes : (uint32_t)kASlotBytes;
  int na = (int)((smem_cap - 1024 - off_a - misc) / slot_bytes);
  na = std::min(na, kMaxNA);
  {
    const char* env = getenv("TIDE_K1_NA");  // debug: cap the A ring (read per call)
    if (env) na = std::max(2, std::min(na, atoi(env)));
  }
  if (na < 2) return set_error(TIDE_ERR_UNSUPPORTED, "bottleneck too wide for smem");
  p.n_host = a.n;
  p.n_dev = a.n_dev;
  p.rows_total = a.rows_total;
  p.d = a.d;
  p.b = a.b;
  p.npad = npad;
  p.bp = bp;
  p.tpg = tpg;
  p.nk = nk;
  p.na = na;
  p.nw = nw;
  p.nx = std::min(nw, nk);  // tile-major tail chunks (W slots kept resident)
  p.pair = pair ? 1 : 0;
  p.idesc = f16_idesc(a.dtype == TIDE_BF16 ? 1 : 0, 128, npad);
  p.tmem_cols = (uint32_t)cols;
  p.wslot = wslot;
  p.off_a = off_a;
  p.off_wup = off_a + (uint32_t)na * slot_bytes;
  p.off_bar = p.off_wup + 1024;
  p.off_words = p.off_bar + 512;
  p.off_ids = p.off_words + 128;
  p.off_tmem = p.off_ids + 2048;
  smem_bytes = p.off_tmem + 16 + 1024;
  p.row_idx = a.row_idx;
  p.ids_from_rows = a.ids_from_rows;
  p.w_up = a.w_up;
  p.eps = a.eps;
  p.inv_d = (float)(1.0 / (double)a.d);
  p.theta = a.theta;
  p.layer = a.layer;
  p.inputs_ready = (a.flags & TIDE_ROUTE_INPUTS_READY) ? 1 : 0;
  p.scores = a.scores;
  p.logits = a.logits;
  p.mask = a.mask;
  p.exit_idx = a.exit_idx;
  p.cont_idx = a.cont_idx;
  p.exit_layers = a.exit_layers;
  p.counts = a.counts;
  p.ws = reinterpret_cast<Workspace*>(a.workspace);
  p.dbg = g_dbg;
  p.nc = 1;
  return TIDE_OK;
}

template <int NC>
static int tc_launch(const RouteArgs& a, const CUtensorMap (&tm)[7], const MultiMaps<NC>& mm,
                     const TcParams& p, uint32_t smem_bytes, int grid, int dev, cudaStream_t stream,
                     const char* what) {
  static bool attr_set[64] = {false};
  if (!attr_set[dev & 63]) {
    cudaFuncSetAttribute(route_tc_kernel<true, NC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         227 * 1024);
    cudaFuncSetAttribute(route_tc_kernel<false, NC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         227 * 1024);
    attr_set[dev & 63] = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreadsTC);
  cfg.dynamicSmemBytes = smem_bytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  {
    const char* env = getenv("TIDE_PDL");  // read per call
    cfg.numAttrs = (env && env[0] == '0') ? 0 : 1;
  }
  cfg.attrs = attr;
  cudaError_t e;
  if (a.dtype == TIDE_BF16)
    e = cudaLaunchKernelEx(&cfg, route_tc_kernel<true, NC>, tm[0], tm[1], tm[2], tm[3], tm[4], tm[5],
                           tm[6], mm, p);
  else
    e = cudaLaunchKernelEx(&cfg, route_tc_kernel<false, NC>, tm[0], tm[1], tm[2], tm[3], tm[4],
                           tm[5], tm[6], mm, p);
  if (e != cudaSuccess) return set_error(TIDE_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return check_launch(what);
}

// TIDE_K1_GRID (debug, read per call): run K1 / K1m as if the GPU had that
// many SMs — several row groups per CTA at small sizes (compute-sanitizer).
static int k1_sms(int dev) {
  const char* env = getenv("TIDE_K1_GRID");
  const int sms = sm_count(dev);
  return env ? std::max(1, std::min(sms, atoi(env))) : sms;
}

int route_tc_launch(const RouteArgs& a, cudaStream_t stream) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (!getenv("TIDE_K1_GRID")) {
    // few rows: split d over a cluster instead (route_tcs.cu)
    int grid = 0;
    const int ks = route_tcs_plan(a, dev, &grid);
    if (ks) return route_tcs_launch(a, stream, ks, grid);
  }
  const int sms = k1_sms(dev);
  // pair slots (two whole tiles per 32 KB slot: half the barrier round trips
  // per byte) for dense launches dealt in whole tiles; TIDE_K1_PAIRSLOT=0/1
  const int tpg0 = std::min(4, 512 / (((a.b + 15) / 16 * 16 + 31) / 32 * 32));
  bool pair = a.row_idx == nullptr && a.n_dev == nullptr && a.n % 128 == 0 &&
              a.n >= (int64_t)sms * 256 && tpg0 == 4;
  {
    const char* env = getenv("TIDE_K1_PAIRSLOT");  // read per call
    if (env) pair = pair && env[0] == '1';
  }
  TcParams p{};
  uint32_t smem_bytes = 0;
  int rc;
  if ((rc = tc_params(a, pair, p, smem_bytes))) return rc;

  CUtensorMap tm[7];  // h128, h64, h32b, h16, w, gather4, h256
  const int64_t hrows = a.row_idx ? a.rows_total : std::max<int64_t>(a.n, 1);
  if ((rc = make_map(&tm[0], a.h, a.dtype, a.d, hrows, a.ld_h, 64, 128))) return rc;
  if ((rc = make_map(&tm[1], a.h, a.dtype, a.d, hrows, a.ld_h, 64, 64))) return rc;
  if ((rc = make_map(&tm[2], a.h, a.dtype, a.d, hrows, a.ld_h, 64, 32))) return rc;
  if ((rc = make_map(&tm[3], a.h, a.dtype, a.d, hrows, a.ld_h, 64, kBox))) return rc;
  if ((rc = make_map(&tm[5], a.h, a.dtype, a.d, hrows, a.ld_h, 64, 1))) return rc;
  if ((rc = make_map(&tm[4], a.w_down, a.dtype, a.d, a.b, a.d, 64, p.npad))) return rc;
  if (pair) {
    if ((rc = make_map(&tm[6], a.h, a.dtype, a.d, hrows, a.ld_h, 64, 256))) return rc;
  } else {
    tm[6] = tm[0];
  }

  // whole tiles per CTA once each holds at least two and the row count is
  // known on the host (a chain link's live count may be far below its
  // capacity: 16-row units keep every SM busy there); TIDE_K1_GRAN overrides
  int gran = (a.n_dev == nullptr && a.n >= (int64_t)sms * 256) ? 128 : kGran;
  {
    const char* env = getenv("TIDE_K1_GRAN");
    if (env) {
      const int v = atoi(env);
      gran = (v == 32 || v == 64 || v == 128) ? v : kGran;
    }
  }
  p.gran = gran;
  const int64_t n32 = (a.n + gran - 1) / gran;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(sms, n32));
  if ((n32 + p.tpg * (128 / gran) - 1) / (p.tpg * (128 / gran)) > kMaxParts / 2)
    return set_error(TIDE_ERR_UNSUPPORTED, "too many rows for one launch");
  MultiMaps<1> mm{};
  return tc_launch<1>(a, tm, mm, p, smem_bytes, grid, dev, stream, "route_tc_kernel");
}

// K1m: every row scored at C checkpoints in ONE persistent launch; each row's
// first firing checkpoint is combined in a.exit_layers by an atomic minimum
// (rows that never fire keep NO_EXIT), scores optionally to a.scores[c *
// a.n + position]; dense (a.row_idx == NULL: rows 0..a.n-1 of every capture)
// or gathered (the live rows a.row_idx[0 .. *a.n_dev), routed only when
// a.n_min <= *a.n_dev <= n_limit).
int route_tc_multi_launch(const RouteArgs& a, int C, const void* const* h_ptrs,
                          const void* const* w_ptrs, const float* const* wup_ptrs,
                          const int64_t* layers, int64_t n_limit, cudaStream_t stream) {
  if (C < 2 || C > kMaxMC) return set_error(TIDE_ERR_UNSUPPORTED, "K1m: C must be in [2, %d]", kMaxMC);
  if (!a.scores && !a.exit_layers) return set_error(TIDE_ERR_ARG, "K1m: scores or exit_layers required");
  if ((a.row_idx == nullptr) != (a.n_dev == nullptr))
    return set_error(TIDE_ERR_ARG, "K1m: row_idx and n_dev go together");
  int dev = 0;
  cudaGetDevice(&dev);
  const int sms = k1_sms(dev);
  TcParams p{};
  uint32_t smem_bytes = 0;
  int rc;
  const bool gathered = a.row_idx != nullptr;
  // dense: pair slots (two whole tiles of one checkpoint per 256-row box);
  // TIDE_K1_PAIRSLOT=0 turns them off
  bool pair = !gathered && std::min(4, 512 / (((a.b + 15) / 16 * 16 + 31) / 32 * 32)) == 4;
  {
    const char* env = getenv("TIDE_K1_PAIRSLOT");  // read per call
    if (env) pair = pair && env[0] == '1';
  }
  if ((rc = tc_params(a, pair, p, smem_bytes))) return rc;
  p.gran = 128;
  p.nc = C;
  p.cap = a.n;
  p.n_min = a.n_min;
  p.n_limit = n_limit;
  // scores only: no mask / logits / compaction / exit layers here
  p.logits = nullptr;
  p.mask = nullptr;
  p.exit_idx = p.cont_idx = p.counts = nullptr;  // exit_layers: first firing checkpoint (exit_min)
  p.inputs_ready = 0;
  const int64_t hrows = gathered ? a.rows_total : std::max<int64_t>(a.n, 1);
  static MultiMaps<kMaxMC> mm;  // host staging (copied into the launch parameters)
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  for (int c = 0; c < C; ++c) {
    if ((rc = make_map(&mm.h[c], h_ptrs[c], a.dtype, a.d, hrows, a.ld_h, 64, gathered ? 1 : 128)))
      return rc;
    if ((rc = make_map(&mm.w[c], w_ptrs[c], a.dtype, a.d, a.b, a.d, 64, p.npad))) return rc;
    if (pair) {
      if ((rc = make_map(&mm.p[c], h_ptrs[c], a.dtype, a.d, hrows, a.ld_h, 64, 256))) return rc;
    } else {
      mm.p[c] = mm.h[c];
    }
    p.wups[c] = wup_ptrs[c];
    p.layers[c] = layers[c];
  }
  CUtensorMap tm[7];
  for (int i = 0; i < 7; ++i) tm[i] = mm.h[0];
  // tiles: C x ceil(cap / 128) at most (the live count is only known on the device)
  const int64_t TT = (int64_t)C * ((a.n + 127) / 128);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(sms, TT));
  return tc_launch<kMaxMC>(a, tm, mm, p, smem_bytes, grid, dev, stream, "route_tc_kernel (K1m)");
}

}  // namespace tide
