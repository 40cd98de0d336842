// K1 for f32 rows (the reference's own dtype): fused RMSNorm + router + exit
// mask + stable compaction on tcgen05 tensor cores with 3xTF32 products.
//
// Restates, for a block of rows at once (same contract as route_tc.cu):
//   ee/router_ops.py:68-87   fused_layernorm_route  (score per row)
//   ee/runtime.py:149,171    mask = score > f32(theta)       (strict)
//   ee/router_ops.py:116-134 _compact_prefix_sum    (stable partition indices)
//   ee/runtime.py:175-178    exited_at / exit_layers / remaining (row_idx mode)
//
// Why 3xTF32: the f32 contract is 1e-5 relative; one TF32
// pass (10-bit mantissa) misses it by three orders of magnitude.  Each f32
// operand is split x = hi + lo with hi = x with the low 13 mantissa bits
// cleared (exactly representable in tf32) and lo = x - hi (exact in f32, its
// tf32 rounding error <= 2^-21 |x|); then
//     x . w  ~=  hi_x . hi_w  +  lo_x . hi_w  +  hi_x . lo_w
// (the dropped lo . lo term is <= 2^-22 relative), all accumulated in f32 in
// TMEM.  Three MMAs (K = 8 each) per 32 bytes of K instead of one.
//
// The hi/lo split is done in shared memory, between the TMA landing and the
// MMA: the RMS warps (which read every element for the sum of squares anyway)
// write each A slot's lo into a lo ring; a W splitter warp does the same for
// each W k-chunk (the MMA reads the staged f32 value as hi).  The kernel's ABI is the
// plain f32 W_down of tide_route; nothing is pre-split on the host.
//
// CTA roles (384 threads, one persistent CTA per SM, groups of up to 4 token
// tiles of 128 rows; the pipeline shape follows route_tc.cu):
//   warp 0      TMA producer (32 f32 columns = 128 B per row per k-chunk;
//               64/32/16-row boxes for the ragged tail, tile::gather4 rows
//               when peeling by row_idx).
//   warp 1      TMEM allocator + MMA issuer: phase 1 K-outer over the first
//               nk - nx chunks (each W chunk feeds every tile), phase 2
//               tile-major over the last nx chunks (W slots resident).
//   warps 2-9   two sets of 4 (set 0: tiles 0, 2; set 1: tiles 1, 3): per A
//               slot, sum of squares + hi/lo split, then the tile epilogue
//               (tcgen05.ld, scale, f32 SiLU, dot w_up, f64 sigmoid, strict
//               threshold, ballots).
//   warp 10     compaction (ballot words -> look-back -> int64 indices).
//   warp 11     W splitter.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "internal.h"

namespace tide {

// 1: the hi half is written back over the staged operand, so the MMA sees an
// exact tf32 value whatever the tensor core does with the low 13 bits of an
// f32 operand; 0 (default): rely on the hardware ignoring them — measured on
// B200: both builds give bit-identical logits (tools/tf32_probe.py).
#ifndef TIDE_TF32_INPLACE
#define TIDE_TF32_INPLACE 0
#endif

constexpr int kThreadsTF = 384;
constexpr int kTfMaxNA = 8;
constexpr int kTfMaxNL = 8;
constexpr int kTfMaxNW = 4;
constexpr int kTfSlot = 128 * 128;  // 128 rows x 32 f32 columns
constexpr int kTfGran = 16;

struct TfParams {
  int64_t n_host;
  const int64_t* n_dev;
  int64_t rows_total;
  int32_t d, b, npad, bp, tpg, nk, na, nl, nw, nx;
  int32_t nacc;  // TMEM accumulators per tile: 1, 2 (hi.hi | small terms), 4 (each by k-chunk parity)
  uint32_t idesc, tmem_cols, wslot, whalf;
  uint32_t off_a, off_l, off_wup, off_bar, off_words, off_ids, off_tmem;
  const int64_t* row_idx;
  int32_t ids_from_rows;
  const float* w_up;
  float eps, inv_d, theta;
  int64_t layer;
  int32_t inputs_ready;  // TIDE_ROUTE_INPUTS_READY
  int32_t w_presplit;    // W's lo half staged in the workspace (tm_wlo): no splitter
  float* scores;
  float* logits;
  uint8_t* mask;
  int64_t* exit_idx;
  int64_t* cont_idx;
  int64_t* exit_layers;
  int64_t* counts;
  Workspace* ws;
};

__device__ __forceinline__ void tf_group_range(int64_t g, int64_t n, int64_t n16, int64_t ng,
                                               int64_t& r0, int64_t& r1) {
  r0 = (g * n16 / ng) * kTfGran;
  r1 = ((g + 1) * n16 / ng) * kTfGran;
  if (r1 > n) r1 = n;
}

// hi = x with the 13 low mantissa bits cleared (a tf32 value), lo = x - hi.
__device__ __forceinline__ void split4(const uint4& v, uint4& hi, uint4& lo) {
  constexpr uint32_t kMask = 0xFFFFE000u;
  hi = make_uint4(v.x & kMask, v.y & kMask, v.z & kMask, v.w & kMask);
  lo = make_uint4(__float_as_uint(__uint_as_float(v.x) - __uint_as_float(hi.x)),
                  __float_as_uint(__uint_as_float(v.y) - __uint_as_float(hi.y)),
                  __float_as_uint(__uint_as_float(v.z) - __uint_as_float(hi.z)),
                  __float_as_uint(__uint_as_float(v.w) - __uint_as_float(hi.w)));
}

// W's lo half (w - tf32(w), exactly split4's) into the workspace once per
// launch: the route kernel then TMA-loads both halves and its splitter warp
// (one warp re-splitting all of W for every row group: ~0.8 us per 32-column
// chunk, as long as the chunk's MMAs) stays idle.
__global__ void __launch_bounds__(256) tf32_split_w_kernel(const float* __restrict__ w,
                                                           float* __restrict__ lo, int64_t n4) {
  const uint4* src = reinterpret_cast<const uint4*>(w);
  uint4* dst = reinterpret_cast<uint4*>(lo);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint4 hi, l;
    split4(src[i], hi, l);
    dst[i] = l;
  }
}

__global__ void __launch_bounds__(kThreadsTF, 1)
    route_tf32_kernel(const __grid_constant__ CUtensorMap tm_h128,
                      const __grid_constant__ CUtensorMap tm_h64,
                      const __grid_constant__ CUtensorMap tm_h32b,
                      const __grid_constant__ CUtensorMap tm_h16,
                      const __grid_constant__ CUtensorMap tm_w,
                      const __grid_constant__ CUtensorMap tm_wlo,
                      const __grid_constant__ CUtensorMap tm_g4, const __grid_constant__ TfParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sW = smem;
  uint8_t* sA = smem + p.off_a;
  uint8_t* sL = smem + p.off_l;
  float* sWup = reinterpret_cast<float*>(smem + p.off_wup);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.off_bar);
  uint64_t* w_full = bars;
  uint64_t* w_ready = w_full + kTfMaxNW;
  uint64_t* w_empty = w_ready + kTfMaxNW;
  uint64_t* a_full = w_empty + kTfMaxNW;
  uint64_t* a_ready = a_full + kTfMaxNA;
  uint64_t* a_empty = a_ready + kTfMaxNA;
  uint64_t* t_full = a_empty + kTfMaxNA;
  uint64_t* t_empty = t_full + 4;
  uint64_t* m_full = t_empty + 4;
  uint64_t* m_empty = m_full + 2;
  uint32_t* words = reinterpret_cast<uint32_t*>(smem + p.off_words);
  uint32_t* ids = reinterpret_cast<uint32_t*>(smem + p.off_ids);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + p.off_tmem);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
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
  const int64_t n = p.n_dev ? *p.n_dev : p.n_host;
  const int64_t n16 = (n + kTfGran - 1) / kTfGran;
  const int64_t G = gridDim.x;
  const int64_t cpg = (int64_t)p.tpg * (128 / kTfGran);
  int64_t NG = n16 < G ? n16 : G;
  if ((n16 + cpg - 1) / cpg > NG) NG = (n16 + cpg - 1) / cpg;
  const bool gathered = p.row_idx != nullptr;
  const bool need_scan = p.exit_idx || p.cont_idx || p.counts;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tm_w);
    if (p.w_presplit) prefetch_tmap(&tm_wlo);
    prefetch_tmap(gathered ? &tm_g4 : &tm_h128);
    for (int i = 0; i < p.nw; ++i) {
      mbar_init(&w_full[i], 1);
      mbar_init(&w_ready[i], 1);  // the splitter warp
      mbar_init(&w_empty[i], 1);  // MMA commit
    }
    for (int i = 0; i < p.na; ++i) {
      mbar_init(&a_full[i], 1);
      mbar_init(&a_ready[i], 4);  // the 4 RMS warps owning the tile (split done)
      mbar_init(&a_empty[i], 1);  // MMA commit (also frees the lo slot it used)
    }
    for (int i = 0; i < 4; ++i) {
      mbar_init(&t_full[i], 1);
      mbar_init(&t_empty[i], 4);
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
  for (int i = threadIdx.x; i < p.b; i += blockDim.x) sWup[i] = p.w_up[i];
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int P1 = p.nk - p.nx;

  if (warp == 0) {
    // ----------------------------------------------------------- producer
    const uint64_t pol_h = policy_evict_first();
    const uint64_t pol_w = policy_evict_last();
    int as = 0, aph = 0, wsl = 0, wph = 0;
    for (int64_t g = blockIdx.x; g < NG; g += G) {
      int64_t r0, r1;
      tf_group_range(g, n, n16, NG, r0, r1);
      const int T = (int)((r1 - r0 + 127) / 128);
      if (gathered) {
        __syncwarp();
        for (int64_t i = r0 + lane; i < r0 + (int64_t)T * 128; i += 32)
          ids[i - r0] = i < r1 ? (uint32_t)p.row_idx[i] : (uint32_t)p.rows_total;
        __syncwarp();
      }
      if (lane == 0) {
        auto load_w = [&](int kc) {
          mbar_wait(&w_empty[wsl], wph ^ 1);
          mbar_arrive_expect_tx(&w_full[wsl], p.w_presplit ? 2 * p.whalf : p.whalf);
          tma_load_2d(sW + (size_t)wsl * p.wslot, &tm_w, &w_full[wsl], kc * 32, 0, pol_w);
          if (p.w_presplit)
            tma_load_2d(sW + (size_t)wsl * p.wslot + p.whalf, &tm_wlo, &w_full[wsl], kc * 32, 0, pol_w);
          if (++wsl == p.nw) { wsl = 0; wph ^= 1; }
        };
        auto load_a = [&](int kc, int t) {
          mbar_wait(&a_empty[as], aph ^ 1);
          uint8_t* dst = sA + (size_t)as * kTfSlot;
          const int64_t rb = r0 + (int64_t)t * 128;
          const int rows_in = (int)((r1 - rb) < 128 ? (r1 - rb) : 128);
          if (!gathered) {
            if (rows_in == 128) {
              mbar_arrive_expect_tx(&a_full[as], kTfSlot);
              tma_load_2d(dst, &tm_h128, &a_full[as], kc * 32, (int)rb, pol_h);
            } else {
              const int rr = (rows_in + kTfGran - 1) / kTfGran * kTfGran;
              mbar_arrive_expect_tx(&a_full[as], (uint32_t)(rr * 128));
              int off = 0;
              if (rr - off >= 64) {
                tma_load_2d(dst, &tm_h64, &a_full[as], kc * 32, (int)rb, pol_h);
                off += 64;
              }
              if (rr - off >= 32) {
                tma_load_2d(dst + off * 128, &tm_h32b, &a_full[as], kc * 32, (int)(rb + off), pol_h);
                off += 32;
              }
              if (rr - off >= 16) {
                tma_load_2d(dst + off * 128, &tm_h16, &a_full[as], kc * 32, (int)(rb + off), pol_h);
                off += 16;
              }
            }
          } else {
            const int ng4 = (rows_in + 3) / 4;
            mbar_arrive_expect_tx(&a_full[as], ng4 * 512);
            const uint32_t* id = ids + t * 128;
            for (int q = 0; q < ng4; ++q)
              tma_gather4(dst + q * 512, &tm_g4, &a_full[as], kc * 32, (int)id[4 * q],
                          (int)id[4 * q + 1], (int)id[4 * q + 2], (int)id[4 * q + 3], pol_h);
          }
          if (++as == p.na) { as = 0; aph ^= 1; }
        };
        for (int kc = 0; kc < P1; ++kc) {
          load_w(kc);
          for (int t = 0; t < T; ++t) load_a(kc, t);
        }
        for (int t = 0; t < T; ++t)
          for (int j = 0; j < p.nx; ++j) {
            if (t == 0) load_w(P1 + j);
            load_a(P1 + j, t);
          }
      }
    }
  } else if (warp == 1) {
    // ----------------------------------------------------------- MMA issuer
    int as = 0, aph = 0, wsl = 0, wph = 0, ls = 0;
    uint32_t accph = 0;
    const uint64_t desc_hi = sw128_kmajor_desc(0);
    const uint32_t wlo_step = p.whalf >> 4;  // descriptor offset of the W lo half
    for (int64_t g = blockIdx.x; g < NG; g += G) {
      int64_t r0, r1;
      tf_group_range(g, n, n16, NG, r0, r1);
      const int T = (int)((r1 - r0 + 127) / 128);
      for (int t = 0; t < T; ++t) mbar_wait(&t_empty[t], ((accph >> t) & 1u) ^ 1u);
      tc_fence_after();
      auto mma_slot = [&](int kc, int t, uint64_t bdesc) {
        mbar_wait(&a_ready[as], aph);
        tc_fence_after();
        if (elect_one()) {
          const uint64_t ax =
              desc_hi | (uint64_t)((smem_u32(sA + (size_t)as * kTfSlot) & 0x3FFFFu) >> 4);
          const uint64_t al =
              desc_hi | (uint64_t)((smem_u32(sL + (size_t)ls * kTfSlot) & 0x3FFFFu) >> 4);
          const uint64_t bl = bdesc + wlo_step;
          // accumulators of this tile: big (hi.hi) and small (lo.hi + hi.lo),
          // each split by k-chunk parity when nacc = 4 — every accumulator
          // sees a fraction of the MMA steps, and the tensor core's per-step
          // loss of low accumulator bits (a bias toward zero that grows with
          // the number of steps) shrinks in proportion
          const uint32_t tb = tmem_base + (uint32_t)(t * p.nacc * p.bp);
          const int par = p.nacc == 4 ? (kc & 1) : 0;
          const uint32_t d_big = tb + (uint32_t)(par * p.bp);
          const uint32_t d_small = p.nacc == 1 ? d_big : tb + (uint32_t)((p.nacc / 2 + par) * p.bp);
          const bool first = kc < (p.nacc == 4 ? 2 : 1);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            tc_mma_tf32(d_big, ax + 2 * k, bdesc + 2 * k, p.idesc, (first && k == 0) ? 0u : 1u);
            tc_mma_tf32(d_small, al + 2 * k, bdesc + 2 * k, p.idesc,
                        (p.nacc != 1 && first && k == 0) ? 0u : 1u);
            tc_mma_tf32(d_small, ax + 2 * k, bl + 2 * k, p.idesc, 1u);
          }
          tc_commit(&a_empty[as]);
          if (kc == p.nk - 1) tc_commit(&t_full[t]);
        }
        __syncwarp();
        if (++as == p.na) { as = 0; aph ^= 1; }
        if (++ls == p.nl) ls = 0;
      };
      auto wdesc = [&](int slot) {
        return desc_hi | (uint64_t)((smem_u32(sW + (size_t)slot * p.wslot) & 0x3FFFFu) >> 4);
      };
      for (int kc = 0; kc < P1; ++kc) {
        mbar_wait(p.w_presplit ? &w_full[wsl] : &w_ready[wsl], wph);
        const uint64_t bdesc = wdesc(wsl);
        for (int t = 0; t < T; ++t) mma_slot(kc, t, bdesc);
        if (elect_one()) tc_commit(&w_empty[wsl]);
        __syncwarp();
        if (++wsl == p.nw) { wsl = 0; wph ^= 1; }
      }
      for (int t = 0; t < T; ++t) {
        int sl = wsl, ph = wph;
        for (int j = 0; j < p.nx; ++j) {
          if (t == 0) mbar_wait(p.w_presplit ? &w_full[sl] : &w_ready[sl], ph);
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
  } else if (warp <= 9) {
    // ----------------------------------------------------------- RMS + split + epilogue
    const int q = warp & 3;
    const int wset = (warp - 2) >> 2;
    const int row = 32 * q + lane;
    // global slot counter: A slot = cnt % na, lo slot = cnt % nl; the lo slot
    // is free once the MMAs of slot cnt - nl retired, i.e. the a_empty phase
    // of A slot (cnt - nl) % na
    int64_t cnt = 0;
    int gi = 0;
    uint32_t accph = 0;
    for (int64_t g = blockIdx.x; g < NG; g += G) {
      int64_t r0, r1;
      tf_group_range(g, n, n16, NG, r0, r1);
      const int T = (int)((r1 - r0 + 127) / 128);
      float ss[2][4];
#pragma unroll
      for (int i = 0; i < 2; ++i) ss[i][0] = ss[i][1] = ss[i][2] = ss[i][3] = 0.0f;
      auto rms_slot = [&](int t, float (&acc)[4]) {
        if ((t & 1) == wset) {
          const int as = (int)(cnt % p.na);
          const int ls = (int)(cnt % p.nl);
          mbar_wait(&a_full[as], (uint32_t)((cnt / p.na) & 1));
          if (cnt >= p.nl) {
            const int64_t prev = cnt - p.nl;
            mbar_wait(&a_empty[prev % p.na], (uint32_t)((prev / p.na) & 1));
          }
          // elementwise work: visit the row's 16-byte chunks in swizzled
          // order so a warp's 32 rows spread over all banks (row stride 128 B)
          uint8_t* rp = sA + (size_t)as * kTfSlot + row * 128;
          uint8_t* lp = sL + (size_t)ls * kTfSlot + row * 128;
          const int swz = row & 7;
          uint4 u[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) u[j] = *reinterpret_cast<const uint4*>(rp + ((j ^ swz) << 4));
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float x0 = __uint_as_float(u[j].x), x1 = __uint_as_float(u[j].y);
            const float x2 = __uint_as_float(u[j].z), x3 = __uint_as_float(u[j].w);
            acc[0] = fmaf(x0, x0, acc[0]);
            acc[1] = fmaf(x1, x1, acc[1]);
            acc[2] = fmaf(x2, x2, acc[2]);
            acc[3] = fmaf(x3, x3, acc[3]);
            uint4 hi, lo;
            split4(u[j], hi, lo);
            if (TIDE_TF32_INPLACE) *reinterpret_cast<uint4*>(rp + ((j ^ swz) << 4)) = hi;
            *reinterpret_cast<uint4*>(lp + ((j ^ swz) << 4)) = lo;
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive(&a_ready[as]);
        }
        ++cnt;
      };
      for (int kc = 0; kc < P1; ++kc) {
#pragma unroll
        for (int t = 0; t < 4; ++t)
          if (t < T) rms_slot(t, ss[t >> 1]);
      }
      const int par = gi & 1;
      mbar_wait(&m_empty[par], (((uint32_t)gi >> 1) & 1u) ^ 1u);
      if (gi == 0) griddep_wait();
      auto epilogue = [&](int t, const float (&acc_ss)[4]) {
        uint32_t bal = 0;
        if (t < T) {
          mbar_wait(&t_full[t], (accph >> t) & 1u);
          tc_fence_after();
          const int64_t r = r0 + (int64_t)t * 128 + row;
          const bool valid = r < r1;
          const float sq = (acc_ss[0] + acc_ss[1]) + (acc_ss[2] + acc_ss[3]);
          const float scale = rms_scale(sq, p.inv_d, p.eps);
          float tl = 0.0f;
          const uint32_t taddr =
              tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)(t * p.nacc * p.bp);
          for (int c0 = 0; c0 < p.b; c0 += 32) {
            uint32_t v[32];
            tmem_ld32(taddr + (uint32_t)c0, v);
            tmem_ld_wait_regs(v);
            // the other accumulators of the tile: (big1) + small0 (+ small1)
            for (int ai = 1; ai < p.nacc; ++ai) {
              uint32_t w[32];
              tmem_ld32(taddr + (uint32_t)(ai * p.bp + c0), w);
              tmem_ld_wait_regs(w);
#pragma unroll
              for (int jj = 0; jj < 32; ++jj)
                v[jj] = __float_as_uint(__uint_as_float(v[jj]) + __uint_as_float(w[jj]));
            }
#pragma unroll
            for (int jj = 0; jj < 32; ++jj)
              if (c0 + jj < p.b)
                tl = fmaf(sWup[c0 + jj], silu_f32(__fmul_rn(__uint_as_float(v[jj]), scale)), tl);
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&t_empty[t]);
          const float score = score_from_logit(tl);
          const bool ex = valid && (score > p.theta);
          if (valid) {
            if (p.scores) p.scores[r] = score;
            if (p.logits) p.logits[r] = tl;
            if (p.mask) p.mask[r] = ex ? 1 : 0;
            if (ex && p.exit_layers) p.exit_layers[gathered ? p.row_idx[r] : r] = p.layer;
          }
          bal = __ballot_sync(0xffffffffu, ex);
        }
        if (lane == 0) words[par * 16 + t * 4 + q] = bal;
      };
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        if (t < T)
          for (int j = 0; j < p.nx; ++j) rms_slot(t, ss[t >> 1]);
        if ((t & 1) == wset) epilogue(t, ss[t >> 1]);
      }
      accph ^= (1u << T) - 1u;
      __syncwarp();
      if (lane == 0) mbar_arrive(&m_full[par]);
      ++gi;
    }
  } else if (warp == 10) {
    // ----------------------------------------------------------- compaction
    griddep_wait();
    const uint32_t tag = launch_tag(p.ws);
    int gi = 0;
    for (int64_t g = blockIdx.x; g < NG; g += G) {
      int64_t r0, r1;
      tf_group_range(g, n, n16, NG, r0, r1);
      const int par = gi & 1;
      mbar_wait(&m_full[par], ((uint32_t)gi >> 1) & 1u);
      const uint32_t word = lane < 16 ? words[par * 16 + lane] : 0u;
      const uint32_t c = __popc(word);
      uint32_t incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const uint32_t excl_w = incl - c;
      const uint32_t agg = __shfl_sync(0xffffffffu, incl, 31);
      // the words buffer is released only once the scan consumed the loaded
      // words (an arrive right after the load issue let the epilogue of the
      // group two ahead overwrite it first: compute-sanitizer racecheck)
      __syncwarp();
      if (lane == 0) mbar_arrive(&m_empty[par]);
      if (need_scan) {
        const uint32_t E = lookback_exclusive(p.ws->status, tag, g, agg);
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
    if (NG == 0 && blockIdx.x == 0 && lane == 0 && p.counts) {
      p.counts[0] = 0;
      p.counts[1] = 0;
    }
  } else {
    // ----------------------------------------------------------- W splitter
    // (idle when W's lo half was staged by tf32_split_w_kernel)
    int wsl = 0, wph = 0;
    for (int64_t g = blockIdx.x; !p.w_presplit && g < NG; g += G) {
      for (int kc = 0; kc < p.nk; ++kc) {
        mbar_wait(&w_full[wsl], wph);
        uint8_t* hp = sW + (size_t)wsl * p.wslot;
        for (int r = lane; r < p.npad; r += 32) {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            uint8_t* e = hp + r * 128 + ((j ^ (r & 7)) << 4);
            uint4 hi, lo;
            split4(*reinterpret_cast<const uint4*>(e), hi, lo);
            if (TIDE_TF32_INPLACE) *reinterpret_cast<uint4*>(e) = hi;
            *reinterpret_cast<uint4*>(e + p.whalf) = lo;
          }
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&w_ready[wsl]);
        if (++wsl == p.nw) { wsl = 0; wph ^= 1; }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, p.tmem_cols);
  }
  if (threadIdx.x == 0) launch_done(p.ws);
}

// Accumulators per tile.  The tensor core's f32 accumulation drops low bits on
// every MMA step, a bias toward zero that grows with the number of steps: with
// every term in one accumulator, max |dt|/max(|t|,m) was 4e-6 at d = 768 but
// 2.2e-5 at d = 4096, outside the 1e-5 f32 contract.  Four accumulators
// (hi.hi and the small terms apart, each split by k-chunk parity) give every
// accumulator 1/2 of the steps and keep the big sum free of the 2/3 of MMAs
// that carry small terms.  TIDE_TF32_ACC = 1 / 2 / 4 overrides (read per call).
// Measured max |dt|/max(|t|,m) on B200 (tools/tf32_probe.py, rows N(0,9)):
//   d      768     4096    8192    16384
//   acc 1  4.0e-6  2.2e-5  4.3e-5  8.9e-5
//   acc 2  1.4e-6  7.1e-6  1.4e-5  2.9e-5
//   acc 4  8.5e-7  3.5e-6  7.2e-6  1.4e-5
// so 2 accumulators (2 tiles per group) up to d = 4096 and 4 (1 tile per
// group: W re-read per tile) up to d = 8192 stay inside the 1e-5 contract.
// Accumulators per tile.  The logit error grows with d and, relative to the
// conditioning magnitude m, as the bottleneck narrows (fewer units average the
// accumulation errors out): tools/tf32_probe.py, 16,384 rows N(0, 9), max
// |dt| / max(|t|, m) with 2 / 4 accumulators —
//   b = 128: d 4096 8.0e-6 / 4.3e-6, d 8192 1.4e-5 / 6.8e-6
//   b =  96: d 4096 7.5e-6 / 3.9e-6, d 8192 1.8e-5 / 8.9e-6
//   b =  64: d 4096 9.9e-6 / 5.6e-6, d 8192 2.0e-5 / 9.8e-6
//   b =  32: d 2048 8.0e-6 / 4.3e-6, d 4096 1.6e-5 / 8.2e-6, d 8192 - / 1.6e-5
//   b =  16: d 4096 3.1e-5 / 1.6e-5
// so 2 only for b >= 128 and d <= 4096 (4 costs TMEM tiles per group there),
// else 4; tf32_max_d below keeps the default path inside 1e-5 with margin.
int tf32_nacc(int d, int nk, int b) {
  const char* env = getenv("TIDE_TF32_ACC");
  int v = env ? atoi(env) : (d <= 4096 && b >= 128 ? 2 : 4);
  if (v != 1 && v != 2 && v != 4) v = 4;
  if (v == 4 && nk < 2) v = 2;
  return v;
}

// f32 rows on tcgen05 (TIDE_F32_TC=0 forces the CUDA-core kernel, =1 this one
// at any shape): the default for d <= tf32_max_d(b) and n >= tf32_min_rows(d).  Below
// that row count every CTA re-reads and re-splits all of W for a few rows
// (W-bound: 0.24 ms at 4,096 x 4096, as the CUDA-core kernel); at 65,536 x 4096
// 0.57 ms against 1.82 ms on CUDA cores.
// Fewest rows the default path takes: below, every CTA still walks all of W
// for a handful of rows (~155 us at d = 4096 whatever n <= 8,192, W-chunk
// latency bound), and the CUDA-core kernel is as fast (tools/remote/tf32_pol.sh:
// d = 4096, n = 2,048: 148 vs 157 us; n = 4,096: 238 vs 158 us; d = 1024,
// n = 4,096: 67 vs 67 us, n = 16,384: 149 vs 67 us).
int64_t tf32_min_rows(int d) { return d >= 2048 ? 4096 : 8192; }
// widest d the default path takes for a bottleneck b (measured errors above:
// <= 9e-6 of the 1e-5 contract with the accumulators tf32_nacc picks)
int tf32_max_d(int b) { return b >= 112 ? 8192 : b >= 48 ? 4096 : b >= 24 ? 2048 : 1024; }
bool route_tf32_supported(int d, int b, int64_t n) {
  const char* env = getenv("TIDE_F32_TC");  // read per call: tests switch it
  if (env && env[0] == '0') return false;
  const bool forced = env && env[0] == '1';
  return d >= 4 && d % 4 == 0 && b >= 1 && b <= 128 &&
         (forced || (d <= tf32_max_d(b) && n >= tf32_min_rows(d)));
}

int route_tf32_launch(const RouteArgs& a, cudaStream_t stream) {
  const int npad = (a.b + 15) / 16 * 16;
  const int bp = (npad + 31) / 32 * 32;
  const int nk = (a.d + 31) / 32;
  const int nacc = tf32_nacc(a.d, nk, a.b);
  const int tpg = std::max(1, std::min(4, 512 / (bp * nacc)));
  if (tpg * bp * nacc > 512) return set_error(TIDE_ERR_UNSUPPORTED, "tf32: TMEM too small");
  int cols = 32;
  while (cols < tpg * bp * nacc) cols <<= 1;
  const uint32_t whalf = (uint32_t)npad * 128u;
  const uint32_t wslot = 2 * whalf;
  // Ring shape: W slots (hi + lo each), A slots, lo slots.  With W's lo half
  // pre-split (below) a W slot needs no splitter pass, and what the MMAs wait
  // on is the lo ring: the RMS warps split A chunk c into a lo slot only once
  // the MMAs that used that slot finished.  So: A slots = max(4, 2 tiles per
  // group) (a ring with 3 A slots for 2 tiles per group was seen to stall for
  // good), 3 W slots when that leaves >= 2 lo slots, the rest to lo (<= 4, <=
  // A slots).  65,536 x 4096 f32 (tools/tf32_ring.py, bit-identical): rings
  // (W, A, lo) = (2, 6, 3) 0.567 ms with the in-kernel split; presplit (4, 4,
  // 1) 0.509, (2, 6, 3) 0.471, (3, 5, 2) 0.428, (3, 4, 3) 0.419 ms.
  // TIDE_TF32_RING="nw,na,nl" (read per call) overrides for sweeps (na, nl 0:
  // the rule for that nw).
  const int smem_cap = 227 * 1024;
  const uint32_t misc = 1024 /*w_up*/ + 512 /*bars*/ + 128 /*words*/ + 2048 /*ids*/ + 16;
  auto slots_for = [&](int w) { return (smem_cap - 1024 - w * (int)wslot - (int)misc) / kTfSlot; };
  int na = std::min(kTfMaxNA, std::max(4, 2 * tpg));
  auto nl_for = [&](int w) { return std::min(std::min(4, na), slots_for(w) - na); };
  int nw = nl_for(3) >= 2 ? 3 : 2, na_req = 0, nl_req = 0;
  if (const char* renv = getenv("TIDE_TF32_RING")) {
    int x = 0, y = 0, z = 0;
    if (sscanf(renv, "%d,%d,%d", &x, &y, &z) == 3 && x >= 1 && x <= kTfMaxNW) nw = x, na_req = y, nl_req = z;
  }
  const uint32_t off_a = (uint32_t)nw * wslot;
  const int slots = slots_for(nw);
  int nl = nl_for(nw);
  if (na_req > 0 && nl_req > 0 && na_req <= kTfMaxNA && nl_req <= kTfMaxNL && na_req + nl_req <= slots)
    na = na_req, nl = nl_req;
  if (na < 2 || nl < 1) return set_error(TIDE_ERR_UNSUPPORTED, "bottleneck too wide for smem");
  TfParams p{};
  p.n_host = a.n;
  p.n_dev = a.n_dev;
  p.rows_total = a.rows_total;
  p.d = a.d;
  p.b = a.b;
  p.npad = npad;
  p.bp = bp;
  p.tpg = tpg;
  p.nacc = nacc;
  p.nk = nk;
  p.na = na;
  p.nl = nl;
  p.nw = nw;
  p.nx = std::min(nw, nk);
  p.idesc = tf32_idesc(128, npad);
  p.tmem_cols = (uint32_t)cols;
  p.wslot = wslot;
  p.whalf = whalf;
  p.off_a = off_a;
  p.off_l = off_a + (uint32_t)na * kTfSlot;
  p.off_wup = p.off_l + (uint32_t)nl * kTfSlot;
  p.off_bar = p.off_wup + 1024;
  p.off_words = p.off_bar + 512;
  p.off_ids = p.off_words + 128;
  p.off_tmem = p.off_ids + 2048;
  const uint32_t smem_bytes = p.off_tmem + 16 + 1024;
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

  CUtensorMap tm_h128, tm_h64, tm_h32b, tm_h16, tm_w, tm_g4;
  const int64_t hrows = a.row_idx ? a.rows_total : std::max<int64_t>(a.n, 1);
  int rc;
  if ((rc = make_map(&tm_h128, a.h, TIDE_F32, a.d, hrows, a.ld_h, 32, 128))) return rc;
  if ((rc = make_map(&tm_h64, a.h, TIDE_F32, a.d, hrows, a.ld_h, 32, 64))) return rc;
  if ((rc = make_map(&tm_h32b, a.h, TIDE_F32, a.d, hrows, a.ld_h, 32, 32))) return rc;
  if ((rc = make_map(&tm_h16, a.h, TIDE_F32, a.d, hrows, a.ld_h, 32, kTfGran))) return rc;
  if ((rc = make_map(&tm_g4, a.h, TIDE_F32, a.d, hrows, a.ld_h, 32, 1))) return rc;
  if ((rc = make_map(&tm_w, a.w_down, TIDE_F32, a.d, a.b, a.d, 32, npad))) return rc;
  // W's lo half staged in the workspace's upper half (TIDE_TF32_PRESPLIT=0,
  // read per call, keeps the in-kernel splitter for A/B runs)
  CUtensorMap tm_wlo = tm_w;
  float* wlo = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(a.workspace) + kWorkspaceScratchOffset);
  const char* penv = getenv("TIDE_TF32_PRESPLIT");
  p.w_presplit = 0;
  if (!(penv && penv[0] == '0') && (size_t)a.b * a.d * 4 <= kWorkspaceScratchBytes &&
      (reinterpret_cast<uintptr_t>(a.w_down) & 15) == 0 &&
      make_map(&tm_wlo, wlo, TIDE_F32, a.d, a.b, a.d, 32, npad) == TIDE_OK) {
    const int64_t n4 = (int64_t)a.b * a.d / 4;
    int blocks = (int)std::min<int64_t>((n4 + 255) / 256, 4 * 148);
    // an ordinary launch: it waits for the kernel in flight, which may read
    // the previous launch's lo half
    tf32_split_w_kernel<<<blocks, 256, 0, stream>>>(static_cast<const float*>(a.w_down), wlo, n4);
    if ((rc = check_launch("tf32_split_w_kernel"))) return rc;
    p.w_presplit = 1;
    p.inputs_ready = 0;  // the route kernel reads what the split kernel just wrote
  }
  cudaGetLastError();

  int dev = 0;
  cudaGetDevice(&dev);
  const int sms = sm_count(dev);
  const int64_t n16 = (a.n + kTfGran - 1) / kTfGran;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(sms, n16));
  if ((n16 + tpg * (128 / kTfGran) - 1) / (tpg * (128 / kTfGran)) > kMaxParts / 2)
    return set_error(TIDE_ERR_UNSUPPORTED, "too many rows for one launch");
  static bool attr_set[64] = {false};
  if (!attr_set[dev & 63]) {
    cudaFuncSetAttribute(route_tf32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         227 * 1024);
    attr_set[dev & 63] = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreadsTF);
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
  cudaLaunchKernelEx(&cfg, route_tf32_kernel, tm_h128, tm_h64, tm_h32b, tm_h16, tm_w, tm_wlo, tm_g4, p);
  return check_launch("route_tf32_kernel");
}

}  // namespace tide
