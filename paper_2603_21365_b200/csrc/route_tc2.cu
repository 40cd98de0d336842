// K1 on CTA pairs: the fused RMSNorm + router + exit mask + stable compaction
// with tcgen05.mma.cta_group::2 (M = 256 tokens per instruction).
//
// Same semantics as route_tc.cu (ee/router_ops.py:68-87, ee/runtime.py:171,
// ee/router_ops.py:116-134, ee/runtime.py:175-178); what changes is the
// mapping onto the hardware:
//   * a cluster of 2 CTAs on one TPC shares each MMA: CTA r holds its own 128
//     token rows of the A tile and half (N/2 rows) of the W_down k-chunk; the
//     leader (rank 0) issues one M=256 instruction for both.  Per token this
//     halves MMA instructions, W smem / L2 traffic and the tensor core's
//     shared-memory operand reads (A 4 KB + B 2 KB per K=16 step per SM);
//   * both CTAs' TMA loads complete on the leader's full barriers (count 2,
//     each producer arrives with its own byte count); the leader forwards
//     "slot ready" to the peer (its RMS warps read their own smem), and its
//     commits multicast to both CTAs' empty / accumulator-full barriers;
//   * each CTA owns a contiguous half of the pair's row range, so every CTA is
//     still one contiguous partition of the stable compaction (partition id
//     2 * pair_group + rank).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "internal.h"

namespace tide {

namespace {

constexpr int kThreads2 = 352;  // producer, MMA, 2 x 4 epilogue, compaction
constexpr int kMaxNA2 = 16;  // A ring depth cap
constexpr int kMaxNW2 = 8;
constexpr int kASlot2 = 128 * 128;
constexpr int kGran2 = 16;

#ifndef TIDE_K1_PROFILE
#define TIDE_K1_PROFILE 0
#endif
__device__ __forceinline__ long long pclk2() {
#if TIDE_K1_PROFILE
  return clock64();
#else
  return 0;
#endif
}
__device__ __forceinline__ unsigned long long gtimer2() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t map_to(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
__device__ __forceinline__ void arrive_remote(uint32_t caddr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(caddr) : "memory");
}
__device__ __forceinline__ void tmem_alloc2(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void tmem_relinquish2() {
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc2(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void mma2_f16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                        uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// commit -> arrive on the barrier at this smem offset in both CTAs of the pair
__device__ __forceinline__ void commit2_both(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], m;\n\t}\n" ::"r"(smem_u32(bar))
      : "memory");
}

struct Tc2Params {
  int64_t n_host;
  const int64_t* n_dev;
  int64_t rows_total;
  int32_t d, b, npad, bp, tpg, nk, na, nw;
  uint32_t idesc, tmem_cols, wslot;
  uint32_t off_a, off_wup, off_bar, off_words, off_ids, off_tmem;
  const int64_t* row_idx;
  int32_t ids_from_rows;
  const float* w_up;
  float eps, inv_d, theta;
  int64_t layer;
  float* scores;
  float* logits;
  uint8_t* mask;
  int64_t* exit_idx;
  int64_t* cont_idx;
  int64_t* exit_layers;
  int64_t* counts;
  Workspace* ws;
  unsigned long long* dbg;
};

// Pair-group g of NGp covers units [g*U/NGp, (g+1)*U/NGp) (kGran2 rows each);
// rank 0 takes the first ceil(half), rank 1 the rest.
__device__ __forceinline__ void half_range(int64_t g, int64_t n, int64_t U, int64_t ngp, int rank,
                                           int64_t& r0, int64_t& r1, int64_t& o0, int64_t& o1) {
  const int64_t u0 = g * U / ngp, u1 = (g + 1) * U / ngp;
  const int64_t um = u0 + (u1 - u0 + 1) / 2;
  const int64_t a0 = u0 * kGran2, am = std::min<int64_t>(um * kGran2, n),
                a1 = std::min<int64_t>(u1 * kGran2, n);
  if (rank == 0) { r0 = a0; r1 = am; o0 = am; o1 = a1; }
  else { r0 = am; r1 = a1; o0 = a0; o1 = am; }
}

}  // namespace

template <bool kBF16>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads2, 1)
    route_tc2_kernel(const __grid_constant__ CUtensorMap tm_h128,
                     const __grid_constant__ CUtensorMap tm_h64,
                     const __grid_constant__ CUtensorMap tm_h32,
                     const __grid_constant__ CUtensorMap tm_h16,
                     const __grid_constant__ CUtensorMap tm_w,
                     const __grid_constant__ CUtensorMap tm_g4, const __grid_constant__ Tc2Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sW = smem;
  uint8_t* sA = smem + p.off_a;
  float* sWup = reinterpret_cast<float*>(smem + p.off_wup);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.off_bar);
  uint64_t* w_land = bars;                     // this CTA's W half landed (TMA tx)
  uint64_t* w_peer = w_land + kMaxNW2;         // leader: the peer's W half landed (forwarded)
  uint64_t* w_empty = w_peer + kMaxNW2;        // both: W slot free (commit multicast)
  uint64_t* a_land = w_empty + kMaxNW2;        // this CTA's A tile landed (TMA tx)
  uint64_t* a_peer = a_land + kMaxNA2;         // leader: the peer's A tile landed (forwarded)
  uint64_t* a_empty = a_peer + kMaxNA2;        // both: slot consumed (MMA commit + RMS)
  uint64_t* t_full = a_empty + kMaxNA2;        // both: accumulator complete
  uint64_t* t_empty = t_full + 4;              // leader: both CTAs drained the accumulator
  uint64_t* m_full = t_empty + 4;
  uint64_t* m_empty = m_full + 2;
  uint32_t* words = reinterpret_cast<uint32_t*>(smem + p.off_words);
  uint32_t* ids = reinterpret_cast<uint32_t*>(smem + p.off_ids);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + p.off_tmem);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int rank = (int)cta_rank();
  const bool leader = rank == 0;
  const int64_t n = p.n_dev ? *p.n_dev : p.n_host;
  const int64_t U = (n + kGran2 - 1) / kGran2;
  const int64_t P = gridDim.x / 2;
  const int64_t pid = blockIdx.x / 2;
  const int64_t cpg = (int64_t)p.tpg * (128 / kGran2);  // units per CTA-group
  int64_t NGp = std::min<int64_t>(P, (U + 1) / 2);
  NGp = std::max<int64_t>(NGp, (U + 2 * cpg - 1) / (2 * cpg));
  const uint32_t tag = launch_tag(p.ws);
  const bool gathered = p.row_idx != nullptr;
  const bool need_scan = p.exit_idx || p.cont_idx || p.counts;
  const uint32_t half_w = (uint32_t)(p.npad / 2) * 128u;  // bytes of this CTA's W half

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tm_w);
    prefetch_tmap(gathered ? &tm_g4 : &tm_h128);
    if (!gathered) {
      prefetch_tmap(&tm_h64);
      prefetch_tmap(&tm_h32);
      prefetch_tmap(&tm_h16);
    }
    for (int i = 0; i < p.nw; ++i) {
      mbar_init(&w_land[i], 1);
      mbar_init(&w_peer[i], 1);
      mbar_init(&w_empty[i], 1);
    }
    for (int i = 0; i < p.na; ++i) {
      mbar_init(&a_land[i], 1);
      mbar_init(&a_peer[i], 1);
      mbar_init(&a_empty[i], 1 + 4);
    }
    for (int i = 0; i < 4; ++i) {
      mbar_init(&t_full[i], 1);
      mbar_init(&t_empty[i], 8);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&m_full[i], 8);
      mbar_init(&m_empty[i], 1);
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    tmem_alloc2(tmem_slot, p.tmem_cols);
    tmem_relinquish2();
  }
  for (int i = threadIdx.x; i < p.b; i += blockDim.x) sWup[i] = p.w_up[i];
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // peer barriers initialised before any remote arrive
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  unsigned long long* dbg = p.dbg ? p.dbg + 24 * blockIdx.x : nullptr;
  if (dbg && threadIdx.x == 0) dbg[0] = gtimer2();

  if (warp == 0) {
    // ----------------------------------------------------------- producer (both CTAs)
    long long pw_cyc = 0, p_begin = pclk2();
    const uint64_t pol_h = policy_evict_first();
    const uint64_t pol_w = policy_evict_last();
    int as = 0, aph = 0, wsl = 0, wph = 0;
    for (int64_t g = pid; g < NGp; g += P) {
      int64_t r0, r1, o0, o1;
      half_range(g, n, U, NGp, rank, r0, r1, o0, o1);
      const int T = (int)std::max<int64_t>((r1 - r0 + 127) / 128, (o1 - o0 + 127) / 128);
      if (gathered) {
        __syncwarp();
        for (int64_t i = r0 + lane; i < r0 + (int64_t)T * 128; i += 32)
          ids[i - r0] = i < r1 ? (uint32_t)p.row_idx[i] : (uint32_t)p.rows_total;
        __syncwarp();
      }
      if (lane == 0) {
        for (int kc = 0; kc < p.nk; ++kc) {
          mbar_wait(&w_empty[wsl], wph ^ 1);
          mbar_arrive_expect_tx(&w_land[wsl], half_w);
          tma_load_2d(sW + (size_t)wsl * p.wslot, &tm_w, &w_land[wsl], kc * 64,
                      rank * (p.npad / 2), pol_w);
          if (++wsl == p.nw) { wsl = 0; wph ^= 1; }
          for (int t = 0; t < T; ++t) {
            const long long q0 = pclk2();
            mbar_wait(&a_empty[as], aph ^ 1);
            pw_cyc += pclk2() - q0;
            uint8_t* dst = sA + (size_t)as * kASlot2;
            uint64_t* abar = &a_land[as];
            auto expect = [&](uint32_t bytes) { mbar_arrive_expect_tx(abar, bytes); };
            const int64_t rb = r0 + (int64_t)t * 128;
            const int rows_in = (int)std::max<int64_t>(0, std::min<int64_t>(128, r1 - rb));
            if (!gathered) {
              if (rows_in == 128) {
                expect(kASlot2);
                tma_load_2d(dst, &tm_h128, abar, kc * 64, (int)rb, pol_h);
              } else {
                // ragged tail: greedy 64/32/16-row boxes (small boxes stream poorly)
                const int rr = (rows_in + kGran2 - 1) / kGran2 * kGran2;
                expect((uint32_t)(rr * 128));
                int off = 0;
                if (rr - off >= 64) { tma_load_2d(dst, &tm_h64, abar, kc * 64, (int)rb, pol_h); off += 64; }
                if (rr - off >= 32) {
                  tma_load_2d(dst + off * 128, &tm_h32, abar, kc * 64, (int)(rb + off), pol_h);
                  off += 32;
                }
                if (rr - off >= 16) {
                  tma_load_2d(dst + off * 128, &tm_h16, abar, kc * 64, (int)(rb + off), pol_h);
                  off += 16;
                }
              }
            } else {
              const int ng4 = (rows_in + 3) / 4;
              expect((uint32_t)(ng4 * 512));
              const uint32_t* id = ids + t * 128;
              for (int q = 0; q < ng4; ++q)
                tma_gather4(dst + q * 512, &tm_g4, abar, kc * 64, (int)id[4 * q],
                            (int)id[4 * q + 1], (int)id[4 * q + 2], (int)id[4 * q + 3], pol_h);
            }
            if (++as == p.na) { as = 0; aph ^= 1; }
          }
        }
      }
    }
    if (dbg && lane == 0) { dbg[1] = gtimer2(); dbg[18] = pw_cyc; dbg[19] = pclk2() - p_begin; }
  } else if (warp == 1) {
    // ----------------------------------------------------------- MMA issuer (leader only)
    if (leader) {
      long long wait_cyc = 0, t_begin = pclk2();
      int as = 0, aph = 0, wsl = 0, wph = 0;
      uint32_t accph = 0;
      const uint64_t desc_hi = sw128_kmajor_desc(0);
      for (int64_t g = pid; g < NGp; g += P) {
        int64_t r0, r1, o0, o1;
        half_range(g, n, U, NGp, rank, r0, r1, o0, o1);
        const int T = (int)std::max<int64_t>((r1 - r0 + 127) / 128, (o1 - o0 + 127) / 128);
        for (int t = 0; t < T; ++t) mbar_wait(&t_empty[t], ((accph >> t) & 1u) ^ 1u);
        tc_fence_after();
        for (int kc = 0; kc < p.nk; ++kc) {
          // per tile: wait both CTAs' A halves, one fence, 4 K-steps, commit -> the
          // slot is released as soon as ITS MMAs retire (not the whole k-chunk's)
          const long long w0 = pclk2();
          mbar_wait(&w_land[wsl], wph);
          mbar_wait(&w_peer[wsl], wph);
          wait_cyc += pclk2() - w0;
          const uint64_t bdesc =
              desc_hi | (uint64_t)((smem_u32(sW + (size_t)wsl * p.wslot) & 0x3FFFFu) >> 4);
          for (int t = 0; t < T; ++t) {
            const long long w1 = pclk2();
            mbar_wait(&a_land[as], aph);
            mbar_wait(&a_peer[as], aph);
            wait_cyc += pclk2() - w1;
            tc_fence_after();
            if (elect_one()) {
              const uint64_t adesc =
                  desc_hi | (uint64_t)((smem_u32(sA + (size_t)as * kASlot2) & 0x3FFFFu) >> 4);
              const uint32_t dt = tmem_base + (uint32_t)(t * p.bp);
#pragma unroll
              for (int k = 0; k < 4; ++k)
                mma2_f16(dt, adesc + 2 * k, bdesc + 2 * k, p.idesc, (kc | k) != 0);
              commit2_both(&a_empty[as]);
              if (kc == p.nk - 1) commit2_both(&t_full[t]);
            }
            __syncwarp();
            if (++as == p.na) { as = 0; aph ^= 1; }
          }
          if (elect_one()) commit2_both(&w_empty[wsl]);
          __syncwarp();
          if (++wsl == p.nw) { wsl = 0; wph ^= 1; }
        }
        accph ^= (1u << T) - 1u;
      }
      if (dbg && lane == 0) { dbg[16] = wait_cyc; dbg[17] = pclk2() - t_begin; }
    } else if (lane == 0) {
      // peer: forward "my half landed" to the leader, slot by slot, in MMA order
      int as = 0, aph = 0, wsl = 0, wph = 0;
      for (int64_t g = pid; g < NGp; g += P) {
        int64_t r0, r1, o0, o1;
        half_range(g, n, U, NGp, rank, r0, r1, o0, o1);
        const int T = (int)std::max<int64_t>((r1 - r0 + 127) / 128, (o1 - o0 + 127) / 128);
        for (int kc = 0; kc < p.nk; ++kc) {
          mbar_wait(&w_land[wsl], wph);
          arrive_remote(map_to(smem_u32(&w_peer[wsl]), 0));
          if (++wsl == p.nw) { wsl = 0; wph ^= 1; }
          for (int t = 0; t < T; ++t) {
            mbar_wait(&a_land[as], aph);
            arrive_remote(map_to(smem_u32(&a_peer[as]), 0));
            if (++as == p.na) { as = 0; aph ^= 1; }
          }
        }
      }
    }
  } else if (warp <= 9) {
    // ----------------------------------------------------------- RMS + epilogue (both CTAs)
    const int q = warp & 3;
    const int wset = (warp - 2) >> 2;
    const int row = 32 * q + lane;
    const uint32_t swz = (uint32_t)(row & 7);
    uint64_t* ready = a_land;
    int as = 0, aph = 0, gi = 0;
    uint32_t accph = 0;
    long long sw_cyc = 0, s_begin = pclk2();
    for (int64_t g = pid; g < NGp; g += P) {
      int64_t r0, r1, o0, o1;
      half_range(g, n, U, NGp, rank, r0, r1, o0, o1);
      const int T = (int)std::max<int64_t>((r1 - r0 + 127) / 128, (o1 - o0 + 127) / 128);
      f32x2 ss[4][2];
#pragma unroll
      for (int t = 0; t < 4; ++t) ss[t][0] = ss[t][1] = 0ull;
      for (int kc = 0; kc < p.nk; ++kc) {
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          if (t < T && (t >> 1) != wset) {
            if (++as == p.na) { as = 0; aph ^= 1; }
          } else if (t < T) {
            const long long s0 = pclk2();
            mbar_wait(&ready[as], aph);
            sw_cyc += pclk2() - s0;
            const uint8_t* rp = sA + (size_t)as * kASlot2 + row * 128;
            uint4 u[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) u[j] = *reinterpret_cast<const uint4*>(rp + ((j ^ swz) << 4));
            __syncwarp();
            if (lane == 0) mbar_arrive(&a_empty[as]);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const uint32_t w[4] = {u[j].x, u[j].y, u[j].z, u[j].w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                f32x2 x;
                if (kBF16) {
                  x = pack2u(w[e] << 16, w[e] & 0xFFFF0000u);
                } else {
                  const float2 f2 = __half22float2(*reinterpret_cast<const __half2*>(&w[e]));
                  x = pack2(f2.x, f2.y);
                }
                ss[t][e & 1] = ffma2(x, x, ss[t][e & 1]);
              }
            }
            if (++as == p.na) { as = 0; aph ^= 1; }
          }
        }
      }
      if (dbg && warp == 2 && lane == 0) { dbg[2] = gtimer2(); dbg[20] = sw_cyc; dbg[21] = pclk2() - s_begin; }
      float ssum[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        float a0, a1, b0, b1;
        unpack2(ss[t][0], a0, a1);
        unpack2(ss[t][1], b0, b1);
        ssum[t] = (a0 + b0) + (a1 + b1);
      }
      const int par = gi & 1;
      mbar_wait(&m_empty[par], (((uint32_t)gi >> 1) & 1u) ^ 1u);
      for (int t = 2 * wset; t < 2 * wset + 2; ++t) {
        uint32_t bal = 0;
        if (t < T) {
          mbar_wait(&t_full[t], (accph >> t) & 1u);
          tc_fence_after();
          const int64_t r = r0 + (int64_t)t * 128 + row;
          const bool valid = r < r1;
          const float sq = t == 0 ? ssum[0] : t == 1 ? ssum[1] : t == 2 ? ssum[2] : ssum[3];
          const float scale = rms_scale(sq, p.inv_d, p.eps);
          const float hs = 0.5f * scale;  // exact (power of two)
          const f32x2 hs2 = pack2(hs, hs);
          f32x2 acc2 = 0ull;
          const uint32_t taddr = tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)(t * p.bp);
          for (int c0 = 0; c0 < p.b; c0 += 32) {
            uint32_t v[32];
            tmem_ld32(taddr + (uint32_t)c0, v);
            tmem_ld_wait();
            if (c0 + 32 <= p.b) {
#pragma unroll
              for (int jj = 0; jj < 32; jj += 4) {
                const float4 w4 = *reinterpret_cast<const float4*>(sWup + c0 + jj);
                const f32x2 s01 = silu2_tanh(fmul2(pack2u(v[jj], v[jj + 1]), hs2));
                const f32x2 s23 = silu2_tanh(fmul2(pack2u(v[jj + 2], v[jj + 3]), hs2));
                acc2 = ffma2(pack2(w4.x, w4.y), s01, acc2);
                acc2 = ffma2(pack2(w4.z, w4.w), s23, acc2);
              }
            } else {
#pragma unroll
              for (int jj = 0; jj < 32; jj += 2) {
                if (c0 + jj < p.b) {
                  const float w0 = sWup[c0 + jj];
                  const float w1 = (c0 + jj + 1 < p.b) ? sWup[c0 + jj + 1] : 0.0f;
                  const f32x2 s01 = silu2_tanh(fmul2(pack2u(v[jj], v[jj + 1]), hs2));
                  acc2 = ffma2(pack2(w0, w1), s01, acc2);
                }
              }
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (leader) mbar_arrive(&t_empty[t]);
            else arrive_remote(map_to(smem_u32(&t_empty[t]), 0));
          }
          float lo, hi;
          unpack2(acc2, lo, hi);
          const float logit = lo + hi;
          const float score = score_from_logit(logit);
          const bool ex = valid && (score > p.theta);
          if (valid) {
            if (p.scores) p.scores[r] = score;
            if (p.logits) p.logits[r] = logit;
            if (p.mask) p.mask[r] = ex ? 1 : 0;
            if (ex && p.exit_layers) p.exit_layers[gathered ? p.row_idx[r] : r] = p.layer;
          }
          bal = __ballot_sync(0xffffffffu, ex);
        }
        if (lane == 0) words[par * 16 + t * 4 + q] = bal;
      }
      accph ^= (1u << T) - 1u;
      __syncwarp();
      if (dbg && warp == 2 && lane == 0) dbg[3] = gtimer2();
      if (lane == 0) mbar_arrive(&m_full[par]);
      ++gi;
    }
  } else {
    // ----------------------------------------------------------- compaction (both CTAs)
    int gi = 0;
    for (int64_t g = pid; g < NGp; g += P) {
      int64_t r0, r1, o0, o1;
      half_range(g, n, U, NGp, rank, r0, r1, o0, o1);
      const int par = gi & 1;
      mbar_wait(&m_full[par], ((uint32_t)gi >> 1) & 1u);
      const uint32_t word = lane < 16 ? words[par * 16 + lane] : 0u;
      __syncwarp();
      if (lane == 0) mbar_arrive(&m_empty[par]);
      const uint32_t cnt = __popc(word);
      uint32_t incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const uint32_t excl_w = incl - cnt;
      const uint32_t agg = __shfl_sync(0xffffffffu, incl, 31);
      if (dbg && lane == 0) dbg[4] = gtimer2();
      if (need_scan) {
        const int64_t part = 2 * g + rank;
        const uint32_t E = lookback_exclusive(p.ws->status, tag, part, agg);
        if (dbg && lane == 0) dbg[5] = gtimer2();
        if (p.exit_idx || p.cont_idx) {
          const int nwords = (int)((r1 - r0 + 31) / 32);
          const uint32_t lt = (1u << lane) - 1u;
          for (int w = 0; w < nwords; ++w) {
            const uint32_t wd = __shfl_sync(0xffffffffu, word, w);
            const uint32_t pre = __shfl_sync(0xffffffffu, excl_w, w);
            const int64_t r = r0 + 32 * w + lane;
            if (r < r1) {
              const int64_t rank_e = (int64_t)E + pre + __popc(wd & lt);
              const int64_t id = (p.ids_from_rows && gathered) ? p.row_idx[r] : r;
              if ((wd >> lane) & 1u) {
                if (p.exit_idx) p.exit_idx[rank_e] = id;
              } else if (p.cont_idx) {
                p.cont_idx[r - rank_e] = id;
              }
            }
          }
        }
        if (part == 2 * NGp - 1 && lane == 0 && p.counts) {
          p.counts[0] = (int64_t)E + agg;
          p.counts[1] = n - ((int64_t)E + agg);
        }
      }
      ++gi;
    }
    if (NGp == 0 && blockIdx.x == 0 && lane == 0 && p.counts) {
      p.counts[0] = 0;
      p.counts[1] = 0;
    }
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // no CTA leaves while its peer may still touch its smem / TMEM
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc2(tmem_base, p.tmem_cols);
  }
  if (dbg && threadIdx.x == 0) dbg[6] = gtimer2();
  if (threadIdx.x == 0) launch_done(p.ws);
}

int route_tc2_launch(const RouteArgs& a, cudaStream_t stream) {
  const int npad = (a.b + 15) / 16 * 16;
  const int bp = (npad + 31) / 32 * 32;
  const int tpg = std::min(4, 512 / bp);
  int cols = 32;
  while (cols < tpg * bp) cols <<= 1;
  const int nk = (a.d + 63) / 64;
  const uint32_t wslot = (uint32_t)(npad / 2) * 128u;  // this CTA's half of a W k-chunk
  const int nw = std::min(kMaxNW2, std::max(3, (int)(24 * 1024 / std::max<uint32_t>(wslot, 1u))));
  const uint32_t off_a = (uint32_t)nw * wslot;
  const uint32_t off_a_al = (off_a + 1023u) & ~1023u;
  const int smem_cap = 227 * 1024;
  const uint32_t misc = 1024 + 768 + 128 + 2048 + 16;
  int na = (int)((smem_cap - 1024 - off_a_al - misc) / kASlot2);
  na = std::min(na, kMaxNA2);
  if (na < 2 || nw < 2) return set_error(TIDE_ERR_UNSUPPORTED, "bottleneck too wide for smem");
  Tc2Params p{};
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
  p.idesc = f16_idesc(a.dtype == TIDE_BF16 ? 1 : 0, 256, npad);
  p.tmem_cols = (uint32_t)cols;
  p.wslot = wslot;
  p.off_a = off_a_al;
  p.off_wup = off_a_al + (uint32_t)na * kASlot2;
  p.off_bar = p.off_wup + 1024;
  p.off_words = p.off_bar + 768;
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
  p.scores = a.scores;
  p.logits = a.logits;
  p.mask = a.mask;
  p.exit_idx = a.exit_idx;
  p.cont_idx = a.cont_idx;
  p.exit_layers = a.exit_layers;
  p.counts = a.counts;
  p.ws = reinterpret_cast<Workspace*>(a.workspace);
  p.dbg = g_dbg;

  CUtensorMap tm_h128, tm_h64, tm_h32, tm_h16, tm_w, tm_g4;
  const int64_t hrows = a.row_idx ? a.rows_total : std::max<int64_t>(a.n, 1);
  int rc;
  if ((rc = make_map(&tm_h128, a.h, a.dtype, a.d, hrows, a.ld_h, 64, 128))) return rc;
  if ((rc = make_map(&tm_h64, a.h, a.dtype, a.d, hrows, a.ld_h, 64, 64))) return rc;
  if ((rc = make_map(&tm_h32, a.h, a.dtype, a.d, hrows, a.ld_h, 64, 32))) return rc;
  if ((rc = make_map(&tm_h16, a.h, a.dtype, a.d, hrows, a.ld_h, 64, kGran2))) return rc;
  if ((rc = make_map(&tm_g4, a.h, a.dtype, a.d, hrows, a.ld_h, 64, 1))) return rc;
  if ((rc = make_map(&tm_w, a.w_down, a.dtype, a.d, a.b, a.d, 64, npad / 2))) return rc;

  int dev = 0;
  cudaGetDevice(&dev);
  const int sms = sm_count(dev);
  const int64_t U = (a.n + kGran2 - 1) / kGran2;
  int64_t pairs = std::max<int64_t>(1, std::min<int64_t>(sms / 2, (U + 1) / 2));
  const int grid = (int)(2 * pairs);
  const int64_t cpg = (int64_t)tpg * (128 / kGran2);
  if (2 * std::max<int64_t>(pairs, (U + 2 * cpg - 1) / (2 * cpg)) > kMaxParts / 2)
    return set_error(TIDE_ERR_UNSUPPORTED, "too many rows for one launch");
  static bool attr_set[64] = {false};
  if (!attr_set[dev & 63]) {
    cudaFuncSetAttribute(route_tc2_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         227 * 1024);
    cudaFuncSetAttribute(route_tc2_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         227 * 1024);
    attr_set[dev & 63] = true;
  }
  if (a.dtype == TIDE_BF16)
    route_tc2_kernel<true><<<grid, kThreads2, smem_bytes, stream>>>(tm_h128, tm_h64, tm_h32, tm_h16, tm_w, tm_g4, p);
  else
    route_tc2_kernel<false><<<grid, kThreads2, smem_bytes, stream>>>(tm_h128, tm_h64, tm_h32, tm_h16, tm_w, tm_g4, p);
  return check_launch("route_tc2_kernel");
}

}  // namespace tide
