// K8: the LM head of posthoc_select on tcgen05 (ee/model.py:329-338,
// ee/runtime.py:176-181: logits = final_norm(rows) @ lm_head^T in f32).
//
//   out[n, V] = A[n, d] . B[V, d]^T
//
// A = the final-normed rows select_project stages, B = the LM head, both
// given as bf16 pairs x = hi + lo (hi = bf16(x), lo = bf16(x - hi): x to
// ~2^-17 relative).  Three kind::f16 MMAs per K step give f32-grade products:
//   acc_big   += A_hi B_hi                 (TMEM columns [0, 256))
//   acc_small += A_hi B_lo + A_lo B_hi     (TMEM columns [256, 512))
// The two small terms accumulate apart from the big one, so their low bits
// are not lost against a large running sum; the epilogue adds them once.
// (lo pointers NULL: one MMA per step, bf16 products.)
//
// Tile 128 rows x 256 vocab columns per CTA, K chunks of 64 (the 128-byte
// swizzle atom), TMA into a 2-stage ring of 96 KB (A_hi, A_lo 16 KB each,
// B_hi, B_lo 32 KB each), one MMA-issuing warp, 4 epilogue warps draining
// TMEM (32 columns at a time) into f32 rows.  Grid x = row tiles (fastest),
// y = vocab tiles: the row tiles of one vocab tile run in the same wave, so
// each 256-row slice of the LM head is read from HBM once and from L2 by the
// others (A, all rows hi + lo, stays L2-resident).  Roofline: tensor —
// 2 n V d flop per term; the 3-term form runs 3 MMAs per step.
// Default form: persistent CTA pairs (lmhead2p_kernel below) with the
// TMA-store epilogue; the one-tile kernels stay for A/B runs and tests.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "internal.h"

namespace tide {

namespace {

constexpr int kLThreads = 192;
constexpr int kLBM = 128, kLBN = 256, kLBK = 64;
constexpr uint32_t kLASlot = kLBM * 128;  // 16 KB
constexpr uint32_t kLBSlot = kLBN * 128;  // 32 KB

struct LmParams {
  int64_t n, V, ld_out;
  int32_t nk, stages, terms;
  uint32_t stage_bytes, idesc;
  float* out;
  int32_t tma_store;  // 1: the epilogue stores through the output tensor map tm_o
};

// ---------------------------------------------------------------------------
// Epilogue: TMEM -> registers (big + small) -> the logits.  With tma_store the
// 32 x 32 f32 block of each warp goes through shared memory (the consumed
// operand ring, 2 x 4 KB per warp, SW128 layout = the map's swizzle) and one
// TMA store per block: the stores leave as whole 128-byte lines instead of
// 32 rows x 16 bytes per warp instruction, and the tensor map clips rows >= n
// and columns >= V.  Without it (an output the map cannot describe)
// row-per-lane float4 stores.
template <int kTerms>
__device__ __forceinline__ void lm_epilogue(const LmParams& p, const CUtensorMap* tm_o, uint32_t taddr,
                                            uint8_t* wbuf, int64_t m0q, int64_t v0) {
  const int lane = threadIdx.x & 31;
  const int64_t row = m0q + lane;
  float* orow = p.out + row * p.ld_out;
#pragma unroll 1
  for (int c0 = 0, it = 0; c0 < kLBN; c0 += 32, ++it) {
    uint32_t v[32];
    tmem_ld32(taddr + (uint32_t)c0, v);
    if (kTerms == 3) {
      uint32_t w[32];
      tmem_ld32(taddr + 256u + (uint32_t)c0, w);
      tmem_ld_wait_regs(v);
      tmem_ld_wait_regs(w);
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(__uint_as_float(v[j]) + __uint_as_float(w[j]));
    } else {
      tmem_ld_wait_regs(v);
    }
    if (p.tma_store) {
      uint8_t* buf = wbuf + (it & 1) * 4096;
      if (it >= 2) {
        // the store issued from this buffer two blocks ago has read it
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        __syncwarp();
      }
      const uint32_t rbase = smem_u32(buf) + (uint32_t)lane * 128u;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(rbase + ((uint32_t)(j ^ (lane & 7)) << 4)),
                     "r"(v[4 * j]), "r"(v[4 * j + 1]), "r"(v[4 * j + 2]), "r"(v[4 * j + 3])
                     : "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        asm volatile(
            "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(tm_o),
            "r"(smem_u32(buf)), "r"((int)(v0 + c0)), "r"((int)m0q)
            : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    } else if (row < p.n) {
      const int64_t col = v0 + c0;
      if (col + 32 <= p.V) {
#pragma unroll
        for (int j = 0; j < 32; j += 4)
          *reinterpret_cast<float4*>(orow + col + j) =
              make_float4(__uint_as_float(v[j]), __uint_as_float(v[j + 1]), __uint_as_float(v[j + 2]),
                          __uint_as_float(v[j + 3]));
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (col + j < p.V) orow[col + j] = __uint_as_float(v[j]);
      }
    }
  }
  if (p.tma_store && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  __syncwarp();
}

template <int kTerms>
__global__ void __launch_bounds__(kLThreads, 1)
    lmhead_kernel(const __grid_constant__ CUtensorMap tm_ah, const __grid_constant__ CUtensorMap tm_al,
                  const __grid_constant__ CUtensorMap tm_bh, const __grid_constant__ CUtensorMap tm_bl,
                  const __grid_constant__ CUtensorMap tm_o, const __grid_constant__ LmParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)p.stages * p.stage_bytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + 8;
  uint64_t* acc_full = bars + 16;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 17);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t m0 = (int64_t)blockIdx.x * kLBM, v0 = (int64_t)blockIdx.y * kLBN;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tm_ah);
    prefetch_tmap(&tm_bh);
    if (kTerms == 3) {
      prefetch_tmap(&tm_al);
      prefetch_tmap(&tm_bl);
    }
    for (int i = 0; i < p.stages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(acc_full, 1);
    fence_mbar_init();
  }
  if (warp == 1) {
    tmem_alloc(tmem_slot, kTerms == 3 ? 512u : 256u);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // the staged rows may come from the kernel just before on the stream
  griddep_wait();

  if (warp == 0) {
    // ----------------------------------------------------------- producer
    if (lane == 0) {
      // A (all rows, hi + lo) is re-read by every vocab tile: keep it; a B
      // slice serves the row tiles of one wave: normal priority.  ncu at
      // 4096 x 50,257 x 4096: 3.8 GB read from DRAM per launch (B is 0.82 GB,
      // A 64 MB; evict_first on B measured the same), ~1 TB/s — far from the
      // bound; the tensor pipe is 71% active (profiles/r02_lmhead_kernel_3term.json)
      const uint64_t pol_a = policy_evict_last();
      uint64_t pol_b;
      asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol_b));
      const uint32_t bytes = kTerms == 3 ? 2u * (kLASlot + kLBSlot) : kLASlot + kLBSlot;
      for (int kc = 0; kc < p.nk; ++kc) {
        const int s = kc % p.stages;
        mbar_wait(&empty[s], ((kc / p.stages) & 1) ^ 1);
        uint8_t* st = smem + (size_t)s * p.stage_bytes;
        mbar_arrive_expect_tx(&full[s], bytes);
        tma_load_2d(st, &tm_ah, &full[s], kc * kLBK, (int)m0, pol_a);
        tma_load_2d(st + kLASlot, &tm_bh, &full[s], kc * kLBK, (int)v0, pol_b);
        if (kTerms == 3) {
          tma_load_2d(st + kLASlot + kLBSlot, &tm_al, &full[s], kc * kLBK, (int)m0, pol_a);
          tma_load_2d(st + 2 * kLASlot + kLBSlot, &tm_bl, &full[s], kc * kLBK, (int)v0, pol_b);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ----------------------------------------------------------- MMA issuer
    const uint64_t dh = sw128_kmajor_desc(0);
    for (int kc = 0; kc < p.nk; ++kc) {
      const int s = kc % p.stages;
      mbar_wait(&full[s], (kc / p.stages) & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint8_t* st = smem + (size_t)s * p.stage_bytes;
        const uint64_t ah = dh | (uint64_t)((smem_u32(st) & 0x3FFFFu) >> 4);
        const uint64_t bh = dh | (uint64_t)((smem_u32(st + kLASlot) & 0x3FFFFu) >> 4);
        const uint64_t al = dh | (uint64_t)((smem_u32(st + kLASlot + kLBSlot) & 0x3FFFFu) >> 4);
        const uint64_t bl = dh | (uint64_t)((smem_u32(st + 2 * kLASlot + kLBSlot) & 0x3FFFFu) >> 4);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t acc = (kc != 0 || k != 0) ? 1u : 0u;
          tc_mma_f16(tmem_base, ah + 2 * k, bh + 2 * k, p.idesc, acc);
          if (kTerms == 3) {
            tc_mma_f16(tmem_base + 256u, ah + 2 * k, bl + 2 * k, p.idesc, acc);
            tc_mma_f16(tmem_base + 256u, al + 2 * k, bh + 2 * k, p.idesc, 1u);
          }
        }
        tc_commit(&empty[s]);
        if (kc == p.nk - 1) tc_commit(acc_full);
      }
      __syncwarp();
    }
  } else {
    // ----------------------------------------------------------- epilogue
    const int q = warp & 3;  // TMEM lane quadrant
    mbar_wait(acc_full, 0);
    tc_fence_after();
    const uint32_t taddr = tmem_base + ((uint32_t)(32 * q) << 16);
    // the operand ring is consumed (every MMA completed): 8 KB per warp of it
    lm_epilogue<kTerms>(p, &tm_o, taddr, smem + (size_t)q * 8192, m0 + 32 * q, v0);
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, kTerms == 3 ? 512u : 256u);
  }
}

// ---------------------------------------------------------------------------
// CTA-pair form (cta_group::2): a cluster of 2 CTAs on one TPC computes a
// 256-row x 256-vocab tile with M = 256 MMAs issued by the leader.  CTA r
// stages its own 128 rows of A and HALF of the vocab tile's B rows (v0 + 128 r
// ..), so each SM streams 64 KB per 64-column chunk (3-term) instead of 96 KB:
// the one-CTA kernel is fed from L2 (A re-read by every vocab tile, B by
// every row tile) and the halved B share is what the pair buys.  The peer
// forwards "my stage landed" to the leader (remote mbarrier arrive); the
// leader's commits arrive on both CTAs' barriers (multicast).  Each CTA's
// TMEM holds its own 128 rows x 256 columns (big, + small at column 256):
// the epilogue is the one-CTA kernel's.
__device__ __forceinline__ uint32_t lm_cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t lm_mapa(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void lm_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" :::
                   "memory");
}
__device__ __forceinline__ void lm_arrive_remote(uint32_t caddr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(caddr) : "memory");
}
__device__ __forceinline__ void lm_tmem_alloc2(uint32_t* dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void lm_tmem_dealloc2(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void lm_mma2(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// commit -> one arrive on the barrier at this smem offset in BOTH CTAs of the pair
__device__ __forceinline__ void lm_commit2_both(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], m;\n\t}\n" ::"r"(smem_u32(bar))
      : "memory");
}

template <int kTerms>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kLThreads, 1)
    lmhead2_kernel(const __grid_constant__ CUtensorMap tm_ah, const __grid_constant__ CUtensorMap tm_al,
                   const __grid_constant__ CUtensorMap tm_bh, const __grid_constant__ CUtensorMap tm_bl,
                   const __grid_constant__ CUtensorMap tm_o, const __grid_constant__ LmParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)p.stages * p.stage_bytes);
  uint64_t* full = bars;             // this CTA's stage landed (TMA bytes)
  uint64_t* peer_full = bars + 8;    // leader: the peer's stage landed (forwarded)
  uint64_t* empty = bars + 16;       // both: stage consumed (leader's commit, multicast)
  uint64_t* acc_full = bars + 24;    // both: accumulator complete (multicast)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 25);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = lm_cta_rank();
  const bool leader = rank == 0;
  const int64_t m0 = (int64_t)blockIdx.x * kLBM;                     // this CTA's 128 rows
  const int64_t v0 = (int64_t)blockIdx.y * kLBN;                     // the pair's 256 vocab columns
  const int64_t vb = v0 + (int64_t)rank * (kLBN / 2);               // this CTA's B half
  constexpr uint32_t kHalfB = (kLBN / 2) * 128;                     // 16 KB
  const uint32_t cols = kTerms == 3 ? 512u : 256u;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tm_ah);
    prefetch_tmap(&tm_bh);
    if (kTerms == 3) {
      prefetch_tmap(&tm_al);
      prefetch_tmap(&tm_bl);
    }
    for (int i = 0; i < p.stages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&peer_full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(acc_full, 1);
    fence_mbar_init();
  }
  if (warp == 1) lm_tmem_alloc2(tmem_slot, cols);
  tc_fence_before();
  __syncthreads();
  lm_cluster_sync();  // the peer's barriers exist before any remote arrive / multicast
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  griddep_wait();  // the staged rows may come from the kernel just before on the stream

  if (warp == 0) {
    // ----------------------------------------------------------- producer (both CTAs)
    if (lane == 0) {
      const uint64_t pol_a = policy_evict_last();
      uint64_t pol_b;
      asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol_b));
      const uint32_t bytes = kTerms == 3 ? 2u * (kLASlot + kHalfB) : kLASlot + kHalfB;
      for (int kc = 0; kc < p.nk; ++kc) {
        const int s = kc % p.stages;
        mbar_wait(&empty[s], ((kc / p.stages) & 1) ^ 1);
        uint8_t* st = smem + (size_t)s * p.stage_bytes;
        mbar_arrive_expect_tx(&full[s], bytes);
        tma_load_2d(st, &tm_ah, &full[s], kc * kLBK, (int)m0, pol_a);
        tma_load_2d(st + kLASlot, &tm_bh, &full[s], kc * kLBK, (int)vb, pol_b);
        if (kTerms == 3) {
          tma_load_2d(st + kLASlot + kHalfB, &tm_al, &full[s], kc * kLBK, (int)m0, pol_a);
          tma_load_2d(st + 2 * kLASlot + kHalfB, &tm_bl, &full[s], kc * kLBK, (int)vb, pol_b);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (leader) {
      // ----------------------------------------------------------- MMA issuer (leader)
      const uint64_t dh = sw128_kmajor_desc(0);
      for (int kc = 0; kc < p.nk; ++kc) {
        const int s = kc % p.stages;
        const uint32_t ph = (kc / p.stages) & 1;
        mbar_wait(&full[s], ph);
        mbar_wait(&peer_full[s], ph);
        tc_fence_after();
        if (elect_one()) {
          const uint8_t* st = smem + (size_t)s * p.stage_bytes;
          const uint64_t ah = dh | (uint64_t)((smem_u32(st) & 0x3FFFFu) >> 4);
          const uint64_t bh = dh | (uint64_t)((smem_u32(st + kLASlot) & 0x3FFFFu) >> 4);
          const uint64_t al = dh | (uint64_t)((smem_u32(st + kLASlot + kHalfB) & 0x3FFFFu) >> 4);
          const uint64_t bl = dh | (uint64_t)((smem_u32(st + 2 * kLASlot + kHalfB) & 0x3FFFFu) >> 4);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint32_t acc = (kc != 0 || k != 0) ? 1u : 0u;
            lm_mma2(tmem_base, ah + 2 * k, bh + 2 * k, p.idesc, acc);
            if (kTerms == 3) {
              lm_mma2(tmem_base + 256u, ah + 2 * k, bl + 2 * k, p.idesc, acc);
              lm_mma2(tmem_base + 256u, al + 2 * k, bh + 2 * k, p.idesc, 1u);
            }
          }
          lm_commit2_both(&empty[s]);
          if (kc == p.nk - 1) lm_commit2_both(acc_full);
        }
        __syncwarp();
      }
    } else if (lane == 0) {
      // ----------------------------------------------------------- peer: forward "landed"
      const uint32_t remote = lm_mapa(smem_u32(peer_full), 0);
      for (int kc = 0; kc < p.nk; ++kc) {
        const int s = kc % p.stages;
        mbar_wait(&full[s], (kc / p.stages) & 1);
        lm_arrive_remote(remote + (uint32_t)s * 8u);
      }
    }
  } else {
    // ----------------------------------------------------------- epilogue (both CTAs)
    const int q = warp & 3;  // TMEM lane quadrant
    mbar_wait(acc_full, 0);
    tc_fence_after();
    const uint32_t taddr = tmem_base + ((uint32_t)(32 * q) << 16);
    // the operand ring is consumed (every MMA completed): 8 KB per warp of it
    lm_epilogue<kTerms>(p, &tm_o, taddr, smem + (size_t)q * 8192, m0 + 32 * q, v0);
    tc_fence_before();
  }
  __syncthreads();
  lm_cluster_sync();  // neither CTA leaves (or frees TMEM) while the pair's MMAs / copies may touch it
  if (warp == 1) {
    tc_fence_after();
    lm_tmem_dealloc2(tmem_base, cols);
  }
}

// ---------------------------------------------------------------------------
// Persistent CTA-pair form: one pair per TPC walks pair tiles t = pair,
// pair + pairs, ... (t % row-pairs fastest, so the pairs in flight share a
// few vocab slices through L2, as the one-tile grid's waves do).  The operand
// ring runs on across tiles: the producer streams the next tile's chunks
// while the epilogue drains the last accumulator, and no tile pays a launch,
// barrier set-up, TMEM allocation or pipeline fill.  TMEM holds kAcc
// accumulator sets (3 terms: one set of 512 columns; hi only: two of 256,
// so the next tile's MMAs run under the epilogue).  acc_full[a]: the leader's
// last commit of a tile (multicast to both CTAs); acc_empty[a] (leader): the
// 4 epilogue warps of each CTA have read set a (the peer's arrive remotely).
// The epilogue stages its TMA stores in 32 KB of its own (the ring is busy).
__device__ __forceinline__ void lm_arrive_remote_release(uint32_t caddr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(caddr) : "memory");
}
__device__ __forceinline__ void lm_wait_cluster(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t spins = 0, ok = 0;
  while (true) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
    if (ok) break;
    if (++spins > TIDE_SPIN_LIMIT) __trap();
  }
}

constexpr uint32_t kLEpiBytes = 4u * 8192u;  // the persistent epilogue's staging

template <int kTerms>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kLThreads, 1)
    lmhead2p_kernel(const __grid_constant__ CUtensorMap tm_ah, const __grid_constant__ CUtensorMap tm_al,
                    const __grid_constant__ CUtensorMap tm_bh, const __grid_constant__ CUtensorMap tm_bl,
                    const __grid_constant__ CUtensorMap tm_o, const __grid_constant__ LmParams p) {
  constexpr int kAcc = kTerms == 3 ? 1 : 2;
  constexpr uint32_t kAccCols = kTerms == 3 ? 512u : 256u;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* epi = smem + (size_t)p.stages * p.stage_bytes;  // 1024-aligned (stage_bytes is)
  uint64_t* bars = reinterpret_cast<uint64_t*>(epi + kLEpiBytes);
  uint64_t* full = bars;             // this CTA's stage landed (TMA bytes)
  uint64_t* peer_full = bars + 8;    // leader: the peer's stage landed (forwarded)
  uint64_t* empty = bars + 16;       // both: stage consumed (leader's commit, multicast)
  uint64_t* acc_full = bars + 24;    // both: accumulator set complete [kAcc]
  uint64_t* acc_empty = bars + 26;   // leader: accumulator set drained [kAcc]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 28);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = lm_cta_rank();
  const bool leader = rank == 0;
  constexpr uint32_t kHalfB = (kLBN / 2) * 128;  // 16 KB
  const int64_t RP = (p.n + 2 * kLBM - 1) / (2 * kLBM);   // row pairs
  const int64_t T = RP * ((p.V + kLBN - 1) / kLBN);        // pair tiles
  const int64_t pair = blockIdx.x >> 1, pairs = gridDim.x >> 1;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tm_ah);
    prefetch_tmap(&tm_bh);
    if (kTerms == 3) {
      prefetch_tmap(&tm_al);
      prefetch_tmap(&tm_bl);
    }
    prefetch_tmap(&tm_o);
    for (int i = 0; i < p.stages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&peer_full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int a = 0; a < kAcc; ++a) {
      mbar_init(&acc_full[a], 1);
      mbar_init(&acc_empty[a], 8);  // 4 epilogue warps x 2 CTAs
    }
    fence_mbar_init();
  }
  if (warp == 1) lm_tmem_alloc2(tmem_slot, 512u);
  tc_fence_before();
  __syncthreads();
  lm_cluster_sync();  // the peer's barriers exist before any remote arrive / multicast
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  griddep_wait();  // the staged rows may come from the kernel just before on the stream

  if (warp == 0) {
    // ----------------------------------------------------------- producer (both CTAs)
    if (lane == 0) {
      const uint64_t pol_a = policy_evict_last();
      uint64_t pol_b;
      asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol_b));
      const uint32_t bytes = kTerms == 3 ? 2u * (kLASlot + kHalfB) : kLASlot + kHalfB;
      uint32_t g = 0;
      for (int64_t t = pair; t < T; t += pairs) {
        const int m0 = (int)((t % RP) * (2 * kLBM) + (int64_t)rank * kLBM);
        const int vb = (int)((t / RP) * kLBN + (int64_t)rank * (kLBN / 2));
        for (int kc = 0; kc < p.nk; ++kc, ++g) {
          const int s = (int)(g % (uint32_t)p.stages);
          mbar_wait(&empty[s], ((g / (uint32_t)p.stages) & 1) ^ 1);
          uint8_t* st = smem + (size_t)s * p.stage_bytes;
          mbar_arrive_expect_tx(&full[s], bytes);
          tma_load_2d(st, &tm_ah, &full[s], kc * kLBK, m0, pol_a);
          tma_load_2d(st + kLASlot, &tm_bh, &full[s], kc * kLBK, vb, pol_b);
          if (kTerms == 3) {
            tma_load_2d(st + kLASlot + kHalfB, &tm_al, &full[s], kc * kLBK, m0, pol_a);
            tma_load_2d(st + 2 * kLASlot + kHalfB, &tm_bl, &full[s], kc * kLBK, vb, pol_b);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (leader) {
      // ----------------------------------------------------------- MMA issuer (leader)
      const uint64_t dh = sw128_kmajor_desc(0);
      uint32_t g = 0, i = 0;
      for (int64_t t = pair; t < T; t += pairs, ++i) {
        const uint32_t a = i % kAcc;
        const uint32_t acc0 = tmem_base + a * kAccCols;
        lm_wait_cluster(&acc_empty[a], ((i / kAcc) & 1) ^ 1);  // both epilogues read set a
        tc_fence_after();
        for (int kc = 0; kc < p.nk; ++kc, ++g) {
          const int s = (int)(g % (uint32_t)p.stages);
          const uint32_t ph = (g / (uint32_t)p.stages) & 1;
          mbar_wait(&full[s], ph);
          mbar_wait(&peer_full[s], ph);
          tc_fence_after();
          if (elect_one()) {
            const uint8_t* st = smem + (size_t)s * p.stage_bytes;
            const uint64_t ah = dh | (uint64_t)((smem_u32(st) & 0x3FFFFu) >> 4);
            const uint64_t bh = dh | (uint64_t)((smem_u32(st + kLASlot) & 0x3FFFFu) >> 4);
            const uint64_t al = dh | (uint64_t)((smem_u32(st + kLASlot + kHalfB) & 0x3FFFFu) >> 4);
            const uint64_t bl = dh | (uint64_t)((smem_u32(st + 2 * kLASlot + kHalfB) & 0x3FFFFu) >> 4);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint32_t acc = (kc != 0 || k != 0) ? 1u : 0u;
              lm_mma2(acc0, ah + 2 * k, bh + 2 * k, p.idesc, acc);
              if (kTerms == 3) {
                lm_mma2(acc0 + 256u, ah + 2 * k, bl + 2 * k, p.idesc, acc);
                lm_mma2(acc0 + 256u, al + 2 * k, bh + 2 * k, p.idesc, 1u);
              }
            }
            lm_commit2_both(&empty[s]);
            if (kc == p.nk - 1) lm_commit2_both(&acc_full[a]);
          }
          __syncwarp();
        }
      }
    } else if (lane == 0) {
      // ----------------------------------------------------------- peer: forward "landed"
      const uint32_t remote = lm_mapa(smem_u32(peer_full), 0);
      uint32_t g = 0;
      for (int64_t t = pair; t < T; t += pairs)
        for (int kc = 0; kc < p.nk; ++kc, ++g) {
          const int s = (int)(g % (uint32_t)p.stages);
          mbar_wait(&full[s], (g / (uint32_t)p.stages) & 1);
          lm_arrive_remote(remote + (uint32_t)s * 8u);
        }
    }
  } else {
    // ----------------------------------------------------------- epilogue (both CTAs)
    const int q = warp & 3;  // TMEM lane quadrant
    uint8_t* wbuf = epi + (size_t)q * 8192;
    const uint32_t empty_addr = lm_mapa(smem_u32(acc_empty), 0);  // the leader's barriers
    uint32_t i = 0, it = 0;
    for (int64_t t = pair; t < T; t += pairs, ++i) {
      const uint32_t a = i % kAcc;
      const int64_t m0q = (t % RP) * (2 * kLBM) + (int64_t)rank * kLBM + 32 * q;
      const int64_t v0 = (t / RP) * kLBN;
      mbar_wait(&acc_full[a], (i / kAcc) & 1);
      tc_fence_after();
      const uint32_t taddr = tmem_base + a * kAccCols + ((uint32_t)(32 * q) << 16);
      const int64_t row = m0q + lane;
      float* orow = p.out + row * p.ld_out;
#pragma unroll 1
      for (int c0 = 0; c0 < kLBN; c0 += 32, ++it) {
        uint32_t v[32];
        tmem_ld32(taddr + (uint32_t)c0, v);
        if (kTerms == 3) {
          uint32_t w[32];
          tmem_ld32(taddr + 256u + (uint32_t)c0, w);
          tmem_ld_wait_regs(v);
          tmem_ld_wait_regs(w);
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(__uint_as_float(v[j]) + __uint_as_float(w[j]));
        } else {
          tmem_ld_wait_regs(v);
        }
        if (c0 + 32 == kLBN) {
          // every column of set a is in registers: hand it back to the MMA warp
          tc_fence_before();
          __syncwarp();
          if (lane == 0) lm_arrive_remote_release(empty_addr + a * 8u);
        }
        if (p.tma_store) {
          uint8_t* buf = wbuf + (it & 1) * 4096;
          if (it >= 2) {
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            __syncwarp();
          }
          const uint32_t rbase = smem_u32(buf) + (uint32_t)lane * 128u;
#pragma unroll
          for (int j = 0; j < 8; ++j)
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(rbase + ((uint32_t)(j ^ (lane & 7)) << 4)),
                         "r"(v[4 * j]), "r"(v[4 * j + 1]), "r"(v[4 * j + 2]), "r"(v[4 * j + 3])
                         : "memory");
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            asm volatile(
                "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(&tm_o),
                "r"(smem_u32(buf)), "r"((int)(v0 + c0)), "r"((int)m0q)
                : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
        } else if (row < p.n) {
          const int64_t col = v0 + c0;
          if (col + 32 <= p.V) {
#pragma unroll
            for (int j = 0; j < 32; j += 4)
              *reinterpret_cast<float4*>(orow + col + j) =
                  make_float4(__uint_as_float(v[j]), __uint_as_float(v[j + 1]), __uint_as_float(v[j + 2]),
                              __uint_as_float(v[j + 3]));
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (col + j < p.V) orow[col + j] = __uint_as_float(v[j]);
          }
        }
      }
    }
    if (p.tma_store && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    __syncwarp();
  }
  __syncthreads();
  lm_cluster_sync();  // neither CTA leaves (or frees TMEM) while the pair's MMAs / copies may touch it
  if (warp == 1) {
    tc_fence_after();
    lm_tmem_dealloc2(tmem_base, 512u);
  }
}

bool lm_persist() {
  const char* env = getenv("TIDE_LM_PERSIST");  // read per call (A/B runs, tests)
  return !(env && env[0] == '0');
}

// CTA pairs: the persistent form for both term counts; one tile per pair
// (TIDE_LM_PERSIST=0) only for 3 terms (the hi-only form: 1.59 one CTA vs
// 1.74 ms paired, one tile per CTA).  TIDE_LM_PAIR=0 / 1 forces either.
bool lm_pair(int terms) {
  const char* env = getenv("TIDE_LM_PAIR");  // read per call
  if (env) return env[0] == '1';
  return terms == 3 || lm_persist();
}

// Co-resident CTA pairs of the persistent kernel (queried once per form).
template <typename K>
int lm_pairs(K kernel, uint32_t smem, int slot) {
  static int cache[2] = {0, 0};
  if (!cache[slot]) {
    cudaLaunchConfig_t q = {};
    q.gridDim = dim3(2 * 1024, 1, 1);
    q.blockDim = dim3(kLThreads, 1, 1);
    q.dynamicSmemBytes = smem;
    int v = 0;
    if (cudaOccupancyMaxActiveClusters(&v, kernel, &q) != cudaSuccess || v <= 0) {
      cudaGetLastError();
      int dev = 0;
      cudaGetDevice(&dev);
      v = sm_count(dev) / 2;
    }
    cache[slot] = v;
  }
  return cache[slot];
}

}  // namespace

int lmhead_launch(const void* a_hi, const void* a_lo, int64_t ld_a, int64_t n, int32_t d,
                  const void* b_hi, const void* b_lo, int64_t ld_b, int64_t V, float* out,
                  int64_t ld_out, cudaStream_t stream) {
  const int terms = (a_lo && b_lo) ? 3 : 1;
  CUtensorMap ah, al, bh, bl;
  int rc;
  if ((rc = make_map(&ah, a_hi, TIDE_BF16, d, n, ld_a, kLBK, kLBM))) return rc;
  const int bbox = lm_pair(terms) ? kLBN / 2 : kLBN;  // pair: each CTA loads half of B
  if ((rc = make_map(&bh, b_hi, TIDE_BF16, d, V, ld_b, kLBK, bbox))) return rc;
  if (terms == 3) {
    if ((rc = make_map(&al, a_lo, TIDE_BF16, d, n, ld_a, kLBK, kLBM))) return rc;
    if ((rc = make_map(&bl, b_lo, TIDE_BF16, d, V, ld_b, kLBK, bbox))) return rc;
  } else {
    al = ah;
    bl = bh;
  }
  // 4,096 x 50,257 x 4096, 3 terms: one CTA 3.87 ms, one-tile pairs 3.41,
  // + TMA-store epilogue 3.27-3.32, persistent pairs 3.16-3.27 ms; hi only:
  // one CTA 1.59-1.8, persistent pairs 1.22-1.33 ms (tools/remote/lm_persist.sh)
  const bool pair = lm_pair(terms);
  const bool persist = pair && lm_persist();
  LmParams p{};
  p.n = n;
  p.V = V;
  p.ld_out = ld_out;
  p.nk = (d + kLBK - 1) / kLBK;
  p.terms = terms;
  p.stage_bytes = pair ? (terms == 3 ? 2u * (kLASlot + kLBSlot / 2) : kLASlot + kLBSlot / 2)
                       : (terms == 3 ? 2u * (kLASlot + kLBSlot) : kLASlot + kLBSlot);
  const uint32_t cap = 227u * 1024u - 1024u - 256u - (persist ? kLEpiBytes : 0u);
  p.stages = (int)std::min<uint32_t>(8u, cap / p.stage_bytes);
  p.idesc = f16_idesc(1, pair ? 2 * kLBM : kLBM, kLBN);
  p.out = out;
  // the epilogue's TMA stores: f32 rows 16-byte aligned (TIDE_LM_TMA_STORE=0,
  // read per call, keeps the per-lane stores for A/B runs)
  CUtensorMap om = ah;
  const char* senv = getenv("TIDE_LM_TMA_STORE");
  p.tma_store = 0;
  if (!(senv && senv[0] == '0') && n > 0 && ld_out % 4 == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0 &&
      make_map(&om, out, TIDE_F32, V, n, ld_out, 32, 32) == TIDE_OK)
    p.tma_store = 1;
  cudaGetLastError();
  const uint32_t smem = (uint32_t)p.stages * p.stage_bytes + (persist ? kLEpiBytes : 0u) + 256u + 1024u;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(lmhead_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(lmhead_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(lmhead2_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(lmhead2_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(lmhead2p_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(lmhead2p_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr = true;
  }
  const int64_t gy = (V + kLBN - 1) / kLBN;
  if (gy > 65535) return set_error(TIDE_ERR_UNSUPPORTED, "tide_lm_head: vocab too large (%lld)", (long long)V);
  cudaLaunchConfig_t cfg = {};
  const int64_t gx = pair ? 2 * ((n + 2 * kLBM - 1) / (2 * kLBM)) : (n + kLBM - 1) / kLBM;
  cfg.gridDim = dim3((unsigned)gx, (unsigned)gy, 1);
  if (persist) {
    // one pair per co-resident TPC slot, each walking pair tiles
    const int64_t tiles = ((n + 2 * kLBM - 1) / (2 * kLBM)) * gy;
    const int pairs = terms == 3 ? lm_pairs(lmhead2p_kernel<3>, smem, 1) : lm_pairs(lmhead2p_kernel<1>, smem, 0);
    cfg.gridDim = dim3((unsigned)(2 * std::min<int64_t>(tiles, pairs)), 1, 1);
  }
  cfg.blockDim = dim3(kLThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr1[1];
  attr1[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr1[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr1;
  cfg.numAttrs = 1;
  const cudaError_t e =
      persist ? (terms == 3 ? cudaLaunchKernelEx(&cfg, lmhead2p_kernel<3>, ah, al, bh, bl, om, p)
                            : cudaLaunchKernelEx(&cfg, lmhead2p_kernel<1>, ah, al, bh, bl, om, p))
      : pair ? (terms == 3 ? cudaLaunchKernelEx(&cfg, lmhead2_kernel<3>, ah, al, bh, bl, om, p)
                         : cudaLaunchKernelEx(&cfg, lmhead2_kernel<1>, ah, al, bh, bl, om, p))
           : (terms == 3 ? cudaLaunchKernelEx(&cfg, lmhead_kernel<3>, ah, al, bh, bl, om, p)
                         : cudaLaunchKernelEx(&cfg, lmhead_kernel<1>, ah, al, bh, bl, om, p));
  if (e != cudaSuccess) return set_error(TIDE_ERR_CUDA, "lmhead_kernel: %s", cudaGetErrorString(e));
  return check_launch("lmhead_kernel");
}

}  // namespace tide
