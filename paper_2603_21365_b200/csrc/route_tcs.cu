// K1s: split-K variant of K1 for small row counts (prefill shards of a few
// thousand tokens, the later links of the peeling chain).
//
// Same contract and numerics as route_tc.cu (ee/router_ops.py:68-87 score,
// ee/runtime.py:149,171 strict threshold, ee/router_ops.py:116-134 stable
// compaction).  With n = 4,096 rows the persistent K1 gives each of 148 SMs
// ~28 rows, so every SM re-reads all of W_down (1 MB at d = 4096) from L2 for
// 56 KB of activations: the launch is bound by W re-reads and their latency,
// not by HBM.  Here a 128-row tile is split over a cluster of KS CTAs along
// d: CTA `rank` streams h[tile, K_rank] and W[:, K_rank] once (W traffic =
// activation traffic), accumulates its partial D = h W^T in TMEM, and the
// cluster reduces the partials through distributed shared memory:
//   1. every CTA pushes column block c of its partial into the smem of the
//      CTA that owns c (remote st.shared::cluster, no round trips), plus its
//      partial sum of squares of each row to every CTA;
//   2. cluster barrier; each CTA sums its columns over the KS partials in
//      fixed rank order, applies scale / SiLU / w_up for them and pushes the
//      partial logit of every row to rank 0;
//   3. cluster barrier; rank 0 sums the KS partial logits (fixed order),
//      thresholds, and compacts the tile with the same ordered look-back as
//      K1 (partition = tile).
// Deterministic (fixed reduction orders); not bit-identical to K1 (different
// f32 summation order), both within the bf16 tolerance of the oracle.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "internal.h"

namespace tide {

namespace {

constexpr int kThreadsS = 320;  // producer, MMA issuer, 4 RMS / epilogue warps, 4 row gatherers
constexpr int kMaxStages = 8;
constexpr int kASlot = 128 * 128;  // 128 rows x 64 cols x 2 B

constexpr int kMaxTailC = 32;  // checkpoints of one chain-tail launch (grid.y)
struct TailLayers {
  int64_t l[kMaxTailC];
};

template <int NC>
struct WMaps {  // W_down tensor map per checkpoint (NC = 1: the plain route)
  CUtensorMap m[NC];
};

struct SplitParams {
  // chain tail (NC > 1): checkpoint c (see the grid order in the kernel) reads its rows from
  // h_bases[c] and w_ups[c] and writes scores[c * cap + position]; the launch
  // does nothing when the live count exceeds n_limit
  const uint8_t* h_bases[kMaxTailC];
  const float* w_ups[kMaxTailC];
  int64_t cap, n_limit, n_min;
  int32_t nc;  // checkpoints of a tail launch (NC > 1)
  int64_t n_host;
  const int64_t* n_dev;
  int64_t rows_total;
  int32_t d, b, bp, nk, ks, cw, stages;
  uint32_t idesc, tmem_cols, wslot, stage_bytes;
  uint32_t off_recv, off_plog, off_wup, off_bar, off_words, off_tmem;
  const int64_t* row_idx;
  int32_t ids_from_rows;
  const uint8_t* h_base;  // gathered rows are copied by the RMS warps (cp.async)
  int64_t ld_bytes;
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
  unsigned long long* dbg;  // optional per-CTA timeline (globaltimer ns), 24 slots per CTA
};

__device__ __forceinline__ unsigned long long gtimer_s() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TL(slot)                                                              \
  do {                                                                        \
    if (p.dbg) p.dbg[24 * blockIdx.x + (slot)] = gtimer_s();                  \
  } while (0)

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// shared::cta address -> the same offset in CTA `rank`'s shared memory
__device__ __forceinline__ uint32_t dsmem_addr(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
// bulk copy local smem -> smem of a CTA in the cluster, completing on its mbarrier
__device__ __forceinline__ void bulk_s2dsmem(uint32_t dst_cluster, uint32_t src_cta, uint32_t bytes,
                                             uint32_t bar_cluster) {
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dst_cluster),
      "r"(src_cta), "r"(bytes), "r"(bar_cluster)
      : "memory");
}
// split arrive / wait: every CTA of the cluster has started (its shared
// memory may be written remotely) once the wait returns
__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait;" ::: "memory"); }
// 16-byte async copy global -> shared (zero-fills when src_bytes == 0) and the
// mbarrier arrive that fires when this thread's prior cp.async have landed
__device__ __forceinline__ void cp_async16(void* dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
               "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void epi_bar() {  // the 4 epilogue warps only
  asm volatile("bar.sync 1, 128;" ::: "memory");
}

template <bool kBF16, int NC>
__global__ void __launch_bounds__(kThreadsS, 1)
    route_tcs_kernel(const __grid_constant__ CUtensorMap tm_h, const __grid_constant__ WMaps<NC> wm,
                     const __grid_constant__ SplitParams p) {
  // Chain tail (NC > 1): the grid is [X clusters per checkpoint] x C along x,
  // checkpoint fastest — cluster g serves checkpoint g % C and per-checkpoint
  // cluster g / C, so the clusters of the low (live) tiles of EVERY checkpoint
  // come first in launch order and the idle rest of a wide tail drains after.
  const uint32_t cl_lin = blockIdx.x / (uint32_t)p.ks;
  const int ck = NC > 1 ? (int)(cl_lin % (uint32_t)p.nc) : 0;
  const uint32_t cl_idx = NC > 1 ? cl_lin / (uint32_t)p.nc : cl_lin;     // cluster within its checkpoint
  const uint32_t cl_cnt = NC > 1 ? gridDim.x / (uint32_t)p.nc : gridDim.x;  // CTAs per checkpoint
  const CUtensorMap& tm_w = wm.m[ck];
  const uint8_t* const h_base = NC > 1 ? p.h_bases[ck] : p.h_base;
  const float* const w_up_c = NC > 1 ? p.w_ups[ck] : p.w_up;
  float* const scores_c = (NC > 1 && p.scores) ? p.scores + (size_t)ck * p.cap : p.scores;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  // partials of this CTA's rows from the ks ranks: [src][bp][R], then ss [src][R]
  float* recv = reinterpret_cast<float*>(smem + p.off_recv);
  // after the stream both live in the (drained) stage ring: this CTA's staged
  // partials [ks][bp][R] + ss [128], then the received ones
  float* stage_out = reinterpret_cast<float*>(smem);
  float* plog = reinterpret_cast<float*>(smem + p.off_plog);  // [column slice][R]
  float* sWup = reinterpret_cast<float*>(smem + p.off_wup);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.off_bar);
  uint64_t* full = bars;
  uint64_t* empty = bars + kMaxStages;
  uint64_t* acc_full = bars + 2 * kMaxStages;
  uint64_t* recv_full = acc_full + 1;
  uint32_t* words = reinterpret_cast<uint32_t*>(smem + p.off_words);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + p.off_tmem);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) TL(0);
  // The cluster (p.ks CTAs, the largest split the shape allows) is cut into
  // groups of ks CTAs, one 128-row tile per group, ks chosen HERE from the live
  // row count (n may come from device memory: later links of a peeling chain
  // split their few remaining tiles further).
  // PDL: the next launch may be scheduled as this grid's CTAs exit.  Setup
  // that touches no global memory (barriers, TMEM, tensor-map prefetch) runs
  // before griddepcontrol.wait, so it overlaps the previous link's tail; the
  // live count and row index it wrote are read after.
  if (threadIdx.x == 0) griddep_launch_dependents();
  if (NC > 1) {
    // tail: a cluster with no live tile leaves before any setup (it only counts
    // itself done for the workspace epoch)
    griddep_wait();
    const int64_t n0 = p.n_dev ? *p.n_dev : p.n_host;
    const int64_t nt0 = (n0 > p.n_limit || n0 < p.n_min) ? 0 : (n0 + 127) / 128;
    int ks0 = p.ks;
    while (ks0 > 1 && nt0 * ks0 > (int64_t)cl_cnt) ks0 >>= 1;
    if ((int64_t)cl_idx * (p.ks / ks0) >= nt0) {
      __syncthreads();
      if (threadIdx.x == 0) launch_done(p.ws);
      return;
    }
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tm_w);
    if (p.row_idx == nullptr) prefetch_tmap(&tm_h);
    for (int i = 0; i < p.stages; ++i) {
      // gathered: + one cp.async arrive per gather thread (warps 6-9 copy the rows)
      mbar_init(&full[i], p.row_idx != nullptr ? 1 + 128 : 1);
      mbar_init(&empty[i], 1 + 4);  // MMA commit + the 4 RMS warps
    }
    mbar_init(acc_full, 1);
    mbar_init(recv_full, 1);
    fence_mbar_init();
  }
  if (warp == 1) {
    tmem_alloc(tmem_slot, p.tmem_cols);
    tmem_relinquish();
  }
  griddep_wait();
  const uint32_t crank = cluster_rank();
  const int64_t n = p.n_dev ? *p.n_dev : p.n_host;
  // tail: outside [n_min, n_limit] -> idle
  const int64_t ntiles = (NC > 1 && (n > p.n_limit || n < p.n_min)) ? 0 : (n + 127) / 128;
  int ks = p.ks;
  while (ks > 1 && ntiles * ks > (int64_t)cl_cnt) ks >>= 1;
  const uint32_t rank = crank % (uint32_t)ks, gbase = crank - rank;
  const int64_t tile = (int64_t)cl_idx * (p.ks / ks) + crank / (uint32_t)ks;
  const int cw = p.bp / ks;
  const uint32_t tag = launch_tag(p.ws);
  if (tile >= ntiles) {
    // idle (its whole group is): still takes part in the two cluster barriers
    if (n == 0 && blockIdx.x == 0 && threadIdx.x == 0 && p.counts) {
      p.counts[0] = 0;
      p.counts[1] = 0;
    }
    // another group of this cluster is live: keep its barrier count (a wholly
    // idle cluster — most of a wide chain tail's grid when few rows are
    // left — leaves at once)
    if ((int64_t)cl_idx * (p.ks / ks) < ntiles) {
      cluster_arrive_relaxed();
      cluster_wait();
      cluster_arrive_relaxed();
      cluster_wait();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
      tc_fence_after();
      tmem_dealloc(*tmem_slot, p.tmem_cols);
    }
    if (threadIdx.x == 0) launch_done(p.ws);
    return;
  }
  const int64_t r0 = tile * 128;
  const int64_t r1 = (r0 + 128 < n) ? r0 + 128 : n;
  const int k0 = (int)((int64_t)p.nk * rank / ks), k1 = (int)((int64_t)p.nk * (rank + 1) / ks);
  const bool gathered = p.row_idx != nullptr;

  // Rank j owns rows [j R, (j+1) R) of the tile in the reduction; ranks whose
  // rows are all past the tile's live rows exchange and finish nothing (a chain
  // link with a handful of rows: one live rank instead of 16).
  const int Rr = 128 / ks;
  const int live_rows = (int)(r1 - r0);
  const bool live_rank = (int)rank * Rr < live_rows;
  if (warp == 0 && lane == 0 && live_rank) {
    // ks - 1 bulk copies of [bp + 1][128 / ks] floats land here (complete_tx may
    // precede this expect_tx: the phase needs the arrive as well)
    mbar_arrive_expect_tx(recv_full, (uint32_t)(ks - 1) * (uint32_t)(p.bp + 1) * (512u / ks));
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) TL(1);
  // Row ids needed on the tail (exit-layer scatter by the finishing threads,
  // index writes by warp 2) are loaded now, while the stream runs: no
  // dependent global loads after the reduction.
  const int64_t pr0e = r0 + (int64_t)rank * Rr;
  const int64_t pr1e = (pr0e + Rr < r1) ? pr0e + Rr : (pr0e < r1 ? r1 : pr0e);
  const int tf = threadIdx.x - 64;
  const int64_t fin_id =
      (gathered && tf >= 0 && tf < Rr && pr0e + tf < pr1e) ? p.row_idx[pr0e + tf] : pr0e + tf;
  int64_t wr_id[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    const int64_t r = pr0e + 32 * w + lane;
    wr_id[w] = (warp == 2 && gathered && p.ids_from_rows && 32 * w < Rr && r < pr1e) ? p.row_idx[r] : r;
  }

  if (warp == 0) {
    // ------------------------------------------------------------- producer
    if (lane == 0) {
      const uint64_t pol_h = policy_evict_first();
      const uint64_t pol_w = policy_evict_last();
      const uint32_t a_bytes = gathered ? 0u : (uint32_t)kASlot;
      int s = 0;
      uint32_t ph = 0;
      for (int kc = k0; kc < k1; ++kc) {
        mbar_wait(&empty[s], ph ^ 1u);
        uint8_t* sa = smem + (size_t)s * p.stage_bytes;
        uint8_t* sw = sa + kASlot;
        mbar_arrive_expect_tx(&full[s], a_bytes + p.wslot);
        if (!gathered) tma_load_2d(sa, &tm_h, &full[s], kc * 64, (int)r0, pol_h);
        tma_load_2d(sw, &tm_w, &full[s], kc * 64, 0, pol_w);
        if (++s == p.stages) { s = 0; ph ^= 1u; }
      }
      TL(2);
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------- MMA issuer
    const uint64_t desc_hi = sw128_kmajor_desc(0);
    int s = 0;
    uint32_t ph = 0;
    for (int kc = k0; kc < k1; ++kc) {
      mbar_wait(&full[s], ph);
      tc_fence_after();
      if (gathered) fence_proxy_async_smem();  // cp.async (generic proxy) -> MMA (async proxy)
      if (elect_one()) {
        const uint8_t* sa = smem + (size_t)s * p.stage_bytes;
        const uint64_t adesc = desc_hi | (uint64_t)((smem_u32(sa) & 0x3FFFFu) >> 4);
        const uint64_t bdesc = desc_hi | (uint64_t)((smem_u32(sa + kASlot) & 0x3FFFFu) >> 4);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          tc_mma_f16(tmem_base, adesc + 2 * k, bdesc + 2 * k, p.idesc, (kc != k0 || k != 0) ? 1u : 0u);
        tc_commit(&empty[s]);
        if (kc == k1 - 1) tc_commit(acc_full);
      }
      __syncwarp();
      if (++s == p.stages) { s = 0; ph ^= 1u; }
    }
  } else if (warp <= 5) {
    // ------------------------------------------------------------- RMS partials
    const int q = warp & 3;  // TMEM lane quadrant of this warp
    const int row = 32 * q + lane;
    const uint32_t swz = (uint32_t)(row & 7);
    float sq[4] = {0.f, 0.f, 0.f, 0.f};
    int s = 0;
    uint32_t ph = 0;
    for (int kc = k0; kc < k1; ++kc) {
      mbar_wait(&full[s], ph);
      const uint8_t* rp = smem + (size_t)s * p.stage_bytes + row * 128;
      uint4 u[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) u[j] = *reinterpret_cast<const uint4*>(rp + ((j ^ swz) << 4));
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        sq2_acc<kBF16>(u[j].x, sq[0], sq[1]);
        sq2_acc<kBF16>(u[j].y, sq[2], sq[3]);
        sq2_acc<kBF16>(u[j].z, sq[0], sq[1]);
        sq2_acc<kBF16>(u[j].w, sq[2], sq[3]);
      }
      // released once the values are consumed (an arrive right after the
      // LDS issue lets the refill race the reads, tools/stress_k1.py)
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (++s == p.stages) { s = 0; ph ^= 1u; }
    }
    const float ssp = (sq[0] + sq[1]) + (sq[2] + sq[3]);
    for (int i = threadIdx.x - 64; i < p.b; i += 128) sWup[i] = w_up_c[i];  // used after recv_full
    if (warp == 2 && lane == 0) TL(3);
    mbar_wait(acc_full, 0);  // every MMA retired: the stage ring is no longer read by the MMAs
    tc_fence_after();
    epi_bar();               // ... nor by the other RMS warps
    // the ring is drained: peers may copy their partials into it (recv) once
    // every CTA of the cluster got here (this also proves they all started)
    cluster_arrive_relaxed();
    if (warp == 2 && lane == 0) TL(4);
    // Stage this CTA's partials by destination: rank j owns rows [j R, (j+1) R)
    // and gets them as one contiguous [bp][R] block (+ their R partial ss).
    const int R = 128 / ks;
    const int jo = row / R, rr = row - jo * R;
    float* so = stage_out + (size_t)jo * p.bp * R + rr;
    const uint32_t taddr = tmem_base + ((uint32_t)(32 * q) << 16);
    const bool warp_live = (32 * q) / R * R < live_rows;  // some destination of this warp's rows is live
    for (int c0 = 0; warp_live && c0 < p.bp; c0 += 32) {
      uint32_t v[32];
      tmem_ld32(taddr + (uint32_t)c0, v);
      tmem_ld_wait();
      if (jo * R < live_rows) {
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) so[(size_t)(c0 + jj) * R] = __uint_as_float(v[jj]);
      }
    }
    float* stage_ss = stage_out + (size_t)p.bp * 128;
    stage_ss[row] = ssp;
    tc_fence_before();
    fence_proxy_async_smem();  // staged partials -> the bulk-copy (async) proxy
    epi_bar();
    cluster_wait();  // every ring in the cluster is drained
    if (warp == 2 && lane == 0) {
      const uint32_t blk = (uint32_t)p.bp * (uint32_t)R * 4u;
      for (uint32_t j = 0; j < (uint32_t)ks; ++j) {
        if (j == rank) continue;  // own rows are read from stage_out in place
        if ((int)j * R >= live_rows) break;  // dead ranks (and all after them) get nothing
        const uint32_t bar = dsmem_addr(smem_u32(recv_full), gbase + j);
        bulk_s2dsmem(dsmem_addr(smem_u32(recv) + rank * blk, gbase + j), smem_u32(stage_out) + j * blk,
                     blk, bar);
        bulk_s2dsmem(dsmem_addr(smem_u32(recv) + (uint32_t)ks * blk + rank * (uint32_t)R * 4u, gbase + j),
                     smem_u32(stage_ss + j * R), (uint32_t)R * 4u, bar);
      }
      TL(5);
    }
  } else if (gathered) {
    // ------------------------------------------------------------- row gatherers
    // Gathered rows by cp.async, warps 6-9 (one per SM sub-partition, 32
    // rows each), issued as far ahead as the ring allows: they wait only for
    // a stage's release (as the TMA producer does), not for the RMS reads of
    // the chunk before.  One instruction moves 4 rows x 128 B (8 lanes per
    // row, 16 B each) so every L2 request is whole sectors.  The byte
    // offsets of a lane's 8 rows stay in registers (-1 = past the tile's
    // live rows: left unwritten, never used).
    const int gq = warp - 6;
    const int sub = lane & 7, rg = lane >> 3;
    int64_t src_off[8];
#pragma unroll
    for (int it = 0; it < 8; ++it) {
      const int64_t r = r0 + 32 * gq + 4 * it + rg;
      src_off[it] = r < r1 ? p.row_idx[r] * p.ld_bytes : -1;
    }
    const int nkr = k1 - k0;
    for (int j = 0; j < nkr; ++j) {
      const int si = j % p.stages;
      mbar_wait(&empty[si], (((uint32_t)(j / p.stages)) & 1u) ^ 1u);
      uint8_t* dst = smem + (size_t)si * p.stage_bytes;
      const int64_t c = (int64_t)(k0 + j) * 64 + 8 * sub;  // this lane's 8 columns
      const bool in = c < p.d;
#pragma unroll
      for (int it = 0; it < 8; ++it) {
        const int rw = 32 * gq + 4 * it + rg;
        if (src_off[it] >= 0)
          cp_async16(dst + rw * 128 + ((sub ^ (rw & 7)) << 4), h_base + src_off[it] + (in ? c * 2 : 0),
                     in ? 16u : 0u);
      }
      cp_async_arrive_noinc(&full[si]);
    }
  }
  if (warp < 2 || warp > 5) {
    cluster_arrive_relaxed();  // (the epilogue warps arrive once the ring is drained ...
    cluster_wait();
    cluster_arrive_relaxed();  // ... and once the partials of their rows landed)
  }

  if (warp >= 2 && warp <= 5) {
    if (live_rank) mbar_wait(recv_full, 0);
    // every copy INTO this CTA has landed; once all CTAs arrive, every copy
    // FROM this CTA's smem has been read, so it may exit
    cluster_arrive_relaxed();
    if (threadIdx.x == 64) TL(6);
    // This CTA's rows [rank R, (rank+1) R): thread t sums column slice t / R
    // of row t % R over the ks partials (fixed order) and applies SiLU / w_up.
    const int R = 128 / ks;
    const int t = threadIdx.x - 64;
    const int rr = t % R, sl = t / R;
    // source j's [bp][R] block: received, or (j == rank) still in stage_out
    const float* own = stage_out + (size_t)rank * p.bp * R + rr;
    const float* rss = recv + (size_t)ks * p.bp * R + rr;
    float ss = 0.f;
    for (int j = 0; j < ks; ++j)
      ss += (j == (int)rank) ? stage_out[(size_t)p.bp * 128 + rank * R + rr] : rss[j * R];
    const float scale = rms_scale(ss, p.inv_d, p.eps);
    const float hs = 0.5f * scale;  // exact (power of two)
    const f32x2 hs2 = pack2(hs, hs);
    // 8 columns at a time: 8 independent sums, then 4 independent SiLU pairs
    // (one warp per SMSP here, so ILP is what hides the latency)
    f32x2 acc2 = 0ull, acc2b = 0ull;
    const int cbase = sl * cw;
    for (int cl0 = 0; live_rank && cl0 < cw; cl0 += 8) {
      if (cbase + cl0 >= p.b) break;
      float sum[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) sum[u] = 0.f;
      for (int j = 0; j < ks; ++j) {
        const float* src = ((j == (int)rank) ? own : recv + (size_t)j * p.bp * R + rr) +
                           (size_t)(cbase + cl0) * R;
#pragma unroll
        for (int u = 0; u < 8; ++u) sum[u] += src[u * R];
      }
#pragma unroll
      for (int u = 0; u < 8; u += 2) {
        const int c = cbase + cl0 + u;
        const float w0 = c < p.b ? sWup[c] : 0.f;
        const float w1 = c + 1 < p.b ? sWup[c + 1] : 0.f;
        const float a0 = c < p.b ? sum[u] : 0.f;
        const float a1 = c + 1 < p.b ? sum[u + 1] : 0.f;
        const f32x2 tt = ffma2(pack2(w0, w1), silu2_tanh(fmul2(pack2(a0, a1), hs2)), 0ull);
        if (u & 2) acc2b = fadd2(acc2b, tt);
        else acc2 = fadd2(acc2, tt);
      }
    }
    acc2 = fadd2(acc2, acc2b);
    float lo, hi;
    unpack2(acc2, lo, hi);
    plog[sl * R + rr] = lo + hi;
    epi_bar();
    if (threadIdx.x == 64) TL(10);
    // rows of this partition: threads t < R finish them (fixed slice order)
    const int64_t pr0 = r0 + (int64_t)rank * R;
    const int64_t pr1 = (pr0 + R < r1) ? pr0 + R : (pr0 < r1 ? r1 : pr0);
    bool ex = false;
    if (t < R) {
      float logit = 0.f;
      for (int j = 0; j < ks; ++j) logit += plog[j * R + t];
      const int64_t r = pr0 + t;
      if (r < pr1) {
        const float score = score_from_logit(logit);
        ex = score > p.theta;
        if (scores_c) scores_c[r] = score;
        if (p.logits) p.logits[r] = logit;
        if (p.mask) p.mask[r] = ex ? 1 : 0;
        if (ex && p.exit_layers) p.exit_layers[fin_id] = p.layer;
      }
    }
    const uint32_t bal = __ballot_sync(0xffffffffu, ex);
    if (lane == 0 && t < R) words[t >> 5] = bal;
    epi_bar();
    if (threadIdx.x == 64) TL(11);
    if (warp == 2 && (p.exit_idx || p.cont_idx || p.counts)) {
      const int nw = (R + 31) / 32;
      const uint32_t word = lane < nw ? words[lane] : 0u;
      const uint32_t cnt = __popc(word);
      uint32_t incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const uint32_t excl_w = incl - cnt;
      const uint32_t agg = __shfl_sync(0xffffffffu, incl, 31);
      const int64_t part = tile * ks + rank;
      const uint32_t E = lookback_exclusive(p.ws->status, tag, part, agg);
      if (lane == 0) TL(8);
      if (p.exit_idx || p.cont_idx) {
        const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          if (w >= nw) break;
          const uint32_t wd = __shfl_sync(0xffffffffu, word, w);
          const uint32_t pre = __shfl_sync(0xffffffffu, excl_w, w);
          const int64_t r = pr0 + 32 * w + lane;
          if (r < pr1) {
            const int64_t rank_e = (int64_t)E + pre + __popc(wd & lt);
            const int64_t id = wr_id[w];
            if ((wd >> lane) & 1u) {
              if (p.exit_idx) p.exit_idx[rank_e] = id;
            } else if (p.cont_idx) {
              p.cont_idx[r - rank_e] = id;
            }
          }
        }
      }
      if (part == ntiles * ks - 1 && lane == 0 && p.counts) {
        p.counts[0] = (int64_t)E + agg;
        p.counts[1] = n - ((int64_t)E + agg);
      }
    }
  }
  if (threadIdx.x == 64) TL(7);
  cluster_wait();  // every bulk copy out of this CTA's smem has been read

  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, p.tmem_cols);
  }
  if (threadIdx.x == 0) {
    TL(9);
    launch_done(p.ws);
  }
}

}  // namespace

namespace {

struct TcsLayout {
  int npad, bp, stages;
  uint32_t wslot, stage_bytes, off_recv, off_plog, off_wup, off_bar, off_words, off_tmem, smem_bytes;
};

// Shared-memory carve-up (depends on the bottleneck width only).  The staged
// and received partials reuse the drained stage ring; small fixed regions after.
bool tcs_layout(int b, TcsLayout& L) {
  L.npad = (b + 15) / 16 * 16;
  L.bp = (L.npad + 31) / 32 * 32;
  L.wslot = (uint32_t)L.npad * 128u;
  L.stage_bytes = (uint32_t)kASlot + L.wslot;
  const uint32_t part_bytes = ((uint32_t)(L.bp + 1) * 512u + 1023u) & ~1023u;
  const uint32_t fixed = 512u /*plog*/ + 1024u /*w_up*/ + 256u /*bars*/ + 64u /*words*/ + 16u;
  const int smem_cap = 227 * 1024 - 1024;
  L.stages = std::min<int>(kMaxStages, (int)((smem_cap - (int)fixed) / (int)L.stage_bytes));
  if (L.npad > 128 || L.stages < 2 || 2u * part_bytes > (uint32_t)L.stages * L.stage_bytes) return false;
  L.off_recv = part_bytes;
  L.off_plog = (uint32_t)L.stages * L.stage_bytes;
  L.off_wup = L.off_plog + 512u;
  L.off_bar = L.off_wup + 1024u;
  L.off_words = L.off_bar + 256u;
  L.off_tmem = L.off_words + 64u;
  L.smem_bytes = L.off_tmem + 16u + 1024u;
  return true;
}

void tcs_set_attrs(int dev) {
  static bool attr_set[64] = {false};
  if (!attr_set[dev & 63]) {
    // clusters of 16 (the chain's links with a handful of live rows) are non-portable
    auto set = [](auto k) {
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    };
    set(route_tcs_kernel<true, 1>);
    set(route_tcs_kernel<false, 1>);
    set(route_tcs_kernel<true, kMaxTailC>);
    set(route_tcs_kernel<false, kMaxTailC>);
    attr_set[dev & 63] = true;
  }
}

// Co-resident clusters of size c (a cluster lives in one GPC, so this is less
// than SMs / c: e.g. clusters of 8 leave several SMs of every GPC idle).
int tcs_max_clusters(int dev, int c, uint32_t smem) {
  static int cache[64][4][2];  // [dev][c = 2, 4, 8, 16][smem class]
  const int ci = c == 2 ? 0 : c == 4 ? 1 : c == 8 ? 2 : 3;
  const int si = smem > 200 * 1024 ? 1 : 0;
  int& mc = cache[dev & 63][ci][si];
  if (!mc) {
    tcs_set_attrs(dev);
    cudaLaunchConfig_t q = {};
    q.gridDim = dim3((unsigned)(c * 64), 1, 1);
    q.blockDim = dim3(kThreadsS, 1, 1);
    q.dynamicSmemBytes = smem;
    cudaLaunchAttribute qa[1];
    qa[0].id = cudaLaunchAttributeClusterDimension;
    qa[0].val.clusterDim.x = (unsigned)c;
    qa[0].val.clusterDim.y = 1;
    qa[0].val.clusterDim.z = 1;
    q.attrs = qa;
    q.numAttrs = 1;
    int v = 0;
    if (cudaOccupancyMaxActiveClusters(&v, route_tcs_kernel<true, 1>, &q) != cudaSuccess || v <= 0) {
      cudaGetLastError();
      v = sm_count(dev) / (2 * c);
    }
    mc = v;
    if (getenv("TIDE_DEBUG_PLAN"))
      fprintf(stderr, "[tide] clusters of %d x %u B smem: %d co-resident\n", c, smem, v);
  }
  return mc;
}

}  // namespace

// Launch plan: cluster size C (the largest split, 0 = use the persistent K1)
// and grid.  Dense launches (row count known on the host): the largest C whose
// co-resident clusters give every tile a full cluster.  Chain links (row
// count in device memory, usually far below the capacity `n`): the largest C
// whose co-resident CTAs cover every tile of the capacity at split 1 — the
// kernel picks the split from the live count (a link that still holds most
// rows runs at split 1-2 on fewer SMs; the links after a large exit wave run
// at split 8-16).  C in {2, 4, 8} (16 for chain links: a non-portable
// cluster size, so links with a handful of live rows stream 1/16 of W per
// CTA): bp / C a multiple of 8 and at least one 64-column k-chunk per rank.
int route_tcs_plan(const RouteArgs& a, int dev, int* grid) {
  // TIDE_SPLIT: "0" forces the persistent K1, 2/4/8 caps the split (tests, sweeps)
  const char* env = getenv("TIDE_SPLIT");
  const int cap = env ? atoi(env) : 16;
  TcsLayout L;
  if (cap <= 1 || a.n < 1 || !tcs_layout(a.b, L)) return 0;
  const int64_t tiles = (a.n + 127) / 128;
  const int nk = (a.d + 63) / 64;
  const bool live = a.n_dev != nullptr;
  for (int c = 16; c >= 2; c >>= 1) {
    if (c > cap || c > nk || L.bp % (8 * c) != 0 || (c == 16 && !live)) continue;
    const int64_t mc = tcs_max_clusters(dev, c, L.smem_bytes);
    if (!live && tiles <= mc) {
      *grid = (int)(tiles * c);
      return c;
    }
    if (live && tiles <= mc * c) {
      *grid = (int)(std::min<int64_t>(mc, tiles) * c);
      return c;
    }
  }
  return 0;
}

namespace {

// Common parameter block of a split-K launch (layout, numerics, outputs).
int tcs_params(const RouteArgs& a, int ks, SplitParams& p, TcsLayout& L) {
  if (!tcs_layout(a.b, L)) return set_error(TIDE_ERR_UNSUPPORTED, "split route: smem too small");
  const int npad = L.npad, bp = L.bp;
  p.n_host = a.n;
  p.n_dev = a.n_dev;
  p.rows_total = a.rows_total;
  p.d = a.d;
  p.b = a.b;
  p.bp = bp;
  p.nk = (a.d + 63) / 64;
  p.ks = ks;
  p.cw = bp / ks;
  p.idesc = f16_idesc(a.dtype == TIDE_BF16 ? 1 : 0, 128, npad);
  p.tmem_cols = bp <= 32 ? 32 : bp <= 64 ? 64 : 128;
  p.wslot = L.wslot;
  p.stage_bytes = L.stage_bytes;
  p.stages = L.stages;
  p.off_recv = L.off_recv;
  p.off_plog = L.off_plog;
  p.off_wup = L.off_wup;
  p.off_bar = L.off_bar;
  p.off_words = L.off_words;
  p.off_tmem = L.off_tmem;
  p.row_idx = a.row_idx;
  p.ids_from_rows = a.ids_from_rows;
  p.h_base = reinterpret_cast<const uint8_t*>(a.h);
  p.ld_bytes = a.ld_h * 2;
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
  const int64_t tiles = (a.n + 127) / 128;
  if (tiles * ks > kMaxParts / 2) return set_error(TIDE_ERR_UNSUPPORTED, "too many rows for one launch");
  return TIDE_OK;
}

template <int NC>
int tcs_launch(const RouteArgs& a, const SplitParams& p, const WMaps<NC>& wm, uint32_t smem_bytes,
               int ks, int grid, int ny, cudaStream_t stream, const char* what) {
  CUtensorMap tm_h;
  const int64_t hrows = a.row_idx ? a.rows_total : std::max<int64_t>(a.n, 1);
  int rc;
  if ((rc = make_map(&tm_h, a.h, a.dtype, a.d, hrows, a.ld_h, 64, 128))) return rc;
  int dev = 0;
  cudaGetDevice(&dev);
  tcs_set_attrs(dev);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid, (unsigned)ny, 1);
  cfg.blockDim = dim3(kThreadsS, 1, 1);
  cfg.dynamicSmemBytes = smem_bytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)ks;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  {
    const char* env = getenv("TIDE_PDL");  // read per call
    cfg.numAttrs = (env && env[0] == '0') ? 1 : 2;
  }
  cudaError_t e;
  if (a.dtype == TIDE_BF16)
    e = cudaLaunchKernelEx(&cfg, route_tcs_kernel<true, NC>, tm_h, wm, p);
  else
    e = cudaLaunchKernelEx(&cfg, route_tcs_kernel<false, NC>, tm_h, wm, p);
  if (e != cudaSuccess) return set_error(TIDE_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return check_launch(what);
}

// Chain tail, step 2: first firing checkpoint of every live row (per-token
// rule of ee/runtime.py:166-178 over the tail's checkpoints, in order) and the
// live count the following links read (0 when the tail handled the rows).
// Dense form (n_dev == row_idx == NULL): rows 0 .. cap-1, row id = position.
__global__ void chain_resolve_kernel(const float* scores, int64_t cap, int nc, TailLayers layers,
                                     float theta, const int64_t* n_dev, int64_t n_min,
                                     int64_t n_limit,
                                     const int64_t* row_idx, int64_t* exit_layers,
                                     int64_t* tail_count, unsigned long long cond) {
  griddep_wait();  // the scoring launch before it may run under PDL
  const int64_t n = n_dev ? *n_dev : cap;
  const bool handled = n >= n_min && n <= n_limit;
  if (blockIdx.x == 0 && threadIdx.x == 0 && tail_count) {
    *tail_count = handled ? 0 : n;
    // in a captured CUDA graph: the IF node holding the remaining links runs
    // only when the tail did not handle the rows (tide_capture_cond_*)
    if (cond) cudaGraphSetConditional((cudaGraphConditionalHandle)cond, handled ? 0u : 1u);
  }
  if (!handled) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rid = row_idx ? row_idx[i] : i;
    // 8 checkpoints' scores in flight per step (the loads are independent)
    for (int c0 = 0; c0 < nc; c0 += 8) {
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = c0 + u < nc ? __ldcg(scores + (size_t)(c0 + u) * cap + i) : 0.f;
      int hit = -1;
#pragma unroll
      for (int u = 7; u >= 0; --u)
        if (c0 + u < nc && v[u] > theta) hit = c0 + u;
      if (hit >= 0) {
        exit_layers[rid] = layers.l[hit];
        break;
      }
    }
  }
}

}  // namespace

int route_tcs_launch(const RouteArgs& a, cudaStream_t stream, int ks, int grid) {
  SplitParams p{};
  TcsLayout L;
  int rc;
  if ((rc = tcs_params(a, ks, p, L))) return rc;
  WMaps<1> wm;
  if ((rc = make_map(&wm.m[0], a.w_down, a.dtype, a.d, a.b, a.d, 64, L.npad))) return rc;
  return tcs_launch<1>(a, p, wm, L.smem_bytes, ks, grid, 1, stream, "route_tcs_kernel");
}

int route_tcs_tail_launch(const RouteArgs& a, int C, const void* const* h_ptrs,
                          const void* const* w_ptrs, const float* const* wup_ptrs,
                          const int64_t* layers, int64_t n_limit, int64_t* tail_count,
                          unsigned long long cond, cudaStream_t stream) {
  if (C < 1 || C > kMaxTailC) return set_error(TIDE_ERR_ARG, "tail: C must be in [1, %d]", kMaxTailC);
  if (!a.row_idx || !a.n_dev || !a.scores || !a.exit_layers || !tail_count)
    return set_error(TIDE_ERR_ARG, "tail: row_idx, n_dev, scores, exit_layers, tail_count required");
  int dev = 0;
  cudaGetDevice(&dev);
  // One wave for every checkpoint at once: X CTAs per checkpoint (a multiple
  // of the cluster size), and at most X tiles of live rows (n_limit clamp).
  TcsLayout L0;
  if (!tcs_layout(a.b, L0)) return set_error(TIDE_ERR_UNSUPPORTED, "tail: smem too small");
  const int nk = (a.d + 63) / 64;
  const int per = std::max(1, sm_count(dev) / C);
  int ks = 1;
  // Cluster size cap 2 (TIDE_TAIL_KS overrides): the tail's rows are few but
  // its checkpoints many, so more clusters per checkpoint, each streaming a
  // longer K range, beat wide splits (tools/tail_sweep.py: config 2
  // 0.109 -> 0.093 ms, config 5 0.252 -> 0.183 ms against a cap of 16).
  const char* kenv = getenv("TIDE_TAIL_KS");
  const int kcap = kenv ? atoi(kenv) : 2;
  for (int c = 16; c >= 2; c >>= 1)
    if (c <= kcap && c <= per && c <= nk && L0.bp % (8 * c) == 0 &&
        tcs_max_clusters(dev, c, L0.smem_bytes) * c >= (per / c) * c * 1) {
      ks = c;
      break;
    }
  int grid = std::max(ks, per / ks * ks);
  if (n_limit >= a.n) {
    // wide tail (n_limit >= capacity): every live count is handled; one
    // cluster per live tile and checkpoint, in as many waves as it takes
    // (clusters past the live tiles exit at once)
    grid = std::max<int64_t>(grid, (a.n + 127) / 128 * ks);
    n_limit = a.n;
  } else {
    n_limit = std::min<int64_t>(n_limit, (int64_t)grid * 128);
  }
  SplitParams p{};
  TcsLayout L;
  int rc;
  if ((rc = tcs_params(a, ks, p, L))) return rc;
  p.cap = a.n;
  p.n_limit = n_limit;
  p.n_min = a.n_min;
  p.logits = nullptr;  // scores only; no mask / compaction / exit layers in the routing step
  p.mask = nullptr;
  p.exit_idx = nullptr;
  p.cont_idx = nullptr;
  p.exit_layers = nullptr;
  p.counts = nullptr;
  static WMaps<kMaxTailC> wm;  // host staging (copied into the launch parameters)
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  for (int c = 0; c < C; ++c) {
    p.h_bases[c] = reinterpret_cast<const uint8_t*>(h_ptrs[c]);
    p.w_ups[c] = wup_ptrs[c];
    if ((rc = make_map(&wm.m[c], w_ptrs[c], a.dtype, a.d, a.b, a.d, 64, L.npad))) return rc;
  }
  p.nc = C;
  if ((rc = tcs_launch<kMaxTailC>(a, p, wm, L.smem_bytes, ks, grid * C, 1, stream,
                                  "route_tcs_kernel (tail)")))
    return rc;
  return chain_resolve_launch((const float*)a.scores, a.n, C, layers, a.theta, a.n_dev, a.n_min,
                              n_limit,
                              a.row_idx, a.exit_layers, tail_count, cond, stream);
}

int chain_resolve_launch(const float* scores, int64_t cap, int C, const int64_t* layers,
                         float theta, const int64_t* n_dev, int64_t n_min, int64_t n_limit,
                         const int64_t* row_idx, int64_t* exit_layers, int64_t* tail_count,
                         unsigned long long cond, cudaStream_t stream) {
  if (C < 1 || C > kMaxTailC) return set_error(TIDE_ERR_ARG, "resolve: C must be in [1, %d]", kMaxTailC);
  TailLayers tl{};
  for (int c = 0; c < C; ++c) tl.l[c] = layers[c];
  // plain launch (full dependency): a conditional graph node may follow it
  const unsigned nb = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n_limit + 255) / 256, 148));
  chain_resolve_kernel<<<nb, 256, 0, stream>>>(scores, cap, C, tl, theta, n_dev, n_min, n_limit, row_idx,
                                               exit_layers, tail_count, cond);
  return check_launch("chain_resolve_kernel");
}

}  // namespace tide
