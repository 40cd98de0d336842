// K5: the decode step — every checkpoint router for n <= 16 rows in ONE
// launch, plus the exit resolution of posthoc_select (ee/runtime.py:151-178).
//
// The step is bound by W_down bytes (C x b x d x e: 9.4 MB for Qwen3-8B's 9
// checkpoints), not by the few hidden rows, and it is short enough that every
// serial memory round trip shows.  CTA (checkpoint c, slice s) owns a column
// slice of W_c (all b rows) and of the n hidden rows:
//   1. every thread issues its share of both slices as 16-byte cp.async at
//      once (one round trip);
//   2. partial pre-activations a[j][r] over the slice: bf16 / f16 on tcgen05
//      (A = W slice, M = 128 rows of W per MMA, B = hidden rows, N = 16,
//      accumulator in TMEM), f32 on CUDA cores;
//   3. the partial tile goes to the workspace; the last CTA of a checkpoint
//      (atomic ticket) sums the tiles in fixed slice order (all loads in
//      flight at once) and applies RMS scale / SiLU / w_up / f64 sigmoid;
//   4. the last checkpoint to finish resolves per-token / batch-unanimous
//      exits.
// Deterministic: every reduction has a fixed order.
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "internal.h"

namespace tide {

namespace {

constexpr int kDThreads = 256;
constexpr int kDWarps = kDThreads / 32;
constexpr int kDMaxRows = TIDE_MAX_DECODE_ROWS;
constexpr int kDMaxC = kMaxTickets;
constexpr int kDMaxB = 256;

constexpr int kDMaxKc = 16;  // 64-column k-chunks per slice (TMA path)

struct DecParams {
  // W of every checkpoint stacked as [C * b, d] (the runtime's decode plan):
  // one tensor map, one TMA box (64 columns x 128 rows) per k-chunk and
  // 128-row block; use_tma = 0 falls back to per-thread cp.async
  CUtensorMap wmap;
  int32_t use_tma;
  const void* h[kDMaxC];
  const void* w[kDMaxC];
  const float* wup[kDMaxC];
  int64_t layers[kDMaxC];
  int32_t C, d, b, S, cs;  // checkpoints, width, bottleneck, slices per checkpoint, slice columns
  int64_t ld_h, n, k_min;
  int32_t mode;
  float eps, inv_d, theta;
  float* scores;
  float* logits;
  int64_t* exit_layers;
  int64_t* exit_count;
  Workspace* ws;
  unsigned long long* dbg;  // optional per-CTA timeline (globaltimer ns), 24 slots per CTA
};

__device__ __forceinline__ unsigned long long dgt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define DTL(slot)                                                             \
  do {                                                                        \
    if (p.dbg && threadIdx.x == 0) p.dbg[24 * blockIdx.x + (slot)] = dgt();   \
  } while (0)

__device__ __forceinline__ void cp_async16_zfill(void* dst, const void* src, bool ok) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
               "r"(ok ? 16u : 0u)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ uint32_t dsmem_addr(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_dsmem_f32(uint32_t addr, float v) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait;" ::: "memory"); }
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}

template <typename T>
__device__ __forceinline__ void lds_vec(const T* p, float (&f)[16 / sizeof(T)]) {
  unpack16(*reinterpret_cast<const uint4*>(p), f, (const T*)nullptr);
}

// Step 5 (+ the exit resolution), shared: one CTA per checkpoint holds the
// row logits in sLogit[NR]; scores out, then the last checkpoint to finish
// (atomic ticket) resolves per-token / batch-unanimous exits.
template <int NR>
__device__ __forceinline__ void decode_finish(const DecParams& p, int c, const float* sLogit,
                                              unsigned int* last_s, bool reset_ticket = true) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = (int)p.n;
  if (threadIdx.x < NR && threadIdx.x < n) {
    const int r = threadIdx.x;
    const float t = sLogit[r];
    const float score = score_from_logit(t);
    if (p.scores) p.scores[(int64_t)c * n + r] = score;
    if (p.logits) p.logits[(int64_t)c * n + r] = t;
    p.ws->dec_scores[c * kDMaxRows + r] = score;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    if (reset_ticket) p.ws->tickets[c] = 0;  // reset for the next launch (graph replay safe)
    const unsigned int prev = atomicAdd(&p.ws->ticket, 1u);
    *last_s = (prev == (unsigned int)(p.C - 1)) ? 2u : 0u;
  }
  __syncthreads();
  DTL(5);
  if (*last_s != 2u || warp != 0) return;
  __threadfence();
  // exit resolution: lanes = rows; scores of 8 checkpoints in flight at once
  const int r = lane;
  int64_t exit_layer = TIDE_NO_EXIT;
  bool done = false;
  for (int cb = 0; cb < p.C && !done; cb += 8) {
    float v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      v[u] = (cb + u < p.C && r < n) ? __ldcg(&p.ws->dec_scores[(cb + u) * kDMaxRows + r]) : 0.f;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int cc = cb + u;
      if (done || cc >= p.C || p.layers[cc] < p.k_min) continue;
      if (p.mode == TIDE_MODE_PER_TOKEN) {
        if (r < n && exit_layer == TIDE_NO_EXIT && v[u] > p.theta) exit_layer = p.layers[cc];
        done = __all_sync(0xffffffffu, r >= n || exit_layer != TIDE_NO_EXIT);
      } else if (__all_sync(0xffffffffu, r >= n || v[u] > p.theta)) {
        exit_layer = p.layers[cc];
        done = true;
      }
    }
  }
  if (r < n && p.exit_layers) p.exit_layers[r] = exit_layer;
  const uint32_t cnt = __popc(__ballot_sync(0xffffffffu, r < n && exit_layer != TIDE_NO_EXIT));
  if (lane == 0) {
    if (p.exit_count) p.exit_count[0] = cnt;
    p.ws->ticket = 0;
  }
  DTL(6);
}

// Steps 3-4, shared by both kernels.  sRes [b][NR] + sSS [NR] hold this CTA's
// partial tile; sWup [b] the checkpoint's w_up; sLog [kDWarps][NR] scratch.
template <int NR>
__device__ __forceinline__ void decode_tail(const DecParams& p, int c, int s, float* sRes, float* sWup,
                                            float* sLog, unsigned int* last_s) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = p.b;
  const int tile = b * NR + NR;
  float* sSS = sRes + (size_t)b * NR;
  float* part = p.ws->partials;
  float* mine = part + ((size_t)c * p.S + s) * tile;
  for (int i = threadIdx.x; i < tile; i += kDThreads) mine[i] = sRes[i];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int prev = atomicAdd(&p.ws->tickets[c], 1u);
    *last_s = (prev == (unsigned int)(p.S - 1)) ? 1u : 0u;
  }
  __syncthreads();
  DTL(3);
  if (!*last_s) return;
  __threadfence();
  // totals over the S slices, fixed order: thread t owns float4 group t of the
  // [b][NR] tile (b * NR / 4 <= 1024 groups) and issues all its S loads at
  // once; threads < NR also sum the ss column
  const float* base = part + (size_t)c * p.S * tile;
  const int G = b * NR / 4;
  for (int g = threadIdx.x; g < G + NR; g += kDThreads) {
    if (g < G) {
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int sl0 = 0; sl0 < p.S; sl0 += 16) {
        float4 v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u)
          v[u] = (sl0 + u < p.S) ? __ldcg(reinterpret_cast<const float4*>(base + (size_t)(sl0 + u) * tile) + g)
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          acc.x += v[u].x;
          acc.y += v[u].y;
          acc.z += v[u].z;
          acc.w += v[u].w;
        }
      }
      reinterpret_cast<float4*>(sRes)[g] = acc;
    } else {
      const int r = g - G;
      float t = 0.f;
      for (int sl = 0; sl < p.S; ++sl) t += __ldcg(base + (size_t)sl * tile + (size_t)b * NR + r);
      sSS[r] = t;
    }
  }
  __syncthreads();
  DTL(4);
  // logit[r] = sum_j w_up[j] * silu(scale_r * a[j][r]); lanes (sub, r)
  {
    constexpr int JL = 32 / NR;
    const int sub = lane / NR, r = lane - sub * NR;
    const float scale = rms_scale(sSS[r], p.inv_d, p.eps);
    float t = 0.f;
#pragma unroll 4
    for (int j = warp * JL + sub; j < b; j += kDWarps * JL)
      t = fmaf(sWup[j], silu_f32(__fmul_rn(sRes[(size_t)j * NR + r], scale)), t);
#pragma unroll
    for (int o = 16; o >= NR; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane < NR) sLog[warp * NR + lane] = t;
  }
  __syncthreads();
  if (threadIdx.x < NR) {
    float t = 0.f;
    for (int w = 0; w < kDWarps; ++w) t += sLog[w * NR + threadIdx.x];
    sLog[kDWarps * NR + threadIdx.x] = t;
  }
  __syncthreads();
  decode_finish<NR>(p, c, sLog + kDWarps * NR, last_s);
}

// ---------------------------------------------------------------------------
// bf16 / f16: tcgen05.  Slice = nkc 64-column k-chunks.  smem (1024-aligned):
//   sA [nkc][MT][128 rows x 128 B]  W slice, SW128 K-major (MT = ceil(b / 128))
//   sB [nkc][16 rows x 128 B]       hidden rows (zero past n), SW128 K-major
//   then sRes [b][NR] + sSS [NR], sLog [8][NR], sWup [b], barrier, TMEM slot
// ---------------------------------------------------------------------------
// kClu: the S slice-CTAs of a checkpoint form one thread-block cluster and
// reduce their partial tiles through distributed shared memory (two cluster
// barriers) instead of partials -> workspace -> ticket -> last-CTA re-read.
template <bool kBF16, int NR, bool kClu>
__global__ void __launch_bounds__(kDThreads, 1) decode_tc_kernel(const __grid_constant__ DecParams p) {
  using T = typename std::conditional<kBF16, __nv_bfloat16, __half>::type;
  constexpr int V = 8;
  extern __shared__ uint8_t dsm_raw[];
  uint8_t* dsm = dsm_raw + ((1024u - (smem_u32(dsm_raw) & 1023u)) & 1023u);
  __shared__ unsigned int last_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x / p.S, s = blockIdx.x - c * p.S;
  const int n = (int)p.n, b = p.b;
  const int MT = (b + 127) / 128;
  const int nkc = p.cs / 64;
  const int c0 = s * p.cs;
  uint8_t* sA = dsm;
  uint8_t* sB = sA + (size_t)nkc * MT * 16384;
  float* sRes = reinterpret_cast<float*>(sB + (size_t)nkc * 2048);
  float* sLog = sRes + (size_t)b * NR + NR;
  float* sWup = sLog + (kDWarps + 1) * NR;
  uint64_t* mma_done = reinterpret_cast<uint64_t*>(sWup + ((b + 1) & ~1));
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mma_done + 1);
  DTL(0);
  if (kClu) cluster_arrive_relaxed();  // this CTA's smem exists (peers write it after step 3a)

  // 1. one round trip: W slice + hidden slice as 16-byte pieces into the
  //    swizzled K-major layout (piece q of row j at ((q ^ (j & 7)) << 4))
  const T* W = reinterpret_cast<const T*>(p.w[c]);
  const T* H = reinterpret_cast<const T*>(p.h[c]);
  const int per_row = nkc * 8;
  uint64_t* wfull = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(tmem_slot) + 8);  // [kDMaxKc]
  if (p.use_tma) {
    // W slice by TMA, one barrier per k-chunk: the MMAs of early chunks run
    // while later chunks land
    if (threadIdx.x == 0) {
      for (int kc = 0; kc < nkc; ++kc) mbar_init(&wfull[kc], 1);
      fence_mbar_init();
      const uint64_t pol = policy_evict_last();  // every decode step re-reads it
      for (int kc = 0; kc < nkc; ++kc) {
        mbar_arrive_expect_tx(&wfull[kc], (uint32_t)MT * 16384u);
        for (int mt = 0; mt < MT; ++mt)
          tma_load_2d(sA + ((size_t)kc * MT + mt) * 16384, &p.wmap, &wfull[kc], c0 + kc * 64,
                      c * b + mt * 128, pol);
      }
    }
  } else {
    for (int i = threadIdx.x; i < b * per_row; i += kDThreads) {
      const int j = i / per_row, rem = i - j * per_row, kc = rem >> 3, q = rem & 7;
      const int col = c0 + kc * 64 + q * 8;
      const bool in = col < p.d;
      uint8_t* dst = sA + ((size_t)kc * MT + (j >> 7)) * 16384 + (j & 127) * 128 + ((q ^ (j & 7)) << 4);
      cp_async16_zfill(dst, W + (int64_t)j * p.d + (in ? col : 0), in);
    }
  }
  for (int i = threadIdx.x; i < 16 * per_row; i += kDThreads) {
    const int r = i / per_row, rem = i - r * per_row, kc = rem >> 3, q = rem & 7;
    const int col = c0 + kc * 64 + q * 8;
    const bool in = col < p.d && r < n;
    uint8_t* dst = sB + (size_t)kc * 2048 + r * 128 + ((q ^ (r & 7)) << 4);
    cp_async16_zfill(dst, H + (in ? (int64_t)r * p.ld_h + col : 0), in);
  }
  for (int j = threadIdx.x; j < b; j += kDThreads) sWup[j] = p.wup[c][j];
  if (threadIdx.x == 0) {
    mbar_init(mma_done, 1);
    fence_mbar_init();
  }
  if (warp == 1) {
    tmem_alloc(tmem_slot, 32);
    tmem_relinquish();
  }
  cp_async_wait_all();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  DTL(1);

  // 2. MMAs (warp 0, one elected lane): D[mt] (128 x 16) += A[kc][mt] . B[kc]^T
  if (warp == 0) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // cp.async -> MMA operands
    tc_fence_after();
    if (elect_one()) {
      const uint64_t desc_hi = sw128_kmajor_desc(0);
      const uint32_t idesc = f16_idesc(kBF16 ? 1 : 0, 128, 16);
      for (int kc = 0; kc < nkc; ++kc) {
        if (p.use_tma) {
          mbar_wait(&wfull[kc], 0);
          tc_fence_after();
        }
        for (int mt = 0; mt < MT; ++mt) {
          const uint64_t ad =
              desc_hi | (uint64_t)((smem_u32(sA + ((size_t)kc * MT + mt) * 16384) & 0x3FFFFu) >> 4);
          const uint64_t bd = desc_hi | (uint64_t)((smem_u32(sB + (size_t)kc * 2048) & 0x3FFFFu) >> 4);
#pragma unroll
          for (int k = 0; k < 4; ++k)
            tc_mma_f16(tmem_base + (uint32_t)(mt * 16), ad + 2 * k, bd + 2 * k, idesc, (kc | k) != 0);
        }
      }
      tc_commit(mma_done);
    }
    __syncwarp();
  } else if (warp >= 4) {
    // partial sums of squares of the hidden rows (8 threads per row, fixed order)
    const int t = threadIdx.x - 128, r = t >> 3, q = t & 7;
    float ss = 0.f;
    if (r < NR) {
      for (int kc = 0; kc < nkc; ++kc) {
        float f[V];
        lds_vec<T>(reinterpret_cast<const T*>(sB + (size_t)kc * 2048 + r * 128 + ((q ^ (r & 7)) << 4)), f);
#pragma unroll
        for (int e = 0; e < V; ++e) ss = fmaf(f[e], f[e], ss);
      }
    }
    ss += __shfl_xor_sync(0xffffffffu, ss, 1);
    ss += __shfl_xor_sync(0xffffffffu, ss, 2);
    ss += __shfl_xor_sync(0xffffffffu, ss, 4);
    if (r < NR && q == 0) sRes[(size_t)b * NR + r] = ss;
  }
  // 3a. accumulators -> sRes[j][r] (warps 0-3: TMEM lane quadrant = warp)
  if (warp < 4) {
    mbar_wait(mma_done, 0);
    tc_fence_after();
    for (int mt = 0; mt < MT; ++mt) {
      uint32_t v[16];
      tmem_ld16(tmem_base + ((uint32_t)(32 * warp) << 16) + (uint32_t)(mt * 16), v);
      tmem_ld_wait();
      const int j = mt * 128 + 32 * warp + lane;
      if (j < b) {
#pragma unroll
        for (int r = 0; r < NR; ++r) sRes[(size_t)j * NR + r] = __uint_as_float(v[r]);
      }
    }
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 32);
  }
  DTL(2);
  if (!kClu) {
    decode_tail<NR>(p, c, s, sRes, sWup, sLog, &last_s);
    return;
  }
  // 3b. DSMEM reduction.  Rank q owns units [q U, (q+1) U); every CTA stores its
  // partial of those units into q's recv[src = own rank], and its partial sum
  // of squares into every CTA's recv_ss[src].
  const uint32_t rank = (uint32_t)s;  // cluster dims (S, 1, 1), blockIdx.x = c S + s
  const int S = p.S, U = (b + S - 1) / S;
  float* recv = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(tmem_slot) + 8 + 8 * kDMaxKc);
  float* recv_ss = recv + (size_t)S * U * NR;
  float* plog = recv_ss + (size_t)S * NR;
  float* yv = plog + (size_t)S * NR;
  const float* sSS = sRes + (size_t)b * NR;
  cluster_wait();  // every peer started
  for (int i = threadIdx.x; i < b * NR; i += kDThreads) {
    const int j = i / NR, r = i - j * NR;
    const int q = j / U, uu = j - q * U;
    st_dsmem_f32(dsmem_addr(smem_u32(recv + ((size_t)rank * U + uu) * NR + r), (uint32_t)q), sRes[i]);
  }
  for (int i = threadIdx.x; i < S * NR; i += kDThreads) {
    const int q = i / NR, r = i - q * NR;
    st_dsmem_f32(dsmem_addr(smem_u32(recv_ss + rank * NR + r), (uint32_t)q), sSS[r]);
  }
  cluster_sync_all();  // release / acquire: every partial landed
  DTL(3);
  // 4. this CTA's units: totals over the S slices (fixed order), scale,
  //    SiLU, w_up; partial logit per row -> rank 0's plog[rank]
  for (int i = threadIdx.x; i < U * NR; i += kDThreads) {
    const int uu = i / NR, r = i - uu * NR;
    const int j = (int)rank * U + uu;
    float a = 0.f, ss = 0.f;
    for (int src = 0; src < S; ++src) {
      a += recv[((size_t)src * U + uu) * NR + r];
      ss += recv_ss[src * NR + r];
    }
    const float scale = rms_scale(ss, p.inv_d, p.eps);
    yv[i] = j < b ? __fmul_rn(sWup[j], silu_f32(__fmul_rn(a, scale))) : 0.f;
  }
  __syncthreads();
  if (threadIdx.x < NR) {
    float t = 0.f;
    for (int uu = 0; uu < U; ++uu) t += yv[uu * NR + threadIdx.x];
    st_dsmem_f32(dsmem_addr(smem_u32(plog + rank * NR + threadIdx.x), 0u), t);
  }
  cluster_sync_all();  // rank 0 holds every partial logit; no DSMEM traffic after this
  DTL(4);
  if (rank != 0) return;
  if (threadIdx.x < NR) {
    float t = 0.f;
    for (int src = 0; src < S; ++src) t += plog[src * NR + threadIdx.x];
    yv[threadIdx.x] = t;
  }
  __syncthreads();
  decode_finish<NR>(p, c, yv, &last_s, false);
}

// ---------------------------------------------------------------------------
// f32: CUDA cores.  smem: sW [b][cs], sH [NR][cs], then the tail buffers.
// ---------------------------------------------------------------------------
template <int NR>
__global__ void __launch_bounds__(kDThreads) decode_f32_kernel(const __grid_constant__ DecParams p) {
  using T = float;
  constexpr int V = 4;
  extern __shared__ uint8_t dsm[];
  __shared__ unsigned int last_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x / p.S, s = blockIdx.x - c * p.S;
  const int n = (int)p.n, b = p.b;
  const int c0 = s * p.cs;
  const int ncol = min(p.cs, p.d - c0);
  const int nch = ncol / V;
  T* sW = reinterpret_cast<T*>(dsm);         // [b][cs]
  T* sH = sW + (size_t)b * p.cs;             // [NR][cs]
  float* sRes = sH + (size_t)NR * p.cs;      // [b][NR] + [NR]
  float* sLog = sRes + (size_t)b * NR + NR;  // [8][NR]
  float* sWup = sLog + (kDWarps + 1) * NR;   // [b]
  DTL(0);
  const T* W = reinterpret_cast<const T*>(p.w[c]);
  const T* H = reinterpret_cast<const T*>(p.h[c]);
  for (int i = threadIdx.x; i < b * nch; i += kDThreads) {
    const int j = i / nch, k = i - j * nch;
    cp_async16_zfill(sW + (size_t)j * p.cs + k * V, W + (int64_t)j * p.d + c0 + k * V, true);
  }
  for (int i = threadIdx.x; i < NR * nch; i += kDThreads) {
    const int r = i / nch, k = i - r * nch;
    cp_async16_zfill(sH + (size_t)r * p.cs + k * V, H + (int64_t)(r < n ? r : 0) * p.ld_h + c0 + k * V,
                     r < n);
  }
  for (int j = threadIdx.x; j < b; j += kDThreads) sWup[j] = p.wup[c][j];
  cp_async_wait_all();
  __syncthreads();
  DTL(1);
  // Warp w owns W rows j0.. in batches of WB; lane l owns 16-byte chunks l,
  // l + 32, ...; WB x NR = 32 dot products per lane, then a butterfly
  // transpose-reduce (each step keeps the half selected by the lane's bit)
  // leaves quantity l = jj * NR + r, summed over the warp, in lane l.
  constexpr int WB = 32 / NR;
  for (int j0 = warp * WB; j0 < b; j0 += kDWarps * WB) {
    float acc[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) acc[i] = 0.f;
    for (int k = lane; k < nch; k += 32) {
      float wf[WB][V];
#pragma unroll
      for (int jj = 0; jj < WB; ++jj) {
        if (j0 + jj < b) {
          lds_vec<T>(sW + (size_t)(j0 + jj) * p.cs + k * V, wf[jj]);
        } else {
#pragma unroll
          for (int e = 0; e < V; ++e) wf[jj][e] = 0.f;
        }
      }
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        float hf[V];
        lds_vec<T>(sH + (size_t)r * p.cs + k * V, hf);
#pragma unroll
        for (int jj = 0; jj < WB; ++jj) {
          float t = acc[jj * NR + r];
#pragma unroll
          for (int e = 0; e < V; ++e) t = fmaf(wf[jj][e], hf[e], t);
          acc[jj * NR + r] = t;
        }
      }
    }
#pragma unroll
    for (int o = 16, m = 32; o > 0; o >>= 1, m >>= 1) {
      const bool upper = (lane & o) != 0;
#pragma unroll
      for (int i = 0; i < m / 2; ++i) {
        const float send = upper ? acc[i] : acc[i + m / 2];
        const float keep = upper ? acc[i + m / 2] : acc[i];
        acc[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
    }
    const int jj = lane / NR, r = lane - jj * NR;
    if (j0 + jj < b) sRes[(size_t)(j0 + jj) * NR + r] = acc[0];
  }
  for (int r = warp; r < NR; r += kDWarps) {
    float t = 0.f;
    for (int k = lane; k < nch; k += 32) {
      float hf[V];
      lds_vec<T>(sH + (size_t)r * p.cs + k * V, hf);
#pragma unroll
      for (int e = 0; e < V; ++e) t = fmaf(hf[e], hf[e], t);
    }
    t = warp_sum_f32(t);
    if (lane == 0) sRes[(size_t)b * NR + r] = t;
  }
  __syncthreads();
  DTL(2);
  decode_tail<NR>(p, c, s, sRes, sWup, sLog, &last_s);
}

size_t tail_bytes(int b, int NR) { return ((size_t)b * NR + NR + (kDWarps + 1) * NR + b + 2) * 4; }

size_t smem_tc(int b, int cs, int NR) {
  const int MT = (b + 127) / 128, nkc = cs / 64;
  return 1024 + (size_t)nkc * MT * 16384 + (size_t)nkc * 2048 + tail_bytes(b, NR) + 32 + 8 * kDMaxKc;
}
// extra smem of the cluster variant: recv [S][U][NR] + recv_ss [S][NR] + plog [S][NR] + yv [U][NR]
size_t smem_clu(int b, int S, int NR) {
  const int U = (b + S - 1) / S;
  return 16 + ((size_t)S * U * NR + 2 * (size_t)S * NR + (size_t)U * NR) * 4;
}
size_t smem_f32(int b, int cs, int NR) { return (size_t)(b + NR) * cs * 4 + tail_bytes(b, NR); }

// Largest-cluster plan: clusters of S slice-CTAs (one per checkpoint) when all
// C of them can be co-resident; else 0 (the global-ticket reduction).
template <typename K>
int launch_cluster(K kernel, const DecParams& p, size_t smem, cudaStream_t s) {
  // co-resident cluster counts per (kernel, S, smem), queried once each
  struct Entry {
    const void* k;
    size_t smem;
    int S, v;
  };
  static Entry cache[16];
  static int used = 0;
  static std::mutex mu;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(p.C * p.S));
  cfg.blockDim = dim3(kDThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeClusterDimension;
  a[0].val.clusterDim.x = (unsigned)p.S;
  a[0].val.clusterDim.y = 1;
  a[0].val.clusterDim.z = 1;
  cfg.attrs = a;
  cfg.numAttrs = 1;
  int ok_for = -1;
  {
    std::lock_guard<std::mutex> lk(mu);
    for (int i = 0; i < used; ++i)
      if (cache[i].k == (const void*)kernel && cache[i].smem == smem && cache[i].S == p.S) ok_for = cache[i].v;
    if (ok_for < 0) {
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cudaFuncSetAttribute(kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      int v = 0;
      if (cudaOccupancyMaxActiveClusters(&v, kernel, &cfg) != cudaSuccess) {
        cudaGetLastError();
        v = 0;
      }
      ok_for = v;
      if (used < 16) cache[used++] = Entry{(const void*)kernel, smem, p.S, v};
      if (getenv("TIDE_DEBUG_PLAN"))
        fprintf(stderr, "[tide] decode clusters of %d x %zu B smem: %d co-resident (need %d)\n",
                p.S, smem, v, p.C);
    }
  }
  {
    // the dynamic-smem attribute is per kernel: keep it at the largest size launched
    static const void* ks[8];
    static size_t kmax[8];
    static int nk = 0;
    std::lock_guard<std::mutex> lk(mu);
    int i = 0;
    while (i < nk && ks[i] != (const void*)kernel) ++i;
    if (i == nk && nk < 8) { ks[nk] = (const void*)kernel; kmax[nk++] = 0; }
    if (i < 8 && kmax[i] < smem) {
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      kmax[i] = smem;
    }
  }
  // The resolution is by ticket, so clusters need not all be co-resident, but
  // a straggler wave costs more than a narrower split (measured: 16-CTA
  // clusters with 7 of 9 resident 11.0 us vs 8-CTA clusters all resident 10.1)
  if (ok_for < p.C) return 1;  // caller tries the next split / falls back
  cudaLaunchKernelEx(&cfg, kernel, p);
  return check_launch("decode_tc_kernel (cluster)") == TIDE_OK ? 0 : -1;
}

template <typename K>
int launch_kernel(K kernel, const DecParams& p, size_t smem, cudaStream_t s, size_t* attr) {
  if (smem > 48 * 1024 && smem > *attr) {
    if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return check_launch("decode_kernel smem attribute");
    *attr = smem;
  }
  kernel<<<p.C * p.S, kDThreads, smem, s>>>(p);
  return check_launch("decode_kernel");
}

}  // namespace

}  // namespace tide

extern "C" int tide_route_decode(const void* const* h_ptrs, int32_t C, int64_t ld_h, int64_t n,
                                 int32_t d, int32_t dtype, const void* const* w_ptrs,
                                 const float* const* wup_ptrs, int32_t b, const int64_t* layers,
                                 float eps, float theta, int64_t k_min, int32_t mode,
                                 float* scores, float* logits, int64_t* exit_layers,
                                 int64_t* exit_count, void* workspace, void* stream) {
  using namespace tide;
  if (C < 1 || C > kDMaxC) return set_error(TIDE_ERR_ARG, "C must be in [1, %d]", kDMaxC);
  if (n < 1 || n > kDMaxRows) return set_error(TIDE_ERR_ARG, "decode rows must be in [1, %d]", kDMaxRows);
  if (d < 1 || b < 1) return set_error(TIDE_ERR_ARG, "bad shape");
  if (b > kDMaxB) return set_error(TIDE_ERR_UNSUPPORTED, "decode path: bottleneck > %d", kDMaxB);
  if (!workspace) return set_error(TIDE_ERR_ARG, "workspace required");
  if (dtype != TIDE_F32 && dtype != TIDE_BF16 && dtype != TIDE_F16)
    return set_error(TIDE_ERR_ARG, "bad dtype %d", dtype);
  const bool tc = dtype != TIDE_F32;
  const int esz = tc ? 2 : 4;
  const int V = 16 / esz;
  if (d % V != 0 || ld_h % V != 0)
    return set_error(TIDE_ERR_UNSUPPORTED, "decode path needs d and ld_h multiples of %d", V);
  DecParams p{};
  for (int c = 0; c < C; ++c) {
    if ((reinterpret_cast<uintptr_t>(h_ptrs[c]) | reinterpret_cast<uintptr_t>(w_ptrs[c])) & 15)
      return set_error(TIDE_ERR_UNSUPPORTED, "decode path needs 16-byte aligned rows");
    p.h[c] = h_ptrs[c];
    p.w[c] = w_ptrs[c];
    p.wup[c] = wup_ptrs[c];
    p.layers[c] = layers[c];
  }
  // Slice width: 512 bytes of every W row per CTA (one 16-byte piece per lane
  // and row), widened while the partial tiles would overflow the workspace.
  const int NR = n <= 8 ? 8 : 16;
  const int64_t tile = (int64_t)b * NR + NR;
  const int unit = 512 / esz;
  int cs = unit;
  size_t smem = 0;
  while (true) {
    const int64_t S = (d + cs - 1) / cs;
    smem = tc ? smem_tc(b, cs, NR) : smem_f32(b, cs, NR);
    if (smem > 220 * 1024) return set_error(TIDE_ERR_UNSUPPORTED, "decode problem too large");
    if ((int64_t)C * S * tile <= kMaxPartials) break;
    cs += unit;
  }
  p.C = C;
  p.d = d;
  p.b = b;
  p.cs = cs;
  p.S = (d + cs - 1) / cs;
  p.ld_h = ld_h;
  p.n = n;
  p.k_min = k_min;
  p.mode = mode;
  p.eps = eps;
  p.inv_d = (float)(1.0 / (double)d);
  p.theta = theta;
  p.scores = scores;
  p.logits = logits;
  p.exit_layers = exit_layers;
  p.exit_count = exit_count;
  p.ws = reinterpret_cast<Workspace*>(workspace);
  p.dbg = g_dbg;
  // stacked W ([C, b, d] contiguous, the runtime's decode plan) -> one tensor map
  p.use_tma = 0;
  if (tc && d % 8 == 0 && cs / 64 <= kDMaxKc) {
    bool stacked = true;
    const char* w0 = reinterpret_cast<const char*>(w_ptrs[0]);
    for (int c = 1; c < C && stacked; ++c)
      stacked = reinterpret_cast<const char*>(w_ptrs[c]) == w0 + (size_t)c * b * d * 2;
    const char* tenv = getenv("TIDE_DECODE_TMA");
    if (stacked && !(tenv && tenv[0] == '0') &&
        make_map(&p.wmap, w_ptrs[0], dtype, d, (int64_t)C * b, d, 64, 128) == TIDE_OK)
      p.use_tma = 1;
    cudaGetLastError();
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  static size_t attr[6] = {0, 0, 0, 0, 0, 0};
  // tensor-core path: slice CTAs of a checkpoint as one cluster (DSMEM
  // reduction) when S <= 16 and all C clusters fit; TIDE_DECODE_CLUSTER=0 disables
  const char* cenv = getenv("TIDE_DECODE_CLUSTER");  // read per call (tests switch it)
  if (tc && !(cenv && cenv[0] == '0')) {
    // widest slice first (S = 16, then 8): fewer bytes per CTA, if co-resident
    for (int cw = cs; cw <= 4 * cs; cw *= 2) {
      DecParams q = p;
      q.cs = cw;
      q.S = (d + cw - 1) / cw;
      if (q.S < 2 || q.S > 16 || q.cs % 64) continue;
      const size_t smc = smem_tc(b, cw, NR) + smem_clu(b, q.S, NR);
      if (smc > 220 * 1024) break;
      int rc;
      if (dtype == TIDE_BF16)
        rc = NR == 8 ? launch_cluster(decode_tc_kernel<true, 8, true>, q, smc, s)
                     : launch_cluster(decode_tc_kernel<true, 16, true>, q, smc, s);
      else
        rc = NR == 8 ? launch_cluster(decode_tc_kernel<false, 8, true>, q, smc, s)
                     : launch_cluster(decode_tc_kernel<false, 16, true>, q, smc, s);
      if (rc <= 0) return rc == 0 ? TIDE_OK : TIDE_ERR_CUDA;
    }
  }
  if (dtype == TIDE_BF16)
    return NR == 8 ? launch_kernel(decode_tc_kernel<true, 8, false>, p, smem, s, &attr[0])
                   : launch_kernel(decode_tc_kernel<true, 16, false>, p, smem, s, &attr[1]);
  if (dtype == TIDE_F16)
    return NR == 8 ? launch_kernel(decode_tc_kernel<false, 8, false>, p, smem, s, &attr[2])
                   : launch_kernel(decode_tc_kernel<false, 16, false>, p, smem, s, &attr[3]);
  return NR == 8 ? launch_kernel(decode_f32_kernel<8>, p, smem, s, &attr[4])
                 : launch_kernel(decode_f32_kernel<16>, p, smem, s, &attr[5]);
}
