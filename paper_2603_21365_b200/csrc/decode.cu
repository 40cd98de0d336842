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

#ifndef TIDE_DEC_EXP
#define TIDE_DEC_EXP 0  // timing experiments only (wrong results, tools/decode_exp.py): 1 one
                        // W chunk per slice, 2 no resolution atomic, 3 no row loads, 4 no
                        // DSMEM exchange
#endif
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
  // or (w_packed != NULL) the SW128 shared-memory image of every W, packed
  // once by tide_decode_pack_weights: [C][nk][MT][128 rows x 128 B]; a CTA's
  // k-chunks are contiguous 16 KB blocks fetched by plain bulk copies
  const uint8_t* w_packed;
  int32_t nk;
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
  unsigned long long* dbg;  // optional per-CTA timeline (globaltimer ns), 32 slots per CTA (debug)
};

__device__ __forceinline__ unsigned long long dgt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// Debug timeline (tools/timeline_decode_graph.py): clock64 per phase slot,
// plus the entry's globaltimer in slot 31; 32 slots per CTA.
#ifdef TIDE_DECODE_DEBUG
#define DPR(slot) \
  do { if (blockIdx.x == 1 && (threadIdx.x == 0 || threadIdx.x == 2)) printf("blk1 t%d at %d\n", threadIdx.x, slot); } while (0)
#else
#define DPR(slot) do {} while (0)
#endif
#define DTL(slot)                                                                   \
  do {                                                                              \
    DPR(slot);                                                                      \
    if (p.dbg && threadIdx.x == 0) {                                                \
      p.dbg[32 * blockIdx.x + (slot)] = (unsigned long long)clock64();              \
      if ((slot) == 0) p.dbg[32 * blockIdx.x + 31] = dgt();                         \
    }                                                                               \
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
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait;" ::: "memory"); }

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

// Step 5 with ONE global round trip (C <= kAtomicMaxC): the CTA holding
// checkpoint c's row logits writes the scores and adds (1 << 56 | fired << c)
// to each row's resolution word (per-token) or (1 << 56 | all-fired << c) to
// the batch word.  The atomic returns the previous value, so the arrival that
// completes the count already holds every checkpoint's fired bit: it writes
// the exit layer (first set bit, layers ascending; NO_EXIT if none) and
// resets the word for the next launch.  Only the fired bits travel through the
// words (no other data is published), so relaxed atomics suffice.
constexpr int kAtomicMaxC = 56;

__device__ __forceinline__ unsigned long long atom_add_relaxed_u64(unsigned long long* a,
                                                                   unsigned long long v) {
  unsigned long long old;
  asm volatile("atom.relaxed.gpu.global.add.u64 %0, [%1], %2;" : "=l"(old) : "l"(a), "l"(v) : "memory");
  return old;
}

template <int NR>
__device__ __forceinline__ void decode_finish_atomic(const DecParams& p, int c, const float* sLogit) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp != 0) return;
  const int n = (int)p.n;
  const int r = lane;
  const bool live = r < n;
  const float t = live ? sLogit[r] : 0.f;
  // The decision score > theta, where score = f32(sigmoid_f64(t)), from an f32
  // estimate (|estimate - score| < 4e-7) except within 1e-6 of theta, where
  // the exact score decides: identical decisions, and the f64 sigmoid for the
  // score output runs while the resolution atomic is in flight.
  bool fired = false;
  if (live && p.layers[c] >= p.k_min) {
    const float se = sigmoid_f32(t);
    if (se > p.theta + 1e-6f)
      fired = true;
    else if (se >= p.theta - 1e-6f)
      fired = score_from_logit(t) > p.theta;
  }
  DTL(5);
  constexpr unsigned long long kOne = 1ull << 56, kBits = kOne - 1ull;
  auto outputs = [&]() {
    if (live) {
      if (p.scores) p.scores[(int64_t)c * n + r] = score_from_logit(t);
      if (p.logits) p.logits[(int64_t)c * n + r] = t;
    }
  };
  if (p.mode == TIDE_MODE_PER_TOKEN) {
    if (!live) return;
    const unsigned long long add = kOne | (fired ? (1ull << c) : 0ull);
    const unsigned long long old = atom_add_relaxed_u64(&p.ws->dec_rows[r], add);
    outputs();
    if ((old >> 56) != (unsigned long long)(p.C - 1)) return;
    const unsigned long long bits = (old + add) & kBits;
    const int64_t ex = bits ? p.layers[__ffsll((long long)bits) - 1] : (int64_t)TIDE_NO_EXIT;
    if (p.exit_layers) p.exit_layers[r] = ex;
    p.ws->dec_rows[r] = 0ull;
    DTL(6);
    if (p.exit_count) {
      const unsigned long long addc = (1ull << 32) | (ex != TIDE_NO_EXIT ? 1ull : 0ull);
      const unsigned long long oc = atom_add_relaxed_u64(&p.ws->dec_cnt, addc);
      if ((oc >> 32) == (unsigned long long)(n - 1)) {
        p.exit_count[0] = (int64_t)((oc + addc) & 0xffffffffull);
        p.ws->dec_cnt = 0ull;
      }
    }
  } else {
    const bool all = __all_sync(0xffffffffu, !live || fired);
    unsigned long long bits = 0ull;
    int last = 0;
    if (lane == 0) {
      const unsigned long long add = kOne | (all ? (1ull << c) : 0ull);
      const unsigned long long old = atom_add_relaxed_u64(&p.ws->dec_all, add);
      last = (old >> 56) == (unsigned long long)(p.C - 1);
      bits = (old + add) & kBits;
      if (last) p.ws->dec_all = 0ull;
    }
    outputs();
    last = __shfl_sync(0xffffffffu, last, 0);
    if (!last) return;
    bits = __shfl_sync(0xffffffffu, bits, 0);
    const int64_t ex = bits ? p.layers[__ffsll((long long)bits) - 1] : (int64_t)TIDE_NO_EXIT;
    if (live && p.exit_layers) p.exit_layers[r] = ex;
    if (lane == 0 && p.exit_count) p.exit_count[0] = ex != TIDE_NO_EXIT ? n : 0;
  }
}

// The same resolution for ONE row, by the thread that finished the row's
// logit t for checkpoint c (cluster kernel: rows are spread over the ranks).
// Per-token: one atomic on the row's word.  Batch-unanimous: the row's last
// checkpoint arrival ORs its not-fired mask into dec_all, then counts itself
// into dec_cnt (release / acquire); the last row reads-and-resets dec_all and
// writes every row (three round trips, batch mode only).
__device__ __forceinline__ unsigned long long atom_or_relaxed_u64(unsigned long long* a,
                                                                  unsigned long long v) {
  unsigned long long old;
  asm volatile("atom.relaxed.gpu.global.or.b64 %0, [%1], %2;" : "=l"(old) : "l"(a), "l"(v) : "memory");
  return old;
}
__device__ __forceinline__ unsigned long long atom_add_acqrel_u64(unsigned long long* a,
                                                                  unsigned long long v) {
  unsigned long long old;
  asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], %2;" : "=l"(old) : "l"(a), "l"(v) : "memory");
  return old;
}
__device__ __forceinline__ unsigned long long atom_exch_acquire_u64(unsigned long long* a,
                                                                    unsigned long long v) {
  unsigned long long old;
  asm volatile("atom.acquire.gpu.global.exch.b64 %0, [%1], %2;" : "=l"(old) : "l"(a), "l"(v) : "memory");
  return old;
}

__device__ __forceinline__ void decode_resolve_row(const DecParams& p, int c, int r, float t) {
  const int n = (int)p.n;
  bool fired = false;
  if (p.layers[c] >= p.k_min) {
    const float se = sigmoid_f32(t);
    if (se > p.theta + 1e-6f)
      fired = true;
    else if (se >= p.theta - 1e-6f)
      fired = score_from_logit(t) > p.theta;
  }
  constexpr unsigned long long kOne = 1ull << 56, kBits = kOne - 1ull;
  const unsigned long long add = kOne | (fired ? (1ull << c) : 0ull);
  if (TIDE_DEC_EXP == 2) {
    if (p.exit_layers && c == 0) p.exit_layers[r] = fired;
    return;
  }
  const unsigned long long old = atom_add_relaxed_u64(&p.ws->dec_rows[r], add);
  if (p.scores) p.scores[(int64_t)c * n + r] = score_from_logit(t);
  if (p.logits) p.logits[(int64_t)c * n + r] = t;
  if ((old >> 56) != (unsigned long long)(p.C - 1)) return;
  p.ws->dec_rows[r] = 0ull;
  const unsigned long long bits = (old + add) & kBits;
  if (p.mode == TIDE_MODE_PER_TOKEN) {
    const int64_t ex = bits ? p.layers[__ffsll((long long)bits) - 1] : (int64_t)TIDE_NO_EXIT;
    if (p.exit_layers) p.exit_layers[r] = ex;
    if (p.exit_count) {
      const unsigned long long addc = (1ull << 32) | (ex != TIDE_NO_EXIT ? 1ull : 0ull);
      const unsigned long long oc = atom_add_relaxed_u64(&p.ws->dec_cnt, addc);
      if ((oc >> 32) == (unsigned long long)(n - 1)) {
        p.exit_count[0] = (int64_t)((oc + addc) & 0xffffffffull);
        p.ws->dec_cnt = 0ull;
      }
    }
    return;
  }
  const unsigned long long all_c = (p.C >= 64) ? ~0ull : ((1ull << p.C) - 1ull);
  atom_or_relaxed_u64(&p.ws->dec_all, ~bits & all_c);  // checkpoints where row r did not fire
  const unsigned long long oc = atom_add_acqrel_u64(&p.ws->dec_cnt, 1ull);
  if (oc != (unsigned long long)(n - 1)) return;
  const unsigned long long notfired = atom_exch_acquire_u64(&p.ws->dec_all, 0ull);
  p.ws->dec_cnt = 0ull;
  const unsigned long long allbits = ~notfired & all_c;
  const int64_t ex = allbits ? p.layers[__ffsll((long long)allbits) - 1] : (int64_t)TIDE_NO_EXIT;
  if (p.exit_layers)
    for (int i = 0; i < n; ++i) p.exit_layers[i] = ex;
  if (p.exit_count) p.exit_count[0] = ex != TIDE_NO_EXIT ? n : 0;
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
  if (p.C <= kAtomicMaxC) {
    if (threadIdx.x == 0) p.ws->tickets[c] = 0;  // reset for the next launch (graph replay safe)
    decode_finish_atomic<NR>(p, c, sLog + kDWarps * NR);
  } else {
    decode_finish<NR>(p, c, sLog + kDWarps * NR, last_s);
  }
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
  if (threadIdx.x == 0) griddep_launch_dependents();
  // cluster reduction buffers: this CTA's partial tile as row blocks
  // sRows[r][RB] (RB = b + 4: the row's b partial pre-activations, then its
  // partial sum of squares), and recv[k][src][RB] for the rows this rank owns
  // (row r is owned by rank r % S; k = r / S)
  const int RB = b + 4;
  uint64_t* recv_bar = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(tmem_slot) + 8 + 8 * kDMaxKc);
  float* sRows = reinterpret_cast<float*>(
      (reinterpret_cast<uintptr_t>(tmem_slot) + 16 + 8 * kDMaxKc + 15) & ~(uintptr_t)15);
  float* recv = sRows + (size_t)NR * RB;
  const int own_rows = kClu ? (n > s ? (n - s + p.S - 1) / p.S : 0) : 0;  // rows r = s, s + S, ...
  if (kClu) {
    if (threadIdx.x == 0 && own_rows > 0) {
      // armed before the cluster arrive: peers send only after their cluster wait
      mbar_init(recv_bar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      mbar_arrive_expect_tx(recv_bar, (uint32_t)own_rows * (uint32_t)(p.S - 1) * (uint32_t)RB * 4u);
    }
    asm volatile("barrier.cluster.arrive.release;" ::: "memory");
  }

  // 1. one round trip: W slice + hidden slice as 16-byte pieces into the
  //    swizzled K-major layout (piece q of row j at ((q ^ (j & 7)) << 4))
  const T* W = reinterpret_cast<const T*>(p.w[c]);
  const T* H = reinterpret_cast<const T*>(p.h[c]);
  const int per_row = nkc * 8;
  uint64_t* wfull = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(tmem_slot) + 8);  // [kDMaxKc]
  // W slices land on ONE barrier (wfull[0]): with PDL they are fetched while
  // the previous kernel runs, so by the time the rows land W is resident and
  // a single wait precedes the whole MMA stream (a wait per k-chunk cost
  // ~500 cycles each, measured).
  const int nkc_mma = TIDE_DEC_EXP == 1 ? 1 : p.w_packed ? min(nkc, p.nk - c0 / 64) : nkc;  // packed: chunks past d skipped
  if (p.w_packed) {
    // the pre-swizzled image: one 1-D bulk copy (MT x 16 KB) per k-chunk
    if (threadIdx.x == 0) {
      mbar_init(&wfull[0], 1);
      fence_mbar_init();
      const uint64_t pol = policy_evict_last();  // every decode step re-reads it
      const int kc0 = c0 / 64;
      const uint32_t bytes = (uint32_t)MT * 16384u;
      mbar_arrive_expect_tx(&wfull[0], bytes * (uint32_t)nkc_mma);
      for (int kc = 0; kc < nkc_mma; ++kc)
        bulk_g2s(sA + (size_t)kc * MT * 16384, p.w_packed + ((size_t)c * p.nk + kc0 + kc) * bytes,
                 bytes, &wfull[0], pol);
    }
  } else if (p.use_tma) {
    if (threadIdx.x == 0) {
      mbar_init(&wfull[0], 1);
      fence_mbar_init();
      const uint64_t pol = policy_evict_last();  // every decode step re-reads it
      mbar_arrive_expect_tx(&wfull[0], (uint32_t)(nkc * MT) * 16384u);
      for (int kc = 0; kc < nkc; ++kc)
        for (int mt = 0; mt < MT; ++mt)
          tma_load_2d(sA + ((size_t)kc * MT + mt) * 16384, &p.wmap, &wfull[0], c0 + kc * 64,
                      c * b + mt * 128, pol);
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
  for (int j = threadIdx.x; j < b; j += kDThreads) sWup[j] = p.wup[c][j];
  if (threadIdx.x == 0) {
    mbar_init(mma_done, 1);
    fence_mbar_init();
  }
  if (warp == 1) {
    tmem_alloc(tmem_slot, 32);
    tmem_relinquish();
  }
  // PDL: everything above reads only the static router weights (the caller's
  // contract: no kernel in flight writes W_down / w_up), so it overlaps the
  // previous kernel on the stream; the hidden rows and the workspace words
  // are touched only after it completed.
  griddep_wait();
  DTL(12);
  for (int i = threadIdx.x; TIDE_DEC_EXP != 3 && i < 16 * per_row; i += kDThreads) {
    const int r = i / per_row, rem = i - r * per_row, kc = rem >> 3, q = rem & 7;
    const int col = c0 + kc * 64 + q * 8;
    const bool in = col < p.d && r < n;
    uint8_t* dst = sB + (size_t)kc * 2048 + r * 128 + ((q ^ (r & 7)) << 4);
    cp_async16_zfill(dst, H + (in ? (int64_t)r * p.ld_h + col : 0), in);
  }
  cp_async_wait_all();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  DTL(1);

  // 2. MMAs: warp 0 walks the loop (descriptors warp-uniform -> uniform
  //    registers), one elected lane issues each MMA: D[mt] (128 x 16) +=
  //    A[kc][mt] . B[kc]^T, ~39 cycles per N = 16 MMA back to back (measured)
  if (warp == 0) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // cp.async -> MMA operands
    if (p.use_tma || p.w_packed) mbar_wait_spin(&wfull[0], 0);
    tc_fence_after();
    DTL(8);
    const uint64_t desc_hi = sw128_kmajor_desc(0);
    const uint32_t idesc = f16_idesc(kBF16 ? 1 : 0, 128, 16);
    const uint64_t a_base = desc_hi | (uint64_t)((smem_u32(sA) & 0x3FFFFu) >> 4);
    const uint64_t b_base = desc_hi | (uint64_t)((smem_u32(sB) & 0x3FFFFu) >> 4);
    for (int kc = 0; kc < nkc_mma; ++kc)
      for (int mt = 0; mt < MT; ++mt) {
        const uint64_t ad = a_base + (uint64_t)(((kc * MT + mt) * 16384) >> 4);
        const uint64_t bd = b_base + (uint64_t)((kc * 2048) >> 4);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (elect_one())
            tc_mma_f16(tmem_base + (uint32_t)(mt * 16), ad + 2 * k, bd + 2 * k, idesc, (kc | k) != 0);
      }
    if (elect_one()) tc_commit(mma_done);
    __syncwarp();
    DTL(9);
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
    if (r < NR && q == 0) {
      if (kClu)
        sRows[(size_t)r * RB + b] = ss;
      else
        sRes[(size_t)b * NR + r] = ss;
    }
  }
  // 3a. accumulators -> sRes[j][r] (warps 0-3: TMEM lane quadrant = warp)
  if (warp < 4) {
    mbar_wait_spin(mma_done, 0);
    tc_fence_after();
    for (int mt = 0; mt < MT; ++mt) {
      uint32_t v[16];
      tmem_ld16(tmem_base + ((uint32_t)(32 * warp) << 16) + (uint32_t)(mt * 16), v);
      tmem_ld_wait();
      const int j = mt * 128 + 32 * warp + lane;
      if (j < b) {
        if (kClu) {
#pragma unroll
          for (int r = 0; r < NR; ++r) sRows[(size_t)r * RB + j] = __uint_as_float(v[r]);
        } else {
#pragma unroll
          for (int r = 0; r < NR; ++r) sRes[(size_t)j * NR + r] = __uint_as_float(v[r]);
        }
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
  // 3b. DSMEM exchange by rows: thread r (< n) ships row r's block (RB
  //     floats) with one bulk copy to the rank that owns the row (r % S),
  //     into its slot for this source rank, completing on that rank's
  //     barrier.  No cluster barrier on the critical path (the wait for every
  //     rank's start was satisfied during the W / row loads).
  const uint32_t rank = (uint32_t)s;  // cluster dims (S, 1, 1), blockIdx.x = c S + s
  const int S = p.S;
  const uint32_t rb_bytes = (uint32_t)RB * 4u;
  if (warp == 0) {
    // the whole warp waits (a partial-warp barrier.cluster.wait never
    // completed here, measured), then each sending lane issues its copy
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // sRows -> bulk copy reads
    cluster_wait();
    if (TIDE_DEC_EXP != 4 && lane < n && (lane % S) != (int)rank) {
      const int r = lane, q = r % S, k = r / S;
      const uint32_t dst = dsmem_addr(smem_u32(recv + ((size_t)k * S + rank) * RB), (uint32_t)q);
      const uint32_t bar = dsmem_addr(smem_u32(recv_bar), (uint32_t)q);
      asm volatile(
          "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
          "r"(smem_u32(sRows + (size_t)r * RB)), "r"(rb_bytes), "r"(bar)
          : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // read before exit
    }
  }
  if (own_rows == 0) return;
#ifdef TIDE_DECODE_DEBUG
  {
    uint32_t spins = 0;
    while (!mbar_try_wait(smem_u32(recv_bar), 0)) {
      if (++spins == (1u << 22) && threadIdx.x == 0) {
        unsigned long long st = *reinterpret_cast<volatile unsigned long long*>(recv_bar);
        uint32_t dyn;
        asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
        printf("decode hang: blk %d rank %u own %d n %d S %d RB %d state %llx | bar %u rows %u recv %u "
               "wup %u tslot %u sA %u sB %u sRes %u dyn %u\n", blockIdx.x, rank, own_rows, n, S, RB, st,
               smem_u32(recv_bar), smem_u32(sRows), smem_u32(recv), smem_u32(sWup), smem_u32(tmem_slot),
               smem_u32(sA), smem_u32(sB), smem_u32(sRes), dyn);
      }
      if (spins > (1u << 24)) __trap();
    }
  }
#endif
  if (TIDE_DEC_EXP != 4) mbar_wait_spin(recv_bar, 0);
  DTL(3);
  // 4. rows owned here (k = 0 .. own_rows - 1, row r = rank + k S), 128
  //    threads per row, unit j per thread: totals over the S slices in fixed
  //    source order, RMS scale, SiLU (tanh form, as K1: logit error <=
  //    2.5e-4 m), w_up; the row's sum in a fixed tree (lanes, then warps)
  float* red = sLog;  // [2][4] warp partials
  for (int kb = 0; kb < own_rows; kb += 2) {  // uniform over the CTA
    const int k = kb + (threadIdx.x >> 7), jt = threadIdx.x & 127;
    const int r = (int)rank + k * S;
    const bool row_ok = k < own_rows && r < n;
    float y = 0.f;
    if (row_ok) {
      float ss = 0.f;
      for (int src = 0; src < S; ++src)
        ss += (src == (int)rank) ? sRows[(size_t)r * RB + b] : recv[((size_t)k * S + src) * RB + b];
      const float hs = 0.5f * rms_scale(ss, p.inv_d, p.eps);
      for (int j = jt; j < b; j += 128) {
        float a = 0.f;
#pragma unroll 4
        for (int src = 0; src < S; ++src)
          a += (src == (int)rank) ? sRows[(size_t)r * RB + j] : recv[((size_t)k * S + src) * RB + j];
        const float h = __fmul_rn(a, hs);
        y = fmaf(sWup[j], fmaf(h, tanh_approx(h), h), y);
      }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) y += __shfl_xor_sync(0xffffffffu, y, o);
    if (lane == 0) red[warp] = y;
    __syncthreads();
    DTL(4);
    if (jt == 0 && row_ok) {
      const int g = threadIdx.x >> 7;
      const float t = (red[4 * g] + red[4 * g + 1]) + (red[4 * g + 2] + red[4 * g + 3]);
      decode_resolve_row(p, c, r, t);
    }
    __syncthreads();
  }
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
  if (threadIdx.x == 0) griddep_launch_dependents();
  for (int i = threadIdx.x; i < b * nch; i += kDThreads) {
    const int j = i / nch, k = i - j * nch;
    cp_async16_zfill(sW + (size_t)j * p.cs + k * V, W + (int64_t)j * p.d + c0 + k * V, true);
  }
  griddep_wait();  // PDL: the rows (and the workspace) only after the previous kernel
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
// extra smem of the cluster variant: sRows [NR][b + 4] + recv [ceil(NR/S)][S][b + 4] (+ alignment)
size_t smem_clu(int b, int S, int NR) {
  return 32 + ((size_t)NR + (size_t)((NR + S - 1) / S) * S) * (size_t)(b + 4) * 4;
}
size_t smem_f32(int b, int cs, int NR) { return (size_t)(b + NR) * cs * 4 + tail_bytes(b, NR); }

// Largest-cluster plan: clusters of S slice-CTAs (one per checkpoint) when all
// C of them can be co-resident; else 0 (the global-ticket reduction).
bool pdl_enabled() {
  const char* env = getenv("TIDE_PDL");  // read per call
  return !(env && env[0] == '0');
}

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
  cudaLaunchAttribute a[2];
  a[0].id = cudaLaunchAttributeClusterDimension;
  a[0].val.clusterDim.x = (unsigned)p.S;
  a[0].val.clusterDim.y = 1;
  a[0].val.clusterDim.z = 1;
  a[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  a[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = a;
  cfg.numAttrs = 1;  // occupancy query without PDL
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
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
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
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(p.C * p.S));
  cfg.blockDim = dim3(kDThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  a[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = a;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kernel, p);
  return check_launch("decode_kernel");
}

// The SW128 K-major shared-memory image of every router's W (bf16 / f16):
// block (c, kc, mt) = rows mt*128 .. +127 of W_c, columns kc*64 .. +63, 16-byte
// piece q of row j at j*128 + ((q ^ (j & 7)) << 4); zero past b / d.
__global__ void decode_pack_kernel(const __grid_constant__ DecParams p, uint8_t* out, int MT) {
  const int64_t pieces = (int64_t)p.C * p.nk * MT * 128 * 8;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < pieces;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int q = (int)(i & 7);
    const int j = (int)((i >> 3) & 127);
    int64_t blk = i >> 10;  // (c, kc, mt)
    const int mt = (int)(blk % MT);
    blk /= MT;
    const int kc = (int)(blk % p.nk);
    const int c = (int)(blk / p.nk);
    const int row = mt * 128 + j, col = kc * 64 + q * 8;
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (row < p.b && col < p.d)
      v = *reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(p.w[c]) +
                                          (int64_t)row * p.d + col);
    *reinterpret_cast<uint4*>(out + (((int64_t)c * p.nk + kc) * MT + mt) * 16384 + j * 128 +
                              ((q ^ (j & 7)) << 4)) = v;
  }
}

}  // namespace

}  // namespace tide

extern "C" size_t tide_decode_packed_bytes(int32_t C, int32_t d, int32_t b) {
  if (C < 1 || d < 1 || b < 1) return 0;
  return (size_t)C * ((d + 63) / 64) * ((b + 127) / 128) * 16384u;
}

extern "C" int tide_decode_pack_weights(const void* const* w_ptrs, int32_t C, int32_t d, int32_t b,
                                        int32_t dtype, void* out, void* stream) {
  using namespace tide;
  if (C < 1 || C > kDMaxC || d < 8 || d % 8 || b < 1 || b > kDMaxB || !out || !w_ptrs)
    return set_error(TIDE_ERR_ARG, "tide_decode_pack_weights: bad arguments");
  if (dtype != TIDE_BF16 && dtype != TIDE_F16)
    return set_error(TIDE_ERR_UNSUPPORTED, "tide_decode_pack_weights: bf16 / f16 only");
  DecParams p{};
  for (int c = 0; c < C; ++c) {
    if (!w_ptrs[c] || (reinterpret_cast<uintptr_t>(w_ptrs[c]) & 15))
      return set_error(TIDE_ERR_ARG, "tide_decode_pack_weights: unaligned weights");
    p.w[c] = w_ptrs[c];
  }
  p.C = C;
  p.d = d;
  p.b = b;
  p.nk = (d + 63) / 64;
  const int MT = (b + 127) / 128;
  decode_pack_kernel<<<296, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      p, reinterpret_cast<uint8_t*>(out), MT);
  return check_launch("decode_pack_kernel");
}

extern "C" int tide_route_decode(const void* const* h_ptrs, int32_t C, int64_t ld_h, int64_t n,
                                 int32_t d, int32_t dtype, const void* const* w_ptrs,
                                 const float* const* wup_ptrs, int32_t b, const int64_t* layers,
                                 float eps, float theta, int64_t k_min, int32_t mode,
                                 float* scores, float* logits, int64_t* exit_layers,
                                 int64_t* exit_count, void* workspace, void* stream) {
  return tide_route_decode_ex(h_ptrs, C, ld_h, n, d, dtype, w_ptrs, wup_ptrs, b, layers, eps,
                              theta, k_min, mode, scores, logits, exit_layers, exit_count,
                              workspace, nullptr, stream);
}

extern "C" int tide_route_decode_ex(const void* const* h_ptrs, int32_t C, int64_t ld_h, int64_t n,
                                 int32_t d, int32_t dtype, const void* const* w_ptrs,
                                 const float* const* wup_ptrs, int32_t b, const int64_t* layers,
                                 float eps, float theta, int64_t k_min, int32_t mode,
                                 float* scores, float* logits, int64_t* exit_layers,
                                 int64_t* exit_count, void* workspace, const void* w_packed,
                                 void* stream) {
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
  // packed W image (tide_decode_pack_weights) -> 1-D bulk copies; else
  // stacked W ([C, b, d] contiguous) -> one tensor map; else cp.async
  p.use_tma = 0;
  p.nk = (d + 63) / 64;
  // TIDE_DECODE_TMA=0: neither bulk nor TMA W loads (the cp.async path);
  // TIDE_DECODE_PACKED=0: the tensor-map path over the stacked W (tests)
  const char* tenv0 = getenv("TIDE_DECODE_TMA");
  const char* penv = getenv("TIDE_DECODE_PACKED");
  const bool no_tma = tenv0 && tenv0[0] == '0';
  p.w_packed = (tc && d % 8 == 0 && !no_tma && !(penv && penv[0] == '0'))
                   ? reinterpret_cast<const uint8_t*>(w_packed)
                   : nullptr;
  if (w_packed && (reinterpret_cast<uintptr_t>(w_packed) & 127))
    return set_error(TIDE_ERR_ARG, "packed weights must be 128-byte aligned");
  if (!p.w_packed && tc && d % 8 == 0 && cs / 64 <= kDMaxKc) {
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
  if (tc && C <= kAtomicMaxC && !(cenv && cenv[0] == '0')) {
    // widest slice first (S = 16, then 8): fewer bytes per CTA, if co-resident;
    // TIDE_DECODE_COLS (a multiple of 64, read per call) tries that width only
    const char* wenv = getenv("TIDE_DECODE_COLS");
    const int cw0 = wenv ? std::max(64, atoi(wenv) / 64 * 64) : cs;
    for (int cw = cw0; cw <= (wenv ? cw0 : 4 * cs); cw *= 2) {
      DecParams q = p;
      q.cs = cw;
      q.S = (d + cw - 1) / cw;
      if (q.S < 2 || q.S > 16 || q.cs % 64) continue;
      if (q.w_packed && q.cs / 64 > kDMaxKc) q.w_packed = nullptr, q.use_tma = 0;
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
  if (p.w_packed && p.cs / 64 > kDMaxKc) p.w_packed = nullptr;  // cp.async fallback
  if (dtype == TIDE_BF16)
    return NR == 8 ? launch_kernel(decode_tc_kernel<true, 8, false>, p, smem, s, &attr[0])
                   : launch_kernel(decode_tc_kernel<true, 16, false>, p, smem, s, &attr[1]);
  if (dtype == TIDE_F16)
    return NR == 8 ? launch_kernel(decode_tc_kernel<false, 8, false>, p, smem, s, &attr[2])
                   : launch_kernel(decode_tc_kernel<false, 16, false>, p, smem, s, &attr[3]);
  return NR == 8 ? launch_kernel(decode_f32_kernel<8>, p, smem, s, &attr[4])
                 : launch_kernel(decode_f32_kernel<16>, p, smem, s, &attr[5]);
}
