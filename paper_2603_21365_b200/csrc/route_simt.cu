// CUDA-core router kernels.
//
// route_simt_kernel  — fused_layernorm_route + mask + stable compaction for
//   shapes the tensor-core kernel does not take (f32 rows: the reference's
//   own dtype, where 1e-5 logit parity needs f32 products; b > 256; d % 8).
//   16 rows x 128 bottleneck columns per pass, K staged through smem in
//   chunks of 32, 2x4 register micro-tile per thread, f32 accumulation.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "internal.h"

namespace tide {

constexpr int kSR = 16;    // rows per CTA
constexpr int kSJ = 128;   // bottleneck columns per pass
constexpr int kSK = 32;    // K chunk
constexpr int kSThreads = 256;

template <typename T>
__device__ __forceinline__ float ldf(const T* p) {
  return to_f32<T>(*p);
}

// acc[r2][c4] += sum_k X[ty + 8 r2][k] * W[j0 + tx + 32 c4][k] over k in [k0, k1)
// Also accumulates sum of squares of the 16 rows into ss_s[16] (if non-null).
template <typename XT>
__device__ __forceinline__ void gemm_16x128(const XT* const* xrow, const XT* W, int64_t ldw,
                                            int j0, int b, int64_t k0, int64_t k1,
                                            float (&acc)[2][4], float (*Xs)[kSK + 1],
                                            float (*Ws)[kSK + 1], float* ss_s) {
  const int tid = threadIdx.x;
  const int tx = tid & 31, ty = tid >> 5;
  for (int64_t kc = k0; kc < k1; kc += kSK) {
    // stage X chunk [16][32]
    for (int e = tid; e < kSR * kSK; e += kSThreads) {
      const int r = e / kSK, kk = e % kSK;
      const int64_t k = kc + kk;
      float v = 0.f;
      if (xrow[r] && k < k1) v = ldf(xrow[r] + k);
      Xs[r][kk] = v;
    }
    // stage W chunk [128][32]
    for (int e = tid; e < kSJ * kSK; e += kSThreads) {
      const int j = e / kSK, kk = e % kSK;
      const int64_t k = kc + kk;
      float v = 0.f;
      if (j0 + j < b && k < k1) v = ldf(W + (int64_t)(j0 + j) * ldw + k);
      Ws[j][kk] = v;
    }
    __syncthreads();
    if (ss_s && j0 == 0 && tid < kSR * 8) {
      // 8 threads per row reduce 4 elements each, then shuffle within the 8
      const int r = tid >> 3, part = tid & 7;
      float s = 0.f;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float x = Xs[r][part * 4 + u];
        s = fmaf(x, x, s);
      }
      s += __shfl_xor_sync(0xffffffffu, s, 1);
      s += __shfl_xor_sync(0xffffffffu, s, 2);
      s += __shfl_xor_sync(0xffffffffu, s, 4);
      if (part == 0) ss_s[r] += s;
    }
#pragma unroll 8
    for (int kk = 0; kk < kSK; ++kk) {
      const float x0 = Xs[ty][kk], x1 = Xs[ty + 8][kk];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const float w = Ws[tx + 32 * c][kk];
        acc[0][c] = fmaf(x0, w, acc[0][c]);
        acc[1][c] = fmaf(x1, w, acc[1][c]);
      }
    }
    __syncthreads();
  }
}

// Vector path (rows and W 16-byte aligned, d and ld multiples of the vector
// width): K chunks of kVK columns staged with 16-byte loads, the next chunk
// prefetched into registers while the current one is multiplied, and the
// inner product read from smem as float4 along k (32 FMAs per 6 LDS.128), so
// the loop is FMA-bound instead of latency- / LDS-bound.
constexpr int kVK = 64;            // K chunk of the vector path
constexpr int kVP = kVK + 4;       // padded smem row (16-byte aligned, conflict-free float4 reads)
constexpr size_t kVSmem = (size_t)(kSR + kSJ) * kVP * sizeof(float);

template <typename XT> struct Vec16;  // 16 bytes of XT -> f32 lanes
template <> struct Vec16<float> { static constexpr int N = 4; };
template <> struct Vec16<__nv_bfloat16> { static constexpr int N = 8; };
template <> struct Vec16<__half> { static constexpr int N = 8; };

template <typename XT>
__device__ __forceinline__ void gemm_16x128_vec(const XT* const* xrow, const XT* W, int64_t ldw,
                                                int j0, int b, int64_t d, float (&acc)[2][4],
                                                float* Xs, float* Ws, float* ss_s) {
  constexpr int V = Vec16<XT>::N;
  constexpr int XN = kSR * kVK / V, WN = kSJ * kVK / V;  // 16-byte pieces per chunk
  constexpr int XPER = (XN + kSThreads - 1) / kSThreads;   // per thread
  constexpr int WPER = (WN + kSThreads - 1) / kSThreads;
  const int tid = threadIdx.x;
  const int tx = tid & 31, ty = tid >> 5;
  uint4 xr[XPER], wr[WPER];
  auto load = [&](int64_t kc) {
#pragma unroll
    for (int u = 0; u < XPER; ++u) {
      const int e = tid + u * kSThreads;
      const int r = e / (kVK / V), kk = (e % (kVK / V)) * V;
      const int64_t k = kc + kk;
      xr[u] = (e < XN && xrow[r] && k < d) ? ld_nc_v4(xrow[r] + k) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < WPER; ++u) {
      const int e = tid + u * kSThreads;
      const int j = e / (kVK / V), kk = (e % (kVK / V)) * V;
      const int64_t k = kc + kk;
      wr[u] = (e < WN && j0 + j < b && k < d) ? ld_nc_v4(W + (int64_t)(j0 + j) * ldw + k)
                                              : make_uint4(0, 0, 0, 0);
    }
  };
  auto store = [&]() {
#pragma unroll
    for (int u = 0; u < XPER; ++u) {
      const int e = tid + u * kSThreads;
      if (e >= XN) break;
      const int r = e / (kVK / V), kk = (e % (kVK / V)) * V;
      float f[V];
      unpack16(xr[u], f, (const XT*)nullptr);
#pragma unroll
      for (int v = 0; v < V; ++v) Xs[r * kVP + kk + v] = f[v];
    }
#pragma unroll
    for (int u = 0; u < WPER; ++u) {
      const int e = tid + u * kSThreads;
      if (e >= WN) break;
      const int j = e / (kVK / V), kk = (e % (kVK / V)) * V;
      float f[V];
      unpack16(wr[u], f, (const XT*)nullptr);
#pragma unroll
      for (int v = 0; v < V; ++v) Ws[j * kVP + kk + v] = f[v];
    }
  };
  load(0);
  for (int64_t kc = 0; kc < d; kc += kVK) {
    store();
    __syncthreads();
    if (kc + kVK < d) load(kc + kVK);  // next chunk in flight during this one's math
    if (ss_s && j0 == 0 && tid < kSR * 8) {
      const int r = tid >> 3, part = tid & 7;
      float sq = 0.f;
#pragma unroll
      for (int u = 0; u < kVK / 8; ++u) {
        const float x = Xs[r * kVP + part * (kVK / 8) + u];
        sq = fmaf(x, x, sq);
      }
      sq += __shfl_xor_sync(0xffffffffu, sq, 1);
      sq += __shfl_xor_sync(0xffffffffu, sq, 2);
      sq += __shfl_xor_sync(0xffffffffu, sq, 4);
      if (part == 0) ss_s[r] += sq;
    }
#pragma unroll 4
    for (int kk = 0; kk < kVK; kk += 4) {
      const float4 x0 = *reinterpret_cast<const float4*>(Xs + ty * kVP + kk);
      const float4 x1 = *reinterpret_cast<const float4*>(Xs + (ty + 8) * kVP + kk);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const float4 w = *reinterpret_cast<const float4*>(Ws + (tx + 32 * c) * kVP + kk);
        acc[0][c] = fmaf(x0.x, w.x, acc[0][c]);
        acc[0][c] = fmaf(x0.y, w.y, acc[0][c]);
        acc[0][c] = fmaf(x0.z, w.z, acc[0][c]);
        acc[0][c] = fmaf(x0.w, w.w, acc[0][c]);
        acc[1][c] = fmaf(x1.x, w.x, acc[1][c]);
        acc[1][c] = fmaf(x1.y, w.y, acc[1][c]);
        acc[1][c] = fmaf(x1.z, w.z, acc[1][c]);
        acc[1][c] = fmaf(x1.w, w.w, acc[1][c]);
      }
    }
    __syncthreads();
  }
}

struct SimtParams {
  int64_t n_host;
  const int64_t* n_dev;
  int32_t d, b;
  int64_t ld_h;
  const void* h;
  const int64_t* row_idx;
  int32_t ids_from_rows;
  const void* w_down;
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
};

template <typename XT, bool kVec>
__global__ void __launch_bounds__(kSThreads) route_simt_kernel(const SimtParams p) {
  // scalar path: [kSR][kSK + 1] and [kSJ][kSK + 1]; vector path: rows of kVP
  extern __shared__ float sm_f[];
  float (*Xs)[kSK + 1] = reinterpret_cast<float (*)[kSK + 1]>(sm_f);
  float (*Ws)[kSK + 1] = reinterpret_cast<float (*)[kSK + 1]>(sm_f + kSR * (kSK + 1));
  __shared__ float ss_s[kSR];
  __shared__ float t_s[kSR];
  __shared__ const XT* xrow[kSR];
  __shared__ uint32_t bits_s;
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
  const int64_t n = p.n_dev ? *p.n_dev : p.n_host;
  const uint32_t tag = launch_tag(p.ws);
  const int64_t nblk = (n + kSR - 1) / kSR;
  const XT* h = reinterpret_cast<const XT*>(p.h);
  const XT* W = reinterpret_cast<const XT*>(p.w_down);
  const bool gathered = p.row_idx != nullptr;
  for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
    const int64_t r0 = blk * kSR;
    if (tid < kSR) {
      const int64_t r = r0 + tid;
      xrow[tid] = r < n ? h + (gathered ? p.row_idx[r] : r) * p.ld_h : nullptr;
      ss_s[tid] = 0.f;
      t_s[tid] = 0.f;
    }
    __syncthreads();
    for (int j0 = 0; j0 < p.b; j0 += kSJ) {
      float acc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
      if (kVec)
        gemm_16x128_vec<XT>(xrow, W, p.d, j0, p.b, p.d, acc, sm_f, sm_f + kSR * kVP, ss_s);
      else
        gemm_16x128<XT>(xrow, W, p.d, j0, p.b, 0, p.d, acc, Xs, Ws, ss_s);
      // all of ss_s is final after the first pass (j0 == 0) completed
#pragma unroll
      for (int r2 = 0; r2 < 2; ++r2) {
        const int r = ty + 8 * r2;
        const float scale = rms_scale(ss_s[r], p.inv_d, p.eps);
        float part = 0.f;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int j = j0 + tx + 32 * c;
          if (j < p.b) part = fmaf(p.w_up[j], silu_f32(__fmul_rn(acc[r2][c], scale)), part);
        }
        part = warp_sum_f32(part);
        if (tx == 0) t_s[r] += part;
      }
      __syncthreads();
    }
    // finalize rows (warp 0), ballot the exit bits
    if (ty == 0) {
      const int64_t r = r0 + tx;
      bool ex = false;
      if (tx < kSR && r < n) {
        const float t = t_s[tx];
        const float score = score_from_logit(t);
        ex = score > p.theta;
        if (p.scores) p.scores[r] = score;
        if (p.logits) p.logits[r] = t;
        if (p.mask) p.mask[r] = ex ? 1 : 0;
        if (ex && p.exit_layers) p.exit_layers[gathered ? p.row_idx[r] : r] = p.layer;
      }
      const uint32_t bits = __ballot_sync(0xffffffffu, ex);
      if (p.exit_idx || p.cont_idx || p.counts) {
        const uint32_t agg = __popc(bits);
        const uint32_t E = lookback_exclusive(p.ws->status, tag, blk, agg);
        if (tx < kSR && r < n) {
          const int64_t rank = (int64_t)E + __popc(bits & ((1u << tx) - 1u));
          const int64_t id = (p.ids_from_rows && gathered) ? p.row_idx[r] : r;
          if (ex) {
            if (p.exit_idx) p.exit_idx[rank] = id;
          } else if (p.cont_idx) {
            p.cont_idx[r - rank] = id;
          }
        }
        if (blk == nblk - 1 && tx == 0 && p.counts) {
          p.counts[0] = (int64_t)E + agg;
          p.counts[1] = n - ((int64_t)E + agg);
        }
      }
      (void)bits_s;
    }
    __syncthreads();
  }
  if (nblk == 0 && blockIdx.x == 0 && tid == 0 && p.counts) {
    p.counts[0] = 0;
    p.counts[1] = 0;
  }
  __syncthreads();
  if (tid == 0) launch_done(p.ws);
}

// Wide variant for many rows (vector path only): 64 rows per CTA, each thread
// 8 rows x 4 bottleneck columns (warp w: rows w, w+8, ..., so the X operand
// is a broadcast read), 128 FMAs per 12 LDS.128 instead of 32 per 6 — the
// 16-row kernel is shared-memory-bound, this one is FMA-bound.  Same
// numerics per output (f32 products, k order).
constexpr int kWR = 64;
constexpr int kWRT = kWR / 8;  // rows per thread
constexpr size_t kWSmem = (size_t)(kWR + kSJ) * kVP * sizeof(float);

template <typename XT>
__device__ __forceinline__ void gemm_wide(const XT* const* xrow, const XT* W, int64_t ldw, int j0,
                                          int b, int64_t d, float (&acc)[kWRT][4], float* Xs,
                                          float* Ws, float* ss_s) {
  constexpr int V = Vec16<XT>::N;
  constexpr int XN = kWR * kVK / V, WN = kSJ * kVK / V;
  constexpr int XPER = XN / kSThreads, WPER = WN / kSThreads;
  static_assert(XN % kSThreads == 0 && WN % kSThreads == 0, "tile pieces");
  const int tid = threadIdx.x;
  const int tx = tid & 31, ty = tid >> 5;
  uint4 xr[XPER], wr[WPER];
  auto load = [&](int64_t kc) {
#pragma unroll
    for (int u = 0; u < XPER; ++u) {
      const int e = tid + u * kSThreads;
      const int r = e / (kVK / V), kk = (e % (kVK / V)) * V;
      const int64_t k = kc + kk;
      xr[u] = (xrow[r] && k < d) ? ld_nc_v4(xrow[r] + k) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < WPER; ++u) {
      const int e = tid + u * kSThreads;
      const int j = e / (kVK / V), kk = (e % (kVK / V)) * V;
      const int64_t k = kc + kk;
      wr[u] = (j0 + j < b && k < d) ? ld_nc_v4(W + (int64_t)(j0 + j) * ldw + k)
                                    : make_uint4(0, 0, 0, 0);
    }
  };
  auto store = [&]() {
#pragma unroll
    for (int u = 0; u < XPER; ++u) {
      const int e = tid + u * kSThreads;
      const int r = e / (kVK / V), kk = (e % (kVK / V)) * V;
      float f[V];
      unpack16(xr[u], f, (const XT*)nullptr);
#pragma unroll
      for (int v = 0; v < V; ++v) Xs[r * kVP + kk + v] = f[v];
    }
#pragma unroll
    for (int u = 0; u < WPER; ++u) {
      const int e = tid + u * kSThreads;
      const int j = e / (kVK / V), kk = (e % (kVK / V)) * V;
      float f[V];
      unpack16(wr[u], f, (const XT*)nullptr);
#pragma unroll
      for (int v = 0; v < V; ++v) Ws[j * kVP + kk + v] = f[v];
    }
  };
  load(0);
  for (int64_t kc = 0; kc < d; kc += kVK) {
    store();
    __syncthreads();
    if (kc + kVK < d) load(kc + kVK);
    if (ss_s && j0 == 0) {
#pragma unroll
      for (int e = tid; e < kWR * 8; e += kSThreads) {
        const int r = e >> 3, part = e & 7;
        float sq = 0.f;
#pragma unroll
        for (int u = 0; u < kVK / 8; ++u) {
          const float x = Xs[r * kVP + part * (kVK / 8) + u];
          sq = fmaf(x, x, sq);
        }
        sq += __shfl_xor_sync(0xffffffffu, sq, 1);
        sq += __shfl_xor_sync(0xffffffffu, sq, 2);
        sq += __shfl_xor_sync(0xffffffffu, sq, 4);
        if (part == 0) ss_s[r] += sq;
      }
    }
#pragma unroll
    for (int kk = 0; kk < kVK; kk += 4) {
      float4 w[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) w[c] = *reinterpret_cast<const float4*>(Ws + (tx + 32 * c) * kVP + kk);
#pragma unroll
      for (int i = 0; i < kWRT; ++i) {
        const float4 x = *reinterpret_cast<const float4*>(Xs + (ty + 8 * i) * kVP + kk);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          acc[i][c] = fmaf(x.x, w[c].x, acc[i][c]);
          acc[i][c] = fmaf(x.y, w[c].y, acc[i][c]);
          acc[i][c] = fmaf(x.z, w[c].z, acc[i][c]);
          acc[i][c] = fmaf(x.w, w[c].w, acc[i][c]);
        }
      }
    }
    __syncthreads();
  }
}

template <typename XT>
__global__ void __launch_bounds__(kSThreads, 1) route_simt_wide_kernel(const SimtParams p) {
  extern __shared__ float sm_f[];
  __shared__ float ss_s[kWR];
  __shared__ float t_s[kWR];
  __shared__ const XT* xrow[kWR];
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
  const int64_t n = p.n_dev ? *p.n_dev : p.n_host;
  const uint32_t tag = launch_tag(p.ws);
  const int64_t nblk = (n + kWR - 1) / kWR;
  const XT* h = reinterpret_cast<const XT*>(p.h);
  const XT* W = reinterpret_cast<const XT*>(p.w_down);
  const bool gathered = p.row_idx != nullptr;
  for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
    const int64_t r0 = blk * kWR;
    if (tid < kWR) {
      const int64_t r = r0 + tid;
      xrow[tid] = r < n ? h + (gathered ? p.row_idx[r] : r) * p.ld_h : nullptr;
      ss_s[tid] = 0.f;
      t_s[tid] = 0.f;
    }
    __syncthreads();
    for (int j0 = 0; j0 < p.b; j0 += kSJ) {
      float acc[kWRT][4];
#pragma unroll
      for (int i = 0; i < kWRT; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
      gemm_wide<XT>(xrow, W, p.d, j0, p.b, p.d, acc, sm_f, sm_f + kWR * kVP, ss_s);
#pragma unroll
      for (int i = 0; i < kWRT; ++i) {
        const int r = ty + 8 * i;
        const float scale = rms_scale(ss_s[r], p.inv_d, p.eps);
        float part = 0.f;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int j = j0 + tx + 32 * c;
          if (j < p.b) part = fmaf(p.w_up[j], silu_f32(__fmul_rn(acc[i][c], scale)), part);
        }
        part = warp_sum_f32(part);
        if (tx == 0) t_s[r] += part;
      }
      __syncthreads();
    }
    if (ty == 0) {
      // two 32-row words: decisions, then one look-back for the block
      uint32_t bits[2];
      bool exr[2];
#pragma unroll
      for (int w = 0; w < 2; ++w) {
        const int64_t r = r0 + 32 * w + tx;
        bool ex = false;
        if (r < n) {
          const float t = t_s[32 * w + tx];
          const float score = score_from_logit(t);
          ex = score > p.theta;
          if (p.scores) p.scores[r] = score;
          if (p.logits) p.logits[r] = t;
          if (p.mask) p.mask[r] = ex ? 1 : 0;
          if (ex && p.exit_layers) p.exit_layers[gathered ? p.row_idx[r] : r] = p.layer;
        }
        exr[w] = ex;
        bits[w] = __ballot_sync(0xffffffffu, ex);
      }
      if (p.exit_idx || p.cont_idx || p.counts) {
        const uint32_t agg = __popc(bits[0]) + __popc(bits[1]);
        const uint32_t E = lookback_exclusive(p.ws->status, tag, blk, agg);
        const uint32_t lt = (1u << tx) - 1u;
#pragma unroll
        for (int w = 0; w < 2; ++w) {
          const int64_t r = r0 + 32 * w + tx;
          if (r < n) {
            const int64_t rank = (int64_t)E + (w ? __popc(bits[0]) : 0) + __popc(bits[w] & lt);
            const int64_t id = (p.ids_from_rows && gathered) ? p.row_idx[r] : r;
            if (exr[w]) {
              if (p.exit_idx) p.exit_idx[rank] = id;
            } else if (p.cont_idx) {
              p.cont_idx[r - rank] = id;
            }
          }
        }
        if (blk == nblk - 1 && tx == 0 && p.counts) {
          p.counts[0] = (int64_t)E + agg;
          p.counts[1] = n - ((int64_t)E + agg);
        }
      }
    }
    __syncthreads();
  }
  if (nblk == 0 && blockIdx.x == 0 && tid == 0 && p.counts) {
    p.counts[0] = 0;
    p.counts[1] = 0;
  }
  __syncthreads();
  if (tid == 0) launch_done(p.ws);
}

// Chain tail for f32 rows (tide_route_tail): the live rows (row_idx[0 ..
// *n_dev)) scored against C checkpoints in ONE launch (grid.y = checkpoint),
// scores [C, cap]; the resolve kernel (route_tcs.cu) then picks each row's
// first firing checkpoint.  Nothing is routed when *n_dev > n_limit.
constexpr int kSimtTailC = 32;
struct SimtTailParams {
  SimtParams base;
  const void* hs[kSimtTailC];
  const void* ws[kSimtTailC];
  const float* wups[kSimtTailC];
  int64_t cap, n_limit, n_min;
};

template <typename XT>
__global__ void __launch_bounds__(kSThreads) route_simt_tail_kernel(const __grid_constant__ SimtTailParams tp) {
  const SimtParams& p = tp.base;
  extern __shared__ float sm_f[];
  __shared__ float ss_s[kSR];
  __shared__ float t_s[kSR];
  __shared__ const XT* xrow[kSR];
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
  const int c = blockIdx.y;
  const int64_t n = *p.n_dev;
  if (n > tp.n_limit || n < tp.n_min) return;
  const XT* h = reinterpret_cast<const XT*>(tp.hs[c]);
  const XT* W = reinterpret_cast<const XT*>(tp.ws[c]);
  const float* w_up = tp.wups[c];
  const int64_t nblk = (n + kSR - 1) / kSR;
  for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
    const int64_t r0 = blk * kSR;
    if (tid < kSR) {
      const int64_t r = r0 + tid;
      xrow[tid] = r < n ? h + p.row_idx[r] * p.ld_h : nullptr;
      ss_s[tid] = 0.f;
      t_s[tid] = 0.f;
    }
    __syncthreads();
    for (int j0 = 0; j0 < p.b; j0 += kSJ) {
      float acc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
      gemm_16x128_vec<XT>(xrow, W, p.d, j0, p.b, p.d, acc, sm_f, sm_f + kSR * kVP, ss_s);
#pragma unroll
      for (int r2 = 0; r2 < 2; ++r2) {
        const int r = ty + 8 * r2;
        const float scale = rms_scale(ss_s[r], p.inv_d, p.eps);
        float part = 0.f;
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          const int j = j0 + tx + 32 * cc;
          if (j < p.b) part = fmaf(w_up[j], silu_f32(__fmul_rn(acc[r2][cc], scale)), part);
        }
        part = warp_sum_f32(part);
        if (tx == 0) t_s[r] += part;
      }
      __syncthreads();
    }
    if (ty == 0 && tx < kSR && r0 + tx < n)
      p.scores[(size_t)c * tp.cap + r0 + tx] = score_from_logit(t_s[tx]);
    __syncthreads();
  }
}

// Same, 64 rows per CTA (gemm_wide): fewer, FMA-bound CTAs.
template <typename XT>
__global__ void __launch_bounds__(kSThreads, 1) route_simt_tail_wide_kernel(const __grid_constant__ SimtTailParams tp) {
  const SimtParams& p = tp.base;
  extern __shared__ float sm_f[];
  __shared__ float ss_s[kWR];
  __shared__ float t_s[kWR];
  __shared__ const XT* xrow[kWR];
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
  const int c = blockIdx.y;
  const int64_t n = *p.n_dev;
  if (n > tp.n_limit || n < tp.n_min) return;
  const XT* h = reinterpret_cast<const XT*>(tp.hs[c]);
  const XT* W = reinterpret_cast<const XT*>(tp.ws[c]);
  const float* w_up = tp.wups[c];
  const int64_t nblk = (n + kWR - 1) / kWR;
  for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
    const int64_t r0 = blk * kWR;
    if (tid < kWR) {
      const int64_t r = r0 + tid;
      xrow[tid] = r < n ? h + p.row_idx[r] * p.ld_h : nullptr;
      ss_s[tid] = 0.f;
      t_s[tid] = 0.f;
    }
    __syncthreads();
    for (int j0 = 0; j0 < p.b; j0 += kSJ) {
      float acc[kWRT][4];
#pragma unroll
      for (int i = 0; i < kWRT; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
      gemm_wide<XT>(xrow, W, p.d, j0, p.b, p.d, acc, sm_f, sm_f + kWR * kVP, ss_s);
#pragma unroll
      for (int i = 0; i < kWRT; ++i) {
        const int r = ty + 8 * i;
        const float scale = rms_scale(ss_s[r], p.inv_d, p.eps);
        float part = 0.f;
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          const int j = j0 + tx + 32 * cc;
          if (j < p.b) part = fmaf(w_up[j], silu_f32(__fmul_rn(acc[i][cc], scale)), part);
        }
        part = warp_sum_f32(part);
        if (tx == 0) t_s[r] += part;
      }
      __syncthreads();
    }
    if (tid < kWR && r0 + tid < n) p.scores[(size_t)c * tp.cap + r0 + tid] = score_from_logit(t_s[tid]);
    __syncthreads();
  }
}

int route_simt_tail_launch(const RouteArgs& a, int C, const void* const* h_ptrs,
                           const void* const* w_ptrs, const float* const* wup_ptrs,
                           const int64_t* layers, int64_t n_limit, int64_t* tail_count,
                           unsigned long long cond, cudaStream_t stream) {
  if (C < 1 || C > kSimtTailC) return set_error(TIDE_ERR_ARG, "tail: C must be in [1, %d]", kSimtTailC);
  if (a.d % 4 || a.ld_h % 4) return set_error(TIDE_ERR_UNSUPPORTED, "f32 tail: d and ld_h must be multiples of 4");
  SimtTailParams tp{};
  SimtParams& p = tp.base;
  p.n_dev = a.n_dev;
  p.d = a.d;
  p.b = a.b;
  p.ld_h = a.ld_h;
  p.row_idx = a.row_idx;
  p.eps = a.eps;
  p.inv_d = (float)(1.0 / (double)a.d);
  p.theta = a.theta;
  p.scores = a.scores;
  for (int c = 0; c < C; ++c) {
    tp.hs[c] = h_ptrs[c];
    tp.ws[c] = w_ptrs[c];
    tp.wups[c] = wup_ptrs[c];
  }
  tp.cap = a.n;
  tp.n_limit = std::min<int64_t>(n_limit, a.n);
  tp.n_min = a.n_min;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(route_simt_tail_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kVSmem);
    cudaFuncSetAttribute(route_simt_tail_wide_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kWSmem);
    attr = true;
  }
  const char* wenv = getenv("TIDE_F32_TAIL_WIDE");
  const bool wide = wenv ? wenv[0] == '1' : true;
  int rc;
  if (wide) {
    const int64_t nblk = std::max<int64_t>(1, (tp.n_limit + kWR - 1) / kWR);
    route_simt_tail_wide_kernel<float><<<dim3((unsigned)nblk, (unsigned)C), kSThreads, kWSmem, stream>>>(tp);
    rc = check_launch("route_simt_tail_wide_kernel");
  } else {
    const int64_t nblk = std::max<int64_t>(1, (tp.n_limit + kSR - 1) / kSR);
    route_simt_tail_kernel<float><<<dim3((unsigned)nblk, (unsigned)C), kSThreads, kVSmem, stream>>>(tp);
    rc = check_launch("route_simt_tail_kernel");
  }
  if (rc) return rc;
  return chain_resolve_launch((const float*)a.scores, a.n, C, layers, a.theta, a.n_dev,
                              tp.n_min, tp.n_limit, a.row_idx, a.exit_layers, tail_count, cond, stream);
}

int route_simt_launch(const RouteArgs& a, cudaStream_t stream) {
  if (a.b < 1 || a.d < 1) return set_error(TIDE_ERR_ARG, "empty router");
  SimtParams p{};
  p.n_host = a.n;
  p.n_dev = a.n_dev;
  p.d = a.d;
  p.b = a.b;
  p.ld_h = a.ld_h;
  p.h = a.h;
  p.row_idx = a.row_idx;
  p.ids_from_rows = a.ids_from_rows;
  p.w_down = a.w_down;
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
  int dev = 0;
  cudaGetDevice(&dev);
  const int64_t nblk = (a.n + kSR - 1) / kSR;
  if (nblk > kMaxParts / 2) return set_error(TIDE_ERR_UNSUPPORTED, "too many rows for one launch");
  // vector path when every 16-byte load is aligned
  const int vw = a.dtype == TIDE_F32 ? 4 : 8;
  const bool vec = a.d % vw == 0 && a.ld_h % vw == 0 &&
                   ((reinterpret_cast<uintptr_t>(a.h) | reinterpret_cast<uintptr_t>(a.w_down)) & 15) == 0;
  const size_t smem = vec ? kVSmem : (size_t)(kSR + kSJ) * (kSK + 1) * sizeof(float);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(route_simt_kernel<float, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kVSmem);
    cudaFuncSetAttribute(route_simt_kernel<__nv_bfloat16, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kVSmem);
    cudaFuncSetAttribute(route_simt_kernel<__half, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kVSmem);
    attr = true;
  }
  void (*kern)(const SimtParams) = nullptr;
  // many rows: the 64-row FMA-bound kernel once it still fills every SM
  static bool wide_attr = false;
  if (!wide_attr) {
    cudaFuncSetAttribute(route_simt_wide_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kWSmem);
    cudaFuncSetAttribute(route_simt_wide_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kWSmem);
    cudaFuncSetAttribute(route_simt_wide_kernel<__half>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kWSmem);
    wide_attr = true;
  }
  const char* wenv = getenv("TIDE_SIMT_WIDE_ROWS");
  // measured (tools/tf32_probe.py, f32): 8,192 x 768 100 -> 64 us, 65,536 x
  // 4096 3.26 -> 1.87 ms; at 2,048 rows (32 CTAs) the 16-row kernel wins
  const int64_t wide_rows = wenv ? atoll(wenv) : (int64_t)sm_count(dev) * 48;
  if (vec && a.n >= wide_rows) {
    switch (a.dtype) {
      case TIDE_F32: kern = route_simt_wide_kernel<float>; break;
      case TIDE_BF16: kern = route_simt_wide_kernel<__nv_bfloat16>; break;
      default: kern = route_simt_wide_kernel<__half>; break;
    }
    const int64_t wblk = (a.n + kWR - 1) / kWR;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kSThreads, kWSmem) !=
            cudaSuccess || per_sm < 1)
      per_sm = 1;
    const int wgrid = (int)std::max<int64_t>(1, std::min<int64_t>(wblk, (int64_t)sm_count(dev) * per_sm));
    kern<<<wgrid, kSThreads, kWSmem, stream>>>(p);
    return check_launch("route_simt_wide_kernel");
  }
  switch (a.dtype) {
    case TIDE_F32: kern = vec ? route_simt_kernel<float, true> : route_simt_kernel<float, false>; break;
    case TIDE_BF16:
      kern = vec ? route_simt_kernel<__nv_bfloat16, true> : route_simt_kernel<__nv_bfloat16, false>;
      break;
    case TIDE_F16: kern = vec ? route_simt_kernel<__half, true> : route_simt_kernel<__half, false>; break;
    default: return set_error(TIDE_ERR_ARG, "bad dtype %d", a.dtype);
  }
  // CTAs walk blocks blk, blk + grid, ... and each block's look-back waits on
  // every lower block: the grid must be fully co-resident, or a CTA spinning
  // on its second block waits for a first block whose CTA cannot be scheduled
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kSThreads, smem) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  const int grid = (int)std::max<int64_t>(
      1, std::min<int64_t>(nblk, (int64_t)sm_count(dev) * std::min(per_sm, 8)));
  kern<<<grid, kSThreads, smem, stream>>>(p);
  return check_launch("route_simt_kernel");
}

}  // namespace tide
