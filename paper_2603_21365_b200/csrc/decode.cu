// K5: the decode step — every checkpoint router for n <= 16 rows in ONE
// launch, plus the exit resolution of posthoc_select (ee/runtime.py:151-178).
//
// Weight-streaming GEMV: the step is bound by W_down bytes (C x b x d x e,
// 9.4 MB for Qwen3-8B's 9 checkpoints) not by the 8 hidden rows.  CTA
// (checkpoint c, slice s) owns a few bottleneck rows of W_c; its warps split
// d, each streaming its slab of W and of the hidden rows once.  Per-slice partial logits
// (sum_j w_up_j SiLU(a_j)) go to the workspace; the last CTA of a checkpoint
// (atomic ticket) reduces them in fixed slice order (deterministic), and the
// last checkpoint to finish resolves per-token / batch-unanimous exits.
#include <cuda_runtime.h>

#include <algorithm>

#include "common.cuh"
#include "internal.h"

namespace tide {

namespace {

constexpr int kDThreads = 256;
constexpr int kDWarps = kDThreads / 32;
constexpr int kDMaxRows = TIDE_MAX_DECODE_ROWS;
constexpr int kDMaxC = kMaxTickets;

struct DecParams {
  const void* h[kDMaxC];
  const void* w[kDMaxC];
  const float* wup[kDMaxC];
  int64_t layers[kDMaxC];
  int32_t C, d, b, slices, rows_per_slice;
  int64_t ld_h, n, k_min;
  int32_t mode;
  float eps, inv_d, theta;
  float* scores;
  float* logits;
  int64_t* exit_layers;
  int64_t* exit_count;
  Workspace* ws;
};

template <typename T>
__device__ __forceinline__ void load_vec(const T* p, float (&f)[16 / sizeof(T)]) {
  unpack16(*reinterpret_cast<const uint4*>(p), f, (const T*)nullptr);
}

// CTA (checkpoint c, slice s): JR bottleneck rows of W_c, all NR tokens.
// Warp w owns the K range [w*d/8, (w+1)*d/8): it streams its JR x (d/8) slab
// of W and the NR x (d/8) slab of the hidden rows exactly once (16-byte loads),
// accumulating JR x NR dot products and NR sums of squares per lane; the
// partial sums are reduced across lanes (shuffles) and warps (smem) in a fixed
// order.
template <typename T, int NR, int JR>
__global__ void __launch_bounds__(kDThreads) decode_kernel(const __grid_constant__ DecParams p) {
  constexpr int V = 16 / sizeof(T);
  __shared__ float red_s[kDWarps][JR * NR + NR];
  __shared__ float a_s[JR][NR];
  __shared__ float ss_s[NR];
  __shared__ unsigned int last_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x, slice = blockIdx.y;
  const T* h = reinterpret_cast<const T*>(p.h[c]);
  const T* W = reinterpret_cast<const T*>(p.w[c]);
  const int n = (int)p.n;
  const int j0 = slice * JR;
  const int nvec = p.d / V;
  const int v0 = (int)((int64_t)nvec * warp / kDWarps), v1 = (int)((int64_t)nvec * (warp + 1) / kDWarps);
  float acc[JR][NR];
  float ss[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    ss[r] = 0.f;
#pragma unroll
    for (int j = 0; j < JR; ++j) acc[j][r] = 0.f;
  }
  for (int v = v0 + lane; v < v1; v += 32) {
    float wf[JR][V];
#pragma unroll
    for (int j = 0; j < JR; ++j) {
      if (j0 + j < p.b) load_vec<T>(W + (int64_t)(j0 + j) * p.d + (int64_t)v * V, wf[j]);
      else {
#pragma unroll
        for (int e = 0; e < V; ++e) wf[j][e] = 0.f;
      }
    }
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      if (r < n) {
        float xf[V];
        load_vec<T>(h + (int64_t)r * p.ld_h + (int64_t)v * V, xf);
#pragma unroll
        for (int e = 0; e < V; ++e) {
          ss[r] = fmaf(xf[e], xf[e], ss[r]);
#pragma unroll
          for (int j = 0; j < JR; ++j) acc[j][r] = fmaf(wf[j][e], xf[e], acc[j][r]);
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    const float sv = warp_sum_f32(ss[r]);
    if (lane == 0) red_s[warp][JR * NR + r] = sv;
#pragma unroll
    for (int j = 0; j < JR; ++j) {
      const float av = warp_sum_f32(acc[j][r]);
      if (lane == 0) red_s[warp][j * NR + r] = av;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < JR * NR + NR; i += kDThreads) {
    float t = 0.f;
    for (int w = 0; w < kDWarps; ++w) t += red_s[w][i];
    if (i < JR * NR) a_s[i / NR][i % NR] = t;
    else ss_s[i - JR * NR] = t;
  }
  __syncthreads();
  float part[NR];
  if (threadIdx.x < NR) {
    const int r = threadIdx.x;
    const float scale = rms_scale(ss_s[r], p.inv_d, p.eps);
    float t = 0.f;
#pragma unroll
    for (int j = 0; j < JR; ++j)
      if (j0 + j < p.b) t = fmaf(p.wup[c][j0 + j], silu_f32(__fmul_rn(a_s[j][r], scale)), t);
    part[0] = t;
  }
  float* partials = p.ws->partials;
  if (threadIdx.x < NR) partials[((int64_t)c * p.slices + slice) * kDMaxRows + threadIdx.x] = part[0];
  // ticket: the last slice CTA of checkpoint c reduces in fixed slice order
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int prev = atomicAdd(&p.ws->tickets[c], 1u);
    last_s = (prev == (unsigned int)(p.slices - 1)) ? 1u : 0u;
  }
  __syncthreads();
  if (!last_s) return;
  __threadfence();
  if (threadIdx.x < NR && threadIdx.x < n) {
    const int r = threadIdx.x;
    float t = 0.f;
    for (int sl = 0; sl < p.slices; ++sl)
      t += __ldcg(&partials[((int64_t)c * p.slices + sl) * kDMaxRows + r]);
    const float score = score_from_logit(t);
    if (p.scores) p.scores[(int64_t)c * n + r] = score;
    if (p.logits) p.logits[(int64_t)c * n + r] = t;
    p.ws->dec_scores[c * kDMaxRows + r] = score;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    p.ws->tickets[c] = 0;  // reset for the next launch
    const unsigned int prev = atomicAdd(&p.ws->ticket, 1u);
    last_s = (prev == (unsigned int)(p.C - 1)) ? 2u : 0u;
  }
  __syncthreads();
  if (last_s != 2u || warp != 0) return;
  __threadfence();
  // exit resolution: lanes = rows
  const int r = lane;
  int64_t exit_layer = TIDE_NO_EXIT;
  if (p.mode == TIDE_MODE_PER_TOKEN) {
    for (int cc = 0; cc < p.C && r < n; ++cc) {
      if (p.layers[cc] < p.k_min) continue;
      if (__ldcg(&p.ws->dec_scores[cc * kDMaxRows + r]) > p.theta) {
        exit_layer = p.layers[cc];
        break;
      }
    }
  } else {
    for (int cc = 0; cc < p.C; ++cc) {
      if (p.layers[cc] < p.k_min) continue;
      const bool fire = r >= n || __ldcg(&p.ws->dec_scores[cc * kDMaxRows + r]) > p.theta;
      if (__all_sync(0xffffffffu, fire)) {
        exit_layer = p.layers[cc];
        break;
      }
    }
  }
  if (r < n && p.exit_layers) p.exit_layers[r] = exit_layer;
  const uint32_t cnt = __popc(__ballot_sync(0xffffffffu, r < n && exit_layer != TIDE_NO_EXIT));
  if (lane == 0) {
    if (p.exit_count) p.exit_count[0] = cnt;
    p.ws->ticket = 0;
  }
}

template <typename T>
int launch_t(const DecParams& p, cudaStream_t s) {
  if (p.n <= 8) {
    decode_kernel<T, 8, 8><<<dim3(p.C, (p.b + 7) / 8), kDThreads, 0, s>>>(p);
  } else {
    decode_kernel<T, 16, 4><<<dim3(p.C, (p.b + 3) / 4), kDThreads, 0, s>>>(p);
  }
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
  if (!workspace) return set_error(TIDE_ERR_ARG, "workspace required");
  const int V = dtype == TIDE_F32 ? 4 : 8;
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
  // slices of JR bottleneck rows (8 for n <= 8, 4 for n <= 16)
  const int rows_per_slice = n <= 8 ? 8 : 4;
  const int slices = (b + rows_per_slice - 1) / rows_per_slice;
  if ((int64_t)C * slices * kDMaxRows > kMaxPartials)
    return set_error(TIDE_ERR_UNSUPPORTED, "decode problem too large for the workspace");
  p.C = C;
  p.d = d;
  p.b = b;
  p.slices = slices;
  p.rows_per_slice = rows_per_slice;
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
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  switch (dtype) {
    case TIDE_F32: return launch_t<float>(p, s);
    case TIDE_BF16: return launch_t<__nv_bfloat16>(p, s);
    case TIDE_F16: return launch_t<__half>(p, s);
    default: return set_error(TIDE_ERR_ARG, "bad dtype %d", dtype);
  }
}
