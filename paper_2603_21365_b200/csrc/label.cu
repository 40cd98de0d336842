// K4: calibration labeller — per-token cosine similarity of every checkpoint
// capture against the final capture, in one pass over HBM.
//
//   ee/tensor_math.py:96-113  batched_cosine_similarity (dot, norms, zero
//                             mask, clip to [-1, 1], zero-norm rows -> 0)
//   ee/calibration.py:201-219 compute_labels (label = sim > f32(tau),
//                             zero_norm_count summed over checkpoints)
//
// One warp per token row.  The final row is streamed once per batch of 8
// checkpoints together with the 8 checkpoint rows (9 independent 16-byte
// loads in flight per lane per step), accumulating dot(h_c, f), |h_c|^2 and
// |f|^2 in f32; lane c of the warp finishes checkpoint c.
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>

#include "common.cuh"
#include "internal.h"

namespace tide {

constexpr int kLThreads = 256;
constexpr int kLBatch = 8;
constexpr int kMaxLabelC = 64;

struct LabelParams {
  const void* ck[kMaxLabelC];
  const void* fin;
  int32_t C, d, vec;
  int64_t ld, n;
  float tau;
  float* sims;
  uint8_t* labels_u8;
  float* labels_f32;
  uint8_t* zero_mask;
  unsigned long long* zero_counts;
};

template <typename T>
__global__ void __launch_bounds__(kLThreads, 2) cos_label_kernel(const __grid_constant__ LabelParams p) {
  constexpr int V = 16 / sizeof(T);
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (kLThreads / 32);
  const bool vec = p.vec && (p.d % V == 0) && (p.ld % V == 0);
  for (int64_t i = (int64_t)blockIdx.x * (kLThreads / 32) + (threadIdx.x >> 5); i < p.n;
       i += warps) {
    const T* f = reinterpret_cast<const T*>(p.fin) + i * p.ld;
    float ssf = 0.f;
    for (int cb = 0; cb < p.C; cb += kLBatch) {
      float dot[kLBatch], ssh[kLBatch];
      const T* hp[kLBatch];
#pragma unroll
      for (int c = 0; c < kLBatch; ++c) {
        dot[c] = 0.f;
        ssh[c] = 0.f;
        hp[c] = (cb + c < p.C) ? reinterpret_cast<const T*>(p.ck[cb + c]) + i * p.ld : nullptr;
      }
      const bool first = cb == 0;
      if (vec && sizeof(T) == 2) {
        // bf16 / f16: mixed-precision FMAs straight on the packed pairs
        constexpr bool kB = sizeof(T) == 2 && !std::is_same<T, __half>::value;
        // two 16-byte steps per iteration: 18 loads in flight per lane (same
        // per-lane element order as one step at a time -> identical sums)
        auto step = [&](const uint4& fr, const uint4 (&raw)[kLBatch]) {
          const uint32_t fw[4] = {fr.x, fr.y, fr.z, fr.w};
          if (first) {
#pragma unroll
            for (int w = 0; w < 4; ++w) dot2_acc<kB>(fw[w], fw[w], ssf);
          }
#pragma unroll
          for (int c = 0; c < kLBatch; ++c) {
            if (hp[c]) {
              const uint32_t hw[4] = {raw[c].x, raw[c].y, raw[c].z, raw[c].w};
#pragma unroll
              for (int w = 0; w < 4; ++w) {
                dot2_acc<kB>(hw[w], fw[w], dot[c]);
                dot2_acc<kB>(hw[w], hw[w], ssh[c]);
              }
            }
          }
        };
        for (int k = lane * V; k < p.d; k += 64 * V) {
          const int k2 = k + 32 * V;
          const bool two = k2 < p.d;
          const uint4 fr0 = ld_nc_v4(f + k);
          const uint4 fr1 = two ? ld_nc_v4(f + k2) : make_uint4(0, 0, 0, 0);
          uint4 raw0[kLBatch], raw1[kLBatch];
#pragma unroll
          for (int c = 0; c < kLBatch; ++c) {
            raw0[c] = hp[c] ? ld_nc_v4(hp[c] + k) : make_uint4(0, 0, 0, 0);
            raw1[c] = (hp[c] && two) ? ld_nc_v4(hp[c] + k2) : make_uint4(0, 0, 0, 0);
          }
          step(fr0, raw0);
          if (two) step(fr1, raw1);
        }
      } else if (vec) {
        for (int k = lane * V; k < p.d; k += 32 * V) {
          float fv[V];
          unpack16(ld_nc_v4(f + k), fv, (const T*)nullptr);
          if (first) {
#pragma unroll
            for (int e = 0; e < V; ++e) ssf = fmaf(fv[e], fv[e], ssf);
          }
          uint4 raw[kLBatch];
#pragma unroll
          for (int c = 0; c < kLBatch; ++c)
            if (hp[c]) raw[c] = ld_nc_v4(hp[c] + k);
#pragma unroll
          for (int c = 0; c < kLBatch; ++c) {
            if (hp[c]) {
              float hv[V];
              unpack16(raw[c], hv, (const T*)nullptr);
#pragma unroll
              for (int e = 0; e < V; ++e) {
                dot[c] = fmaf(hv[e], fv[e], dot[c]);
                ssh[c] = fmaf(hv[e], hv[e], ssh[c]);
              }
            }
          }
        }
      } else {
        for (int k = lane; k < p.d; k += 32) {
          const float fv = to_f32<T>(f[k]);
          if (first) ssf = fmaf(fv, fv, ssf);
#pragma unroll
          for (int c = 0; c < kLBatch; ++c) {
            if (hp[c]) {
              const float hv = to_f32<T>(hp[c][k]);
              dot[c] = fmaf(hv, fv, dot[c]);
              ssh[c] = fmaf(hv, hv, ssh[c]);
            }
          }
        }
      }
      if (first) ssf = warp_sum_f32(ssf);
      float my_dot = 0.f, my_ss = 0.f;
#pragma unroll
      for (int c = 0; c < kLBatch; ++c) {
        const float dsum = warp_sum_f32(dot[c]);
        const float ssum = warp_sum_f32(ssh[c]);
        if (lane == c) {
          my_dot = dsum;
          my_ss = ssum;
        }
      }
      const int c = cb + lane;
      if (lane < kLBatch && c < p.C) {
        const float na = __fsqrt_rn(my_ss);
        const float nb = __fsqrt_rn(ssf);
        const bool zero = (na == 0.0f) || (nb == 0.0f);
        float s = 0.0f;
        if (!zero) s = fminf(1.0f, fmaxf(-1.0f, __fdiv_rn(my_dot, __fmul_rn(na, nb))));
        const int64_t o = (int64_t)c * p.n + i;
        if (p.sims) p.sims[o] = s;
        const bool lab = s > p.tau;
        if (p.labels_u8) p.labels_u8[o] = lab ? 1 : 0;
        if (p.labels_f32) p.labels_f32[o] = lab ? 1.0f : 0.0f;
        if (p.zero_mask) p.zero_mask[o] = zero ? 1 : 0;
        if (zero && p.zero_counts) atomicAdd(&p.zero_counts[c], 1ull);
      }
    }
  }
}

}  // namespace tide

using namespace tide;

extern "C" int tide_cos_label(const void* const* ckpt_ptrs, int32_t C, const void* final_h,
                              int64_t ld, int32_t dtype, int64_t n, int32_t d, float tau,
                              float* sims, uint8_t* labels_u8, float* labels_f32,
                              uint8_t* zero_mask, int64_t* zero_counts, void* stream) {
  if (C < 1 || C > kMaxLabelC || d < 1 || n < 0 || !final_h || !ckpt_ptrs)
    return set_error(TIDE_ERR_ARG, "tide_cos_label: bad arguments (C in [1, %d])", kMaxLabelC);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (zero_counts) {
    if (cudaMemsetAsync(zero_counts, 0, sizeof(int64_t) * C, s) != cudaSuccess)
      return set_error(TIDE_ERR_CUDA, "memset zero_counts failed");
  }
  if (n == 0) return TIDE_OK;
  LabelParams p{};
  for (int c = 0; c < C; ++c) {
    if (!ckpt_ptrs[c]) return set_error(TIDE_ERR_ARG, "null checkpoint pointer %d", c);
    p.ck[c] = ckpt_ptrs[c];
  }
  p.fin = final_h;
  p.vec = (reinterpret_cast<uintptr_t>(final_h) & 15) == 0;
  for (int c = 0; c < C; ++c)
    if (reinterpret_cast<uintptr_t>(ckpt_ptrs[c]) & 15) p.vec = 0;
  p.C = C;
  p.d = d;
  p.ld = ld;
  p.n = n;
  p.tau = tau;
  p.sims = sims;
  p.labels_u8 = labels_u8;
  p.labels_f32 = labels_f32;
  p.zero_mask = zero_mask;
  p.zero_counts = reinterpret_cast<unsigned long long*>(zero_counts);
  int dev = 0;
  cudaGetDevice(&dev);
  const int64_t blocks = (n + (kLThreads / 32) - 1) / (kLThreads / 32);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(blocks, (int64_t)sm_count(dev) * 8));
  switch (dtype) {
    case TIDE_F32: cos_label_kernel<float><<<grid, kLThreads, 0, s>>>(p); break;
    case TIDE_BF16: cos_label_kernel<__nv_bfloat16><<<grid, kLThreads, 0, s>>>(p); break;
    case TIDE_F16: cos_label_kernel<__half><<<grid, kLThreads, 0, s>>>(p); break;
    default: return set_error(TIDE_ERR_ARG, "bad dtype %d", dtype);
  }
  return check_launch("cos_label_kernel");
}
