// Router training step kernels: the elementwise / per-row
// parts of one minibatch of ee/calibration.py:238-343 on the GPU; the three
// contractions (u = z W^T, d_w_up = g_t a, d_w_down = g_u^T z) are plain
// library GEMMs issued by the host (training.py).
//
//   train_act_kernel  ee/calibration.py:238-260 bce_loss_and_grads, per row:
//                     su = sigma(u), a = u su, t = a . w_up, the BCE term,
//                     g_t = (sigma(t) - y) / n, g_u = g_t w_up su (1 + u (1 - su))
//   adam_kernel       ee/calibration.py:277-290 _Adam.step, elementwise
//
// Every f32 operation is written out with _rn intrinsics in the reference's
// evaluation order (numpy f32 arrays with weakly typed Python scalars), so no
// FMA contraction changes a rounding the reference does not do.
#include <cuda_runtime.h>

#include <algorithm>

#include "common.cuh"
#include "internal.h"

namespace tide {

constexpr int kTrainWarps = 8;

__global__ void __launch_bounds__(32 * kTrainWarps)
    train_act_kernel(const float* __restrict__ u, int64_t rows, int b,
                     const float* __restrict__ w_up, const float* __restrict__ y,
                     float* __restrict__ a_out, float* __restrict__ gu_out,
                     float* __restrict__ gt_out, float* __restrict__ t_out, double* loss_sum) {
  const int lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * kTrainWarps + (threadIdx.x >> 5);
  if (i >= rows) return;
  const float* ur = u + i * b;
  float t = 0.0f;
  for (int j = lane; j < b; j += 32) {
    const float uj = ur[j];
    const float aj = __fmul_rn(uj, sigmoid_f32(uj));
    if (a_out) a_out[i * b + j] = aj;
    t = fmaf(aj, w_up[j], t);
  }
  t = warp_sum_f32(t);
  const float yi = y[i];
  const float gt = __fdiv_rn(__fsub_rn(sigmoid_f32(t), yi), (float)rows);
  if (gu_out) {
    for (int j = lane; j < b; j += 32) {
      const float uj = ur[j];
      const float su = sigmoid_f32(uj);
      // g_a * (su * (1.0 + u * (1.0 - su)))
      const float dsilu = __fmul_rn(su, __fadd_rn(1.0f, __fmul_rn(uj, __fsub_rn(1.0f, su))));
      gu_out[i * b + j] = __fmul_rn(__fmul_rn(gt, w_up[j]), dsilu);
    }
  }
  if (lane == 0) {
    if (gt_out) gt_out[i] = gt;
    if (t_out) t_out[i] = t;
    if (loss_sum) {
      // max(t, 0) - t*y + log1p(exp(-|t|))
      const float term = __fadd_rn(__fsub_rn(fmaxf(t, 0.0f), __fmul_rn(t, yi)),
                                   log1pf(expf(-fabsf(t))));
      atomicAdd(loss_sum, (double)term);
    }
  }
}

__global__ void adam_kernel(float* __restrict__ w, const float* __restrict__ g,
                            float* __restrict__ m, float* __restrict__ v, int64_t count, float b1,
                            float c1, float b2, float c2, const float* __restrict__ bc_table,
                            const int64_t* __restrict__ step_base, int64_t step_offset,
                            float bc1, float bc2, float lr, float eps) {
  if (bc_table) {  // step-dependent bias corrections from device memory (graph replay)
    const int64_t t = *step_base + step_offset;
    bc1 = bc_table[2 * t];
    bc2 = bc_table[2 * t + 1];
  }
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count;
       k += (int64_t)gridDim.x * blockDim.x) {
    const float gk = g[k];
    const float mk = __fadd_rn(__fmul_rn(b1, m[k]), __fmul_rn(c1, gk));
    const float vk = __fadd_rn(__fmul_rn(b2, v[k]), __fmul_rn(c2, __fmul_rn(gk, gk)));
    m[k] = mk;
    v[k] = vk;
    const float mh = __fdiv_rn(mk, bc1);
    const float vh = __fdiv_rn(vk, bc2);
    w[k] = __fsub_rn(w[k], __fdiv_rn(__fmul_rn(lr, mh), __fadd_rn(__fsqrt_rn(vh), eps)));
  }
}

}  // namespace tide

using namespace tide;

extern "C" int tide_train_act(const float* u, int64_t rows, int32_t b, const float* w_up,
                              const float* labels, float* a_out, float* gu_out, float* gt_out,
                              float* t_out, double* loss_sum, void* stream) {
  if (rows < 0 || b < 1) return set_error(TIDE_ERR_ARG, "tide_train_act: bad shape");
  if (rows > 0 && (!u || !w_up || !labels))
    return set_error(TIDE_ERR_ARG, "tide_train_act: null input");
  if (rows == 0) return TIDE_OK;
  const int64_t blocks = (rows + kTrainWarps - 1) / kTrainWarps;
  train_act_kernel<<<(unsigned)blocks, 32 * kTrainWarps, 0, (cudaStream_t)stream>>>(
      u, rows, b, w_up, labels, a_out, gu_out, gt_out, t_out, loss_sum);
  return check_launch("train_act_kernel");
}

extern "C" int tide_adam_step(float* w, const float* g, float* m, float* v, int64_t count,
                              float beta1, float one_minus_beta1, float beta2,
                              float one_minus_beta2, const float* bias_corr_table,
                              const int64_t* step_base, int64_t step_offset, float bias_corr1,
                              float bias_corr2, float lr, float eps, void* stream) {
  if (count < 0) return set_error(TIDE_ERR_ARG, "tide_adam_step: bad count");
  if (bias_corr_table && !step_base)
    return set_error(TIDE_ERR_ARG, "tide_adam_step: bias_corr_table needs step_base");
  if (count > 0 && (!w || !g || !m || !v))
    return set_error(TIDE_ERR_ARG, "tide_adam_step: null buffer");
  if (count == 0) return TIDE_OK;
  int dev = 0;
  cudaGetDevice(&dev);
  const int64_t want = (count + 255) / 256;
  const int grid = (int)std::min<int64_t>(want, (int64_t)sm_count(dev) * 8);
  adam_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(
      w, g, m, v, count, beta1, one_minus_beta1, beta2, one_minus_beta2, bias_corr_table,
      step_base, step_offset, bias_corr1, bias_corr2, lr, eps);
  return check_launch("adam_kernel");
}
