// K3: exit scatter / exit projection and the posthoc output staging.
//
//   exit_scatter    ee/router_ops.py:170-176   out[pos] = rows
//   exit_projection ee/router_ops.py:179-188   out[pos] = rmsnorm(rows, gain, eps)
//   select_project  ee/runtime.py:176,180 + ee/model.py:329-338: every row is
//                   final-normed from the layer it exits at (or the final
//                   capture), producing the LM-head input in one pass.
// rmsnorm follows ee/tensor_math.py:35-49 in f32, bit-exactly (numpy's pairwise
// order for the mean of squares, see np_pairwise_sumsq): x / sqrt(sum(x^2)/d + eps) * gain.
// One warp per row, 16-byte vector loads, the row held in registers between
// the two passes when it fits (d <= 32 lanes x 8 x 4 elements).
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>
#include <cstdlib>

#include "common.cuh"
#include "internal.h"

namespace tide {

constexpr int kPThreads = 256;

// Sum of squares of one row in numpy's order, so the f32 result is bit-equal
// to the reference's np.mean(np.square(x), axis=-1) * d (ee/tensor_math.py:43):
// numpy reduces a contiguous row with FLOAT_pairwise_sum
// (numpy/_core/src/umath/loops_utils.h.src): n < 8 -> sequential; n <= 128 ->
// eight strided accumulators r[j] (j, j+8, ...) combined as
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then the n % 8 tail sequentially;
// else split at n2 = n/2 - (n/2) % 8 and add the two halves.  Each square is
// rounded to f32 first (np.square).  Warp-uniform recursion; the leaf's 8
// chains run on lanes 0-7.  Returns the sum in every lane.
template <typename T>
__device__ __forceinline__ float sq_at(const T* a, int i) {
  const float x = to_f32<T>(a[i]);
  return __fmul_rn(x, x);
}

template <typename T>
__device__ float np_leaf_sumsq(const T* __restrict__ a, int n) {
  const int lane = threadIdx.x & 31;
  float res = 0.0f;
  if (n < 8) {
    if (lane == 0)
      for (int i = 0; i < n; ++i) res = __fadd_rn(res, sq_at<T>(a, i));
  } else {
    const int body = n - (n % 8);
    float r = 0.0f;
    if (lane < 8) {
      r = sq_at<T>(a, lane);
      for (int i = 8 + lane; i < body; i += 8) r = __fadd_rn(r, sq_at<T>(a, i));
    }
    r = __fadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 1));  // r0+r1, r2+r3, ...
    r = __fadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 2));  // (r0+r1)+(r2+r3), ...
    r = __fadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 4));  // both halves
    if (lane == 0) {
      res = r;
      for (int i = body; i < n; ++i) res = __fadd_rn(res, sq_at<T>(a, i));
    }
  }
  return __shfl_sync(0xffffffffu, res, 0);
}

template <typename T>
__device__ __noinline__ float np_pairwise_sumsq(const T* __restrict__ a, int n) {
  if (n <= 128) return np_leaf_sumsq<T>(a, n);
  int n2 = n / 2;
  n2 -= n2 % 8;
  const float lo = np_pairwise_sumsq<T>(a, n2);
  const float hi = np_pairwise_sumsq<T>(a + n2, n - n2);
  return __fadd_rn(lo, hi);
}

// rmsnorm of one row (warp): x / sqrt(f32(sum x^2) / f32(d) + eps) * gain with
// every operation rounded as numpy does it (no FMA contraction): bit-equal to
// ee/tensor_math.py:35-49 on the f32 (or exactly upcast bf16/f16) row.
template <typename T>
__device__ __forceinline__ void norm_row(const T* __restrict__ src, float* __restrict__ dst, int d,
                                         const float* __restrict__ gain, float eps,
                                         int normalize) {
  const int lane = threadIdx.x & 31;
  constexpr int V = 16 / sizeof(T);
  const bool vec = ((reinterpret_cast<uintptr_t>(src) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(dst) & 15) == 0) && (d % V == 0);
  const float ss = normalize ? np_pairwise_sumsq<T>(src, d) : 0.0f;
  const float den = normalize ? __fsqrt_rn(__fadd_rn(__fdiv_rn(ss, (float)d), eps)) : 1.0f;
  if (vec) {
    for (int k = lane * V; k < d; k += 32 * V) {
      float f[V];
      unpack16(*reinterpret_cast<const uint4*>(src + k), f, (const T*)nullptr);
#pragma unroll
      for (int e = 0; e < V; ++e) {
        float y = normalize ? __fdiv_rn(f[e], den) : f[e];
        if (normalize && gain) y = __fmul_rn(y, gain[k + e]);
        f[e] = y;
      }
#pragma unroll
      for (int e = 0; e < V; e += 4)
        *reinterpret_cast<float4*>(dst + k + e) = make_float4(f[e], f[e + 1], f[e + 2], f[e + 3]);
    }
  } else {
    for (int k = lane; k < d; k += 32) {
      float y = to_f32<T>(src[k]);
      if (normalize) {
        y = __fdiv_rn(y, den);
        if (gain) y = __fmul_rn(y, gain[k]);
      }
      dst[k] = y;
    }
  }
}

// The same row as norm_row, written as a bf16 pair y = hi + lo (hi = bf16(y),
// lo = bf16(y - hi)): the A operand of the 3-term tensor-core LM head.
template <typename T>
__device__ __forceinline__ void norm_row_split(const T* __restrict__ src, __nv_bfloat16* __restrict__ hi,
                                               __nv_bfloat16* __restrict__ lo, int d,
                                               const float* __restrict__ gain, float eps) {
  const int lane = threadIdx.x & 31;
  const float ss = np_pairwise_sumsq<T>(src, d);
  const float den = __fsqrt_rn(__fadd_rn(__fdiv_rn(ss, (float)d), eps));
  for (int k = lane; k < d; k += 32) {
    float y = __fdiv_rn(to_f32<T>(src[k]), den);
    if (gain) y = __fmul_rn(y, gain[k]);
    const __nv_bfloat16 h = __float2bfloat16_rn(y);
    hi[k] = h;
    lo[k] = __float2bfloat16_rn(y - __bfloat162float(h));  // y - h is exact in f32
  }
}

template <typename T>
__global__ void __launch_bounds__(kPThreads)
    exit_project_kernel(const T* rows, int64_t ld_rows, const int64_t* src_idx, int64_t n_e_host,
                        const int64_t* n_e_dev, int d, const float* gain, float eps, int normalize,
                        const int64_t* positions, float* out, int64_t ld_out) {
  const int64_t n_e = n_e_dev ? *n_e_dev : n_e_host;
  const int64_t warps = (int64_t)gridDim.x * (kPThreads / 32);
  for (int64_t j = (int64_t)blockIdx.x * (kPThreads / 32) + (threadIdx.x >> 5); j < n_e;
       j += warps) {
    const int64_t s = src_idx ? src_idx[j] : j;
    norm_row<T>(rows + s * ld_rows, out + positions[j] * ld_out, d, gain, eps, normalize);
  }
}

// ---------------------------------------------------------------------------
// Staged form (round 2).  numpy's pairwise order is a fixed tree for a given
// d, so the host lays it out once per launch (PairPlan: the <= 128-element
// leaves in order, and the post-order additions of the leaf / node sums).
// A warp copies its row into shared memory as f32 (coalesced 16-byte loads),
// sums four leaves at a time (8-lane groups, each lane's <= 16 squares
// loaded before its sequential chain), lane 0 replays the additions, and the
// row is normalized from shared memory: one read of the row, no recursion,
// no per-element global latency.  Bit-identical to np_pairwise_sumsq.
constexpr int kPlanLeaves = 256;
constexpr int kStageWarps = 4;
struct PairPlan {
  int32_t L, nops;                  // leaves, additions (L - 1)
  int32_t off[kPlanLeaves];         // leaf k = elements [off, off + len)
  int16_t len[kPlanLeaves];
  int16_t opa[kPlanLeaves], opb[kPlanLeaves];  // slot L + m = slot opa + slot opb
};

static int plan_build(int n, PairPlan& P) {
  // iterative post-order of the recursion in np_pairwise_sumsq
  struct Fr { int off, n, state, left; };
  Fr st[64];
  int sp = 0, L = 0, ops = 0;
  st[sp++] = {0, n, 0, -1};
  // first pass: leaves in order (slots 0..L-1), second: the additions
  // (done together: each frame returns the slot of its sum)
  int16_t ret = -1;
  while (sp) {
    Fr& f = st[sp - 1];
    if (f.n <= 128) {
      if (L >= kPlanLeaves) return -1;
      P.off[L] = f.off;
      P.len[L] = (int16_t)f.n;
      ret = (int16_t)L++;
      --sp;
      continue;
    }
    int n2 = f.n / 2;
    n2 -= n2 % 8;
    if (f.state == 0) {
      f.state = 1;
      st[sp++] = {f.off, n2, 0, -1};
    } else if (f.state == 1) {
      f.left = ret;
      f.state = 2;
      st[sp++] = {f.off + n2, f.n - n2, 0, -1};
    } else {
      if (ops >= kPlanLeaves) return -1;
      P.opa[ops] = (int16_t)f.left;
      P.opb[ops] = ret;
      ret = (int16_t)(kPlanLeaves + ops);  // node slots after the leaf slots
      ++ops;
      --sp;
    }
    if (sp >= 62) return -1;
  }
  P.L = L;
  P.nops = ops;
  return 0;
}

// the warp's shared region: kPlanLeaves leaf slots + kPlanLeaves node slots
// (f32), then the row in its own dtype (16-byte padded)
__host__ __device__ __forceinline__ size_t stage_bytes(int d, int esz) {
  return (size_t)2 * kPlanLeaves * sizeof(float) + (((size_t)d * esz + 15) & ~(size_t)15);
}

template <typename T>
__device__ __forceinline__ void stage_row(const T* __restrict__ src, T* __restrict__ buf, int d) {
  const int lane = threadIdx.x & 31;
  constexpr int V = 16 / sizeof(T);
  if (((reinterpret_cast<uintptr_t>(src) & 15) == 0) && d % V == 0) {
    for (int k = lane * V; k < d; k += 32 * V)
      *reinterpret_cast<uint4*>(buf + k) = ld_nc_v4(src + k);
  } else {
    for (int k = lane; k < d; k += 32) buf[k] = src[k];
  }
  __syncwarp();
}

// 4 consecutive staged elements as f32 (exact upcast)
template <typename T>
__device__ __forceinline__ void lds4(const T* p, float (&f)[4]);
template <>
__device__ __forceinline__ void lds4<float>(const float* p, float (&f)[4]) {
  const float4 x = *reinterpret_cast<const float4*>(p);
  f[0] = x.x;
  f[1] = x.y;
  f[2] = x.z;
  f[3] = x.w;
}
template <>
__device__ __forceinline__ void lds4<__nv_bfloat16>(const __nv_bfloat16* p, float (&f)[4]) {
  const uint2 u = *reinterpret_cast<const uint2*>(p);
  f[0] = __uint_as_float(u.x << 16);
  f[1] = __uint_as_float(u.x & 0xffff0000u);
  f[2] = __uint_as_float(u.y << 16);
  f[3] = __uint_as_float(u.y & 0xffff0000u);
}
template <>
__device__ __forceinline__ void lds4<__half>(const __half* p, float (&f)[4]) {
  f[0] = __half2float(p[0]);
  f[1] = __half2float(p[1]);
  f[2] = __half2float(p[2]);
  f[3] = __half2float(p[3]);
}

// numpy-ordered sum of squares of the staged row; every lane gets it
template <typename T>
__device__ __forceinline__ float sumsq_planned(const T* __restrict__ buf, float* __restrict__ slots,
                                               const PairPlan& P) {
  const int lane = threadIdx.x & 31;
  const int g = lane >> 3, j = lane & 7;
  for (int k0 = 0; k0 < P.L; k0 += 4) {
    const int k = k0 + g;
    const bool valid = k < P.L;
    const int n = valid ? P.len[k] : 8;
    const T* a = buf + (valid ? P.off[k] : 0);
    const int body = n - (n % 8);
    float v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int i = j + 8 * u;
      const float x = (valid && i < body) ? to_f32<T>(a[i]) : 0.0f;
      v[u] = __fmul_rn(x, x);
    }
    float r = v[0];
#pragma unroll
    for (int u = 1; u < 16; ++u)
      if (j + 8 * u < body) r = __fadd_rn(r, v[u]);
    r = __fadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 1));
    r = __fadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 2));
    r = __fadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 4));
    if (valid && j == 0) {
      if (n < 8) {  // numpy: fewer than 8 elements are summed sequentially
        r = 0.0f;
        for (int i = 0; i < n; ++i) {
          const float x = to_f32<T>(a[i]);
          r = __fadd_rn(r, __fmul_rn(x, x));
        }
      } else {
        for (int i = body; i < n; ++i) {
          const float x = to_f32<T>(a[i]);
          r = __fadd_rn(r, __fmul_rn(x, x));
        }
      }
      slots[k] = r;
    }
  }
  __syncwarp();
  float res = 0.0f;
  if (lane == 0) {
    for (int m = 0; m < P.nops; ++m)
      slots[kPlanLeaves + m] = __fadd_rn(slots[P.opa[m]], slots[P.opb[m]]);
    res = P.nops ? slots[kPlanLeaves + P.nops - 1] : slots[0];
  }
  return __shfl_sync(0xffffffffu, res, 0);
}

template <typename T>
__device__ __forceinline__ void norm_row_planned(const T* __restrict__ src, float* __restrict__ dst,
                                                 __nv_bfloat16* __restrict__ hi,
                                                 __nv_bfloat16* __restrict__ lo, int d,
                                                 const float* __restrict__ gain, float eps, int normalize,
                                                 uint8_t* region, const PairPlan& P) {
  const int lane = threadIdx.x & 31;
  float* slots = reinterpret_cast<float*>(region);
  T* buf = reinterpret_cast<T*>(region + 2 * kPlanLeaves * sizeof(float));
  stage_row<T>(src, buf, d);
  const float ss = normalize ? sumsq_planned<T>(buf, slots, P) : 0.0f;
  const float den = normalize ? __fsqrt_rn(__fadd_rn(__fdiv_rn(ss, (float)d), eps)) : 1.0f;
  if (hi) {
    for (int k = lane; k < d; k += 32) {
      float y = __fdiv_rn(to_f32<T>(buf[k]), den);
      if (gain) y = __fmul_rn(y, gain[k]);
      const __nv_bfloat16 h = __float2bfloat16_rn(y);
      hi[k] = h;
      lo[k] = __float2bfloat16_rn(y - __bfloat162float(h));  // y - h is exact in f32
    }
  } else if (((reinterpret_cast<uintptr_t>(dst) & 15) == 0) && d % 4 == 0 &&
             ((reinterpret_cast<uintptr_t>(gain) & 15) == 0)) {
    // 4 elements per step: staged row from shared memory, float4 gains
    // (read-only path), float4 stores
    for (int k = lane * 4; k < d; k += 128) {
      float f[4];
      lds4<T>(buf + k, f);
      if (normalize) {
#pragma unroll
        for (int e = 0; e < 4; ++e) f[e] = __fdiv_rn(f[e], den);
        if (gain) {
          const float4 gv = __ldg(reinterpret_cast<const float4*>(gain + k));
          f[0] = __fmul_rn(f[0], gv.x);
          f[1] = __fmul_rn(f[1], gv.y);
          f[2] = __fmul_rn(f[2], gv.z);
          f[3] = __fmul_rn(f[3], gv.w);
        }
      }
      *reinterpret_cast<float4*>(dst + k) = make_float4(f[0], f[1], f[2], f[3]);
    }
  } else {
    for (int k = lane; k < d; k += 32) {
      float y = normalize ? __fdiv_rn(to_f32<T>(buf[k]), den) : to_f32<T>(buf[k]);
      if (normalize && gain) y = __fmul_rn(y, gain[k]);
      dst[k] = y;
    }
  }
  __syncwarp();  // the region is reused for the warp's next row
}

template <typename T>
__global__ void __launch_bounds__(32 * kStageWarps)
    exit_project_staged_kernel(const T* rows, int64_t ld_rows, const int64_t* src_idx, int64_t n_e_host,
                               const int64_t* n_e_dev, int d, const float* gain, float eps,
                               int normalize, const int64_t* positions, float* out, int64_t ld_out,
                               const __grid_constant__ PairPlan plan) {
  extern __shared__ __align__(16) uint8_t stage_smem[];
  const int64_t n_e = n_e_dev ? *n_e_dev : n_e_host;
  uint8_t* region = stage_smem + (size_t)(threadIdx.x >> 5) * stage_bytes(d, (int)sizeof(T));
  const int64_t warps = (int64_t)gridDim.x * kStageWarps;
  for (int64_t j = (int64_t)blockIdx.x * kStageWarps + (threadIdx.x >> 5); j < n_e; j += warps) {
    const int64_t s = src_idx ? src_idx[j] : j;
    norm_row_planned<T>(rows + s * ld_rows, out + positions[j] * ld_out, nullptr, nullptr, d, gain, eps,
                        normalize, region, plan);
  }
}

constexpr int kMaxPtrs = TIDE_MAX_LAYERS + 1;
struct SelectParams {
  const void* layer[kMaxPtrs];
  int32_t num;
  int64_t ld_h, n, ld_out;
  int32_t d;
  const int64_t* exit_layers;
  const float* gain;
  float eps;
  float* out;
  __nv_bfloat16* out_hi;  // split mode (out == NULL): bf16 pair rows, leading dim ld_out
  __nv_bfloat16* out_lo;
};

template <typename T>
__global__ void __launch_bounds__(kPThreads) select_project_kernel(const __grid_constant__ SelectParams p) {
  const int64_t warps = (int64_t)gridDim.x * (kPThreads / 32);
  for (int64_t i = (int64_t)blockIdx.x * (kPThreads / 32) + (threadIdx.x >> 5); i < p.n;
       i += warps) {
    int64_t src = p.num - 1;
    if (p.exit_layers) {
      const int64_t k = p.exit_layers[i];
      if (k != TIDE_NO_EXIT && k + 1 >= 0 && k + 1 < p.num) src = k + 1;
    }
    const T* row = reinterpret_cast<const T*>(p.layer[src]) + i * p.ld_h;
    if (p.out_hi)
      norm_row_split<T>(row, p.out_hi + i * p.ld_out, p.out_lo + i * p.ld_out, p.d, p.gain, p.eps);
    else
      norm_row<T>(row, p.out + i * p.ld_out, p.d, p.gain, p.eps, 1);
  }
}

template <typename T>
__global__ void __launch_bounds__(32 * kStageWarps)
    select_project_staged_kernel(const __grid_constant__ SelectParams p, const __grid_constant__ PairPlan plan) {
  extern __shared__ __align__(16) uint8_t stage_smem[];
  uint8_t* region = stage_smem + (size_t)(threadIdx.x >> 5) * stage_bytes(p.d, (int)sizeof(T));
  const int64_t warps = (int64_t)gridDim.x * kStageWarps;
  for (int64_t i = (int64_t)blockIdx.x * kStageWarps + (threadIdx.x >> 5); i < p.n; i += warps) {
    int64_t src = p.num - 1;
    if (p.exit_layers) {
      const int64_t k = p.exit_layers[i];
      if (k != TIDE_NO_EXIT && k + 1 >= 0 && k + 1 < p.num) src = k + 1;
    }
    const T* row = reinterpret_cast<const T*>(p.layer[src]) + i * p.ld_h;
    norm_row_planned<T>(row, p.out ? p.out + i * p.ld_out : nullptr,
                        p.out_hi ? p.out_hi + i * p.ld_out : nullptr,
                        p.out_hi ? p.out_lo + i * p.ld_out : nullptr, p.d, p.gain, p.eps, 1, region, plan);
  }
}

// The staged kernels take d >= 8 up to ~13,500 (4 rows in shared memory);
// TIDE_PROJECT_STAGED=0 keeps the one-pass global-read kernels.
static bool staged_plan(int d, int esz, PairPlan& P) {
  const char* env = getenv("TIDE_PROJECT_STAGED");  // read per call
  if (env && env[0] == '0') return false;
  if (d < 8 || kStageWarps * stage_bytes(d, esz) > 220 * 1024) return false;
  return plan_build(d, P) == 0;
}
// the dynamic-smem limit of a staged kernel is raised once, to the largest size used
template <typename K>
static void staged_smem_attr(K kernel, size_t smem) {
  if (smem <= 48 * 1024) return;
  static const void* ks[16];
  static size_t sz[16];
  static int nk = 0;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  int i = 0;
  while (i < nk && ks[i] != (const void*)kernel) ++i;
  if (i == nk && nk < 16) {
    ks[nk] = (const void*)kernel;
    sz[nk++] = 0;
  }
  if (i >= 16 || sz[i] < smem) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (i < 16) sz[i] = smem;
  }
}

static int grid_for(int64_t rows) {
  int dev = 0;
  cudaGetDevice(&dev);
  const int64_t blocks = (rows + (kPThreads / 32) - 1) / (kPThreads / 32);
  return (int)std::max<int64_t>(1, std::min<int64_t>(blocks, (int64_t)sm_count(dev) * 8));
}

}  // namespace tide

using namespace tide;

extern "C" int tide_exit_project(const void* rows, int64_t ld_rows, int32_t dtype,
                                 const int64_t* src_idx, int64_t n_e, const int64_t* n_e_dev,
                                 int32_t d, const float* gain, float eps, int32_t normalize,
                                 const int64_t* positions, float* out, int64_t ld_out,
                                 void* stream) {
  if (d < 1 || n_e < 0 || !out || !positions || (!rows && n_e > 0))
    return set_error(TIDE_ERR_ARG, "tide_exit_project: bad arguments");
  if (n_e == 0 && !n_e_dev) return TIDE_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  PairPlan plan;
  const int esz = dtype == TIDE_F32 ? 4 : 2;
  if (staged_plan(d, esz, plan)) {
    const size_t smem = kStageWarps * stage_bytes(d, esz);
    int dev = 0;
    cudaGetDevice(&dev);
    const int grid = (int)std::max<int64_t>(
        1, std::min<int64_t>((std::max<int64_t>(n_e, 1) + kStageWarps - 1) / kStageWarps,
                             (int64_t)sm_count(dev) * 8));
    switch (dtype) {
      case TIDE_F32:
        staged_smem_attr(exit_project_staged_kernel<float>, smem);
        exit_project_staged_kernel<float><<<grid, 32 * kStageWarps, smem, s>>>(
            (const float*)rows, ld_rows, src_idx, n_e, n_e_dev, d, gain, eps, normalize, positions, out,
            ld_out, plan);
        break;
      case TIDE_BF16:
        staged_smem_attr(exit_project_staged_kernel<__nv_bfloat16>, smem);
        exit_project_staged_kernel<__nv_bfloat16><<<grid, 32 * kStageWarps, smem, s>>>(
            (const __nv_bfloat16*)rows, ld_rows, src_idx, n_e, n_e_dev, d, gain, eps, normalize,
            positions, out, ld_out, plan);
        break;
      case TIDE_F16:
        staged_smem_attr(exit_project_staged_kernel<__half>, smem);
        exit_project_staged_kernel<__half><<<grid, 32 * kStageWarps, smem, s>>>(
            (const __half*)rows, ld_rows, src_idx, n_e, n_e_dev, d, gain, eps, normalize, positions,
            out, ld_out, plan);
        break;
      default:
        return set_error(TIDE_ERR_ARG, "bad dtype %d", dtype);
    }
    return check_launch("exit_project_staged_kernel");
  }
  const int grid = grid_for(std::max<int64_t>(n_e, 1));
  switch (dtype) {
    case TIDE_F32:
      exit_project_kernel<float><<<grid, kPThreads, 0, s>>>((const float*)rows, ld_rows, src_idx,
                                                            n_e, n_e_dev, d, gain, eps, normalize,
                                                            positions, out, ld_out);
      break;
    case TIDE_BF16:
      exit_project_kernel<__nv_bfloat16><<<grid, kPThreads, 0, s>>>(
          (const __nv_bfloat16*)rows, ld_rows, src_idx, n_e, n_e_dev, d, gain, eps, normalize,
          positions, out, ld_out);
      break;
    case TIDE_F16:
      exit_project_kernel<__half><<<grid, kPThreads, 0, s>>>((const __half*)rows, ld_rows, src_idx,
                                                             n_e, n_e_dev, d, gain, eps, normalize,
                                                             positions, out, ld_out);
      break;
    default:
      return set_error(TIDE_ERR_ARG, "bad dtype %d", dtype);
  }
  return check_launch("exit_project_kernel");
}

static int select_project_impl(const void* const* layer_ptrs, int32_t num_ptrs, int64_t ld_h,
                               int32_t dtype, const int64_t* exit_layers, int64_t n, int32_t d,
                               const float* gain, float eps, float* out, __nv_bfloat16* out_hi,
                               __nv_bfloat16* out_lo, int64_t ld_out, void* stream);

extern "C" int tide_select_project(const void* const* layer_ptrs, int32_t num_ptrs, int64_t ld_h,
                                   int32_t dtype, const int64_t* exit_layers, int64_t n,
                                   int32_t d, const float* gain, float eps, float* out,
                                   int64_t ld_out, void* stream) {
  if (!out) return set_error(TIDE_ERR_ARG, "tide_select_project: bad arguments");
  return select_project_impl(layer_ptrs, num_ptrs, ld_h, dtype, exit_layers, n, d, gain, eps, out,
                             nullptr, nullptr, ld_out, stream);
}

extern "C" int tide_select_project_split(const void* const* layer_ptrs, int32_t num_ptrs,
                                         int64_t ld_h, int32_t dtype, const int64_t* exit_layers,
                                         int64_t n, int32_t d, const float* gain, float eps,
                                         void* out_hi, void* out_lo, int64_t ld_out, void* stream) {
  if (!out_hi || !out_lo) return set_error(TIDE_ERR_ARG, "tide_select_project_split: null output");
  return select_project_impl(layer_ptrs, num_ptrs, ld_h, dtype, exit_layers, n, d, gain, eps,
                             nullptr, reinterpret_cast<__nv_bfloat16*>(out_hi),
                             reinterpret_cast<__nv_bfloat16*>(out_lo), ld_out, stream);
}

static int select_project_impl(const void* const* layer_ptrs, int32_t num_ptrs, int64_t ld_h,
                               int32_t dtype, const int64_t* exit_layers, int64_t n, int32_t d,
                               const float* gain, float eps, float* out, __nv_bfloat16* out_hi,
                               __nv_bfloat16* out_lo, int64_t ld_out, void* stream) {
  if (num_ptrs < 1 || num_ptrs > kMaxPtrs || d < 1 || n < 0 || ld_out < d || !layer_ptrs ||
      !layer_ptrs[num_ptrs - 1])
    return set_error(TIDE_ERR_ARG, "tide_select_project: bad arguments");
  if (n == 0) return TIDE_OK;
  SelectParams p{};
  for (int i = 0; i < num_ptrs; ++i) p.layer[i] = layer_ptrs[i];
  p.num = num_ptrs;
  p.ld_h = ld_h;
  p.n = n;
  p.ld_out = ld_out;
  p.d = d;
  p.exit_layers = exit_layers;
  p.gain = gain;
  p.eps = eps;
  p.out = out;
  p.out_hi = out_hi;
  p.out_lo = out_lo;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  PairPlan plan;
  const int esz = dtype == TIDE_F32 ? 4 : 2;
  if (staged_plan(d, esz, plan)) {
    const size_t smem = kStageWarps * stage_bytes(d, esz);
    int dev = 0;
    cudaGetDevice(&dev);
    const int grid = (int)std::max<int64_t>(
        1, std::min<int64_t>((n + kStageWarps - 1) / kStageWarps, (int64_t)sm_count(dev) * 8));
    switch (dtype) {
      case TIDE_F32:
        staged_smem_attr(select_project_staged_kernel<float>, smem);
        select_project_staged_kernel<float><<<grid, 32 * kStageWarps, smem, s>>>(p, plan);
        break;
      case TIDE_BF16:
        staged_smem_attr(select_project_staged_kernel<__nv_bfloat16>, smem);
        select_project_staged_kernel<__nv_bfloat16><<<grid, 32 * kStageWarps, smem, s>>>(p, plan);
        break;
      case TIDE_F16:
        staged_smem_attr(select_project_staged_kernel<__half>, smem);
        select_project_staged_kernel<__half><<<grid, 32 * kStageWarps, smem, s>>>(p, plan);
        break;
      default:
        return set_error(TIDE_ERR_ARG, "bad dtype %d", dtype);
    }
    return check_launch("select_project_staged_kernel");
  }
  const int grid = grid_for(n);
  switch (dtype) {
    case TIDE_F32: select_project_kernel<float><<<grid, kPThreads, 0, s>>>(p); break;
    case TIDE_BF16: select_project_kernel<__nv_bfloat16><<<grid, kPThreads, 0, s>>>(p); break;
    case TIDE_F16: select_project_kernel<__half><<<grid, kPThreads, 0, s>>>(p); break;
    default: return set_error(TIDE_ERR_ARG, "bad dtype %d", dtype);
  }
  return check_launch("select_project_kernel");
}
