// C ABI entry points (include/tide_b200.h): argument checks, path selection
// (tcgen05 vs CUDA-core), thread-local error reporting, device queries.
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "internal.h"

namespace tide {

static thread_local char g_err[512] = "";

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int check_launch(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(TIDE_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return TIDE_OK;
}

int sm_count(int device) {
  static int cache[64] = {0};
  if (device < 0 || device >= 64) return 148;
  if (!cache[device]) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || v <= 0)
      v = 148;
    cache[device] = v;
  }
  return cache[device];
}

}  // namespace tide

using namespace tide;

extern "C" {

const char* tide_version(void) { return "tide_b200 0.1.0 (sm_100a)"; }

const char* tide_last_error(void) { return g_err; }

int tide_sm_count(int device) { return sm_count(device); }

size_t tide_workspace_bytes(void) { return TIDE_WORKSPACE_BYTES; }

int tide_workspace_init(void* workspace, void* stream) {
  if (!workspace) return set_error(TIDE_ERR_ARG, "null workspace");
  if (cudaMemsetAsync(workspace, 0, TIDE_WORKSPACE_BYTES, reinterpret_cast<cudaStream_t>(stream)) !=
      cudaSuccess)
    return set_error(TIDE_ERR_CUDA, "workspace memset failed");
  return TIDE_OK;
}

int tide_route_uses_tensor_cores(int32_t dtype, int32_t d, int32_t b) {
  if (dtype == TIDE_F32) return route_tf32_supported(d, b, 1 << 30) ? 1 : 0;
  return route_tc_supported(dtype, d, b) ? 1 : 0;
}

int tide_route(const void* h, int64_t ld_h, int64_t n, const int64_t* n_dev, int64_t rows_total,
               int32_t d, int32_t dtype, const int64_t* row_idx, const void* w_down,
               const float* w_up, int32_t b, float eps, float theta, int64_t layer,
               float* scores, float* logits, uint8_t* mask, int64_t* exit_idx,
               int64_t* cont_idx, int32_t ids_from_rows, int64_t* exit_layers,
               int64_t* counts, void* workspace, void* stream) {
  return tide_route_ex(h, ld_h, n, n_dev, rows_total, d, dtype, row_idx, w_down, w_up, b, eps,
                       theta, layer, scores, logits, mask, exit_idx, cont_idx, ids_from_rows,
                       exit_layers, counts, workspace, 0u, stream);
}

int tide_route_ex(const void* h, int64_t ld_h, int64_t n, const int64_t* n_dev,
                  int64_t rows_total, int32_t d, int32_t dtype, const int64_t* row_idx,
                  const void* w_down, const float* w_up, int32_t b, float eps, float theta,
                  int64_t layer, float* scores, float* logits, uint8_t* mask, int64_t* exit_idx,
                  int64_t* cont_idx, int32_t ids_from_rows, int64_t* exit_layers,
                  int64_t* counts, void* workspace, uint32_t flags, void* stream) {
  if (d < 1 || b < 1 || n < 0) return set_error(TIDE_ERR_ARG, "tide_route: bad shape");
  if (!w_down || !w_up || !workspace)
    return set_error(TIDE_ERR_ARG, "tide_route: null weights or workspace");
  if (n > 0 && !h) return set_error(TIDE_ERR_ARG, "tide_route: null hidden rows");
  if (ld_h < d) return set_error(TIDE_ERR_ARG, "tide_route: ld_h < d");
  if (dtype != TIDE_F32 && dtype != TIDE_F16 && dtype != TIDE_BF16)
    return set_error(TIDE_ERR_ARG, "tide_route: bad dtype %d", dtype);
  if (row_idx && rows_total < 1) return set_error(TIDE_ERR_ARG, "tide_route: rows_total required");
  if (flags & ~(uint32_t)TIDE_ROUTE_INPUTS_READY)
    return set_error(TIDE_ERR_ARG, "tide_route: unknown flags 0x%x", flags);
  if (n == 0 && !n_dev) {
    if (counts)
      if (cudaMemsetAsync(counts, 0, 2 * sizeof(int64_t), reinterpret_cast<cudaStream_t>(stream)) !=
          cudaSuccess)
        return set_error(TIDE_ERR_CUDA, "memset counts failed");
    return TIDE_OK;
  }
  RouteArgs a{};
  a.h = h;
  a.ld_h = ld_h;
  a.n = n;
  a.n_dev = n_dev;
  a.rows_total = row_idx ? rows_total : n;
  a.d = d;
  a.dtype = dtype;
  a.row_idx = row_idx;
  a.w_down = w_down;
  a.w_up = w_up;
  a.b = b;
  a.eps = eps;
  a.theta = theta;
  a.layer = layer;
  a.scores = scores;
  a.logits = logits;
  a.mask = mask;
  a.exit_idx = exit_idx;
  a.cont_idx = cont_idx;
  a.ids_from_rows = ids_from_rows;
  a.exit_layers = exit_layers;
  a.counts = counts;
  a.workspace = workspace;
  a.flags = flags;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const bool aligned = ((reinterpret_cast<uintptr_t>(h) & 15) == 0) &&
                       ((reinterpret_cast<uintptr_t>(w_down) & 15) == 0) && (ld_h % 8 == 0);
  if (route_tc_supported(dtype, d, b) && aligned) return route_tc_launch(a, s);
  // f32 rows: the 3xTF32 tensor-core kernel (route_tf32.cu) where its error
  // bound holds and the rows are 16-byte aligned for TMA, else CUDA cores
  if (dtype == TIDE_F32 && route_tf32_supported(d, b, n) && ld_h % 4 == 0 &&
      ((reinterpret_cast<uintptr_t>(h) | reinterpret_cast<uintptr_t>(w_down)) & 15) == 0)
    return route_tf32_launch(a, s);
  return route_simt_launch(a, s);
}

int tide_route_tail(const void* const* h_ptrs, int32_t C, int64_t ld_h, int64_t rows_total,
                    int32_t d, int32_t dtype, const int64_t* row_idx, const int64_t* n_dev,
                    int64_t cap, int64_t n_limit, const void* const* w_ptrs,
                    const float* const* wup_ptrs, int32_t b, const int64_t* layers, float eps,
                    float theta, float* scores, int64_t* exit_layers, int64_t* tail_count,
                    uint64_t cond_handle, void* workspace, void* stream) {
  return tide_route_tail_ex(h_ptrs, C, ld_h, rows_total, d, dtype, row_idx, n_dev, cap, 0, n_limit,
                            w_ptrs, wup_ptrs, b, layers, eps, theta, scores, exit_layers,
                            tail_count, cond_handle, workspace, stream);
}

int tide_route_tail_ex(const void* const* h_ptrs, int32_t C, int64_t ld_h, int64_t rows_total,
                       int32_t d, int32_t dtype, const int64_t* row_idx, const int64_t* n_dev,
                       int64_t cap, int64_t n_min, int64_t n_limit, const void* const* w_ptrs,
                       const float* const* wup_ptrs, int32_t b, const int64_t* layers, float eps,
                       float theta, float* scores, int64_t* exit_layers, int64_t* tail_count,
                       uint64_t cond_handle, void* workspace, void* stream) {
  if (n_min < 0) return set_error(TIDE_ERR_ARG, "tide_route_tail: n_min < 0");
  if (C < 1 || !h_ptrs || !w_ptrs || !wup_ptrs || !layers)
    return set_error(TIDE_ERR_ARG, "tide_route_tail: bad checkpoint arrays");
  if (d < 1 || b < 1 || cap < 1 || ld_h < d || rows_total < 1 || n_limit < 0)
    return set_error(TIDE_ERR_ARG, "tide_route_tail: bad shape");
  if (!row_idx || !n_dev || !scores || !exit_layers || !tail_count || !workspace)
    return set_error(TIDE_ERR_ARG, "tide_route_tail: null device buffer");
  if (dtype != TIDE_F32 && dtype != TIDE_F16 && dtype != TIDE_BF16)
    return set_error(TIDE_ERR_ARG, "tide_route_tail: bad dtype %d", dtype);
  if (dtype != TIDE_F32 && !route_tc_supported(dtype, d, b))
    return set_error(TIDE_ERR_UNSUPPORTED, "tide_route_tail: shape");
  for (int c = 0; c < C; ++c)
    if (((reinterpret_cast<uintptr_t>(h_ptrs[c]) | reinterpret_cast<uintptr_t>(w_ptrs[c])) & 15) ||
        (c && layers[c] <= layers[c - 1]))
      return set_error(TIDE_ERR_ARG, "tide_route_tail: unaligned pointer or unordered layers");
  RouteArgs a{};
  a.h = h_ptrs[0];
  a.ld_h = ld_h;
  a.n = cap;
  a.n_dev = n_dev;
  a.rows_total = rows_total;
  a.d = d;
  a.dtype = dtype;
  a.row_idx = row_idx;
  a.w_down = w_ptrs[0];
  a.w_up = wup_ptrs[0];
  a.b = b;
  a.eps = eps;
  a.theta = theta;
  a.scores = scores;
  a.exit_layers = exit_layers;
  a.workspace = workspace;
  a.n_min = n_min;
  if (dtype == TIDE_F32)  // CUDA-core kernel, f32 products (the 1e-5 contract)
    return route_simt_tail_launch(a, C, h_ptrs, w_ptrs, wup_ptrs, layers, n_limit, tail_count,
                                  (unsigned long long)cond_handle,
                                  reinterpret_cast<cudaStream_t>(stream));
  return route_tcs_tail_launch(a, C, h_ptrs, w_ptrs, wup_ptrs, layers, n_limit, tail_count,
                               (unsigned long long)cond_handle, reinterpret_cast<cudaStream_t>(stream));
}

int tide_route_multi(const void* const* h_ptrs, int32_t C, int64_t ld_h, int64_t n,
                     const int64_t* n_dev, int64_t rows_total, int32_t d, int32_t dtype,
                     const int64_t* row_idx, const void* const* w_ptrs,
                     const float* const* wup_ptrs, int32_t b, const int64_t* layers, float eps,
                     float theta, float* scores, int64_t* exit_layers, void* workspace,
                     void* stream) {
  if (C < 1 || !h_ptrs || !w_ptrs || !wup_ptrs || !layers)
    return set_error(TIDE_ERR_ARG, "tide_route_multi: bad checkpoint arrays");
  if (d < 1 || b < 1 || n < 0 || ld_h < d || (row_idx && rows_total < 1))
    return set_error(TIDE_ERR_ARG, "tide_route_multi: bad shape");
  if ((row_idx == nullptr) != (n_dev == nullptr))
    return set_error(TIDE_ERR_ARG, "tide_route_multi: row_idx and n_dev go together");
  if (!exit_layers || !workspace)
    return set_error(TIDE_ERR_ARG, "tide_route_multi: null device buffer");
  if ((dtype != TIDE_F16 && dtype != TIDE_BF16) || !route_tc_supported(dtype, d, b) || ld_h % 8)
    return set_error(TIDE_ERR_UNSUPPORTED, "tide_route_multi: bf16/f16 rows, d %% 8 == 0, b <= 256");
  for (int c = 0; c < C; ++c)
    if (((reinterpret_cast<uintptr_t>(h_ptrs[c]) | reinterpret_cast<uintptr_t>(w_ptrs[c])) & 15) ||
        (c && layers[c] <= layers[c - 1]))
      return set_error(TIDE_ERR_ARG, "tide_route_multi: unaligned pointer or unordered layers");
  if (n == 0) return TIDE_OK;
  RouteArgs a{};
  a.h = h_ptrs[0];
  a.ld_h = ld_h;
  a.n = n;
  a.n_dev = n_dev;
  a.rows_total = row_idx ? rows_total : n;
  a.d = d;
  a.dtype = dtype;
  a.row_idx = row_idx;
  a.w_down = w_ptrs[0];
  a.w_up = wup_ptrs[0];
  a.b = b;
  a.eps = eps;
  a.theta = theta;
  a.scores = scores;
  a.exit_layers = exit_layers;
  a.workspace = workspace;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (C == 1) {  // one checkpoint: the plain route (strict mask -> exit layer)
    a.layer = layers[0];
    return route_tc_launch(a, s);
  }
  return route_tc_multi_launch(a, C, h_ptrs, w_ptrs, wup_ptrs, layers, n, s);
}

// --- CUDA-graph conditional for the links after a chain tail -----------------
int tide_capture_cond_create(void* stream, uint64_t* handle) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  cudaGraph_t g = nullptr;
  if (cudaStreamGetCaptureInfo(s, &st, nullptr, &g, nullptr, nullptr) != cudaSuccess)
    return set_error(TIDE_ERR_CUDA, "capture info failed");
  if (st != cudaStreamCaptureStatusActive) {
    *handle = 0;
    return TIDE_OK;  // not capturing: nothing to do
  }
  cudaGraphConditionalHandle h;
  if (cudaGraphConditionalHandleCreate(&h, g, 1u, cudaGraphCondAssignDefault) != cudaSuccess)
    return set_error(TIDE_ERR_CUDA, "conditional handle");
  *handle = (uint64_t)h;
  return TIDE_OK;
}

int tide_capture_cond_open(void* stream, uint64_t handle, void** body_stream) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  cudaGraph_t g = nullptr;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  if (cudaStreamGetCaptureInfo(s, &st, nullptr, &g, &deps, &nd) != cudaSuccess ||
      st != cudaStreamCaptureStatusActive)
    return set_error(TIDE_ERR_CUDA, "tide_capture_cond_open: stream not capturing");
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = (cudaGraphConditionalHandle)handle;
  cp.conditional.type = cudaGraphCondTypeIf;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  if (cudaGraphAddNode(&node, g, deps, nd, &cp) != cudaSuccess)
    return set_error(TIDE_ERR_CUDA, "conditional node");
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  if (cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies) != cudaSuccess)
    return set_error(TIDE_ERR_CUDA, "capture dependencies");
  cudaStream_t side;
  if (cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking) != cudaSuccess)
    return set_error(TIDE_ERR_CUDA, "side stream");
  if (cudaStreamBeginCaptureToGraph(side, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed) !=
      cudaSuccess)
    return set_error(TIDE_ERR_CUDA, "capture to the conditional body");
  *body_stream = side;
  return TIDE_OK;
}

int tide_capture_cond_close(void* body_stream) {
  cudaStream_t side = reinterpret_cast<cudaStream_t>(body_stream);
  cudaGraph_t out = nullptr;
  const cudaError_t e = cudaStreamEndCapture(side, &out);
  cudaStreamDestroy(side);
  if (e != cudaSuccess) return set_error(TIDE_ERR_CUDA, "end of the conditional body capture");
  return TIDE_OK;
}

int tide_compact(const uint8_t* mask, int64_t n, const int64_t* n_dev, const int64_t* row_idx,
                 int32_t ids_from_rows, const void* rows, int64_t ld_rows, int32_t d,
                 int32_t elem_bytes, int64_t* exit_idx, int64_t* cont_idx, void* exit_rows,
                 void* cont_rows, int64_t* counts, void* workspace, void* stream) {
  if (n < 0 || (!mask && n > 0) || !workspace)
    return set_error(TIDE_ERR_ARG, "tide_compact: bad arguments");
  if (rows && (d < 1 || elem_bytes < 1 || ld_rows < d))
    return set_error(TIDE_ERR_ARG, "tide_compact: bad row geometry");
  return compact_launch(mask, n, n_dev, row_idx, ids_from_rows, rows, ld_rows, d, elem_bytes,
                        exit_idx, cont_idx, exit_rows, cont_rows, counts, workspace,
                        reinterpret_cast<cudaStream_t>(stream));
}

int tide_lm_head(const void* a_hi, const void* a_lo, int64_t ld_a, int64_t n, int32_t d,
                 const void* b_hi, const void* b_lo, int64_t ld_b, int64_t V, float* out,
                 int64_t ld_out, void* stream) {
  if (n < 0 || V < 0 || d < 1 || !a_hi || !b_hi || (n > 0 && V > 0 && !out))
    return set_error(TIDE_ERR_ARG, "tide_lm_head: bad arguments");
  if ((a_lo == nullptr) != (b_lo == nullptr))
    return set_error(TIDE_ERR_ARG, "tide_lm_head: give both lo operands or neither");
  if (ld_a % 8 || ld_b % 8 || ld_a < d || ld_b < d || ld_out % 4 || ld_out < V)
    return set_error(TIDE_ERR_UNSUPPORTED,
                     "tide_lm_head: ld_a, ld_b multiples of 8 (>= d); ld_out a multiple of 4 (>= V)");
  const uintptr_t al = reinterpret_cast<uintptr_t>(a_hi) | reinterpret_cast<uintptr_t>(a_lo) |
                       reinterpret_cast<uintptr_t>(b_hi) | reinterpret_cast<uintptr_t>(b_lo) |
                       reinterpret_cast<uintptr_t>(out);
  if (al & 15) return set_error(TIDE_ERR_ARG, "tide_lm_head: pointers must be 16-byte aligned");
  if (n == 0 || V == 0) return TIDE_OK;
  return lmhead_launch(a_hi, a_lo, ld_a, n, d, b_hi, b_lo, ld_b, V, out, ld_out,
                       reinterpret_cast<cudaStream_t>(stream));
}

int tide_exit_encode(const int64_t* exit_layers, int64_t n, uint8_t* code, void* stream) {
  if (n < 0 || (n > 0 && (!exit_layers || !code)))
    return set_error(TIDE_ERR_ARG, "tide_exit_encode: bad arguments");
  return exit_code_launch(exit_layers, n, code, 0, reinterpret_cast<cudaStream_t>(stream));
}

int tide_exit_decode(const uint8_t* code, int64_t n, int64_t* exit_layers, void* stream) {
  if (n < 0 || (n > 0 && (!exit_layers || !code)))
    return set_error(TIDE_ERR_ARG, "tide_exit_decode: bad arguments");
  return exit_code_launch(exit_layers, n, const_cast<uint8_t*>(code), 1,
                          reinterpret_cast<cudaStream_t>(stream));
}

}  // extern "C"
