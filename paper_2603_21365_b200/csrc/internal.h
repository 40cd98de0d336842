// Host-side internals shared by the launchers and the C ABI (capi.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/tide_b200.h"

namespace tide {

struct RouteArgs {
  const void* h;
  int64_t ld_h;
  int64_t n;
  const int64_t* n_dev;
  int64_t rows_total;
  int32_t d;
  int32_t dtype;
  const int64_t* row_idx;
  const void* w_down;
  const float* w_up;
  int32_t b;
  float eps;
  float theta;
  int64_t layer;
  float* scores;
  float* logits;
  uint8_t* mask;
  int64_t* exit_idx;
  int64_t* cont_idx;
  int32_t ids_from_rows;
  int64_t* exit_layers;
  int64_t* counts;
  void* workspace;
  uint32_t flags;  // TIDE_ROUTE_* (tide_route_ex)
  int64_t n_min;   // chain tail: handle the live rows only when n_min <= n <= n_limit
};

int set_error(int code, const char* fmt, ...);
int check_launch(const char* what);
int sm_count(int device);

bool route_tc_supported(int dtype, int d, int b);
int make_map(CUtensorMap* m, const void* base, int dtype, int64_t cols, int64_t rows,
             int64_t ld_elems, int box_cols, int box_rows);
extern unsigned long long* g_dbg;
int route_tc_launch(const RouteArgs& a, cudaStream_t stream);
int route_tcs_plan(const RouteArgs& a, int dev, int* grid);
int route_tcs_launch(const RouteArgs& a, cudaStream_t stream, int ks, int grid);
int route_tcs_tail_launch(const RouteArgs& a, int C, const void* const* h_ptrs,
                          const void* const* w_ptrs, const float* const* wup_ptrs,
                          const int64_t* layers, int64_t n_limit, int64_t* tail_count,
                          unsigned long long cond, cudaStream_t stream);
int route_tc_multi_launch(const RouteArgs& a, int C, const void* const* h_ptrs,
                          const void* const* w_ptrs, const float* const* wup_ptrs,
                          const int64_t* layers, int64_t n_limit, cudaStream_t stream);
int route_simt_launch(const RouteArgs& a, cudaStream_t stream);
int route_simt_tail_launch(const RouteArgs& a, int C, const void* const* h_ptrs,
                           const void* const* w_ptrs, const float* const* wup_ptrs,
                           const int64_t* layers, int64_t n_limit, int64_t* tail_count,
                           unsigned long long cond, cudaStream_t stream);
int chain_resolve_launch(const float* scores, int64_t cap, int C, const int64_t* layers,
                         float theta, const int64_t* n_dev, int64_t n_min, int64_t n_limit,
                         const int64_t* row_idx, int64_t* exit_layers, int64_t* tail_count,
                         unsigned long long cond, cudaStream_t stream);
bool route_tf32_supported(int d, int b, int64_t n);
int route_tf32_launch(const RouteArgs& a, cudaStream_t stream);
int compact_launch(const uint8_t* mask, int64_t n, const int64_t* n_dev, const int64_t* row_idx,
                   int32_t ids_from_rows, const void* rows, int64_t ld_rows, int32_t d,
                   int32_t elem_bytes, int64_t* exit_idx, int64_t* cont_idx, void* exit_rows,
                   void* cont_rows, int64_t* counts, void* workspace, cudaStream_t stream);
int lmhead_launch(const void* a_hi, const void* a_lo, int64_t ld_a, int64_t n, int32_t d,
                  const void* b_hi, const void* b_lo, int64_t ld_b, int64_t V, float* out,
                  int64_t ld_out, cudaStream_t stream);
int exit_code_launch(const int64_t* layers, int64_t n, uint8_t* code, int decode,
                     cudaStream_t stream);

}  // namespace tide
