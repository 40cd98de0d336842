/*
 * tide_b200.h — C ABI of the B200-native TIDE exit-decision hot path.
 *
 * Drop-in boundary for the reference's routing ops (earlyexit 0.1.0,
 * /root/reference/pkg/src/earlyexit, "ee/" below) and for the four CUDA ops
 * the paper registers as torch.ops.tide.* (PAPER.md:376-392, 413-419).
 *
 * Conventions
 *   - Every pointer argument is a DEVICE pointer unless stated otherwise; the
 *     caller allocates every output (the kernels never allocate global
 *     memory).  `stream` is a cudaStream_t passed as void*.
 *   - All calls are asynchronous and stream-ordered; none synchronises the
 *     host.  Return value: TIDE_OK (0) or a negative TIDE_ERR_* code;
 *     tide_last_error() returns the message of the calling thread's last
 *     failure.
 *   - dtype codes: TIDE_F32, TIDE_F16, TIDE_BF16.  Hidden rows are row-major
 *     with a leading dimension `ld` in ELEMENTS.
 *   - `workspace` is a TIDE_WORKSPACE_BYTES device buffer, zeroed once with
 *     tide_workspace_init() and then reused by calls on ONE stream (it holds
 *     the ordered look-back state of the stable compaction; its upper half
 *     is per-launch scratch, e.g. the f32 router's pre-split W).
 *   - There is no CPU fallback: unsupported shapes return
 *     TIDE_ERR_UNSUPPORTED.
 */
#ifndef TIDE_B200_H_
#define TIDE_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TIDE_F32 0
#define TIDE_F16 1
#define TIDE_BF16 2

#define TIDE_OK 0
#define TIDE_ERR_ARG (-1)
#define TIDE_ERR_UNSUPPORTED (-2)
#define TIDE_ERR_CUDA (-3)
#define TIDE_ERR_NODEVICE (-4)

#define TIDE_MODE_PER_TOKEN 0       /* ee/runtime.py:28 */
#define TIDE_MODE_BATCH_UNANIMOUS 1 /* ee/runtime.py:29 */
#define TIDE_NO_EXIT (-1)           /* ee/runtime.py:35 */

#define TIDE_WORKSPACE_BYTES (16u << 20)
#define TIDE_MAX_LAYERS 256
#define TIDE_MAX_DECODE_ROWS 16

const char* tide_version(void);
const char* tide_last_error(void);
int tide_sm_count(int device);
size_t tide_workspace_bytes(void);
int tide_workspace_init(void* workspace, void* stream);

/* 1 when (dtype, d, b) runs on a tcgen05 tensor-core kernel for large row
 * counts, else 0.  bf16 / f16: route_tc (all row counts).  f32: the 3xTF32
 * kernel for d <= 8192 from 16,384 rows (within the 1e-5 f32 contract); fewer
 * rows and other shapes take the CUDA-core kernel (f32 products). */
int tide_route_uses_tensor_cores(int32_t dtype, int32_t d, int32_t b);

/*
 * Fused RMSNorm + router + exit mask + stable compaction.
 *
 * Replaces, per checkpoint:
 *   ee/router_ops.py:68-87    fused_layernorm_route(h, router, eps) -> scores
 *   ee/runtime.py:149,171     mask = scores > np.float32(theta)
 *   ee/router_ops.py:137-154  batch_compact(...).{exiting,continuing}_indices
 *   ee/runtime.py:175-178     exited_at / exit_layers[exited_at] = k / remaining
 *
 * Rows routed: i in [0, n) — or [0, *n_dev) when n_dev != NULL (n is then the
 * capacity, the device count was produced by a previous call's counts[1]).
 * Row i reads h[row_idx[i]] when row_idx != NULL (peeling; rows_total bounds
 * row_idx values), else h[i].
 *   w_down  [b, d] row-major, dtype == h dtype (bf16/f16: tensor cores;
 *           f32: CUDA cores).     w_up [b] f32.
 * Outputs (each optional, NULL to skip), i = routed row:
 *   scores[i] f32, logits[i] f32 (pre-sigmoid), mask[i] u8,
 *   exit_idx[0..n_exit) / cont_idx[0..n-n_exit): stable partition, values are
 *   i (ids_from_rows = 0) or row_idx[i] (ids_from_rows = 1),
 *   exit_layers[row_idx ? row_idx[i] : i] = layer for exiting rows,
 *   counts[0] = n_exit, counts[1] = n - n_exit.
 */
int tide_route(const void* h, int64_t ld_h, int64_t n, const int64_t* n_dev, int64_t rows_total,
               int32_t d, int32_t dtype, const int64_t* row_idx, const void* w_down,
               const float* w_up, int32_t b, float eps, float theta, int64_t layer,
               float* scores, float* logits, uint8_t* mask, int64_t* exit_idx,
               int64_t* cont_idx, int32_t ids_from_rows, int64_t* exit_layers,
               int64_t* counts, void* workspace, void* stream);

/*
 * tide_route with launch flags.  tide_route(...) == tide_route_ex(..., 0, stream).
 *
 * TIDE_ROUTE_INPUTS_READY: the caller asserts that no kernel still in flight
 * on `stream` writes h, w_down or w_up (e.g. back-to-back routing of one
 * resident buffer).  The tensor-core kernel is launched with programmatic
 * dependent launch; by default it executes griddepcontrol.wait before its
 * first read of h / w_down / w_up, so rows written by the kernel just before
 * it on the stream (a layer's last kernel in a forward hook, a producer of
 * the capture) are visible.  With the flag its TMA stream starts while the
 * previous grid drains; only its writes and look-back wait.  Launches that
 * read a previous launch's row_idx / n_dev always wait first.
 */
#define TIDE_ROUTE_INPUTS_READY 1u
int tide_route_ex(const void* h, int64_t ld_h, int64_t n, const int64_t* n_dev,
                  int64_t rows_total, int32_t d, int32_t dtype, const int64_t* row_idx,
                  const void* w_down, const float* w_up, int32_t b, float eps, float theta,
                  int64_t layer, float* scores, float* logits, uint8_t* mask, int64_t* exit_idx,
                  int64_t* cont_idx, int32_t ids_from_rows, int64_t* exit_layers,
                  int64_t* counts, void* workspace, uint32_t flags, void* stream);

/*
 * Stable partition of a u8 mask (ee/router_ops.py:107-154, both strategies —
 * they agree bitwise by contract).  Index outputs as tide_route; when `rows`
 * != NULL also gathers rows (elem_bytes * d bytes each, leading dim ld_rows
 * elements) into exit_rows [n_exit, d] / cont_rows [n - n_exit, d]
 * (contiguous), which the caller sizes from a previous count.
 */
int tide_compact(const uint8_t* mask, int64_t n, const int64_t* n_dev, const int64_t* row_idx,
                 int32_t ids_from_rows, const void* rows, int64_t ld_rows, int32_t d,
                 int32_t elem_bytes, int64_t* exit_idx, int64_t* cont_idx, void* exit_rows,
                 void* cont_rows, int64_t* counts, void* workspace, void* stream);

/*
 * The LM head of posthoc_select (ee/model.py:329-338, ee/runtime.py:176-181:
 * logits = final_norm(rows) @ lm_head^T) on the tensor cores:
 *   out[n, V] (f32, leading dim ld_out) = A[n, d] . B[V, d]^T
 * with A, B as bf16 pairs (x = hi + lo, lo = bf16(x - bf16(x))): three MMA
 * terms hi.hi + hi.lo + lo.hi, f32 accumulation (small terms apart) — f32-grade
 * logits.  a_lo = b_lo = NULL: hi only (bf16 products).  ld_a, ld_b
 * multiples of 8 (any d <= ld), ld_out a multiple of 4, 16-byte aligned
 * pointers.  Columns [V, ceil4(V)) of every output row (inside ld_out) are
 * written with 0 (the epilogue stores whole 16-byte pieces); nothing past
 * ceil4(V) or row n is written.
 */
int tide_lm_head(const void* a_hi, const void* a_lo, int64_t ld_a, int64_t n, int32_t d,
                 const void* b_hi, const void* b_lo, int64_t ld_b, int64_t V, float* out,
                 int64_t ld_out, void* stream);

/*
 * select_project writing the LM head's A operand directly: every row final-
 * normed in f32 exactly as tide_select_project computes it, stored as the
 * bf16 pair hi = bf16(y), lo = bf16(y - hi) ([n, d] each, leading dim ld_out).
 */
int tide_select_project_split(const void* const* layer_ptrs, int32_t num_ptrs, int64_t ld_h,
                              int32_t dtype, const int64_t* exit_layers, int64_t n, int32_t d,
                              const float* gain, float eps, void* out_hi, void* out_lo,
                              int64_t ld_out, void* stream);

/*
 * u8 exit codes for the multi-GPU exit-map exchange (the
 * reference's exit map is ee/runtime.py:153-178's int64 exit_layers):
 * code[i] = exit_layers[i] + 1, so NO_EXIT (-1) -> 0 and checkpoint k -> k+1
 * (layers must lie in [-1, 254]).  tide_exit_decode is the inverse.  A
 * gathered code array is itself a valid tide_compact mask (nonzero = exited).
 */
int tide_exit_encode(const int64_t* exit_layers, int64_t n, uint8_t* code, void* stream);
int tide_exit_decode(const uint8_t* code, int64_t n, int64_t* exit_layers, void* stream);

/*
 * exit_scatter (ee/router_ops.py:170-176, normalize = 0) and exit_projection
 * (ee/router_ops.py:179-188, normalize = 1):
 *   out[positions[j]] = normalize ? rmsnorm(rows[src(j)], gain, eps) : rows[src(j)]
 * src(j) = src_idx ? src_idx[j] : j.  out is f32 [*, d] with leading dim ld_out.
 * gain may be NULL (no gain).  Positions are trusted (validated by caller).
 */
int tide_exit_project(const void* rows, int64_t ld_rows, int32_t dtype, const int64_t* src_idx,
                      int64_t n_e, const int64_t* n_e_dev, int32_t d, const float* gain,
                      float eps, int32_t normalize, const int64_t* positions, float* out,
                      int64_t ld_out, void* stream);

/*
 * The output staging of posthoc_select (ee/runtime.py:176,180, ee/model.py:329-338):
 *   out[i] = rmsnorm(H_{src(i)}[i], gain, eps), src(i) = exit_layers[i] + 1, or the
 *   final capture (layer_ptrs[num_ptrs-1]) when exit_layers[i] == TIDE_NO_EXIT
 *   (or exit_layers == NULL).  layer_ptrs is a HOST array of num_ptrs (= L+1)
 *   device pointers, NULL allowed for layers never referenced.
 */
int tide_select_project(const void* const* layer_ptrs, int32_t num_ptrs, int64_t ld_h,
                        int32_t dtype, const int64_t* exit_layers, int64_t n, int32_t d,
                        const float* gain, float eps, float* out, int64_t ld_out, void* stream);

/*
 * Calibration labeller (ee/tensor_math.py:96-113, ee/calibration.py:201-219):
 * one pass over the final rows and C checkpoint tensors (HOST array of C
 * device pointers, same dtype / ld as final_h).  Per checkpoint c, row i:
 *   sims[c*n+i] = clip(dot / (|h|*|f|), -1, 1), 0 for zero-norm rows;
 *   labels_u8 / labels_f32 [c*n+i] = sims > f32(tau);
 *   zero_mask[c*n+i] = 1 when either side has zero norm;
 *   zero_counts[c] = #rows with a zero-norm side (int64; zeroed by the call).
 * Any output may be NULL.
 */
int tide_cos_label(const void* const* ckpt_ptrs, int32_t C, const void* final_h, int64_t ld,
                   int32_t dtype, int64_t n, int32_t d, float tau, float* sims,
                   uint8_t* labels_u8, float* labels_f32, uint8_t* zero_mask,
                   int64_t* zero_counts, void* stream);

/*
 * Router training, one minibatch (ee/calibration.py:238-290; host side in
 * training.py, whose GEMMs are library calls).  Per row i of u [rows, b] f32
 * (= z_batch W_down^T):  su = sigma(u), a = u*su, t = a . w_up,
 *   gt[i] = (sigma(t) - labels[i]) / rows,  gu = gt * w_up * su*(1 + u*(1 - su)),
 *   *loss_sum += max(t,0) - t*y + log1p(exp(-|t|))   (f64 accumulator).
 * Outputs a_out / gu_out [rows, b], gt_out / t_out [rows], loss_sum: any may
 * be NULL.
 */
int tide_train_act(const float* u, int64_t rows, int32_t b, const float* w_up,
                   const float* labels, float* a_out, float* gu_out, float* gt_out,
                   float* t_out, double* loss_sum, void* stream);

/*
 * One Adam step over count f32 elements (ee/calibration.py:277-290), the
 * reference's rounding order: m = b1*m + (1-b1)*g; v = b2*v + (1-b2)*g*g;
 * w -= lr * (m / bias_corr1) / (sqrt(v / bias_corr2) + eps), with
 * bias_corr_k = f32(1 - beta_k^t) computed by the caller: the two scalars,
 * or (bias_corr_table != NULL, for a captured CUDA graph replayed every
 * epoch) the pair table[2 t], table[2 t + 1] at t = *step_base + step_offset
 * (device memory).
 */
int tide_adam_step(float* w, const float* g, float* m, float* v, int64_t count, float beta1,
                   float one_minus_beta1, float beta2, float one_minus_beta2,
                   const float* bias_corr_table, const int64_t* step_base, int64_t step_offset,
                   float bias_corr1, float bias_corr2, float lr, float eps, void* stream);

/*
 * Decode-step router (n <= TIDE_MAX_DECODE_ROWS rows, every checkpoint in ONE
 * launch) + exit resolution of posthoc_select (ee/runtime.py:151-178):
 * per-token = first checkpoint >= k_min whose score > theta; batch-unanimous
 * = first checkpoint where every row's score > theta.  Checkpoint c reads
 * h_ptrs[c] [n, d] (ld_h) with router (w_ptrs[c] [b,d] dtype, wup_ptrs[c] [b]
 * f32); HOST pointer arrays of length C, layers[c] ascending (host array).
 * Outputs: scores/logits [C, n] f32, exit_layers [n] int64 (TIDE_NO_EXIT),
 * exit_count[0] = rows that exited.
 */
int tide_route_decode(const void* const* h_ptrs, int32_t C, int64_t ld_h, int64_t n, int32_t d,
                      int32_t dtype, const void* const* w_ptrs, const float* const* wup_ptrs,
                      int32_t b, const int64_t* layers, float eps, float theta, int64_t k_min,
                      int32_t mode, float* scores, float* logits, int64_t* exit_layers,
                      int64_t* exit_count, void* workspace, void* stream);

/*
 * tide_route_decode with the routers' W_down in the packed shared-memory
 * image made by tide_decode_pack_weights (w_packed, 128-byte aligned; NULL =
 * tide_route_decode).  The kernel then fetches its W slices with plain 1-D
 * bulk copies.  Launched with programmatic dependent launch: the W / w_up
 * fetch overlaps the previous kernel on the stream (the caller's contract:
 * no kernel in flight writes the router weights); the hidden rows are read
 * only after it completed.
 */
int tide_route_decode_ex(const void* const* h_ptrs, int32_t C, int64_t ld_h, int64_t n, int32_t d,
                         int32_t dtype, const void* const* w_ptrs, const float* const* wup_ptrs,
                         int32_t b, const int64_t* layers, float eps, float theta, int64_t k_min,
                         int32_t mode, float* scores, float* logits, int64_t* exit_layers,
                         int64_t* exit_count, void* workspace, const void* w_packed, void* stream);

/* Bytes of the packed decode image of C routers ([C][ceil(d/64)][ceil(b/128)] x 16 KB). */
size_t tide_decode_packed_bytes(int32_t C, int32_t d, int32_t b);

/* Pack C routers' W_down (bf16 / f16 [b, d], HOST array of device pointers)
 * into the image tide_route_decode_ex reads (out: tide_decode_packed_bytes). */
int tide_decode_pack_weights(const void* const* w_ptrs, int32_t C, int32_t d, int32_t b,
                             int32_t dtype, void* out, void* stream);

/*
 * Tail of a per-token peeling chain (ee/runtime.py:166-178) in ONE routing
 * launch: after some links of the chain, the rows still live (row_idx[0 .. *n_dev),
 * device memory, as written by tide_route's cont_idx / counts[1]) are scored
 * against the C remaining checkpoints at once (checkpoint c: captures
 * h_ptrs[c], router w_ptrs[c] / wup_ptrs[c], layer layers[c]; HOST pointer
 * arrays, ascending layers) and each row gets the first checkpoint whose
 * score > theta in exit_layers[row id].  Only when *n_dev <= n_limit; else
 * nothing is routed.  *tail_count receives the live count the following
 * links must read (0 when the tail handled the rows, else *n_dev), so links
 * launched after it with n_dev = tail_count become no-ops (or are skipped
 * entirely inside a captured CUDA graph, see tide_capture_cond_*).  scores: device
 * scratch of C * cap f32 (cap = the chain's row capacity).  bf16 / f16
 * (split-K tensor-core kernel) or f32 (CUDA-core kernel, f32 products).
 * (No reference counterpart: an execution strategy of posthoc_select.)
 */
int tide_route_tail(const void* const* h_ptrs, int32_t C, int64_t ld_h, int64_t rows_total,
                    int32_t d, int32_t dtype, const int64_t* row_idx, const int64_t* n_dev,
                    int64_t cap, int64_t n_limit, const void* const* w_ptrs,
                    const float* const* wup_ptrs, int32_t b, const int64_t* layers, float eps,
                    float theta, float* scores, int64_t* exit_layers, int64_t* tail_count,
                    uint64_t cond_handle, void* workspace, void* stream);

/*
 * CUDA-graph capture helpers for the links after a chain tail: during stream
 * capture, tide_capture_cond_create makes a conditional handle (pass it as
 * tide_route_tail's cond_handle: the tail's resolve step sets it to 0 when it
 * handled the rows), tide_capture_cond_open adds an IF node on it after the
 * captured work and returns a side stream capturing into the node's body (launch
 * the remaining links there), tide_capture_cond_close ends that body.  Outside
 * capture, cond_create returns handle 0 and the links run as plain launches.
 */
/*
 * tide_route_tail with a lower bound: the tail handles the live rows only when
 * n_min <= *n_dev <= n_limit (else it leaves *tail_count = *n_dev for the
 * links).  n_limit >= cap makes it a WIDE tail: one cluster per live tile and
 * checkpoint, any live count — the speculative "score every remaining
 * checkpoint" step the chain takes right after its first link when few rows
 * exited there (n_min = the caller's break-even live count).
 * tide_route_tail(...) == tide_route_tail_ex(..., n_min = 0, ...).
 */
int tide_route_tail_ex(const void* const* h_ptrs, int32_t C, int64_t ld_h, int64_t rows_total,
                       int32_t d, int32_t dtype, const int64_t* row_idx, const int64_t* n_dev,
                       int64_t cap, int64_t n_min, int64_t n_limit, const void* const* w_ptrs,
                       const float* const* wup_ptrs, int32_t b, const int64_t* layers, float eps,
                       float theta, float* scores, int64_t* exit_layers, int64_t* tail_count,
                       uint64_t cond_handle, void* workspace, void* stream);

/*
 * Per-token exit decision over C checkpoints (ee/runtime.py:166-178, the
 * per-token rule of posthoc_select) in ONE persistent tensor-core launch:
 * every row is scored at every checkpoint (speculative: no peeling between
 * checkpoints) and exit_layers[row id] = layers[first c whose score >
 * theta], combined across CTAs by an atomic minimum; the routed rows'
 * entries must hold TIDE_NO_EXIT on entry, rows that never fire keep it.
 * Dense (row_idx = n_dev = NULL: rows 0..n-1 of every capture, row id = row)
 * or gathered (the live rows row_idx[0 .. *n_dev), n = the list's
 * capacity).  h_ptrs / w_ptrs / wup_ptrs / layers: HOST arrays of C entries
 * (ascending layers, C <= 24).  scores: NULL or device memory of C * n f32
 * (score of position i at checkpoint c -> scores[c * n + i]).  bf16 / f16
 * rows only.  Same exit map as the peeling chain (a row's score at a
 * checkpoint depends only on that row).
 * (No reference counterpart: an execution strategy of posthoc_select.)
 */
int tide_route_multi(const void* const* h_ptrs, int32_t C, int64_t ld_h, int64_t n,
                     const int64_t* n_dev, int64_t rows_total, int32_t d, int32_t dtype,
                     const int64_t* row_idx, const void* const* w_ptrs,
                     const float* const* wup_ptrs, int32_t b, const int64_t* layers, float eps,
                     float theta, float* scores, int64_t* exit_layers, void* workspace,
                     void* stream);

int tide_capture_cond_create(void* stream, uint64_t* handle);
int tide_capture_cond_open(void* stream, uint64_t handle, void** body_stream);
int tide_capture_cond_close(void* body_stream);

#ifdef __cplusplus
}
#endif

#endif /* TIDE_B200_H_ */
