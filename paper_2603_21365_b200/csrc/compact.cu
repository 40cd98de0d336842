// K2 standalone: stable partition of an exit mask (batch_compact,
// ee/router_ops.py:107-154) with optional row gather.
//
// 2048 mask entries per partition (256 threads x 8 bytes, one 8-byte load
// each), block scan of exit counts, ordered decoupled look-back across
// partitions (bit-exact stable order), then int64 index writes and, when
// rows are given, a warp-per-row gather into the exiting / continuing blocks.
#include <cuda_runtime.h>

#include <algorithm>

#include "common.cuh"
#include "internal.h"

namespace tide {

constexpr int kCThreads = 256;
constexpr int kCPer = 8;
constexpr int kCTile = kCThreads * kCPer;

struct CompactParams {
  const uint8_t* mask;
  int64_t n_host;
  const int64_t* n_dev;
  const int64_t* row_idx;
  int32_t ids_from_rows;
  const uint8_t* rows;
  int64_t row_pitch;   // bytes
  int64_t row_bytes;   // d * elem_bytes
  int64_t* exit_idx;
  int64_t* cont_idx;
  uint8_t* exit_rows;
  uint8_t* cont_rows;
  int64_t* counts;
  Workspace* ws;
};

__global__ void __launch_bounds__(kCThreads) compact_kernel(const CompactParams p) {
  __shared__ uint32_t warp_tot[kCThreads / 32];
  __shared__ uint32_t E_s;
  __shared__ int32_t dst_s[kCTile];  // destination row in its half (exit: rank, cont: i-rank) tile-local offset
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t n = p.n_dev ? *p.n_dev : p.n_host;
  const int64_t ntiles = (n + kCTile - 1) / kCTile;
  const uint32_t tag = launch_tag(p.ws);
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t base = tile * kCTile + (int64_t)tid * kCPer;
    uint8_t m[kCPer];
    if (base + kCPer <= n && ((reinterpret_cast<uintptr_t>(p.mask + base) & 7) == 0)) {
      const uint2 v = *reinterpret_cast<const uint2*>(p.mask + base);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        m[e] = (v.x >> (8 * e)) & 0xFF;
        m[4 + e] = (v.y >> (8 * e)) & 0xFF;
      }
    } else {
#pragma unroll
      for (int e = 0; e < kCPer; ++e) m[e] = (base + e < n) ? p.mask[base + e] : 0;
    }
    uint32_t cnt = 0;
#pragma unroll
    for (int e = 0; e < kCPer; ++e) cnt += m[e] ? 1u : 0u;
    uint32_t incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    uint32_t wpre = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < kCThreads / 32; ++w) {
      const uint32_t t = warp_tot[w];
      if (w < warp) wpre += t;
      tot += t;
    }
    if (warp == 0) {
      const uint32_t E = lookback_exclusive(p.ws->status, tag, tile, tot);
      if (lane == 0) {
        E_s = E;
        if (tile == ntiles - 1 && p.counts) {
          p.counts[0] = (int64_t)E + tot;
          p.counts[1] = n - ((int64_t)E + tot);
        }
      }
    }
    __syncthreads();
    const int64_t E = E_s;
    uint32_t run = wpre + incl - cnt;  // exclusive within the tile
#pragma unroll
    for (int e = 0; e < kCPer; ++e) {
      const int64_t i = base + e;
      if (i < n) {
        const int64_t rank = E + run;
        const int64_t id = (p.ids_from_rows && p.row_idx) ? p.row_idx[i] : i;
        if (m[e]) {
          if (p.exit_idx) p.exit_idx[rank] = id;
          dst_s[tid * kCPer + e] = (int32_t)(rank - E);
        } else {
          if (p.cont_idx) p.cont_idx[i - rank] = id;
          dst_s[tid * kCPer + e] = (int32_t)((i - rank) - (tile * kCTile - E)) | (int32_t)0x80000000;
        }
        run += m[e] ? 1u : 0u;
      }
    }
    if (p.rows) {
      __syncthreads();
      const int64_t t0 = tile * kCTile;
      const int64_t cont_base = t0 - E;  // first continuing rank of this tile
      const int lim = (int)std::min<int64_t>(kCTile, n - t0);
      const bool vec = (p.row_bytes % 16 == 0) && (p.row_pitch % 16 == 0) &&
                       ((reinterpret_cast<uintptr_t>(p.rows) & 15) == 0);
      for (int r = warp; r < lim; r += kCThreads / 32) {
        const int32_t code = dst_s[r];
        const int64_t i = t0 + r;
        const int64_t src_row = p.row_idx ? p.row_idx[i] : i;
        const uint8_t* src = p.rows + src_row * p.row_pitch;
        uint8_t* dst;
        if (code & 0x80000000) {
          if (!p.cont_rows) continue;
          dst = p.cont_rows + (cont_base + (code & 0x7FFFFFFF)) * p.row_bytes;
        } else {
          if (!p.exit_rows) continue;
          dst = p.exit_rows + (E + code) * p.row_bytes;
        }
        if (vec && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
          for (int64_t o = (int64_t)lane * 16; o < p.row_bytes; o += 32 * 16)
            *reinterpret_cast<uint4*>(dst + o) = *reinterpret_cast<const uint4*>(src + o);
        } else {
          for (int64_t o = lane; o < p.row_bytes; o += 32) dst[o] = src[o];
        }
      }
    }
    __syncthreads();
  }
  if (ntiles == 0 && blockIdx.x == 0 && tid == 0 && p.counts) {
    p.counts[0] = 0;
    p.counts[1] = 0;
  }
  __syncthreads();
  if (tid == 0) launch_done(p.ws);
}

// Row gather from the index lists the scan wrote (dense rows): output row j
// is rows[exit_idx[j]] for j < counts[0], else rows[cont_idx[j - counts[0]]]
// into the continuing block.  A warp per output row with 8 16-byte loads in
// flight per lane, every SM busy (the scan's own warp-per-row gather runs on
// one CTA per 2,048-row partition: 32 CTAs at 65,536 rows, 0.5 TB/s).
__global__ void __launch_bounds__(256) gather_rows_kernel(
    const int64_t* __restrict__ exit_idx, const int64_t* __restrict__ cont_idx,
    const int64_t* __restrict__ counts, const uint8_t* __restrict__ rows, int64_t pitch,
    int64_t row_bytes, uint8_t* __restrict__ exit_rows, uint8_t* __restrict__ cont_rows) {
  griddep_wait();  // the scan kernel just before wrote the indices and counts
  const int64_t ne = counts[0], nt = counts[0] + counts[1];
  const int lane = threadIdx.x & 31;
  const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const bool vec = (row_bytes % 16 == 0) && (pitch % 16 == 0) &&
                   ((reinterpret_cast<uintptr_t>(rows) | reinterpret_cast<uintptr_t>(exit_rows) |
                     reinterpret_cast<uintptr_t>(cont_rows)) & 15) == 0;
  for (int64_t j = wid; j < nt; j += nw) {
    const bool ex = j < ne;
    if (ex ? exit_rows == nullptr : cont_rows == nullptr) continue;
    const int64_t src_row = ex ? exit_idx[j] : cont_idx[j - ne];
    const uint8_t* src = rows + src_row * pitch;
    uint8_t* dst = ex ? exit_rows + j * row_bytes : cont_rows + (j - ne) * row_bytes;
    if (vec) {
      for (int64_t o0 = (int64_t)lane * 16; o0 < row_bytes; o0 += 32 * 16 * 8) {
        uint4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (o0 + u * 512 < row_bytes) v[u] = ld_nc_v4(src + o0 + u * 512);
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (o0 + u * 512 < row_bytes) __stcs(reinterpret_cast<uint4*>(dst + o0 + u * 512), v[u]);
      }
    } else {
      for (int64_t o = lane; o < row_bytes; o += 32) dst[o] = src[o];
    }
  }
}

int compact_launch(const uint8_t* mask, int64_t n, const int64_t* n_dev, const int64_t* row_idx,
                   int32_t ids_from_rows, const void* rows, int64_t ld_rows, int32_t d,
                   int32_t elem_bytes, int64_t* exit_idx, int64_t* cont_idx, void* exit_rows,
                   void* cont_rows, int64_t* counts, void* workspace, cudaStream_t stream) {
  const int64_t ntiles = (n + kCTile - 1) / kCTile;
  if (ntiles > kMaxParts / 2) return set_error(TIDE_ERR_UNSUPPORTED, "mask too long for one launch");
  CompactParams p{};
  p.mask = mask;
  p.n_host = n;
  p.n_dev = n_dev;
  p.row_idx = row_idx;
  p.ids_from_rows = ids_from_rows;
  p.rows = reinterpret_cast<const uint8_t*>(rows);
  p.row_pitch = ld_rows * elem_bytes;
  p.row_bytes = (int64_t)d * elem_bytes;
  p.exit_idx = exit_idx;
  p.cont_idx = cont_idx;
  p.exit_rows = reinterpret_cast<uint8_t*>(exit_rows);
  p.cont_rows = reinterpret_cast<uint8_t*>(cont_rows);
  p.counts = counts;
  p.ws = reinterpret_cast<Workspace*>(workspace);
  int dev = 0;
  cudaGetDevice(&dev);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)sm_count(dev) * 4));
  // dense rows with the index lists and counts requested: scan, then the
  // parallel gather over those lists (same outputs as the in-scan gather)
  const bool split_gather = rows && !row_idx && exit_idx && cont_idx && counts;
  if (split_gather) {
    p.rows = nullptr;
    p.exit_rows = p.cont_rows = nullptr;
  }
  compact_kernel<<<grid, kCThreads, 0, stream>>>(p);
  int rc = check_launch("compact_kernel");
  if (rc || !split_gather) return rc;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(sm_count(dev) * 8));
  cfg.blockDim = dim3(256);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, gather_rows_kernel, (const int64_t*)exit_idx, (const int64_t*)cont_idx,
                     (const int64_t*)counts, reinterpret_cast<const uint8_t*>(rows),
                     (int64_t)(ld_rows * elem_bytes), (int64_t)d * elem_bytes,
                     reinterpret_cast<uint8_t*>(exit_rows), reinterpret_cast<uint8_t*>(cont_rows));
  return check_launch("gather_rows_kernel");
}

// ---------------------------------------------------------------------------
// u8 exit codes for the multi-GPU exchange: code = layer + 1
// for a token that exited at checkpoint `layer`, 0 for NO_EXIT (-1).  One byte
// per token is what crosses NVLink; every rank then rebuilds the global exit
// list with one compact_kernel scan of the gathered codes (nonzero = exited).
__global__ void exit_encode_kernel(const int64_t* __restrict__ layers, int64_t n,
                                   uint8_t* __restrict__ code) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    code[i] = (uint8_t)(layers[i] + 1);
}

__global__ void exit_decode_kernel(const uint8_t* __restrict__ code, int64_t n,
                                   int64_t* __restrict__ layers) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    layers[i] = (int64_t)code[i] - 1;
}

int exit_code_launch(const int64_t* layers, int64_t n, uint8_t* code, int decode,
                     cudaStream_t stream) {
  if (n == 0) return 0;
  int dev = 0;
  cudaGetDevice(&dev);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256,
                                                               (int64_t)sm_count(dev) * 8));
  if (decode)
    exit_decode_kernel<<<grid, 256, 0, stream>>>(code, n, const_cast<int64_t*>(layers));
  else
    exit_encode_kernel<<<grid, 256, 0, stream>>>(layers, n, code);
  return check_launch(decode ? "exit_decode_kernel" : "exit_encode_kernel");
}

}  // namespace tide
