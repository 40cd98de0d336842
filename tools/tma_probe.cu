// TMA read-bandwidth probe on B200: which access pattern streams a
// [65536 x 4096] bf16 tensor (512 MiB) fastest into shared memory?
// Producer = one thread issuing TMA into a ring of 16 KB slots; consumer = one
// warp that releases each slot as soon as it lands (no compute).  Reports GB/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_probe tma_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void mb_expect(uint64_t* b, uint32_t x) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(x) : "memory"); }
__device__ __forceinline__ void mb_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory"); }
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t ph) {
  uint32_t ok = 0, spins = 0;
  while (!ok && ++spins < (1u << 26)) asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0,1,0,p;\n}\n" : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, uint64_t* b, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(su32(dst)), "l"(m), "r"(su32(b)), "r"(c0), "r"(c1) : "memory");
}
__device__ __forceinline__ void bulk1d(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)), "l"(src), "r"(bytes), "r"(su32(b)) : "memory");
}

constexpr int SLOT = 16384;
struct P { int mode, ns, tiles, rows, cols, nk, wload; const uint8_t* base; long ld_bytes; int kq; };

__global__ void __launch_bounds__(64, 1) probe(const __grid_constant__ CUtensorMap m128, const __grid_constant__ CUtensorMap m32, const __grid_constant__ CUtensorMap mw, const __grid_constant__ P p) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = raw + ((1024 - (su32(raw) & 1023)) & 1023);
  uint64_t* full = (uint64_t*)(sm + p.ns * SLOT);
  uint64_t* empty = full + 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { for (int i = 0; i < p.ns; ++i) { mb_init(&full[i], 1); mb_init(&empty[i], 1); } asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  // rows of this CTA: contiguous balanced range
  const int G = gridDim.x;
  long r0 = (long)blockIdx.x * p.rows / G, r1 = (long)(blockIdx.x + 1) * p.rows / G;
  const int T = p.tiles;  // tiles per group (rows per group = 128*T)
  // enumerate the (tile, kchunk) schedule
  long total = 0;
  for (long g0 = r0; g0 < r1; g0 += 128L * T) {
    int tt = (int)((r1 - g0 + 127) / 128); if (tt > T) tt = T;
    total += (p.mode == 1) ? (long)tt * p.nk * (1 + p.wload) : (long)tt * p.nk + (p.wload ? p.nk : 0);
  }
  if (warp == 0 && lane == 0) {
    int s = 0, ph = 0;
    auto next = [&](uint32_t bytes) -> uint8_t* { mb_wait(&empty[s], ph ^ 1); mb_expect(&full[s], bytes); return sm + s * SLOT; };
    auto adv = [&]() { if (++s == p.ns) { s = 0; ph ^= 1; } };
    for (long g0 = r0; g0 < r1; g0 += 128L * T) {
      int tt = (int)((r1 - g0 + 127) / 128); if (tt > T) tt = T;
      if (p.mode == 0 || p.mode == 4) {          // k-outer, M-inner
        for (int kc = 0; kc < p.nk; ++kc) {
          if (p.wload) { uint8_t* d = next(SLOT); tma2d(d, &mw, &full[s], kc * 64, 0); adv(); }
          for (int t = 0; t < tt; ++t) {
            long rb = g0 + 128L * t;
            if (p.mode == 0) { uint8_t* d = next(SLOT); tma2d(d, &m128, &full[s], kc * 64, (int)rb); adv(); }
            else { uint8_t* d = next(SLOT); for (int q = 0; q < 4; ++q) tma2d(d + q * 4096, &m32, &full[s], kc * 64, (int)(rb + 32 * q)); adv(); }
          }
        }
      } else if (p.mode == 1) {                    // tile-major, K-inner
        for (int t = 0; t < tt; ++t) for (int kc = 0; kc < p.nk; ++kc) {
          if (p.wload) { uint8_t* d = next(SLOT); tma2d(d, &mw, &full[s], kc * 64, 0); adv(); }
          long rb = g0 + 128L * t; uint8_t* d = next(SLOT); tma2d(d, &m128, &full[s], kc * 64, (int)rb); adv();
        }
      } else if (p.mode == 2) {                    // k-quads: 4 consecutive k-chunks per tile
        for (int kq = 0; kq < p.nk; kq += p.kq) {
          if (p.wload) for (int kk = 0; kk < p.kq; ++kk) { uint8_t* d = next(SLOT); tma2d(d, &mw, &full[s], (kq + kk) * 64, 0); adv(); }
          for (int t = 0; t < tt; ++t) for (int kk = 0; kk < p.kq; ++kk) {
            long rb = g0 + 128L * t; uint8_t* d = next(SLOT); tma2d(d, &m128, &full[s], (kq + kk) * 64, (int)rb); adv();
          }
        }
      } else if (p.mode == 3) {                    // contiguous 1D bulk copies of 16 KB
        const uint8_t* src = p.base + g0 * p.ld_bytes;
        long bytes = (long)tt * 128 * p.ld_bytes;
        for (long o = 0; o < bytes; o += SLOT) { uint8_t* d = next(SLOT); bulk1d(d, src + o, SLOT, &full[s]); adv(); }
      }
    }
  } else if (warp == 1) {
    int s = 0, ph = 0;
    for (long i = 0; i < total; ++i) {
      mb_wait(&full[s], ph);
      __syncwarp();
      if (lane == 0) mb_arrive(&empty[s]);
      if (++s == p.ns) { s = 0; ph ^= 1; }
    }
  }
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static void mk(EncFn enc, CUtensorMap* m, void* base, long cols, long rows, int bc, int br, CUtensorMapL2promotion prom) {
  cuuint64_t gd[2] = {(cuuint64_t)cols, (cuuint64_t)rows}; cuuint64_t gs[1] = {(cuuint64_t)cols * 2};
  cuuint32_t bx[2] = {(cuuint32_t)bc, (cuuint32_t)br}; cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, gd, gs, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, prom, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r) { printf("encode failed %d\n", r); exit(1); }
}

int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  const long rows = 65536, cols = 4096;
  void* h; CK(cudaMalloc(&h, rows * cols * 2)); CK(cudaMemset(h, 1, rows * cols * 2));
  void* w; CK(cudaMalloc(&w, 128 * cols * 2)); CK(cudaMemset(w, 1, 128 * cols * 2));
  void* fp; cudaDriverEntryPointQueryResult q; CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q));
  EncFn enc = (EncFn)fp;
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[] = {"k-outer 4 tiles box64x128", "tile-major k-inner", "k-quads per tile", "1D bulk 16KB contiguous", "k-outer box64x32 x4"};
  CUtensorMap m128, m32, mw;
  CUtensorMapL2promotion pr = CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  mk(enc, &m128, h, cols, rows, 64, 128, pr); mk(enc, &m32, h, cols, rows, 64, 32, pr); mk(enc, &mw, w, cols, 128, 64, 128, pr);
  struct Cfg { int mode, kq, tiles, ns, wl; };
  std::vector<Cfg> cfgs = {{0,1,4,9,1},{0,1,4,7,1},{2,2,4,7,1},{2,2,4,9,1},{2,4,4,7,1},{2,4,4,5,1},{2,8,4,9,1},{2,2,2,9,1},{2,4,2,9,1},{1,1,4,9,1},{2,2,4,12,1},{2,4,4,12,1},{2,1,4,9,0},{2,4,4,9,0},{2,8,4,9,0}};
  for (auto c : cfgs) {
      P p{c.mode, c.ns, c.tiles, (int)rows, (int)cols, (int)(cols / 64), c.wl, (const uint8_t*)h, cols * 2, c.kq};
      size_t smem = c.ns * SLOT + 1024 + 1024;
      for (int it = 0; it < 2; ++it) probe<<<sms, 64, smem>>>(m128, m32, mw, p);
      CK(cudaDeviceSynchronize());
      const int reps = 5;
      cudaEventRecord(e0);
      for (int it = 0; it < reps; ++it) probe<<<sms, 64, smem>>>(m128, m32, mw, p);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= reps;
      double gbs = rows * cols * 2 / (ms * 1e-3) / 1e9;
      printf("mode=%d kq=%d tiles=%d ns=%2d wload=%d  %8.1f us  %7.0f GB/s (h bytes only)\n", c.mode, c.kq, c.tiles, c.ns, c.wl, ms * 1e3, gbs);
  }
  return 0;
}
