// Per-SM streaming ceiling on B200: G CTAs each stream its own slice of a
// buffer into a ring of 16 KB smem slots by TMA (one producer thread, one
// consumer warp releasing each slot; optionally 4 consumer warps reading the
// slot like the RMS warps).  Reports GB/s total and per CTA, for G and for
// L2-resident (32 MB) vs HBM (512 MB) buffers.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sm_stream_probe sm_stream_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void mb_expect(uint64_t* b, uint32_t x) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(x) : "memory"); }
__device__ __forceinline__ void mb_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory"); }
__device__ int g_wait_mode;  // 0 try_wait, 1 test_wait spin, 2 try_wait + 1000 ns hint, 3 try_wait + 20 ns hint
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t ph) {
  uint32_t ok = 0;
  const int m = g_wait_mode;
  if (m == 1) {
    while (!ok) asm volatile("{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0,1,0,p;\n}\n" : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory");
  } else if (m >= 2) {
    const uint32_t hint = m == 2 ? 1000u : 20u;
    while (!ok) asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\nselp.u32 %0,1,0,p;\n}\n" : "=r"(ok) : "r"(su32(b)), "r"(ph), "r"(hint) : "memory");
  } else {
    while (!ok) asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0,1,0,p;\n}\n" : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory");
  }
}
__device__ __forceinline__ void bulk1d(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)), "l"(src), "r"(bytes), "r"(su32(b)) : "memory");
}
constexpr int SLOT = 16384;
__global__ void __launch_bounds__(192, 1) probe(const uint8_t* base, long bytes_per_cta, int ns, int readers, int slot, int split) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = raw + ((1024 - (su32(raw) & 1023)) & 1023);
  uint64_t* full = (uint64_t*)(sm + ns * slot);
  uint64_t* empty = full + 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { for (int i = 0; i < ns; ++i) { mb_init(&full[i], 1); mb_init(&empty[i], readers); } asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  const uint8_t* src = base + blockIdx.x * bytes_per_cta;
  const long nchunks = bytes_per_cta / slot;
  if (warp == 0) {
    if (lane == 0) {
      for (long i = 0; i < nchunks; ++i) {
        int s = i % ns; uint32_t ph = (i / ns) & 1;
        mb_wait(&empty[s], ph ^ 1); mb_expect(&full[s], slot);
        for (int q = 0; q < split; ++q)
          bulk1d(sm + s * slot + q * (slot / split), src + i * slot + q * (slot / split), slot / split, &full[s]);
      }
    }
  } else if (warp >= 2 && warp < 2 + readers) {
    float acc = 0.f;
    for (long i = 0; i < nchunks; ++i) {
      int s = i % ns; uint32_t ph = (i / ns) & 1;
      mb_wait(&full[s], ph);
      const uint4* rp = (const uint4*)(sm + s * slot) + lane;
      for (int j = 0; j < slot / 16 / 32 / readers; ++j) { uint4 u = rp[(warp - 2) * (slot / 16 / readers) + j * 32]; acc += __uint_as_float(u.x); }
      __syncwarp();
      if (lane == 0) mb_arrive(&empty[s]);
    }
    if (acc == 12345.f) printf("x");
  }
}
int main() {
  const long total = 512l << 20;
  uint8_t* buf; CK(cudaMalloc(&buf, total)); CK(cudaMemset(buf, 1, total));
  CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int mode : {0}) for (int slot : {16384, 32768, 65536}) for (int split : {1, 2, 4, 8}) for (int readers : {4}) for (long region : {512l << 20}) for (int G : {32, 148}) {
    if (slot / split < 4096) continue;
    CK(cudaMemcpyToSymbol(g_wait_mode, &mode, sizeof(int)));
    const int ns = (200 * 1024) / slot;
    long per = (region / G) / slot * slot;
    for (int it = 0; it < 2; ++it) probe<<<G, 192, ns * slot + 2048>>>(buf, per, ns, readers, slot, split);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    const int reps = 5;
    for (int it = 0; it < reps; ++it) probe<<<G, 192, ns * slot + 2048>>>(buf, per, ns, readers, slot, split);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= reps;
    double gbs = (double)per * G / (ms * 1e-3) / 1e9;
    printf("split=%d mode=%d slot=%5d readers=%d region=%4ld MB G=%3d: %7.1f us  %7.0f GB/s  %6.1f GB/s/CTA\n", split, mode, slot, readers, region >> 20, G, ms * 1e3, gbs, gbs / G);
  }
  return 0;
}
