// tcgen05.mma (kind::f16, SS mode, cta_group::1) throughput vs M / N and the
// number of independent accumulators: cycles per MMA over a stream of MMAs
// (K = 16 each) issued by one elected lane of a warp that walks the loop
// (operands in uniform registers), then one commit + wait.  One CTA per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_rate_probe mma_rate_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ bool elect() {
  uint32_t pred = 0;
  asm volatile("{\n.reg .pred p;\nelect.sync _|p, 0xffffffff;\nselp.u32 %0, 1, 0, p;\n}" : "=r"(pred));
  return pred != 0;
}
template <int M, int N, int NACC>
__global__ void __launch_bounds__(64, 1) probe(int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0x3f803f80u;
  if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
  const uint64_t a0 = desc(su32(base)), b0 = desc(su32(base + 48 * 1024));
  if (warp == 0) {
    const long long t0 = clock64();
    for (int i = 0; i < iters; i += 4 * NACC) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int a = 0; a < NACC; ++a)
          if (elect()) mma(tmem + a * N, a0 + 2 * k, b0 + 2 * k, idesc, (i | k) != 0);
    }
    if (elect()) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
    uint32_t ok = 0;
    while (!ok) asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0,1,0,p;\n}\n" : "=r"(ok) : "r"(su32(&bar)) : "memory");
    const long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}
template <int M, int N, int NACC>
void run(long long* d) {
  const int iters = 4096;
  CK(cudaFuncSetAttribute(probe<M, N, NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
  probe<M, N, NACC><<<148, 64, 100 * 1024>>>(iters, d);
  CK(cudaDeviceSynchronize());
  long long o;
  CK(cudaMemcpy(&o, d, 8, cudaMemcpyDeviceToHost));
  printf("M=%3d N=%3d acc=%d: %6.1f cyc/MMA\n", M, N, NACC, (double)o / iters);
}
int main() {
  long long* d; CK(cudaMalloc(&d, 8 * 148));
  run<128, 16, 1>(d); run<128, 16, 4>(d); run<128, 32, 1>(d); run<128, 64, 1>(d);
  run<128, 128, 1>(d); run<128, 128, 2>(d); run<128, 256, 1>(d);
  run<64, 16, 1>(d); run<64, 64, 1>(d); run<64, 128, 1>(d); run<64, 256, 1>(d);
  return 0;
}
