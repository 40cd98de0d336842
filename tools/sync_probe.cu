// Microbenchmarks of the synchronisation / MMA primitives the route kernel is
// built from (B200, sm_100a).  One CTA per SM, timings in SM cycles.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sync_probe sync_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void mb_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory"); }
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t ph) {
  uint32_t ok = 0;
  while (!ok) asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0,1,0,p;\n}\n" : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void commit(uint64_t* b) { asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(b)) : "memory"); }
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ uint64_t desc(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}

struct Out { long long cyc[16]; };

// mode 0: mbarrier ping-pong between warp 0 and warp 1 (round trip)
// mode 1: commit + wait (no MMA) loop
// mode 2: 4 MMAs (N) + commit + wait  (latency)
// mode 3: throughput: 4 MMAs + commit to ring of 9, wait 8 behind
// mode 4: throughput with 8 MMAs per commit (two 64-col chunks per stage)
// mode 5: MMA issue only (no commits) for 4096 MMAs, one final commit + wait
__global__ void __launch_bounds__(256, 1) probe(int mode, int N, int iters, Out* out, int opt) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  uint64_t* bars = (uint64_t*)(base + 208 * 1024);
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { for (int i = 0; i < 32; ++i) mb_init(&bars[i], 1); bars[29] = 0; asm volatile("fence.mbarrier_init.release.cluster;"); }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  const uint32_t a0 = su32(base), b0 = su32(base + 32 * 1024);
  long long t0 = 0, t1 = 0;
  if (mode == 0) {
    if (lane == 0) {
      uint32_t ph = 0;
      __syncwarp(1);
      if (warp == 0) t0 = clock64();
      for (int i = 0; i < iters; ++i) {
        if (warp == 0) { mb_arrive(&bars[0]); mb_wait(&bars[1], ph); }
        else { mb_wait(&bars[0], ph); mb_arrive(&bars[1]); }
        ph ^= 1;
      }
      if (warp == 0) { t1 = clock64(); out[blockIdx.x].cyc[0] = (t1 - t0) / iters; }
    }
  } else if (warp >= 2) {
    // spinner warps (opt bit4: spin on try_wait of a barrier that completes at the end;
    // bit5: spin with nanosleep backoff); else idle
    if (opt & 48) {
      volatile uint32_t* stop = (volatile uint32_t*)&bars[29];
      while (*stop == 0) {
        uint32_t ok;
        asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0,1,0,p;\n}\n" : "=r"(ok) : "r"(su32(&bars[30])), "r"(0u) : "memory");
        if (opt & 32) __nanosleep(200);
      }
    }
  } else if (warp == 0 && lane == 0) {
    uint32_t ph = 0;
    t0 = clock64();
    if (mode == 1) {
      for (int i = 0; i < iters; ++i) { commit(&bars[0]); mb_wait(&bars[0], ph); ph ^= 1; }
    } else if (mode == 2) {
      for (int i = 0; i < iters; ++i) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        for (int k = 0; k < 4; ++k) mma(tmem, desc(a0 + 32 * k), desc(b0 + 32 * k), idesc, (i | k) != 0);
        commit(&bars[0]); mb_wait(&bars[0], ph); ph ^= 1;
      }
    } else if (mode == 3 || mode == 4) {
      const int per = mode == 3 ? 4 : 8;
      uint32_t phs = 0;  // bit per barrier
      for (int i = 0; i < iters; ++i) {
        const int s = i % 9;
        if (i >= 9) { mb_wait(&bars[s], (phs >> s) & 1); phs ^= (1u << s); }
        asm volatile("tcgen05.fence::after_thread_sync;");
        for (int k = 0; k < per; ++k) mma(tmem + (i & 1) * 256, desc(a0 + 32 * (k & 3) + 16384 * (k >> 2)), desc(b0 + 32 * (k & 3) + 16384 * (k >> 2)), idesc, k != 0);
        commit(&bars[s]);
      }
      for (int i = iters; i < iters + 9; ++i) { const int s = i % 9; mb_wait(&bars[s], (phs >> s) & 1); phs ^= (1u << s); }
    } else if (mode == 6 || mode == 7) {
      // independent accumulators: mode 6 = 4 MMAs to 4 different accumulators per commit;
      // mode 7 = 16 MMAs per commit, k-outer over 4 accumulators (4 tiles x 4 k-steps)
      const int per = mode == 6 ? 4 : 16;
      const uint32_t stride = N <= 128 ? 128 : 256;
      const int nacc = N <= 128 ? 4 : 2;
      uint32_t phs = 0;
      for (int i = 0; i < iters; ++i) {
        const int s = i % 9;
        if (i >= 9) { mb_wait(&bars[s], (phs >> s) & 1); phs ^= (1u << s); }
        asm volatile("tcgen05.fence::after_thread_sync;");
        for (int k = 0; k < per; ++k) {
          const int acc = k % nacc, kk = (k / nacc) & 3;
          mma(tmem + acc * stride, desc(a0 + 32 * kk + 16384 * (acc & 1)), desc(b0 + 32 * kk), idesc, (i | (k / nacc)) != 0);
        }
        commit(&bars[s]);
      }
      for (int i = iters; i < iters + 9; ++i) { const int s = i % 9; mb_wait(&bars[s], (phs >> s) & 1); phs ^= (1u << s); }
    } else if (mode >= 8 && mode <= 11) {
      // mode 3 variants: 8 = no fence, 9 = no wait, 10 = no commit (no wait), 11 = wait on the
      // barrier committed 2 iterations ago (shallow ring)
      uint32_t phs = 0;
      for (int i = 0; i < iters; ++i) {
        const int s = i % 9;
        if (mode == 8 || mode == 11) { if (i >= 9) { mb_wait(&bars[s], (phs >> s) & 1); phs ^= (1u << s); } }
        if (mode != 8) asm volatile("tcgen05.fence::after_thread_sync;");
        for (int k = 0; k < 4; ++k) mma(tmem + (i & 1) * 256, desc(a0 + 32 * k), desc(b0 + 32 * k), idesc, k != 0);
        if (mode != 10) commit(&bars[s]);
      }
      if (mode == 8 || mode == 11) for (int i = iters; i < iters + 9; ++i) { const int s = i % 9; mb_wait(&bars[s], (phs >> s) & 1); phs ^= (1u << s); }
      else { commit(&bars[15]); mb_wait(&bars[15], 0); }
    } else if (mode == 12) {
      // the route kernel's MMA pattern: per k-chunk, 4 tiles x 4 K-steps (same acc x4),
      // A slots cycling through 9 x 16 KB, W slots through 4 x 16 KB.
      // opt bit0: one commit per k-chunk instead of 5; bit1: fixed A/W slot addresses;
      // bit2: wait on the k-chunk barrier from 2 chunks ago; bit3: no fence
      uint32_t phs = 0;
      int as = 0;
      for (int i = 0; i < iters; ++i) {
        const int s = i % 8;
        if ((opt & 4) && i >= 8) { mb_wait(&bars[s], (phs >> s) & 1); phs ^= (1u << s); }
        if (!(opt & 8)) asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t wb = (opt & 2) ? b0 : su32(base + 144 * 1024 + (i % 4) * 16384);
        for (int t = 0; t < 4; ++t) {
          const uint32_t ab = (opt & 2) ? a0 : su32(base + ((as + t) % 9) * 16384);
          for (int k = 0; k < 4; ++k) mma(tmem + t * 128, desc(ab + 32 * k), desc(wb + 32 * k), idesc, (i | k) != 0);
        }
        as = (as + 4) % 9;
        if (opt & 1) commit(&bars[s]);
        else { for (int t = 0; t < 4; ++t) commit(&bars[16 + t]); commit(&bars[s]); }
      }
      if (opt & 4) { for (int i = iters; i < iters + 8; ++i) { const int s = i % 8; mb_wait(&bars[s], (phs >> s) & 1); phs ^= (1u << s); } }
      else { commit(&bars[31]); mb_wait(&bars[31], 0); }
    } else if (mode == 13) {
      // commit-only throughput: one commit per slot into a ring of 9, waiting 8 behind
      uint32_t phs = 0;
      for (int i = 0; i < iters; ++i) {
        const int s = i % 9;
        if (i >= 9) { mb_wait(&bars[s], (phs >> s) & 1); phs ^= (1u << s); }
        asm volatile("tcgen05.fence::after_thread_sync;");
        commit(&bars[s]);
      }
      for (int i = iters; i < iters + 9; ++i) { const int s = i % 9; mb_wait(&bars[s], (phs >> s) & 1); phs ^= (1u << s); }
    } else if (mode == 5) {
      for (int i = 0; i < iters; ++i)
        for (int k = 0; k < 4; ++k) mma(tmem + (i & 1) * 256, desc(a0 + 32 * k), desc(b0 + 32 * k), idesc, k != 0);
      commit(&bars[0]); mb_wait(&bars[0], 0);
    }
    t1 = clock64();
    out[blockIdx.x].cyc[0] = (t1 - t0) / iters;
    *(volatile uint32_t*)&bars[29] = 1;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  Out* d; CK(cudaMalloc(&d, sizeof(Out) * 148));
  CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  const char* names[] = {"mbarrier ping-pong (round trip)", "commit+wait, no MMA", "4 MMA + commit + wait (latency)", "4 MMA/commit, ring of 9 (thru)", "8 MMA/commit, ring of 9 (thru)", "MMA issue only (per 4 MMAs)", "4 indep-acc MMA/commit, ring 9", "16 MMA (4acc x 4k)/commit, ring 9", "mode3 without fence", "mode3 without wait", "mode3 no commit/wait", "mode3 again"};
  for (int mode : {0, 1, 2, 3, 13}) {
    probe<<<148, 64, 220 * 1024>>>(mode, 128, 1000, d, 0); CK(cudaDeviceSynchronize());
    Out o; CK(cudaMemcpy(&o, d, sizeof(Out), cudaMemcpyDeviceToHost));
    printf("mode %2d %-40s: %lld cyc/iter\n", mode, mode == 13 ? "commit-only ring of 9 (thru)" : names[mode], o.cyc[0]);
  }
  for (int opt : {0, 2, 5, 7}) for (int nthr : {64}) {
    const int N = 128;
    const int iters = 1000;
    probe<<<148, nthr, 220 * 1024>>>(12, N, iters, d, opt);
    CK(cudaDeviceSynchronize());
    Out o; CK(cudaMemcpy(&o, d, sizeof(Out), cudaMemcpyDeviceToHost));
    printf("route pattern opt=%2d threads=%3d (1commit=%d wait=%d spinners=%d sleep=%d): %6lld cyc per k-chunk = %5.1f per MMA\n", opt, nthr, opt & 1, (opt >> 2) & 1, (opt >> 4) & 1, (opt >> 5) & 1, o.cyc[0], o.cyc[0] / 16.0);
  }
  { probe<<<148, 64, 220 * 1024>>>(5, 128, 1000, d, 0); CK(cudaDeviceSynchronize()); Out o; CK(cudaMemcpy(&o, d, sizeof(Out), cudaMemcpyDeviceToHost)); printf("issue-only reference N=128: %lld per 4 MMAs\n", o.cyc[0]); }
  return 0;
}
