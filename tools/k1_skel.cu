// Streaming-skeleton probe for K1 (route_tc.cu): the same TMA ring / tcgen05
// MMA / RMS-read structure over 65,536 x 4096 bf16 rows, without the epilogue
// or compaction, with compile-time variants of the synchronisation scheme.
// Prints the kernel time of each variant (CUDA events, best of 5).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o k1_skel k1_skel.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include <vector>

#define TIDE_SPIN_LIMIT 0x40000000u
#include "../paper_2603_21365_b200/csrc/common.cuh"

using namespace tide;

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e = (x);                                                              \
    if (e != cudaSuccess) {                                                           \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));              \
      exit(1);                                                                        \
    }                                                                                 \
  } while (0)

constexpr int kSlot = 16384;
constexpr int kGranS = 16;

struct SkelParams {
  int n, d, nk, na, nw;
  uint32_t flags;  // 1 = MMA, 2 = RMS reads, 4 = TMA
  uint32_t idesc, idesc2, idesc64;
  float* out;
};

// CM: 0 = commit per tile + per W slot (base); 1 = one commit per k-chunk (stage);
//     2 = commit per tile, W slot freed by the chunk's last tile commit
// NR: RMS warps (4: one set reads every tile; 8: two sets split tiles 0-1 / 2-3)
// RL: RMS release point: 0 = right after the smem loads, 1 = after the math
template <int CM, int NR, int RL>
__global__ void __launch_bounds__(64 + 32 * NR, 1)
    skel(const __grid_constant__ CUtensorMap tm_h, const __grid_constant__ CUtensorMap tm_w,
         const __grid_constant__ SkelParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sW = smem;
  uint8_t* sA = smem + p.nw * kSlot;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sA + p.na * kSlot);
  uint64_t* w_full = bars;            // 8
  uint64_t* w_empty = bars + 8;       // 8
  uint64_t* a_full = bars + 16;       // 16
  uint64_t* a_empty = bars + 32;      // 16 (CM 0/2) or stage barriers (CM 1)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 64);
  uint32_t* slot_st = tslot + 4;      // CM 1: stage (+1) that last used each A slot

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n32 = (p.n + kGranS - 1) / kGranS;
  const int G = gridDim.x;
  const int r0 = (int)((long long)blockIdx.x * n32 / G) * kGranS;
  int r1 = (int)((long long)(blockIdx.x + 1) * n32 / G) * kGranS;
  if (r1 > p.n) r1 = p.n;
  const int T = (r1 - r0 + 127) / 128;
  const int rms_per_tile = NR == 8 ? 4 : 4;  // warps reading each tile
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) { mbar_init(&w_full[i], 1); mbar_init(&w_empty[i], 1); }
    for (int i = 0; i < 16; ++i) {
      mbar_init(&a_full[i], 1);
      mbar_init(&a_empty[i], CM == 1 ? 1 + NR : 1 + rms_per_tile);
      slot_st[i] = 0;
    }
    fence_mbar_init();
  }
  if (warp == 1) { tmem_alloc(tslot, 512); tmem_relinquish(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  long long c_start = clock64();
  unsigned long long g_start;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_start));

  if (warp == 0) {
    if (lane == 0 && (p.flags & 128)) {
      // quad order: W for 4 k-chunks, then per tile its 4 k-chunks back to back
      // (the 4 boxes of a row's 512 contiguous bytes are requested together)
      const uint64_t pol_h = policy_evict_first(), pol_w = policy_evict_last();
      int as = 0, aph = 0, wsl = 0, wph = 0;
      for (int kq = 0; kq < p.nk; kq += 4) {
        for (int kc = kq; kc < kq + 4 && kc < p.nk; ++kc) {
          mbar_wait(&w_empty[wsl], wph ^ 1);
          mbar_arrive_expect_tx(&w_full[wsl], kSlot);
          tma_load_2d(sW + wsl * kSlot, &tm_w, &w_full[wsl], kc * 64, 0, pol_w);
          if (++wsl == p.nw) { wsl = 0; wph ^= 1; }
        }
        for (int t = 0; t < T; ++t)
          for (int kc = kq; kc < kq + 4 && kc < p.nk; ++kc) {
            mbar_wait(&a_empty[as], aph ^ 1);
            mbar_arrive_expect_tx(&a_full[as], kSlot);
            tma_load_2d(sA + as * kSlot, &tm_h, &a_full[as], kc * 64, r0 + 128 * t, pol_h);
            if (++as == p.na) { as = 0; aph ^= 1; }
          }
      }
    } else if (lane == 0) {
      const uint64_t pol_h = policy_evict_first(), pol_w = policy_evict_last();
      int as = 0, aph = 0, wsl = 0, wph = 0;
      for (int kc = 0; kc < p.nk; ++kc) {
        if (CM == 1) {
          if (kc >= p.nw) mbar_wait(&a_empty[(kc - p.nw) & 15], ((kc - p.nw) >> 4) & 1);
        } else {
          mbar_wait(&w_empty[wsl], wph ^ 1);
        }
        if ((p.flags & 4) && !((p.flags & 8) && kc >= p.nw)) {
          mbar_arrive_expect_tx(&w_full[wsl], kSlot);
          tma_load_2d(sW + wsl * kSlot, &tm_w, &w_full[wsl], kc * 64, 0, pol_w);
        } else {
          mbar_arrive(&w_full[wsl]);
        }
        if (++wsl == p.nw) { wsl = 0; wph ^= 1; }
        for (int t = 0; t < T; ++t) {
          if (CM == 1) {
            const uint32_t prev = slot_st[as];
            if (prev) mbar_wait(&a_empty[(prev - 1) & 15], ((prev - 1) >> 4) & 1);
            slot_st[as] = kc + 1;
          } else {
            mbar_wait(&a_empty[as], aph ^ 1);
          }
          if (p.flags & 4) {
            mbar_arrive_expect_tx(&a_full[as], kSlot);
            tma_load_2d(sA + as * kSlot, &tm_h, &a_full[as], kc * 64, r0 + 128 * t, pol_h);
          } else {
            mbar_arrive(&a_full[as]);
          }
          if (++as == p.na) { as = 0; aph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    int as = 0, aph = 0, wsl = 0, wph = 0;
    const uint64_t dhi = sw128_kmajor_desc(0);
    for (int kc = 0; kc < p.nk; ++kc) {
      mbar_wait(&w_full[wsl], wph);
      const uint64_t bdesc = dhi | (uint64_t)((smem_u32(sW + wsl * kSlot) & 0x3FFFFu) >> 4);
      if (p.flags & 32) {
        // transposed: D^T[b, 256 tokens] = W (A, M=128) x tokens (B, N=256) over
        // two adjacent 128-row slots; one MMA per k-step covers two tiles
        for (int t0 = 0; t0 < T; t0 += 2) {
          int sl0 = as;
          for (int u = 0; u < 2; ++u) {
            mbar_wait(&a_full[as], aph);
            if (++as == p.na) { as = 0; aph ^= 1; }
          }
          tc_fence_after();
          if (elect_one()) {
            const uint64_t tdesc = dhi | (uint64_t)((smem_u32(sA + sl0 * kSlot) & 0x3FFFFu) >> 4);
#pragma unroll
            for (int k = 0; k < 4; ++k)
              tc_mma_f16(tmem + (t0 >> 1) * 256, bdesc + 2 * k, tdesc + 2 * k, p.idesc2, (kc | k) != 0);
            tc_commit(&a_empty[sl0]);
            tc_commit(&a_empty[sl0 + 1]);
          }
          __syncwarp();
        }
        if (elect_one()) tc_commit(&w_empty[wsl]);
        __syncwarp();
        if (++wsl == p.nw) { wsl = 0; wph ^= 1; }
        continue;
      }
      if (p.flags & 16) {
        // k-step-outer: all T slots of the chunk, then W slice k for every tile
        // pairs of tiles: W slice k feeds two tiles back to back
        for (int t0 = 0; t0 < T; t0 += 2) {
          const int np = (T - t0) < 2 ? 1 : 2;
          int sl[2];
          for (int u = 0; u < np; ++u) {
            sl[u] = as;
            mbar_wait(&a_full[as], aph);
            if (++as == p.na) { as = 0; aph ^= 1; }
          }
          tc_fence_after();
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < 4; ++k)
#pragma unroll
              for (int u = 0; u < 2; ++u)
                if (u < np) {
                  const uint64_t adesc = dhi | (uint64_t)((smem_u32(sA + sl[u] * kSlot) & 0x3FFFFu) >> 4);
                  tc_mma_f16(tmem + (t0 + u) * 128, adesc + 2 * k, bdesc + 2 * k, p.idesc, (kc | k) != 0);
                }
            for (int u = 0; u < np; ++u) tc_commit(&a_empty[sl[u]]);
          }
          __syncwarp();
        }
        if (elect_one()) tc_commit(&w_empty[wsl]);
        __syncwarp();
        if (++wsl == p.nw) { wsl = 0; wph ^= 1; }
        continue;
      }
      for (int t = 0; t < T; ++t) {
        mbar_wait(&a_full[as], aph);
        tc_fence_after();
        if (elect_one()) {
          const uint64_t adesc = dhi | (uint64_t)((smem_u32(sA + as * kSlot) & 0x3FFFFu) >> 4);
          if (p.flags & 1) {
            const uint32_t id = ((p.flags & 64) && t == T - 1) ? p.idesc64 : p.idesc;
#pragma unroll
            for (int k = 0; k < 4; ++k)
              tc_mma_f16(tmem + t * 128, adesc + 2 * k, bdesc + 2 * k, id, (kc | k) != 0);
          }
          if (CM == 0 || CM == 2) tc_commit(&a_empty[as]);
          if (CM == 2 && t == T - 1) tc_commit(&w_empty[wsl]);
        }
        __syncwarp();
        if (++as == p.na) { as = 0; aph ^= 1; }
      }
      if (elect_one()) {
        if (CM == 0) tc_commit(&w_empty[wsl]);
        if (CM == 1) tc_commit(&a_empty[kc & 15]);
      }
      __syncwarp();
      if (++wsl == p.nw) { wsl = 0; wph ^= 1; }
    }
  } else {
    const int rw = warp - 2;           // 0..NR-1
    const int q = warp & 3;
    const int set = NR == 8 ? rw >> 2 : 0;
    const int row = 32 * q + lane;
    const uint32_t swz = row & 7;
    int as = 0, aph = 0;
    f32x2 acc = 0ull;
    for (int kc = 0; kc < p.nk; ++kc) {
      for (int t = 0; t < T; ++t) {
        const bool mine = NR == 4 || (t >> 1) == set;
        if (mine) {
          mbar_wait(&a_full[as], aph);
          const uint8_t* rp = sA + as * kSlot + row * 128;
          uint4 u[8];
          if (p.flags & 2) {
#pragma unroll
            for (int j = 0; j < 8; ++j) u[j] = *reinterpret_cast<const uint4*>(rp + ((j ^ swz) << 4));
          } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) u[j] = make_uint4(0, 0, 0, 0);
          }
          if (CM != 1 && RL == 0) {
            __syncwarp();
            if (lane == 0) mbar_arrive(&a_empty[as]);
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint32_t w[4] = {u[j].x, u[j].y, u[j].z, u[j].w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const f32x2 x = pack2u(w[e] << 16, w[e] & 0xFFFF0000u);
              acc = ffma2(x, x, acc);
            }
          }
          if (CM != 1 && RL == 1) {
            __syncwarp();
            if (lane == 0) mbar_arrive(&a_empty[as]);
          }
        }
        if (++as == p.na) { as = 0; aph ^= 1; }
      }
      if (CM == 1) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&a_empty[kc & 15]);
      }
    }
    float lo, hi;
    unpack2(acc, lo, hi);
    if (lo + hi == 1234.5f) p.out[0] = lo;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) { tc_fence_after(); tmem_dealloc(tmem, 512); }
  if (threadIdx.x == 0) {
    unsigned long long g_end;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_end));
    p.out[2 + 2 * blockIdx.x] = (float)(clock64() - c_start);
    p.out[3 + 2 * blockIdx.x] = (float)(g_end - g_start);
  }
}

__global__ void fill_rand(uint16_t* p, size_t n, uint32_t seed, float scale) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t x = (uint32_t)i * 2654435761u ^ seed;
    x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
    const float f = ((float)(x & 0xFFFFFF) / 16777216.0f - 0.5f) * 3.4f * scale;
    const uint32_t b = __float_as_uint(f);
    p[i] = (uint16_t)(b >> 16);
  }
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                          const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                          CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                          CUtensorMapFloatOOBfill);

static CUtensorMap make(void* base, int cols, int rows, int bc, int br) {
  static EncFn enc = nullptr;
  if (!enc) {
    void* ptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q));
    enc = (EncFn)ptr;
  }
  CUtensorMap m;
  cuuint64_t gd[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t gs[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {(cuuint32_t)bc, (cuuint32_t)br};
  cuuint32_t es[2] = {1, 1};
  if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, gd, gs, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    printf("encode failed\n");
    exit(1);
  }
  return m;
}

template <int CM, int NR, int RL>
float run(const CUtensorMap& th, const CUtensorMap& tw, SkelParams p, int grid) {
  const int smem = 1024 + (p.nw + p.na) * kSlot + 64 * 8 + 128;
  CK(cudaFuncSetAttribute(skel<CM, NR, RL>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) skel<CM, NR, RL><<<grid, 64 + 32 * NR, smem>>>(th, tw, p);
  CK(cudaDeviceSynchronize());
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    for (int i = 0; i < 10; ++i) skel<CM, NR, RL><<<grid, 64 + 32 * NR, smem>>>(th, tw, p);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms / 10 < best) best = ms / 10;
  }
  float o[300];
  CK(cudaMemcpy(o, p.out, sizeof(o), cudaMemcpyDeviceToHost));
  double cyc = 0, ns = 0;
  for (int i = 0; i < 148; ++i) { cyc += o[2 + 2 * i]; ns += o[3 + 2 * i]; }
  printf("[clock %.0f MHz] ", cyc / ns * 1e3);
  return best * 1e3f;
}

int main(int argc, char** argv) {
  setvbuf(stdout, NULL, _IONBF, 0);
  const int n = 65536, d = 4096, b = 128;
  void *h, *w;
  float* out;
  CK(cudaMalloc(&h, (size_t)n * d * 2));
  CK(cudaMalloc(&w, (size_t)b * d * 2));
  CK(cudaMalloc(&out, 4096));
  if (argc > 1 && argv[1][0] == 'z') {
    CK(cudaMemset(h, 0, (size_t)n * d * 2));
    CK(cudaMemset(w, 0, (size_t)b * d * 2));
    printf("zero data\n");
  } else {
    fill_rand<<<1024, 256>>>((uint16_t*)h, (size_t)n * d, 1u, 1.0f);
    fill_rand<<<64, 256>>>((uint16_t*)w, (size_t)b * d, 7u, 0.05f);
    CK(cudaDeviceSynchronize());
    printf("random data\n");
  }
  CUtensorMap th = make(h, d, n, 64, 128), tw = make(w, d, b, 64, 128);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  SkelParams p{n, d, d / 64, 9, 4, 7u, f16_idesc(1, 128, 128), f16_idesc(1, 128, 256), f16_idesc(1, 64, 128), out};
  const double bytes = (double)n * d * 2;
  auto show = [&](const char* name, float us) {
    printf("%-58s %8.1f us  %6.0f GB/s\n", name, us, bytes / us / 1e3);
  };
  struct Cfg { int na, nw; };
  for (Cfg c : {Cfg{9, 4}}) {
    p.na = c.na;
    p.nw = c.nw;
    char nm[128];
    // flag 8: W loaded once (first nw chunks), no per-chunk W re-reads from L2
    for (uint32_t f : {4u, 12u, 7u, 15u, 7u, 15u}) {
      p.flags = f;
      const char* fs = f == 4 ? "TMA" : f == 12 ? "TMA, no W reload" : f == 7 ? "TMA+MMA+RMS" : "TMA+MMA+RMS no W rel";
      snprintf(nm, sizeof nm, "na=%d nw=%d %-16s CM0 NR8 RL0 (base)", c.na, c.nw, fs);
      show(nm, run<0, 8, 0>(th, tw, p, sms));

    }
  }
  return 0;
}
