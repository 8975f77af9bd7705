// Micro-benchmark (dev tool): tcgen05.mma (kind::f16, bf16 -> fp32, cta_group::1) cycles per
// instruction for the attention backward's shapes, SS (A and B from smem) vs TS (A from TMEM),
// one CTA per SM, one thread issuing back-to-back MMAs into one accumulator.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2205_05198_b200/csrc -o bench_umma bench_umma.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "tc_common.cuh"

using namespace spl::k::tc;

// mode 0: SS, K-major A and B (A rows M, B rows N; 64-element SW128 atoms)
// mode 1: TS, A from TMEM, B K-major from smem
// mode 2: SS, A MN-major (M contiguous), B MN-major (N contiguous)
__device__ __forceinline__ void ld32x(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
}
__device__ volatile int g_stop;
__device__ float g_sink;

// STRESS 0: none; 1: 8 warps of back-to-back tcgen05.ld (TMEM reads of other columns);
// 2: 8 warps of ld.shared.v4 broadcast loops; 3: 8 warps of st.shared.v4
template <int M, int N, int MODE, int STRESS = 0>
__global__ void __launch_bounds__(384, 1) umma_k(int iters, unsigned long long* cyc) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;  // small bf16 values
  fence_proxy_async();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tmem_alloc_warp(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  __shared__ volatile int done;
  if (threadIdx.x == 0) done = 0;
  __syncthreads();
  if (STRESS != 0 && warp >= 4) {
    float acc = 0.f;
    uint32_t r[32];
    const uint32_t sa = smem_u32(smem + 65536) + (threadIdx.x & 31) * 16;
    while (!done) {
      if constexpr (STRESS == 1) {
        ld32x(tmem + ((uint32_t)((warp & 3) * 32) << 16) + 384 + ((warp >> 2) & 3) * 32, r);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        acc += __uint_as_float(r[0]) + __uint_as_float(r[31]);
      } else if constexpr (STRESS == 2) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          uint32_t a0, a1, a2, a3;
          asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3) : "r"(sa + j * 512));
          acc += __uint_as_float(a0 ^ a3);
        }
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j)
          asm volatile("st.shared.v4.b32 [%0], {%1,%1,%1,%1};" ::"r"(sa + j * 512), "r"(j) : "memory");
      }
    }
    g_sink = acc;
  }
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = make_idesc(M, N, MODE == 2, MODE == 2);
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const int kk = i & 3;
      if constexpr (MODE == 0)
        umma_bf16(tmem, smem_desc(a + kk * 32, 16, 1024), smem_desc(b + kk * 32, 16, 1024), idesc, 1u);
      else if constexpr (MODE == 1)
        umma_bf16_ts(tmem, tmem + 256 + kk * 8, smem_desc(b + kk * 32, 16, 1024), idesc, 1u);
      else
        umma_bf16(tmem, smem_desc(a + kk * 2048, 16384, 1024), smem_desc(b + kk * 2048, 8192, 1024), idesc, 1u);
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    const long long t1 = clock64();
    cyc[blockIdx.x] = (unsigned long long)(t1 - t0);
    done = 1;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc_warp(tmem, 512);
  }
}

template <int M, int N, int MODE, int STRESS = 0>
void run(const char* name, int sms, unsigned long long* cyc) {
  const int iters = 4096;
  cudaFuncSetAttribute(umma_k<M, N, MODE, STRESS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  umma_k<M, N, MODE, STRESS><<<sms, STRESS ? 384 : 128, 100 * 1024>>>(iters, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[256];
  cudaMemcpy(h, cyc, sms * 8, cudaMemcpyDeviceToHost);
  double c = 0;
  for (int i = 0; i < sms; ++i) c += h[i];
  c /= sms;
  const double per = c / iters;
  const double flops = 2.0 * M * N * 16;
  printf("%-28s M=%3d N=%3d: %6.1f cycles/MMA  (%5.0f flop/clk/SM = %4.0f%% of 8192)  %s\n", name,
         M, N, per, flops / per, 100.0 * flops / per / 8192, cudaGetErrorString(e));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* cyc;
  cudaMalloc(&cyc, sms * 8);
  run<128, 64, 0>("SS K-major", sms, cyc);
  run<128, 96, 0>("SS K-major", sms, cyc);
  run<128, 128, 0>("SS K-major", sms, cyc);
  run<128, 256, 0>("SS K-major", sms, cyc);
  run<64, 96, 0>("SS K-major", sms, cyc);
  run<64, 128, 0>("SS K-major", sms, cyc);
  run<128, 64, 1>("TS", sms, cyc);
  run<128, 96, 1>("TS", sms, cyc);
  run<128, 128, 1>("TS", sms, cyc);
  run<128, 256, 1>("TS", sms, cyc);
  run<128, 64, 2>("SS MN-major", sms, cyc);
  run<128, 96, 2>("SS MN-major", sms, cyc);
  run<64, 96, 2>("SS MN-major", sms, cyc);
  run<128, 64, 0, 1>("SS + 8w TMEM-ld stress", sms, cyc);
  run<128, 96, 1, 1>("TS + 8w TMEM-ld stress", sms, cyc);
  run<128, 64, 0, 2>("SS + 8w LDS stress", sms, cyc);
  run<128, 96, 1, 2>("TS + 8w LDS stress", sms, cyc);
  run<128, 64, 0, 3>("SS + 8w STS stress", sms, cyc);
  return 0;
}
