// Micro-benchmark (dev tool): tcgen05.ld throughput per SM — W warps (W/4 per TMEM lane
// quadrant) each repeatedly load 32 lanes x 32 columns x 4 B with 32x32b.x32, optionally while
// one thread keeps the tensor core busy with M=128 N=128 K=16 SS MMAs into other TMEM columns.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2205_05198_b200/csrc tmem_ld_bw.cu
#include <cstdio>
#include <cuda.h>
#include "../../paper_2205_05198_b200/csrc/tc_common.cuh"
using namespace spl::k::tc;

__global__ void __launch_bounds__(544, 1) k(int iters, int with_mma, unsigned long long* out) {
  __shared__ uint32_t slot;
  __shared__ __align__(1024) uint8_t ab[2 * 16384];
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5;
  const int nld = (blockDim.x >> 5) - 1;  // warps 0..nld-1 load, the last warp issues MMAs
  if (warp == 0) tmem_alloc_warp(&slot, 512);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  for (int i = threadIdx.x; i < 2 * 16384 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(ab)[i] = 0;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  unsigned long long t0 = clock64();
  if (warp < nld) {
    const uint32_t tl = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) % 4) * 32;
    uint32_t acc = 0;
    for (int it = 0; it < iters; ++it) {
      uint32_t r[32];
      tmem_ld32_nw(tl, r);
      tmem_wait();
#pragma unroll
      for (int i = 0; i < 32; ++i) acc += r[i];
    }
    if (acc == 0x12345678u) out[2] = acc;
  } else if (with_mma) {
    if ((threadIdx.x & 31) == 0) {
      constexpr uint32_t idesc = make_idesc(128, 128, false, false);
      const uint32_t a = smem_u32(ab), b = smem_u32(ab + 16384);
      for (int it = 0; it < iters / 2; ++it) {
        for (int kk = 0; kk < 4; ++kk)
          umma_bf16(tmem + 256, smem_desc(a + kk * 32, 16, 1024), smem_desc(b + kk * 32, 16, 1024), idesc, 1u);
        umma_commit(&bar);
        mbar_wait(&bar, it & 1);
      }
    }
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) { out[0] = t1 - t0; }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc_warp(tmem, 512); }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64);
  const int iters = 4096;
  for (int w : {4, 8, 16}) for (int mma : {0, 1}) {
    k<<<148, (w + 1) * 32>>>(iters, mma, d);
    cudaDeviceSynchronize();
    k<<<148, (w + 1) * 32>>>(iters, mma, d);
    unsigned long long h[3];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    const double bytes = (double)w * iters * 32 * 32 * 4;
    printf("warps %2d mma %d: %llu cycles, %.1f B/clk/SM tcgen05.ld (%s)\n", w, mma, h[0], bytes / h[0],
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
