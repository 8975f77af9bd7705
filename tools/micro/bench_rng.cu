// Micro-benchmark (dev tool): keep-bit RNG throughput vs warps per SM and registers (ILP).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2205_05198_b200/csrc tools/micro/bench_rng.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "rng_fast.cuh"
using namespace spl::rngk;

template <int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) kb(uint64_t mixed, uint64_t tsh, int nrows, int W, int s,
                                              uint32_t* bits, ShiftMuls sm) {
  const uint32_t mixed_lo = (uint32_t)mixed, mixed_hi = (uint32_t)(mixed >> 32);
  const uint32_t t_lo = (uint32_t)tsh, t_hi = (uint32_t)(tsh >> 32);
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < nrows; row += warps) {
    const uint64_t base = (uint64_t)row * s + kC + kG;
    for (int w = lane; w < W; w += 32) {
      const uint64_t bw = base + 32u * w;
      const uint32_t blo = (uint32_t)bw, bhi = (uint32_t)(bw >> 32);
      uint32_t word = 0;
      if (blo <= 0xffffffffu - 31u) {
        const uint32_t hx = bhi ^ (bhi >> 30);
        const uint32_t hc = hx * 0x1ce4e5b9u;
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (keep_fast(blo + j, bhi, hc, hx, mixed_lo, mixed_hi, t_lo, t_hi, sm)) word |= 1u << j;
      }
      bits[(int64_t)row * W + w] = word;
    }
  }
}

template <int NT, int MINB>
void run(const char* name, int ctas_per_sm, uint32_t* bits, int nrows, int W, int s) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  ShiftMuls sm{4u, 32u, 2u, 1u};
  int grid = 148 * ctas_per_sm;
  kb<NT, MINB><<<grid, NT>>>(0x1234567890abcdefULL, 0x0CCCCCCCCCCCCC00ULL, nrows, W, s, bits, sm);
  cudaEventRecord(a);
  for (int i = 0; i < 5; ++i)
    kb<NT, MINB><<<grid, NT>>>(0x1234567890abcdefULL, 0x0CCCCCCCCCCCCC00ULL, nrows, W, s, bits, sm);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  ms /= 5;
  cudaFuncAttributes at;
  cudaFuncGetAttributes(&at, kb<NT, MINB>);
  printf("%-28s warps/SM=%3d regs=%3d  %.3f ms  %.3g hashes/s\n", name, ctas_per_sm * NT / 32,
         at.numRegs, ms, (double)nrows * s / (ms * 1e-3));
}

int main() {
  const int s = 2048, nrows = 64 * 4 * 2048, W = s / 32;
  uint32_t* bits;
  cudaMalloc(&bits, (size_t)nrows * W * 4);
  run<256, 8>("256thr x8 (current)", 8, bits, nrows, W, s);
  run<256, 8>("256thr x4", 4, bits, nrows, W, s);
  run<256, 8>("256thr x2", 2, bits, nrows, W, s);
  run<256, 8>("256thr x1", 1, bits, nrows, W, s);
  run<256, 2>("256thr x1 (128 regs)", 1, bits, nrows, W, s);
  run<256, 2>("256thr x2 (128 regs)", 2, bits, nrows, W, s);
  run<128, 1>("128thr x1 (255 regs)", 1, bits, nrows, W, s);
  run<128, 4>("128thr x4 (128 regs)", 4, bits, nrows, W, s);
  run<512, 1>("512thr x1 (128 regs)", 1, bits, nrows, W, s);
  run<512, 2>("512thr x2 (64 regs)", 2, bits, nrows, W, s);
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
