// Micro-benchmark (dev tool): TMEM read throughput per SM (tcgen05.ld.32x32b.x32 + wait::ld)
// with 4 / 8 / 16 warps per CTA, one CTA per SM; and the same loads interleaved with a fixed
// amount of FP work per loaded column (does the load overlap other warps' math?).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bench_tmem_ld bench_tmem_ld.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void ld32(uint32_t taddr, uint32_t (&r)[32]) {
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

template <int MATH>
__global__ void tmem_k(int iters, float* out, unsigned long long* cyc) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot + ((uint32_t)((warp & 3) * 32) << 16);
  float acc = 0.f;
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    uint32_t a[32], b[32];
    const uint32_t col = (uint32_t)(((i * 2 + (warp >> 2)) & 7) * 64);
    ld32(tmem + col, a);
    ld32(tmem + col + 32, b);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      float x = __uint_as_float(a[j]) + __uint_as_float(b[j]);
#pragma unroll
      for (int m = 0; m < MATH; ++m) x = fmaf(x, 1.0001f, 0.5f);
      acc += x;
    }
  }
  const long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = (unsigned long long)(t1 - t0);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

template <int MATH>
void run(int warps, int sms, float* out, unsigned long long* cyc) {
  const int iters = 2000;
  tmem_k<MATH><<<sms, warps * 32>>>(iters, out, cyc);
  cudaDeviceSynchronize();
  unsigned long long h[256];
  cudaMemcpy(h, cyc, sms * 8, cudaMemcpyDeviceToHost);
  double c = 0;
  for (int i = 0; i < sms; ++i) c += h[i];
  c /= sms;
  const double bytes = (double)iters * warps * 2 * 32 * 32 * 4;  // per CTA
  printf("math %2d warps %2d: %.1f B/clk/SM TMEM read, %.0f cycles per warp-iteration\n", MATH,
         warps, bytes / c, c / iters);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  unsigned long long* cyc;
  cudaMalloc(&out, sms * 1024 * 4);
  cudaMalloc(&cyc, sms * 8);
  for (int w : {4, 8, 16}) run<0>(w, sms, out, cyc);
  for (int w : {4, 8, 16}) run<4>(w, sms, out, cyc);
  for (int w : {4, 8, 16}) run<12>(w, sms, out, cyc);
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
