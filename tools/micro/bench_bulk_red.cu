// Micro-benchmark (dev tool): throughput of fp32 reductions into L2-resident global memory, the
// dQ accumulation pattern of a fused attention backward (each CTA adds a [64 x HD] fp32 tile
// per step into a per-(head, batch) accumulator shared by the head's key-block CTAs).
//   mode 0: cp.reduce.async.bulk .add.f32 of the whole tile from smem (one thread issues)
//   mode 1: red.global.add.f32 per element (coalesced, lanes = consecutive floats)
//   mode 2: red.global.add.v4.f32 per 4 elements
//   mode 3: plain st.global of the tile (bandwidth reference)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bench_bulk_red bench_bulk_red.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int HD = 96, QT = 64, TILE = HD * QT;  // floats per tile
constexpr int NKB = 16, NQT = 32;               // key blocks per head, query tiles per head

template <int MODE>
__global__ void __launch_bounds__(256) red_k(float* __restrict__ acc, int nhb, int steps) {
  __shared__ __align__(128) float st[TILE];
  for (int i = threadIdx.x; i < TILE; i += blockDim.x) st[i] = 1.0f + (i & 7) * 0.125f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  // CTA c = (head-batch hb, key block j); step = query tile (staggered start per key block)
  for (int c = blockIdx.x; c < nhb * NKB; c += gridDim.x) {
    const int hb = c / NKB, j = c % NKB;
    for (int it = 0; it < steps; ++it) {
      const int qt = (it + 2 * j) % NQT;
      float* dst = acc + ((int64_t)hb * NQT + qt) * TILE;
      if constexpr (MODE == 0) {
        if (threadIdx.x == 0) {
          asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;"
                       ::"l"(dst), "r"((uint32_t)__cvta_generic_to_shared(st)), "r"(TILE * 4) : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        }
        __syncthreads();
      } else if constexpr (MODE == 1) {
        for (int i = threadIdx.x; i < TILE; i += blockDim.x)
          asm volatile("red.global.add.f32 [%0], %1;" ::"l"(dst + i), "f"(st[i]) : "memory");
      } else if constexpr (MODE == 2) {
        for (int i = threadIdx.x * 4; i < TILE; i += blockDim.x * 4)
          asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(dst + i), "f"(st[i]),
                       "f"(st[i + 1]), "f"(st[i + 2]), "f"(st[i + 3]) : "memory");
      } else {
        for (int i = threadIdx.x * 4; i < TILE; i += blockDim.x * 4)
          *reinterpret_cast<float4*>(dst + i) = *reinterpret_cast<const float4*>(st + i);
      }
    }
  }
  if constexpr (MODE == 0) {
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

template <int MODE>
double run(float* acc, int nhb, int steps, int grid) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  red_k<MODE><<<grid, 256>>>(acc, nhb, steps);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) red_k<MODE><<<grid, 256>>>(acc, nhb, steps);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double bytes = 5.0 * nhb * NKB * (double)steps * TILE * 4;
  return bytes / (ms * 1e-3) / 1e9;
}

int main() {
  const int nhb = 256;  // 22B: 64 heads x 4 batch
  const size_t n = (size_t)nhb * NQT * TILE;
  float* acc;
  cudaMalloc(&acc, n * 4);
  cudaMemset(acc, 0, n * 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int grid : {sms, 2 * sms, 4 * sms}) {
    printf("grid %d: bulk-red %.0f GB/s | red.f32 %.0f GB/s | red.v4.f32 %.0f GB/s | store %.0f GB/s\n",
           grid, run<0>(acc, nhb, NQT, grid), run<1>(acc, nhb, NQT, grid), run<2>(acc, nhb, NQT, grid),
           run<3>(acc, nhb, NQT, grid));
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
