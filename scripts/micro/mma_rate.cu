// Microbenchmark: tcgen05.mma (kind::f16, cta_group::1, M = 128, K = 16) issue and
// completion cost per instruction for N = 64 / 128 / 256, A from smem (SS) or from
// TMEM (TS, the attention P.V form), one issuing thread per SM, 148 CTAs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/mma_rate scripts/micro/mma_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2504_11765_b200/csrc/ptx.cuh"
using namespace rdkv;

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) mma_rate(int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (128 + 256) * 128 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  fence_proxy_async_smem();
  if (warp == 0) tmem_alloc(&slot, 512);
  if (threadIdx.x == 32) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(smem), b = a + 128 * 128;
    constexpr uint32_t idesc = idesc_bf16_f32(128, N) | (TS ? (1u << 16) : 0u);
    const uint32_t d = slot + 256;  // accumulator columns [256, 256 + N)
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        if constexpr (TS)
          umma_bf16_ts(d, slot + kk * 8, sdesc_k_sw128(b + (kk & 3) * 32), idesc, 1u);
        else
          umma_bf16(d, sdesc_k_sw128(a + (kk & 3) * 32), sdesc_k_sw128(b + (kk & 3) * 32), idesc, 1u);
      }
    }
    long long t1 = clock64();
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t2 = clock64();
    out[blockIdx.x * 2] = t1 - t0;
    out[blockIdx.x * 2 + 1] = t2 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(slot, 512);
  }
}

template <int N, bool TS>
void run(int iters) {
  long long* out;
  cudaMalloc(&out, 148 * 16);
  const int smem = (128 + 256) * 128 + 1024;
  cudaFuncSetAttribute(mma_rate<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  mma_rate<N, TS><<<148, 128, smem>>>(iters, out);
  cudaDeviceSynchronize();
  long long h[296];
  cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
  const double n = 8.0 * iters;
  const double ideal = 2.0 * 128 * N * 16 / 8192.0;
  printf("N=%3d %s: issue %.1f cyc/MMA, complete %.1f cyc/MMA (ideal %.0f at 8192 FLOP/clk) err=%s\n", N,
         TS ? "TS" : "SS", h[0] / n, h[1] / n, ideal, cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}

int main() {
  run<64, false>(2000);
  run<128, false>(2000);
  run<256, false>(2000);
  run<64, true>(2000);
  run<128, true>(2000);
  run<256, true>(2000);
  return 0;
}
