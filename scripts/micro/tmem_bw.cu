// Microbenchmark: TMEM read bandwidth (tcgen05.ld 32x32b.x32) per SM, W warps.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2504_11765_b200/csrc/ptx.cuh"
using namespace rdkv;

template <int W>
__global__ void __launch_bounds__(W * 32, 1) tmem_read(uint32_t* out, int iters, long long* cyc) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = slot + ((uint32_t)((warp & 3) * 32) << 16) + ((warp >> 2) & 3) * 128;
  uint32_t acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t v[4][32];
#pragma unroll
    for (int c = 0; c < 4; ++c) tmem_ld32(tm + c * 32, v[c]);
    tmem_ld_wait();
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int i = 0; i < 32; ++i) acc ^= v[c][i];
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(slot, 512); }
}

template <int W>
void run(int iters) {
  uint32_t* out; long long* cyc;
  cudaMalloc(&out, 148 * W * 32 * 4); cudaMalloc(&cyc, 148 * 8);
  tmem_read<W><<<148, W * 32>>>(out, iters, cyc);
  cudaDeviceSynchronize();
  long long h[148]; cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double bytes = (double)W * 32 * 4 * 32 * 4 * iters;  // per SM
  printf("warps %2d: %.1f B/cycle/SM (%lld cycles) err=%s\n", W, bytes / h[0], h[0], cudaGetErrorString(cudaGetLastError()));
  cudaFree(out); cudaFree(cyc);
}

int main() {
  run<4>(1000); run<8>(1000); run<12>(1000);
  return 0;
}
