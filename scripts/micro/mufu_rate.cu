// Microbenchmark: MUFU ex2 throughput, fp32 vs packed bf16x2 / f16x2 (results per clock per SM).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(512) k(uint32_t* out, int iters, long long* cyc) {
  uint32_t v[8];
  for (int i = 0; i < 8; ++i) v[i] = 0x3c003c00u ^ (threadIdx.x * 7 + i);
  float f[8];
  for (int i = 0; i < 8; ++i) f[i] = -0.001f * (threadIdx.x + i);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(f[i]));
      if (MODE == 1) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(v[i]));
      if (MODE == 2) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(v[i]));
    }
  }
  long long t1 = clock64();
  uint32_t acc = 0;
  for (int i = 0; i < 8; ++i) acc ^= v[i] ^ __float_as_uint(f[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  uint32_t* out; long long* cyc;
  cudaMalloc(&out, 148 * 512 * 4); cudaMalloc(&cyc, 148 * 8);
  const int iters = 4096;
  const char* names[3] = {"f32", "bf16x2", "f16x2"};
  for (int m = 0; m < 3; ++m) {
    if (m == 0) k<0><<<148, 512>>>(out, iters, cyc);
    if (m == 1) k<1><<<148, 512>>>(out, iters, cyc);
    if (m == 2) k<2><<<148, 512>>>(out, iters, cyc);
    cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    double instr = 512.0 * iters * 8;  // per SM (thread-instructions)
    double results = instr * (m == 0 ? 1 : 2);
    printf("%-7s %.1f results/clk/SM (%.1f instr/clk/SM) %s\n", names[m], results / h, instr / h, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
