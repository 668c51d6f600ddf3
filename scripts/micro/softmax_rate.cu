// Microbenchmark: the attention softmax instruction stream alone (no TMEM, no MMA, no
// barriers), i.e. the per-tile work of one softmax thread over KH scores held in
// registers: row max (FMNMX3), P = 2^(s*scale - m) (FFMA2 + MUFU.EX2 / degree-2
// polynomial on the FMA pipe), fp32 row sum (FADD2), bf16 packing (F2FP).
// Reports cycles per tile per warp with W softmax warps per SM (W/4 per SMSP).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2504_11765_b200/csrc scripts/micro/softmax_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "ptx.cuh"

using namespace rdkv;

// FLAGS: 1 max, 2 row sum, 4 pack, 8 exp
template <int KH, int EMU, int FLAGS, int NT>
__global__ void __launch_bounds__(NT, 1) k(uint32_t* out, int iters, long long* cyc) {
  float sv[KH];
#pragma unroll
  for (int e = 0; e < KH; ++e) sv[e] = -0.01f * ((threadIdx.x * 7 + e * 13) & 255);
  const float sl2 = 0.18f;
  float m_used = 0.5f;
  uint32_t sink = 0;
  float lsum = 0.f;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
    if (FLAGS & 1) {
#pragma unroll
      for (int e = 0; e < KH; e += 8)
#pragma unroll
        for (int q = 0; q < 4; ++q) mx4[q] = fmax3(mx4[q], sv[e + 2 * q], sv[e + 2 * q + 1]);
      const float mt = fmax3(fmaxf(mx4[0], mx4[1]), mx4[2], mx4[3]) * sl2;
      if (__any_sync(0xffffffffu, mt > m_used + 8.f)) m_used = mt;
    }
    const float nb = -m_used - 1e-7f * it;
    float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
    uint32_t pk[KH / 2];
#pragma unroll
    for (int e = 0; e < KH; e += 4) {
      float x0, x1, x2, x3;
      ffma2(x0, x1, sv[e], sv[e + 1], sl2, sl2, nb, nb);
      ffma2(x2, x3, sv[e + 2], sv[e + 3], sl2, sl2, nb, nb);
      if (FLAGS & 8) {
        if (((e / 4) * 3) % 8 < EMU) {
          exp2_emu2(x0, x1, x0, x1);
          exp2_emu2(x2, x3, x2, x3);
        } else {
          x0 = ex2_approx(x0);
          x1 = ex2_approx(x1);
          x2 = ex2_approx(x2);
          x3 = ex2_approx(x3);
        }
      }
      if (FLAGS & 2) {
        fadd2(s0, s1, s0, s1, x0, x1);
        fadd2(s2, s3, s2, s3, x2, x3);
      }
      if (FLAGS & 4) {
        pk[e / 2] = pack_bf16(x0, x1);
        pk[e / 2 + 1] = pack_bf16(x2, x3);
      } else {
        pk[e / 2] = __float_as_uint(x0) ^ __float_as_uint(x1);
        pk[e / 2 + 1] = __float_as_uint(x2) ^ __float_as_uint(x3);
      }
    }
    lsum += (s0 + s1) + (s2 + s3);
    uint32_t x = 0;
#pragma unroll
    for (int e = 0; e < KH / 2; ++e) x ^= pk[e];
    sink ^= x;
  }
  const long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = sink ^ __float_as_uint(lsum);
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int KH, int EMU, int FLAGS>
void run(const char* name, int warps, uint32_t* out, long long* cyc) {
  const int iters = 2000;
  if (warps == 8) k<KH, EMU, FLAGS, 256><<<148, 256>>>(out, iters, cyc);
  else k<KH, EMU, FLAGS, 512><<<148, 512>>>(out, iters, cyc);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  const double per = avg / iters;  // cycles per tile (every warp did one tile)
  printf("KH=%3d emu=%d/8 flags=%2d %-28s warps/SM=%2d: %7.1f cyc/tile  (%.2f cyc per score per SMSP) %s\n", KH, EMU,
         FLAGS, name, warps, per, per / (KH * warps / 4.0), cudaGetErrorString(cudaGetLastError()));
}

int main() {
  uint32_t* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 512 * 4);
  cudaMalloc(&cyc, 148 * 8);
  {
    const int w = 8;  // two softmax warps per SMSP, as in the kernel
    run<128, 3, 15>("full (max+exp+sum+pack)", w, out, cyc);
    run<128, 3, 14>("no max", w, out, cyc);
    run<128, 3, 13>("no sum", w, out, cyc);
    run<128, 3, 11>("no pack", w, out, cyc);
    run<128, 3, 7>("no exp (max+scale+sum+pack)", w, out, cyc);
    run<128, 0, 15>("full, all MUFU", w, out, cyc);
    run<128, 2, 15>("full, 2/8 poly", w, out, cyc);
    run<128, 4, 15>("full, 4/8 poly", w, out, cyc);
    run<128, 5, 15>("full, 5/8 poly", w, out, cyc);
    run<128, 8, 15>("full, all poly", w, out, cyc);
    run<64, 3, 15>("dh128 tile: full", w, out, cyc);
    run<64, 0, 15>("dh128 tile: all MUFU", w, out, cyc);
    run<64, 2, 15>("dh128 tile: 2/8 poly", w, out, cyc);
    run<64, 4, 15>("dh128 tile: 4/8 poly", w, out, cyc);
    run<64, 3, 13>("dh128 tile: no sum", w, out, cyc);
    run<64, 3, 14>("dh128 tile: no max", w, out, cyc);
  }
  run<64, 3, 15>("KH 64 x 16 warps: full", 16, out, cyc);
  run<64, 4, 15>("KH 64 x 16 warps: 4/8 poly", 16, out, cyc);
  return 0;
}
