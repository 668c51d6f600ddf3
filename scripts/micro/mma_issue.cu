// Microbenchmark: tcgen05.mma issue cost with several issuing warps and with warp-uniform
// issue.  NI warps each issue iters x 8 MMAs (kind::f16, M = 128, K = 16, N, both operands in
// smem) into their own accumulator columns; aggregate cycles per MMA over all issuers.
//   UNI = 0: the issuing thread runs alone inside `if (lane == 0)` (descriptors in per-thread
//            registers: every UTCHMMA sits in an ELECT / R2UR.BROADCAST / BRA.U.ANY loop)
//   UNI = 1: the whole warp runs the loop with warp-uniform operands and elects one lane for the
//            instruction itself (descriptors can live in uniform registers)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o scripts/micro/mma_issue scripts/micro/mma_issue.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2504_11765_b200/csrc/ptx.cuh"
using namespace rdkv;

template <int N, int NI, int UNI>
__global__ void __launch_bounds__(32 * (NI + 1), 1) mma_issue(int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar[NI];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < (128 + 256) * 128 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  fence_proxy_async_smem();
  if (warp == NI) tmem_alloc(&slot, 512);
  if (threadIdx.x == 0) {
    for (int i = 0; i < NI; ++i) mbar_init(&bar[i], 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp < NI) {
    const uint32_t a = smem_u32(smem), b = a + 128 * 128;
    constexpr uint32_t idesc = idesc_bf16_f32(128, N);
    const uint32_t d = slot + warp * N;
    long long t0 = clock64();
    if (UNI) {
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t da = sdesc_k_sw128(a + (kk & 3) * 32), db = sdesc_k_sw128(b + (kk & 3) * 32);
          if (elect_one()) umma_bf16(d, da, db, idesc, 1u);
          __syncwarp();
        }
      }
      if (elect_one()) umma_commit(&bar[warp]);
      __syncwarp();
    } else if (lane == 0) {
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_bf16(d, sdesc_k_sw128(a + (kk & 3) * 32), sdesc_k_sw128(b + (kk & 3) * 32), idesc, 1u);
      }
      umma_commit(&bar[warp]);
    }
    mbar_wait(&bar[warp], 0);
    long long t1 = clock64();
    if (lane == 0) out[blockIdx.x * NI + warp] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == NI) {
    tc_fence_after();
    tmem_dealloc(slot, 512);
  }
}

template <int N, int NI, int UNI>
void run(int iters) {
  long long* out;
  cudaMalloc(&out, 148 * NI * 8);
  const int smem = (128 + 256) * 128 + 1024;
  cudaFuncSetAttribute(mma_issue<N, NI, UNI>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  mma_issue<N, NI, UNI><<<148, 32 * (NI + 1), smem>>>(iters, out);
  cudaDeviceSynchronize();
  long long h[148 * 4];
  cudaMemcpy(h, out, 148 * NI * 8, cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < NI; ++i) mx = h[i] > mx ? h[i] : mx;
  const double n = 8.0 * iters * NI;
  printf("N=%3d issuers=%d %s: %.1f cyc per MMA aggregate (%.1f per issuer-MMA) err=%s\n", N, NI,
         UNI ? "warp-uniform+elect" : "lane-0 branch     ", mx / n, mx / (8.0 * iters),
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}

int main() {
  run<64, 1, 0>(2000);
  run<64, 1, 1>(2000);
  run<64, 2, 0>(2000);
  run<64, 2, 1>(2000);
  run<64, 4, 0>(2000);
  run<64, 4, 1>(2000);
  run<128, 1, 0>(2000);
  run<128, 1, 1>(2000);
  run<128, 2, 0>(2000);
  run<128, 2, 1>(2000);
  return 0;
}
