// C-ABI entry points for the device side of librdkv.
#include <cuda_runtime.h>
#include <cstdlib>

#include "common.cuh"
#include "gemm_tc.cuh"

namespace rdkv {

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("RDKV_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

int num_sms() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!cached[dev]) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = n > 0 ? n : 148;
  }
  return cached[dev];
}

}  // namespace rdkv

using namespace rdkv;

extern "C" int rdkv_gemm_bf16(const void* A, int64_t lda, const void* B, int64_t ldb, void* D, int64_t ldd,
                              const void* R, int64_t ldr, int M, int N, int K, int epilogue, void* stream) {
  return rdkv_gemm_bf16_ex(A, lda, B, ldb, D, ldd, R, ldr, M, N, K, epilogue, 0, nullptr, 0, stream);
}

extern "C" int rdkv_gemm_bf16_ex(const void* A, int64_t lda, const void* B, int64_t ldb, void* D, int64_t ldd,
                                 const void* R, int64_t ldr, int M, int N, int K, int epilogue, int tile_n,
                                 void* scratch, size_t scratch_bytes, void* stream) {
  if (epilogue < RDKV_EPI_STORE || epilogue > RDKV_EPI_SWIGLU)
    return set_error(RDKV_ERR_ARG, "rdkv_gemm_bf16: epilogue %d not exposed", epilogue);
  GemmEpi ep{};
  ep.out = D;
  ep.ldo = ldd;
  ep.resid = static_cast<const __nv_bfloat16*>(epilogue == RDKV_EPI_RESID ? (R ? R : D) : nullptr);
  ep.ldr = R ? ldr : ldd;
  ep.splitk_ws = scratch;
  ep.splitk_bytes = scratch ? scratch_bytes : 0;
  return launch_gemm(static_cast<const __nv_bfloat16*>(A), lda, static_cast<const __nv_bfloat16*>(B), ldb, M, N,
                     K, epilogue, 0, ep, static_cast<cudaStream_t>(stream), tile_n);
}
