// C-ABI entry points for the device side of librdkv.
#include <cuda_runtime.h>
#include <cmath>
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

#include "attention.cuh"

extern "C" int rdkv_attention(const void* q, int64_t ldq, void* o, int64_t ldo, const void* kplane,
                              const void* vplane, int64_t kv_slots, const int32_t* seq_start,
                              const int32_t* seq_new, const int32_t* seq_cached, const int32_t* block_table,
                              int bt_stride, int block_size, int n_seqs, int n_tokens, int max_new, int max_ctx,
                              int n_heads, int kv_heads, int head_dim, int impl, void* scratch,
                              size_t scratch_bytes, void* stream) {
  if (!q || !o || !kplane || !vplane || n_seqs <= 0 || n_tokens <= 0 || kv_heads <= 0 || n_heads % kv_heads)
    return set_error(RDKV_ERR_ARG, "rdkv_attention: bad arguments");
  AttnParams ap{};
  ap.q = static_cast<const __nv_bfloat16*>(q);
  ap.ldq = ldq;
  ap.o = static_cast<__nv_bfloat16*>(o);
  ap.ldo = ldo;
  ap.kplane = static_cast<const __nv_bfloat16*>(kplane);
  ap.vplane = static_cast<const __nv_bfloat16*>(vplane);
  ap.head_stride = kv_slots * head_dim;
  ap.seq_start = seq_start;
  ap.seq_new = seq_new;
  ap.seq_cached = seq_cached;
  ap.block_table = block_table;
  ap.bt_stride = bt_stride;
  ap.block_size = block_size;
  ap.hq = n_heads;
  ap.hkv = kv_heads;
  ap.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)head_dim));
  ap.contiguous = bt_stride == 1 ? 1 : 0;
  ap.kv_splits = 1;
  ap.n_tokens = n_tokens;
  ap.max_ctx = max_ctx;
  const size_t need = attention_split_scratch_bytes(n_tokens, n_heads, head_dim);
  if (scratch && need && scratch_bytes >= need) {
    ap.split_o = static_cast<float*>(scratch);
    ap.split_ml = reinterpret_cast<float2*>(static_cast<uint8_t*>(scratch) + (size_t)attention_split_cap(n_tokens) * n_tokens * n_heads * head_dim * 4);
    ap.split_bytes = need;
  }
  auto st = static_cast<cudaStream_t>(stream);
  const size_t sk = attention_sk_scratch_bytes(num_sms(), head_dim);
  if (scratch && scratch_bytes >= need + sk) {
    attention_sk_carve(ap, static_cast<uint8_t*>(scratch) + need, num_sms(), head_dim);
    RDKV_TRY(attention_sk_zero_flags(ap, st));
  }
  if (impl == 2) {  // tcgen05 kernel, stream-K schedule where it applies
    ap.sk_mode = 1;
    impl = 0;
  }
  if (impl == 0) {
    if (!attention_tc_supported(ap, head_dim))
      return set_error(RDKV_ERR_ARG, "rdkv_attention: shape not supported by the tcgen05 kernel");
    return launch_attention_tc(ap, head_dim, n_seqs, max_new, st);
  }
  return launch_attention(ap, head_dim, n_seqs, max_new, st);
}

extern "C" size_t rdkv_attention_scratch_bytes(int n_tokens, int n_heads, int head_dim) {
  return attention_split_scratch_bytes(n_tokens, n_heads, head_dim) + attention_sk_scratch_bytes(num_sms(), head_dim);
}
