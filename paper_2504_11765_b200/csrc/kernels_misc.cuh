#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include "../../include/rdkv.h"

namespace rdkv {

using UnpackJob = rdkv_unpack_job;

__device__ __forceinline__ uint32_t pack_bf16_f(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ float2 unpack_bf16_f(uint32_t u) {
  __nv_bfloat162 v = *reinterpret_cast<__nv_bfloat162*>(&u);
  return __bfloat1622float2(v);
}

int launch_kv_unpack(const UnpackJob* jobs_dev, int n_jobs, int max_tokens, const int* bt, int block_size,
                     void* pool, int layer_begin, int layer_end, int hkv, int dh, long long slots, int elem_width,
                     cudaStream_t st, int head_begin = 0, int src_kv_heads = 0);
int launch_embed(const int* tok, const __nv_bfloat16* table, __nv_bfloat16* out, int n, int d, int vocab,
                 cudaStream_t st, float* ssq = nullptr);
int launch_rmsnorm(const __nv_bfloat16* x, long long ldx, const int* rows, const float* gain, __nv_bfloat16* out,
                   long long ldo, int n_rows, int d, float eps, cudaStream_t st);
size_t argmax_scratch_bytes(int rows);
int launch_argmax(const float* logits, long long ld, int rows, int n, int* out, void* scratch, cudaStream_t st);

}  // namespace rdkv
