#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace rdkv {

struct AttnParams {
  const __nv_bfloat16* q;   // [T, hq*dh] token-major (post-RoPE)
  long long ldq;
  __nv_bfloat16* o;         // [T, hq*dh]
  long long ldo;
  const __nv_bfloat16* kplane;  // this layer's K plane [hkv][slots][dh]
  const __nv_bfloat16* vplane;
  long long head_stride;        // slots * dh
  const int* seq_start;         // [S] first row in T
  const int* seq_new;           // [S] new tokens
  const int* seq_cached;        // [S] cached-prefix tokens (positions start here)
  const int* block_table;       // [S][bt_stride]
  int bt_stride;
  int block_size;
  int hq, hkv;
  float scale_log2;             // log2(e) / sqrt(dh)
  int contiguous;               // 1: each sequence's KV is one block (blob layout)
};

// mma.sync kernel (any group size dividing 128, any block size)
int launch_attention(const AttnParams& p, int head_dim, int n_seqs, int max_new, cudaStream_t st);
// tcgen05 kernel (block_size % 64 == 0 or contiguous)
bool attention_tc_supported(const AttnParams& p, int head_dim);
int launch_attention_tc(const AttnParams& p, int head_dim, int n_seqs, int max_new, cudaStream_t st);

}  // namespace rdkv
