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
  // split-KV (tensor-core kernel): scratch for per-split partials, chosen at launch
  int kv_splits;
  int seq_off;                  // first sequence of this launch's split units (grid z = sequences seq_off..)
  int tail_ctas;                // > 0: tail-split grid, CTAs [0, tail_ctas) are whole units of sequences [0, seq_off)
  int n_tokens;                 // T (rows of q / o)
  int max_ctx;                  // max over sequences of n_cached + n_new
  float* split_o;               // [splits][T][hq][dh] fp32
  float2* split_ml;             // [splits][T][hq] (max, sum)
  size_t split_bytes;
  // stream-K (tensor-core kernel, chosen at launch): per-CTA partial of the unit it
  // shares with its predecessor CTA, and the publish flags (zero between launches)
  int n_seqs;
  int sk_qblocks;               // query blocks per sequence (set by the launcher)
  float* sk_o;                  // [ctas][2 Q tiles x 128 rows][dh] fp32
  float2* sk_ml;                // [ctas][256] (max, sum)
  int* sk_flag;                 // [ctas]
  int sk_ctas;                  // CTAs the scratch was sized for (0 = no stream-K)
  int sk_mode;                  // 1: use stream-K where it applies (rdkv_attention impl 2, RDKV_ATTN_SK=1)
  // L2 prefetch of the next kernel's weights (the O projection) by the Q-loader warp;
  // the K/V stream itself is loaded evict-first so it does not push them out.  Null = off.
  const void* l2_next;
  long long l2_next_bytes;
  int kv_evict_first;           // set by the launcher: every K/V tile is read by one CTA only
};

// stream-K scratch: partials + flags for `ctas` CTAs; carve() points p's sk_* into it
size_t attention_sk_scratch_bytes(int ctas, int dh);
void attention_sk_carve(AttnParams& p, void* base, int ctas, int dh);
int attention_sk_zero_flags(const AttnParams& p, cudaStream_t st);

// split-KV scratch: attention_split_cap(T) partial slabs of [T][hq][dh] fp32, then
// as many [T][hq] (max, sum) pairs
inline int attention_split_cap(int T) { return T <= 512 ? 16 : 4; }
size_t attention_split_scratch_bytes(int T, int hq, int dh);

// mma.sync kernel (any group size dividing 128, any block size)
int launch_attention(const AttnParams& p, int head_dim, int n_seqs, int max_new, cudaStream_t st);
// tcgen05 kernel (block_size % 64 == 0 or contiguous)
bool attention_tc_supported(const AttnParams& p, int head_dim);
int launch_attention_tc(const AttnParams& p, int head_dim, int n_seqs, int max_new, cudaStream_t st);

}  // namespace rdkv
