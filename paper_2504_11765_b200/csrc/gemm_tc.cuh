// K1: persistent, warp-specialised tcgen05 GEMM for sm_100a.
//
//   D[M, N] = A[M, K] . B[N, K]^T      A, B bf16 K-major, fp32 accumulate in TMEM
//
// Roles (256 threads): warp 0 = TMA producer, warp 1 = MMA issuer (one thread),
// warp 2 = TMEM allocator, warps 4..7 = epilogue (one TMEM lane = one output row
// per thread).  Operand tiles are staged by TMA with 128-byte swizzle into a
// STAGES-deep smem ring guarded by full/empty mbarriers; the fp32 accumulator
// is double-buffered in TMEM so the epilogue of tile i overlaps the MMAs of
// tile i+1.  Fused epilogues replace the separate elementwise passes of a
// plain transformer layer:
//   STORE      bf16 D
//   STORE_F32  fp32 D (LM-head logits)
//   RESID      D = R + A.B^T (residual add; R may alias D)
//   SWIGLU     weights interleaved in BN/2 blocks [gate | up]; D = silu(g) * u
//   QKV        RoPE on q/k heads, q -> token-major buffer, k/v -> head-major
//              KV planes at per-row slots (document blob layout or paged pool)
//   PUSH       bf16 D stored into every TP rank's receive slot (NVLink P2P
//              stores): the GEMM and the all-reduce's data movement are one kernel
#pragma once
#include <cuda_runtime.h>
#include "ptx.cuh"

namespace rdkv {

enum EpiKind : int { EPI_STORE = 0, EPI_STORE_F32 = 1, EPI_RESID = 2, EPI_SWIGLU = 3, EPI_QKV = 4, EPI_PARTIAL = 5, EPI_PUSH = 6 };

struct GemmEpi {
  void* out;                 // bf16 (or fp32 for STORE_F32)
  long long ldo;             // elements
  const __nv_bfloat16* resid;
  long long ldr;
  // QKV
  __nv_bfloat16* q;
  long long ldq;
  __nv_bfloat16* kplane;     // K plane of this layer: [Hkv][slots][dh]
  __nv_bfloat16* vplane;     // V plane of this layer
  long long head_stride;     // elements between consecutive kv heads in a plane
  const int* slot;           // per row: slot index inside the head plane
  const int* pos;            // per row: RoPE position
  const float* rope;         // [max_pos][dh/2] x (cos, sin)
  int hq, hkv;
  // split-K scratch (fp32 slabs); null disables split-K
  void* splitk_ws;
  size_t splitk_bytes;
  // optional RMSNorm fused into the split-K RESID finalize: norm_out = rmsnorm(out) * norm_gain
  const float* norm_gain;
  __nv_bfloat16* norm_out;
  float norm_eps;
  // PUSH (tensor-parallel row-parallel projections): the bf16 tile is stored into
  // every rank's receive slot for this rank (dense [M][ldo]); peers' slots are
  // CUDA-IPC mappings, so the stores cross NVLink while later tiles still compute
  __nv_bfloat16* push[8];
  int npush;
  // RMSNorm fused across GEMMs (RDKV_MODEL_NORM_FOLDED: the norm gains are folded into
  // the consuming weights).  RESID writes, per output row and 32-column chunk, the
  // sum of squares of its bf16 outputs to ssq_out[chunk][M]; QKV / SWIGLU read the
  // ssq_parts partials of their A rows in a fixed order and scale the accumulators
  // by rsqrt(sum / ssq_dim + norm_eps) before RoPE / SiLU.  Null = off.
  float* ssq_out;
  const float* ssq_in;
  int ssq_parts;
  int ssq_dim;
  // L2 prefetch of the NEXT kernel's weights (126 MB of L2: the following projection's
  // weights are pulled in by this kernel's idle warp while its own tiles compute, so a
  // single-wave GEMM does not start on a cold weight stream).  Null = off; launch_gemm
  // clears it unless RDKV_L2_PREFETCH=1 (measured no faster in the C3 step).
  const void* l2_next;
  long long l2_next_bytes;
  // L2 policy of the weight (B) loads: 0 evict-last (like the activations), 1 evict-first
  // (a weight tile is read by the M tiles of one wave at the same time, then never again
  // in this kernel: streaming it evict-first keeps the prefetched next weights resident).
  // Set by launch_gemm (RDKV_GEMM_WPOL, default 0).
  int w_policy;
  // L2 prefetch of this GEMM's own weight (B) tiles b_pf k-blocks ahead of the TMA loads
  // (cp.async.bulk.prefetch.tensor, duty spread over the M tiles sharing a B tile): the
  // smem ring holds only a few k-blocks, too little to cover DRAM latency when a
  // single-wave GEMM streams its weights cold.  0 = off.  Set by launch_gemm (RDKV_GEMM_PF).
  int b_pf;
  // Small-M fused split-K (swap-AB GEMM, no finalize kernel): one ticket counter per 128-column
  // weight tile, zero before the launch and left zero by it (the last split resets it).
  // Null = the split-K partials go through a separate finalize kernel.
  int* counters;
  int n_counters;
  // Large-M stream-K (CTA-pair GEMM): fp32 partial tiles [2 per pair][128 rows][tile N]
  // and one release flag per slot, zero before the launch and left zero by it (the pair
  // holding a split tile's first k-block adds the later pairs' partials).  Null = off.
  float* sk_part;
  int* sk_flag;
  int sk_slots;
  // Which units the stream-K launch splits: the first sk_dp tiles run whole, round-robin
  // over the pairs; the k-blocks of the rest are shared equally by the first sk_tp pairs
  // (pure stream-K: sk_dp = 0, sk_tp = every pair; the DP + split-tail hybrid: sk_dp =
  // the full rounds, sk_tp = tail tiles x split).  Set by the launcher.
  int sk_dp;
  int sk_tp;
};

// Bytes of stream-K scratch (partials + flags) for the CTA-pair GEMM on this GPU, and the
// RDKV_GEMM_SK mode (0 off, 1 grids leaving pairs idle, 2 any partial last round,
// 3 whole tiles for the full rounds + the partial last round's tiles split in k).
size_t gemm_sk_scratch_bytes();
int gemm_sk_mode();

// True when launch_gemm will take the split-K path for this shape (small M).
bool gemm_splits(int M, int N, int K, size_t splitk_bytes);

// Scratch bytes split-K would use for this GEMM shape (0 if it would not split).
size_t splitk_scratch_bytes(int M, int N, int K);

// bn = tile N (128 or 256), 0 = choose by wave quantisation
int launch_gemm(const __nv_bfloat16* A, long long lda, const __nv_bfloat16* B, long long ldb, int M,
                int N, int K, int kind, int dh, const GemmEpi& ep, cudaStream_t stream, int bn = 0);

}  // namespace rdkv
