// K2/K4: causal prefill attention over a (possibly cached) KV prefix, GQA.
//
// One kernel serves both document prefill (n_cached = 0, KV in the blob
// layout) and query prefill over cached document KV (new tokens at positions
// [n_cached, n_cached + n_new) attend over every slot of positions <= their
// own, reference semantics of cached_prefill_work, costs.py:89-99).  KV lives
// in head-major planes [Hkv][slots][dh]; logical position p of sequence s sits
// at slot block_table[s][p / bs] * bs + p % bs, so the same code reads a
// contiguous document blob (one block) or a paged pool.
//
// Tiling: a CTA owns 128 query *rows* of ONE kv head, where row r is
// (token t0 + r / G, q-head kvh*G + r % G) and G = hq / hkv.  All G query
// heads that share a K/V head therefore read each K/V tile once (GQA
// packing: 4x less KV traffic than one CTA per q head).  8 warps x 16 rows;
// K/V tiles of 64 positions in a 3-stage cp.async ring with XOR-swizzled
// smem; S = Q.K^T and O += P.V on mma.sync m16n8k16 bf16 (fp32 accumulate)
// with an exp2-domain online softmax.  CTAs are issued longest-first so the
// causal tail does not straggle.
#include <cuda_bf16.h>
#include <cstdint>

#include "attention.cuh"
#include "common.cuh"
#include "pdl.cuh"

namespace rdkv {
namespace {

constexpr int ROWS = 128;  // query rows per CTA
constexpr int BN = 64;     // key positions per tile
constexpr int STAGES = 3;
constexpr int THREADS = 256;

__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool pred) {
  const int n = pred ? 16 : 0;  // src-size 0 => zero fill
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void ldsm_x4(uint32_t a, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(a));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t a, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(a));
}
__device__ __forceinline__ void mma16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

// byte offset of (row, 16-B chunk) inside a [rows][DH] bf16 tile with XOR swizzle
template <int DH>
__device__ __forceinline__ uint32_t swz(int row, int chunk) {
  return (uint32_t)(row * DH * 2 + ((chunk ^ (row & 7)) << 4));
}

template <int DH>
__global__ void __launch_bounds__(THREADS, DH == 64 ? 2 : 1) attn_prefill_kernel(AttnParams p) {
  pdl_trigger();
  pdl_wait();
  constexpr int CH = DH / 8;  // 16-B chunks per row
  constexpr uint32_t TILE = BN * DH * 2;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + ROWS * DH * 2;        // [STAGES][BN][DH]
  uint8_t* sV = sK + STAGES * TILE;        // [STAGES][BN][DH]

  const int G = p.hq / p.hkv;
  const int s = blockIdx.z, kvh = blockIdx.y;
  const int qb = gridDim.x - 1 - blockIdx.x;  // longest causal rows first
  const int n_new = p.seq_new[s];
  const int tok_per_cta = ROWS / G;
  const int tok0 = qb * tok_per_cta;
  if (tok0 >= n_new) return;
  const int ntok = min(tok_per_cta, n_new - tok0);
  const int nrows = ntok * G;
  const int n_cached = p.seq_cached[s];
  const int row_base = p.seq_start[s] + tok0;    // first token row in T
  const int pos0 = n_cached + tok0;              // position of the CTA's first token
  const int kv_len = pos0 + ntok;                // positions [0, kv_len) are needed
  const int n_tiles = (kv_len + BN - 1) / BN;
  const __nv_bfloat16* kp = p.kplane + (long long)kvh * p.head_stride;
  const __nv_bfloat16* vp = p.vplane + (long long)kvh * p.head_stride;
  const int* bt = p.block_table + (long long)s * p.bt_stride;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // ---- Q tile -> smem: row r = (token r/G, head kvh*G + r%G); rows >= nrows zero-filled
  for (int i = tid; i < ROWS * CH; i += THREADS) {
    const int r = i / CH, c = i % CH;
    const bool ok = r < nrows;
    const int rr = ok ? r : 0;
    const __nv_bfloat16* src =
        p.q + (long long)(row_base + rr / G) * p.ldq + (long long)(kvh * G + rr % G) * DH + c * 8;
    cp_async16(saddr(sQ) + swz<DH>(r, c), src, ok);
  }
  auto load_kv = [&](int tile, int buf) {
    for (int i = tid; i < BN * CH; i += THREADS) {
      const int r = i / CH, c = i % CH;
      const int pos = tile * BN + r;
      const bool ok = pos < kv_len;
      long long slot = 0;
      if (ok) slot = (long long)bt[pos / p.block_size] * p.block_size + pos % p.block_size;
      const uint32_t off = (uint32_t)buf * TILE + swz<DH>(r, c);
      cp_async16(saddr(sK) + off, kp + slot * DH + c * 8, ok);
      cp_async16(saddr(sV) + off, vp + slot * DH + c * 8, ok);
    }
  };
  load_kv(0, 0);
  cp_commit();                       // group: Q + tile 0
  if (n_tiles > 1) load_kv(1, 1);
  cp_commit();                       // group: tile 1 (possibly empty)

  // ---- per-warp state: rows g and g+8 of this warp's 16
  const int g = lane >> 2, c4 = lane & 3;
  const int wr = warp * 16;
  const int qpos_a = pos0 + (wr + g) / G;
  const int qpos_b = pos0 + (wr + g + 8) / G;
  const int warp_min_pos = pos0 + wr / G;
  const int warp_max_pos = pos0 + (wr + 15) / G;
  float m_a = -INFINITY, m_b = -INFINITY, l_a = 0.f, l_b = 0.f;
  float o[DH / 8][4];
#pragma unroll
  for (int i = 0; i < DH / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  uint32_t qf[DH / 16][4];

  for (int tile = 0; tile < n_tiles; ++tile) {
    const int buf = tile % STAGES;
    if (tile + 2 < n_tiles) load_kv(tile + 2, (tile + 2) % STAGES);
    cp_commit();
    cp_wait<2>();
    __syncthreads();
    if (tile == 0) {
#pragma unroll
      for (int kk = 0; kk < DH / 16; ++kk) {
        const int r = wr + (lane & 15);
        const int c = kk * 2 + (lane >> 4);
        ldsm_x4(saddr(sQ) + swz<DH>(r, c), qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3]);
      }
    }
    if (tile * BN <= warp_max_pos && wr < nrows) {  // this tile holds keys visible to the warp
      const uint32_t kb = saddr(sK) + buf * TILE;
      const uint32_t vb = saddr(sV) + buf * TILE;
      float sc[BN / 8][4];
#pragma unroll
      for (int j = 0; j < BN / 8; ++j) sc[j][0] = sc[j][1] = sc[j][2] = sc[j][3] = 0.f;
#pragma unroll
      for (int kk = 0; kk < DH / 16; ++kk) {
#pragma unroll
        for (int jj = 0; jj < BN / 16; ++jj) {
          uint32_t b0, b1, b2, b3;
          const int r = jj * 16 + ((lane >> 4) << 3) + (lane & 7);
          const int c = kk * 2 + ((lane >> 3) & 1);
          ldsm_x4(kb + swz<DH>(r, c), b0, b1, b2, b3);
          mma16816(sc[2 * jj], qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3], b0, b1);
          mma16816(sc[2 * jj + 1], qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3], b2, b3);
        }
      }
      const bool need_mask = (tile * BN + BN - 1) > warp_min_pos || (tile * BN + BN) > kv_len;
      float mx_a = m_a, mx_b = m_b;
#pragma unroll
      for (int j = 0; j < BN / 8; ++j) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int kpos = tile * BN + j * 8 + c4 * 2 + e;
          float va = sc[j][e] * p.scale_log2, vb2 = sc[j][2 + e] * p.scale_log2;
          if (need_mask) {
            if (kpos > qpos_a || kpos >= kv_len) va = -INFINITY;
            if (kpos > qpos_b || kpos >= kv_len) vb2 = -INFINITY;
          }
          sc[j][e] = va;
          sc[j][2 + e] = vb2;
          mx_a = fmaxf(mx_a, va);
          mx_b = fmaxf(mx_b, vb2);
        }
      }
      mx_a = fmaxf(mx_a, __shfl_xor_sync(0xffffffff, mx_a, 1));
      mx_a = fmaxf(mx_a, __shfl_xor_sync(0xffffffff, mx_a, 2));
      mx_b = fmaxf(mx_b, __shfl_xor_sync(0xffffffff, mx_b, 1));
      mx_b = fmaxf(mx_b, __shfl_xor_sync(0xffffffff, mx_b, 2));
      const float base_a = mx_a == -INFINITY ? 0.f : mx_a;
      const float base_b = mx_b == -INFINITY ? 0.f : mx_b;
      const float corr_a = exp2f(m_a - base_a), corr_b = exp2f(m_b - base_b);
      m_a = mx_a;
      m_b = mx_b;
      float sum_a = 0.f, sum_b = 0.f;
#pragma unroll
      for (int j = 0; j < BN / 8; ++j) {
        sc[j][0] = exp2f(sc[j][0] - base_a);
        sc[j][1] = exp2f(sc[j][1] - base_a);
        sc[j][2] = exp2f(sc[j][2] - base_b);
        sc[j][3] = exp2f(sc[j][3] - base_b);
        sum_a += sc[j][0] + sc[j][1];
        sum_b += sc[j][2] + sc[j][3];
      }
      l_a = l_a * corr_a + sum_a;
      l_b = l_b * corr_b + sum_b;
#pragma unroll
      for (int i = 0; i < DH / 8; ++i) {
        o[i][0] *= corr_a;
        o[i][1] *= corr_a;
        o[i][2] *= corr_b;
        o[i][3] *= corr_b;
      }
#pragma unroll
      for (int kk = 0; kk < BN / 16; ++kk) {
        const uint32_t a0 = pack2(sc[2 * kk][0], sc[2 * kk][1]);
        const uint32_t a1 = pack2(sc[2 * kk][2], sc[2 * kk][3]);
        const uint32_t a2 = pack2(sc[2 * kk + 1][0], sc[2 * kk + 1][1]);
        const uint32_t a3 = pack2(sc[2 * kk + 1][2], sc[2 * kk + 1][3]);
#pragma unroll
        for (int jj = 0; jj < DH / 16; ++jj) {
          uint32_t b0, b1, b2, b3;
          const int r = kk * 16 + (lane & 7) + (((lane >> 3) & 1) << 3);
          const int c = jj * 2 + (lane >> 4);
          ldsm_x4_t(vb + swz<DH>(r, c), b0, b1, b2, b3);
          mma16816(o[2 * jj], a0, a1, a2, a3, b0, b1);
          mma16816(o[2 * jj + 1], a0, a1, a2, a3, b2, b3);
        }
      }
    }
    __syncthreads();
  }
  cp_wait<0>();

  // ---- normalise and store (row-sum across the quad)
  l_a += __shfl_xor_sync(0xffffffff, l_a, 1);
  l_a += __shfl_xor_sync(0xffffffff, l_a, 2);
  l_b += __shfl_xor_sync(0xffffffff, l_b, 1);
  l_b += __shfl_xor_sync(0xffffffff, l_b, 2);
  const float inv_a = l_a > 0.f ? 1.f / l_a : 0.f;
  const float inv_b = l_b > 0.f ? 1.f / l_b : 0.f;
  const int ra = wr + g, rb = ra + 8;
  __nv_bfloat16* oa = p.o + (long long)(row_base + ra / G) * p.ldo + (long long)(kvh * G + ra % G) * DH;
  __nv_bfloat16* ob = p.o + (long long)(row_base + rb / G) * p.ldo + (long long)(kvh * G + rb % G) * DH;
#pragma unroll
  for (int i = 0; i < DH / 8; ++i) {
    const int col = i * 8 + c4 * 2;
    if (ra < nrows) *reinterpret_cast<uint32_t*>(oa + col) = pack2(o[i][0] * inv_a, o[i][1] * inv_a);
    if (rb < nrows) *reinterpret_cast<uint32_t*>(ob + col) = pack2(o[i][2] * inv_b, o[i][3] * inv_b);
  }
}

template <int DH>
int launch_dh(const AttnParams& p, int n_seqs, int max_new, cudaStream_t st) {
  constexpr size_t smem = (size_t)ROWS * DH * 2 + 2 * STAGES * (size_t)BN * DH * 2;
  static bool attr = false;
  if (!attr) {
    CUDA_TRY(cudaFuncSetAttribute(attn_prefill_kernel<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  const int G = p.hq / p.hkv;
  const int tok_per_cta = ROWS / G;
  dim3 grid((max_new + tok_per_cta - 1) / tok_per_cta, p.hkv, n_seqs);
  CUDA_TRY(launch_k(attn_prefill_kernel<DH>, grid, dim3(THREADS), smem, st, p));
  CUDA_TRY(cudaGetLastError());
  return 0;
}

}  // namespace

int launch_attention(const AttnParams& p, int head_dim, int n_seqs, int max_new, cudaStream_t st) {
  if (n_seqs <= 0 || max_new <= 0) return 0;
  if (p.hq % p.hkv != 0) return set_error(RDKV_ERR_ARG, "attention: hq %% hkv != 0");
  const int G = p.hq / p.hkv;
  if (G > 128 || 128 % G != 0) return set_error(RDKV_ERR_ARG, "attention: group size %d must divide 128", G);
  if (head_dim == 64) return launch_dh<64>(p, n_seqs, max_new, st);
  if (head_dim == 128) return launch_dh<128>(p, n_seqs, max_new, st);
  return set_error(RDKV_ERR_ARG, "attention: head_dim %d unsupported", head_dim);
}

}  // namespace rdkv
