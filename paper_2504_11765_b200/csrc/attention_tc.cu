// K2/K4 on the 5th-generation tensor cores: causal prefill attention over a
// (possibly cached) KV prefix with grouped-query packing.
//
// Semantics are those of attention.cu (reference: cached_prefill_work,
// costs.py:89-99 — new tokens at positions [n_cached, n_cached+n_new) attend
// over every position <= their own).  A CTA owns 128 query rows of ONE kv
// head, row r = (token t0 + r / G, q-head kvh*G + r % G), so the G query heads
// sharing a K/V head read each K/V tile once.
//
// Warp roles (256 threads, one CTA per SM):
//   warp 0      TMA producer: K and V tiles of 128 positions (two 64-row boxes
//               each, one per KV block of the paged pool / blob) into a
//               STAGES-deep smem ring, 128-byte swizzle
//   warp 1      MMA issuer (one thread): S[b] = Q.K^T  (M=128, N=128, K=dh) into
//               TMEM, then O_tile[b] = P.V (M=128, N=dh, K=128; V is the
//               MN-major B operand) into TMEM; order QK0, QK1, PV0, QK2, PV1, ...
//   warp 2      TMEM allocator (512 columns: S x2, O_tile x2)
//   warps 4..7  softmax (one query row per thread = one TMEM lane): load Q,
//               then per tile: tcgen05.ld S, mask, online max / exp2 / sum,
//               write P (bf16, swizzled K-major) to smem; fold the previous
//               tile's O_tile into a register accumulator with the running
//               rescale; finally normalise and store O.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>
#include <cstdint>

#include "attention.cuh"
#include "common.cuh"
#include "pdl.cuh"
#include "ptx.cuh"

namespace rdkv {

int make_tmap(CUtensorMap* m, const void* base, long long rows, long long K, long long ld, int box_rows);

namespace {

constexpr int ROWS = 128;
constexpr int BKV = 128;  // key positions per tile
constexpr int HALF = 64;  // rows per TMA box (= one KV block of the pool)

template <int DH>
struct TcCfg {
  static constexpr int STAGES = DH == 64 ? 3 : 2;
  static constexpr uint32_t QB = ROWS * DH * 2;    // Q tile bytes
  static constexpr uint32_t KB = BKV * DH * 2;     // one K (or V) tile
  static constexpr uint32_t PB = ROWS * BKV * 2;   // one P tile
  static constexpr uint32_t OFF_Q = 0;
  static constexpr uint32_t OFF_K = OFF_Q + QB;
  static constexpr uint32_t OFF_V = OFF_K + STAGES * KB;
  static constexpr uint32_t OFF_P = OFF_V + STAGES * KB;
  static constexpr uint32_t OFF_RED = OFF_P + 2 * PB;  // [2 parity][2 half][128] fp32 row-max / row-sum exchange
  static constexpr uint32_t OFF_BAR = OFF_RED + 4 * ROWS * 4;
  // no alignment slack: DH=128 uses all but ~0.6 KB of the 227 KB; the base is checked at run time
  static constexpr size_t SMEM = OFF_BAR + 8 * (1 + 3 * STAGES + 12) + 16;
};

// K-major SW128 operand (rows of 128 B, 8-row atoms 1024 B apart)
__device__ __forceinline__ uint64_t desc_k(uint32_t saddr) { return sdesc_k_sw128(saddr); }

// MN-major SW128 operand: 64 MN elements (128 B) per swizzle row, 8 K rows per
// 1024-B atom (SBO), next 64 MN elements `lbo` bytes away (LBO).
__device__ __forceinline__ uint64_t desc_mn(uint32_t saddr, uint32_t lbo) {
  return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

template <int DH>
__global__ void __launch_bounds__(384, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV, AttnParams p) {
  using C = TcCfg<DH>;
  constexpr int ST = C::STAGES;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  const uint32_t sb = smem_u32(smem);
  if (sb & 1023) __trap();  // SW128 operands need 1024-B alignment
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;             // [ST]
  uint64_t* v_full = k_full + ST;          // [ST]
  uint64_t* kv_empty = v_full + ST;        // [ST]
  uint64_t* s_full = kv_empty + ST;        // [2]
  uint64_t* s_empty = s_full + 2;          // [2]
  uint64_t* p_full = s_empty + 2;          // [2]
  uint64_t* p_empty = p_full + 2;          // [2]
  uint64_t* o_full = p_empty + 2;          // [2]
  uint64_t* o_empty = o_full + 2;          // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_empty + 2);

  const int G = p.hq / p.hkv;
  const int s = blockIdx.z, kvh = blockIdx.y;
  const int xb = gridDim.x - 1 - blockIdx.x;  // longest causal rows first
  const int qb = xb / p.kv_splits, ks = xb % p.kv_splits;  // query block, KV split
  const int n_new = p.seq_new[s];
  const int tok_per_cta = ROWS / G;
  const int tok0 = qb * tok_per_cta;
  if (tok0 >= n_new) return;
  const int ntok = min(tok_per_cta, n_new - tok0);
  const int nrows = ntok * G;
  const int pos0 = p.seq_cached[s] + tok0;
  const int kv_len = pos0 + ntok;
  // this CTA's share of the KV tiles (split-KV when the grid alone cannot fill the GPU)
  const int n_all = (kv_len + BKV - 1) / BKV;
  const int per_split = (n_all + p.kv_splits - 1) / p.kv_splits;
  const int t_begin = ks * per_split;
  const int n_tiles = max(0, min(n_all, t_begin + per_split) - t_begin);
  const int row_base = p.seq_start[s] + tok0;
  const int* bt = p.block_table + (long long)s * p.bt_stride;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
  }
  if (warp == 1 && lane == 0) {
    mbar_init(q_full, 8);
    for (int i = 0; i < ST; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&v_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], 8);
      mbar_init(&p_full[i], 8);
      mbar_init(&p_empty[i], 1);
      mbar_init(&o_full[i], 1);
      mbar_init(&o_empty[i], 8);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  pdl_wait();  // q / KV planes written by the predecessor are visible from here
  const uint32_t tS = tmem;             // S buffers at columns [0,128) and [128,256)
  const uint32_t tO = tmem + 2 * BKV;   // O_tile buffers at 256 and 256 + DH

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      const long long row0 = (long long)kvh * (p.head_stride / DH);  // first row of this head in the plane view
      for (int j = 0; j < n_tiles; ++j) {
        const int st = j % ST;
        mbar_wait_sleep(&kv_empty[st], ((j / ST) & 1) ^ 1);
        int rows[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          int pos = (t_begin + j) * BKV + h * HALF;
          if (pos >= kv_len) pos = (t_begin + j) * BKV;  // masked half: any valid, finite block
          rows[h] = (int)(row0 + (long long)bt[pos / p.block_size] * p.block_size + pos % p.block_size);
        }
        mbar_arrive_expect_tx(&k_full[st], C::KB);
#pragma unroll
        for (int c = 0; c < DH / 64; ++c)
#pragma unroll
          for (int h = 0; h < 2; ++h)
            tma_load_2d_nohint(&tmK, &k_full[st], smem + C::OFF_K + st * C::KB + c * (BKV * 128) + h * (HALF * 128),
                               c * 64, rows[h]);
        mbar_arrive_expect_tx(&v_full[st], C::KB);
#pragma unroll
        for (int c = 0; c < DH / 64; ++c)
#pragma unroll
          for (int h = 0; h < 2; ++h)
            tma_load_2d_nohint(&tmV, &v_full[st], smem + C::OFF_V + st * C::KB + c * (BKV * 128) + h * (HALF * 128),
                               c * 64, rows[h]);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc_qk = idesc_bf16_f32(ROWS, BKV);
      constexpr uint32_t idesc_pv = idesc_bf16_f32(ROWS, DH) | (1u << 16);  // B (V) is MN-major
      mbar_wait_sleep(q_full, 0);
      tc_fence_after();
      auto issue_qk = [&](int j) {
        const int st = j % ST, b = j & 1;
        mbar_wait_sleep(&k_full[st], (j / ST) & 1);
        mbar_wait_sleep(&s_empty[b], ((j >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t qa = sb + C::OFF_Q, ka = sb + C::OFF_K + st * C::KB;
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) {
          const uint32_t blk = (kk >> 2) * (ROWS * 128), sub = (kk & 3) * 32;
          umma_bf16(tS + b * BKV, desc_k(qa + blk + sub), desc_k(ka + (kk >> 2) * (BKV * 128) + sub), idesc_qk,
                    kk > 0 ? 1u : 0u);
        }
        umma_commit(&s_full[b]);
      };
      auto issue_pv = [&](int j) {
        const int st = j % ST, b = j & 1;
        mbar_wait_sleep(&v_full[st], (j / ST) & 1);
        mbar_wait_sleep(&p_full[b], (j >> 1) & 1);
        mbar_wait_sleep(&o_empty[b], ((j >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t pa = sb + C::OFF_P + b * C::PB, va = sb + C::OFF_V + st * C::KB;
#pragma unroll
        for (int kk = 0; kk < BKV / 16; ++kk) {
          const uint32_t a_off = (kk >> 2) * (ROWS * 128) + (kk & 3) * 32;
          umma_bf16(tO + b * DH, desc_k(pa + a_off), desc_mn(va + kk * 2048, BKV * 128), idesc_pv, kk > 0 ? 1u : 0u);
        }
        umma_commit(&o_full[b]);
        umma_commit(&p_empty[b]);
        umma_commit(&kv_empty[st]);
      };
      if (n_tiles > 0) issue_qk(0);
      for (int j = 0; j < n_tiles; ++j) {
        if (j + 1 < n_tiles) issue_qk(j + 1);
        issue_pv(j);
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ softmax warps
    // 8 warps: warp 4+q and warp 8+q both own TMEM lanes [32q, 32q+32) (query
    // rows); half h = (warp-4)/4 takes S columns [64h, 64h+64) and O columns
    // [h*DH/2, (h+1)*DH/2).  The pair exchanges the row max per tile.
    const int quad = (warp - 4) & 3, h = (warp - 4) >> 2;
    const int r = quad * 32 + lane;  // query row == TMEM lane
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    float* red = reinterpret_cast<float*>(smem + C::OFF_RED);  // [2 parity][2 half][128 rows]
    auto pair_sync = [&]() { asm volatile("bar.sync %0, 64;" ::"r"(1 + quad) : "memory"); };
    // Q row half -> smem (K-major SW128, DH/64 column blocks of [128 rows][128 B])
    {
      const bool ok = r < nrows;
      const int rr = ok ? r : 0;
      const uint4* src = reinterpret_cast<const uint4*>(p.q + (long long)(row_base + rr / G) * p.ldq +
                                                        (long long)(kvh * G + rr % G) * DH);
#pragma unroll
      for (int cc = 0; cc < DH / 16; ++cc) {
        const int c = h * (DH / 16) + cc;
        const uint4 v = ok ? src[c] : make_uint4(0, 0, 0, 0);
        const uint32_t a = sb + C::OFF_Q + (c >> 3) * (ROWS * 128) + r * 128 + (((c & 7) ^ (r & 7)) << 4);
        st_shared_v4(a, v.x, v.y, v.z, v.w);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(q_full);
    }
    // padded rows pretend to be the last valid position so no row is fully masked
    const int qpos = (r < nrows) ? pos0 + r / G : kv_len - 1;
    const int kmax = min(qpos, kv_len - 1);  // last visible key position of this row
    const float sl2 = p.scale_log2;
    constexpr int OD = DH / 2;  // O columns owned by this half
    float o_acc[OD];
#pragma unroll
    for (int i = 0; i < OD; ++i) o_acc[i] = 0.f;
    float m_run = -INFINITY;   // max used for the newest P
    float m_acc = -INFINITY;   // scale of o_acc
    float m_pend = -INFINITY;  // max of the tile whose O_tile is pending
    float l = 0.f;             // this half's share of the row sum (same scale as o_acc after the last fold)

    auto consume = [&](int t, float m_t) {
      const int b = t & 1;
      mbar_wait(&o_full[b], (t >> 1) & 1);
      tc_fence_after();
      const float f = ex2_approx(m_acc - m_t);
#pragma unroll
      for (int c = 0; c < OD / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(tO + b * DH + h * OD + c * 32 + lane_off, v);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) o_acc[c * 32 + i] = fmaf(o_acc[c * 32 + i], f, __uint_as_float(v[i]));
      }
      m_acc = m_t;
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_empty[b]);
    };

    for (int j = 0; j < n_tiles; ++j) {
      const int b = j & 1;
      mbar_wait(&s_full[b], (j >> 1) & 1);
      tc_fence_after();
      const int kbase = (t_begin + j) * BKV + h * 64;  // first key of this half
      const int lim0 = kmax - kbase;            // element e visible iff e <= lim0
      const bool need_mask = lim0 < 63;
      const uint32_t scol = tS + b * BKV + h * 64 + lane_off;
      // this half's 64 scores stay in registers for both passes
      uint32_t va[32], vb[32];
      tmem_ld32(scol, va);
      tmem_ld32(scol + 32, vb);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[b]);  // S buffer may be overwritten now
      if (need_mask) {
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          if (i > lim0) va[i] = __float_as_uint(-INFINITY);
          if (32 + i > lim0) vb[i] = __float_as_uint(-INFINITY);
        }
      }
      // pass 1: raw max (scale > 0 commutes with max), 4 chains
      float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
      for (int i = 0; i < 32; i += 4)
#pragma unroll
        for (int u = 0; u < 4; ++u)
          m4[u] = fmaxf(m4[u], fmaxf(__uint_as_float(va[i + u]), __uint_as_float(vb[i + u])));
      const float mine = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
      red[((j & 1) * 2 + h) * ROWS + r] = mine;
      pair_sync();
      const float other = red[((j & 1) * 2 + (h ^ 1)) * ROWS + r];
      const float mx = fmaxf(m_run, fmaxf(mine, other) * sl2);
      const float nmx = -mx;
      // pass 2: P = exp2(S*scale - max) -> smem (bf16, swizzled K-major), partial row sum
      mbar_wait(&p_empty[b], ((j >> 1) & 1) ^ 1);
      float s4[4] = {0.f, 0.f, 0.f, 0.f};
      const uint32_t pbase = sb + C::OFF_P + b * C::PB + h * (ROWS * 128) + r * 128;
      auto emit = [&](const uint32_t(&v)[32], const int c) {
        uint32_t w[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          // masked scores are -inf: ex2(-inf) = +0
          const float e0 = ex2_approx(fmaf(__uint_as_float(v[2 * i]), sl2, nmx));
          const float e1 = ex2_approx(fmaf(__uint_as_float(v[2 * i + 1]), sl2, nmx));
          s4[i & 3] += e0 + e1;
          w[i] = pack_bf16(e0, e1);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int chunk = c * 4 + q;
          st_shared_v4(pbase + ((chunk ^ (r & 7)) << 4), w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
        }
      };
      emit(va, 0);
      emit(vb, 1);
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[b]);
      l = l * ex2_approx(m_run - mx) + ((s4[0] + s4[1]) + (s4[2] + s4[3]));
      m_run = mx;
      if (j >= 1) consume(j - 1, m_pend);
      m_pend = mx;
    }
    if (n_tiles > 0) consume(n_tiles - 1, m_pend);
    // total row sum = both halves; then normalise and store this half of the row
    // the parity slot the last tile did NOT use is free (its readers passed the last pair_sync)
    const int fs = n_tiles & 1;
    red[(fs * 2 + h) * ROWS + r] = l;
    pair_sync();
    const float lt = l + red[(fs * 2 + (h ^ 1)) * ROWS + r];
    if (r < nrows) {
      const long long trow = row_base + r / G;  // token row in [0, T)
      const int head = kvh * G + r % G;
      if (p.kv_splits > 1) {
        // unnormalised partial at scale m_acc; combined by attn_split_combine_kernel
        float* dst = p.split_o + (((long long)ks * p.n_tokens + trow) * p.hq + head) * DH + h * OD;
#pragma unroll
        for (int c = 0; c < OD / 4; ++c)
          reinterpret_cast<float4*>(dst)[c] =
              make_float4(o_acc[4 * c], o_acc[4 * c + 1], o_acc[4 * c + 2], o_acc[4 * c + 3]);
        if (h == 0) p.split_ml[((long long)ks * p.n_tokens + trow) * p.hq + head] = make_float2(m_acc, lt);
      } else {
        const float inv = 1.f / lt;
        uint4* dst = reinterpret_cast<uint4*>(p.o + trow * p.ldo + (long long)head * DH + h * OD);
#pragma unroll
        for (int c = 0; c < OD / 8; ++c)
          dst[c] = make_uint4(pack_bf16(o_acc[8 * c] * inv, o_acc[8 * c + 1] * inv),
                              pack_bf16(o_acc[8 * c + 2] * inv, o_acc[8 * c + 3] * inv),
                              pack_bf16(o_acc[8 * c + 4] * inv, o_acc[8 * c + 5] * inv),
                              pack_bf16(o_acc[8 * c + 6] * inv, o_acc[8 * c + 7] * inv));
      }
    }
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// Merge the KV-split partials of every (token, head): O = sum_s o_s 2^(m_s-M) / sum_s l_s 2^(m_s-M).
template <int DH>
__global__ void __launch_bounds__(256) attn_split_combine_kernel(AttnParams p) {
  pdl_trigger();
  pdl_wait();
  const int t = blockIdx.x, head = blockIdx.y * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (head >= p.hq) return;
  float M = -INFINITY;
  for (int k = 0; k < p.kv_splits; ++k) M = fmaxf(M, p.split_ml[((long long)k * p.n_tokens + t) * p.hq + head].x);
  constexpr int PER = DH / 32;
  float acc[PER] = {};
  float L = 0.f;
  for (int k = 0; k < p.kv_splits; ++k) {
    const float2 ml = p.split_ml[((long long)k * p.n_tokens + t) * p.hq + head];
    if (ml.x == -INFINITY) continue;
    const float w = ex2_approx(ml.x - M);
    L += ml.y * w;
    const float* src = p.split_o + (((long long)k * p.n_tokens + t) * p.hq + head) * DH;
#pragma unroll
    for (int e = 0; e < PER; ++e) acc[e] += src[lane + 32 * e] * w;
  }
  const float inv = L > 0.f ? 1.f / L : 0.f;
  __nv_bfloat16* dst = p.o + (long long)t * p.ldo + (long long)head * DH;
#pragma unroll
  for (int e = 0; e < PER; ++e) dst[lane + 32 * e] = __float2bfloat16(acc[e] * inv);
}

template <int DH>
int launch_tc(const AttnParams& p, int n_seqs, int max_new, cudaStream_t st) {
  using C = TcCfg<DH>;
  static bool attr = false;
  if (!attr) {
    CUDA_TRY(cudaFuncSetAttribute(attn_tc_kernel<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
    attr = true;
  }
  // plane view: rows = hkv * slots, cols = dh
  const long long rows = (long long)p.hkv * (p.head_stride / DH);
  CUtensorMap tk, tv;
  RDKV_TRY(make_tmap(&tk, p.kplane, rows, DH, DH, HALF));
  RDKV_TRY(make_tmap(&tv, p.vplane, rows, DH, DH, HALF));
  const int tok_per_cta = ROWS / (p.hq / p.hkv);
  const int qblocks = (max_new + tok_per_cta - 1) / tok_per_cta;
  // split the KV range when the (query block x kv head x sequence) grid is too
  // small for 148 SMs (single-query TTFT) and scratch is available
  AttnParams q = p;
  q.kv_splits = 1;
  const int ctas = qblocks * p.hkv * n_seqs, sms = num_sms();
  const int max_tiles = (p.max_ctx + BKV - 1) / BKV;
  if (p.split_o && ctas * 2 <= sms && max_tiles >= 4) {
    int k = sms / ctas;
    k = k < max_tiles / 2 ? k : max_tiles / 2;
    k = k < 16 ? k : 16;
    if (k >= 2 && (size_t)k * p.n_tokens * p.hq * (DH * 4 + 8) <= p.split_bytes) q.kv_splits = k;
  }
  dim3 grid(qblocks * q.kv_splits, p.hkv, n_seqs);
  CUDA_TRY(launch_k(attn_tc_kernel<DH>, grid, dim3(384), C::SMEM, st, tk, tv, q));
  CUDA_TRY(cudaGetLastError());
  if (q.kv_splits > 1) {
    CUDA_TRY(launch_k(attn_split_combine_kernel<DH>, dim3(p.n_tokens, (p.hq + 7) / 8), dim3(256), 0, st, q));
    CUDA_TRY(cudaGetLastError());
  }
  return 0;
}

}  // namespace

bool attention_tc_supported(const AttnParams& p, int head_dim) {
  const int G = p.hq / p.hkv;
  return (head_dim == 64 || head_dim == 128) && 128 % G == 0 && (p.block_size % HALF == 0 || p.contiguous);
}

int launch_attention_tc(const AttnParams& p, int head_dim, int n_seqs, int max_new, cudaStream_t st) {
  if (n_seqs <= 0 || max_new <= 0) return 0;
  if (!attention_tc_supported(p, head_dim))
    return set_error(RDKV_ERR_ARG, "attention_tc: unsupported shape (dh %d, group %d, block %d)", head_dim,
                     p.hq / p.hkv, p.block_size);
  if (head_dim == 64) return launch_tc<64>(p, n_seqs, max_new, st);
  return launch_tc<128>(p, n_seqs, max_new, st);
}

}  // namespace rdkv

namespace rdkv {
size_t attention_split_scratch_bytes(int T, int hq, int dh) {
  if (T <= 0 || T > 512) return 0;
  return (size_t)16 * T * hq * (dh * 4 + 8);
}
}  // namespace rdkv
