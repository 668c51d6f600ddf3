// K1 implementation: see gemm_tc.cuh for the design summary.
//
// Work units: (output tile, K split).  With split = 1 (the normal case) the
// epilogue applies the fused op straight from TMEM.  Small-M GEMMs (a single
// query's 64 rows) have too few tiles to occupy 148 SMs and are weight-
// bandwidth bound, so they split K: each unit writes an fp32 partial tile to
// its own slab and `splitk_finalize` sums the slabs in a fixed order (bit-for-
// bit deterministic, no atomics) and applies the same fused epilogue.
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <type_traits>
#include "common.cuh"
#include "gemm_tc.cuh"
#include "pdl.cuh"

namespace rdkv {

namespace {

constexpr int BM = 128;
constexpr int BK = 64;  // 64 bf16 = 128 B = one swizzle row
// warps 0 TMA, 1 MMA, 2 TMEM, 3 idle, 4-7 and 8-11: two epilogue warpgroups that
// split each tile's columns (a single-wave GEMM cannot hide its epilogue)
constexpr int GEMM_THREADS = 384;

template <int BN>
struct GemmCfg {
  static constexpr int STAGES = BN == 256 ? 4 : 6;
  static constexpr uint32_t A_BYTES = BM * BK * 2;
  static constexpr uint32_t B_BYTES = BN * BK * 2;
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr uint32_t TMEM_COLS = 2 * BN;  // double-buffered accumulator
  static constexpr size_t SMEM = 1024 + (size_t)STAGES * STAGE_BYTES + 256;
};

__device__ __forceinline__ float silu(float x) { return __fdividef(x, 1.0f + __expf(-x)); }

// One 32-byte (full L2 sector) store; `dst` must be 32-B aligned.
__device__ __forceinline__ void st_global_256(void* dst, const uint32_t (&w)[8]) {
  asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(dst), "r"(w[0]), "r"(w[1]),
               "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
               : "memory");
}

// Store 32 consecutive bf16 values (packed in 16 words) with 16-byte stores.
__device__ __forceinline__ void st_bf16x32(__nv_bfloat16* dst, const uint32_t (&w)[16]) {
  uint4* d = reinterpret_cast<uint4*>(dst);
#pragma unroll
  for (int i = 0; i < 4; ++i) d[i] = make_uint4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]);
}

// ---------------------------------------------------------------- shared epilogue math
// RoPE (rotate-half) on one head held in registers, then bf16 store to its destination.
template <int DH>
__device__ __forceinline__ void qkv_head_out(float (&v)[DH], int g, int row, int p, int sl, const GemmEpi& ep) {
  if (g < ep.hq + ep.hkv) {
    // the position's (cos, sin) row is DH contiguous floats: 16-B loads, two pairs each
    const float4* cs = reinterpret_cast<const float4*>(ep.rope + (long long)p * DH);
#pragma unroll
    for (int i = 0; i < DH / 4; ++i) {
      const float4 t = cs[i];
      const float a1 = v[2 * i], a2 = v[2 * i + DH / 2], b1 = v[2 * i + 1], b2 = v[2 * i + 1 + DH / 2];
      v[2 * i] = a1 * t.x - a2 * t.y;
      v[2 * i + DH / 2] = a2 * t.x + a1 * t.y;
      v[2 * i + 1] = b1 * t.z - b2 * t.w;
      v[2 * i + 1 + DH / 2] = b2 * t.z + b1 * t.w;
    }
  }
  __nv_bfloat16* dst;
  if (g < ep.hq)
    dst = ep.q + (long long)row * ep.ldq + (long long)g * DH;
  else if (g < ep.hq + ep.hkv)
    dst = ep.kplane + (long long)(g - ep.hq) * ep.head_stride + (long long)sl * DH;
  else
    dst = ep.vplane + (long long)(g - ep.hq - ep.hkv) * ep.head_stride + (long long)sl * DH;
#pragma unroll
  for (int c = 0; c < DH / 32; ++c) {
    uint32_t w[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) w[i] = pack_bf16(v[c * 32 + 2 * i], v[c * 32 + 2 * i + 1]);
    st_bf16x32(dst + c * 32, w);
  }
}

// One accumulator tile -> fused epilogue -> global.  `row` is this thread's output row
// (its TMEM lane), `taddr` the tile's TMEM address for this warp's lane quadrant.
// Per-row RMSNorm scale from the producer's per-chunk sums of squares (fixed
// summation order: row-deterministic).
__device__ __forceinline__ float row_rscale(const GemmEpi& ep, int row, int M) {
  float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
  const float* p = ep.ssq_in + row;
  int c = 0;
  for (; c + 4 <= ep.ssq_parts; c += 4) {
    s0 += p[(long long)c * M];
    s1 += p[(long long)(c + 1) * M];
    s2 += p[(long long)(c + 2) * M];
    s3 += p[(long long)(c + 3) * M];
  }
  for (; c < ep.ssq_parts; ++c) s0 += p[(long long)c * M];
  return rsqrtf(((s0 + s1) + (s2 + s3)) / (float)ep.ssq_dim + ep.norm_eps);
}

template <int EPI>
__device__ __forceinline__ float epi_rscale(const GemmEpi& ep, int row, int M) {
  if constexpr (EPI == EPI_QKV || EPI == EPI_SWIGLU)
    return ep.ssq_in && row < M ? row_rscale(ep, row, M) : 1.f;
  return 1.f;
}

template <int BN, int EPI, int DH>
__device__ __forceinline__ void epilogue_rows(uint32_t taddr, int row, int nb, int sp, int M, int N,
                                              const GemmEpi& ep, int half, float rs) {
  // rs: the fused RMSNorm scale of this A row (QKV / SWIGLU consumers; 1 otherwise),
  // computed by the caller while the tile's MMAs were still running
  const bool row_ok = row < M;

  if constexpr (EPI == EPI_STORE || EPI == EPI_STORE_F32 || EPI == EPI_RESID || EPI == EPI_PARTIAL || EPI == EPI_PUSH) {
#pragma unroll 1
    for (int c = half * (BN / 64); c < (half + 1) * (BN / 64); ++c) {
      uint32_t r[32];
      tmem_ld32(taddr + c * 32, r);
      tmem_ld_wait();
      const int col = nb * BN + c * 32;
      if (row_ok && col < N) {
        if constexpr (EPI == EPI_STORE_F32 || EPI == EPI_PARTIAL) {
          float* base = static_cast<float*>(ep.out);
          if constexpr (EPI == EPI_PARTIAL) base += (long long)sp * M * N;  // this split's slab
          float4* dst = reinterpret_cast<float4*>(base + (long long)row * (EPI == EPI_PARTIAL ? N : ep.ldo) + col);
#pragma unroll
          for (int i = 0; i < 8; ++i)
            dst[i] = make_float4(__uint_as_float(r[4 * i]), __uint_as_float(r[4 * i + 1]),
                                 __uint_as_float(r[4 * i + 2]), __uint_as_float(r[4 * i + 3]));
        } else {
          uint32_t w[16];
          if constexpr (EPI == EPI_RESID) {
            const uint4* src = reinterpret_cast<const uint4*>(ep.resid + (long long)row * ep.ldr + col);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const uint4 q = src[i];
              const uint32_t uu[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const float2 f = unpack_bf16(uu[j]);
                const int e = 8 * i + 2 * j;
                w[4 * i + j] = pack_bf16(f.x + __uint_as_float(r[e]), f.y + __uint_as_float(r[e + 1]));
              }
            }
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) w[i] = pack_bf16(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1]));
          }
          if constexpr (EPI == EPI_PUSH) {
            for (int p = 0; p < ep.npush; ++p) st_bf16x32(ep.push[p] + (long long)row * ep.ldo + col, w);
          } else {
            st_bf16x32(static_cast<__nv_bfloat16*>(ep.out) + (long long)row * ep.ldo + col, w);
          }
          if constexpr (EPI == EPI_RESID) {
            if (ep.ssq_out) {  // the next RMSNorm's statistics, from the values just stored
              float ss = 0.f;
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                const float2 f = unpack_bf16(w[i]);
                ss = fmaf(f.x, f.x, ss);
                ss = fmaf(f.y, f.y, ss);
              }
              ep.ssq_out[(long long)(col >> 5) * M + row] = ss;
            }
          }
        }
      }
    }
  } else if constexpr (EPI == EPI_SWIGLU) {
    // weights interleaved in 64-row blocks: tile column block 2i = gate, 2i+1 = up
#pragma unroll 1
    for (int c = half * (BN / 128); c < (half + 1) * (BN / 128); ++c) {
      const int pb = c >> 1, hf = c & 1;
      uint32_t g[32], v[32];
      tmem_ld32(taddr + pb * 128 + hf * 32, g);
      tmem_ld32(taddr + pb * 128 + 64 + hf * 32, v);
      tmem_ld_wait();
      const int col = nb * (BN / 2) + pb * 64 + hf * 32;  // output column
      if (row_ok && col < N / 2) {
        uint32_t w[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float a0 = silu(rs * __uint_as_float(g[2 * i])) * (rs * __uint_as_float(v[2 * i]));
          const float a1 = silu(rs * __uint_as_float(g[2 * i + 1])) * (rs * __uint_as_float(v[2 * i + 1]));
          w[i] = pack_bf16(a0, a1);
        }
        st_bf16x32(static_cast<__nv_bfloat16*>(ep.out) + (long long)row * ep.ldo + col, w);
      }
    }
  } else if constexpr (EPI == EPI_QKV && (DH == 64 || DH == 128)) {
    // each epilogue warpgroup takes a quarter of every head's columns and their RoPE
    // partners (frequencies [half DH/4, (half+1) DH/4): columns f and f + DH/2), in
    // chunks of 16 frequencies, so both halves do the same work for any head count per
    // tile (a 256x384 tile holds 3 heads of 128, a 256x192 one 3 heads of 64) and the
    // (cos, sin) of this token's 16 frequencies is loaded once per chunk for all heads
    static_assert(BN % DH == 0, "tile must hold whole heads");
    constexpr int HEADS = BN / DH;
    constexpr int NCH = DH / 64;  // 16-frequency chunks per warpgroup
    const int p = row_ok ? ep.pos[row] : 0;
    const int sl = row_ok ? ep.slot[row] : 0;
#pragma unroll 1
    for (int ch = 0; ch < NCH; ++ch) {
      const int f0 = half * (DH / 4) + ch * 16;  // first frequency of this chunk
      float2 cs[16];
      {
        const float4* src = reinterpret_cast<const float4*>(ep.rope + (long long)p * DH + 2 * f0);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float4 t = src[i];
          cs[2 * i] = make_float2(t.x, t.y);
          cs[2 * i + 1] = make_float2(t.z, t.w);
        }
      }
#pragma unroll 1
      for (int hh = 0; hh < HEADS; ++hh) {
        uint32_t ra[16], rb[16];
        tmem_ld16(taddr + hh * DH + f0, ra);
        tmem_ld16(taddr + hh * DH + DH / 2 + f0, rb);
        tmem_ld_wait();
        const int g = (nb * BN + hh * DH) / DH;  // global head index in [q | k | v]
        if (!row_ok || g >= ep.hq + 2 * ep.hkv) continue;
        uint32_t wa[8], wb[8];
        if (g < ep.hq + ep.hkv) {
#pragma unroll
          for (int i = 0; i < 16; i += 2) {
            const float a0 = rs * __uint_as_float(ra[i]), a1 = rs * __uint_as_float(ra[i + 1]);
            const float b0 = rs * __uint_as_float(rb[i]), b1 = rs * __uint_as_float(rb[i + 1]);
            wa[i / 2] = pack_bf16(a0 * cs[i].x - b0 * cs[i].y, a1 * cs[i + 1].x - b1 * cs[i + 1].y);
            wb[i / 2] = pack_bf16(b0 * cs[i].x + a0 * cs[i].y, b1 * cs[i + 1].x + a1 * cs[i + 1].y);
          }
        } else {
#pragma unroll
          for (int i = 0; i < 16; i += 2) {
            wa[i / 2] = pack_bf16(rs * __uint_as_float(ra[i]), rs * __uint_as_float(ra[i + 1]));
            wb[i / 2] = pack_bf16(rs * __uint_as_float(rb[i]), rs * __uint_as_float(rb[i + 1]));
          }
        }
        __nv_bfloat16* dst;
        if (g < ep.hq)
          dst = ep.q + (long long)row * ep.ldq + (long long)g * DH;
        else if (g < ep.hq + ep.hkv)
          dst = ep.kplane + (long long)(g - ep.hq) * ep.head_stride + (long long)sl * DH;
        else
          dst = ep.vplane + (long long)(g - ep.hq - ep.hkv) * ep.head_stride + (long long)sl * DH;
        st_global_256(dst + f0, wa);  // 32-B aligned: f0 is a multiple of 16
        st_global_256(dst + DH / 2 + f0, wb);
      }
    }
  } else if constexpr (EPI == EPI_QKV) {
    static_assert(BN % DH == 0, "tile must hold whole heads");
    const int p = row_ok ? ep.pos[row] : 0;
    const int sl = row_ok ? ep.slot[row] : 0;
    constexpr int HEADS = BN / DH, PER = (HEADS + 1) / 2;  // heads per epilogue warpgroup
#pragma unroll 1
    for (int hh = half * PER; hh < (half + 1) * PER && hh < HEADS; ++hh) {
      float v[DH];
#pragma unroll
      for (int c = 0; c < DH / 32; ++c) {
        uint32_t r[32];
        tmem_ld32(taddr + hh * DH + c * 32, r);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) v[c * 32 + i] = rs * __uint_as_float(r[i]);
      }
      const int g = (nb * BN + hh * DH) / DH;  // global head index in [q | k | v]
      if (!row_ok || g >= ep.hq + 2 * ep.hkv) continue;
      qkv_head_out<DH>(v, g, row, p, sl, ep);
    }
  }
}

template <int BN, int EPI, int DH>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    gemm_bf16_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                        int M, int N, int K, int splits, GemmEpi ep) {
  using C = GemmCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int m_tiles = (M + BM - 1) / BM;
  const int n_tiles = (N + BN - 1) / BN;
  const int units = m_tiles * n_tiles * splits;
  const int kblocks = K / BK;
  const int kb_per = (kblocks + splits - 1) / splits;
  // unit -> (tile, k-range); tiles are M-fastest so CTAs resident together share weight tiles
  auto decode = [&](int u, int& mb, int& nb, int& kb0, int& kb1, int& sp) {
    const int t = u / splits;
    sp = u - t * splits;
    mb = t % m_tiles;
    nb = t / m_tiles;
    kb0 = sp * kb_per;
    kb1 = min(kb0 + kb_per, kblocks);
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 8);  // 2 epilogue warpgroups x 4 warps
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_trigger();
  pdl_wait();  // predecessor's outputs (activations, residual) are visible from here

  if (warp == 0) {
    // ---------------- TMA producer
    if (lane == 0) {
      const uint64_t pol_act = policy_evict_last();
      const uint64_t pol_w = ep.w_policy ? policy_evict_first() : pol_act;
      int stage = 0;
      uint32_t phase = 0;
      const int pf = ep.b_pf;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        int mb, nb, kb0, kb1, sp;
        decode(u, mb, nb, kb0, kb1, sp);
        // this CTA's share (k-blocks kb with kb % m_tiles == mb) of the B prefetch stream
        auto prefetch_b = [&](int kb) {
          if (kb < kb1 && kb % m_tiles == mb) tma_prefetch_2d(&tmB, kb * BK, nb * BN);
        };
        if (pf > 0)
          for (int kb = kb0; kb < kb0 + pf; ++kb) prefetch_b(kb);
        for (int kb = kb0; kb < kb1; ++kb) {
          if (pf > 0) prefetch_b(kb + pf);
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES);
          tma_load_2d(&tmA, &full[stage], sA + stage * C::A_BYTES, kb * BK, mb * BM, pol_act);
          if (ep.w_policy)
            tma_load_2d(&tmB, &full[stage], sB + stage * C::B_BYTES, kb * BK, nb * BN, pol_w);
          else
            tma_load_2d_nohint(&tmB, &full[stage], sB + stage * C::B_BYTES, kb * BK, nb * BN);
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (single thread)
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16_f32(BM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        int mb, nb, kb0, kb1, sp;
        decode(u, mb, nb, kb0, kb1, sp);
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t ad = sdesc_k_sw128(smem_u32(sA + stage * C::A_BYTES));
          const uint64_t bd = sdesc_k_sw128(smem_u32(sB + stage * C::B_BYTES));
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            umma_bf16(d, ad + 2 * k, bd + 2 * k, idesc, (kb != kb0 || k != 0) ? 1u : 0u);
          umma_commit(&empty[stage]);
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&tfull[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else if (warp == 3) {
    // idle warp: pull the next kernel's weights into L2 while this GEMM computes
    l2_prefetch_share(ep.l2_next, ep.l2_next_bytes, blockIdx.x, gridDim.x, lane);
  } else if (warp >= 4) {
    // ---------------- epilogue: TMEM -> registers -> fused op -> global
    const int wq = warp & 3;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      int mb, nb, kb0, kb1, sp;
      decode(u, mb, nb, kb0, kb1, sp);
      const int row = mb * BM + wq * 32 + lane;
      const float rs = epi_rscale<EPI>(ep, row, M);  // overlaps this tile's MMAs
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t taddr = tmem_base + acc * BN + ((uint32_t)(wq * 32) << 16);
      epilogue_rows<BN, EPI, DH>(taddr, row, nb, sp, M, N, ep, (warp - 4) >> 2, rs);
      if constexpr (EPI == EPI_PUSH) __threadfence_system();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
}

// ---------------------------------------------------------------- CTA-pair GEMM
// cta_group::2 variant for large M: a cluster of 2 CTAs (one SM pair) owns a
// 256 x 256 output tile.  Each CTA stages its 128 rows of A and its 128 of the
// 256 B rows (TMA completes on the leader's barrier); the leader issues M=256
// MMAs that read both CTAs' smem and write each CTA's 128 accumulator rows to
// its own TMEM.  Operand bytes per FLOP halve vs the 128 x 256 single-CTA tile,
// which is what lifts the L2 -> SM traffic ceiling (~12 TB/s on B200).
template <int BN>
struct PairCfg {
  // BN = 384: a single TMEM accumulator (384 of 512 columns) filled by two MMAs per
  // k-step (N = 256 + 128); only planned when every pair gets at most one tile
  static constexpr int NACC = BN == 384 ? 1 : 2;
  static constexpr int STAGES = BN == 384 ? 5 : BN == 256 ? 6 : BN == 192 ? 7 : 8;
  static constexpr uint32_t A_BYTES = 128 * BK * 2, B_BYTES = (BN / 2) * BK * 2, STAGE = A_BYTES + B_BYTES;
  static constexpr size_t SMEM = 1024 + (size_t)STAGES * STAGE + 256;
};

__device__ __forceinline__ int ld_acquire_flag(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_flag(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int BN, int EPI, int DH, bool SK = false, bool MC = false>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    gemm_bf16_tc2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M,
                         int N, int K, GemmEpi ep) {
  using C = PairCfg<BN>;
  constexpr int STAGES = C::STAGES;
  constexpr uint32_t A_BYTES = C::A_BYTES, B_BYTES = C::B_BYTES, STAGE = C::STAGE;
  constexpr int NACC = C::NACC;
  constexpr uint32_t TMEM_COLS = NACC * BN <= 256 ? NACC * BN : 512;  // a power of two >= NACC x BN
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // MC: clusters of two CTA pairs that own M tiles 2j, 2j + 1 of the same B tile; each CTA
  // loads half of its B rows and multicasts them to its counterpart in the other pair
  const uint32_t crank = cluster_ctarank();
  const uint32_t rank = crank & 1u, grp = MC ? crank >> 1 : 0u, lead = crank & ~1u;
  const int pair = MC ? (int)cluster_id_x() * 2 + (int)grp : (int)cluster_id_x();
  const int npairs = MC ? 2 * (int)nclusters_x() : (int)nclusters_x();
  const int m_tiles = (M + 255) / 256, n_tiles = (N + BN - 1) / BN;
  const int units = m_tiles * n_tiles, kblocks = K / BK;
  // Work items: whole tiles round-robin over the pairs, or (SK, stream-K) equal shares of
  // the unit-major k-block order, cut at tile boundaries into segments [kb0, kb1)
  // (hybrid: the first sk_dp units whole and round-robin, then the k-blocks of the rest
  // shared by the first sk_tp pairs)
  const int sk_dp = SK ? ep.sk_dp : 0, sk_tp = SK ? ep.sk_tp : npairs;
  const long long W0 = (long long)sk_dp * kblocks, W = (long long)units * kblocks - W0;
  auto share = [&](int p) { return W0 + W * min(p, sk_tp) / sk_tp; };
  auto for_segments = [&](auto&& fn) {  // fn(unit, kb0, kb1)
    if constexpr (SK) {
      for (int u = pair; u < sk_dp; u += npairs) fn(u, 0, kblocks);
      const long long hi = share(pair + 1);
      for (long long w = share(pair); w < hi;) {
        const int u = (int)(w / kblocks), kb0 = (int)(w % kblocks);
        const int kb1 = (int)min((long long)kblocks, kb0 + (hi - w));
        fn(u, kb0, kb1);
        w += kb1 - kb0;
      }
    } else if constexpr (MC) {
      for (int j = (int)cluster_id_x(); j < units / 2; j += (int)nclusters_x()) fn(2 * j + (int)grp, 0, kblocks);
    } else {
      for (int u = pair; u < units; u += npairs) fn(u, 0, kblocks);
    }
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], MC ? 2 : 1);  // MC: both pairs' MMAs read the multicast B
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 16);  // 2 epilogue warpgroups x 4 warps in each CTA of the pair
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_2sm(tmem_slot, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // peer barriers initialised before any remote arrive / complete_tx
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_trigger();
  pdl_wait();

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol_act = policy_evict_last();
      const uint64_t pol_w = ep.w_policy ? policy_evict_first() : pol_act;
      int stage = 0;
      uint32_t phase = 0;
      const int pf = ep.b_pf;
      for_segments([&](int u, int kb0, int kb1) {
        const int mb = u % m_tiles, nb = u / m_tiles;
        // this CTA's half of B, k-blocks kb with kb % m_tiles == mb (the M tiles sharing the
        // B tile split the prefetch stream)
        auto prefetch_b = [&](int kb) {
          if (kb >= kb1 || kb % m_tiles != mb) return;
          if constexpr (BN == 384) {
            tma_prefetch_2d(&tmB, kb * BK, nb * BN + (int)rank * 128);
            tma_prefetch_2d(&tmB, kb * BK, nb * BN + (int)rank * 128 + 64);
            tma_prefetch_2d(&tmB, kb * BK, nb * BN + 256 + (int)rank * 64);
          } else {
            tma_prefetch_2d(&tmB, kb * BK, nb * BN + (int)rank * (BN / 2));
          }
        };
        if (pf > 0)
          for (int kb = kb0; kb < kb0 + pf; ++kb) prefetch_b(kb);
        for (int kb = kb0; kb < kb1; ++kb) {
          if (pf > 0) prefetch_b(kb + pf);
          mbar_wait(&empty[stage], phase ^ 1);
          if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * STAGE);
          const uint32_t bar = mapa_shared(smem_u32(&full[stage]), lead);
          tma_load_2d_2sm(&tmA, bar, sA + stage * A_BYTES, kb * BK, mb * 256 + (int)rank * 128, pol_act);
          if constexpr (BN == 384) {
            // each CTA holds its N-half of both MMAs: rows [128 r, +128) of the N = 256 one and
            // [256 + 64 r, +64) of the N = 128 one (64-row boxes)
            uint8_t* b = sB + stage * B_BYTES;
            tma_load_2d_2sm(&tmB, bar, b, kb * BK, nb * BN + (int)rank * 128, pol_w);
            tma_load_2d_2sm(&tmB, bar, b + 64 * 128, kb * BK, nb * BN + (int)rank * 128 + 64, pol_w);
            tma_load_2d_2sm(&tmB, bar, b + 128 * 128, kb * BK, nb * BN + 256 + (int)rank * 64, pol_w);
          } else if constexpr (MC) {
            tma_load_2d_2sm_mc(&tmB, bar, sB + stage * B_BYTES + grp * (BN / 4) * 128, kb * BK,
                               nb * BN + (int)rank * (BN / 2) + (int)grp * (BN / 4), (uint16_t)(0x5u << rank), pol_w);
          } else {
            tma_load_2d_2sm(&tmB, bar, sB + stage * B_BYTES, kb * BK, nb * BN + (int)rank * (BN / 2), pol_w);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      });
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      constexpr int BN1 = BN == 384 ? 256 : BN;  // first (or only) MMA's N
      constexpr uint32_t idesc = idesc_bf16_f32(256, BN1);
      constexpr uint32_t idesc2 = idesc_bf16_f32(256, 128);
      int stage = 0, acc = 0;
      uint32_t phase = 0, acc_phase = 0;
      for_segments([&](int, int kb0, int kb1) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t ad = sdesc_k_sw128(smem_u32(sA + stage * A_BYTES));
          const uint64_t bd = sdesc_k_sw128(smem_u32(sB + stage * B_BYTES));
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            umma_bf16_2sm(d, ad + 2 * k, bd + 2 * k, idesc, ((kb - kb0) | k) != 0 ? 1u : 0u);
          if constexpr (BN == 384) {
            const uint64_t bd2 = sdesc_k_sw128(smem_u32(sB + stage * B_BYTES + 128 * 128));
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              umma_bf16_2sm(d + 256, ad + 2 * k, bd2 + 2 * k, idesc2, ((kb - kb0) | k) != 0 ? 1u : 0u);
          }
          umma_commit_2sm(&empty[stage], MC ? 0xF : 0x3);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit_2sm(&tfull[acc], (uint16_t)(0x3u << (2 * grp)));
        if (NACC == 2) acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      });
    }
  } else if (warp == 3) {
    // idle warp: pull the next kernel's weights into L2 while this GEMM computes
    l2_prefetch_share(ep.l2_next, ep.l2_next_bytes, blockIdx.x, gridDim.x, lane);
  } else if (warp >= 4) {
    const int wq = warp & 3;
    int acc = 0;
    uint32_t acc_phase = 0;
    const uint32_t tempty0 = mapa_shared(smem_u32(&tempty[0]), lead), tempty1 = mapa_shared(smem_u32(&tempty[1]), lead);
    const int half = (warp - 4) >> 2;
    auto epi_bar = [&]() { asm volatile("bar.sync 2, 256;" ::: "memory"); };  // the 8 epilogue warps
    for_segments([&](int u, int kb0, int kb1) {
      const int mb = u % m_tiles, nb = u / m_tiles;
      const int row = mb * 256 + (int)rank * 128 + wq * 32 + lane;
      const float rs = kb0 == 0 ? epi_rscale<EPI>(ep, row, M) : 1.f;  // overlaps this tile's MMAs
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t taddr = tmem_base + acc * BN + ((uint32_t)(wq * 32) << 16);
      if constexpr (SK) {
        // partial tiles: [BN/4][128 rows][4] fp32 per (pair, CTA) slot, so a warp's float4
        // accesses of one column group cover 512 contiguous bytes
        auto slot = [&](int p) {
          return reinterpret_cast<float4*>(ep.sk_part + (size_t)(p * 2 + (int)rank) * 128 * BN) + wq * 32 + lane;
        };
        if (kb0 > 0) {  // a later part of a tile whose first k-blocks another pair holds
          float4* dst = slot(pair);
#pragma unroll 1
          for (int c = half * (BN / 64); c < (half + 1) * (BN / 64); ++c) {
            uint32_t r[32];
            tmem_ld32(taddr + c * 32, r);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 8; ++e)
              dst[(c * 8 + e) * 128] = make_float4(__uint_as_float(r[4 * e]), __uint_as_float(r[4 * e + 1]),
                                                   __uint_as_float(r[4 * e + 2]), __uint_as_float(r[4 * e + 3]));
          }
          __threadfence();
          epi_bar();
          if (warp == 4 && lane == 0) st_release_flag(ep.sk_flag + pair * 2 + (int)rank, 1);
        } else if (kb1 < kblocks) {  // the tile's first k-blocks: add the later pairs' parts
          const long long uend = (long long)(u + 1) * kblocks;
          for (int q = pair + 1; q < npairs && share(q) < uend; ++q) {
            if (lane == 0) {
              long long spins = 0;
              while (ld_acquire_flag(ep.sk_flag + q * 2 + (int)rank) == 0)
                if (++spins > (1ll << 31)) __trap();
            }
            __syncwarp();
            const float4* src = slot(q);
#pragma unroll 1
            for (int c = half * (BN / 64); c < (half + 1) * (BN / 64); ++c) {
              uint32_t r[32];
              tmem_ld32(taddr + c * 32, r);
              tmem_ld_wait();
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                const float4 t = __ldcg(src + (c * 8 + e) * 128);
                r[4 * e] = __float_as_uint(__uint_as_float(r[4 * e]) + t.x);
                r[4 * e + 1] = __float_as_uint(__uint_as_float(r[4 * e + 1]) + t.y);
                r[4 * e + 2] = __float_as_uint(__uint_as_float(r[4 * e + 2]) + t.z);
                r[4 * e + 3] = __float_as_uint(__uint_as_float(r[4 * e + 3]) + t.w);
              }
              tmem_st32(taddr + c * 32, r);
            }
          }
          tmem_st_wait();
          tc_fence_before();
          epi_bar();  // every column of the summed tile is in TMEM before any epilogue reads it
          tc_fence_after();
          if (warp == 4 && lane == 0)  // consumed: re-arm the parts' flags for the next launch
            for (int q = pair + 1; q < npairs && share(q) < uend; ++q) ep.sk_flag[q * 2 + (int)rank] = 0;
        }
      }
      if (kb0 == 0) epilogue_rows<BN, EPI, DH>(taddr, row, nb, 0, M, N, ep, half, rs);
      if constexpr (EPI == EPI_PUSH) __threadfence_system();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(acc ? tempty1 : tempty0);
      if (NACC == 2) acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    });
  }
  __syncthreads();
  cluster_sync();  // the leader's MMAs into this CTA's TMEM / smem are complete
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_2sm(tmem_base, TMEM_COLS);
  }
}

template <int BN, int EPI, int DH, bool SK = false, bool MC = false>
int launch_pair(const CUtensorMap& ta, const CUtensorMap& tb, int M, int N, int K, const GemmEpi& ep,
                cudaStream_t stream, int sk_pairs = 0) {
  constexpr size_t SMEM = PairCfg<BN>::SMEM;
  auto kern = gemm_bf16_tc2_kernel<BN, EPI, DH, SK, MC>;
  static bool attr_set = false;
  if (!attr_set) {
    CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM));
    attr_set = true;
  }
  const int units = ((M + 255) / 256) * ((N + BN - 1) / BN);
  const int max_pairs = num_sms() / 2;
  // stream-K: every pair co-resident (a split tile's first pair waits for the later ones)
  int pairs = SK ? sk_pairs : units < max_pairs ? units : max_pairs;
  if constexpr (MC) {
    // clusters of two pairs, one M-tile couple each; a persistent grid only as large as the
    // 4-CTA clusters that fit at once (GPCs whose SM count is not a multiple of 4 hold fewer)
    static int fit = -1;
    if (fit < 0) {
      cudaLaunchConfig_t q{};
      q.gridDim = dim3(num_sms());
      q.blockDim = dim3(GEMM_THREADS);
      q.dynamicSmemBytes = SMEM;
      cudaLaunchAttribute a{};
      a.id = cudaLaunchAttributeClusterDimension;
      a.val.clusterDim.x = 4;
      a.val.clusterDim.y = 1;
      a.val.clusterDim.z = 1;
      q.attrs = &a;
      q.numAttrs = 1;
      int c = 0;
      fit = cudaOccupancyMaxActiveClusters(&c, kern, &q) == cudaSuccess && c > 0 ? std::min(c, num_sms() / 4) : 1;
      cudaGetLastError();
      if (std::getenv("RDKV_GEMM_MC_VERBOSE")) std::fprintf(stderr, "rdkv: %d 4-CTA clusters fit\n", fit);
    }
    pairs = std::min(units, 2 * fit) & ~1;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(GEMM_THREADS);
  cfg.dynamicSmemBytes = SMEM;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = MC ? 4 : 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, ta, tb, M, N, K, ep));
  return 0;
}

// ---------------------------------------------------------------- small-M swap-AB
// D^T = W . X^T for M <= 128 tokens: the weights are the 128-row A operand
// (every weight byte crosses L2->SM once), the NT-row token tile is UMMA N.  Each
// unit (128 weight rows, K split) writes fp32 partial rows part[split][m][n]
// (thread = weight row n, so a warp writes 32 consecutive n per token: coalesced);
// splitk_finalize applies the fused epilogue.
//
// EPI != EPI_PARTIAL (fused small-M path): no finalize kernel.  With one split the epilogue
// warps apply the epilogue straight from TMEM; otherwise every split's CTA writes its partial,
// and the CTA whose atomic ticket on the weight tile comes last (after a __threadfence)
// sums the partials in split order (deterministic) and applies the epilogue for that tile's
// 128 output columns.  Norms use the per-chunk sum-of-squares scheme (ep.ssq_out / ssq_in).
// Token tiles of <= 64 rows (decode steps, single queries): two CTAs per SM (RDKV_SWAPAB_2CTA), each with a
// shallower ring, so one CTA's prologue / epilogue overlaps the other's weight stream.
#ifndef RDKV_SWAPAB_2CTA
#define RDKV_SWAPAB_2CTA 1
#endif
#ifndef RDKV_SWAPAB_2CTA_MAXNT
#define RDKV_SWAPAB_2CTA_MAXNT 64
#endif
template <int NT>
struct SwapCfg {
  static constexpr int CTAS_PER_SM = (RDKV_SWAPAB_2CTA && NT <= RDKV_SWAPAB_2CTA_MAXNT) ? 2 : 1;
  static constexpr int STAGES = NT >= 128 ? 6 : CTAS_PER_SM == 2 ? (NT >= 64 ? 4 : 5) : 8;
};
template <int NT, int EPI = EPI_PARTIAL, int DH = 0>
__global__ void __launch_bounds__(256, SwapCfg<NT>::CTAS_PER_SM)
    gemm_swapab_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX, int M, int N,
                       int K, int splits, float* __restrict__ part, GemmEpi ep) {
  constexpr bool FUSED = EPI != EPI_PARTIAL;
  constexpr int STAGES = SwapCfg<NT>::STAGES;
  constexpr uint32_t W_BYTES = 128 * BK * 2, X_BYTES = NT * BK * 2, STAGE = W_BYTES + X_BYTES;
  constexpr uint32_t ACC = NT < 32 ? 32 : NT;  // accumulator column stride (tcgen05.ld reads 32 columns)
  constexpr uint32_t TMEM_COLS = 2 * ACC;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sW = smem;
  uint8_t* sX = smem + STAGES * W_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int w_tiles = (N + 127) / 128;
  const int units = w_tiles * splits;
  const int kblocks = K / BK, kb_per = (kblocks + splits - 1) / splits;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmW);
    tma_prefetch_desc(&tmX);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol_act = policy_evict_last();
      // The weights are never written by the preceding kernels: the first unit's first
      // STAGES weight tiles are requested BEFORE griddepcontrol.wait, so their cold DRAM
      // latency overlaps the predecessor's tail (programmatic dependent launch); the
      // activation tiles (the predecessor's output) follow once it has completed.
      int pre = 0;
      if (blockIdx.x < units) {
        const int wt = blockIdx.x / splits, sp = blockIdx.x % splits;
        const int kb0 = sp * kb_per, kb1 = min(kb0 + kb_per, kblocks);
        pre = min(STAGES, kb1 - kb0);
        for (int s = 0; s < pre; ++s) {
          mbar_arrive_expect_tx(&full[s], STAGE);
          tma_load_2d_nohint(&tmW, &full[s], sW + s * W_BYTES, (kb0 + s) * BK, wt * 128);
        }
      }
      pdl_wait();
      int stage = 0, n = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int wt = u / splits, sp = u % splits;
        const int kb0 = sp * kb_per, kb1 = min(kb0 + kb_per, kblocks);
        for (int kb = kb0; kb < kb1; ++kb, ++n) {
          if (n >= pre) {
            mbar_wait(&empty[stage], phase ^ 1);
            mbar_arrive_expect_tx(&full[stage], STAGE);
            tma_load_2d_nohint(&tmW, &full[stage], sW + stage * W_BYTES, kb * BK, wt * 128);
          }
          tma_load_2d(&tmX, &full[stage], sX + stage * X_BYTES, kb * BK, 0, pol_act);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16_f32(128, NT);
      int stage = 0, acc = 0;
      uint32_t phase = 0, acc_phase = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int sp = u % splits;
        const int kb0 = sp * kb_per, kb1 = min(kb0 + kb_per, kblocks);
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + acc * ACC;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t ad = sdesc_k_sw128(smem_u32(sW + stage * W_BYTES));
          const uint64_t bd = sdesc_k_sw128(smem_u32(sX + stage * X_BYTES));
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) umma_bf16(d, ad + 2 * k, bd + 2 * k, idesc, (kb != kb0 || k != 0) ? 1u : 0u);
          umma_commit(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&tfull[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else if (warp == 3) {
    // idle warp: this CTA's share of the next kernel's weights into L2 (weights are never
    // written by a predecessor: no griddepcontrol.wait needed)
    l2_prefetch_share(ep.l2_next, ep.l2_next_bytes, blockIdx.x, gridDim.x, lane);
  } else if (warp >= 4) {
    pdl_wait();  // the split-K scratch may still be read by the predecessor's finalize
    const int wq = warp & 3;
    const int r = wq * 32 + lane;  // weight row within the tile == output column offset
    int acc = 0;
    uint32_t acc_phase = 0;
    // fused epilogue scratch (after the stage ring): RoPE / SwiGLU partner exchange [32][128] fp32,
    // per-row RMSNorm scales [128], the last-split flag
    float* xs = reinterpret_cast<float*>(smem + STAGES * STAGE + 1024);
    float* rs_s = xs + 32 * 128;
    int* last_s = reinterpret_cast<int*>(rs_s + 128);
    auto epi_bar = [&]() { asm volatile("bar.sync 1, 128;" ::: "memory"); };
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int wt = u / splits, sp = u % splits;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int n = wt * 128 + r;  // weight row == output column
      const uint32_t taddr = tmem_base + acc * ACC + ((uint32_t)(wq * 32) << 16);
      float* dst = part + (long long)sp * M * N + n;
      bool direct = false;  // fused, one split: epilogue straight from TMEM
      if constexpr (FUSED) direct = splits == 1;
      if (!direct) {
#pragma unroll
        for (int c = 0; c < (NT + 31) / 32; ++c) {
          uint32_t rr[32];
          tmem_ld32(taddr + c * 32, rr);
          tmem_ld_wait();
          if (n < N) {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (c * 32 + i < M) dst[(long long)(c * 32 + i) * N] = __uint_as_float(rr[i]);
          }
        }
      }
      if constexpr (FUSED) {
        bool mine = direct;
        if (!direct) {  // last split of this weight tile does the epilogue
          __threadfence();
          epi_bar();
          if (r == 0) *last_s = atomicAdd(&ep.counters[wt], 1) == splits - 1;
          epi_bar();
          mine = *last_s != 0;
          if (mine) __threadfence();
        }
        if (mine) {
          if (ep.ssq_in && (EPI == EPI_QKV || EPI == EPI_SWIGLU)) {  // per-row RMSNorm scales
            if (r < M) {
              float v0 = 0.f, v1 = 0.f, v2 = 0.f, v3 = 0.f;
              const float* p = ep.ssq_in + r;
              int c = 0;
              for (; c + 4 <= ep.ssq_parts; c += 4) {
                v0 += p[(long long)c * M];
                v1 += p[(long long)(c + 1) * M];
                v2 += p[(long long)(c + 2) * M];
                v3 += p[(long long)(c + 3) * M];
              }
              for (; c < ep.ssq_parts; ++c) v0 += p[(long long)c * M];
              rs_s[r] = rsqrtf(((v0 + v1) + (v2 + v3)) / (float)ep.ssq_dim + ep.norm_eps);
            }
            epi_bar();
          }
#pragma unroll 1
          for (int c = 0; c < (M + 31) / 32; ++c) {
            float v[32];
            if (direct) {
              uint32_t rr[32];
              tmem_ld32(taddr + c * 32, rr);
              tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(rr[i]);
            } else {
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] = 0.f;
              for (int k = 0; k < splits; ++k) {  // split order: deterministic
                const float* src = part + (long long)k * M * N + n;
#pragma unroll
                for (int i = 0; i < 32; ++i)
                  if (c * 32 + i < M && n < N) v[i] += __ldcg(src + (long long)(c * 32 + i) * N);
              }
            }
            if constexpr (EPI == EPI_QKV || EPI == EPI_SWIGLU) {
              if (ep.ssq_in) {
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] *= rs_s[min(c * 32 + i, 127)];
              }
            }
            if constexpr (EPI == EPI_STORE_F32 || EPI == EPI_STORE || EPI == EPI_RESID) {
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                const int m = c * 32 + i;
                float y = v[i];
                if (m < M && n < N) {
                  if constexpr (EPI == EPI_STORE_F32) {
                    static_cast<float*>(ep.out)[(long long)m * ep.ldo + n] = y;
                  } else {
                    if constexpr (EPI == EPI_RESID) y += __bfloat162float(ep.resid[(long long)m * ep.ldr + n]);
                    const __nv_bfloat16 yb = __float2bfloat16(y);
                    static_cast<__nv_bfloat16*>(ep.out)[(long long)m * ep.ldo + n] = yb;
                    y = __bfloat162float(yb);
                  }
                } else {
                  y = 0.f;
                }
                if constexpr (EPI == EPI_RESID) {
                  if (ep.ssq_out) {  // the next RMSNorm's statistics: this warp's 32 columns = one chunk
                    float q = y * y;
#pragma unroll
                    for (int o = 16; o; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
                    if (lane == 0 && m < M) ep.ssq_out[(long long)(n >> 5) * M + m] = q;
                  }
                }
              }
            } else if constexpr (EPI == EPI_SWIGLU) {
              // weight rows [0, 64) of the tile are gate, [64, 128) up, for output columns wt*64 + r % 64
              if (r >= 64) {
#pragma unroll
                for (int i = 0; i < 32; ++i) xs[i * 128 + r] = v[i];
              }
              epi_bar();
              if (r < 64) {
                const int o = wt * 64 + r;
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                  const int m = c * 32 + i;
                  if (m < M && o < N / 2)
                    static_cast<__nv_bfloat16*>(ep.out)[(long long)m * ep.ldo + o] =
                        __float2bfloat16(silu(v[i]) * xs[i * 128 + r + 64]);
                }
              }
              epi_bar();
            } else if constexpr (EPI == EPI_QKV) {
              // DH = 128: the tile is one head; DH = 64: two.  RoPE pairs (d, d + DH/2) within a head.
#pragma unroll
              for (int i = 0; i < 32; ++i) xs[i * 128 + r] = v[i];
              epi_bar();
              const int g = (wt * 128 + r) / DH, d = r % DH;
              const bool rot = g < ep.hq + ep.hkv;
#pragma unroll 4
              for (int i = 0; i < 32; ++i) {
                const int m = c * 32 + i;
                if (m >= M || n >= N) continue;
                float y = v[i];
                if (rot) {
                  const int p = ep.pos[m];
                  const float2 cs = reinterpret_cast<const float2*>(ep.rope)[(long long)p * (DH / 2) + (d % (DH / 2))];
                  const int base = r - d;  // this head's first row in the tile
                  y = d < DH / 2 ? v[i] * cs.x - xs[i * 128 + base + d + DH / 2] * cs.y
                                 : v[i] * cs.x + xs[i * 128 + base + d - DH / 2] * cs.y;
                }
                __nv_bfloat16* o;
                if (g < ep.hq)
                  o = ep.q + (long long)m * ep.ldq + (long long)g * DH + d;
                else if (g < ep.hq + ep.hkv)
                  o = ep.kplane + (long long)(g - ep.hq) * ep.head_stride + (long long)ep.slot[m] * DH + d;
                else
                  o = ep.vplane + (long long)(g - ep.hq - ep.hkv) * ep.head_stride + (long long)ep.slot[m] * DH + d;
                *o = __float2bfloat16(y);
              }
              epi_bar();
            }
          }
          if (!direct && r == 0) ep.counters[wt] = 0;  // ticket reset for the next launch
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, TMEM_COLS);
  }
}

template <int NT, int EPI = EPI_PARTIAL, int DH = 0>
int launch_swapab(const CUtensorMap& tw, const CUtensorMap& tx, int M, int N, int K, int splits, float* part,
                  const GemmEpi& ep, cudaStream_t stream) {
  // stage ring + the fused epilogue's exchange [32][128] fp32, row scales [128], flag
  constexpr size_t SMEM = 1024 + SwapCfg<NT>::STAGES * ((size_t)128 * BK * 2 + (size_t)NT * BK * 2) + 256 +
                          (EPI != EPI_PARTIAL ? 1024 + 32 * 128 * 4 + 128 * 4 + 16 : 0);
  static bool attr_set = false;
  auto kern = gemm_swapab_kernel<NT, EPI, DH>;
  if (!attr_set) {
    CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM));
    attr_set = true;
  }
  const int units = ((N + 127) / 128) * splits, slots = num_sms() * SwapCfg<NT>::CTAS_PER_SM;
  const int grid = units < slots ? units : slots;
  CUDA_TRY(launch_k(kern, dim3(grid), dim3(256), SMEM, stream, tw, tx, M, N, K, splits, part, ep));
  return 0;
}

// ---------------------------------------------------------------- split-K finalize
// Sum the split slabs in a fixed order (deterministic) and apply the epilogue.
// Grid: (rows, column chunks); 4 consecutive columns per thread (float4 loads).
template <int EPI, int DH>
__global__ void __launch_bounds__(256) splitk_finalize_kernel(const float* __restrict__ part, int splits, int M,
                                                              int N, GemmEpi ep) {
  pdl_trigger();
  pdl_wait();
  const int row = blockIdx.x;
  const long long slab = (long long)M * N;
  const float* pr = part + (long long)row * N;
  // splits summed in order (deterministic); unrolled so the partial loads are in flight together
  auto sum4 = [&](int col) {
    float4 s = *reinterpret_cast<const float4*>(pr + col);
#pragma unroll 4
    for (int k = 1; k < splits; ++k) {
      const float4 t = *reinterpret_cast<const float4*>(pr + k * slab + col);
      s.x += t.x;
      s.y += t.y;
      s.z += t.z;
      s.w += t.w;
    }
    return s;
  };
  // RMSNorm fused across GEMMs (QKV / SwiGLU consumers): this row's rsqrt, reduced once per
  // CTA from the producer's per-chunk sums of squares (fixed order: deterministic)
  float rs = 1.f;
  if constexpr (EPI == EPI_QKV || EPI == EPI_SWIGLU) {
    if (ep.ssq_in) {
      __shared__ float red[8];
      float v = 0.f;
      for (int c = threadIdx.x; c < ep.ssq_parts; c += blockDim.x) v += ep.ssq_in[(long long)c * M + row];
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
      __syncthreads();
      float t = 0.f;
#pragma unroll
      for (int w = 0; w < 8; ++w) t += red[w];
      rs = rsqrtf(t / (float)ep.ssq_dim + ep.norm_eps);
    }
  }
  if constexpr (EPI == EPI_QKV) {
    // one warp per head (8 heads per CTA); lane owns elements lane + 32k, so RoPE
    // pairs (i, i + DH/2) stay in-lane
    constexpr int PER = DH / 32;
    const int g = blockIdx.y * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (g >= N / DH) return;
    const int p = ep.pos[row], sl = ep.slot[row];
    float v[PER];
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int col = g * DH + lane + 32 * k;
      float t = pr[col];
#pragma unroll 4
      for (int q = 1; q < splits; ++q) t += pr[q * slab + col];
      v[k] = t * rs;
    }
    if (g < ep.hq + ep.hkv) {
      const float2* cs = reinterpret_cast<const float2*>(ep.rope) + (long long)p * (DH / 2);
#pragma unroll
      for (int k = 0; k < PER / 2; ++k) {
        const float2 t = cs[lane + 32 * k];
        const float x1 = v[k], x2 = v[k + PER / 2];
        v[k] = x1 * t.x - x2 * t.y;
        v[k + PER / 2] = x2 * t.x + x1 * t.y;
      }
    }
    __nv_bfloat16* dst;
    if (g < ep.hq)
      dst = ep.q + (long long)row * ep.ldq + (long long)g * DH;
    else if (g < ep.hq + ep.hkv)
      dst = ep.kplane + (long long)(g - ep.hq) * ep.head_stride + (long long)sl * DH;
    else
      dst = ep.vplane + (long long)(g - ep.hq - ep.hkv) * ep.head_stride + (long long)sl * DH;
#pragma unroll
    for (int k = 0; k < PER; ++k) dst[lane + 32 * k] = __float2bfloat16(v[k]);
  } else if constexpr (EPI == EPI_SWIGLU) {
    const int j = (blockIdx.y * 256 + threadIdx.x) * 4;  // 4 outputs inside one 64-block
    if (j >= N / 2) return;
    const int gc = (j / 64) * 128 + (j % 64);
    float4 g = sum4(gc), u = sum4(gc + 64);
    if (ep.ssq_in) {
      g = make_float4(g.x * rs, g.y * rs, g.z * rs, g.w * rs);
      u = make_float4(u.x * rs, u.y * rs, u.z * rs, u.w * rs);
    }
    uint2 w;
    w.x = pack_bf16(silu(g.x) * u.x, silu(g.y) * u.y);
    w.y = pack_bf16(silu(g.z) * u.z, silu(g.w) * u.w);
    *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(ep.out) + (long long)row * ep.ldo + j) = w;
  } else {
    const int j = (blockIdx.y * 256 + threadIdx.x) * 4;
    if (EPI != EPI_RESID && j >= N) return;  // RESID: every lane joins the chunk sums below
    float4 s = j < N ? sum4(j) : make_float4(0.f, 0.f, 0.f, 0.f);
    if constexpr (EPI == EPI_STORE_F32) {
      *reinterpret_cast<float4*>(static_cast<float*>(ep.out) + (long long)row * ep.ldo + j) = s;
    } else {
      if constexpr (EPI == EPI_RESID) {
        const uint2 r = *reinterpret_cast<const uint2*>(ep.resid + (long long)row * ep.ldr + j);
        const float2 a = unpack_bf16(r.x), b = unpack_bf16(r.y);
        s.x += a.x;
        s.y += a.y;
        s.z += b.x;
        s.w += b.y;
      }
      uint2 w;
      w.x = pack_bf16(s.x, s.y);
      w.y = pack_bf16(s.z, s.w);
      if constexpr (EPI == EPI_PUSH) {
        for (int p = 0; p < ep.npush; ++p) *reinterpret_cast<uint2*>(ep.push[p] + (long long)row * ep.ldo + j) = w;
        __threadfence_system();
      } else {
        if (j < N) *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(ep.out) + (long long)row * ep.ldo + j) = w;
        if constexpr (EPI == EPI_RESID) {
          if (ep.ssq_out) {  // the next RMSNorm's statistics: per 32-column chunk (8 lanes), bf16 outputs
            const float2 p0 = unpack_bf16(w.x), p1 = unpack_bf16(w.y);
            float ss = j < N ? (p0.x * p0.x + p0.y * p0.y) + (p1.x * p1.x + p1.y * p1.y) : 0.f;
            ss += __shfl_xor_sync(0xffffffffu, ss, 1);
            ss += __shfl_xor_sync(0xffffffffu, ss, 2);
            ss += __shfl_xor_sync(0xffffffffu, ss, 4);
            if ((threadIdx.x & 7) == 0 && j < N) ep.ssq_out[(long long)(j >> 5) * M + row] = ss;
          }
        }
      }
    }
  }
}

// RESID finalize with the following RMSNorm fused in (one CTA per row, N <= 8192):
// x = resid + sum(partials) -> bf16 -> out; h = x * rsqrt(mean(x^2) + eps) * gain -> norm_out.
// 1024 threads x <= 2 float4 chunks; every split's partial of a chunk is requested before
// any is summed (a decode step has only M = 16 rows = 16 CTAs: the kernel is latency-bound,
// so the loads must all be in flight at once), summed in split order (deterministic).
constexpr int RN_THREADS = 1024, RN_MAXC = 2, RN_G = 4;
__global__ void __launch_bounds__(RN_THREADS) splitk_resid_norm_kernel(const float* __restrict__ part, int splits,
                                                                       int M, int N, GemmEpi ep) {
  pdl_trigger();
  pdl_wait();
  const int row = blockIdx.x;
  const long long slab = (long long)M * N;
  const float* pr = part + (long long)row * N;
  float xs[RN_MAXC][4];
  float ss = 0.f;
  float4 t[RN_MAXC];
  uint2 rr[RN_MAXC];
#pragma unroll
  for (int c = 0; c < RN_MAXC; ++c) {
    const int j = (c * RN_THREADS + threadIdx.x) * 4;
    t[c] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (j < N) rr[c] = *reinterpret_cast<const uint2*>(ep.resid + (long long)row * ep.ldr + j);
  }
  for (int k0 = 0; k0 < splits; k0 += RN_G) {  // RN_G splits x every chunk in flight per round
    float4 u[RN_MAXC][RN_G];
#pragma unroll
    for (int c = 0; c < RN_MAXC; ++c) {
      const int j = (c * RN_THREADS + threadIdx.x) * 4;
#pragma unroll
      for (int g = 0; g < RN_G; ++g)
        if (j < N && k0 + g < splits) u[c][g] = __ldcg(reinterpret_cast<const float4*>(pr + (k0 + g) * slab + j));
    }
#pragma unroll
    for (int c = 0; c < RN_MAXC; ++c)
#pragma unroll
      for (int g = 0; g < RN_G; ++g)
        if (k0 + g < splits) {  // split order: bit-identical to a serial sum
          t[c].x += u[c][g].x;
          t[c].y += u[c][g].y;
          t[c].z += u[c][g].z;
          t[c].w += u[c][g].w;
        }
  }
#pragma unroll
  for (int c = 0; c < RN_MAXC; ++c) {
    const int j = (c * RN_THREADS + threadIdx.x) * 4;
    if (j < N) {
      const float2 a = unpack_bf16(rr[c].x), b = unpack_bf16(rr[c].y);
      uint2 w;
      w.x = pack_bf16(t[c].x + a.x, t[c].y + a.y);
      w.y = pack_bf16(t[c].z + b.x, t[c].w + b.y);
      *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(ep.out) + (long long)row * ep.ldo + j) = w;
      const float2 p0 = unpack_bf16(w.x), p1 = unpack_bf16(w.y);  // normalise the rounded residual
      xs[c][0] = p0.x;
      xs[c][1] = p0.y;
      xs[c][2] = p1.x;
      xs[c][3] = p1.y;
      ss += p0.x * p0.x + p0.y * p0.y + p1.x * p1.x + p1.y * p1.y;
    }
  }
  __shared__ float red[RN_THREADS / 32];
  for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffff, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  float tot = 0.f;
#pragma unroll
  for (int w = 0; w < RN_THREADS / 32; ++w) tot += red[w];
  const float inv = rsqrtf(tot / (float)N + ep.norm_eps);
#pragma unroll
  for (int c = 0; c < RN_MAXC; ++c) {
    const int j = (c * RN_THREADS + threadIdx.x) * 4;
    if (j < N) {
      const float4 g = *reinterpret_cast<const float4*>(ep.norm_gain + j);
      uint2 w;
      w.x = pack_bf16(xs[c][0] * inv * g.x, xs[c][1] * inv * g.y);
      w.y = pack_bf16(xs[c][2] * inv * g.z, xs[c][3] * inv * g.w);
      *reinterpret_cast<uint2*>(ep.norm_out + (long long)row * N + j) = w;
    }
  }
}

template <int BN, int EPI, int DH>
int launch_impl(const CUtensorMap& ta, const CUtensorMap& tb, int M, int N, int K, int splits, const GemmEpi& ep,
                cudaStream_t stream) {
  using C = GemmCfg<BN>;
  auto kern = gemm_bf16_tc_kernel<BN, EPI, DH>;
  static bool attr_set = false;  // per template instance
  if (!attr_set) {
    CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
    attr_set = true;
  }
  const int units = ((M + BM - 1) / BM) * ((N + BN - 1) / BN) * splits;
  const int grid = units < num_sms() ? units : num_sms();
  CUDA_TRY(launch_k(kern, dim3(grid), dim3(GEMM_THREADS), C::SMEM, stream, ta, tb, M, N, K, splits, ep));
  CUDA_TRY(cudaGetLastError());
  return 0;
}

template <int EPI, int DH>
int launch_finalize(const float* part, int splits, int M, int N, const GemmEpi& ep, cudaStream_t stream) {
  int gy;
  if (EPI == EPI_QKV) gy = (N / (DH ? DH : 1) + 7) / 8;
  else if (EPI == EPI_SWIGLU) gy = (N / 2 + 1023) / 1024;
  else gy = (N + 1023) / 1024;
  CUDA_TRY(launch_k(splitk_finalize_kernel<EPI, DH>, dim3(M, gy), dim3(256), 0, stream, part, splits, M, N, ep));
  CUDA_TRY(cudaGetLastError());
  return 0;
}

}  // namespace

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2-D bf16 K-major operand map: dims {K, rows}, box {64, box_rows}, 128-B swizzle.
int make_tmap(CUtensorMap* m, const void* base, long long rows, long long K, long long ld, int box_rows) {
  auto fn = encode_fn();
  if (!fn) return set_error(RDKV_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(RDKV_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return 0;
}

// Tile-N choice: fewer, larger tiles are cheaper per FLOP (smem traffic per MMA
// drops from 128 to 96 B/clk) but quantise worse on 148 SMs; estimate both.
int pick_bn(int M, int N) {
  const int m_tiles = (M + BM - 1) / BM, sms = num_sms();
  auto cost = [&](int bn, double eff) {
    const long long tiles = (long long)m_tiles * ((N + bn - 1) / bn);
    return (double)((tiles + sms - 1) / sms) * bn * eff;
  };
  return cost(256, 1.0) <= cost(128, 1.15) ? 256 : 128;
}

// K splits for a GEMM whose tiles cannot fill the SMs (small M): enough units
// for ~one wave, at least 4 k-blocks per split.
int pick_splits(int M, int N, int K, int bn) {
  const int tiles = ((M + BM - 1) / BM) * ((N + bn - 1) / bn), sms = num_sms();
  const int kblocks = K / BK;
  if (tiles * 2 > sms || kblocks < 8) return 1;
  int s = (sms + tiles - 1) / tiles;
  s = s < kblocks / 4 ? s : kblocks / 4;
  if (s < 2) return 1;
  const int kb_per = (kblocks + s - 1) / s;  // make every split non-empty
  return (kblocks + kb_per - 1) / kb_per;
}

// Small-M plan: <= 128 tokens make every layer GEMM weight-bandwidth bound.  Run
// it swap-AB (weights = 128-row A operand, tokens = UMMA N) with enough K splits
// for about one wave; fp32 partials are reduced by splitk_finalize, which also
// applies the fused epilogue.
struct SplitPlan {
  int nt, splits;  // token tile (0 = not small-M) and K splits
};
SplitPlan pick_split_plan(int M, int N, int K) {
  if (M > 128 || K % BK) return {0, 1};
  const int nt = M <= 16 ? 16 : M <= 32 ? 32 : M <= 64 ? 64 : 128;
  const int sms = num_sms() * ((RDKV_SWAPAB_2CTA && nt <= RDKV_SWAPAB_2CTA_MAXNT) ? 2 : 1), kblocks = K / BK,
            w_tiles = (N + 127) / 128;
  int s = w_tiles >= sms ? 1 : sms / w_tiles;
  s = s < kblocks / 4 ? s : kblocks / 4;
  if (s < 1) s = 1;
  const int kb_per = (kblocks + s - 1) / s;
  return {nt, (kblocks + kb_per - 1) / kb_per};
}

bool gemm_splits(int M, int N, int K, size_t splitk_bytes) {
  const SplitPlan sp = pick_split_plan(M, N, K);
  return sp.nt > 0 && (size_t)sp.splits * M * N * sizeof(float) <= splitk_bytes;
}

size_t splitk_scratch_bytes(int M, int N, int K) {
  const SplitPlan sp = pick_split_plan(M, N, K);
  return sp.nt > 0 ? (size_t)sp.splits * M * N * sizeof(float) : 0;
}

// RDKV_GEMM_SK: stream-K for the CTA-pair GEMM — 1: only grids that leave pairs idle
// (single-wave projections at M = 1024: 64 tiles on 74 pairs), 2: any grid whose last
// round is partial, 3: whole tiles for the full rounds and only the partial last round's
// tiles split in k (gate/up at M = 1024: 448 tiles = 6 x 74 + 4).  0 (default): whole tiles.
int gemm_sk_mode() {
  static const int m = [] {
    const char* e = std::getenv("RDKV_GEMM_SK");
    return e ? std::atoi(e) : 0;
  }();
  return m;
}

size_t gemm_sk_scratch_bytes() {
  const size_t slots = (size_t)num_sms();  // two per pair
  return slots * 128 * 384 * sizeof(float) + slots * sizeof(int);
}

namespace {

// Sum `splits` fp32 partial slabs and apply the requested epilogue.
int finalize(int kind, int dh, const float* part, int splits, int M, int N, const GemmEpi& ep, cudaStream_t stream) {
  switch (kind) {
    case EPI_STORE: return launch_finalize<EPI_STORE, 0>(part, splits, M, N, ep, stream);
    case EPI_STORE_F32: return launch_finalize<EPI_STORE_F32, 0>(part, splits, M, N, ep, stream);
    case EPI_RESID:
      if (ep.norm_out) {
        if (N > RN_THREADS * RN_MAXC * 4 || N % 4)
          return set_error(RDKV_ERR_ARG, "resid+norm finalize: N must be <= 8192, %% 4");
        CUDA_TRY(launch_k(splitk_resid_norm_kernel, dim3(M), dim3(RN_THREADS), 0, stream, part, splits, M, N, ep));
        return 0;
      }
      return launch_finalize<EPI_RESID, 0>(part, splits, M, N, ep, stream);
    case EPI_SWIGLU: return launch_finalize<EPI_SWIGLU, 0>(part, splits, M, N, ep, stream);
    case EPI_PUSH: return launch_finalize<EPI_PUSH, 0>(part, splits, M, N, ep, stream);
    case EPI_QKV:
      if (dh == 64) return launch_finalize<EPI_QKV, 64>(part, splits, M, N, ep, stream);
      if (dh == 128) return launch_finalize<EPI_QKV, 128>(part, splits, M, N, ep, stream);
      return set_error(RDKV_ERR_ARG, "qkv: head_dim %d unsupported (64 or 128)", dh);
    default: return set_error(RDKV_ERR_ARG, "gemm: unknown epilogue %d", kind);
  }
}

int launch_small_m(const __nv_bfloat16* A, long long lda, const __nv_bfloat16* B, long long ldb, int M, int N, int K,
                   int kind, int dh, const GemmEpi& ep, cudaStream_t stream, SplitPlan sp) {
  CUtensorMap tw, tx;
  RDKV_TRY(make_tmap(&tw, B, N, K, ldb, 128));
  RDKV_TRY(make_tmap(&tx, A, M, K, lda, sp.nt));
  auto* part = static_cast<float*>(ep.splitk_ws);
  // fused split-K (no finalize kernel) for every epilogue that works per 128-column tile: not
  // the row-wide resid+norm finalize (norm_out) nor the tensor-parallel push
  const int w_tiles = (N + 127) / 128;
  const bool fuse = ep.counters && w_tiles <= ep.n_counters && !(kind == EPI_RESID && ep.norm_out) &&
                    kind != EPI_PUSH && (kind != EPI_QKV || dh == 64 || dh == 128);
  if (fuse) {
    auto go = [&](auto nt) -> int {
      constexpr int NT = decltype(nt)::value;
      switch (kind) {
        case EPI_STORE: return launch_swapab<NT, EPI_STORE, 0>(tw, tx, M, N, K, sp.splits, part, ep, stream);
        case EPI_STORE_F32: return launch_swapab<NT, EPI_STORE_F32, 0>(tw, tx, M, N, K, sp.splits, part, ep, stream);
        case EPI_RESID: return launch_swapab<NT, EPI_RESID, 0>(tw, tx, M, N, K, sp.splits, part, ep, stream);
        case EPI_SWIGLU: return launch_swapab<NT, EPI_SWIGLU, 0>(tw, tx, M, N, K, sp.splits, part, ep, stream);
        case EPI_QKV:
          if (dh == 64) return launch_swapab<NT, EPI_QKV, 64>(tw, tx, M, N, K, sp.splits, part, ep, stream);
          return launch_swapab<NT, EPI_QKV, 128>(tw, tx, M, N, K, sp.splits, part, ep, stream);
        default: return set_error(RDKV_ERR_ARG, "gemm: unknown epilogue %d", kind);
      }
    };
    switch (sp.nt) {
      case 16: return go(std::integral_constant<int, 16>{});
      case 32: return go(std::integral_constant<int, 32>{});
      case 64: return go(std::integral_constant<int, 64>{});
      default: return go(std::integral_constant<int, 128>{});
    }
  }
  switch (sp.nt) {
    case 16: RDKV_TRY(launch_swapab<16>(tw, tx, M, N, K, sp.splits, part, ep, stream)); break;
    case 32: RDKV_TRY(launch_swapab<32>(tw, tx, M, N, K, sp.splits, part, ep, stream)); break;
    case 64: RDKV_TRY(launch_swapab<64>(tw, tx, M, N, K, sp.splits, part, ep, stream)); break;
    default: RDKV_TRY(launch_swapab<128>(tw, tx, M, N, K, sp.splits, part, ep, stream)); break;
  }
  return finalize(kind, dh, part, sp.splits, M, N, ep, stream);
}

}  // namespace

template <int BN>
int dispatch(const __nv_bfloat16* A, long long lda, const __nv_bfloat16* B, long long ldb, int M, int N, int K,
             int kind, int dh, const GemmEpi& ep, cudaStream_t stream, int splits) {
  CUtensorMap ta, tb;
  RDKV_TRY(make_tmap(&ta, A, M, K, lda, BM));
  RDKV_TRY(make_tmap(&tb, B, N, K, ldb, BN));
  if (splits > 1) {
    GemmEpi pe = ep;
    pe.out = ep.splitk_ws;
    RDKV_TRY((launch_impl<BN, EPI_PARTIAL, 0>(ta, tb, M, N, K, splits, pe, stream)));
    return finalize(kind, dh, static_cast<const float*>(ep.splitk_ws), splits, M, N, ep, stream);
  }
  switch (kind) {
    case EPI_STORE: return launch_impl<BN, EPI_STORE, 0>(ta, tb, M, N, K, 1, ep, stream);
    case EPI_STORE_F32: return launch_impl<BN, EPI_STORE_F32, 0>(ta, tb, M, N, K, 1, ep, stream);
    case EPI_RESID: return launch_impl<BN, EPI_RESID, 0>(ta, tb, M, N, K, 1, ep, stream);
    case EPI_SWIGLU: return launch_impl<BN, EPI_SWIGLU, 0>(ta, tb, M, N, K, 1, ep, stream);
    case EPI_PUSH: return launch_impl<BN, EPI_PUSH, 0>(ta, tb, M, N, K, 1, ep, stream);
    case EPI_QKV:
      if (dh == 64) return launch_impl<BN, EPI_QKV, 64>(ta, tb, M, N, K, 1, ep, stream);
      if (dh == 128) return launch_impl<BN, EPI_QKV, 128>(ta, tb, M, N, K, 1, ep, stream);
      return set_error(RDKV_ERR_ARG, "qkv: head_dim %d unsupported (64 or 128)", dh);
    default: return set_error(RDKV_ERR_ARG, "gemm: unknown epilogue %d", kind);
  }
}

// Co-resident 2-CTA clusters of the pair kernel (all of them must be, for stream-K).
template <int BN, int EPI, int DH>
int sk_resident_pairs() {
  static int n = -1;
  if (n < 0) {
    auto kern = gemm_bf16_tc2_kernel<BN, EPI, DH, true>;
    constexpr size_t SMEM = PairCfg<BN>::SMEM;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM) != cudaSuccess ||
        cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 0) != cudaSuccess) {
      n = 0;
      return n;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(num_sms());
    cfg.blockDim = dim3(GEMM_THREADS);
    cfg.dynamicSmemBytes = SMEM;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int c = 0;
    n = cudaOccupancyMaxActiveClusters(&c, kern, &cfg) == cudaSuccess ? std::min(c, num_sms() / 2) : 0;
    cudaGetLastError();
  }
  return n;
}

// RDKV_GEMM_MC: B-tile TMA multicast across two CTA pairs (clusters of 4) for 256 x 256 pair
// tiles with an even number of M tiles — 1: every such grid, 2: only multi-wave grids, 3: only
// single-wave grids (units <= the pairs).  0: off.  Default 2 (C3 step, 5 interleaved pairs:
// gate/up -3%, 1034 vs 1023 q/s, profiles/r2s4_gemm_mc_ab.txt).
int gemm_mc_mode() {
  static const int m = [] {
    const char* e = std::getenv("RDKV_GEMM_MC");
    return e ? std::atoi(e) : 2;
  }();
  return m;
}
template <int BN>
bool use_mc(int M, int N, int kind) {
  const int mode = gemm_mc_mode(), m_tiles = (M + 255) / 256, units = m_tiles * ((N + BN - 1) / BN);
  const bool multi = units > num_sms() / 2;
  return BN == 256 && mode > 0 && kind != EPI_PUSH && m_tiles % 2 == 0 && (mode == 1 || (mode == 2) == multi);
}

template <int BN, int EPI, int DH>
int launch_pair_auto(const CUtensorMap& ta, const CUtensorMap& tb, int M, int N, int K, const GemmEpi& ep,
                     cudaStream_t stream) {
  if constexpr (BN == 256)
    if (use_mc<BN>(M, N, EPI)) return launch_pair<BN, EPI, DH, false, true>(ta, tb, M, N, K, ep, stream);
  const int mode = gemm_sk_mode();
  if (mode > 0 && EPI != EPI_PUSH && ep.sk_part && ep.sk_flag) {
    const int units = ((M + 255) / 256) * ((N + BN - 1) / BN), kblocks = K / BK;
    const int P = sk_resident_pairs<BN, EPI, DH>();
    const bool partial = P > 0 && units % P != 0 && (mode >= 2 || units < P);
    if (mode == 3) {
      // whole tiles for the full rounds; the last round's `tail` tiles each split in k over
      // s pairs (s - 1 fp32 partial tiles added by the first), so the round costs ~1/s
      const int tail = P > 0 ? units % P : 0;
      static const int smax = [] {
        const char* e = std::getenv("RDKV_GEMM_SK_SPLIT");
        return e ? std::max(1, std::atoi(e)) : 4;
      }();
      const int s = tail ? std::min(smax, P / tail) : 0;
      if (units > P && s >= 2 && kblocks >= 4 * s && 2 * P <= ep.sk_slots) {
        GemmEpi e = ep;
        e.sk_dp = units - tail;
        e.sk_tp = tail * s;
        return launch_pair<BN, EPI, DH, true>(ta, tb, M, N, K, e, stream, P);
      }
    } else if (partial && (long long)units * kblocks >= 8ll * P && 2 * P <= ep.sk_slots) {
      GemmEpi e = ep;
      e.sk_dp = 0;
      e.sk_tp = P;
      return launch_pair<BN, EPI, DH, true>(ta, tb, M, N, K, e, stream, P);
    }
  }
  return launch_pair<BN, EPI, DH>(ta, tb, M, N, K, ep, stream);
}

template <int BN>
int dispatch_pair(const __nv_bfloat16* A, long long lda, const __nv_bfloat16* B, long long ldb, int M, int N, int K,
                  int kind, int dh, const GemmEpi& ep, cudaStream_t stream) {
  CUtensorMap ta, tb;
  RDKV_TRY(make_tmap(&ta, A, M, K, lda, 128));
  RDKV_TRY(make_tmap(&tb, B, N, K, ldb, BN == 384 ? 64 : use_mc<BN>(M, N, kind) ? BN / 4 : BN / 2));
  switch (kind) {
    case EPI_STORE: return launch_pair_auto<BN, EPI_STORE, 0>(ta, tb, M, N, K, ep, stream);
    case EPI_STORE_F32: return launch_pair_auto<BN, EPI_STORE_F32, 0>(ta, tb, M, N, K, ep, stream);
    case EPI_RESID: return launch_pair_auto<BN, EPI_RESID, 0>(ta, tb, M, N, K, ep, stream);
    case EPI_SWIGLU:
      if constexpr (BN % 128 == 0) return launch_pair_auto<BN, EPI_SWIGLU, 0>(ta, tb, M, N, K, ep, stream);
      return set_error(RDKV_ERR_ARG, "swiglu: tile N %d must hold whole gate/up block pairs", BN);
    case EPI_PUSH: return launch_pair<BN, EPI_PUSH, 0>(ta, tb, M, N, K, ep, stream);
    case EPI_QKV:
      if (dh == 64) return launch_pair_auto<BN, EPI_QKV, 64>(ta, tb, M, N, K, ep, stream);
      if constexpr (BN % 128 == 0)
        if (dh == 128) return launch_pair_auto<BN, EPI_QKV, 128>(ta, tb, M, N, K, ep, stream);
      return set_error(RDKV_ERR_ARG, "qkv: head_dim %d unsupported with tile N %d", dh, BN);
    default: return set_error(RDKV_ERR_ARG, "gemm: unknown epilogue %d", kind);
  }
}

// Tile plan for the unsplit path: {1-CTA 128x128, 1-CTA 128x256, pair 256x256},
// cost = waves x per-SM tile work / efficiency.  Efficiencies are the measured
// tensor-pipe ceilings set by L2->SM operand traffic per FLOP.
struct TilePlan {
  bool pair;
  int bn;
};
bool pairs_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("RDKV_GEMM_PAIRS");
    return !(e && e[0] == '0');
  }();
  return on;
}
TilePlan pick_tiles(int M, int N, int K, bool allow192) {
  const int sms = num_sms();
  struct Cand {
    bool pair;
    int bn;
    double eff;
  } cands[5] = {{false, 128, 0.60}, {false, 256, 0.83}, {true, 256, 0.975}, {true, 192, 0.95}, {true, 384, 0.975}};
  // Cost = waves x k-blocks x tile width / efficiency + a per-kernel fixed cost (prologue,
  // pipeline fill, the last tile's exposed epilogue), calibrated with scripts/gemm_tiles.py:
  // at N = 2048 single-CTA 128x256 tiles take 15.2 / 52.3 us for K = 2048 / 8192 and
  // 256x256 CTA pairs 16.3 / 47.9 us -> pairs stream k-blocks ~18% faster but pay ~3 us
  // more of fixed cost (cluster launch, 2-SM TMEM allocation and barriers), so short-K
  // single-wave GEMMs (the O projection) run on single CTAs.  The 256 x 128 CTA-pair tile
  // measured slower than both neighbours and is only reachable explicitly (tile_n = 384).
  // 256 x 192 pairs fit N = 3072 into 128 tiles (not for SwiGLU, whose tiles hold gate/up
  // 64-column block pairs, nor for 128-wide heads); 256 x 384 pairs (one accumulator) only
  // when every pair gets at most one tile.
  constexpr double F_SINGLE = 2255.0, F_PAIR = 4597.0;  // in (k-block x 256 / 0.83) units ~ 1.25 ns
  const double kb = K / (double)BK;
  double best = 1e30;
  TilePlan plan{false, 256};
  for (const Cand& c : cands) {
    if (c.pair && (M < 256 || !pairs_enabled())) continue;
    if (c.bn == 192 && (!allow192 || N % 192)) continue;
    static const bool allow384 = [] {
      const char* e = std::getenv("RDKV_GEMM_384");  // "0": no 256 x 384 pair tiles (A/B)
      return !(e && e[0] == '0');
    }();
    if (c.bn == 384 && (!allow384 || N % 384 || (long long)((M + 255) / 256) * (N / 384) > sms / 2)) continue;
    const int rows = c.pair ? 256 : 128;
    const long long units = (long long)((M + rows - 1) / rows) * ((N + c.bn - 1) / c.bn);
    const int slots = c.pair ? sms / 2 : sms;
    const double t = (double)((units + slots - 1) / slots) * kb * c.bn / c.eff + (c.pair ? F_PAIR : F_SINGLE);
    if (t < best - 1e-9) {
      best = t;
      plan = {c.pair, c.bn};
    }
  }
  return plan;
}

#ifndef RDKV_GEMM_PF_DEFAULT
#define RDKV_GEMM_PF_DEFAULT 0
#endif
int launch_gemm(const __nv_bfloat16* A, long long lda, const __nv_bfloat16* B, long long ldb, int M, int N, int K,
                int kind, int dh, const GemmEpi& ep_in, cudaStream_t stream, int bn) {
  // opt-in A/B knobs, measured no faster inside the C3 step (profiles/r2_l2_prefetch_ab.txt):
  // RDKV_GEMM_WPOL=1 streams the weights evict-first, RDKV_L2_PREFETCH=1 lets the idle
  // warp pull the next projection's weights into L2
  static const int wpol = [] {
    const char* e = std::getenv("RDKV_GEMM_WPOL");
    return e && e[0] == '1' ? 1 : 0;
  }();
  static const bool l2pf = [] {
    const char* e = std::getenv("RDKV_L2_PREFETCH");
    return e && e[0] == '1';
  }();
  static const int b_pf = [] {
    const char* e = std::getenv("RDKV_GEMM_PF");  // weight L2 prefetch distance in k-blocks
    return e ? std::atoi(e) : RDKV_GEMM_PF_DEFAULT;
  }();
  GemmEpi ep = ep_in;
  ep.w_policy = wpol;
  ep.b_pf = b_pf;
  // RDKV_SMALLM_L2PF=all: on the small-M (split-K swap-AB) path the idle warp pulls the next
  // projection's weights into L2 (gate/up -> w_down, down -> next w_qkv).  Measured slower
  // (single-query TTFT 4.50 -> 5.09 ms, decode step 5.20 -> 5.68 ms: the prefetch competes with
  // the weight stream it is meant to hide); off.  Large M only with RDKV_L2_PREFETCH=1.
  static const bool small_l2pf = [] {
    const char* e = std::getenv("RDKV_SMALLM_L2PF");
    return e && e[0] == 'a';
  }();
  if (!l2pf && !(small_l2pf && M <= 128)) ep.l2_next = nullptr;
  if (M <= 0 || N <= 0) return 0;
  if (K <= 0 || K % BK != 0) return set_error(RDKV_ERR_ARG, "gemm: K=%d must be a positive multiple of 64", K);
  if (N % 32 != 0) return set_error(RDKV_ERR_ARG, "gemm: N=%d must be a multiple of 32", N);
  if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15)
    return set_error(RDKV_ERR_ARG, "gemm: operands must be 16-byte aligned");
  if ((lda | ldb) & 7) return set_error(RDKV_ERR_ARG, "gemm: leading dims must be multiples of 8");
  if (bn != 0 && bn != 128 && bn != 256 && bn != 384 && bn != 512 && bn != 640)
    return set_error(RDKV_ERR_ARG, "gemm: tile N %d must be 128, 256 (or 384/512/640 for CTA pairs)", bn);
  if (kind == EPI_SWIGLU && N % 128 != 0) return set_error(RDKV_ERR_ARG, "swiglu: N must be a multiple of 128");
  int splits = 1;
  if (ep.splitk_ws) {
    if (bn == 0) {
      const SplitPlan sp = pick_split_plan(M, N, K);
      if (sp.nt > 0 && (size_t)sp.splits * M * N * sizeof(float) <= ep.splitk_bytes)
        return launch_small_m(A, lda, B, ldb, M, N, K, kind, dh, ep, stream, sp);
    } else {  // explicit tile width (tests): split-K with that tile when it would help
      splits = pick_splits(M, N, K, bn);
      if ((size_t)splits * M * N * sizeof(float) > ep.splitk_bytes) splits = 1;
    }
  }
  if (bn == 0 && splits == 1) {
    static const bool allow192_env = [] {
      const char* e = std::getenv("RDKV_GEMM_192");  // "0": no 256 x 192 pair tiles (A/B)
      return !(e && e[0] == '0');
    }();
    const bool allow192 = allow192_env && kind != EPI_SWIGLU && !(kind == EPI_QKV && dh != 64);
    const TilePlan tp = pick_tiles(M, N, K, allow192);
    if (tp.pair && !(kind == EPI_SWIGLU && N % tp.bn != 0)) {
      if (tp.bn == 128) return dispatch_pair<128>(A, lda, B, ldb, M, N, K, kind, dh, ep, stream);
      if (tp.bn == 192) return dispatch_pair<192>(A, lda, B, ldb, M, N, K, kind, dh, ep, stream);
      if (tp.bn == 384) return dispatch_pair<384>(A, lda, B, ldb, M, N, K, kind, dh, ep, stream);
      // RDKV_GEMM_TAIL=1: a last round that holds only the final column of 256-wide tiles
      // (gate/up at M = 1024: 448 tiles on 74 pairs, the 7th round has 4) runs as its own launch
      // of 256 x 128 tiles.  Correct, measured slower (gate/up 169.8 -> 175.1 us alone, 6.03 ->
      // 6.29 ms per C3 step: the second launch's ramp costs more than the half round it saves).
      static const bool tail_env = [] {
        const char* e = std::getenv("RDKV_GEMM_TAIL");
        return e && e[0] == '1';
      }();
      const int m_t = (M + 255) / 256, n_t = N / 256, npairs = num_sms() / 2;
      const int units = m_t * n_t, rem = units % npairs;
      if (tail_env && (kind == EPI_SWIGLU || kind == EPI_STORE) && N % 256 == 0 && units > npairs && rem > 0 &&
          rem <= m_t && (units - m_t) % npairs == 0) {
        const int n_main = N - 256;
        RDKV_TRY(dispatch_pair<256>(A, lda, B, ldb, M, n_main, K, kind, dh, ep, stream));
        GemmEpi et = ep;  // the last 256 output columns (128 for SwiGLU): shifted B rows and output
        et.out = static_cast<__nv_bfloat16*>(ep.out) + (kind == EPI_SWIGLU ? n_main / 2 : n_main);
        return dispatch_pair<128>(A, lda, B + (long long)n_main * ldb, ldb, M, 256, K, kind, dh, et, stream);
      }
      return dispatch_pair<256>(A, lda, B, ldb, M, N, K, kind, dh, ep, stream);
    }
    bn = tp.bn;
  }
  if (bn == 512 || bn == 384 || bn == 640) {  // explicit CTA-pair request (tests): 512 -> 256 x 256, 384 -> 256 x 128,
    // 640 -> 256 x 384 (one accumulator)
    if (M < 256) return set_error(RDKV_ERR_ARG, "gemm: CTA-pair tiles need M >= 256");
    if (bn == 384) return dispatch_pair<128>(A, lda, B, ldb, M, N, K, kind, dh, ep, stream);
    if (bn == 640) {
      if (N % 384) return set_error(RDKV_ERR_ARG, "gemm: 256 x 384 tiles need N %% 384 == 0");
      return dispatch_pair<384>(A, lda, B, ldb, M, N, K, kind, dh, ep, stream);
    }
    return dispatch_pair<256>(A, lda, B, ldb, M, N, K, kind, dh, ep, stream);
  }
  if (bn == 0) bn = pick_bn(M, N);
  if (kind == EPI_SWIGLU && N % bn != 0) bn = 128;
  if (bn == 128) return dispatch<128>(A, lda, B, ldb, M, N, K, kind, dh, ep, stream, splits);
  return dispatch<256>(A, lda, B, ldb, M, N, K, kind, dh, ep, stream, splits);
}

}  // namespace rdkv
