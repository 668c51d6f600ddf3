// K2/K4 on the 5th-generation tensor cores: causal prefill attention over a
// (possibly cached) KV prefix with grouped-query packing.
//
// Semantics are those of attention.cu (reference: cached_prefill_work,
// costs.py:89-99 — new tokens at positions [n_cached, n_cached+n_new) attend
// over every position <= their own).  A Q tile is 128 query rows of ONE kv
// head, row r = (token t0 + r / G, q-head kvh*G + r % G), so the G query heads
// sharing a K/V head read each K/V tile once.  A CTA owns TWO consecutive Q
// tiles (for G = 4: 64 query tokens = a whole C2 query) that share every K/V
// tile the TMA brings in.
//
// Warp roles (320 threads, one CTA per SM):
//   warps 0-3   softmax of Q tile 0, warps 4-7 softmax of Q tile 1: one query
//               row per thread (= one TMEM lane).  Per KV tile: tcgen05.ld the
//               128 scores, mask, row max (FMNMX3), P = 2^(s*scale - m) with
//               packed FFMA2 + MUFU ex2, tcgen05.st of P (bf16 pairs) into TMEM.
//               The row max is moved lazily (only when it grows by > 2^8), and
//               only then is the O row in TMEM rescaled.  The two warpgroups
//               run independently, so one's exp2 overlaps the other's loads.
//   warp 8      TMA producer: K and V tiles of 128 positions (two 64-row boxes
//               each, one per KV block of the paged pool / blob), STAGES-deep
//               smem ring, 128-byte swizzle.
//   warps 9,10  MMA issuers, one thread per Q tile (warp 9 also allocates
//               TMEM): S_i = Q_i.K^T (M=128, N=128, K=dh, smem operands) and
//               O_i += P_i.V with P_i read from TMEM (tcgen05.mma A-from-TMEM,
//               V as the MN-major B).  Separate issuers keep the two Q tiles'
//               pipelines independent.
// TMEM (512 columns): S_0 S_1 (128 each), O_0 O_1 (dh each), P_0 P_1 (64 each,
// dh=64) or P_i over S_i (dh=128, after S_i is in registers).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>
#include <cstdint>
#include <cstdlib>

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
  // dh=128 fills TMEM with S0,S1,O0,O1 (4 x 128 columns), so P_i is written over
  // S_i (already in registers); dh=64 has room for separate P buffers
  static constexpr bool ALIAS = DH == 128;
  static constexpr int STAGES = DH == 64 ? 5 : 2;
  static constexpr uint32_t QB = ROWS * DH * 2;    // one Q tile
  static constexpr uint32_t KB = BKV * DH * 2;     // one K (or V) tile
  static constexpr uint32_t OFF_Q = 0;             // [2 Q tiles]
  static constexpr uint32_t OFF_K = OFF_Q + 2 * QB;
  static constexpr uint32_t OFF_V = OFF_K + STAGES * KB;
  static constexpr uint32_t OFF_RED = OFF_V + STAGES * KB;  // [2 parity][2 Q tiles][2 halves][128 rows] fp32
  static constexpr uint32_t OFF_BAR = OFF_RED + 2 * 2 * 2 * ROWS * 4;
  static constexpr size_t SMEM = OFF_BAR + 8 * (1 + 3 * STAGES + 8) + 16;
  // TMEM columns
  static constexpr uint32_t COL_S = 0;                          // S_i at 128 i
  static constexpr uint32_t COL_O = 2 * BKV;                    // O_i at 256 + DH i
  static constexpr uint32_t COL_P = ALIAS ? 0 : 2 * BKV + 2 * DH;  // P_i at COL_P + (ALIAS ? 128 : 64) i
  static constexpr uint32_t P_STRIDE = ALIAS ? BKV : BKV / 2;
};

// SPL softmax warps per query row (each takes BKV / SPL keys of a tile):
//   warps [0, NS): softmax, NS = 8 * SPL (Q tile i, key half h, TMEM quadrant q);
//   NS: TMA producer; NS+1 / NS+2: MMA issuers of Q tile 0 / 1; NS+3 idle.
template <int SPL>
struct Roles {
  static constexpr int NS = 8 * SPL;
  static constexpr int THREADS = 32 * (NS + 4);
  // setmaxnreg budgets: the CTA keeps its launch allocation (THREADS x launch-bound registers),
  // so NS x 32 x REG_SOFTMAX + 4 x 32 x REG_AUX must not exceed it (SPL=1: 384 x 168, SPL=2: 640 x 96)
  static constexpr int REG_SOFTMAX = SPL == 1 ? 224 : 104;
  static constexpr int REG_AUX = SPL == 1 ? 56 : 40;
};
constexpr float RESCALE_LOG2 = 8.f;   // lazy O rescale: keep a stale row max until it is 2^8 too small
#ifndef RDKV_ATTN_TRACE
#define RDKV_ATTN_TRACE 0  // 1: per-tile clock64 timeline of CTA 0 (debug builds only)
#endif
#if RDKV_ATTN_TRACE
__device__ long long g_attn_trace[4][64][8];
#define TRACE(who, j, ev) \
  do { if (blockIdx.x == gridDim.x - 1 && blockIdx.y == 0 && blockIdx.z == 0 && (j) < 64) g_attn_trace[who][j][ev] = clock64(); } while (0)
#else
#define TRACE(who, j, ev) do { } while (0)
#endif
#ifndef RDKV_ATTN_EMU
#define RDKV_ATTN_EMU 3
#endif
constexpr int EMU_OF_8 = RDKV_ATTN_EMU;  // exp2 of this many of every 8 score groups runs as a polynomial

#ifndef RDKV_ATTN_SPIN
#define RDKV_ATTN_SPIN 1
#endif
// MMA issuers spin (prompt wake-up: the issue latency sits on the P -> P.V chain)
__device__ __forceinline__ void issuer_wait(uint64_t* bar, uint32_t parity) {
  if (RDKV_ATTN_SPIN)
    mbar_wait(bar, parity);
  else
    mbar_wait_sleep(bar, parity);
}

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

template <int DH, int SPL>
__global__ void __launch_bounds__(Roles<SPL>::THREADS, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV, AttnParams p) {
  using C = TcCfg<DH>;
  using R = Roles<SPL>;
  constexpr int NS = R::NS;
  constexpr int KH = BKV / SPL;  // keys of a tile per softmax thread
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
  uint64_t* s_full = kv_empty + ST;        // [2] per Q tile: S_i = Q_i.K^T landed
  uint64_t* s_empty = s_full + 2;          // [2] S_i read into registers
  uint64_t* p_full = s_empty + 2;          // [2] P_i written (and O_i rescaled)
  uint64_t* o_done = p_full + 2;           // [2] O_i += P_i.V retired (P_i free)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 2);

  const int G = p.hq / p.hkv;
  const int TPT = ROWS / G;                 // tokens per Q tile
  const int s = blockIdx.z, kvh = blockIdx.y;
  const int xb = gridDim.x - 1 - blockIdx.x;  // longest causal rows first
  const int qb = xb / p.kv_splits, ks = xb % p.kv_splits;  // query-tile pair, KV split
  const int n_new = p.seq_new[s];
  const int tok0 = qb * 2 * TPT;
  if (tok0 >= n_new) return;
  const int ntok = min(2 * TPT, n_new - tok0);
  const int n_q = ntok > TPT ? 2 : 1;       // active Q tiles
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

  if (warp == NS && lane == 0) {
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    mbar_init(q_full, NS);
    for (int i = 0; i < ST; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&v_full[i], 1);
      mbar_init(&kv_empty[i], n_q);  // released by both Q tiles' P.V
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], 4 * SPL);
      mbar_init(&p_full[i], 4 * SPL);
      mbar_init(&o_done[i], 1);
    }
    fence_barrier_init();
  }
  if (warp == NS + 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  pdl_wait();  // q / KV planes written by the predecessor are visible from here

  // register budget: the softmax warpgroups hold a 128-score row per thread,
  // the TMA / MMA warpgroup gives its registers up
  if (warp >= NS) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(R::REG_AUX) : "memory");
  if (warp == NS) {
    // ------------------------------------------------------------ TMA producer
    // The whole warp walks the tiles: every 32 tiles each lane resolves one
    // tile's two block-table rows (32 global loads in parallel instead of a
    // dependent load per tile on the issue path); lane 0 issues the TMA.
    const long long row0 = (long long)kvh * (p.head_stride / DH);  // first row of this head in the plane view
    int my_rows[2] = {0, 0};
    for (int j = 0; j < n_tiles; ++j) {
      if ((j & 31) == 0 && j + lane < n_tiles) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          int pos = (t_begin + j + lane) * BKV + h * HALF;
          if (pos >= kv_len) pos = (t_begin + j + lane) * BKV;  // masked half: any valid, finite block
          my_rows[h] = (int)(row0 + (long long)bt[pos / p.block_size] * p.block_size + pos % p.block_size);
        }
      }
      const int rows[2] = {__shfl_sync(0xffffffffu, my_rows[0], j & 31), __shfl_sync(0xffffffffu, my_rows[1], j & 31)};
      if (lane == 0) {
        const int st = j % ST;
        mbar_wait_sleep(&kv_empty[st], ((j / ST) & 1) ^ 1);
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
      __syncwarp();
    }
  } else if (warp == NS + 1 || warp == NS + 2) {
    // ------------------------------------------------------------ MMA issuers
    // one issuing thread per Q tile, so neither softmax warpgroup ever waits on
    // the other's progress (their exp2 phases drift apart and overlap)
    const int i = warp - NS - 1;
    if (lane == 0 && n_tiles > 0 && i < n_q) {
      constexpr uint32_t idesc_qk = idesc_bf16_f32(ROWS, BKV);
      constexpr uint32_t idesc_pv = idesc_bf16_f32(ROWS, DH) | (1u << 16);  // B (V) is MN-major
      const uint32_t qa = sb + C::OFF_Q + i * C::QB;
      const uint32_t tS = tmem + C::COL_S + i * BKV, tO = tmem + C::COL_O + i * DH;
      const uint32_t tP = tmem + C::COL_P + i * C::P_STRIDE;
      auto issue_qk = [&](int j) {  // S_i = Q_i . K(j)^T
        const uint32_t ka = sb + C::OFF_K + (j % ST) * C::KB;
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) {
          const uint32_t sub = (kk & 3) * 32;
          umma_bf16(tS, desc_k(qa + (kk >> 2) * (ROWS * 128) + sub), desc_k(ka + (kk >> 2) * (BKV * 128) + sub),
                    idesc_qk, kk > 0 ? 1u : 0u);
        }
        umma_commit(&s_full[i]);
      };
      issuer_wait(q_full, 0);
      issuer_wait(&k_full[0], 0);
      tc_fence_after();
      issue_qk(0);
      for (int j = 0; j < n_tiles; ++j) {
        const int st = j % ST;
        const bool more = j + 1 < n_tiles;
        if (!C::ALIAS && more) {  // next S_i while the softmax still works on this tile
          issuer_wait(&k_full[(j + 1) % ST], ((j + 1) / ST) & 1);
          issuer_wait(&s_empty[i], j & 1);
          tc_fence_after();
          issue_qk(j + 1);
          TRACE(2 + i, j, 0);
        }
        issuer_wait(&v_full[st], (j / ST) & 1);
        issuer_wait(&p_full[i], j & 1);
        tc_fence_after();
        const uint32_t va = sb + C::OFF_V + st * C::KB;
#pragma unroll
        for (int kk = 0; kk < BKV / 16; ++kk) {  // O_i (+)= P_i . V(j), P_i from TMEM
          // P of keys [16kk, 16kk+16): with P over S each half writes inside its own S columns
          const uint32_t pcol = C::ALIAS ? (kk / (KH / 16)) * KH + (kk % (KH / 16)) * 8 : kk * 8;
          umma_bf16_ts(tO, tP + pcol, desc_mn(va + kk * 2048, BKV * 128), idesc_pv, (j > 0 || kk > 0) ? 1u : 0u);
        }
        umma_commit(&o_done[i]);
        TRACE(2 + i, j, 1);
        umma_commit(&kv_empty[st]);
        if (C::ALIAS && more) {  // S_i overwrites P_i only after the P.V above (issue order)
          issuer_wait(&k_full[(j + 1) % ST], ((j + 1) / ST) & 1);
          tc_fence_after();
          issue_qk(j + 1);
        }
      }
    }
  } else if (warp < NS) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(R::REG_SOFTMAX) : "memory");
    // ------------------------------------------------------------ softmax warps
    // warp w < NS: Q tile i, key half h (SPL = 2: keys [64h, 64h+64) of every tile,
    // O columns [h dh/2, (h+1) dh/2)), TMEM lanes [32 (w % 4), +32) = query rows.
    // With SPL = 2 the two halves of a row exchange their row max per tile (and
    // the row sum at the end) through smem under a 64-thread named barrier.
    const int i = warp / (4 * SPL), h = (warp / 4) % SPL, quad = warp & 3;
    const int r = quad * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const int nrows = max(0, min(TPT, ntok - i * TPT)) * G;
    float* red = reinterpret_cast<float*>(smem + C::OFF_RED);  // [parity][tile][half][row]
    auto pair_sync = [&]() {
      if constexpr (SPL == 2) asm volatile("bar.sync %0, 64;" ::"r"(1 + i * 4 + quad) : "memory");
    };
    auto exchange = [&](float v, int parity, bool use_max) {  // combine with the partner half of this row
      if constexpr (SPL == 1) {
        return v;
      } else {
        red[((parity * 2 + i) * 2 + h) * ROWS + r] = v;
        pair_sync();
        const float o = red[((parity * 2 + i) * 2 + (h ^ 1)) * ROWS + r];
        return use_max ? fmaxf(v, o) : v + o;
      }
    };
    // Q row (this half's 16-B chunks) -> smem (K-major SW128, DH/64 column blocks of [128 rows][128 B])
    {
      const bool ok = r < nrows;
      const int rr = ok ? r : 0;
      const uint4* src = reinterpret_cast<const uint4*>(
          p.q + (long long)(row_base + i * TPT + rr / G) * p.ldq + (long long)(kvh * G + rr % G) * DH);
#pragma unroll
      for (int cc = 0; cc < DH / 8 / SPL; ++cc) {
        const int c = h * (DH / 8 / SPL) + cc;
        const uint4 v = ok ? src[c] : make_uint4(0, 0, 0, 0);
        const uint32_t a = sb + C::OFF_Q + i * C::QB + (c >> 3) * (ROWS * 128) + r * 128 + (((c & 7) ^ (r & 7)) << 4);
        st_shared_v4(a, v.x, v.y, v.z, v.w);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(q_full);
    }
    if (i < n_q && n_tiles > 0) {
      // padded rows pretend to be the last valid position so no row is fully masked
      const int qpos = (r < nrows) ? pos0 + i * TPT + r / G : kv_len - 1;
      const float sl2 = p.scale_log2;
      constexpr int OH = DH / SPL;  // O columns of this half
      const uint32_t tS = tmem + C::COL_S + i * BKV + h * KH + lane_off;
      const uint32_t tO = tmem + C::COL_O + i * DH + h * OH + lane_off;
      // P columns of this half: inside its own S columns when P is written over S
      const uint32_t tP = tmem + C::COL_P + i * C::P_STRIDE + h * (C::ALIAS ? KH : KH / 2) + lane_off;
      float m_used = -INFINITY;  // row max the P values and O are scaled to (log2 domain)
      float l = 0.f;             // this half's row sum at scale m_used
      for (int j = 0; j < n_tiles; ++j) {
        mbar_wait(&s_full[i], j & 1);
        tc_fence_after();
        uint32_t sv[KH];
#pragma unroll
        for (int c = 0; c < KH / 32; ++c) tmem_ld32(tS + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&sv[c * 32]));
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_empty[i]);
        const int lim = qpos - (t_begin + j) * BKV - h * KH;  // key e of this half visible iff e <= lim
        if (lim < KH - 1) {
#pragma unroll
          for (int e = 0; e < KH; ++e)
            if (e > lim) sv[e] = __float_as_uint(-INFINITY);
        }
        float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int e = 0; e < KH; e += 8)
#pragma unroll
          for (int u = 0; u < 4; ++u)
            mx4[u] = fmax3(mx4[u], __uint_as_float(sv[e + 2 * u]), __uint_as_float(sv[e + 2 * u + 1]));
        const float mt = exchange(fmax3(fmaxf(mx4[0], mx4[1]), mx4[2], mx4[3]), j & 1, true) * sl2;
        // lazy rescale: move the reference max only when it grew by more than 2^8
        const bool need = mt > m_used + RESCALE_LOG2;
        const bool rescale = __any_sync(0xffffffffu, need) && j > 0;
        float f = 1.f;
        if (need) {
          f = ex2_approx(m_used - mt);  // 0 when m_used = -inf
          l *= f;
          m_used = mt;
        }
        // P = 2^(S*scale - m_used) as bf16 pairs (registers), row sum in fp32; this
        // overlaps P_i.V(j-1), which still reads the P_i buffer
        const float nb = m_used == -INFINITY ? 0.f : -m_used;
        float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
        uint32_t pk[KH / 2];
#pragma unroll
        for (int k = 0; k < KH; k += 4) {
          float x0, x1, x2, x3;
          ffma2(x0, x1, __uint_as_float(sv[k]), __uint_as_float(sv[k + 1]), sl2, sl2, nb, nb);
          ffma2(x2, x3, __uint_as_float(sv[k + 2]), __uint_as_float(sv[k + 3]), sl2, sl2, nb, nb);
          if (((k / 4) * 3) % 8 < EMU_OF_8) {  // this group of 4 on the FMA pipe
            exp2_emu2(x0, x1, x0, x1);
            exp2_emu2(x2, x3, x2, x3);
          } else {  // on the MUFU
            x0 = ex2_approx(x0);
            x1 = ex2_approx(x1);
            x2 = ex2_approx(x2);
            x3 = ex2_approx(x3);
          }
          fadd2(s0, s1, s0, s1, x0, x1);
          fadd2(s2, s3, s2, s3, x2, x3);
          pk[k / 2] = pack_bf16(x0, x1);
          pk[k / 2 + 1] = pack_bf16(x2, x3);
        }
        // P_i (and O_i) are free once P_i.V(j-1) has retired (implied by s_full when P aliases S)
        if (j > 0) {
          mbar_wait(&o_done[i], (j - 1) & 1);
          tc_fence_after();
        }
#pragma unroll
        for (int c = 0; c < KH / 64; ++c) tmem_st32(tP + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&pk[c * 32]));
        l += (s0 + s1) + (s2 + s3);
        if (rescale) {  // this half of the O_i row *= f before P_i.V(j) accumulates into it
#pragma unroll
          for (int c = 0; c < OH / 32; ++c) {
            uint32_t ov[32];
            tmem_ld32(tO + c * 32, ov);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; e += 2) {
              float a0, a1;
              fmul2(a0, a1, __uint_as_float(ov[e]), __uint_as_float(ov[e + 1]), f, f);
              ov[e] = __float_as_uint(a0);
              ov[e + 1] = __float_as_uint(a1);
            }
            tmem_st32(tO + c * 32, ov);
          }
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[i]);
      }
      // final O row: wait for the last P.V, normalise, store (each half its O columns)
      const float lt = exchange(l, n_tiles & 1, false);  // the parity the last tile did NOT use
      mbar_wait(&o_done[i], (n_tiles - 1) & 1);
      tc_fence_after();
      const bool ok = r < nrows;  // every lane joins the .sync.aligned TMEM loads; valid rows store
      const long long trow = row_base + i * TPT + (ok ? r : 0) / G;  // token row in [0, T)
      const int head = kvh * G + (ok ? r : 0) % G;
      const float inv = lt > 0.f ? 1.f / lt : 0.f;
#pragma unroll
      for (int c = 0; c < OH / 32; ++c) {
        uint32_t ov[32];
        tmem_ld32(tO + c * 32, ov);
        tmem_ld_wait();
        if (!ok) continue;
        const int col = h * OH + c * 32;
        if (p.kv_splits > 1) {
          // unnormalised partial at scale m_used; combined by attn_split_combine_kernel
          float4* dst =
              reinterpret_cast<float4*>(p.split_o + (((long long)ks * p.n_tokens + trow) * p.hq + head) * DH + col);
#pragma unroll
          for (int e = 0; e < 8; ++e)
            dst[e] = make_float4(__uint_as_float(ov[4 * e]), __uint_as_float(ov[4 * e + 1]),
                                 __uint_as_float(ov[4 * e + 2]), __uint_as_float(ov[4 * e + 3]));
        } else {
          uint4* dst = reinterpret_cast<uint4*>(p.o + trow * p.ldo + (long long)head * DH + col);
#pragma unroll
          for (int e = 0; e < 4; ++e)
            dst[e] = make_uint4(pack_bf16(__uint_as_float(ov[8 * e]) * inv, __uint_as_float(ov[8 * e + 1]) * inv),
                                pack_bf16(__uint_as_float(ov[8 * e + 2]) * inv, __uint_as_float(ov[8 * e + 3]) * inv),
                                pack_bf16(__uint_as_float(ov[8 * e + 4]) * inv, __uint_as_float(ov[8 * e + 5]) * inv),
                                pack_bf16(__uint_as_float(ov[8 * e + 6]) * inv, __uint_as_float(ov[8 * e + 7]) * inv));
        }
      }
      if (ok && h == 0 && p.kv_splits > 1)
        p.split_ml[((long long)ks * p.n_tokens + trow) * p.hq + head] = make_float2(m_used, lt);
    } else if (p.kv_splits > 1 && n_tiles == 0 && r < nrows && h == 0) {
      // empty split: mark the partial as absent
      const long long trow = row_base + i * TPT + r / G;
      p.split_ml[((long long)ks * p.n_tokens + trow) * p.hq + kvh * G + r % G] = make_float2(-INFINITY, 0.f);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == NS + 1) {
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

template <int DH, int SPL>
int launch_tc(const AttnParams& p, int n_seqs, int max_new, cudaStream_t st) {
  using C = TcCfg<DH>;
  static bool attr = false;
  if (!attr) {
    CUDA_TRY(cudaFuncSetAttribute(attn_tc_kernel<DH, SPL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
    attr = true;
  }
  // plane view: rows = hkv * slots, cols = dh
  const long long rows = (long long)p.hkv * (p.head_stride / DH);
  CUtensorMap tk, tv;
  RDKV_TRY(make_tmap(&tk, p.kplane, rows, DH, DH, HALF));
  RDKV_TRY(make_tmap(&tv, p.vplane, rows, DH, DH, HALF));
  const int tok_per_cta = 2 * ROWS / (p.hq / p.hkv);  // two Q tiles per CTA
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
  CUDA_TRY(launch_k(attn_tc_kernel<DH, SPL>, grid, dim3(Roles<SPL>::THREADS), C::SMEM, st, tk, tv, q));
  CUDA_TRY(cudaGetLastError());
  if (q.kv_splits > 1) {
    CUDA_TRY(launch_k(attn_split_combine_kernel<DH>, dim3(p.n_tokens, (p.hq + 7) / 8), dim3(256), 0, st, q));
    CUDA_TRY(cudaGetLastError());
  }
  return 0;
}

}  // namespace

#if RDKV_ATTN_TRACE
extern "C" RDKV_API int rdkv_debug_attn_trace(long long* out) {
  return cudaMemcpyFromSymbol(out, g_attn_trace, sizeof(g_attn_trace)) == cudaSuccess ? 0 : -8;
}
#endif

bool attention_tc_supported(const AttnParams& p, int head_dim) {
  const int G = p.hq / p.hkv;
  return (head_dim == 64 || head_dim == 128) && 128 % G == 0 && (p.block_size % HALF == 0 || p.contiguous);
}

int launch_attention_tc(const AttnParams& p, int head_dim, int n_seqs, int max_new, cudaStream_t st) {
  if (n_seqs <= 0 || max_new <= 0) return 0;
  if (!attention_tc_supported(p, head_dim))
    return set_error(RDKV_ERR_ARG, "attention_tc: unsupported shape (dh %d, group %d, block %d)", head_dim,
                     p.hq / p.hkv, p.block_size);
  static const int spl = [] {  // softmax warps per query row (RDKV_ATTN_SPL=2: two, 640 threads; measured slower)
    const char* e = std::getenv("RDKV_ATTN_SPL");
    return e && e[0] == '2' ? 2 : 1;
  }();
  if (head_dim == 64) return spl == 2 ? launch_tc<64, 2>(p, n_seqs, max_new, st) : launch_tc<64, 1>(p, n_seqs, max_new, st);
  return spl == 2 ? launch_tc<128, 2>(p, n_seqs, max_new, st) : launch_tc<128, 1>(p, n_seqs, max_new, st);
}

}  // namespace rdkv

namespace rdkv {
size_t attention_split_scratch_bytes(int T, int hq, int dh) {
  if (T <= 0 || T > 512) return 0;
  return (size_t)16 * T * hq * (dh * 4 + 8);
}
}  // namespace rdkv
