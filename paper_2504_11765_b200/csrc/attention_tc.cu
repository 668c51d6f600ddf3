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
// Warp roles (384 threads, one CTA per SM):
//   warps 0-3   softmax of Q tile 0, warps 4-7 softmax of Q tile 1: one query
//               row per thread (= one TMEM lane).  Per KV tile: tcgen05.ld the
//               BKV scores, mask, row max (FMNMX3), P = 2^(s*scale - m) with
//               packed FFMA2 + MUFU ex2, tcgen05.st of P (bf16 pairs) into TMEM.
//               The row max is moved lazily (only when it grows by > 2^8), and
//               only then is the O row in TMEM rescaled.  The two warpgroups
//               run independently, so one's exp2 overlaps the other's loads.
//   warp 8      TMA producer: K and V tiles of BKV positions (64-row boxes, one
//               per KV block of the paged pool / blob), STAGES-deep smem ring,
//               128-byte swizzle.  BKV = 128 at dh = 64, 64 at dh = 128.
//   warps 9,10  MMA issuers, one thread per Q tile (warp 9 also allocates
//               TMEM): S_i = Q_i.K^T (M=128, N=BKV, K=dh, smem operands) and
//               O_i += P_i.V with P_i read from TMEM (tcgen05.mma A-from-TMEM,
//               V as the MN-major B).  Separate issuers keep the two Q tiles'
//               pipelines independent.
//   warp 11     Q loader: TMA of each segment's Q tiles (3-D map: dh x heads x
//               tokens, so the G heads of one kv head land as consecutive rows)
//               as soon as the previous segment's last Q.K^T has retired.
// TMEM: S_0 S_1 (BKV each), O_0 O_1 (dh each), P_0 P_1 (BKV/2 each): 512 columns
// at dh = 64, 448 at dh = 128.  Q.K^T of tile j+1 is issued as soon as the
// softmax has read S(j), so the tensor pipe works while the softmax does.
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
PFN_cuTensorMapEncodeTiled_v12000 encode_fn();

// Q as a 3-D bf16 map {dh, heads, tokens} (token stride ldq elements), box {64, G, TPT}, 128-B swizzle
static int make_tmap_q(CUtensorMap* m, const void* q, long long tokens, int hq, int dh, long long ldq, int G, int tpt) {
  auto fn = encode_fn();
  if (!fn) return set_error(RDKV_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {(cuuint64_t)dh, (cuuint64_t)hq, (cuuint64_t)tokens};
  cuuint64_t strides[2] = {(cuuint64_t)dh * 2, (cuuint64_t)ldq * 2};
  cuuint32_t box[3] = {64, (cuuint32_t)G, (cuuint32_t)tpt};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(q), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(RDKV_ERR_CUDA, "cuTensorMapEncodeTiled (q) failed (%d)", (int)r);
  return 0;
}

#ifndef RDKV_ATTN_BYKIND
#define RDKV_ATTN_BYKIND 1  // MMA issuers by kind and Q tile (Q.K^T_0, Q.K^T_1, P.V_0, P.V_1) instead of one per Q tile
#endif
#ifndef RDKV_ATTN_QTMEM
#define RDKV_ATTN_QTMEM 1  // Q tile 0 in TMEM for its Q.K^T (issuers by kind, dh = 128)
#endif
#ifndef RDKV_ATTN_ONES
#define RDKV_ATTN_ONES 0  // 1: row sums through a ones column in V (issuers by kind, dh = 128)
#endif
#ifndef RDKV_ATTN_PDB
#define RDKV_ATTN_PDB 0  // 1: double-buffered P with the issuers by kind (dh = 128)
#endif
#ifndef RDKV_ATTN_BYK64
#define RDKV_ATTN_BYK64 0  // 1: issuers by kind at dh = 64 too
#endif
#ifndef RDKV_ATTN_SPLITKV
#define RDKV_ATTN_SPLITKV 0  // 1: separate K / V stage releases in the two-issuer schedule (measured: C3 98.5 vs 96.3 us, C2 77.5 vs 78.3)
#endif
#ifndef RDKV_ATTN_LSUM
#define RDKV_ATTN_LSUM 0  // 1: dh = 128 row sums on the tensor cores (L += P.ones; measured slower: 111 vs 98 us)
#endif
namespace {

constexpr int ROWS = 128;
constexpr int HALF = 64;  // rows per TMA box (= one KV block of the pool)

template <int DH, bool PP = false, bool BYK = false>
struct TcCfg {
  // key positions per tile: 128 at dh = 64; 64 at dh = 128, so S_i (BKV columns),
  // O_i (dh) and P_i (BKV / 2) of both Q tiles fit the 512 TMEM columns (448) and
  // Q_i.K^T of the next tile is issued while the softmax still works on this one
  // (with 128-key tiles at dh = 128, P_i had to live over S_i and each Q tile's
  // S -> P -> P.V -> next S chain serialised: ~4.3k cycles per 128 keys).
  // PP (ping-pong, dh = 128): 128-key tiles with P_i over S_i, ONE issuer that interleaves
  // the Q tiles (P.V_0, Q.K^T_0, P.V_1, Q.K^T_1, ...) so one tile's softmax runs while the
  // tensor pipe works on the other tile; Q.K^T at N = 128 (N = 64 MMAs run at 2/3 rate,
  // profiles/r2_l2_prefetch_ab.txt), separate K and V rings (K released after both
  // Q.K^T, V after both P.V; K loaded two tiles ahead).
  static constexpr int BKV = PP ? 128 : (DH == 128 ? 64 : 128);
  static constexpr bool ALIAS = PP;  // P_i over S_i
#ifndef RDKV_ATTN_ST64
#define RDKV_ATTN_ST64 5
#endif
#ifndef RDKV_ATTN_ST128
#define RDKV_ATTN_ST128 4
#endif
#ifndef RDKV_ATTN_ST128_BYK
#define RDKV_ATTN_ST128_BYK 5
#endif
  // BYK (issuers by kind, one segment): no row-exchange / stream-K regions, so dh = 128
  // affords a fifth K/V stage (the stage of tile j + ST is released only when the later Q
  // tile's P.V(j) retired; K/V loads under full load take ~3.8k cycles)
  static constexpr int STAGES = DH == 64 ? RDKV_ATTN_ST64 : BYK ? (RDKV_ATTN_ONES ? 4 : RDKV_ATTN_ST128_BYK) : RDKV_ATTN_ST128;
  static constexpr int KST = PP ? 3 : STAGES;  // K stages (PP: own ring)
  static constexpr int VST = PP ? 2 : STAGES;  // V stages (PP: own ring)
  static constexpr uint32_t QB = ROWS * DH * 2;    // one Q tile
  static constexpr uint32_t KB = BKV * DH * 2;     // one K (or V) tile
  static constexpr uint32_t OFF_Q = 0;             // [2 Q tiles]
  static constexpr uint32_t OFF_K = OFF_Q + 2 * QB;
  static constexpr uint32_t OFF_V = OFF_K + KST * KB;
  // RDKV_ATTN_ONES (BYK, dh = 128): each V stage carries a third 64-column chunk of bf16 ones
  // (written once), so P.V runs at N = DH + 16 and O's extra columns accumulate the row sums
  // of the bf16 P the tensor cores multiplied (no FADD2 row sum in the softmax)
  static constexpr bool ONES = RDKV_ATTN_ONES && BYK && DH == 128 && !PP;
  static constexpr uint32_t VKB = KB + (ONES ? BKV * 128 : 0);  // V stage stride
  static constexpr uint32_t OW = DH + (ONES ? 16 : 0);          // O columns per Q tile
  // row max / sum exchange of the two halves of a row (SPL = 2): [parity][2 Q tiles][2
  // halves][128 rows] fp32; PP has room for one parity only (a second barrier orders reuse)
  static constexpr int RED_PAR = PP ? 1 : 2;
  static constexpr uint32_t OFF_RED = OFF_V + VST * VKB;
  static constexpr uint32_t OFF_BAR = OFF_RED + (BYK ? 0 : RED_PAR * 2 * 2 * ROWS * 4);
  // RDKV_ATTN_PDB (BYK at dh = 128): P double-buffered (TMEM has the room: S 128 + O 256 + P 4 x 32
  // = 512), so the softmax stores P(j) once P.V(j-2) retired instead of waiting for P.V(j-1).
  // Correct but measured no faster (C3 attn_perf 92.3 vs 91.7 us): off
  static constexpr int P_BUFS = RDKV_ATTN_PDB && BYK && DH == 128 ? 2 : 1;
  static constexpr uint32_t N_BARS = 4 + 2 * KST + 2 * VST + 4 + 4 * P_BUFS;
  static constexpr uint32_t OFF_MISC = (OFF_BAR + 8 * N_BARS + 15) / 16 * 16;  // TMEM base, segment count, W
  static constexpr uint32_t OFF_SEG = OFF_MISC + 16;                        // stream-K segments (int4)
  static constexpr uint32_t OFF_SEQ = OFF_SEG + 16 * 512;                   // stream-K: [3][512] seq start/new/cached
  // row sums on the tensor cores (dh = 128, where TMEM has room): L_i += P_i . ones, with a
  // constant [16 x BKV] bf16 ones tile as the K-major B operand (16 columns of L_i, all equal)
  static constexpr bool LSUM = RDKV_ATTN_LSUM && DH == 128 && !ALIAS;
  static constexpr uint32_t OFF_ONES = (OFF_SEQ + 3 * 4 * 512 + 1023) / 1024 * 1024;
  static constexpr size_t SMEM = PP || BYK ? OFF_MISC + 16 : LSUM ? OFF_ONES + 16 * 128 : OFF_SEQ + 3 * 4 * 512;
  static_assert(SMEM <= 232448, "attention smem exceeds 227 KB");
  // TMEM columns
  static constexpr uint32_t COL_S = 0;                          // S_i at BKV i
  static constexpr uint32_t COL_O = 2 * BKV;                    // O_i at 2 BKV + OW i
  static constexpr uint32_t COL_P = ALIAS ? 0 : 2 * BKV + 2 * OW;  // P_i at COL_P + (ALIAS ? BKV : BKV / 2) i
  static constexpr uint32_t P_STRIDE = ALIAS ? BKV : P_BUFS * BKV / 2;  // per Q tile (all P buffers)
  static_assert(COL_P + 2 * P_STRIDE <= 512, "TMEM: P does not fit");
  static constexpr uint32_t COL_L = COL_P + 2 * P_STRIDE;     // L_i at COL_L + 16 i (LSUM)
  // RDKV_ATTN_QTMEM (BYK, dh = 128, single P buffer): Q tile 0 staged in the last 64 TMEM columns
  // (tcgen05.cp), so its Q.K^T reads only K from smem: M = 128, N = 64 MMAs are smem-bound at
  // 48 cycles with both operands in smem (4 KB of Q + 2 KB of K per K = 16 step)
  static constexpr bool QTMEM = RDKV_ATTN_QTMEM && BYK && DH == 128 && P_BUFS == 1 && !ONES;
  static constexpr uint32_t COL_Q0 = COL_P + 2 * P_STRIDE;
  static_assert(!QTMEM || COL_Q0 + DH / 2 <= 512, "TMEM: Q tile 0 does not fit");
  static_assert(!LSUM || COL_L + 32 <= 512, "TMEM: L columns do not fit");
  static_assert(COL_O + 2 * OW <= 512, "TMEM: S and O do not fit");
  static_assert(!ONES || P_BUFS == 1, "ones-column row sums with a single P buffer");
};

// SPL softmax warps per query row (each takes BKV / SPL keys of a tile):
//   warps [0, NS): softmax, NS = 8 * SPL (Q tile i, key half h, TMEM quadrant q);
//   NS: TMA producer; NS+1 / NS+2: MMA issuers of Q tile 0 / 1; NS+3: Q loader.
//   BYK (MMA issuers by kind, see ISSUE_BY_KIND): NS+1 / NS+2 issue Q.K^T of Q tile 0 / 1,
//   NS+3 loads Q then issues P.V of Q tile 0, the TMA producer NS also issues P.V of Q tile 1.
template <int SPL, bool BYK = false>
struct Roles {
  static constexpr int NS = 8 * SPL;
  static constexpr int THREADS = 32 * (NS + 4);
  // setmaxnreg budgets: the CTA keeps its launch allocation (THREADS x launch-bound registers),
  // so NS x 32 x REG_SOFTMAX + 4 x 32 x REG_AUX must not exceed it (SPL=1: 384 x 168, SPL=2: 640 x 96)
  static constexpr int REG_SOFTMAX = SPL == 1 ? 224 : 104;
  static constexpr int REG_AUX = SPL == 1 ? 56 : 40;
};
// Q.K^T and P.V issued by separate threads, one per (kind, Q tile): single-segment grids
// with the default TMEM layout (not stream-K, ping-pong or tensor-core row sums)
// (dh = 128: at dh = 64 the default schedule measured 1% faster)
template <int DH, int SPL, bool SK, bool PP>
constexpr bool issue_by_kind() {
  return RDKV_ATTN_BYKIND && (DH == 128 || RDKV_ATTN_BYK64) && SPL == 1 && !SK && !PP && !RDKV_ATTN_LSUM && !(RDKV_ATTN_SPLITKV != 0);
}
template <int DH, int SPL, bool SK, bool PP>
using RolesOf = Roles<SPL, issue_by_kind<DH, SPL, SK, PP>()>;
template <int DH, int SPL, bool SK, bool PP>
using CfgOf = TcCfg<DH, PP, issue_by_kind<DH, SPL, SK, PP>()>;
constexpr float RESCALE_LOG2 = 8.f;   // lazy O rescale: keep a stale row max until it is 2^8 too small
#ifndef RDKV_ATTN_TRACE
#define RDKV_ATTN_TRACE 0  // 1: per-tile clock64 timeline of CTA 0 (debug builds only)
#endif
#if RDKV_ATTN_TRACE
__device__ long long g_attn_trace[6][64][8];
__device__ long long g_attn_cta[2048][4];  // per CTA: smid, start, after prologue, end (globaltimer ns)
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define CTA_TRACE(ev)                                                                              \
  do {                                                                                             \
    const int _c = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);                 \
    if (threadIdx.x == 0 && _c < 2048) {                                                           \
      if ((ev) == 1) {                                                                             \
        unsigned _sm;                                                                              \
        asm volatile("mov.u32 %0, %smid;" : "=r"(_sm));                                           \
        g_attn_cta[_c][0] = _sm;                                                                   \
      }                                                                                            \
      g_attn_cta[_c][ev] = gtimer();                                                               \
    }                                                                                              \
  } while (0)
#define TRACE(who, j, ev) \
  do { if (blockIdx.x == gridDim.x - 1 && blockIdx.y == 0 && blockIdx.z == 0 && (j) < 64) g_attn_trace[who][j][ev] = clock64(); } while (0)
#else
#define TRACE(who, j, ev) do { } while (0)
#define CTA_TRACE(ev) do { } while (0)
#endif
#ifndef RDKV_ATTN_EMU
#define RDKV_ATTN_EMU 3
#endif
constexpr int EMU_OF_8 = RDKV_ATTN_EMU;  // exp2 of this many of every 8 score groups runs as a polynomial
#ifndef RDKV_ATTN_SPEC
#define RDKV_ATTN_SPEC 0  // 1: P at the current reference max while the tile max is taken (redo if it moved); measured slower
#endif

#ifndef RDKV_ATTN_PF
#define RDKV_ATTN_PF 0  // TMA producer L2 prefetch distance in tiles (0: off; 2-8 measured no faster)
#endif
#ifndef RDKV_ATTN_PPF
#define RDKV_ATTN_PPF 0  // ping-pong producer: L2 prefetch distance in tiles ahead of the K stream (2-8 slower)
#endif
#ifndef RDKV_ATTN_IDLE
#define RDKV_ATTN_IDLE 0  // 1: softmax warps with no real query row skip the exp work (decode: G valid
                          // rows of 128); measured no faster — decode attention is HBM-bound (5.15-5.19
                          // vs 5.16-5.22 ms per C3 decode step, identical tokens)
#endif
constexpr bool IDLE_SKIP = RDKV_ATTN_IDLE != 0;
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


// One unit of attention work: two Q tiles (query block qb) of sequence s against KV head kvh.
struct Unit {
  int s, kvh, tok0, ntok, n_q, pos0, kv_len, n_all, row_base;
};
template <int BKV>
__device__ __forceinline__ Unit unit_of(const int* seq_start, const int* seq_new, const int* seq_cached, int s, int qb,
                                       int kvh, int TPT) {
  Unit u;
  u.s = s;
  u.kvh = kvh;
  const int n_new = seq_new[s];
  u.tok0 = qb * 2 * TPT;
  u.ntok = max(0, min(2 * TPT, n_new - u.tok0));
  u.n_q = u.ntok > TPT ? 2 : (u.ntok > 0 ? 1 : 0);
  u.pos0 = seq_cached[s] + u.tok0;
  u.kv_len = u.pos0 + u.ntok;
  u.n_all = u.ntok > 0 ? (u.kv_len + BKV - 1) / BKV : 0;
  u.row_base = seq_start[s] + u.tok0;
  return u;
}

// Segment kinds: a CTA's share [ta, tb) of one unit's KV tiles
enum : int { SEG_WHOLE = 0, SEG_SPLIT = 1, SEG_PART = 2, SEG_HEAD = 3 };
constexpr int SK_MAXSEG = 512;     // stream-K: segments per CTA (<= units, checked at launch)
constexpr int SK_BAR = 9;          // named barrier of the softmax warps (stream-K hand-off)
constexpr int SK_PUB = 10;         // softmax warps + the Q-loader warp: a part's rows are written

// stream-K: first global tile of CTA b when W tiles are spread over G CTAs
__device__ __forceinline__ long long sk_bound(int b, long long W, int G) { return (long long)b * W / G; }

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// SK = false: one CTA per (query block, kv head, sequence[, KV split]), as the grid says.
// SK = true (stream-K, SPL = 1): a persistent grid of G CTAs; the W = sum of all units' KV
// tiles are dealt out as G equal contiguous ranges of the (sequence, query block, kv head)
// -major tile order, so every SM gets the same number of tile iterations whatever the
// unit count.  A unit cut by a range boundary is finished by the CTA that holds its
// first tiles (SEG_HEAD, always that CTA's last segment): it merges the (m, l, O)
// partials that the following CTAs wrote as their FIRST segment (SEG_PART, published
// with a release flag before they do anything else, so the waits cannot deadlock).
template <int DH, int SPL, bool SK, bool PP = false>
__global__ void __launch_bounds__(RolesOf<DH, SPL, SK, PP>::THREADS, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                   const __grid_constant__ CUtensorMap tmQ, AttnParams p) {
  using C = CfgOf<DH, SPL, SK, PP>;
  using R = RolesOf<DH, SPL, SK, PP>;
  static_assert(!SK || SPL == 1, "stream-K runs one softmax warp per row");
  static_assert(!PP || !SK, "ping-pong runs one segment per CTA");
  constexpr int NS = R::NS;
  constexpr int BKV = C::BKV;
  constexpr int NH = BKV / HALF;  // TMA boxes (KV blocks) per tile
  constexpr int KH = BKV / SPL;   // keys of a tile per softmax thread
  static_assert(KH % 64 == 0, "a softmax thread stores P in 32-column TMEM chunks");
  constexpr int ST = C::STAGES;
  constexpr bool SPEC = RDKV_ATTN_SPEC != 0;
  // Q.K^T and P.V issued by separate threads (single-segment grids, default two-issuer layout)
  constexpr bool ISSUE_BY_KIND = issue_by_kind<DH, SPL, SK, PP>();
  static_assert(!ISSUE_BY_KIND || (!C::LSUM && !C::ALIAS), "issuers by kind need separate S / P buffers");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  CTA_TRACE(1);
  uint8_t* smem = smem_raw;
  const uint32_t sb = smem_u32(smem);
  if (sb & 1023) __trap();  // SW128 operands need 1024-B alignment
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* q_full = bars + 0;             // [2] per Q tile: Q_i staged
  uint64_t* q_empty = bars + 2;            // [2] per Q tile: the segment's last Q_i.K^T retired
  constexpr int KST = C::KST, VST = C::VST;
  // separate K and V releases: a K stage frees after both Q.K^T, a V stage after both P.V,
  // and the producer runs K LEAD tiles ahead of V (stream-K keeps the shared stages)
  constexpr bool SPLIT = PP || (RDKV_ATTN_SPLITKV && !SK);
  constexpr int LEAD = PP ? 2 : 1;
  uint64_t* k_full = bars + 4;             // [KST]
  uint64_t* v_full = k_full + KST;         // [VST]
  uint64_t* kv_empty = v_full + VST;       // [KST] stage free (PP: K consumed by both Q.K^T)
  uint64_t* v_empty = kv_empty + KST;      // [VST] PP only: V consumed by both P.V
  uint64_t* s_full = v_empty + (SPLIT ? VST : 0);  // [2] per Q tile: S_i = Q_i.K^T landed
  uint64_t* s_empty = s_full + 2;          // [2] S_i read into registers
  // per P buffer (the softmax runs up to P_BUFS tiles ahead of the P.V issuer, so one barrier
  // per buffer keeps every parity wait within one phase of the barrier's state)
  uint64_t* p_full = s_empty + 2;          // [2][P_BUFS] P_i(buffer b) written (and O_i rescaled)
  uint64_t* o_done = p_full + 2 * C::P_BUFS;  // [2][P_BUFS] O_i += P_i(buffer b).V retired (that P buffer free)
  // the barriers and parity of tile t of Q tile i: P(t) written, P.V_i(t) retired
  auto pf = [&](int i, int t) { return &p_full[i * C::P_BUFS + t % C::P_BUFS]; };
  auto od = [&](int i, int t) { return &o_done[i * C::P_BUFS + t % C::P_BUFS]; };
  auto od_par = [&](int t) { return (uint32_t)((t / C::P_BUFS) & 1); };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::OFF_MISC);
  int* nseg_s = reinterpret_cast<int*>(smem + C::OFF_MISC + 4);
  long long* wtot_s = reinterpret_cast<long long*>(smem + C::OFF_MISC + 8);
  int4* segs = reinterpret_cast<int4*>(smem + C::OFF_SEG);  // {unit code, ta, tb, kind}

  const int G = p.hq / p.hkv;
  const int TPT = ROWS / G;                 // tokens per Q tile
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int QBn = SK || p.tail_ctas ? p.sk_qblocks : gridDim.x / p.kv_splits;
  // the single segment of a non-stream-K CTA, and its KV split index
  int4 seg0 = make_int4(0, 0, 0, SEG_WHOLE);
  int ks0 = 0;
  if constexpr (!SK) {
    int s, kvh, qb, ks = 0, nsplit = p.kv_splits;
    if (p.tail_ctas) {
      // tail-split grid (1-D): CTAs [0, tail_ctas) = whole units of sequences
      // [0, seq_off) (dispatched first: the full waves); the rest = units of the
      // remaining sequences in kv_splits KV ranges each, filling the last wave
      const int ups = QBn * p.hkv;
      int r;
      if ((int)blockIdx.x < p.tail_ctas) {
        s = blockIdx.x / ups;
        r = blockIdx.x % ups;
        nsplit = 1;
      } else {
        const int v = blockIdx.x - p.tail_ctas;
        s = p.seq_off + v / (ups * p.kv_splits);
        r = v % (ups * p.kv_splits);
        ks = r % p.kv_splits;
        r /= p.kv_splits;
      }
      kvh = r % p.hkv;
      qb = r / p.hkv;
    } else {
      s = blockIdx.z + p.seq_off;
      kvh = blockIdx.y;
      const int xb = gridDim.x - 1 - blockIdx.x;  // longest causal rows first
      qb = xb / p.kv_splits;
      ks = xb % p.kv_splits;
    }
    const Unit u = unit_of<BKV>(p.seq_start, p.seq_new, p.seq_cached, s, qb, kvh, TPT);
    if (u.ntok == 0) return;
    const int per_split = (u.n_all + nsplit - 1) / nsplit;
    const int ta = min(u.n_all, ks * per_split), tb = min(u.n_all, ta + per_split);
    seg0 = make_int4((s * QBn + qb) * p.hkv + kvh, ta, tb, nsplit > 1 ? SEG_SPLIT : SEG_WHOLE);
    ks0 = ks;
  }

  if (warp == NS) {
    if (lane == 0) {
      tma_prefetch_desc(&tmK);
      tma_prefetch_desc(&tmV);
      tma_prefetch_desc(&tmQ);
      for (int i = 0; i < 2; ++i) {
        mbar_init(&q_full[i], 1);
        mbar_init(&q_empty[i], 1);
      }
      if constexpr (PP) {  // one issuer commits each release once
        for (int i = 0; i < KST; ++i) {
          mbar_init(&k_full[i], 1);
          mbar_init(&kv_empty[i], 1);
        }
        for (int i = 0; i < VST; ++i) {
          mbar_init(&v_full[i], 1);
          mbar_init(&v_empty[i], 1);
        }
      } else {
        for (int i = 0; i < ST; ++i) {
          mbar_init(&k_full[i], 1);
          mbar_init(&v_full[i], 1);
          mbar_init(&kv_empty[i], 2);  // both Q tiles' (P.V) issuers release every stage
          if constexpr (SPLIT) mbar_init(&v_empty[i], 2);
        }
      }
      for (int i = 0; i < 2; ++i) {
        mbar_init(&s_full[i], 1);
        mbar_init(&s_empty[i], 4 * SPL);
        for (int b = 0; b < C::P_BUFS; ++b) mbar_init(&p_full[i * C::P_BUFS + b], 4 * SPL);
        for (int b = 0; b < C::P_BUFS; ++b) mbar_init(&o_done[i * C::P_BUFS + b], 1);
      }
      fence_barrier_init();
    }
    if constexpr (SK) {
      // stream-K schedule (batch metadata only: valid before the predecessor finishes).
      // Lane l walks a contiguous chunk of (sequence, query block) pairs; every pair
      // holds hkv units of equal cost (KV tiles).
      const int npair = p.n_seqs * QBn;
      // the batch metadata the roles re-read per segment, cached in smem (n_seqs <= units <= 512)
      int* seq_s = reinterpret_cast<int*>(smem + C::OFF_SEQ);
      for (int q = lane; q < p.n_seqs; q += 32) {
        seq_s[q] = p.seq_start[q];
        seq_s[512 + q] = p.seq_new[q];
        seq_s[1024 + q] = p.seq_cached[q];
      }
      auto cost = [&](int pr) { return unit_of<BKV>(p.seq_start, p.seq_new, p.seq_cached, pr / QBn, pr % QBn, 0, TPT).n_all; };
      const int chunk = (npair + 31) / 32;
      const int c0 = min(npair, lane * chunk), c1 = min(npair, c0 + chunk);
      long long mine = 0;
      for (int pr = c0; pr < c1; ++pr) mine += (long long)cost(pr) * p.hkv;
      long long incl = mine;
      for (int o = 1; o < 32; o <<= 1) {
        const long long t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      const long long W = __shfl_sync(0xffffffffu, incl, 31);
      const long long B0 = sk_bound(blockIdx.x, W, gridDim.x), B1 = sk_bound(blockIdx.x + 1, W, gridDim.x);
      int base = 0;
      for (int pass = 0; pass < 2; ++pass) {
        long long g = incl - mine;
        int cnt = 0;
        for (int pr = c0; pr < c1 && g < B1; ++pr) {
          const int c = cost(pr);
          if (c == 0 || g + (long long)c * p.hkv <= B0) {
            g += (long long)c * p.hkv;
            continue;
          }
          for (int kvh = 0; kvh < p.hkv; ++kvh, g += c) {
            const long long lo = max(g, B0), hi = min(g + c, B1);
            if (lo >= hi) continue;
            if (pass == 1) {
              const int ta = (int)(lo - g), tb = (int)(hi - g);
              segs[base + cnt] = make_int4(pr * p.hkv + kvh, ta, tb, ta > 0 ? SEG_PART : tb < c ? SEG_HEAD : SEG_WHOLE);
            }
            ++cnt;
          }
        }
        if (pass == 0) {  // exclusive scan of the per-lane counts -> write offsets
          int ic = cnt;
          for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, ic, o);
            if (lane >= o) ic += t;
          }
          base = ic - cnt;
          if (lane == 31) {
            *nseg_s = ic;
            *wtot_s = W;
          }
        }
      }
    }
  }
  if (warp == NS + 1) tmem_alloc(tmem_slot, 512);
  if constexpr (C::ONES) {
    if (warp == NS + 3) {  // every V stage's third chunk: bf16 1.0 (never written by the TMA)
      for (int st2 = 0; st2 < C::VST; ++st2) {
        uint32_t* ones = reinterpret_cast<uint32_t*>(smem + C::OFF_V + st2 * C::VKB + C::KB);
        for (int w = lane; w < BKV * 128 / 4; w += 32) ones[w] = 0x3F803F80u;
      }
      fence_proxy_async_smem();  // generic-proxy stores -> visible to the tensor core (async proxy)
    }
  }
  if constexpr (C::LSUM) {
    if (warp == NS + 3) {  // constant B operand of the row-sum MMA: bf16 1.0 everywhere
      uint32_t* ones = reinterpret_cast<uint32_t*>(smem + C::OFF_ONES);
      for (int w = lane; w < 16 * 128 / 4; w += 32) ones[w] = 0x3F803F80u;
      fence_proxy_async_smem();  // generic-proxy stores -> visible to the tensor core (async proxy)
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int nseg = SK ? *nseg_s : 1;
  const long long Wtot = SK ? *wtot_s : 0;  // stream-K: total KV tiles of the launch
  auto seg_at = [&](int k) { return SK ? segs[k] : seg0; };
  const int* seq_s = reinterpret_cast<const int*>(smem + C::OFF_SEQ);
  auto unit_at = [&](int code) {
    const int pr = code / p.hkv;
    if constexpr (SK) return unit_of<BKV>(seq_s, seq_s + 512, seq_s + 1024, pr / QBn, pr % QBn, code % p.hkv, TPT);
    return unit_of<BKV>(p.seq_start, p.seq_new, p.seq_cached, pr / QBn, pr % QBn, code % p.hkv, TPT);
  };
  pdl_trigger();
  pdl_wait();  // q / KV planes written by the predecessor are visible from here
  CTA_TRACE(2);

  // register budget: the softmax warpgroups hold a 128-score row per thread,
  // the TMA / MMA warpgroup gives its registers up
  if (warp >= NS) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(R::REG_AUX) : "memory");
  // P.V of Q tile i for KV tile j (ISSUE_BY_KIND; lane 0): P.V_i(j) is issued only after the
  // softmax consumed S_i(j), i.e. after Q.K^T_i(j) retired, so this thread's commit after
  // P.V_i(j) also covers K(j); each Q tile's P.V issuer releases the stage once (count 2).
  auto pv_step = [&](int i, int j, bool mine) {
    constexpr uint32_t idesc_pv = idesc_bf16_f32(ROWS, C::OW) | (1u << 16);  // B (V) is MN-major
    const int st = j % ST;
    issuer_wait(&v_full[st], (j / ST) & 1);
    if (!mine) {  // no Q tile i in this unit: just release the stage
      mbar_arrive(&kv_empty[st]);
      return;
    }
    issuer_wait(pf(i, j), od_par(j));
    TRACE(2 + i, j, 5);
    tc_fence_after();
    const uint32_t va = sb + C::OFF_V + st * C::VKB;
    const uint32_t tO = tmem + C::COL_O + i * C::OW;
    const uint32_t tP = tmem + C::COL_P + i * C::P_STRIDE + (j % C::P_BUFS) * (BKV / 2);
#pragma unroll
    for (int kk = 0; kk < BKV / 16; ++kk)  // O_i (+)= P_i . V(j), P_i from TMEM
      umma_bf16_ts(tO, tP + kk * 8, desc_mn(va + kk * 2048, BKV * 128), idesc_pv, (j > 0 || kk > 0) ? 1u : 0u);
    umma_commit(od(i, j));
    umma_commit(&kv_empty[st]);
    TRACE(2 + i, j, 1);
  };
  if (warp == NS) {
    if constexpr (SPLIT) {
      // ---------------------------------------------------------- TMA producer (split K / V rings)
      // K runs LEAD tiles ahead of V: order K(0..LEAD-1), then V(j), K(j + LEAD).  Each stream
      // keeps a warp-wide cache of 32 tiles' block-table rows (lane l holds tile base + l).
      const int4 sg = seg0;
      const Unit u = unit_at(sg.x);
      const long long row0 = (long long)u.kvh * (p.head_stride / DH);
      const int* bt = p.block_table + (long long)u.s * p.bt_stride;
      const uint64_t pol_kv = policy_evict_first();
      auto fetch = [&](int base, int (&cache)[NH]) {
        const int j = base + lane;
        if (j < sg.z) {
#pragma unroll
          for (int h = 0; h < NH; ++h) {
            int pos = j * BKV + h * HALF;
            if (pos >= u.kv_len) pos = j * BKV;  // masked half: any valid, finite block
            cache[h] = (int)(row0 + (long long)bt[pos / p.block_size] * p.block_size + pos % p.block_size);
          }
        }
      };
      int kbase = -64, vbase = -64, kc[NH] = {}, vc[NH] = {};
      auto load = [&](bool isk, int j) {  // whole warp (uniform j)
        int& base = isk ? kbase : vbase;
        int(&cache)[NH] = isk ? kc : vc;
        if (j < base || j >= base + 32) {
          base = j;
          fetch(base, cache);
        }
        int rows[NH];
#pragma unroll
        for (int h = 0; h < NH; ++h) rows[h] = __shfl_sync(0xffffffffu, cache[h], j - base);
        if (lane == 0) {
          const int jl = j - sg.y, ns = isk ? KST : VST, st = jl % ns;
          mbar_wait_sleep(isk ? &kv_empty[st] : &v_empty[st], ((jl / ns) & 1) ^ 1);
          uint64_t* bar = isk ? &k_full[st] : &v_full[st];
          mbar_arrive_expect_tx(bar, C::KB);
          const CUtensorMap* tm = isk ? &tmK : &tmV;
          uint8_t* dst = smem + (isk ? C::OFF_K + st * C::KB : C::OFF_V + st * C::VKB);
#pragma unroll
          for (int c = 0; c < DH / 64; ++c)
#pragma unroll
            for (int h = 0; h < NH; ++h) {
              if (p.kv_evict_first)
                tma_load_2d(tm, bar, dst + c * (BKV * 128) + h * (HALF * 128), c * 64, rows[h], pol_kv);
              else
                tma_load_2d_nohint(tm, bar, dst + c * (BKV * 128) + h * (HALF * 128), c * 64, rows[h]);
            }
        }
        __syncwarp();
      };
      // the K/V stream outruns the smem rings' lead (~5k cycles of DRAM latency under load at
      // 3 + 2 stages): warm L2 with K and V of tile j + RDKV_ATTN_PPF when K(j) is requested
      auto prefetch = [&](int j) {
        if (RDKV_ATTN_PPF <= 0 || j >= sg.z) return;
        int pcache[NH];
        // rows of tile j: this lane's cache covers it only if j is in the K window
        if (j >= kbase && j < kbase + 32) {
#pragma unroll
          for (int h = 0; h < NH; ++h) pcache[h] = __shfl_sync(0xffffffffu, kc[h], j - kbase);
        } else {
#pragma unroll
          for (int h = 0; h < NH; ++h) {
            int pos = j * BKV + h * HALF;
            if (pos >= u.kv_len) pos = j * BKV;
            pcache[h] = (int)(row0 + (long long)bt[pos / p.block_size] * p.block_size + pos % p.block_size);
          }
        }
        if (lane == 0) {
#pragma unroll
          for (int h = 0; h < NH; ++h) {
            if (j * BKV + h * HALF >= u.kv_len) continue;
#pragma unroll
            for (int c = 0; c < DH / 64; ++c) {
              tma_prefetch_2d(&tmK, c * 64, pcache[h]);
              tma_prefetch_2d(&tmV, c * 64, pcache[h]);
            }
          }
        }
        __syncwarp();
      };
      int kj = sg.y;
      for (int j = sg.y; j < sg.z && j < sg.y + RDKV_ATTN_PPF; ++j) prefetch(j + LEAD);
      for (; kj < sg.z && kj < sg.y + LEAD; ++kj) load(true, kj);
      for (int j = sg.y; j < sg.z; ++j) {
        load(false, j);
        if (kj < sg.z) {
          load(true, kj);
          prefetch(kj + RDKV_ATTN_PPF);
          ++kj;
        }
      }
    } else if constexpr (ISSUE_BY_KIND) {
      // ---------------------------------------------------------- TMA producer + P.V_1 issuer
      // The first ST tiles are requested up front; afterwards tile j + ST goes into the stage
      // that P.V_0(j) and P.V_1(j) release, right after this thread issued P.V_1(j).
      const int4 sg = seg0;
      const Unit u = unit_at(sg.x);
      const int nt = sg.z - sg.y;
      const bool mine1 = nt > 0 && u.n_q > 1;
      const long long row0 = (long long)u.kvh * (p.head_stride / DH);
      const int* bt = p.block_table + (long long)u.s * p.bt_stride;
      int my_rows[NH] = {};
      auto produce = [&](int jl) {  // whole warp, jl = 0, 1, 2, ... in order
        const int j = sg.y + jl;
        if ((jl & 31) == 0 && j + lane < sg.z) {
#pragma unroll
          for (int h = 0; h < NH; ++h) {
            int pos = (j + lane) * BKV + h * HALF;
            if (pos >= u.kv_len) pos = (j + lane) * BKV;  // masked half: any valid, finite block
            my_rows[h] = (int)(row0 + (long long)bt[pos / p.block_size] * p.block_size + pos % p.block_size);
          }
        }
        int rows[NH];
#pragma unroll
        for (int h = 0; h < NH; ++h) rows[h] = __shfl_sync(0xffffffffu, my_rows[h], jl & 31);
        if (lane == 0) {
          const int st = jl % ST;
          TRACE(4, jl, 0);
          issuer_wait(&kv_empty[st], ((jl / ST) & 1) ^ 1);  // prompt: P.V_1 follows on this thread
          TRACE(4, jl, 1);
          mbar_arrive_expect_tx(&k_full[st], C::KB);
#pragma unroll
          for (int c = 0; c < DH / 64; ++c)
#pragma unroll
            for (int h = 0; h < NH; ++h)
              tma_load_2d_nohint(&tmK, &k_full[st], smem + C::OFF_K + st * C::KB + c * (BKV * 128) + h * (HALF * 128),
                                 c * 64, rows[h]);
          mbar_arrive_expect_tx(&v_full[st], C::KB);
#pragma unroll
          for (int c = 0; c < DH / 64; ++c)
#pragma unroll
            for (int h = 0; h < NH; ++h)
              tma_load_2d_nohint(&tmV, &v_full[st], smem + C::OFF_V + st * C::VKB + c * (BKV * 128) + h * (HALF * 128),
                                 c * 64, rows[h]);
        }
        __syncwarp();
      };
      for (int jl = 0; jl < nt && jl < ST; ++jl) produce(jl);
      for (int j = 0; j < nt; ++j) {
        if (lane == 0) pv_step(1, j, mine1);
        __syncwarp();
        if (j + ST < nt) produce(j + ST);
      }
    } else {
    // ------------------------------------------------------------ TMA producer
    // The whole warp walks the tiles: every 32 tiles each lane resolves one
    // tile's two block-table rows (32 global loads in parallel instead of a
    // dependent load per tile on the issue path); lane 0 issues the TMA.
    int it = 0;  // stage counter over every tile of every segment
    for (int k = 0; k < nseg; ++k) {
      const int4 sg = seg_at(k);
      const Unit u = unit_at(sg.x);
      const long long row0 = (long long)u.kvh * (p.head_stride / DH);  // first row of this head in the plane view
      const int* bt = p.block_table + (long long)u.s * p.bt_stride;
      int my_rows[NH] = {};
      for (int j = sg.y; j < sg.z; ++j, ++it) {
        if (((j - sg.y) & 31) == 0 && j + lane < sg.z) {
#pragma unroll
          for (int h = 0; h < NH; ++h) {
            int pos = (j + lane) * BKV + h * HALF;
            if (pos >= u.kv_len) pos = (j + lane) * BKV;  // masked half: any valid, finite block
            my_rows[h] = (int)(row0 + (long long)bt[pos / p.block_size] * p.block_size + pos % p.block_size);
          }
        }
        int rows[NH];
#pragma unroll
        for (int h = 0; h < NH; ++h) rows[h] = __shfl_sync(0xffffffffu, my_rows[h], (j - sg.y) & 31);
        if (lane == 0) {
          const int st = it % ST;
          const uint64_t pol_kv = policy_evict_first();
          TRACE(4, it, 0);
          mbar_wait_sleep(&kv_empty[st], ((it / ST) & 1) ^ 1);
          TRACE(4, it, 1);
          mbar_arrive_expect_tx(&k_full[st], C::KB);
#pragma unroll
          for (int c = 0; c < DH / 64; ++c)
#pragma unroll
            for (int h = 0; h < NH; ++h)
              if (p.kv_evict_first)  // a streamed K/V tile is read once: keep L2 for the prefetched weights
                tma_load_2d(&tmK, &k_full[st], smem + C::OFF_K + st * C::KB + c * (BKV * 128) + h * (HALF * 128),
                            c * 64, rows[h], pol_kv);
              else
                tma_load_2d_nohint(&tmK, &k_full[st], smem + C::OFF_K + st * C::KB + c * (BKV * 128) + h * (HALF * 128),
                                   c * 64, rows[h]);
          mbar_arrive_expect_tx(&v_full[st], C::KB);
#pragma unroll
          for (int c = 0; c < DH / 64; ++c)
#pragma unroll
            for (int h = 0; h < NH; ++h)
              if (p.kv_evict_first)  // a streamed K/V tile is read once: keep L2 for the prefetched weights
                tma_load_2d(&tmV, &v_full[st], smem + C::OFF_V + st * C::VKB + c * (BKV * 128) + h * (HALF * 128),
                            c * 64, rows[h], pol_kv);
              else
                tma_load_2d_nohint(&tmV, &v_full[st], smem + C::OFF_V + st * C::VKB + c * (BKV * 128) + h * (HALF * 128),
                                   c * 64, rows[h]);
          // the smem ring holds only STAGES tiles and a stage is refilled only after its
          // P.V retired: with the KV stream coming from HBM under full load (~4.5k cycles
          // latency measured) the ring alone runs dry, so warm L2 RDKV_ATTN_PF tiles ahead
          if (RDKV_ATTN_PF > 0 && j + RDKV_ATTN_PF < sg.z) {
            const int jp = j + RDKV_ATTN_PF;
#pragma unroll
            for (int h = 0; h < NH; ++h) {
              int pos = jp * BKV + h * HALF;
              if (pos >= u.kv_len) continue;
              const int prow = (int)(row0 + (long long)bt[pos / p.block_size] * p.block_size + pos % p.block_size);
#pragma unroll
              for (int c = 0; c < DH / 64; ++c) {
                tma_prefetch_2d(&tmK, c * 64, prow);
                tma_prefetch_2d(&tmV, c * 64, prow);
              }
            }
          }
        }
        __syncwarp();
      }
    }
    }
  } else if (warp == NS + 1 || warp == NS + 2) {
    if constexpr (PP) {
      // ---------------------------------------------------------- MMA issuer (ping-pong)
      // One thread issues for both Q tiles in the order P.V_0(j), Q.K^T_0(j+1), P.V_1(j),
      // Q.K^T_1(j+1): the tensor pipe executes in issue order, so Q.K^T_i(j+1) overwrites
      // S_i (= P_i) only after P.V_i(j) has read P_i, and S_i(j+1) landing tells the softmax
      // that O_i is idle.  While softmax 0 works on S_0(j) the pipe runs tile 1's P.V and
      // Q.K^T and vice versa.
      if (warp == NS + 1 && lane == 0) {
        constexpr uint32_t idesc_qk = idesc_bf16_f32(ROWS, BKV);
        constexpr uint32_t idesc_pv = idesc_bf16_f32(ROWS, DH) | (1u << 16);  // B (V) is MN-major
        const int4 sg = seg0;
        const int nt = sg.z - sg.y;
        const int nq = unit_at(sg.x).n_q;
        auto qk = [&](int i, int jl) {  // S_i = Q_i . K(jl)^T
          const uint32_t qa = sb + C::OFF_Q + i * C::QB;
          const uint32_t ka = sb + C::OFF_K + (jl % KST) * C::KB;
          const uint32_t tS = tmem + C::COL_S + i * BKV;
#pragma unroll
          for (int kk = 0; kk < DH / 16; ++kk) {
            const uint32_t sub = (kk & 3) * 32;
            umma_bf16(tS, desc_k(qa + (kk >> 2) * (ROWS * 128) + sub), desc_k(ka + (kk >> 2) * (BKV * 128) + sub),
                      idesc_qk, kk > 0 ? 1u : 0u);
          }
          umma_commit(&s_full[i]);
          if (jl + 1 == nt) umma_commit(&q_empty[i]);  // the segment's last Q_i.K^T
        };
        if (nt > 0 && nq > 0) {
          for (int i = 0; i < nq; ++i) issuer_wait(&q_full[i], 0);
          issuer_wait(&k_full[0], 0);
          tc_fence_after();
          for (int i = 0; i < nq; ++i) qk(i, 0);
          umma_commit(&kv_empty[0]);
          for (int jl = 0; jl < nt; ++jl) {
            const int vs = jl % VST;
            const uint32_t va = sb + C::OFF_V + vs * C::VKB;
            for (int i = 0; i < nq; ++i) {
              issuer_wait(pf(i, jl), od_par(jl));
              if (i == 0) issuer_wait(&v_full[vs], (jl / VST) & 1);
              TRACE(2 + i, jl, 4);
              tc_fence_after();
              const uint32_t tO = tmem + C::COL_O + i * C::OW, tP = tmem + C::COL_P + i * C::P_STRIDE;
#pragma unroll
              for (int kk = 0; kk < BKV / 16; ++kk) {  // O_i (+)= P_i . V(jl); each key half's P inside its S columns
                const uint32_t pcol = (kk / (KH / 16)) * KH + (kk % (KH / 16)) * 8;
                umma_bf16_ts(tO, tP + pcol, desc_mn(va + kk * 2048, BKV * 128), idesc_pv, (jl > 0 || kk > 0) ? 1u : 0u);
              }
              umma_commit(od(i, jl));
              TRACE(2 + i, jl, 1);
              if (jl + 1 < nt) {
                if (i == 0) issuer_wait(&k_full[(jl + 1) % KST], ((jl + 1) / KST) & 1);
                tc_fence_after();
                qk(i, jl + 1);
                TRACE(2 + i, jl, 0);
              }
            }
            umma_commit(&v_empty[vs]);
            if (jl + 1 < nt) umma_commit(&kv_empty[(jl + 1) % KST]);
          }
        }
      }
    } else if constexpr (ISSUE_BY_KIND) {
      // ---------------------------------------------------------- Q.K^T issuers
      // warp NS+1+i issues Q.K^T_i of every tile; the P.V of both Q tiles is issued by the
      // Q-loader warp once Q is requested (below).  Separate Q.K^T and P.V streams touch
      // disjoint TMEM (S vs P / O), so their relative order does not matter: Q.K^T_i(j+1)
      // goes out as soon as the softmax has read S_i(j), never queued behind the P.V of a
      // tile whose softmax is still running, and each issuer's barrier-observation latency
      // (~90 cycles per satisfied try_wait) overlaps the other issuers' MMAs.
      const int i = warp - NS - 1;
      if (lane == 0) {
        constexpr uint32_t idesc_qk = idesc_bf16_f32(ROWS, BKV);
        const int4 sg = seg0;
        const int nt = sg.z - sg.y;
        if (nt > 0 && i < unit_at(sg.x).n_q) {
          issuer_wait(&q_full[i], 0);
          const uint32_t qa = sb + C::OFF_Q + i * C::QB;
          const uint32_t tS = tmem + C::COL_S + i * BKV;
          const bool q_in_tmem = C::QTMEM && i == 0;
          if (q_in_tmem) {  // stage Q_0 in TMEM: one 128 x 16 slice per K = 16 step, same descriptors as the MMA
            tc_fence_after();
#pragma unroll
            for (int kk = 0; kk < DH / 16; ++kk)
              tmem_cp_128x256b(tmem + C::COL_Q0 + kk * 8, desc_k(qa + (kk >> 2) * (ROWS * 128) + (kk & 3) * 32));
          }
          for (int j = 0; j < nt; ++j) {
            const int st = j % ST;
            issuer_wait(&k_full[st], (j / ST) & 1);
            if (j > 0) issuer_wait(&s_empty[i], (j - 1) & 1);  // the softmax read S_i(j-1)
            TRACE(2 + i, j, 2);
            tc_fence_after();
            const uint32_t ka = sb + C::OFF_K + st * C::KB;
            if (q_in_tmem) {
#pragma unroll
              for (int kk = 0; kk < DH / 16; ++kk)
                umma_bf16_ts(tS, tmem + C::COL_Q0 + kk * 8, desc_k(ka + (kk >> 2) * (BKV * 128) + (kk & 3) * 32),
                             idesc_qk, kk > 0 ? 1u : 0u);
            } else {
#pragma unroll
              for (int kk = 0; kk < DH / 16; ++kk) {
                const uint32_t sub = (kk & 3) * 32;
                umma_bf16(tS, desc_k(qa + (kk >> 2) * (ROWS * 128) + sub), desc_k(ka + (kk >> 2) * (BKV * 128) + sub),
                          idesc_qk, kk > 0 ? 1u : 0u);
              }
            }
            umma_commit(&s_full[i]);
            if (j + 1 == nt) umma_commit(&q_empty[i]);
            TRACE(2 + i, j, 0);
          }
        }
      }
    } else {
    // ------------------------------------------------------------ MMA issuers
    // one issuing thread per Q tile, so neither softmax warpgroup ever waits on
    // the other's progress (their exp2 phases drift apart and overlap)
    const int i = warp - NS - 1;
    if (lane == 0) {
      constexpr uint32_t idesc_qk = idesc_bf16_f32(ROWS, BKV);
      constexpr uint32_t idesc_pv = idesc_bf16_f32(ROWS, DH) | (1u << 16);  // B (V) is MN-major
      const uint32_t qa = sb + C::OFF_Q + i * C::QB;
      const uint32_t tS = tmem + C::COL_S + i * BKV, tO = tmem + C::COL_O + i * C::OW;
      const uint32_t tP = tmem + C::COL_P + i * C::P_STRIDE;
      auto issue_qk = [&](int stg, bool last) {  // S_i = Q_i . K^T of the tile in stage stg
        const uint32_t ka = sb + C::OFF_K + stg * C::KB;
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) {
          const uint32_t sub = (kk & 3) * 32;
          umma_bf16(tS, desc_k(qa + (kk >> 2) * (ROWS * 128) + sub), desc_k(ka + (kk >> 2) * (BKV * 128) + sub),
                    idesc_qk, kk > 0 ? 1u : 0u);
        }
        umma_commit(&s_full[i]);
        if (last) umma_commit(&q_empty[i]);  // Q_i may be overwritten by the next segment's
      };
      int it = 0, ti = 0, qi = 0;  // stage counter, this Q tile's tiles, this Q tile's segments
      for (int k = 0; k < nseg; ++k) {
        const int4 sg = seg_at(k);
        const int nt = sg.z - sg.y;
        if (nt == 0) continue;
        if (i >= unit_at(sg.x).n_q) {  // no Q tile i in this unit: release its stages
          for (int j = 0; j < nt; ++j, ++it) {
            if constexpr (SPLIT) {
              issuer_wait(&k_full[it % ST], (it / ST) & 1);
              mbar_arrive(&kv_empty[it % ST]);
              issuer_wait(&v_full[it % ST], (it / ST) & 1);
              mbar_arrive(&v_empty[it % ST]);
            } else {
              issuer_wait(&v_full[it % ST], (it / ST) & 1);
              mbar_arrive(&kv_empty[it % ST]);
            }
          }
          continue;
        }
        TRACE(2 + i, ti, 2);
        issuer_wait(&q_full[i], qi & 1);
        ++qi;
        TRACE(2 + i, ti, 3);
        issuer_wait(&k_full[it % ST], (it / ST) & 1);
        TRACE(2 + i, ti, 4);
        if (!C::ALIAS && ti > 0) issuer_wait(&s_empty[i], (ti - 1) & 1);
        TRACE(2 + i, ti, 5);
        tc_fence_after();
        issue_qk(it % ST, nt == 1);
        if constexpr (SPLIT) umma_commit(&kv_empty[it % ST]);  // K(j) consumed by this Q.K^T
        for (int j = 0; j < nt; ++j, ++it, ++ti) {
          const int st = it % ST;
          const bool more = j + 1 < nt;
          if (!C::ALIAS && more) {  // next S_i while the softmax still works on this tile
            issuer_wait(&k_full[(it + 1) % ST], ((it + 1) / ST) & 1);
            if (j > 0) TRACE(2 + i, ti, 2);
            issuer_wait(&s_empty[i], ti & 1);
            if (j > 0) TRACE(2 + i, ti, 3);
            tc_fence_after();
            issue_qk((it + 1) % ST, j + 2 == nt);
            if constexpr (SPLIT) umma_commit(&kv_empty[(it + 1) % ST]);
            TRACE(2 + i, ti, 0);
          }
          issuer_wait(&v_full[st], (it / ST) & 1);
          if (j > 0) TRACE(2 + i, ti, 4);
          issuer_wait(pf(i, ti), od_par(ti));
          if (j > 0) TRACE(2 + i, ti, 5);
          tc_fence_after();
          const uint32_t va = sb + C::OFF_V + st * C::VKB;
#pragma unroll
          for (int kk = 0; kk < BKV / 16; ++kk) {  // O_i (+)= P_i . V(j), P_i from TMEM
            // P of keys [16kk, 16kk+16): with P over S each half writes inside its own S columns
            const uint32_t pcol = C::ALIAS ? (kk / (KH / 16)) * KH + (kk % (KH / 16)) * 8 : kk * 8;
            umma_bf16_ts(tO, tP + pcol, desc_mn(va + kk * 2048, BKV * 128), idesc_pv, (j > 0 || kk > 0) ? 1u : 0u);
          }
          if constexpr (C::LSUM) {  // L_i (+)= P_i . ones: the row sums, off the softmax warps
            constexpr uint32_t idesc_l = idesc_bf16_f32(ROWS, 16);
            const uint32_t oa = sb + C::OFF_ONES;
#pragma unroll
            for (int kk = 0; kk < BKV / 16; ++kk)
              umma_bf16_ts(tmem + C::COL_L + i * 16, tP + kk * 8, desc_k(oa + (kk & 3) * 32), idesc_l,
                           (j > 0 || kk > 0) ? 1u : 0u);
          }
          umma_commit(od(i, ti));
          TRACE(2 + i, ti, 1);
          umma_commit(SPLIT ? &v_empty[st] : &kv_empty[st]);
          if (C::ALIAS && more) {  // S_i overwrites P_i only after the P.V above (issue order)
            issuer_wait(&k_full[(it + 1) % ST], ((it + 1) / ST) & 1);
            tc_fence_after();
            issue_qk((it + 1) % ST, j + 2 == nt);
          }
        }
      }
    }
    }
  } else if (warp == NS + 3) {
    // ------------------------------------------------------------ Q loader
    // rows of a Q tile = (token, head of this kv group) pairs, token-major: the
    // box {64 dh, G heads, TPT tokens} lands exactly as [128 rows][128 B] SW128.
    // Rows past the unit's tokens hold other tokens' queries (or TMA zero fill):
    // finite, and their scores only reach their own (discarded) O rows.
    // Stream-K: this warp also publishes the CTA's part (its first segment) once
    // the softmax warps have written it, so they never wait for the release.
    int qn[2] = {0, 0};
    const bool part = SK && nseg > 0 && seg_at(0).w == SEG_PART;
    const int k_pub = part ? min(2, nseg) : -1;  // publish after requesting this many segments' Q
    for (int k = 0; k < nseg; ++k) {
      const int4 sg = seg_at(k);
      if (lane == 0 && sg.z > sg.y) {
        const Unit u = unit_at(sg.x);
        for (int i = 0; i < u.n_q; ++i) {
          TRACE(5, 2 * k + i, 0);
          if (qn[i] > 0) mbar_wait_sleep(&q_empty[i], (qn[i] - 1) & 1);
          TRACE(5, 2 * k + i, 1);
          ++qn[i];
          mbar_arrive_expect_tx(&q_full[i], C::QB);
#pragma unroll
          for (int c = 0; c < DH / 64; ++c)
            tma_load_3d_nohint(&tmQ, &q_full[i], smem + C::OFF_Q + i * C::QB + c * (ROWS * 128), c * 64, u.kvh * G,
                               u.row_base + i * TPT);
        }
      }
      if (k + 1 == k_pub) {
        __syncwarp();
        asm volatile("bar.sync %0, %1;" ::"n"(SK_PUB), "n"(NS * 32 + 32) : "memory");
        if (lane == 0) st_release_gpu(p.sk_flag + blockIdx.x, 1);
      }
      if constexpr (ISSUE_BY_KIND) {  // then issue P.V of Q tile 0 (the producer: Q tile 1)
        // this CTA's share of the next projection's weights into L2 first (a few bulk prefetches)
        __syncwarp();
        l2_prefetch_share(p.l2_next, p.l2_next_bytes, blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z),
                          gridDim.x * gridDim.y * gridDim.z, lane);
        if (lane == 0) {
          const int nt = sg.z - sg.y;
          const bool mine = nt > 0 && unit_at(sg.x).n_q > 0;
          for (int j = 0; j < nt; ++j) pv_step(0, j, mine);
        }
        __syncwarp();
        continue;
      }
      if (k == 0) {  // Q requested: pull the O projection's weights into L2 meanwhile
        __syncwarp();
        l2_prefetch_share(p.l2_next, p.l2_next_bytes, blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z),
                          gridDim.x * gridDim.y * gridDim.z, lane);
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
    float* red = reinterpret_cast<float*>(smem + C::OFF_RED);  // [parity][tile][half][row]
    auto pair_sync = [&]() {
      if constexpr (SPL == 2) asm volatile("bar.sync %0, 64;" ::"r"(1 + i * 4 + quad) : "memory");
    };
    auto exchange = [&](float v, int parity, bool use_max) {  // combine with the partner half of this row
      if constexpr (SPL == 1) {
        return v;
      } else {
        const int pa = C::RED_PAR == 2 ? parity : 0;
        red[((pa * 2 + i) * 2 + h) * ROWS + r] = v;
        pair_sync();
        const float o = red[((pa * 2 + i) * 2 + (h ^ 1)) * ROWS + r];
        if constexpr (C::RED_PAR == 1) pair_sync();  // both read before either writes the slot again
        return use_max ? fmaxf(v, o) : v + o;
      }
    };
    auto softmax_bar = [&]() { asm volatile("bar.sync %0, %1;" ::"n"(SK_BAR), "n"(NS * 32) : "memory"); };
    constexpr int OH = DH / SPL;  // O columns of this half
    const uint32_t tS = tmem + C::COL_S + i * BKV + h * KH + lane_off;
    const uint32_t tO = tmem + C::COL_O + i * C::OW + h * OH + lane_off;
    // P columns of this half: inside its own S columns when P is written over S
    const uint32_t tP = tmem + C::COL_P + i * C::P_STRIDE + h * (C::ALIAS ? KH : KH / 2) + lane_off;
    const float sl2 = p.scale_log2;
    int ti = 0;  // this Q tile's tiles so far (barrier parities)
    for (int k = 0; k < nseg; ++k) {
      const int4 sg = seg_at(k);
      const Unit u = unit_at(sg.x);
      const int nt = sg.z - sg.y;
      const bool act = i < u.n_q && nt > 0;
      const int nrows = max(0, min(TPT, u.ntok - i * TPT)) * G;
      const bool ok = r < nrows;
      const long long trow = u.row_base + i * TPT + (ok ? r : 0) / G;  // token row in [0, T)
      const int head = u.kvh * G + (ok ? r : 0) % G;
      float m_used = -INFINITY;  // row max the P values and O are scaled to (log2 domain)
      float l = 0.f;             // this half's row sum at scale m_used
      if (act) {
        // padded rows pretend to be the last valid position so no row is fully masked
        const int qpos = ok ? u.pos0 + i * TPT + r / G : u.kv_len - 1;
        // a warp none of whose rows is a real query row (decode: G valid rows of 128) only
        // keeps the handshakes: its P rows feed O rows that are never stored
        const bool idle = IDLE_SKIP && !PP && SPL == 1 && !C::LSUM && !C::ONES && !__any_sync(0xffffffffu, ok);
        TRACE(i, ti, 6);
        for (int j = 0; j < nt; ++j, ++ti) {
          mbar_wait(&s_full[i], ti & 1);
          tc_fence_after();
          if (idle) {
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_empty[i]);
            // as below: no p_full arrival for tile ti before P.V(ti - P_BUFS) retired, or the
            // early arrival would complete the previous tile's phase
            const int tw = ti - C::P_BUFS;
            if (!PP && tw >= ti - j) {
              mbar_wait(od(i, tw), od_par(tw));
              tc_fence_after();
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(pf(i, ti));
            continue;
          }
          if (j == 0) TRACE(i, ti, 7);
          if (j + 1 < nt) TRACE(i, ti, 2);
          uint32_t sv[KH];
#pragma unroll
          for (int c = 0; c < KH / 32; ++c) tmem_ld32(tS + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&sv[c * 32]));
          tmem_ld_wait();
          tc_fence_before();
          __syncwarp();
          if (!PP && lane == 0) mbar_arrive(&s_empty[i]);
          const int lim = qpos - (sg.y + j) * BKV - h * KH;  // key e of this half visible iff e <= lim
          if (lim < KH - 1) {
#pragma unroll
            for (int e = 0; e < KH; ++e)
              if (e > lim) sv[e] = __float_as_uint(-INFINITY);
          }
          // P = 2^(S*scale - m_used) as bf16 pairs (registers), row sum in fp32; this
          // overlaps P_i.V(j-1), which still reads the P_i buffer.  With `track`, the
          // tile's row max is taken in the same pass (speculative: P at the current
          // reference max, redone below in the rare case that the max moved).
          float s0, s1, s2, s3;
          uint32_t pk[KH / 2];
          float mx4[4];
          auto exp_pass = [&](float nb, bool track) {
            s0 = s1 = s2 = s3 = 0.f;
#pragma unroll
            for (int e = 0; e < KH; e += 4) {
              if (track) {
                mx4[(e / 4) & 3] = fmax3(mx4[(e / 4) & 3], __uint_as_float(sv[e]), __uint_as_float(sv[e + 1]));
                mx4[(e / 4 + 2) & 3] = fmax3(mx4[(e / 4 + 2) & 3], __uint_as_float(sv[e + 2]), __uint_as_float(sv[e + 3]));
              }
              float x0, x1, x2, x3;
              ffma2(x0, x1, __uint_as_float(sv[e]), __uint_as_float(sv[e + 1]), sl2, sl2, nb, nb);
              ffma2(x2, x3, __uint_as_float(sv[e + 2]), __uint_as_float(sv[e + 3]), sl2, sl2, nb, nb);
              if (((e / 4) * 3) % 8 < EMU_OF_8) {  // this group of 4 on the FMA pipe
                exp2_emu2(x0, x1, x0, x1);
                exp2_emu2(x2, x3, x2, x3);
              } else {  // on the MUFU
                x0 = ex2_approx(x0);
                x1 = ex2_approx(x1);
                x2 = ex2_approx(x2);
                x3 = ex2_approx(x3);
              }
              if constexpr (!C::LSUM && !C::ONES) {
                fadd2(s0, s1, s0, s1, x0, x1);
                fadd2(s2, s3, s2, s3, x2, x3);
              }
              pk[e / 2] = pack_bf16(x0, x1);
              pk[e / 2 + 1] = pack_bf16(x2, x3);
            }
          };
          mx4[0] = mx4[1] = mx4[2] = mx4[3] = -INFINITY;
          // speculative pass once the reference max is finite (every tile after the first)
          const bool spec = SPEC && __all_sync(0xffffffffu, m_used != -INFINITY);
          if (spec) {
            exp_pass(-m_used, true);
          } else {
#pragma unroll
            for (int e = 0; e < KH; e += 8)
#pragma unroll
              for (int q = 0; q < 4; ++q)
                mx4[q] = fmax3(mx4[q], __uint_as_float(sv[e + 2 * q]), __uint_as_float(sv[e + 2 * q + 1]));
          }
          const float mt = exchange(fmax3(fmaxf(mx4[0], mx4[1]), mx4[2], mx4[3]), ti & 1, true) * sl2;
          // lazy rescale: move the reference max only when it grew by more than 2^8
          const bool need = mt > m_used + RESCALE_LOG2;
          const bool any_need = __any_sync(0xffffffffu, need);
          const bool rescale = any_need && j > 0;
          float f = 1.f;
          if (need) {
            f = ex2_approx(m_used - mt);  // 0 when m_used = -inf
            l *= f;
            m_used = mt;
          }
          if (!spec || any_need) exp_pass(m_used == -INFINITY ? 0.f : -m_used, false);
          // P_i (and O_i) are free once P_i.V(j-1) has retired (implied by s_full when P aliases S)
          if (j + 1 < nt) TRACE(i, ti, 3);
          // (P double-buffered: P.V_i(j-2) frees this tile's buffer; a rescale of O needs P.V_i(j-1))
          if (!PP) {  // PP: S_i(j) landing already implies P.V_i(j-1) retired
            const int tw = rescale ? ti - 1 : ti - C::P_BUFS;
            if (tw >= ti - j) {  // a P.V of this segment
              mbar_wait(od(i, tw), od_par(tw));
              tc_fence_after();
            }
          }
          if (j + 1 < nt) TRACE(i, ti, 4);
          const uint32_t tPb = tP + (ti % C::P_BUFS) * (BKV / 2);
#pragma unroll
          for (int c = 0; c < KH / 64; ++c) tmem_st32(tPb + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&pk[c * 32]));
          l += (s0 + s1) + (s2 + s3);
          if (C::LSUM && rescale) {  // L_i (tensor-core row sums) at the new scale too
            uint32_t lv[16];
            tmem_ld16(tmem + C::COL_L + i * 16 + lane_off, lv);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 16; ++e) lv[e] = __float_as_uint(__uint_as_float(lv[e]) * f);
            tmem_st16(tmem + C::COL_L + i * 16 + lane_off, lv);
          }
          if (C::ONES && rescale) {  // the ones-column row sums at the new scale too
            uint32_t lv[16];
            tmem_ld16(tO + DH, lv);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 16; ++e) lv[e] = __float_as_uint(__uint_as_float(lv[e]) * f);
            tmem_st16(tO + DH, lv);
          }
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
          if (lane == 0) mbar_arrive(pf(i, ti));
          TRACE(i, ti, 0);
        }
        l = exchange(l, ti & 1, false);  // the parity the last tile did NOT use
        TRACE(i, ti, 1);
        mbar_wait(od(i, ti - 1), od_par(ti - 1));
        tc_fence_after();
        if constexpr (C::LSUM) {  // the row sum of the bf16 P the tensor cores multiplied V by
          uint32_t lv[16];
          tmem_ld16(tmem + C::COL_L + i * 16 + lane_off, lv);
          tmem_ld_wait();
          l = __uint_as_float(lv[0]);
        }
        if constexpr (C::ONES) {  // the ones columns of O_i: the row sum of the bf16 P
          uint32_t lv[16];
          tmem_ld16(tO + DH, lv);
          tmem_ld_wait();
          l = __uint_as_float(lv[0]);
        }
        TRACE(i, ti, 2);
      }
      // ---- the segment's O rows (every lane of an active tile joins the .sync.aligned TMEM loads)
      if (sg.w == SEG_HEAD) {  // wait until every later part of this unit is published
        if (threadIdx.x == 0) {
          const long long W = Wtot;
          const long long uend = sk_bound(blockIdx.x + 1, W, gridDim.x) + (u.n_all - sg.z);
          for (int c = blockIdx.x + 1; c < (int)gridDim.x && sk_bound(c, W, gridDim.x) < uend; ++c) {
            if (sk_bound(c + 1, W, gridDim.x) == sk_bound(c, W, gridDim.x)) continue;
            long long spins = 0;
            while (ld_acquire_gpu(p.sk_flag + c) == 0)
              if (++spins > (1ll << 31)) __trap();
          }
        }
        softmax_bar();
      }
      if (act) {
        if (sg.w == SEG_PART) {
          // unnormalised partial at scale m_used for the unit's head CTA; slot layout
          // [dh/4][256 rows][4] so a warp's float4 stores cover 512 contiguous bytes
          float4* dst = reinterpret_cast<float4*>(p.sk_o + (long long)blockIdx.x * 2 * ROWS * DH) + i * ROWS + r;
#pragma unroll
          for (int c = 0; c < DH / 32; ++c) {
            uint32_t ov[32];
            tmem_ld32(tO + c * 32, ov);
            tmem_ld_wait();
            if (ok)
#pragma unroll
              for (int e = 0; e < 8; ++e)
                dst[(c * 8 + e) * 2 * ROWS] = make_float4(__uint_as_float(ov[4 * e]), __uint_as_float(ov[4 * e + 1]),
                                                          __uint_as_float(ov[4 * e + 2]), __uint_as_float(ov[4 * e + 3]));
          }
          if (ok) p.sk_ml[(long long)blockIdx.x * 2 * ROWS + i * ROWS + r] = make_float2(m_used, l);
        } else {
          // merge the later parts (SEG_HEAD): O = sum_c o_c 2^(m_c - M), L likewise
          float M = m_used, L = 0.f;
          long long W = 0, uend = 0;
          if (sg.w == SEG_HEAD) {
            W = Wtot;
            uend = sk_bound(blockIdx.x + 1, W, gridDim.x) + (u.n_all - sg.z);
          }
          auto for_parts = [&](auto&& fn) {  // fn(slot row index, part CTA)
            if (sg.w != SEG_HEAD || !ok) return;
            for (int c = blockIdx.x + 1; c < (int)gridDim.x && sk_bound(c, W, gridDim.x) < uend; ++c)
              if (sk_bound(c + 1, W, gridDim.x) > sk_bound(c, W, gridDim.x)) fn((long long)c * 2 * ROWS + i * ROWS + r, c);
          };
          for_parts([&](long long slot, int) { M = fmaxf(M, __ldcg(&p.sk_ml[slot].x)); });
          const float w0 = M == m_used ? 1.f : ex2_approx(m_used - M);
          L = l * w0;
          for_parts([&](long long slot, int) {
            const float2 ml = __ldcg(&p.sk_ml[slot]);
            L += ml.y * ex2_approx(ml.x - M);
          });
          const float inv = L > 0.f ? 1.f / L : 0.f;
#pragma unroll
          for (int c = 0; c < OH / 32; ++c) {
            uint32_t ov[32];
            tmem_ld32(tO + c * 32, ov);
            tmem_ld_wait();
            if (!ok) continue;
            const int col = h * OH + c * 32;
            if (sg.w == SEG_SPLIT) {
              // unnormalised partial at scale m_used; combined by attn_split_combine_kernel
              const int ks = ks0;
              float4* dst = reinterpret_cast<float4*>(p.split_o + (((long long)ks * p.n_tokens + trow) * p.hq + head) * DH + col);
#pragma unroll
              for (int e = 0; e < 8; ++e)
                dst[e] = make_float4(__uint_as_float(ov[4 * e]), __uint_as_float(ov[4 * e + 1]),
                                     __uint_as_float(ov[4 * e + 2]), __uint_as_float(ov[4 * e + 3]));
              continue;
            }
            float a[32];
#pragma unroll
            for (int e = 0; e < 32; ++e) a[e] = __uint_as_float(ov[e]) * w0;
            for_parts([&](long long slot, int pc) {
              const float wc = ex2_approx(__ldcg(&p.sk_ml[slot].x) - M);
              const float4* src =
                  reinterpret_cast<const float4*>(p.sk_o + (long long)pc * 2 * ROWS * DH) + (slot - (long long)pc * 2 * ROWS);
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                const float4 t = __ldcg(src + (col / 4 + e) * 2 * ROWS);
                a[4 * e] += t.x * wc;
                a[4 * e + 1] += t.y * wc;
                a[4 * e + 2] += t.z * wc;
                a[4 * e + 3] += t.w * wc;
              }
            });
            uint4* dst = reinterpret_cast<uint4*>(p.o + trow * p.ldo + (long long)head * DH + col);
#pragma unroll
            for (int e = 0; e < 4; ++e)
              dst[e] = make_uint4(pack_bf16(a[8 * e] * inv, a[8 * e + 1] * inv), pack_bf16(a[8 * e + 2] * inv, a[8 * e + 3] * inv),
                                  pack_bf16(a[8 * e + 4] * inv, a[8 * e + 5] * inv), pack_bf16(a[8 * e + 6] * inv, a[8 * e + 7] * inv));
          }
          if (ok && h == 0 && sg.w == SEG_SPLIT) {
            const int ks = ks0;
            p.split_ml[((long long)ks * p.n_tokens + trow) * p.hq + head] = make_float2(m_used, l);
          }
        }
      } else if (sg.w == SEG_SPLIT && nt == 0 && i < u.n_q && ok && h == 0) {
        // empty split: mark the partial as absent
        const int ks = ks0;
        p.split_ml[((long long)ks * p.n_tokens + trow) * p.hq + head] = make_float2(-INFINITY, 0.f);
      }
      if (sg.w == SEG_PART) {  // rows written: the Q-loader warp publishes them (release store)
        TRACE(i, ti, 3);
        asm volatile("bar.sync %0, %1;" ::"n"(SK_PUB), "n"(NS * 32 + 32) : "memory");
        TRACE(i, ti, 4);
      } else if (sg.w == SEG_HEAD) {  // consumed: re-arm the parts' flags for the next launch
        softmax_bar();
        if (threadIdx.x == 0) {
          const long long W = Wtot;
          const long long uend = sk_bound(blockIdx.x + 1, W, gridDim.x) + (u.n_all - sg.z);
          for (int c = blockIdx.x + 1; c < (int)gridDim.x && sk_bound(c, W, gridDim.x) < uend; ++c) p.sk_flag[c] = 0;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  CTA_TRACE(3);
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
  if (head >= p.hq || t < p.seq_start[p.seq_off]) return;  // tokens of this launch's sequences only
  // (split loops unrolled: the partials' loads are in flight together — a single-query
  // combine is latency-bound; summation order unchanged, so results are bit-identical)
  float M = -INFINITY;
#pragma unroll 8
  for (int k = 0; k < p.kv_splits; ++k) M = fmaxf(M, p.split_ml[((long long)k * p.n_tokens + t) * p.hq + head].x);
  constexpr int PER = DH / 32;
  float acc[PER] = {};
  float L = 0.f;
#pragma unroll 4  // (8 / 16 measured slower: 14.9 vs 10.0 us per single-query layer)
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

template <int DH, int SPL, bool SK, bool PP = false>
int set_smem_attr() {
  static bool attr = false;
  if (!attr) {
    CUDA_TRY(cudaFuncSetAttribute(attn_tc_kernel<DH, SPL, SK, PP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)CfgOf<DH, SPL, SK, PP>::SMEM));
    attr = true;
  }
  return 0;
}

template <int DH, int SPL, bool PP = false>
int launch_tc(const AttnParams& p, int n_seqs, int max_new, cudaStream_t st) {
  using C = CfgOf<DH, SPL, false, PP>;
  // plane view: rows = hkv * slots, cols = dh
  const long long rows = (long long)p.hkv * (p.head_stride / DH);
  CUtensorMap tk, tv;
  RDKV_TRY(make_tmap(&tk, p.kplane, rows, DH, DH, HALF));
  RDKV_TRY(make_tmap(&tv, p.vplane, rows, DH, DH, HALF));
  CUtensorMap tq;
  RDKV_TRY(make_tmap_q(&tq, p.q, p.n_tokens, p.hq, DH, p.ldq, p.hq / p.hkv, ROWS / (p.hq / p.hkv)));
  const int tok_per_cta = 2 * ROWS / (p.hq / p.hkv);  // two Q tiles per CTA
  const int qblocks = (max_new + tok_per_cta - 1) / tok_per_cta;
  AttnParams q = p;
  q.kv_splits = 1;
  q.n_seqs = n_seqs;
  q.sk_qblocks = qblocks;
  // K/V evict-first only alongside the (opt-in) weight prefetch it protects
  q.kv_evict_first = qblocks == 1 && p.l2_next ? 1 : 0;
  const int ctas = qblocks * p.hkv * n_seqs, sms = num_sms();
  const int max_tiles = (p.max_ctx + C::BKV - 1) / C::BKV;
  // stream-K (opt-in: p.sk_mode) when the unit grid is at least half a wave; measured
  // slower than one CTA per unit on the C2/C3 shapes (profiles/r1_attn_experiments.md)
  if constexpr (SPL == 1 && !PP) {
    if (p.sk_mode && p.sk_o && p.sk_ctas >= sms && ctas * 2 > sms && ctas <= SK_MAXSEG) {
      RDKV_TRY((set_smem_attr<DH, SPL, true>()));
      CUDA_TRY(launch_k(attn_tc_kernel<DH, SPL, true>, dim3(sms), dim3(RolesOf<DH, SPL, true, false>::THREADS),
                        CfgOf<DH, SPL, true, false>::SMEM, st, tk, tv, tq, q));
      CUDA_TRY(cudaGetLastError());
      return 0;
    }
  }
  // More than one wave whose last wave would leave many SMs idle (the C2 batch: 256
  // units on 148 SMs): the sequences that fill whole waves run one CTA per unit, the
  // rest split their KV range in 4 and are merged by the combine kernel; launched
  // back to back (PDL), the small split CTAs fill the SMs as the first wave drains.
  static const bool tail_env = [] {
    const char* e = std::getenv("RDKV_ATTN_TAIL");  // "0": whole units only (A/B)
    return !(e && e[0] == '0');
  }();
  const int ups = qblocks * p.hkv;  // units per sequence
  const int s_a = ups > 0 ? (ctas / sms) * sms / ups : 0;
  const double last = (double)(ctas % sms) / sms;
  constexpr int KT = 4;
  // (only when a split keeps >= 8 KV tiles: a CTA's fixed cost — TMEM / barrier setup,
  // pipeline fill, the O store — is several tiles' worth; the C2 batch, 21 tiles per
  // unit, measured 77 -> 103 us with 5-tile splits, a 41-tile dh=128 batch 212 -> 189 us)
  static const int tail_min = [] {  // KV tiles a split must keep (RDKV_ATTN_TAIL_MIN, A/B)
    const char* e = std::getenv("RDKV_ATTN_TAIL_MIN");
    return e ? std::atoi(e) : 8;
  }();
  if (tail_env && p.split_o && ctas > sms && last > 0.0 && last < 0.9 && s_a >= 1 && s_a < n_seqs &&
      max_tiles >= tail_min * KT && (size_t)KT * p.n_tokens * p.hq * (DH * 4 + 8) <= p.split_bytes) {
    RDKV_TRY((set_smem_attr<DH, SPL, false, PP>()));
    AttnParams b = q;
    b.seq_off = s_a;
    b.kv_splits = KT;
    b.tail_ctas = s_a * ups;
    const int grid = s_a * ups + (n_seqs - s_a) * ups * KT;
    CUDA_TRY(launch_k(attn_tc_kernel<DH, SPL, false, PP>, dim3(grid), dim3(RolesOf<DH, SPL, false, PP>::THREADS), C::SMEM, st, tk, tv, tq, b));
    CUDA_TRY(launch_k(attn_split_combine_kernel<DH>, dim3(p.n_tokens, (p.hq + 7) / 8), dim3(256), 0, st, b));
    CUDA_TRY(cudaGetLastError());
    return 0;
  }
  // split the KV range when the (query block x kv head x sequence) grid is too
  // small for 148 SMs (single-query TTFT) and scratch is available
  if (p.split_o && ctas * 2 <= sms && max_tiles >= 4) {
    int k = sms / ctas;
    k = k < max_tiles / 2 ? k : max_tiles / 2;
    k = k < 16 ? k : 16;
    if (k >= 2 && (size_t)k * p.n_tokens * p.hq * (DH * 4 + 8) <= p.split_bytes) q.kv_splits = k;
  }
  RDKV_TRY((set_smem_attr<DH, SPL, false, PP>()));
  dim3 grid(qblocks * q.kv_splits, p.hkv, n_seqs);
  CUDA_TRY(launch_k(attn_tc_kernel<DH, SPL, false, PP>, grid, dim3(RolesOf<DH, SPL, false, PP>::THREADS), C::SMEM, st, tk, tv, tq, q));
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
extern "C" RDKV_API int rdkv_debug_attn_cta_trace(long long* out) {
  return cudaMemcpyFromSymbol(out, g_attn_cta, sizeof(g_attn_cta)) == cudaSuccess ? 0 : -8;
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
  // RDKV_ATTN_PP=1: the ping-pong schedule (opt-in: measured slower, 102-107 vs 98-99 us at
  // the C3 shape and 98 vs 93 us with every K/V tile L2-hot — one softmax warp per SMSP at a
  // time needs ~1510 cycles per 128 keys, profiles/r2_attn_experiments.md)
  static const bool pp = [] {
    const char* e = std::getenv("RDKV_ATTN_PP");
    return e && e[0] == '1';
  }();
  // stream-K (opt-in) runs the two-issuer schedule; RDKV_ATTN_SPL=2: two softmax warps per row
  if (pp && !p.sk_mode) return spl == 2 ? launch_tc<128, 2, true>(p, n_seqs, max_new, st)
                                        : launch_tc<128, 1, true>(p, n_seqs, max_new, st);
  return launch_tc<128, 1>(p, n_seqs, max_new, st);  // 64-key tiles at dh = 128: one softmax warp per row
}

}  // namespace rdkv

namespace rdkv {
size_t attention_split_scratch_bytes(int T, int hq, int dh) {
  if (T <= 0) return 0;
  // up to 16 KV splits for small batches (single-query TTFT), 4 for the tail of large ones
  return (size_t)attention_split_cap(T) * T * hq * (dh * 4 + 8);
}

size_t attention_sk_scratch_bytes(int ctas, int dh) {
  const size_t o = (size_t)ctas * 2 * ROWS * dh * 4, ml = (size_t)ctas * 2 * ROWS * 8, fl = (size_t)ctas * 4;
  return o + ml + ((fl + 255) / 256) * 256;
}

void attention_sk_carve(AttnParams& p, void* base, int ctas, int dh) {
  auto* b = static_cast<uint8_t*>(base);
  p.sk_o = reinterpret_cast<float*>(b);
  p.sk_ml = reinterpret_cast<float2*>(b + (size_t)ctas * 2 * ROWS * dh * 4);
  p.sk_flag = reinterpret_cast<int*>(b + (size_t)ctas * 2 * ROWS * dh * 4 + (size_t)ctas * 2 * ROWS * 8);
  p.sk_ctas = ctas;
}

int attention_sk_zero_flags(const AttnParams& p, cudaStream_t st) {
  if (p.sk_flag) CUDA_TRY(cudaMemsetAsync(p.sk_flag, 0, (size_t)p.sk_ctas * 4, st));
  return 0;
}
}  // namespace rdkv
