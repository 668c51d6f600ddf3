// Llama-shaped decoder forward over a batch of sequences with a (possibly
// cached) KV prefix — the device half of document-KV generation (replaces
// codec.synth_blob, codec.py:188-224) and of prefill-with-cached-prefix
// (replaces costs.ttft, costs.py:121-144).
//
// Per layer: RMSNorm -> QKV GEMM (RoPE + KV write epilogue) -> attention ->
// O GEMM (+residual) -> RMSNorm -> gate/up GEMM (SwiGLU epilogue) -> down GEMM
// (+residual).  The last row of each sequence then goes through the final
// RMSNorm, the LM head (fp32 logits) and argmax = the first token.
#include <cmath>
#include <cstdlib>
#include <mutex>
#include <new>
#include <algorithm>
#include <vector>

#include "attention.cuh"
#include "common.cuh"
#include "gemm_tc.cuh"
#include "kernels_misc.cuh"
#include "tp.cuh"

struct rdkv_model {
  rdkv_model_desc d;
  std::vector<const void*> w;  // see rdkv.h for the order
  float* rope = nullptr;        // [max_pos][dh/2] (cos, sin)
  float* ones = nullptr;        // unit gain [hidden] (norm gains folded into the weights)
  int device = 0;
  rdkv_tp_comm* tp = nullptr;  // tensor-parallel group (row-parallel outputs all-reduced), or null
  // measurement (rdkv_profile_*)
  bool prof = false;
  struct Rec {
    int cat;
    cudaEvent_t a, b;
  };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> spare;
  int64_t launches[RDKV_PROF_N] = {};
  double flops[RDKV_PROF_N] = {};
  // forwards may run concurrently on several streams (serving and queue-time
  // generation share the handle): counters and event records are guarded
  std::mutex mu;

  cudaEvent_t event() {
    if (!spare.empty()) {
      cudaEvent_t e = spare.back();
      spare.pop_back();
      return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
  }
};

namespace {
// Brackets one launch: counts it and, when profiling, records events around it.
struct ProfScope {
  rdkv_model* m;
  int cat;
  cudaStream_t st;
  cudaEvent_t a = nullptr;
  ProfScope(rdkv_model* m_, int cat_, cudaStream_t st_, double fl = 0.0) : m(m_), cat(cat_), st(st_) {
    std::lock_guard<std::mutex> g(m->mu);
    m->launches[cat] += 1;
    m->flops[cat] += fl;
    if (m->prof) {
      a = m->event();
      cudaEventRecord(a, st);
    }
  }
  ~ProfScope() {
    if (m->prof) {
      std::lock_guard<std::mutex> g(m->mu);
      cudaEvent_t b = m->event();
      cudaEventRecord(b, st);
      m->recs.push_back({cat, a, b});
    }
  }
};
}  // namespace

namespace rdkv {
namespace {

constexpr size_t kAlign = 256;
inline size_t up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

struct Ws {
  __nv_bfloat16 *x, *h, *q, *o, *a, *hl;
  float* ssq;  // fused-RMSNorm statistics [hidden/32][T]
  void* splitk;
  size_t splitk_bytes;
  void* attn_split;
  size_t attn_split_bytes;
  void* attn_sk;  // stream-K attention partials + flags (num_sms() CTAs)
  void* gemm_sk;  // stream-K CTA-pair GEMM partials + flags (RDKV_GEMM_SK; large M only)
  void* argmax;
  int* counters;  // fused small-M split-K tickets (zeroed at the start of every forward)
};
constexpr int N_SPLITK_COUNTERS = 2048;

size_t ws_layout(const rdkv_model_desc& d, int T, int S, Ws* ws, void* base) {
  const size_t qd = (size_t)d.n_heads * d.head_dim;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += up(bytes);
    return o;
  };
  const size_t ox = take((size_t)T * d.hidden * 2), oh = take((size_t)T * d.hidden * 2);
  const size_t oq = take((size_t)T * qd * 2), oo = take((size_t)T * qd * 2);
  const size_t oa = take((size_t)T * d.ffn * 2), ol = take((size_t)(S > 0 ? S : 1) * d.hidden * 2);
  // split-K scratch for small-M GEMMs (largest of the per-layer shapes and the LM head)
  const int qkv_n = (d.n_heads + 2 * d.kv_heads) * d.head_dim;
  size_t sk = splitk_scratch_bytes(T, qkv_n, d.hidden);
  sk = std::max(sk, splitk_scratch_bytes(T, d.hidden, (int)qd));
  sk = std::max(sk, splitk_scratch_bytes(T, 2 * d.ffn, d.hidden));
  sk = std::max(sk, splitk_scratch_bytes(T, d.hidden, d.ffn));
  sk = std::max(sk, splitk_scratch_bytes(S > 0 ? S : 1, d.vocab, d.hidden));
  const size_t osk = take(sk);
  const size_t ask = attention_split_scratch_bytes(T, d.n_heads, d.head_dim);
  const size_t oask = take(ask);
  const size_t osk_attn = take(attention_sk_scratch_bytes(num_sms(), d.head_dim));
  const size_t gsk = T >= 256 && gemm_sk_mode() > 0 ? gemm_sk_scratch_bytes() : 0;
  const size_t ogsk = take(gsk);
  const size_t oam = take(argmax_scratch_bytes(S));
  const size_t ossq = take((size_t)(d.hidden / 32) * T * sizeof(float));
  const size_t octr = take((size_t)N_SPLITK_COUNTERS * sizeof(int));
  if (ws && base) {
    ws->counters = reinterpret_cast<int*>(static_cast<uint8_t*>(base) + octr);
    ws->ssq = reinterpret_cast<float*>(static_cast<uint8_t*>(base) + ossq);
    ws->argmax = static_cast<uint8_t*>(base) + oam;
    ws->attn_split = ask ? static_cast<uint8_t*>(base) + oask : nullptr;
    ws->attn_split_bytes = ask;
    ws->attn_sk = static_cast<uint8_t*>(base) + osk_attn;
    ws->gemm_sk = gsk ? static_cast<uint8_t*>(base) + ogsk : nullptr;
    ws->splitk = sk ? static_cast<uint8_t*>(base) + osk : nullptr;
    ws->splitk_bytes = sk;
    auto* b = static_cast<uint8_t*>(base);
    ws->x = reinterpret_cast<__nv_bfloat16*>(b + ox);
    ws->h = reinterpret_cast<__nv_bfloat16*>(b + oh);
    ws->q = reinterpret_cast<__nv_bfloat16*>(b + oq);
    ws->o = reinterpret_cast<__nv_bfloat16*>(b + oo);
    ws->a = reinterpret_cast<__nv_bfloat16*>(b + oa);
    ws->hl = reinterpret_cast<__nv_bfloat16*>(b + ol);
  }
  return off;
}

inline const __nv_bfloat16* W(const rdkv_model* m, int i) { return static_cast<const __nv_bfloat16*>(m->w[i]); }
inline const float* G(const rdkv_model* m, int i) { return static_cast<const float*>(m->w[i]); }

}  // namespace
}  // namespace rdkv

using namespace rdkv;

#define LAUNCH(cat, fl, expr)            \
  do {                                   \
    ProfScope _ps(m, (cat), st, (fl));   \
    RDKV_TRY(expr);                      \
  } while (0)

extern "C" {

int rdkv_model_create(const rdkv_model_desc* desc, const void* const* weights, size_t n_weights, rdkv_model** out) {
  if (!desc || !weights || !out) return set_error(RDKV_ERR_ARG, "model_create: null argument");
  const rdkv_model_desc& d = *desc;
  if (d.layers < 1 || d.hidden < 64 || d.n_heads < 1 || d.kv_heads < 1 || d.n_heads % d.kv_heads)
    return set_error(RDKV_ERR_ARG, "model_create: bad dimensions");
  if (d.head_dim != 64 && d.head_dim != 128) return set_error(RDKV_ERR_ARG, "model_create: head_dim must be 64/128");
  if (d.hidden % 64 || d.ffn % 64 || (d.n_heads * d.head_dim) % 64 || d.vocab % 32)
    return set_error(RDKV_ERR_ARG, "model_create: hidden/ffn/heads*dh must be multiples of 64, vocab of 32");
  const size_t need = (size_t)RDKV_WEIGHTS_PER_LAYER * d.layers + 3;
  if (n_weights != need) return set_error(RDKV_ERR_ARG, "model_create: expected %zu weights, got %zu", need, n_weights);
  for (size_t i = 0; i < n_weights; ++i)
    if (!weights[i] || (reinterpret_cast<uintptr_t>(weights[i]) & 15))
      return set_error(RDKV_ERR_ARG, "model_create: weight %zu null or not 16-byte aligned", i);
  auto* m = new (std::nothrow) rdkv_model;
  if (!m) return set_error(RDKV_ERR_ARG, "model_create: out of host memory");
  m->d = d;
  m->w.assign(weights, weights + n_weights);
  cudaGetDevice(&m->device);
  // RoPE table in double precision, rounded once to fp32 (same as the oracle).
  const int half = d.head_dim / 2;
  std::vector<float> tab((size_t)d.max_pos * half * 2);
  for (int p = 0; p < d.max_pos; ++p)
    for (int i = 0; i < half; ++i) {
      const double inv = std::pow((double)d.rope_theta, -2.0 * i / (double)d.head_dim);
      const double a = (double)p * inv;
      tab[((size_t)p * half + i) * 2] = (float)std::cos(a);
      tab[((size_t)p * half + i) * 2 + 1] = (float)std::sin(a);
    }
  const std::vector<float> ones((size_t)d.hidden, 1.0f);
  if (cudaMalloc(&m->rope, tab.size() * sizeof(float)) != cudaSuccess ||
      cudaMemcpy(m->rope, tab.data(), tab.size() * sizeof(float), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMalloc(&m->ones, ones.size() * sizeof(float)) != cudaSuccess ||
      cudaMemcpy(m->ones, ones.data(), ones.size() * sizeof(float), cudaMemcpyHostToDevice) != cudaSuccess) {
    cudaFree(m->rope);
    cudaFree(m->ones);
    delete m;
    return set_error(RDKV_ERR_CUDA, "model_create: rope / gain table upload failed");
  }
  *out = m;
  return 0;
}

void rdkv_model_destroy(rdkv_model* m) {
  if (!m) return;
  for (auto& r : m->recs) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  for (auto e : m->spare) cudaEventDestroy(e);
  cudaFree(m->rope);
  cudaFree(m->ones);
  delete m;
}

size_t rdkv_workspace_bytes(const rdkv_model* m, int n_tokens, int n_seqs) {
  if (!m) return 0;
  return ws_layout(m->d, n_tokens, n_seqs, nullptr, nullptr);
}

namespace {
// PUSH epilogue for all-reduce number `ar` of this forward: this rank's slot in
// every rank's receive buffer of parity ar & 1 (dense rows of `cols`).
rdkv::GemmEpi tp_push_epi(const rdkv::GemmEpi& base, const rdkv_tp_comm* tp, int ar, int cols) {
  rdkv::GemmEpi ep = base;
  ep.out = nullptr;
  ep.ldo = cols;
  ep.norm_gain = nullptr;
  ep.norm_out = nullptr;
  ep.npush = tp->size;
  for (int p = 0; p < tp->size; ++p) ep.push[p] = tp->args.push[ar & 1][p];
  return ep;
}
}  // namespace

int rdkv_forward(rdkv_model* m, const rdkv_batch* b, void* ws_base, size_t ws_bytes, void* stream) {
  if (!m || !b) return set_error(RDKV_ERR_ARG, "forward: null argument");
  const rdkv_model_desc& d = m->d;
  const int T = b->n_tokens, S = b->n_seqs;
  if (T <= 0 || S <= 0) return set_error(RDKV_ERR_ARG, "forward: empty batch");
  if (b->block_size <= 0 || b->kv_slots <= 0 || !b->kv_base) return set_error(RDKV_ERR_ARG, "forward: bad KV pool");
  Ws ws;
  if (ws_layout(d, T, S, &ws, ws_base) > ws_bytes) return set_error(RDKV_ERR_ARG, "forward: workspace too small");
  auto st = static_cast<cudaStream_t>(stream);
  const int dh = d.head_dim, hq = d.n_heads, hkv = d.kv_heads;
  const long long qd = (long long)hq * dh;
  const long long plane = (long long)hkv * b->kv_slots * dh;  // elements per (layer, k|v) plane
  auto* kv = static_cast<__nv_bfloat16*>(b->kv_base);
  static const bool use_tc_attn = [] {
    const char* e = std::getenv("RDKV_ATTN");  // "mma" forces the legacy kernel (A/B measurements)
    return !(e && e[0] == 'm');
  }();

  if (b->flags & RDKV_BATCH_ROW_DETERMINISTIC) {  // no shape-dependent reduction orders
    ws.splitk = nullptr;
    ws.splitk_bytes = 0;
    ws.attn_split = nullptr;
    ws.attn_split_bytes = 0;
    ws.attn_sk = nullptr;
    ws.gemm_sk = nullptr;
  }
  float* gsk_part = nullptr;
  int* gsk_flag = nullptr;
  if (ws.gemm_sk) {  // GEMM stream-K flags start at zero (every launch leaves them zero)
    gsk_part = static_cast<float*>(ws.gemm_sk);
    gsk_flag = reinterpret_cast<int*>(gsk_part + (size_t)num_sms() * 128 * 384);
    CUDA_TRY(cudaMemsetAsync(gsk_flag, 0, (size_t)num_sms() * sizeof(int), st));
  }
  auto set_sk = [&](GemmEpi& e) {
    e.sk_part = gsk_part;
    e.sk_flag = gsk_flag;
    e.sk_slots = num_sms();
  };
  if (ws.attn_sk) {  // stream-K flags start at zero (every launch leaves them zero)
    AttnParams z{};
    attention_sk_carve(z, ws.attn_sk, num_sms(), dh);
    RDKV_TRY(attention_sk_zero_flags(z, st));
  }
  // small batches run the residual GEMMs split-K; their finalize also applies the
  // following RMSNorm, saving a launch per norm
  rdkv_tp_comm* tp = m->tp && m->tp->size > 1 ? m->tp : nullptr;
  const bool o_fused = !tp && gemm_splits(T, d.hidden, (int)qd, ws.splitk_bytes);
  const bool down_fused = !tp && gemm_splits(T, d.hidden, d.ffn, ws.splitk_bytes);
  // norm gains folded into w_qkv / w_gate_up: the attention / MLP norms carry unit gain
  const bool folded = (d.flags & RDKV_MODEL_NORM_FOLDED) != 0;
  auto gain = [&](int i) { return folded ? static_cast<const float*>(m->ones) : G(m, i); };
  // large batches fuse the norms across GEMMs (no rmsnorm launches): the embedding and
  // residual epilogues emit per-row sums of squares, the QKV / gate-up epilogues scale
  const int qkv_n = (int)((hq + 2 * hkv) * dh);
  static const bool fuse_norm_env = [] {
    const char* e = std::getenv("RDKV_FUSED_NORM");  // "0": rmsnorm launches instead (A/B)
    return !(e && e[0] == '0');
  }();
  // RDKV_SMALLM_FUSED=1: the swap-AB split-K GEMMs reduce their partials in-kernel (the last
  // split of each weight tile applies the epilogue: no finalize launches) and the norms use the
  // per-chunk statistics of large batches.  Correct (tests pass with it on) but slower: only the
  // w_tiles last CTAs do the whole epilogue (single-query TTFT 4.50 -> 9.94 ms, decode step
  // 5.22 -> 6.89 ms); the finalize kernels spread it over rows x column chunks.  Off.
  // (RDKV_SMALLM_SSQ=1 with the finalize kernels: correct, measured no faster — decode step
  // 5.20 vs 5.20 ms, single-query TTFT 4.52 vs 4.51 ms.)
  static const bool small_fused_env = [] {
    const char* e = std::getenv("RDKV_SMALLM_FUSED");
    return e && e[0] == '1';
  }();
  static const bool small_ssq_env = [] {
    const char* e = std::getenv("RDKV_SMALLM_SSQ");
    return (e && e[0] == '1') || small_fused_env;
  }();
  int* counters = small_fused_env && !tp ? ws.counters : nullptr;
  if (counters) CUDA_TRY(cudaMemsetAsync(counters, 0, N_SPLITK_COUNTERS * sizeof(int), st));
  const bool split_any = o_fused || down_fused || gemm_splits(T, qkv_n, d.hidden, ws.splitk_bytes) ||
                         gemm_splits(T, 2 * d.ffn, d.hidden, ws.splitk_bytes);
  const bool ssq_path = fuse_norm_env && folded && !tp && d.hidden % 256 == 0 && (small_ssq_env || !split_any);
  LAUNCH(RDKV_PROF_MISC, 0.0, launch_embed(b->tokens, W(m, 0), ws.x, T, d.hidden, d.vocab, st,
                                           ssq_path ? ws.ssq : nullptr));
  int ar = 0;  // all-reduces issued by this forward (2 per layer: parity selects the partial buffer)
  bool h_ready = false;  // ws.h already holds this layer's attention-norm output
  for (int l = 0; l < d.layers; ++l) {
    const int wb = 1 + RDKV_WEIGHTS_PER_LAYER * l;
    __nv_bfloat16* kpl = kv + (2LL * l) * plane;
    __nv_bfloat16* vpl = kv + (2LL * l + 1) * plane;
    // attention block
    if (!h_ready && !ssq_path)
      LAUNCH(RDKV_PROF_MISC, 0.0, launch_rmsnorm(ws.x, d.hidden, nullptr, gain(wb + 0), ws.h, d.hidden, T, d.hidden, d.norm_eps, st));
    GemmEpi eq{};
    eq.counters = counters;
    eq.n_counters = N_SPLITK_COUNTERS;
    eq.splitk_ws = ws.splitk;  // small M: split-K (the finalize handles the norm statistics)
    eq.splitk_bytes = ws.splitk_bytes;
    set_sk(eq);
    if (ssq_path) {
      eq.ssq_in = ws.ssq;
      eq.ssq_parts = d.hidden / 32;
      eq.ssq_dim = d.hidden;
      eq.norm_eps = d.norm_eps;
    }
    eq.q = ws.q;
    eq.ldq = qd;
    eq.kplane = kpl;
    eq.vplane = vpl;
    eq.head_stride = b->kv_slots * dh;
    eq.slot = b->slot;
    eq.pos = b->pos;
    eq.rope = m->rope;
    eq.hq = hq;
    eq.hkv = hkv;
    LAUNCH(RDKV_PROF_QKV, 2.0 * T * (hq + 2 * hkv) * dh * d.hidden,
           launch_gemm(ssq_path ? ws.x : ws.h, d.hidden, W(m, wb + 1), d.hidden, T, qkv_n, d.hidden, EPI_QKV, dh,
                         eq, st));
    // document-KV generation (no logits): the last layer's KV is written by the QKV
    // epilogue above; its attention, O projection and MLP feed nothing
    if (!b->want_logits && l == d.layers - 1) break;
    AttnParams ap{};
    ap.q = ws.q;
    ap.ldq = qd;
    ap.o = ws.o;
    ap.ldo = qd;
    ap.kplane = kpl;
    ap.vplane = vpl;
    ap.head_stride = b->kv_slots * dh;
    ap.seq_start = b->seq_start;
    ap.seq_new = b->seq_new;
    ap.seq_cached = b->seq_cached;
    ap.block_table = b->block_table;
    ap.bt_stride = b->bt_stride;
    ap.block_size = b->block_size;
    ap.hq = hq;
    ap.hkv = hkv;
    ap.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)dh));
    ap.contiguous = b->bt_stride == 1 ? 1 : 0;
    ap.kv_splits = 1;
    ap.n_tokens = T;
    ap.max_ctx = b->max_ctx > 0 ? b->max_ctx : 0;
    if (ws.attn_split && b->max_ctx > 0) {
      const size_t o_bytes = (size_t)attention_split_cap(T) * T * hq * dh * 4;
      ap.split_o = static_cast<float*>(ws.attn_split);
      ap.split_ml = reinterpret_cast<float2*>(static_cast<uint8_t*>(ws.attn_split) + o_bytes);
      ap.split_bytes = ws.attn_split_bytes;
    }
    static const bool attn_sk = [] {
      const char* e = std::getenv("RDKV_ATTN_SK");  // "1": stream-K attention schedule (A/B)
      return e && e[0] == '1';
    }();
    if (ws.attn_sk && attn_sk) {
      ap.sk_mode = 1;
      attention_sk_carve(ap, ws.attn_sk, num_sms(), dh);
    }
    // the attention kernel pulls the O projection's weights into L2 (its K/V stream is evict-first)
    static const bool attn_l2pf = [] {
      const char* e = std::getenv("RDKV_L2_PREFETCH");  // opt-in: measured no faster in the C3 step
      return e && e[0] == '1';
    }();
    static const bool small_l2pf = [] {  // RDKV_SMALLM_L2PF=attn|all: small batches pull w_o while attending
      const char* e = std::getenv("RDKV_SMALLM_L2PF");
      return e && (e[0] == 'a');
    }();
    if (attn_l2pf || (small_l2pf && T <= 128)) {
      ap.l2_next = W(m, wb + 2);
      ap.l2_next_bytes = (long long)d.hidden * qd * 2;
    }
    if (b->layer_ready && b->layer_ready[l])  // layer-wise streaming: this layer's cached KV has landed
      CUDA_TRY(cudaStreamWaitEvent(st, static_cast<cudaEvent_t>(b->layer_ready[l]), 0));
    // the tcgen05 kernel is the product path: an unsupported shape is an error, not a
    // silent fallback; the legacy mma.sync kernel runs only when asked for (RDKV_ATTN=mma, A/B)
    if (use_tc_attn)
      LAUNCH(RDKV_PROF_ATTN, 0.0, launch_attention_tc(ap, dh, S, b->max_new, st));
    else
      LAUNCH(RDKV_PROF_ATTN, 0.0, launch_attention(ap, dh, S, b->max_new, st));
    GemmEpi er{};
    er.counters = counters;
    er.n_counters = N_SPLITK_COUNTERS;
    er.splitk_ws = ws.splitk;  // small M: split-K (the finalize handles the norm statistics)
    er.splitk_bytes = ws.splitk_bytes;
    set_sk(er);
    er.out = ws.x;
    er.ldo = d.hidden;
    er.resid = ws.x;
    er.ldr = d.hidden;
    er.norm_eps = d.norm_eps;
    if (ssq_path) er.ssq_out = ws.ssq;
    if (o_fused && !ssq_path) {
      er.norm_gain = gain(wb + 3);
      er.norm_out = ws.h;
    }
    if (tp) {  // row-parallel: the GEMM pushes its bf16 tiles to every rank (NVLink), then reduce + residual
      const GemmEpi ep = tp_push_epi(er, tp, ar, d.hidden);
      LAUNCH(RDKV_PROF_O, 2.0 * T * qd * d.hidden, launch_gemm(ws.o, qd, W(m, wb + 2), qd, T, d.hidden, (int)qd, EPI_PUSH, 0, ep, st));
      LAUNCH(RDKV_PROF_O, 0.0, launch_tp_reduce_resid(tp, ws.x, d.hidden, T, d.hidden, ar & 1, st));
      ++ar;
    } else {
      LAUNCH(RDKV_PROF_O, 2.0 * T * qd * d.hidden, launch_gemm(ws.o, qd, W(m, wb + 2), qd, T, d.hidden, (int)qd, EPI_RESID, 0, er, st));
    }
    // MLP block
    if (!o_fused && !ssq_path)
      LAUNCH(RDKV_PROF_MISC, 0.0, launch_rmsnorm(ws.x, d.hidden, nullptr, gain(wb + 3), ws.h, d.hidden, T, d.hidden, d.norm_eps, st));
    GemmEpi eg{};
    eg.counters = counters;
    eg.n_counters = N_SPLITK_COUNTERS;
    eg.splitk_ws = ws.splitk;  // small M: split-K (the finalize handles the norm statistics)
    eg.splitk_bytes = ws.splitk_bytes;
    set_sk(eg);
    eg.out = ws.a;
    eg.ldo = d.ffn;
    if (ssq_path) {
      eg.ssq_in = ws.ssq;
      eg.ssq_parts = d.hidden / 32;
      eg.ssq_dim = d.hidden;
      eg.norm_eps = d.norm_eps;
    }
    eg.l2_next = W(m, wb + 5);  // the down projection's weights (kept only on the small-M path)
    eg.l2_next_bytes = (long long)d.ffn * d.hidden * 2;
    LAUNCH(RDKV_PROF_GU, 4.0 * T * d.ffn * d.hidden, launch_gemm(ssq_path ? ws.x : ws.h, d.hidden, W(m, wb + 4), d.hidden, T, 2 * d.ffn, d.hidden, EPI_SWIGLU, 0, eg, st));
    h_ready = down_fused && !ssq_path && l + 1 < d.layers;
    // the down projection pulls the next layer's QKV weights into L2
    if (l + 1 < d.layers) {
      er.l2_next = W(m, wb + RDKV_WEIGHTS_PER_LAYER + 1);
      er.l2_next_bytes = (long long)qkv_n * d.hidden * 2;
    }
    er.norm_gain = h_ready ? gain(wb + RDKV_WEIGHTS_PER_LAYER + 0) : nullptr;  // next layer's attention norm
    er.norm_out = h_ready ? ws.h : nullptr;
    if (tp) {
      const GemmEpi ep = tp_push_epi(er, tp, ar, d.hidden);
      LAUNCH(RDKV_PROF_DOWN, 2.0 * T * d.ffn * d.hidden, launch_gemm(ws.a, d.ffn, W(m, wb + 5), d.ffn, T, d.hidden, d.ffn, EPI_PUSH, 0, ep, st));
      LAUNCH(RDKV_PROF_DOWN, 0.0, launch_tp_reduce_resid(tp, ws.x, d.hidden, T, d.hidden, ar & 1, st));
      ++ar;
    } else {
      LAUNCH(RDKV_PROF_DOWN, 2.0 * T * d.ffn * d.hidden, launch_gemm(ws.a, d.ffn, W(m, wb + 5), d.ffn, T, d.hidden, d.ffn, EPI_RESID, 0, er, st));
    }
  }
  if (b->want_logits) {
    if (!b->logits || !b->last_row) return set_error(RDKV_ERR_ARG, "forward: logits requested without buffers");
    const int fn = 1 + RDKV_WEIGHTS_PER_LAYER * d.layers;
    LAUNCH(RDKV_PROF_HEAD, 0.0, launch_rmsnorm(ws.x, d.hidden, b->last_row, G(m, fn), ws.hl, d.hidden, S, d.hidden, d.norm_eps, st));
    GemmEpi el{};
    el.counters = counters;
    el.n_counters = N_SPLITK_COUNTERS;
    el.splitk_ws = ws.splitk;
    el.splitk_bytes = ws.splitk_bytes;
    el.out = b->logits;
    el.ldo = d.vocab;
    LAUNCH(RDKV_PROF_HEAD, 2.0 * S * d.vocab * d.hidden, launch_gemm(ws.hl, d.hidden, W(m, fn + 1), d.hidden, S, d.vocab, d.hidden, EPI_STORE_F32, 0, el, st));
    if (b->next_token) LAUNCH(RDKV_PROF_HEAD, 0.0, launch_argmax(b->logits, d.vocab, S, d.vocab, b->next_token, ws.argmax, st));
  }
  return 0;
}

int rdkv_model_set_tp(rdkv_model* m, rdkv_tp_comm* comm) {
  if (!m) return set_error(RDKV_ERR_ARG, "model_set_tp: null model");
  m->tp = comm;
  return 0;
}

int rdkv_profile_enable(rdkv_model* m, int on) {
  if (!m) return set_error(RDKV_ERR_ARG, "profile_enable: null model");
  m->prof = on != 0;
  return 0;
}

int rdkv_profile_collect(rdkv_model* m, double* ms, int64_t* launches, double* flops) {
  if (!m) return set_error(RDKV_ERR_ARG, "profile_collect: null model");
  double acc[RDKV_PROF_N] = {};
  std::lock_guard<std::mutex> g(m->mu);
  for (auto& r : m->recs) {
    CUDA_TRY(cudaEventSynchronize(r.b));
    float t = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&t, r.a, r.b));
    acc[r.cat] += t;
    m->spare.push_back(r.a);
    m->spare.push_back(r.b);
  }
  m->recs.clear();
  for (int c = 0; c < RDKV_PROF_N; ++c) {
    if (ms) ms[c] = acc[c];
    if (launches) launches[c] = m->launches[c];
    if (flops) flops[c] = m->flops[c];
    m->launches[c] = 0;
    m->flops[c] = 0;
  }
  return 0;
}

int rdkv_kv_copy_block(void* pool_base, int layers, int kv_heads, int head_dim, int64_t pool_slots, int block_size,
                       int src_block, int dst_block, int n_tokens, void* stream) {
  if (!pool_base || block_size <= 0 || n_tokens < 0 || n_tokens > block_size || src_block < 0 || dst_block < 0 ||
      (int64_t)(src_block + 1) * block_size > pool_slots || (int64_t)(dst_block + 1) * block_size > pool_slots)
    return set_error(RDKV_ERR_ARG, "kv_copy_block: bad arguments");
  if (n_tokens == 0) return 0;
  const size_t row = (size_t)head_dim * 2, pitch = (size_t)pool_slots * row;
  auto* base = static_cast<uint8_t*>(pool_base);
  CUDA_TRY(cudaMemcpy2DAsync(base + (size_t)dst_block * block_size * row, pitch,
                             base + (size_t)src_block * block_size * row, pitch, (size_t)n_tokens * row,
                             (size_t)layers * 2 * kv_heads, cudaMemcpyDeviceToDevice, static_cast<cudaStream_t>(stream)));
  return 0;
}

int rdkv_kv_unpack(const rdkv_unpack_job* jobs_dev, int n_jobs, int max_tokens, const int32_t* block_table_dev,
                   int block_size, void* pool_base, int layers, int kv_heads, int head_dim, int64_t pool_slots,
                   int elem_width, int layer_begin, int layer_end, void* stream) {
  return rdkv_kv_unpack_heads(jobs_dev, n_jobs, max_tokens, block_table_dev, block_size, pool_base, layers, kv_heads,
                              head_dim, pool_slots, elem_width, layer_begin, layer_end, 0, kv_heads, stream);
}

int rdkv_kv_stream_layers(const rdkv_unpack_job* jobs_dev, int n_jobs, int max_tokens, const int32_t* block_table_dev,
                          int block_size, void* pool_base, int layers, int kv_heads, int head_dim, int64_t pool_slots,
                          int elem_width, int head_begin, int src_kv_heads, int n_copies, void* const* host_src,
                          void* const* dev_dst, const size_t* bytes_per_layer, int copy_layers, void* h2d_stream,
                          void* unpack_stream, void* const* copied_events, void* const* layer_events) {
  if (block_size <= 0 || !pool_base || !jobs_dev || layers <= 0 || !layer_events || copy_layers <= 0 ||
      (n_copies > 0 && (!host_src || !dev_dst || !bytes_per_layer || !copied_events)))
    return set_error(RDKV_ERR_ARG, "kv_stream_layers: bad arguments");
  auto h2d = static_cast<cudaStream_t>(h2d_stream), up = static_cast<cudaStream_t>(unpack_stream);
  for (int l = 0; l < layers; ++l) {
    if (n_copies > 0 && l % copy_layers == 0) {
      const int l1 = std::min(layers, l + copy_layers);
      for (int c = 0; c < n_copies; ++c) {
        const size_t per = bytes_per_layer[c];
        CUDA_TRY(cudaMemcpyAsync(static_cast<uint8_t*>(dev_dst[c]) + (size_t)l * per,
                                 static_cast<const uint8_t*>(host_src[c]) + (size_t)l * per, (size_t)(l1 - l) * per,
                                 cudaMemcpyHostToDevice, h2d));
      }
      for (int ll = l; ll < l1; ++ll) CUDA_TRY(cudaEventRecord(static_cast<cudaEvent_t>(copied_events[ll]), h2d));
    }
    if (n_copies > 0) CUDA_TRY(cudaStreamWaitEvent(up, static_cast<cudaEvent_t>(copied_events[l]), 0));
    RDKV_TRY(launch_kv_unpack(jobs_dev, n_jobs, max_tokens, block_table_dev, block_size, pool_base, l, l + 1, kv_heads,
                              head_dim, pool_slots, elem_width, up, head_begin, src_kv_heads));
    CUDA_TRY(cudaEventRecord(static_cast<cudaEvent_t>(layer_events[l]), up));
  }
  return 0;
}

int rdkv_kv_unpack_heads(const rdkv_unpack_job* jobs_dev, int n_jobs, int max_tokens, const int32_t* block_table_dev,
                         int block_size, void* pool_base, int layers, int kv_heads, int head_dim, int64_t pool_slots,
                         int elem_width, int layer_begin, int layer_end, int head_begin, int src_kv_heads,
                         void* stream) {
  if (block_size <= 0 || !pool_base || !jobs_dev) return set_error(RDKV_ERR_ARG, "kv_unpack: bad arguments");
  if (layer_begin < 0 || layer_end > layers || layer_begin > layer_end)
    return set_error(RDKV_ERR_ARG, "kv_unpack: bad layer range [%d, %d) of %d", layer_begin, layer_end, layers);
  return launch_kv_unpack(jobs_dev, n_jobs, max_tokens, block_table_dev, block_size, pool_base, layer_begin,
                          layer_end, kv_heads, head_dim, pool_slots, elem_width, static_cast<cudaStream_t>(stream),
                          head_begin, src_kv_heads);
}

}  // extern "C"
