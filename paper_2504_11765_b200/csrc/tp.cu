// Tensor parallelism inside one instance (C5: Llama-3-70B-shaped, TP=4;
// SURVEY §8e "C5 exception", §8f rank 1).  Each TP rank owns 1/T of the query
// heads, KV heads and FFN columns; the attention-output and down projections
// are row-parallel, so their outputs are partial sums that must be all-reduced
// before the residual add — the only collective on the hot path.
//
// No NCCL: the reduction runs over NVLink peer memory in two steps.
//   1. The row-parallel GEMM itself is the transfer: its PUSH epilogue stores
//      every finished bf16 output tile into this rank's receive slot of EVERY
//      rank (CUDA-IPC mappings, P2P stores over NVLink), so the data moves
//      tile by tile while later tiles are still on the tensor cores.
//   2. tp_reduce_resid_kernel (per rank) publishes "my pushes for epoch e are
//      complete" into every peer's flag array (st.release.sys), waits until all
//      peers published e (ld.acquire.sys), then sums the T received slots from
//      LOCAL HBM in fp32 together with the residual stream and writes the new
//      residual (bf16) — reduction and residual add in one pass.
// Epochs live in device memory (a per-rank counter bumped by the last CTA of
// each reduce), so the forward stays CUDA-graph capturable.  Receive slots are
// double-buffered by all-reduce parity: rank r pushes into parity b again only
// two all-reduces later, after every peer published the intermediate epoch —
// i.e. finished reading parity b — so no "done" flags are needed.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <new>

#include "common.cuh"
#include "pdl.cuh"
#include "tp.cuh"

namespace rdkv {
namespace {

constexpr size_t kHdr = 128;  // flags[16] u32 | seq u32 | ticket u32 | pad

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint4 ld_volatile_v4(const void* p) {  // slots are rewritten by peers
  uint4 r;
  asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void add_bf16x8(float (&a)[8], uint4 v) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&w[i]);
    const float2 f = __bfloat1622float2(b);
    a[2 * i] += f.x;
    a[2 * i + 1] += f.y;
  }
}

__global__ void __launch_bounds__(256) tp_reduce_resid_kernel(TpArgs t, __nv_bfloat16* __restrict__ x, long long ldx,
                                                              int rows, int cols, int buf) {
  pdl_trigger();
  pdl_wait();  // this rank's pushes (the preceding GEMM) are complete
  __shared__ uint32_t s_epoch;
  if (threadIdx.x == 0) s_epoch = *t.seq + 1;
  __syncthreads();
  const uint32_t e = s_epoch;
  if (threadIdx.x < t.size) {
    // publish our pushes to peer threadIdx.x, then wait for its pushes to us
    __threadfence_system();
    st_release_sys(t.flags[threadIdx.x] + t.rank, e);
    const uint32_t* mine = t.flags[t.rank] + threadIdx.x;
    while (ld_acquire_sys(mine) < e) {
    }
  }
  __syncthreads();
  const int vec_per_row = cols / 8;
  const long long nvec = (long long)rows * vec_per_row;
  for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < nvec; v += (long long)gridDim.x * blockDim.x) {
    const long long r = v / vec_per_row;
    const int c = (int)(v % vec_per_row) * 8;
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    __nv_bfloat16* xp = x + r * ldx + c;
    add_bf16x8(acc, *reinterpret_cast<const uint4*>(xp));
    const long long off = r * cols + c;
#pragma unroll 8
    for (int q = 0; q < t.size; ++q) add_bf16x8(acc, ld_volatile_v4(t.recv[buf][q] + off));
    uint4 o;
    uint32_t* ow = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __nv_bfloat162 b = __floats2bfloat162_rn(acc[2 * i], acc[2 * i + 1]);
      ow[i] = *reinterpret_cast<uint32_t*>(&b);
    }
    *reinterpret_cast<uint4*>(xp) = o;
  }
  // the last CTA to finish advances this rank's epoch (every CTA read it at its start)
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const uint32_t tk = atomicAdd(t.ticket, 1u);
    if (tk == gridDim.x - 1) {
      *t.ticket = 0;
      __threadfence();
      atomicExch(t.seq, e);
    }
  }
}

__global__ void __launch_bounds__(256) tp_push_kernel(TpArgs t, const __nv_bfloat16* __restrict__ src, long long n8,
                                                      int buf) {
  pdl_trigger();
  pdl_wait();
  for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < n8; v += (long long)gridDim.x * blockDim.x) {
    const uint4 d = reinterpret_cast<const uint4*>(src)[v];
    for (int p = 0; p < t.size; ++p) reinterpret_cast<uint4*>(t.push[buf][p])[v] = d;
  }
  __threadfence_system();
}

}  // namespace

int launch_tp_reduce_resid(const rdkv_tp_comm* c, __nv_bfloat16* x, long long ldx, int rows, int cols, int buf,
                           cudaStream_t st) {
  if (rows <= 0) return 0;
  if (cols % 8 || (size_t)rows * cols > c->max_elems)
    return set_error(RDKV_ERR_ARG, "tp_reduce: %d x %d exceeds the comm buffer or is not a multiple of 8", rows,
                     cols);
  const long long nvec = (long long)rows * cols / 8;
  long long grid = (nvec + 255) / 256;
  const long long cap = 2LL * num_sms();
  if (grid > cap) grid = cap;
  CUDA_TRY(launch_k(tp_reduce_resid_kernel, dim3((unsigned)grid), dim3(256), 0, st, c->args, x, ldx, rows, cols,
                    buf & 1));
  CUDA_TRY(cudaGetLastError());
  return 0;
}

int launch_tp_push(const rdkv_tp_comm* c, const __nv_bfloat16* src, int rows, int cols, int buf, cudaStream_t st) {
  if (rows <= 0) return 0;
  if (cols % 8 || (size_t)rows * cols > c->max_elems)
    return set_error(RDKV_ERR_ARG, "tp_push: %d x %d exceeds the comm buffer or is not a multiple of 8", rows, cols);
  const long long n8 = (long long)rows * cols / 8;
  long long grid = (n8 + 255) / 256;
  const long long cap = 2LL * num_sms();
  if (grid > cap) grid = cap;
  CUDA_TRY(launch_k(tp_push_kernel, dim3((unsigned)grid), dim3(256), 0, st, c->args, src, n8, buf & 1));
  CUDA_TRY(cudaGetLastError());
  return 0;
}

}  // namespace rdkv

using namespace rdkv;

static size_t slot_bytes(size_t max_elems) { return (max_elems * 2 + 127) / 128 * 128; }

extern "C" size_t rdkv_tp_comm_bytes(size_t max_elems, int size) {
  return kHdr + 2 * (size_t)size * slot_bytes(max_elems);
}

extern "C" int rdkv_tp_comm_create(int rank, int size, void* const* bases, size_t max_elems, rdkv_tp_comm** out) {
  if (!bases || !out || size < 1 || size > RDKV_TP_MAX || rank < 0 || rank >= size || max_elems == 0)
    return set_error(RDKV_ERR_ARG, "tp_comm_create: bad arguments (rank %d, size %d)", rank, size);
  auto* c = new (std::nothrow) rdkv_tp_comm();
  if (!c) return set_error(RDKV_ERR_ARG, "tp_comm_create: out of memory");
  c->rank = rank;
  c->size = size;
  c->max_elems = max_elems;
  const size_t sb = slot_bytes(max_elems);
  TpArgs& a = c->args;
  a.rank = rank;
  a.size = size;
  auto* mine = static_cast<uint8_t*>(bases[rank]);
  for (int p = 0; p < size; ++p) {
    auto* b = static_cast<uint8_t*>(bases[p]);
    if (!b) {
      delete c;
      return set_error(RDKV_ERR_ARG, "tp_comm_create: null buffer for rank %d", p);
    }
    a.flags[p] = reinterpret_cast<uint32_t*>(b);
    for (int par = 0; par < 2; ++par) {
      a.recv[par][p] = reinterpret_cast<const __nv_bfloat16*>(mine + kHdr + ((size_t)par * size + p) * sb);
      a.push[par][p] = reinterpret_cast<__nv_bfloat16*>(b + kHdr + ((size_t)par * size + rank) * sb);
    }
  }
  a.seq = reinterpret_cast<uint32_t*>(mine + 64);
  a.ticket = reinterpret_cast<uint32_t*>(mine + 68);
  *out = c;
  return 0;
}

extern "C" void rdkv_tp_comm_destroy(rdkv_tp_comm* c) { delete c; }

extern "C" int rdkv_tp_push(rdkv_tp_comm* c, const void* src, int rows, int cols, int buf, void* stream) {
  if (!c || !src) return set_error(RDKV_ERR_ARG, "tp_push: null argument");
  return launch_tp_push(c, static_cast<const __nv_bfloat16*>(src), rows, cols, buf, static_cast<cudaStream_t>(stream));
}

extern "C" int rdkv_tp_reduce_resid(rdkv_tp_comm* c, void* x, int64_t ldx, int rows, int cols, int buf,
                                    void* stream) {
  if (!c || !x) return set_error(RDKV_ERR_ARG, "tp_reduce: null argument");
  return launch_tp_reduce_resid(c, static_cast<__nv_bfloat16*>(x), ldx, rows, cols, buf,
                                static_cast<cudaStream_t>(stream));
}
