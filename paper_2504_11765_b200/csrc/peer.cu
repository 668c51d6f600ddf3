// Multi-instance sharing: one model instance per GPU, and a cached
// prefix already resident in a PEER GPU's HBM tier is pulled over NVLink
// instead of from the host tier or disk.
//
//   rdkv_ipc_handle / rdkv_ipc_open / rdkv_ipc_close
//       CUDA IPC: each rank exports the allocation holding its paged KV pool;
//       every other rank maps it (peer access enabled lazily), so a kernel on
//       rank r can load straight from rank s's pool over NVLink / NVSwitch.
//   K3p rdkv_kv_peer_gather
//       block gather pool -> pool: (layer, K|V, head, block) runs of
//       block_size*dh bf16 read from the source pool (a peer's, through the
//       IPC mapping, or the local one) and written into freshly reserved local
//       blocks.  One warp per run, 16-B loads, 4 in flight per lane, so the
//       NVLink reads are deep enough to cover the remote latency.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstring>
#include <mutex>

#include "common.cuh"
#include "pdl.cuh"

namespace rdkv {
namespace {

__device__ __forceinline__ uint4 ld_nc(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__global__ void __launch_bounds__(256) kv_gather_kernel(const __nv_bfloat16* __restrict__ src, long long src_slots,
                                                        const int* __restrict__ src_blocks,
                                                        __nv_bfloat16* __restrict__ dst, long long dst_slots,
                                                        const int* __restrict__ dst_blocks, int n_blocks, int planes,
                                                        int dh, int block_size) {
  pdl_trigger();
  pdl_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long runs = (long long)planes * n_blocks;
  const long long nvec = (long long)block_size * dh / 8;  // 16-B vectors per run
  constexpr int U = 4;
  for (long long run = (long long)blockIdx.x * 8 + warp; run < runs; run += (long long)gridDim.x * 8) {
    const long long plane = run / n_blocks;
    const int b = (int)(run % n_blocks);
    const __nv_bfloat16* s = src + (plane * src_slots + (long long)src_blocks[b] * block_size) * dh;
    __nv_bfloat16* d = dst + (plane * dst_slots + (long long)dst_blocks[b] * block_size) * dh;
    long long i = lane;
    for (; i + 32 * (U - 1) < nvec; i += 32 * U) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = ld_nc(s + (i + 32 * u) * 8);
#pragma unroll
      for (int u = 0; u < U; ++u) *reinterpret_cast<uint4*>(d + (i + 32 * u) * 8) = v[u];
    }
    for (; i < nvec; i += 32) *reinterpret_cast<uint4*>(d + i * 8) = ld_nc(s + i * 8);
  }
}

PFN_cuMemGetAddressRange_v3020 range_fn() {
  static PFN_cuMemGetAddressRange_v3020 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(p);
  });
  return fn;
}

}  // namespace
}  // namespace rdkv

using namespace rdkv;

extern "C" int rdkv_ipc_handle(const void* dev_ptr, void* handle_out, int64_t* offset_out) {
  if (!dev_ptr || !handle_out || !offset_out) return set_error(RDKV_ERR_ARG, "ipc_handle: null argument");
  CUdeviceptr base = 0;
  size_t size = 0;
  auto range = range_fn();
  if (!range || range(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS)
    return set_error(RDKV_ERR_CUDA, "ipc_handle: cuMemGetAddressRange failed");
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  static_assert(sizeof(h) == 64, "CUDA IPC handles are 64 bytes");
  std::memcpy(handle_out, &h, sizeof(h));
  *offset_out = (int64_t)(reinterpret_cast<CUdeviceptr>(dev_ptr) - base);
  return 0;
}

extern "C" int rdkv_ipc_open(const void* handle, void** base_out) {
  if (!handle || !base_out) return set_error(RDKV_ERR_ARG, "ipc_open: null argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  CUDA_TRY(cudaIpcOpenMemHandle(base_out, h, cudaIpcMemLazyEnablePeerAccess));
  return 0;
}

extern "C" int rdkv_ipc_close(void* base) {
  if (!base) return 0;
  CUDA_TRY(cudaIpcCloseMemHandle(base));
  return 0;
}

extern "C" int rdkv_kv_peer_gather(const void* src_pool, int64_t src_slots, const int32_t* src_blocks,
                                   void* dst_pool, int64_t dst_slots, const int32_t* dst_blocks, int n_blocks,
                                   int layers, int kv_heads, int head_dim, int block_size, void* stream) {
  if (!src_pool || !dst_pool || !src_blocks || !dst_blocks || n_blocks < 0 || block_size <= 0 || head_dim % 8)
    return set_error(RDKV_ERR_ARG, "kv_peer_gather: bad arguments");
  if (n_blocks == 0) return 0;
  const int planes = layers * 2 * kv_heads;
  long long runs = (long long)planes * n_blocks;
  long long gx = (runs + 7) / 8;
  const long long cap = 4LL * num_sms();
  if (gx > cap) gx = cap;
  CUDA_TRY(launch_k(kv_gather_kernel, dim3((unsigned)gx), dim3(256), 0, static_cast<cudaStream_t>(stream),
                    static_cast<const __nv_bfloat16*>(src_pool), (long long)src_slots, src_blocks,
                    static_cast<__nv_bfloat16*>(dst_pool), (long long)dst_slots, dst_blocks, n_blocks, planes,
                    head_dim, block_size));
  CUDA_TRY(cudaGetLastError());
  return 0;
}

extern "C" int rdkv_memcpy_2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t height,
                              void* stream) {
  if (!dst || !src || width > dpitch || width > spitch) return set_error(RDKV_ERR_ARG, "memcpy_2d: bad arguments");
  CUDA_TRY(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, cudaMemcpyDefault,
                             static_cast<cudaStream_t>(stream)));
  return 0;
}
