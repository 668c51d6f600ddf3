// Tensor-parallel communicator (see tp.cu).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstddef>
#include <cstdint>

#define RDKV_TP_MAX 8

namespace rdkv {

// Kernel-side view: every rank's comm buffer, mapped into this process.
struct TpArgs {
  int rank, size;
  uint32_t* flags[RDKV_TP_MAX];                   // rank p's flag array (flags[p][q] = epoch q published)
  const __nv_bfloat16* part[RDKV_TP_MAX][2];      // rank p's partial buffers
  uint32_t* seq;                                  // this rank's completed-epoch counter
  uint32_t* ticket;                               // this rank's CTA ticket
};

}  // namespace rdkv

struct rdkv_tp_comm {
  int rank = 0, size = 1;
  size_t max_elems = 0;
  rdkv::TpArgs args{};
  __nv_bfloat16* local_part[2] = {nullptr, nullptr};
};

namespace rdkv {
// x[rows, cols] (ld ldx) += sum over ranks of partial buffer `buf` (dense [rows, cols]).
int launch_tp_allreduce_resid(const rdkv_tp_comm* c, __nv_bfloat16* x, long long ldx, int rows, int cols, int buf,
                              cudaStream_t st);
}  // namespace rdkv
