// Tensor-parallel communicator (see tp.cu).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstddef>
#include <cstdint>

#define RDKV_TP_MAX 8

namespace rdkv {

// Kernel-side view of the group.  Each rank's comm buffer holds a header (flags,
// epoch counter, ticket) and receive slots recv[2 parities][size][max_elems] bf16;
// slot (b, q) of rank p receives rank q's partial for all-reduces of parity b.
struct TpArgs {
  int rank, size;
  uint32_t* flags[RDKV_TP_MAX];                   // rank p's flag array (flags[p][q] = epoch q published)
  const __nv_bfloat16* recv[2][RDKV_TP_MAX];      // this rank's receive slots (local HBM)
  __nv_bfloat16* push[2][RDKV_TP_MAX];            // this rank's slot in rank p's buffer (peer HBM)
  uint32_t* seq;                                  // this rank's completed-epoch counter
  uint32_t* ticket;                               // this rank's CTA ticket
};

}  // namespace rdkv

struct rdkv_tp_comm {
  int rank = 0, size = 1;
  size_t max_elems = 0;
  rdkv::TpArgs args{};
};

namespace rdkv {
// x[rows, cols] (ld ldx) += sum over ranks of the partials received in parity
// `buf` (pushed by every rank's PUSH-epilogue GEMM or rdkv_tp_push).
int launch_tp_reduce_resid(const rdkv_tp_comm* c, __nv_bfloat16* x, long long ldx, int rows, int cols, int buf,
                           cudaStream_t st);
// Copy a local dense [rows, cols] partial into every rank's slot (what the PUSH
// epilogue does from inside the GEMM).
int launch_tp_push(const rdkv_tp_comm* c, const __nv_bfloat16* src, int rows, int cols, int buf, cudaStream_t st);
}  // namespace rdkv
