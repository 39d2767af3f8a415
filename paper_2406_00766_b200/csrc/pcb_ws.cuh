// Shared pieces of the warp-specialised tcgen05 kernels (pcb_tc_ws.cu,
// pcb_tc_pf.cu): mbarrier ring bookkeeping and TMA tensor maps over the
// node-major fp32 buffers.
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>

#include "pcb_internal.cuh"
#include "pcb_tc.cuh"

namespace pcb {
namespace ws {

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

// ring position: slot and wait parities of use u of a ring with S stages
// stage ring of S slots: slot index and mbarrier phase parity, kept
// incrementally (no division per access)
template <int S>
struct Ring {
  int s = 0;
  uint32_t par = 0;
  __device__ int slot() const { return s; }
  __device__ uint32_t full_par() const { return par; }
  __device__ uint32_t empty_par() const { return par ^ 1u; }
  __device__ void next() {
    if (++s == S) {
      s = 0;
      par ^= 1u;
    }
  }
};

__device__ __forceinline__ int next_real(const int32_t* __restrict__ ids, int cap, int c) {
  while (c < cap && __ldg(ids + c) == 0) ++c;
  return c;
}



inline PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 2-D fp32 map over a node-major buffer [rows x ldb], box [box_rows x box_cols
// samples]; swizzle_bytes (64 / 128) permutes the 16-byte chunks of each box
// row so row-parallel shared-memory reads are bank-conflict free
inline int make_rows_map(CUtensorMap* m, const float* base, int64_t rows, int ldb, int box_rows,
                         int box_cols = 128, int swizzle_bytes = 0) {
  auto fn = encode_fn();
  if (!fn) return PCB_CUDA;
  const cuuint64_t dims[2] = {(cuuint64_t)ldb, (cuuint64_t)(rows > 0 ? rows : 1)};
  const cuuint64_t strides[1] = {(cuuint64_t)ldb * 4};
  const cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  swizzle_bytes == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                  : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                        : CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? PCB_OK : PCB_CUDA;
}

}  // namespace ws
}  // namespace pcb
