// Host-side TMA tensor-map creation for THD [rows][heads][D] bf16 tensors.
// cuTensorMapEncodeTiled is fetched through the runtime's driver entry point so
// the library does not link libcuda directly.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include "common.cuh"

namespace wlb {

inline PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 3-D map over a THD tensor: dims {D, H, rows}, box {64, 1, box_rows},
// 128-B swizzle (one 64-element slab = one 128-B swizzle row per token).
inline int make_thd_tmap(CUtensorMap* map, const void* base, int rows, int heads, int dim,
                         int box_rows) {
  auto enc = tmap_encoder();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return WLB_ECUDA;
  }
  cuuint64_t gdim[3] = {(cuuint64_t)dim, (cuuint64_t)heads, (cuuint64_t)rows};
  cuuint64_t gstride[2] = {(cuuint64_t)dim * 2, (cuuint64_t)heads * dim * 2};
  cuuint32_t box[3] = {64, 1, (cuuint32_t)box_rows};
  cuuint32_t estride[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), gdim,
                   gstride, box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d) rows=%d heads=%d dim=%d", (int)r, rows, heads,
              dim);
    return WLB_ECUDA;
  }
  return WLB_OK;
}

// 3-D map over the 128-query backward's fp32 dQ accumulator [H][D/4][rows][4]:
// dims {rows*4, D/4, H}, box {128, 8, 1} = 32 rows x 32 head-dims (4 KB, laid
// out [8][32][4] in shared memory), no swizzle; the drain warps reduce into it
// with TMA tile reduce-adds (rows past `rows` are clipped).
inline int make_dq_acc_tmap(CUtensorMap* map, void* base, int rows, int heads, int dim) {
  auto enc = tmap_encoder();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return WLB_ECUDA;
  }
  // (rows, 4) flattened: each box row is 32 query rows x 4 floats = 512
  // contiguous bytes (a 16-B inner box dimension made 256 separate 16-B
  // requests per box and measured 1.8x slower)
  cuuint64_t gdim[3] = {(cuuint64_t)rows * 4, (cuuint64_t)dim / 4, (cuuint64_t)heads};
  cuuint64_t gstride[2] = {(cuuint64_t)rows * 16, (cuuint64_t)rows * 16 * (dim / 4)};
  cuuint32_t box[3] = {128, 8, 1};
  cuuint32_t estride[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, base, gdim, gstride, box, estride,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (dQ accumulator) failed (%d) rows=%d heads=%d", (int)r,
              rows, heads);
    return WLB_ECUDA;
  }
  return WLB_OK;
}

}  // namespace wlb
