// tma_host.h -- host-side TMA tensor-map encoding through the driver entry
// point (no link-time dependency on libcuda).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>

namespace dkv {

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiledFn encode_tiled_fn() {
  static const EncodeTiledFn fn = [] {  // resolved once (thread-safe static initialisation)
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<EncodeTiledFn>(p);
    return static_cast<EncodeTiledFn>(nullptr);
  }();
  return fn;
}

// 3-D bf16 map over a row-major [rows, heads, dim] tensor: dims (dim, heads, rows),
// box (64, box_heads, box_rows), SWIZZLE_128B (64 bf16 = 128 B inner box).
inline bool make_map_3d_bf16(CUtensorMap* m, const void* base, int64_t rows, int64_t heads, int64_t dim,
                             uint32_t box_heads, uint32_t box_rows) {
  std::memset(m, 0, sizeof(*m));
  EncodeTiledFn fn = encode_tiled_fn();
  if (!fn || rows <= 0) return false;
  cuuint64_t gdim[3] = {static_cast<cuuint64_t>(dim), static_cast<cuuint64_t>(heads),
                        static_cast<cuuint64_t>(rows)};
  cuuint64_t gstride[2] = {static_cast<cuuint64_t>(dim * 2), static_cast<cuuint64_t>(heads * dim * 2)};
  cuuint32_t box[3] = {64u, box_heads, box_rows};
  cuuint32_t estr[3] = {1u, 1u, 1u};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), gdim, gstride, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// 3-D fp32 map over [rows, heads, dim] (no swizzle), box (dim, box_heads, box_rows);
// used as the destination of TMA bulk reduce-adds (dQ accumulation).
inline bool make_map_3d_f32(CUtensorMap* m, const void* base, int64_t rows, int64_t heads, int64_t dim,
                            uint32_t box_heads, uint32_t box_rows, uint32_t box_dim) {
  std::memset(m, 0, sizeof(*m));
  EncodeTiledFn fn = encode_tiled_fn();
  if (!fn || rows <= 0) return false;
  cuuint64_t gdim[3] = {static_cast<cuuint64_t>(dim), static_cast<cuuint64_t>(heads),
                        static_cast<cuuint64_t>(rows)};
  cuuint64_t gstride[2] = {static_cast<cuuint64_t>(dim * 4), static_cast<cuuint64_t>(heads * dim * 4)};
  cuuint32_t box[3] = {box_dim, box_heads, box_rows};
  cuuint32_t estr[3] = {1u, 1u, 1u};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), gdim, gstride, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// 2-D fp32 map over a row-major [rows][cols] buffer (row stride in elements), box (box_cols, 1)
inline bool make_map_2d_f32(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int64_t stride,
                            uint32_t box_cols) {
  std::memset(m, 0, sizeof(*m));
  EncodeTiledFn fn = encode_tiled_fn();
  if (!fn || rows <= 0 || cols <= 0) return false;
  cuuint64_t gdim[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t gstride[1] = {static_cast<cuuint64_t>(stride * 4)};
  cuuint32_t box[2] = {box_cols, 1u};
  cuuint32_t estr[2] = {1u, 1u};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), gdim, gstride, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// 2-D bf16 map over a row-major [rows][cols] buffer, box (box_cols, box_rows), SWIZZLE_32B
// (box_cols * 2 == 32 bytes): the UMMA K-major SW32 operand layout straight from TMA.
inline bool make_map_2d_bf16_sw32(CUtensorMap* m, const void* base, int64_t rows, int64_t cols,
                                  uint32_t box_cols, uint32_t box_rows) {
  std::memset(m, 0, sizeof(*m));
  EncodeTiledFn fn = encode_tiled_fn();
  if (!fn || rows <= 0 || cols <= 0) return false;
  cuuint64_t gdim[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t gstride[1] = {static_cast<cuuint64_t>(cols * 2)};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1u, 1u};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), gdim, gstride, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace dkv
