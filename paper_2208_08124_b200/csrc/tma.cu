// Host-side TMA tensor-map creation (cuTensorMapEncodeTiled via the runtime's driver
// entry point, so the library does not link libcuda directly).
#include <mutex>

#include "fmha_common.cuh"

namespace ub {

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

ub_status make_tmap_bf16(CUtensorMap* map, const void* base, uint64_t cols, uint64_t rows, uint64_t pitch_bytes,
                         uint32_t box_cols, uint32_t box_rows, int swizzle_bytes) {
  auto enc = get_encode();
  UB_REQUIRE(enc != nullptr, UB_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  UB_REQUIRE(pitch_bytes % 16 == 0, UB_ERR_INVALID_ARG, "TMA row pitch must be a multiple of 16 B");
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {pitch_bytes};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  const CUtensorMapSwizzle sw = swizzle_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                               : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_NONE;
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  UB_REQUIRE(r == CUDA_SUCCESS, UB_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return UB_OK;
}

ub_status make_tmap_f32(CUtensorMap* map, const void* base, uint64_t cols, uint64_t rows, uint64_t pitch_bytes,
                        uint32_t box_cols, uint32_t box_rows, int swizzle_bytes) {
  auto enc = get_encode();
  UB_REQUIRE(enc != nullptr, UB_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {pitch_bytes};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  const CUtensorMapSwizzle sw = swizzle_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                               : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_NONE;
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  UB_REQUIRE(r == CUDA_SUCCESS, UB_ERR_CUDA, "cuTensorMapEncodeTiled (f32) failed (%d)", (int)r);
  return UB_OK;
}

ub_status make_tmap_f32_1d(CUtensorMap* map, const void* base, uint64_t n, uint32_t box) {
  auto enc = get_encode();
  UB_REQUIRE(enc != nullptr, UB_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[1] = {n};
  cuuint64_t strides[1] = {n * 4};
  cuuint32_t boxd[1] = {box};
  cuuint32_t estr[1] = {1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 1, const_cast<void*>(base), dims, strides, boxd, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  UB_REQUIRE(r == CUDA_SUCCESS, UB_ERR_CUDA, "cuTensorMapEncodeTiled (f32 1-D) failed (%d)", (int)r);
  return UB_OK;
}

}  // namespace ub
