// Host-side TMA descriptor encoding (cuTensorMapEncodeIm2col / Tiled), fetched
// through cudaGetDriverEntryPoint so the library does not link libcuda.
#include "tmap.h"

#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <mutex>

namespace gemel {

namespace {
PFN_cuTensorMapEncodeTiled_v12000 g_tiled = nullptr;
PFN_cuTensorMapEncodeIm2col_v12000 g_im2col = nullptr;
int g_driver_version = 0;
std::once_flag g_once;

void init() {
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&g_tiled), cudaEnableDefault, &q);
  cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", reinterpret_cast<void**>(&g_im2col), cudaEnableDefault, &q);
  cudaDriverGetVersion(&g_driver_version);
}

CUtensorMapSwizzle swz(int bytes) {
  switch (bytes) {
    case 128: return CU_TENSOR_MAP_SWIZZLE_128B;
    case 64: return CU_TENSOR_MAP_SWIZZLE_64B;
    case 32: return CU_TENSOR_MAP_SWIZZLE_32B;
    default: return CU_TENSOR_MAP_SWIZZLE_NONE;
  }
}

// Driver <= 13.1 workaround for tensors smaller than 128 KiB (mirrors the
// public CUTLASS fix): clear bit 21 of the descriptor's second word.
void small_tensor_fix(CUtensorMap* m, uint64_t bytes) {
  if (g_driver_version <= 13010 && bytes < 131072) reinterpret_cast<uint64_t*>(m)[1] &= ~(1ull << 21);
}
}  // namespace

int tmap_encode_im2col(CUtensorMap* m, const void* ptr, int n, int h, int w, int c, int c_pitch, int lower_w,
                       int lower_h, int upper_w, int upper_h, int chunk, int pixels, int stride_w, int stride_h) {
  std::call_once(g_once, init);
  if (!g_im2col) return -1;
  cuuint64_t dims[4] = {cuuint64_t(c), cuuint64_t(w), cuuint64_t(h), cuuint64_t(n)};
  cuuint64_t strides[3] = {cuuint64_t(c_pitch) * 2, cuuint64_t(c_pitch) * 2 * w, cuuint64_t(c_pitch) * 2 * w * h};
  int lower[2] = {lower_w, lower_h};
  int upper[2] = {upper_w, upper_h};
  cuuint32_t estr[4] = {1, cuuint32_t(stride_w), cuuint32_t(stride_h), 1};
  CUresult r = g_im2col(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(ptr), dims, strides, lower, upper,
                        cuuint32_t(chunk), cuuint32_t(pixels), estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz(chunk * 2),
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return int(r);
  small_tensor_fix(m, uint64_t(c_pitch) * 2 * w * h * n);
  return 0;
}

int tmap_encode_2d(CUtensorMap* m, const void* ptr, uint64_t cols, uint64_t rows, uint64_t pitch_bytes,
                   int box_cols, int box_rows, int swizzle_bytes) {
  std::call_once(g_once, init);
  if (!g_tiled) return -1;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {pitch_bytes};
  cuuint32_t box[2] = {cuuint32_t(box_cols), cuuint32_t(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_tiled(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, swz(swizzle_bytes), CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return int(r);
  small_tensor_fix(m, pitch_bytes * rows);
  return 0;
}

}  // namespace gemel
