#pragma once
#include <cuda.h>
#include <cstdint>

namespace gemel {

// im2col map over an NHWC bf16 tensor [n, h, w, c] with channel pitch c_pitch
// (elements).  The pixel bounding box is [lower, dim-1+upper] per spatial dim,
// traversed with the conv stride; `chunk` channels x `pixels` pixels per box.
int tmap_encode_im2col(CUtensorMap* m, const void* ptr, int n, int h, int w, int c, int c_pitch, int lower_w,
                       int lower_h, int upper_w, int upper_h, int chunk, int pixels, int stride_w, int stride_h);

// 2-D tiled map over a row-major bf16 matrix [rows, cols] with row pitch in bytes.
int tmap_encode_2d(CUtensorMap* m, const void* ptr, uint64_t cols, uint64_t rows, uint64_t pitch_bytes,
                   int box_cols, int box_rows, int swizzle_bytes);

}  // namespace gemel
