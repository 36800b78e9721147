// Fused frame ingest + first convolution (SURVEY.md §8(a) a6 + a7 for the
// models' first layer): uint8 RGB frames -> normalised bf16 im2col rows built in
// shared memory -> tcgen05 MMA (M = 128 output pixels, N = Cout, K = kh*kw*3
// padded to 16) -> folded BN/bias + activation -> NHWC bf16.  The im2col matrix
// is never written to HBM (it was 3-20x the frame's bytes).
#pragma once
#include <cstdint>

namespace gemel {

struct StemTask {           // one member (model) of a first-conv problem
  const uint8_t* src;       // frames [n_img, h, w, 3] uint8 (staging buffer)
  const void* wgt;          // bf16 [N, ldw], column k = (r * kw + s) * 3 + c, zero beyond K
  const float* scale;       // fp32 [N] folded epilogue: y = act(acc * scale + shift)
  const float* shift;
  void* out;                // bf16 NHWC [n_img, ho, wo, N] (channel pitch == N)
  int64_t tile_begin;       // prefix over tasks of stem_tile_count(n_img, ho, wo, sub)
  int32_t n_img, h, w, ho, wo;
  int32_t kh, kw, sh, sw, ph, pw;
  int32_t K, ldw, N;        // K = kh*kw*3; ldw = weight row pitch (elements, multiple of 8); N % 16 == 0
  int32_t act;
  float slope;
  int32_t pad_;
};

// Padded K of the fused stem: each filter row's 3*kw (column, channel) bytes take
// stem_row_groups(kw) 8-column groups, the total rounded up to the MMA's K = 16.
#ifdef __CUDACC__
#define GEMEL_STEM_HD __host__ __device__
#else
#define GEMEL_STEM_HD
#endif
inline GEMEL_STEM_HD int stem_row_groups(int kw) { return (3 * kw + 7) / 8; }
inline GEMEL_STEM_HD int stem_kp(int kh, int kw) { return (kh * 8 * stem_row_groups(kw) + 15) / 16 * 16; }

// 128-row MMA sub-tiles per tile: two for narrow K (K' <= 64: the per-tile pipeline
// round trips, not the bytes, bound those stems), one otherwise (a 7x7 stem's A stage is
// already 44 KB).
inline GEMEL_STEM_HD int stem_sub(int kp) { return kp <= 64 ? 2 : 1; }

// A member's tiles: 128 * sub consecutive output pixels each (flattened (image, row, column)).
inline int64_t stem_tile_count(int n_img, int ho, int wo, int sub) {
  return (int64_t(n_img) * ho * wo + 128 * sub - 1) / (128 * sub);
}

// Frame-row slot bytes of a first conv (kh, sh, output width wo, input width w): the
// receptive rows of up to (128 sub - 1)/wo + 2 output rows, full width; 0 = read the frame
// from global memory (row pitch w*3 not a multiple of 16 bytes: no bulk copies).
inline int stem_in_slot_bytes(int kh, int sh, int wo, int w, int sub) {
  if ((w * 3) % 16) return 0;
  return ((128 * sub - 1) / wo + 2) * sh * w * 3 + kh * w * 3;
}

// Dynamic shared memory of a launch whose tasks have at most these sizes.
int stem_smem_bytes(int n_max, int kp16_max, int in_slot);
// Tiles [tile0, tile0 + tiles) of the task table (tile_begin prefixes over the whole table);
// every task in that range is a member of ONE first-conv problem (same weight and shape;
// frames of one width).  in_slot = stem_in_slot_bytes(...) of that problem.
int launch_stem(const StemTask* tasks, int n_tasks, int64_t tile0, int64_t tiles, int n_max, int kp16_max,
                int in_slot, int sm_count, void* stream);

}  // namespace gemel
