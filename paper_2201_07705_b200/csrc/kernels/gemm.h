// Grouped implicit-GEMM convolution / linear problem table (host + device).
//
// One launch runs a list of problems (a "wave").  A
// problem is D[m, n] = sum_k A[m, k] * W[n, k] with
//   m = (image, out_row, out_col) flattened over the problem's concatenated
//       batch (all models sharing the weight, PAPER.md:70/203 -- one weight
//       copy; SURVEY.md §8(a) a7 "batch union"),
//   k = (tap r, tap s, channel) with channels innermost (NHWC),
//   n = output channel.
// A is gathered by TMA im2col straight from the NHWC bf16 activation (no
// materialised im2col), W is the bf16 [N, K] weight.  Each problem carries a
// list of segments (one per member model) whose fp32 epilogue applies that
// model's folded BN (scale, shift), optional residual add and activation.
#pragma once
#include <cuda.h>
#include <cstdint>

namespace gemel {

enum GemmAct : int32_t { ACT_NONE = 0, ACT_RELU = 1, ACT_LEAKY = 2 };

struct alignas(128) GemmSeg {
  CUtensorMap out_map;         // bf16 out: 2-D [rows = m_end - m_begin, N] tiled, box 32x32, 64B swizzle
  CUtensorMap res_map;         // residual: same geometry (valid when res != nullptr)
  int32_t m_begin, m_end;      // problem rows [m_begin, m_end) belong to this member
  int32_t act;                 // GemmAct
  float slope;                 // LeakyReLU negative slope
  const float* scale;          // [N] fp32
  const float* shift;          // [N] fp32
  void* out;                   // bf16 or fp32; row (m - m_begin) at out + (m - m_begin) * ldo
  const void* res;             // optional bf16 residual, same row indexing with ldr
  int64_t ldo, ldr;            // row pitches (elements)
  int32_t out_fp32;            // 1: store fp32 (final logits / YOLO heads), 0: bf16
  int32_t res_post;            // 1: residual added after the activation (darknet shortcut)
  int32_t res_up;              // > 1: the residual is read nearest-upsampled by this factor
                               // (FPN top-down): row (img, y, x) reads coarse row
                               // img * res_hw + (y / res_up) * res_w + x / res_up
  int32_t res_w, res_hw;       // coarse residual W and H*W
  int32_t out_w, out_hw;       // this member's output Wo and Ho*Wo
  int32_t pad_[3];
};

struct alignas(128) GemmProblem {
  CUtensorMap tmap_a;          // im2col map over the input slab [img, H, W, Cs]
  CUtensorMap tmap_b;          // tiled map over W [N, Ktot]
  int32_t M, N, Ktot;
  int32_t HoWo, Wo;
  int32_t sh, sw, ph, pw;
  int32_t kw, dh, dw;
  int32_t cin_k;               // channels per tap in K (multiple of chunk)
  int32_t chunk;               // channels per TMA box: 8, 16, 32 or 64
  int32_t n_sub;               // (tap, channel-chunk) sub-tiles in K
  int32_t n_kstages;           // ceil(n_sub / (64 / chunk))
  int32_t c_oob;               // channel coordinate that is entirely out of bounds
  int32_t bn;                  // N tile (multiple of 16, <= 256)
  int32_t m_tiles, n_tiles, tile_begin;
  int32_t item_begin, run;     // tile-queue grabs: item i covers tiles [tile_begin + (i - item_begin) * run, +run)
  int32_t msub;                // 128-row sub-tiles per tile (1, 2, 4; a tile = msub consecutive m-tiles)
  int32_t seg_begin, n_seg;
  int32_t n_deps;              // producer problems (same launch) that must finish first
  int32_t deps[31];            // their indices in the launch's problem table
  int32_t ksplit;              // split-K factor (1 = none); tiles = m_tiles * n_tiles * ksplit
  int32_t kst_split;           // K stages per split (last split may have fewer)
  float* ws;                   // split-K fp32 partials [m*n tiles][ksplit][round_up(bn,32) cols][128 rows]
  int32_t* tcnt;               // split-K arrival counters per (m, n) tile (zeroed every step)
  int32_t a_tiled;             // 1: tmap_a is a plain 2-D tiled map over [M, C] (1x1 stride-1 conv / linear)
  int32_t cnt_off;             // its per-m-tile completion counters: sched[cnt_off + m_tile] (n-tiles done)
  const int32_t* dep_rng;      // [m_tiles][n_deps][2]: producer m-tiles [lo, hi] this m-tile reads (lo > hi: none)
};

static_assert(sizeof(CUtensorMap) == 128, "CUtensorMap size");

constexpr int GEMM_BM = 128;
constexpr int GEMM_BK = 64;            // K elements per pipeline stage
constexpr int GEMM_THREADS = 352;      // warp0 TMA, warp1 MMA, warps 2-9 epilogue (2 groups x 4 quadrants), warp10 scheduler
constexpr int GEMM_MAX_DEPS = 31;

struct GemmLaunch {
  const GemmProblem* probs;    // device
  const GemmSeg* segs;         // device
  int32_t* sched;              // device: [0] = next grab (dynamic queue), then per-m-tile completion counters
  unsigned long long* trace;   // optional [total_tiles][4] ns timestamps: grab, deps ready, acc ready, done
  int32_t n_probs;
  int32_t total_tiles;
  int32_t total_items;         // tile-queue grabs (sum over problems of ceil(tiles / run))
  int32_t bn_max;
  int32_t stages;
  int32_t cg;                  // 1: 128-row tiles, one CTA; 2: 256-row tiles on a CTA pair (cta_group::2)
  int32_t acc_w;               // TMEM columns of one accumulator: max over problems of msub * bn (<= 256)
  int32_t epi_flags;           // bit 0: output chunks leave through TMA stores (else the LSU transpose path);
                               // bit 1: the producer prefetches each tile's residual rows into L2;
                               // bit 2: one output staging buffer per warp instead of two
  int32_t dbg;                 // developer probes: bit0 skip MMA, bit1 skip operand TMA (0 in production)
};

// Host: smem bytes for a launch and the launcher (stream = cudaStream_t).
size_t gemm_smem_bytes(int bn_max, int stages, int cg);
int gemm_pick_stages(int bn_max, int cg);
int gemm_launch(const GemmLaunch& L, int grid, void* stream);

}  // namespace gemel
