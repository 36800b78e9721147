// Fused frame ingest + first convolution on the 5th-gen tensor cores (SURVEY.md
// §8(a) a6 + a7; §2.1's models all open with a 3-channel conv).
//
// Persistent, warp-specialised (one CTA per SM, 576 threads).  A tile = 128
// consecutive output pixels of one member (flattened (image, row, column) order), so
// its output rows are one contiguous NHWC byte range.
//   warp 17    : frame loader.  The input rows a tile reads (one contiguous byte range
//                of the uint8 staging buffer: its receptive rows, full width) are
//                fetched by one bulk async copy (cp.async.bulk -> mbarrier) into a ring
//                of up to ST_MAX_IN shared-memory slots, that many tiles ahead.
//   warps 0-7  : A builders.  Thread (row p, half h) assembles im2col row p of the
//                tile -- column k = (r*kw + s)*3 + c, zero beyond K and outside the
//                frame -- for the 8-column groups j = h, h+2, ...: the frame bytes are
//                read from the slot, normalised with the preprocess kernel's fma
//                ((x/255 - mean)/std as x * a + b, fp32) and stored as bf16 in the
//                no-swizzle K-major UMMA layout.  Up to ST_MAX_STAGES tiles in flight.  (Frames
//                whose row pitch is not a multiple of 16 bytes are read from global
//                memory directly.)
//   warp 16    : TMEM allocator + single-thread tcgen05.mma issuer (M = 128, N = Cout,
//                K = 16 per instruction; weights resident in shared memory for the whole
//                launch), four TMEM accumulators (two when N > 128).
//   warps 8-15 : epilogue, two groups of four (one warp per TMEM lane quadrant) taking
//                alternate tiles, so one tile's epilogue latency overlaps the next's: tcgen05.ld -> folded BN/bias +
//                activation (the GEMM epilogue's arithmetic) -> bf16, transposed through a
//                per-warp swizzled smem slice -> coalesced 512-byte st.global.v4 rows.
// The im2col matrix the unfused path materialises in HBM (K8 x 2 bytes per output pixel,
// written by the ingest kernel and re-read by the GEMM) never leaves the SM: HBM traffic
// is the frame bytes in and the NHWC activation out.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "gemm.h"
#include "memops.h"
#include "smem_attr.cuh"
#include "sm100_ptx.cuh"
#include "stem.h"

namespace gemel {
namespace {

constexpr int ST_BM = 128;
constexpr int ST_PROD_WARPS = 8;                 // A builders: 2 threads per tile row
constexpr int ST_EPI_WARPS = 8;                  // two groups of 4 (one per TMEM lane quadrant), alternate tiles
constexpr int ST_MMA_WARP = ST_PROD_WARPS + ST_EPI_WARPS;   // warp 16
constexpr int ST_LOAD_WARP = ST_MMA_WARP + 1;               // warp 17
constexpr int ST_THREADS = 32 * (ST_LOAD_WARP + 1);
constexpr int ST_MAX_STAGES = 6;                 // A tiles in flight: as many as shared memory allows
constexpr int ST_MAX_IN = 6;                     // frame-row slots in flight (as many as fit)
constexpr int ST_KMAX = 256;

#define GEMEL_NA0 (1.f / (255.f * 0.229f))
#define GEMEL_NA1 (1.f / (255.f * 0.224f))
#define GEMEL_NA2 (1.f / (255.f * 0.225f))
#define GEMEL_NB0 (-0.485f / 0.229f)
#define GEMEL_NB1 (-0.456f / 0.224f)
#define GEMEL_NB2 (-0.406f / 0.225f)
__constant__ float kNormA[3] = {GEMEL_NA0, GEMEL_NA1, GEMEL_NA2};
__constant__ float kNormB[3] = {GEMEL_NB0, GEMEL_NB1, GEMEL_NB2};
__host__ __device__ constexpr int st_align(int x, int a) { return (x + a - 1) / a * a; }

struct StemLayout {
  int bars, vec, b, a, o, in, total;
};
__host__ __device__ inline StemLayout stem_layout(int n_max, int kp_max, int in_slot, int stages, int n_in) {
  const int sub = stem_sub(kp_max);
  StemLayout L;
  L.bars = 0;   // 2*ST_MAX_STAGES + 8 + 2*ST_MAX_IN mbarriers (256 B); [256, 280) slot rows g0; TMEM slot at 288
  L.vec = 320;                                         // float [2 groups][2][n_max]: scale, shift of the member
  L.b = st_align(L.vec + 4 * n_max * 4, 1024);         // bf16 B: [kp/8][n][8]
  L.a = st_align(L.b + n_max * kp_max * 2, 1024);      // stages x bf16 A: [kp/8][128][8]
  L.o = st_align(L.a + stages * sub * ST_BM * kp_max * 2, 1024);   // [8 warps][32][n] bf16 output transpose
  L.in = st_align(L.o + 2 * ST_BM * n_max * 2, 128);   // n_in x in_slot bytes of frame rows
  L.total = st_align(L.in + n_in * in_slot + 16, 128);   // (+16: word loads of a run's tail)
  return L;
}

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

__device__ __forceinline__ float u8f(uint32_t b) {   // exact float(b) for b < 2^23, no I2F
  return __uint_as_float(0x4B000000u | b) - 8388608.f;
}

__device__ __forceinline__ int task_of(const StemTask* t, int n, int64_t tile, int k) {
  while (k + 1 < n && tile >= t[k + 1].tile_begin) ++k;
  return k;
}

// First global input row (image * h + row) a tile reads and the row count (0: none):
// the receptive rows of its first to its last output pixel, clipped to the frames.
// (A member's pixels, n_img * ho * wo, and its frames' rows fit 32 bits: checked at bind.)
__device__ __forceinline__ int tile_rows(const StemTask& T, int64_t t, int tm, int& n_rows) {
  const int HoWo = T.ho * T.wo, M = T.n_img * HoWo;
  const int m0 = int(t - T.tile_begin) * tm, m1 = min(M, m0 + tm) - 1;
  const int img0 = m0 / HoWo, img1 = m1 / HoWo;
  const int oh0 = (m0 - img0 * HoWo) / T.wo, oh1 = (m1 - img1 * HoWo) / T.wo;
  const int g0 = img0 * T.h + max(0, oh0 * T.sh - T.ph);
  const int g1 = img1 * T.h + min(T.h - 1, oh1 * T.sh - T.ph + T.kh - 1);
  n_rows = g1 >= g0 ? g1 - g0 + 1 : 0;
  return g0;
}

// byte b of x as an exact float: 0x4B0000bb - 2^23 (one byte permute + one add, no I2F)
__device__ __forceinline__ float byte_f(uint32_t x, int b) {
  return __uint_as_float(__byte_perm(x, 0x4B000000u, 0x7440u | uint32_t(b))) - 8388608.f;
}

__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

__device__ __forceinline__ void put_group(uint8_t* As, int j, int p, const float (&v)[8]) {
  *reinterpret_cast<uint4*>(As + j * (ST_BM * 16) + p * 16) =
      make_uint4(pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]), pack_bf16x2(v[4], v[5]), pack_bf16x2(v[6], v[7]));
}

// Interior pixel, GPR groups per filter row (3*kw <= 8*GPR bytes): rows half, half + 2, ...
template <int GPR>
__device__ __forceinline__ void build_rows(const uint8_t* slot, int base, int row3, int kh, int half, uint8_t* As,
                                           int p) {
  constexpr int NW = 2 * GPR + 1;   // words covering a run plus its byte offset
  const float A0 = kNormA[0], A1 = kNormA[1], A2 = kNormA[2], B0 = kNormB[0], B1 = kNormB[1], B2 = kNormB[2];
  for (int r = half; r < kh; r += 2) {   // (hoisting every row's loads first measured slower)
    const int so = base + r * row3;
    const uint32_t* wp = reinterpret_cast<const uint32_t*>(slot + (so & ~3));
    const uint32_t sh = uint32_t(so & 3) * 8u;
    uint32_t w[NW];
#pragma unroll
    for (int k = 0; k < NW; ++k) w[k] = wp[k];
#pragma unroll
    for (int u = 0; u < GPR; ++u) {
      const uint32_t lo = __funnelshift_r(w[2 * u], w[2 * u + 1], sh);
      const uint32_t hi = __funnelshift_r(w[2 * u + 1], w[2 * u + 2], sh);
      float v[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int c = (2 * u + e) % 3;   // compile-time
        v[e] = fmaf(byte_f(e < 4 ? lo : hi, e & 3), c == 0 ? A0 : (c == 1 ? A1 : A2), c == 0 ? B0 : (c == 1 ? B1 : B2));
      }
      put_group(As, r * GPR + u, p, v);   // bytes past the run (group tail) meet zero weight columns
    }
  }
}

__global__ void __launch_bounds__(ST_THREADS, 1) stem_kernel(const StemTask* __restrict__ tasks, int n_tasks,
                                                            int64_t tile0, int64_t tile_end, int n_max, int kp_max,
                                                            int in_slot, int stages, int n_in) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const StemLayout SL = stem_layout(n_max, kp_max, in_slot, stages, n_in);
  const bool direct = in_slot == 0;   // frames read from global memory (row pitch not 16-byte aligned)
  const uint32_t bars = ptx::smem_u32(sm + SL.bars);
  const uint32_t bar_full = bars, bar_empty = bars + 8 * ST_MAX_STAGES;
  const uint32_t bar_tfull = bars + 16 * ST_MAX_STAGES, bar_tempty = bar_tfull + 32;
  const uint32_t bar_ifull = bar_tempty + 32, bar_iempty = bar_ifull + 8 * ST_MAX_IN;   // 32 barriers: [0, 256)
  int* s_g0 = reinterpret_cast<int*>(sm + 256);            // first global frame row of each slot
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + 288);
  float* s_vec = reinterpret_cast<float*>(sm + SL.vec);
  uint8_t* sB = sm + SL.b;
  uint8_t* sA = sm + SL.a;
  uint8_t* sO = sm + SL.o;
  const uint8_t* sIn = sm + SL.in;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // every member of a launch is one merged problem: one weight, one layer shape
  const int t_first = task_of(tasks, n_tasks, tile0 + blockIdx.x, 0);
  const StemTask& T0 = tasks[t_first];
  // K layout: filter row r owns G8 = 8 * stem_row_groups(kw) columns (r*G8 + s*3 + c; the
  // rest zero), so each 8-column group of A is 8 consecutive bytes of one frame row
  const int N = T0.N, KW3 = 3 * T0.kw, G8 = 8 * stem_row_groups(T0.kw), kp = stem_kp(T0.kh, T0.kw), nj = kp / 8;
  const int sub = stem_sub(kp), TM = ST_BM * sub;   // 128-row MMA sub-tiles per tile, tile rows
  const uint32_t a_sub = uint32_t(ST_BM) * kp * 2, a_stage = a_sub * sub;
  // TMEM accumulators: 4 when they fit (N <= 128), else 2 -- the MMA runs ahead of the
  // two epilogue groups
  const int n_acc = 4 * stem_sub(kp) * N <= 512 ? 4 : 2;   // an accumulator holds sub x N columns
  uint32_t ncols = 32;
  while (ncols < uint32_t(n_acc * stem_sub(kp) * N)) ncols <<= 1;

  if (tid == 0) {
    for (int s = 0; s < stages; ++s) {
      ptx::mbar_init(bar_full + 8 * s, 32 * ST_PROD_WARPS);
      ptx::mbar_init(bar_empty + 8 * s, 1);
    }
    for (int a = 0; a < 4; ++a) {
      ptx::mbar_init(bar_tfull + 8 * a, 1);
      ptx::mbar_init(bar_tempty + 8 * a, 4);
    }
    for (int i = 0; i < n_in; ++i) {
      ptx::mbar_init(bar_ifull + 8 * i, 1);
      ptx::mbar_init(bar_iempty + 8 * i, 32 * ST_PROD_WARPS);
    }
    ptx::fence_mbar_init();
  }
  if (warp == ST_MMA_WARP) ptx::tmem_alloc(ptx::smem_u32(tmem_slot), ncols);
  {   // weights, remapped to the padded K: column k' of row n at (k'/8)*N*16 + n*16 + (k'%8)*2
      // (no-swizzle K-major core matrices); k' = r*G8 + q holds the registered column
      // r*3*kw + q for q < 3*kw, zero otherwise
    const uint16_t* wg = static_cast<const uint16_t*>(T0.wgt);
    for (int i = tid; i < N * kp; i += ST_THREADS) {
      const int n = i / kp, k2 = i - n * kp, r = k2 / G8, q = k2 - r * G8;
      const uint16_t v = (r < T0.kh && q < KW3) ? wg[int64_t(n) * T0.ldw + r * KW3 + q] : uint16_t(0);
      *reinterpret_cast<uint16_t*>(sB + (k2 >> 3) * (N * 16) + n * 16 + (k2 & 7) * 2) = v;
    }
  }
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < ST_PROD_WARPS) {
    // ------------------------------------------------------------ A builders
    const int p = tid & (ST_BM - 1), half = tid >> 7;
    const int GPR = G8 / 8;   // 8-column groups per filter row
    const int kh = T0.kh;
    int ti = t_first, s = 0, is = 0;
    uint32_t ph = 0, iph = 0;
    for (int64_t t = tile0 + blockIdx.x; t < tile_end; t += gridDim.x) {
      ti = task_of(tasks, n_tasks, t, ti);
      const StemTask& T = tasks[ti];
      const int HoWo = T.ho * T.wo;
      const uint8_t* slot = sIn + is * in_slot;
      const int row3 = T.w * 3;
      int g0 = 0;
      if (!direct) {   // this tile's frame rows, landed in slot `is`
        ptx::mbar_wait(bar_ifull + 8 * is, iph);
        g0 = s_g0[is];
      }
      ptx::mbar_wait(bar_empty + 8 * s, ph ^ 1);
      for (int sb = 0; sb < sub; ++sb) {   // the tile's 128-row sub-tiles
      const int m = int(t - T.tile_begin) * TM + sb * ST_BM + p;
      const bool valid = m < T.n_img * HoWo;
      const int img = m / HoWo, rem = m - img * HoWo, oh = rem / T.wo, ow = rem - oh * T.wo;
      const int ih0 = oh * T.sh - T.ph, iw0 = ow * T.sw - T.pw;
      const bool interior = valid && ih0 >= 0 && ih0 + kh <= T.h && iw0 >= 0 && iw0 + T.kw <= T.w;
      uint8_t* As = sA + s * a_stage + sb * a_sub;
      auto put = [&](int j, const float (&v)[8]) {
        *reinterpret_cast<uint4*>(As + j * (ST_BM * 16) + p * 16) =
            make_uint4(pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]), pack_bf16x2(v[4], v[5]),
                       pack_bf16x2(v[6], v[7]));
      };
      if (interior && !direct && (GPR == 2 || GPR == 3)) {
        // this thread's filter rows r = half, half + 2, ...: each row's 3*kw frame bytes (one
        // run) are loaded as aligned words -- every row's words first, so the loads overlap
        // -- then each 8-byte group is funnel-shifted out and its bytes permuted into exact
        // floats; the group's first channel (8u mod 3) is a compile-time constant, so the
        // preprocess constants stay in registers
        const int base = ((img * T.h + ih0 - g0) * T.w + iw0) * 3;
        if (GPR == 2) build_rows<2>(slot, base, row3, kh, half, As, p);
        else build_rows<3>(slot, base, row3, kh, half, As, p);
        for (int j = kh * GPR + half; j < nj; j += 2) {   // K padding groups
          const float z[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
          put(j, z);
        }
      } else {   // frame border, padding rows / columns, other widths or unaligned frames
        for (int j = half; j < nj; j += 2) {
          const int r = j / GPR, u = j - r * GPR;
          float v[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int qq = 8 * u + e, s2 = qq / 3, c = qq - s2 * 3;
            const int ih = ih0 + r, iw = iw0 + s2;
            float x = 0.f;
            if (valid && r < kh && qq < KW3 && ih >= 0 && ih < T.h && iw >= 0 && iw < T.w) {
              const uint32_t b = direct ? __ldg(T.src + (int64_t(img * T.h + ih) * T.w + iw) * 3 + c)
                                        : slot[(img * T.h + ih - g0) * row3 + iw * 3 + c];
              x = fmaf(u8f(b), kNormA[c], kNormB[c]);
            }
            v[e] = x;
          }
          put(j, v);
        }
      }
      }   // sub-tiles
      ptx::fence_proxy_async_smem();   // generic-proxy smem writes -> the tensor core reads
      ptx::mbar_arrive(bar_full + 8 * s);
      if (++s == stages) { s = 0; ph ^= 1; }
      if (!direct) {   // the frame-row slot may be refilled
        ptx::mbar_arrive(bar_iempty + 8 * is);
        if (++is == n_in) { is = 0; iph ^= 1; }
      }
    }
  } else if (warp == ST_LOAD_WARP) {
    // ------------------------------------------------------------ frame loader
    if (lane == 0 && !direct) {
      int ti = t_first, is = 0;
      uint32_t iph = 0;
      for (int64_t t = tile0 + blockIdx.x; t < tile_end; t += gridDim.x) {
        ti = task_of(tasks, n_tasks, t, ti);
        const StemTask& T = tasks[ti];
        int n_rows;
        const int g0 = tile_rows(T, t, TM, n_rows);
        const uint32_t bytes = uint32_t(n_rows) * uint32_t(T.w) * 3u;
        ptx::mbar_wait(bar_iempty + 8 * is, iph ^ 1);
        s_g0[is] = g0;   // published to the builders by the slot's mbarrier (release / acquire)
        if (bytes) {
          ptx::mbar_arrive_expect_tx(bar_ifull + 8 * is, bytes);
          bulk_load(ptx::smem_u32(sIn + is * in_slot), T.src + int64_t(g0) * T.w * 3, bytes, bar_ifull + 8 * is);
        } else {
          ptx::mbar_arrive(bar_ifull + 8 * is);
        }
        if (++is == n_in) { is = 0; iph ^= 1; }
      }
    }
  } else if (warp == ST_MMA_WARP) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t idesc = ptx::idesc_bf16_m128(uint32_t(N));
      const uint64_t b0 = ptx::umma_desc(ptx::smem_u32(sB), uint32_t(N) * 16, 128, 0);
      int s = 0, k = 0;
      uint32_t ph = 0;
      for (int64_t t = tile0 + blockIdx.x; t < tile_end; t += gridDim.x, ++k) {
        const uint32_t acc = uint32_t(k % n_acc), acc_ph = uint32_t(k / n_acc) & 1u;
        ptx::mbar_wait(bar_tempty + 8 * acc, acc_ph ^ 1);
        ptx::mbar_wait(bar_full + 8 * s, ph);
        ptx::tc_fence_after();
        for (int sb = 0; sb < sub; ++sb) {   // sub-tile sb accumulates in columns [sb*N, sb*N + N)
          const uint64_t a0 = ptx::umma_desc(ptx::smem_u32(sA + s * a_stage + sb * a_sub), ST_BM * 16, 128, 0);
          for (int st = 0; st < kp / 16; ++st)
            ptx::umma_bf16(tmem + acc * uint32_t(sub * N) + uint32_t(sb * N), a0 + uint64_t((2 * st * ST_BM * 16) >> 4),
                           b0 + uint64_t((2 * st * N * 16) >> 4), idesc, st ? 1u : 0u);
        }
        ptx::umma_commit(bar_empty + 8 * s);   // the A stage is free once these MMAs retire
        ptx::umma_commit(bar_tfull + 8 * acc);
        if (++s == stages) { s = 0; ph ^= 1; }
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    // Each warp drains its 32 TMEM lanes (= tile rows) and transposes them through its own
    // smem slice (16-byte units XOR-swizzled by row: conflict-free both ways), then writes
    // the rows back in linear order -- every st.global.v4 of the warp covers 512
    // contiguous bytes (a tile's output rows are contiguous in NHWC).
    const int q = warp & 3;                    // TMEM lane quadrant
    const int grp = (warp - ST_PROD_WARPS) >> 2;   // epilogue group: tiles k with k % 2 == grp
    const int row = q * 32 + lane;
    float* s_scale = s_vec + grp * 2 * N;
    float* s_shift = s_scale + N;
    const int nv = N / 8;                      // 16-byte units per output row (2, 4, ..., 32)
    const bool pow2 = (nv & (nv - 1)) == 0;
    auto swz = [&](int r, int u) {             // unit u of slice row r -> its slot in the row
      if (!pow2) return u;                     // (Cout not a power of two: plain layout)
      return nv >= 8 ? (u ^ (r & 7)) : (u ^ ((r / (8 / nv)) & (nv - 1)));
    };
    uint8_t* slice = sO + (warp - ST_PROD_WARPS) * (32 * N * 2);
    int ti = t_first, cur = -1, k = 0;
    for (int64_t t = tile0 + blockIdx.x; t < tile_end; t += gridDim.x, ++k) {
      if ((k & 1) != grp) continue;            // the other group's tile
      ti = task_of(tasks, n_tasks, t, ti);
      const StemTask& T = tasks[ti];
      const uint32_t acc = uint32_t(k % n_acc), acc_ph = uint32_t(k / n_acc) & 1u;
      if (ti != cur) {   // this member's folded BN / bias
        ptx::named_bar_sync(2 + grp, 128);
        for (int n = row; n < N; n += 128) {
          s_scale[n] = T.scale[n];
          s_shift[n] = T.shift[n];
        }
        ptx::named_bar_sync(2 + grp, 128);
        cur = ti;
      }
      const float ns = T.act == ACT_RELU ? 0.f : (T.act == ACT_LEAKY ? T.slope : 1.f);
      ptx::mbar_wait(bar_tfull + 8 * acc, acc_ph);
      ptx::tc_fence_after();
      for (int sb = 0; sb < sub; ++sb) {   // the tile's 128-row sub-tiles, columns [sb*N, sb*N + N)
        for (int c0 = 0; c0 < N; c0 += 32) {
          uint32_t v[32];
          __syncwarp();
          ptx::tmem_ld_32x32b_x32(tmem + (uint32_t(q * 32) << 16) + acc * uint32_t(sub * N) + uint32_t(sb * N + c0), v);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (c0 + 8 * u >= N) break;
            uint32_t pk[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int n0 = c0 + 8 * u + 2 * e;
              float y0 = fmaf(__uint_as_float(v[8 * u + 2 * e]), s_scale[n0], s_shift[n0]);
              float y1 = fmaf(__uint_as_float(v[8 * u + 2 * e + 1]), s_scale[n0 + 1], s_shift[n0 + 1]);
              y0 = fmaf(ns, fminf(y0, 0.f), fmaxf(y0, 0.f));
              y1 = fmaf(ns, fminf(y1, 0.f), fmaxf(y1, 0.f));
              pk[e] = pack_bf16x2(y0, y1);
            }
            *reinterpret_cast<uint4*>(slice + lane * (N * 2) + swz(lane, c0 / 8 + u) * 16) =
                make_uint4(pk[0], pk[1], pk[2], pk[3]);
          }
        }
        if (sb == sub - 1) {   // every TMEM column of the tile has been read
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(bar_tempty + 8 * acc);   // the accumulator may be overwritten
        }
        const int64_t m0 = (t - T.tile_begin) * TM + sb * ST_BM + q * 32;   // this warp's first row
        const int64_t rows = min(int64_t(32), int64_t(T.n_img) * T.ho * T.wo - m0);
        uint4* dst = reinterpret_cast<uint4*>(static_cast<uint8_t*>(T.out) + m0 * N * 2);
        __syncwarp();
        for (int g = lane; g < 32 * nv; g += 32) {
          const int r = g / nv, u = g - r * nv;
          if (r < rows) dst[g] = *reinterpret_cast<const uint4*>(slice + r * (N * 2) + swz(r, u) * 16);
        }
        __syncwarp();   // the slice is rewritten by the next sub-tile / tile
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == ST_MMA_WARP) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, ncols);
  }
}

}  // namespace

int stem_smem_bytes(int n_max, int kp16_max, int in_slot) {
  return stem_layout(n_max, kp16_max, in_slot, 2, 2).total;   // the minimum (two A stages, two slots)
}

int launch_stem(const StemTask* tasks, int n_tasks, int64_t tile0, int64_t tiles, int n_max, int kp16_max,
                int in_slot, int sm_count, void* stream) {
  if (tiles <= 0) return 0;
  if (kp16_max > ST_KMAX || n_max > 256 || n_max % 16 || in_slot % 16) return int(cudaErrorInvalidValue);
  int dev = 0, optin = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (e != cudaSuccess) return int(e);
  // as many frame-row slots (latency of the bulk copies) and A stages as fit, keeping >= 3
  // stages while slots can be given up
  int stages = ST_MAX_STAGES, n_in = in_slot ? ST_MAX_IN : 1;
  auto fits = [&](int st, int ni) { return stem_layout(n_max, kp16_max, in_slot, st, ni).total <= optin; };
  while (!fits(stages, n_in) && stages > 3) --stages;
  while (!fits(stages, n_in) && n_in > 2) --n_in;
  while (!fits(stages, n_in) && stages > 2) --stages;
  const int smem = stem_layout(n_max, kp16_max, in_slot, stages, n_in).total;
  if (smem > optin) return int(cudaErrorInvalidValue);
  e = allow_max_dyn_smem(stem_kernel);
  if (e != cudaSuccess) return int(e);
  const int64_t grid = tiles < int64_t(sm_count) ? tiles : int64_t(sm_count);
  stem_kernel<<<unsigned(grid), ST_THREADS, smem, static_cast<cudaStream_t>(stream)>>>(
      tasks, n_tasks, tile0, tile0 + tiles, n_max, kp16_max, in_slot, stages, n_in);
  return int(cudaGetLastError());
}

}  // namespace gemel
