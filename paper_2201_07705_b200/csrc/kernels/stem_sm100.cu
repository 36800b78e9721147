// Fused frame ingest + first convolution on the 5th-gen tensor cores (SURVEY.md
// §8(a) a6 + a7; §2.1's models all open with a 3-channel conv).
//
// One tile = up to 128 consecutive output pixels of one output row of one frame.
// Per tile, a 128-thread CTA
//   1. normalises the receptive-field input rows of the tile once into shared
//      memory (fp32, the same (x/255 - mean)/std fma as the preprocess kernel),
//   2. assembles the tile's im2col rows in shared memory (thread = output pixel,
//      column k = (r*kw + s)*3 + c, zero beyond K) as bf16 in the no-swizzle
//      K-major UMMA layout (8-column core-matrix groups of 128 rows x 16 B),
//   3. one thread issues K/16 tcgen05.mma (M = 128, N = Cout) into TMEM,
//   4. each warp drains its 32 TMEM lanes (tcgen05.ld), applies the folded
//      BN/bias + activation, stages its rows in shared memory (XOR-swizzled, no
//      bank conflicts) and writes them back as fully coalesced 16-byte stores
//      (a tile's output rows are contiguous in NHWC).
// The weights of the current task stay in shared memory across its tiles.  Several
// CTAs per SM overlap one another's load / MMA / store phases.  The im2col matrix
// the unfused path materialised in HBM (K8 x 2 bytes per output pixel, written by
// the ingest kernel and re-read by the GEMM) never leaves the SM.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "gemm.h"
#include "sm100_ptx.cuh"
#include "stem.h"

namespace gemel {
namespace {

constexpr int ST_THREADS = 128;   // = tile rows = TMEM lanes
constexpr int ST_BM = 128;

__host__ __device__ constexpr int st_align(int x, int a) { return (x + a - 1) / a * a; }

struct StemLayout {
  int koff, scale, shift, b, a, u, total;
};
__host__ __device__ inline StemLayout stem_layout(int n_max, int kp_max, int patch_max) {
  StemLayout L;
  L.koff = 16;                                   // [0, 16): TMEM address, mbarrier
  L.scale = st_align(L.koff + kp_max * 4, 16);
  L.shift = L.scale + n_max * 4;
  L.b = st_align(L.shift + n_max * 4, 128);
  L.a = st_align(L.b + n_max * kp_max * 2, 128);
  L.u = st_align(L.a + ST_BM * kp_max * 2, 128);  // input patch (fp32), later the output staging
  const int u_bytes = patch_max * 4 > ST_BM * n_max * 2 ? patch_max * 4 : ST_BM * n_max * 2;
  L.total = st_align(L.u + u_bytes, 128);
  return L;
}

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// 16-byte unit v of staged row r (nv units per row): XOR swizzle so that 8 consecutive
// rows' unit v (the write pattern) and 8 consecutive units of the linear row-major
// order (the read-back pattern) both fall in distinct bank groups
__device__ __forceinline__ int stage_unit(int r, int v, int nv) {
  const int sw = nv >= 8 ? (r & 7) : ((r / (8 / nv)) & (nv - 1));
  return v ^ sw;
}

constexpr int ST_PF = 12;   // prefetched 4-byte words of input per thread (7x7/s2 tiles need <= 11)

// A tile's receptive field: kh input rows x wspan pixels starting at (ih0, iw0); the
// in-frame columns [px_lo, px_hi) of each in-frame row are fetched as aligned 4-byte
// words, S word slots per row
struct Geo {
  const uint8_t* fb;        // the frame
  int h, w, kh, ih0, iw0, wspan, px_lo, px_hi, S;
  int ow0, nvalid, oh;
  int64_t img;
};

__device__ __forceinline__ Geo tile_geo(const StemTask& T, int64_t tile) {
  Geo G;
  const int tpr = (T.wo + ST_BM - 1) / ST_BM;
  int64_t q = tile - T.tile_begin;
  const int seg = int(q % tpr);
  q /= tpr;
  G.oh = int(q % T.ho);
  G.img = q / T.ho;
  G.ow0 = seg * ST_BM;
  G.nvalid = min(ST_BM, T.wo - G.ow0);
  G.h = T.h; G.w = T.w; G.kh = T.kh;
  G.wspan = (G.nvalid - 1) * T.sw + T.kw;
  G.ih0 = G.oh * T.sh - T.ph;
  G.iw0 = G.ow0 * T.sw - T.pw;
  G.px_lo = max(G.iw0, 0);
  G.px_hi = min(G.iw0 + G.wspan, T.w);
  G.S = (G.wspan * 3 + 3) / 4 + 1;
  G.fb = T.src + G.img * int64_t(T.h) * T.w * 3;
  return G;
}

// word slots i0, i0 + 128, ... (row y = i / S, word j = i % S of the row's byte range)
__device__ __forceinline__ void patch_load(const Geo& G, int i0, uint32_t (&w)[ST_PF]) {
#pragma unroll
  for (int u = 0; u < ST_PF; ++u) {
    const int i = i0 + u * ST_THREADS;
    w[u] = 0u;
    if (i < G.kh * G.S) {
      const int y = i / G.S, j = i - y * G.S, ih = G.ih0 + y;
      if (ih >= 0 && ih < G.h && G.px_lo < G.px_hi) {
        const uintptr_t a0 = reinterpret_cast<uintptr_t>(G.fb + (int64_t(ih) * G.w + G.px_lo) * 3);
        const uintptr_t a1 = reinterpret_cast<uintptr_t>(G.fb + (int64_t(ih) * G.w + G.px_hi) * 3);
        const uintptr_t A = (a0 & ~uintptr_t(3)) + 4u * uintptr_t(j);
        if (A < a1) w[u] = __ldg(reinterpret_cast<const unsigned int*>(A));
      }
    }
  }
}

// normalise the loaded bytes into the fp32 patch [kh][wsp][3] (ImageNet (x/255 - mean) / std
// as x * a + b, the preprocess kernel's constants and fma)
__device__ __forceinline__ void patch_store(const Geo& G, int i0, const uint32_t (&w)[ST_PF], float* patch, int wsp) {
  const float A0 = 1.f / (255.f * 0.229f), A1 = 1.f / (255.f * 0.224f), A2 = 1.f / (255.f * 0.225f);
  const float B0 = -0.485f / 0.229f, B1 = -0.456f / 0.224f, B2 = -0.406f / 0.225f;
#pragma unroll
  for (int u = 0; u < ST_PF; ++u) {
    const int i = i0 + u * ST_THREADS;
    if (i >= G.kh * G.S) continue;
    const int y = i / G.S, j = i - y * G.S, ih = G.ih0 + y;
    if (ih < 0 || ih >= G.h || G.px_lo >= G.px_hi) continue;
    const uintptr_t row = reinterpret_cast<uintptr_t>(G.fb + int64_t(ih) * G.w * 3);
    const uintptr_t a0 = row + uintptr_t(G.px_lo) * 3;
    const int off0 = int(((a0 & ~uintptr_t(3)) + 4u * uintptr_t(j)) - row);   // byte offset in the row (< 2^31)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int off = off0 + b;
      if (off < G.px_lo * 3 || off >= G.px_hi * 3) continue;
      const int p = off / 3, c = off - p * 3;
      const float x = float((w[u] >> (8 * b)) & 0xFFu);
      const float v = c == 0 ? fmaf(x, A0, B0) : (c == 1 ? fmaf(x, A1, B1) : fmaf(x, A2, B2));
      patch[(y * wsp + (p - G.iw0)) * 3 + c] = v;
    }
  }
}

__global__ void __launch_bounds__(ST_THREADS) stem_kernel(const StemTask* __restrict__ tasks, int n_tasks,
                                                         int64_t tile0, int64_t total, int n_max, int kp_max,
                                                         int patch_max) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const StemLayout SL = stem_layout(n_max, kp_max, patch_max);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm);
  const uint32_t bar = ptx::smem_u32(sm + 8);
  int* koff = reinterpret_cast<int*>(sm + SL.koff);
  float* s_scale = reinterpret_cast<float*>(sm + SL.scale);
  float* s_shift = reinterpret_cast<float*>(sm + SL.shift);
  uint8_t* sB = sm + SL.b;
  uint8_t* sA = sm + SL.a;
  uint8_t* sU = sm + SL.u;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint32_t ncols = 32;
  while (ncols < uint32_t(n_max)) ncols <<= 1;
  if (warp == 0) ptx::tmem_alloc(ptx::smem_u32(tmem_slot), ncols);
  if (tid == 0) {
    ptx::mbar_init(bar, 1);
    ptx::fence_mbar_init();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  int ti = 0, cur = -1;
  uint32_t phase = 0;
  uint32_t pw[ST_PF];   // the next tile's input bytes, loaded while this tile's MMA and epilogue run
  int64_t tile = tile0 + blockIdx.x;   // tiles [tile0, total) of the task table
  if (tile < total) {
    while (ti + 1 < n_tasks && tile >= tasks[ti + 1].tile_begin) ++ti;
    const Geo g = tile_geo(tasks[ti], tile);
    if (g.kh * g.S <= ST_THREADS * ST_PF) patch_load(g, tid, pw);
  }
  for (; tile < total; tile += gridDim.x) {
    while (ti + 1 < n_tasks && tile >= tasks[ti + 1].tile_begin) ++ti;   // tiles visit tasks in order
    const StemTask& T = tasks[ti];
    const int kp = st_align(T.K, 16), nj = kp / 8, N = T.N;
    const int wsp = (ST_BM - 1) * T.sw + T.kw;   // patch row pitch (pixels)
    if (ti != cur) {   // the task's weights, column offsets and epilogue vectors
      for (int k = tid; k < kp; k += ST_THREADS) {
        int o = -1;
        if (k < T.K) {
          const int tap = k / 3, c = k - tap * 3, r = tap / T.kw, s = tap - r * T.kw;
          o = (r * wsp + s) * 3 + c;
        }
        koff[k] = o;
      }
      for (int n = tid; n < N; n += ST_THREADS) {
        s_scale[n] = T.scale[n];
        s_shift[n] = T.shift[n];
      }
      const uint4* wg = static_cast<const uint4*>(T.wgt);
      const int ldv = T.ldw / 8;
      for (int i = tid; i < N * nj; i += ST_THREADS) {   // B: 8-column group j of row n at j*N*16 + n*16
        const int n = i % N, j = i / N;
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        if (j < ldv) v = wg[int64_t(n) * ldv + j];
        *reinterpret_cast<uint4*>(sB + j * (N * 16) + n * 16) = v;
      }
      cur = ti;
    }
    // tile -> (frame, output row, first output column) and its receptive input rows
    const Geo G = tile_geo(T, tile);
    const int ow0 = G.ow0, nvalid = G.nvalid;
    const int64_t img = G.img;
    const int oh = G.oh;
    float* patch = reinterpret_cast<float*>(sU);
    // zero padding (rows outside the frame, columns left / right of it), then the frame bytes
    for (int y = 0; y < G.kh; ++y) {
      const int ih = G.ih0 + y;
      const bool rv = ih >= 0 && ih < G.h && G.px_lo < G.px_hi;
      const int left = rv ? G.px_lo - G.iw0 : G.wspan, right = rv ? G.iw0 + G.wspan - G.px_hi : 0;
      for (int x = tid; x < left + right; x += ST_THREADS) {
        const int xx = x < left ? x : G.wspan - right + (x - left);
        float* d = patch + (y * wsp + xx) * 3;
        d[0] = 0.f;
        d[1] = 0.f;
        d[2] = 0.f;
      }
    }
    if (G.kh * G.S <= ST_THREADS * ST_PF) {
      patch_store(G, tid, pw, patch, wsp);
    } else {   // wider than the prefetch registers: load and store in rounds
      for (int i0 = tid; i0 < G.kh * G.S; i0 += ST_THREADS * ST_PF) {
        uint32_t tmp[ST_PF];
        patch_load(G, i0, tmp);
        patch_store(G, i0, tmp, patch, wsp);
      }
    }
    __syncthreads();
    {   // im2col row `tid` (rows past nvalid read stale patch values and are never stored)
      const float* base = patch + tid * T.sw * 3;
      for (int j = 0; j < nj; ++j) {
        float v[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int o = koff[j * 8 + e];
          v[e] = o >= 0 ? base[o] : 0.f;
        }
        *reinterpret_cast<uint4*>(sA + j * (ST_BM * 16) + tid * 16) =
            make_uint4(pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]), pack_bf16x2(v[4], v[5]),
                       pack_bf16x2(v[6], v[7]));
      }
    }
    ptx::fence_proxy_async_smem();   // generic-proxy smem writes -> visible to the tensor core
    __syncthreads();
    if (tid == 0) {
      ptx::tc_fence_after();
      const uint32_t idesc = ptx::idesc_bf16_m128(uint32_t(N));
      const uint64_t a0 = ptx::umma_desc(ptx::smem_u32(sA), ST_BM * 16, 128, 0);
      const uint64_t b0 = ptx::umma_desc(ptx::smem_u32(sB), uint32_t(N) * 16, 128, 0);
      for (int st = 0; st < kp / 16; ++st)
        ptx::umma_bf16(tmem, a0 + uint64_t((2 * st * ST_BM * 16) >> 4), b0 + uint64_t((2 * st * N * 16) >> 4), idesc,
                       st ? 1u : 0u);
      ptx::umma_commit(bar);
    }
    {   // the next tile's input bytes: in flight while this tile's MMA and epilogue run
      const int64_t nt = tile + gridDim.x;
      if (nt < total) {
        int tn = ti;
        while (tn + 1 < n_tasks && nt >= tasks[tn + 1].tile_begin) ++tn;
        const Geo g = tile_geo(tasks[tn], nt);
        if (g.kh * g.S <= ST_THREADS * ST_PF) patch_load(g, tid, pw);
      }
    }
    ptx::mbar_wait(bar, phase);
    phase ^= 1u;
    ptx::tc_fence_after();
    // epilogue: warp w owns TMEM lanes / tile rows [32w, 32w + 32); the patch is dead
    // (all reads happened before the last barrier), its space stages the output rows
    const int nv = N / 8;
    uint8_t* stg = sU + warp * 32 * N * 2;
    for (int c0 = 0; c0 < N; c0 += 32) {
      uint32_t v[32];
      ptx::tmem_ld_32x32b_x32(tmem + (uint32_t(warp * 32) << 16) + uint32_t(c0), v);
      ptx::tmem_ld_wait();
      const float ns = T.act == ACT_RELU ? 0.f : (T.act == ACT_LEAKY ? T.slope : 1.f);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (c0 + u * 8 >= N) break;
        uint32_t p[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int n0 = c0 + u * 8 + 2 * e;
          float y0 = fmaf(__uint_as_float(v[u * 8 + 2 * e]), s_scale[n0], s_shift[n0]);
          float y1 = fmaf(__uint_as_float(v[u * 8 + 2 * e + 1]), s_scale[n0 + 1], s_shift[n0 + 1]);
          y0 = fmaf(ns, fminf(y0, 0.f), fmaxf(y0, 0.f));
          y1 = fmaf(ns, fminf(y1, 0.f), fmaxf(y1, 0.f));
          p[e] = pack_bf16x2(y0, y1);
        }
        const int vv = c0 / 8 + u;
        *reinterpret_cast<uint4*>(stg + lane * N * 2 + 16 * stage_unit(lane, vv, nv)) = make_uint4(p[0], p[1], p[2], p[3]);
      }
    }
    __syncwarp();
    {
      const int r0 = warp * 32;
      const int vr = max(0, min(32, nvalid - r0));
      uint4* dst = reinterpret_cast<uint4*>(static_cast<uint8_t*>(T.out) +
                                            (((img * T.ho + oh) * int64_t(T.wo)) + ow0 + r0) * int64_t(N) * 2);
      for (int g = lane; g < vr * nv; g += 32) {
        const int row = g / nv, vv = g - row * nv;
        dst[g] = *reinterpret_cast<const uint4*>(stg + row * N * 2 + 16 * stage_unit(row, vv, nv));
      }
    }
    ptx::tc_fence_before();
    __syncthreads();   // TMEM, A, patch / staging free for the next tile
  }
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc(tmem, ncols);
}

}  // namespace

int stem_smem_bytes(int n_max, int kp16_max, int patch_floats_max) {
  return stem_layout(n_max, kp16_max, patch_floats_max).total;
}

int launch_stem(const StemTask* tasks, int n_tasks, int64_t tile0, int64_t tiles, int n_max, int kp16_max,
                int patch_floats_max, int sm_count, void* stream) {
  if (tiles <= 0) return 0;
  const int smem = stem_smem_bytes(n_max, kp16_max, patch_floats_max);
  cudaError_t e = cudaFuncSetAttribute(stem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return int(e);
  int occ = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, stem_kernel, ST_THREADS, smem);
  if (e != cudaSuccess) return int(e);
  int ncols = 32;
  while (ncols < n_max) ncols <<= 1;
  occ = occ < 512 / ncols ? occ : 512 / ncols;   // every resident CTA holds its TMEM columns
  if (occ < 1) occ = 1;
  const int64_t grid = tiles < int64_t(sm_count) * occ ? tiles : int64_t(sm_count) * occ;
  stem_kernel<<<unsigned(grid), ST_THREADS, smem, static_cast<cudaStream_t>(stream)>>>(
      tasks, n_tasks, tile0, tile0 + tiles, n_max, kp16_max, patch_floats_max);
  return int(cudaGetLastError());
}

}  // namespace gemel
