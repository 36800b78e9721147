// K1/K2: grouped implicit-GEMM convolution + linear on 5th-gen tensor cores.
//
// Persistent, warp-specialised sm_100a kernel (one CTA per SM, 192 threads):
//   warp 0      : TMA producer.  A tiles come from the NHWC bf16 activation via
//                 TMA *im2col* mode (128 output pixels x one (tap, channel-chunk)
//                 per box; conv padding = OOB zero fill, stride = traversal
//                 stride, dilation = tap offset); B tiles from the [N, K] weight
//                 via tiled TMA.  Both land in the same swizzle layout.
//   warp 1      : TMEM allocator + single-thread tcgen05.mma issuer (M=128,
//                 N=bn<=256, K=16 per instruction), fp32 accumulators in TMEM,
//                 double-buffered so the epilogue of tile i overlaps tile i+1.
//   warps 2..5  : epilogue: tcgen05.ld -> per-segment fp32 scale/shift (folded
//                 BN + bias), residual add, ReLU/LeakyReLU -> bf16 (or fp32) store.
// A launch runs every GEMM problem of one scheduler wave; a problem whose
// weight is shared by several models runs once over their concatenated
// batches (one weight copy), each model a segment.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "gemm.h"
#include "sm100_ptx.cuh"

namespace gemel {

namespace {

constexpr uint32_t A_STAGE_BYTES = GEMM_BM * GEMM_BK * 2;   // 16 KB

__device__ __forceinline__ int find_problem(const GemmProblem* __restrict__ P, int n, int tile) {
  int p = 0;
  while (p + 1 < n && tile >= P[p + 1].tile_begin) ++p;
  return p;
}

struct KLayout {
  uint32_t layout, sbo_a, sbo_b, lbo_a, lbo_b, region_a, region_b;
};

__device__ __forceinline__ KLayout k_layout(int chunk, int bn) {
  KLayout k;
  k.region_a = GEMM_BM * chunk * 2;
  k.region_b = bn * chunk * 2;
  switch (chunk) {
    case 64: k.layout = 2; k.sbo_a = k.sbo_b = 1024; k.lbo_a = k.lbo_b = 16; break;
    case 32: k.layout = 4; k.sbo_a = k.sbo_b = 512; k.lbo_a = k.lbo_b = 16; break;
    case 16: k.layout = 6; k.sbo_a = k.sbo_b = 256; k.lbo_a = k.lbo_b = 16; break;
    default: k.layout = 0; k.sbo_a = k.sbo_b = 128; k.lbo_a = k.region_a; k.lbo_b = k.region_b; break;
  }
  return k;
}

__device__ __forceinline__ float act_apply(float y, int act, float slope) {
  if (act == ACT_RELU) return fmaxf(y, 0.f);
  if (act == ACT_LEAKY) return y >= 0.f ? y : y * slope;
  return y;
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

__device__ __forceinline__ float bf16_lo(uint32_t u) { return __uint_as_float(u << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t u) { return __uint_as_float(u & 0xFFFF0000u); }

}  // namespace

extern "C" __global__ void __launch_bounds__(GEMM_THREADS, 1) gemel_gemm_sm100(const GemmLaunch L) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int stages = L.stages;
  const uint32_t b_stage_bytes = uint32_t(L.bn_max) * GEMM_BK * 2;
  uint8_t* sA = smem;
  uint8_t* sB = sA + stages * A_STAGE_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + stages * b_stage_bytes);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * stages + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t bar_full = ptx::smem_u32(bars);
  const uint32_t bar_empty = bar_full + 8 * stages;
  const uint32_t bar_tfull = bar_empty + 8 * stages;
  const uint32_t bar_tempty = bar_tfull + 16;
  const GemmProblem* __restrict__ probs = L.probs;

  uint32_t tmem_cols = 32;
  while (tmem_cols < uint32_t(2 * L.bn_max)) tmem_cols <<= 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      ptx::mbar_init(bar_full + 8 * s, 1);
      ptx::mbar_init(bar_empty + 8 * s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(bar_tfull + 8 * a, 1);
      ptx::mbar_init(bar_tempty + 8 * a, 4);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc(ptx::smem_u32(tmem_slot), tmem_cols);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      for (int p = 0; p < L.n_probs; ++p) {
        ptx::prefetch_tmap(&probs[p].tmap_a);
        ptx::prefetch_tmap(&probs[p].tmap_b);
      }
      int s = 0;
      uint32_t ph = 0;
      for (int tile = blockIdx.x; tile < L.total_tiles; tile += gridDim.x) {
        const GemmProblem& P = probs[find_problem(probs, L.n_probs, tile)];
        const int local = tile - P.tile_begin;
        const int m_tile = local / P.n_tiles, n_tile = local - m_tile * P.n_tiles;
        const int m0 = m_tile * GEMM_BM;
        const int img = m0 / P.HoWo, rem = m0 - img * P.HoWo;
        const int oh = rem / P.Wo, ow = rem - oh * P.Wo;
        const int w0 = ow * P.sw - P.pw, h0 = oh * P.sh - P.ph;
        const int chunk = P.chunk, R = GEMM_BK / chunk, cpt = P.cin_k / chunk;
        const KLayout kl = k_layout(chunk, P.bn);
        const uint32_t tx = uint32_t(R) * (kl.region_a + kl.region_b);
        const int n0 = n_tile * P.bn;
        for (int ks = 0; ks < P.n_kstages; ++ks) {
          ptx::mbar_wait(bar_empty + 8 * s, ph ^ 1);
          const uint32_t fb = bar_full + 8 * s;
          ptx::mbar_arrive_expect_tx(fb, tx);
          const uint32_t a_dst = ptx::smem_u32(sA + s * A_STAGE_BYTES);
          const uint32_t b_dst = ptx::smem_u32(sB + s * b_stage_bytes);
          for (int j = 0; j < R; ++j) {
            const int sub = ks * R + j;
            if (sub < P.n_sub) {
              const int tap = sub / cpt, c0 = (sub - tap * cpt) * chunk;
              const int r = tap / P.kw, t = tap - r * P.kw;
              ptx::tma_load_im2col_4d(a_dst + j * kl.region_a, &P.tmap_a, fb, c0, w0, h0, img,
                                      uint16_t(t * P.dw), uint16_t(r * P.dh));
              ptx::tma_load_2d(b_dst + j * kl.region_b, &P.tmap_b, fb, tap * P.cin_k + c0, n0);
            } else {  // K tail of the last stage: fully out-of-bounds boxes (zero fill)
              ptx::tma_load_im2col_4d(a_dst + j * kl.region_a, &P.tmap_a, fb, P.c_oob, w0, h0, img, 0, 0);
              ptx::tma_load_2d(b_dst + j * kl.region_b, &P.tmap_b, fb, P.Ktot, n0);
            }
          }
          if (++s == stages) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0, acc = 0, acc_ph = 0;
      for (int tile = blockIdx.x; tile < L.total_tiles; tile += gridDim.x) {
        const GemmProblem& P = probs[find_problem(probs, L.n_probs, tile)];
        const int chunk = P.chunk;
        const KLayout kl = k_layout(chunk, P.bn);
        const uint32_t idesc = ptx::idesc_bf16_m128(uint32_t(P.bn));
        ptx::mbar_wait(bar_tempty + 8 * acc, acc_ph ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * uint32_t(L.bn_max);
        for (int ks = 0; ks < P.n_kstages; ++ks) {
          ptx::mbar_wait(bar_full + 8 * s, ph);
          ptx::tc_fence_after();
          const uint32_t a_base = ptx::smem_u32(sA + s * A_STAGE_BYTES);
          const uint32_t b_base = ptx::smem_u32(sB + s * b_stage_bytes);
#pragma unroll
          for (int st = 0; st < GEMM_BK / 16; ++st) {
            uint32_t a_addr, b_addr;
            if (chunk >= 16) {
              const int kel = st * 16, j = kel / chunk, kk = (kel - j * chunk) / 16;
              a_addr = a_base + j * kl.region_a + kk * 32;
              b_addr = b_base + j * kl.region_b + kk * 32;
            } else {
              a_addr = a_base + (2 * st) * kl.region_a;
              b_addr = b_base + (2 * st) * kl.region_b;
            }
            const uint64_t ad = ptx::umma_desc(a_addr, kl.lbo_a, kl.sbo_a, kl.layout);
            const uint64_t bd = ptx::umma_desc(b_addr, kl.lbo_b, kl.sbo_b, kl.layout);
            ptx::umma_bf16(d_tmem, ad, bd, idesc, (ks | st) != 0 ? 1u : 0u);
          }
          ptx::umma_commit(bar_empty + 8 * s);   // frees the smem stage when these MMAs retire
          if (++s == stages) { s = 0; ph ^= 1; }
        }
        ptx::umma_commit(bar_tfull + 8 * acc);   // accumulator ready for the epilogue
        acc ^= 1;
        if (acc == 0) acc_ph ^= 1;
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;                  // TMEM lane quadrant this warp may access
    uint32_t acc = 0, acc_ph = 0;
    for (int tile = blockIdx.x; tile < L.total_tiles; tile += gridDim.x) {
      const GemmProblem& P = probs[find_problem(probs, L.n_probs, tile)];
      const int local = tile - P.tile_begin;
      const int m_tile = local / P.n_tiles, n_tile = local - m_tile * P.n_tiles;
      const int row = m_tile * GEMM_BM + q * 32 + lane;
      const int n0 = n_tile * P.bn, N = P.N;
      const bool valid = row < P.M;
      const GemmSeg* seg = L.segs + P.seg_begin;
      if (valid) {
        int si = 0;
        while (si + 1 < P.n_seg && row >= seg[si].m_end) ++si;
        seg += si;
      }
      const int64_t lrow = row - seg->m_begin;
      ptx::mbar_wait(bar_tfull + 8 * acc, acc_ph);
      ptx::tc_fence_after();
      for (int c = 0; c < P.bn; c += 32) {
        uint32_t v[32];
        ptx::tmem_ld_32x32b_x32(tmem_base + (uint32_t(q * 32) << 16) + acc * uint32_t(L.bn_max) + c, v);
        ptx::tmem_ld_wait();
        const int col0 = n0 + c;
        if (!valid || col0 >= N) continue;
        const float* __restrict__ sc = seg->scale + col0;
        const float* __restrict__ sf = seg->shift + col0;
        const int act = seg->act;
        const float slope = seg->slope;
        float y[32];
        if (col0 + 32 <= N) {
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            const float4 a = *reinterpret_cast<const float4*>(sc + j);
            const float4 b = *reinterpret_cast<const float4*>(sf + j);
            y[j + 0] = fmaf(__uint_as_float(v[j + 0]), a.x, b.x);
            y[j + 1] = fmaf(__uint_as_float(v[j + 1]), a.y, b.y);
            y[j + 2] = fmaf(__uint_as_float(v[j + 2]), a.z, b.z);
            y[j + 3] = fmaf(__uint_as_float(v[j + 3]), a.w, b.w);
          }
          if (seg->res) {
            const uint4* rp = reinterpret_cast<const uint4*>(
                reinterpret_cast<const __nv_bfloat16*>(seg->res) + lrow * seg->ldr + col0);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const uint4 r4 = rp[j];
              y[8 * j + 0] += bf16_lo(r4.x); y[8 * j + 1] += bf16_hi(r4.x);
              y[8 * j + 2] += bf16_lo(r4.y); y[8 * j + 3] += bf16_hi(r4.y);
              y[8 * j + 4] += bf16_lo(r4.z); y[8 * j + 5] += bf16_hi(r4.z);
              y[8 * j + 6] += bf16_lo(r4.w); y[8 * j + 7] += bf16_hi(r4.w);
            }
          }
#pragma unroll
          for (int j = 0; j < 32; ++j) y[j] = act_apply(y[j], act, slope);
          if (seg->out_fp32) {
            float4* op = reinterpret_cast<float4*>(reinterpret_cast<float*>(seg->out) + lrow * seg->ldo + col0);
#pragma unroll
            for (int j = 0; j < 8; ++j) op[j] = make_float4(y[4 * j], y[4 * j + 1], y[4 * j + 2], y[4 * j + 3]);
          } else {
            uint4* op = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(seg->out) + lrow * seg->ldo + col0);
#pragma unroll
            for (int j = 0; j < 4; ++j)
              op[j] = make_uint4(pack_bf16(y[8 * j + 0], y[8 * j + 1]), pack_bf16(y[8 * j + 2], y[8 * j + 3]),
                                 pack_bf16(y[8 * j + 4], y[8 * j + 5]), pack_bf16(y[8 * j + 6], y[8 * j + 7]));
          }
        } else {
          const __nv_bfloat16* rp =
              seg->res ? reinterpret_cast<const __nv_bfloat16*>(seg->res) + lrow * seg->ldr + col0 : nullptr;
          for (int j = 0; j < 32 && col0 + j < N; ++j) {
            float t = fmaf(__uint_as_float(v[j]), sc[j], sf[j]);
            if (rp) t += __bfloat162float(rp[j]);
            t = act_apply(t, act, slope);
            if (seg->out_fp32)
              reinterpret_cast<float*>(seg->out)[lrow * seg->ldo + col0 + j] = t;
            else
              reinterpret_cast<__nv_bfloat16*>(seg->out)[lrow * seg->ldo + col0 + j] = __float2bfloat16_rn(t);
          }
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(bar_tempty + 8 * acc);
      acc ^= 1;
      if (acc == 0) acc_ph ^= 1;
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem_base, tmem_cols);
  }
}

size_t gemm_smem_bytes(int bn_max, int stages) {
  return 1024 + size_t(stages) * (A_STAGE_BYTES + size_t(bn_max) * GEMM_BK * 2) + (2 * stages + 4) * 8 + 16;
}

int gemm_pick_stages(int bn_max) {
  int s = 8;
  while (s > 2 && gemm_smem_bytes(bn_max, s) > 227 * 1024) --s;
  return s;
}

int gemm_launch(const GemmLaunch& L, int grid, void* stream) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(gemel_gemm_sm100, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return int(e);
    attr_set = true;
  }
  const size_t smem = gemm_smem_bytes(L.bn_max, L.stages);
  gemel_gemm_sm100<<<grid, GEMM_THREADS, smem, static_cast<cudaStream_t>(stream)>>>(L);
  return int(cudaGetLastError());
}

}  // namespace gemel
