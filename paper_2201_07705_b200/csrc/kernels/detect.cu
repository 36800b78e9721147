// Faster R-CNN R50-FPN irregular stages on B200 (SURVEY.md §8(a) a9 "RPN top-k +
// NMS(0.7) + MultiScaleRoIAlign(7x7, sr = 2)", a11 box decode; include/gemel.h
// RPN_LEVEL / RPN_MERGE / ROI_ALIGN / BOX_POST give the exact semantics, DESIGN.md
// readings R15-R18 the choices the paper leaves open).
//
//  rpn_level_kernel  one CTA (1024 threads) per (model level, frame): radix select of
//                    the K highest objectness logits straight from the fp32 head (4
//                    passes of 8-bit histograms, L2-resident), index-ordered compaction,
//                    a bitonic sort of the K survivors (logit desc, index asc), BoxCoder
//                    decode + clip in fp32, the K x K IoU bitmask in shared memory (one
//                    thread per 32-column word, warp lanes on consecutive rows so box
//                    reads broadcast) and the greedy NMS scan by one warp (lane w owns
//                    removed-word w).  All levels of a step run in ONE launch (the
//                    planner schedules RPN_LEVEL as late as possible).
//  rpn_merge_kernel  one CTA per frame: bitonic sort of every level's kept rows, the
//                    first post_n written as proposals.
//  roi_align_kernel  a CTA per proposal, a thread per (bin, 8 channels): level from the
//                    box area, 4 bilinear samples of 16-byte NHWC bf16 vectors, fp32 average.
//  box_post_kernel   a warp per proposal: softmax over the class logits (warp
//                    reductions), BoxCoder(10,10,5,5) decode + clip per class.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "memops.h"

namespace gemel {
namespace {

constexpr float kXformClip = 4.135166556742356f;   // log(1000 / 16)

__device__ __forceinline__ uint32_t okey(float f) {   // order-preserving float -> uint32
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// exclusive prefix of a per-thread flag over a 1024-thread block; returns the block total
__device__ __forceinline__ int scan1024(bool flag, int* warp_tot, int& excl) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned b = __ballot_sync(0xffffffffu, flag);
  const int in_warp = __popc(b & ((1u << lane) - 1u));
  __syncthreads();
  if (lane == 0) warp_tot[wid] = __popc(b);
  __syncthreads();
  if (wid == 0) {
    const int v = warp_tot[lane];
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    warp_tot[lane] = incl - v;
    if (lane == 31) warp_tot[32] = incl;
  }
  __syncthreads();
  excl = warp_tot[wid] + in_warp;
  return warp_tot[32];
}

// ascending bitonic sort of P (power of two) 64-bit keys in shared memory, 1024 threads
__device__ void bitonic_sort(unsigned long long* a, int P) {
  for (int k = 2; k <= P; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      __syncthreads();
      for (int i = threadIdx.x; i < P; i += blockDim.x) {
        const int l = i ^ j;
        if (l > i) {
          const unsigned long long x = a[i], y = a[l];
          const bool up = (i & k) == 0;
          if ((x > y) == up) { a[i] = y; a[l] = x; }
        }
      }
    }
  __syncthreads();
}

// torchvision BoxCoder.decode_single, fp32, same operation order
__device__ __forceinline__ float4 decode(float4 b, float d0, float d1, float d2, float d3, const float* w) {
  const float widths = b.z - b.x, heights = b.w - b.y;
  const float cx = b.x + 0.5f * widths, cy = b.y + 0.5f * heights;
  const float dx = d0 / w[0], dy = d1 / w[1];
  const float dw = fminf(d2 / w[2], kXformClip), dh = fminf(d3 / w[3], kXformClip);
  const float pcx = dx * widths + cx, pcy = dy * heights + cy;
  const float pw = expf(dw) * widths, ph = expf(dh) * heights;
  const float hw = 0.5f * pw, hh = 0.5f * ph;
  return make_float4(pcx - hw, pcy - hh, pcx + hw, pcy + hh);
}

__device__ __forceinline__ float4 clip(float4 b, float W, float H) {
  return make_float4(fminf(fmaxf(b.x, 0.f), W), fminf(fmaxf(b.y, 0.f), H), fminf(fmaxf(b.z, 0.f), W),
                     fminf(fmaxf(b.w, 0.f), H));
}

__device__ __forceinline__ bool iou_above(float4 a, float4 b, float thr) {
  const float aa = (a.z - a.x) * (a.w - a.y), ab = (b.z - b.x) * (b.w - b.y);
  const float iw = fmaxf(0.f, fminf(a.z, b.z) - fmaxf(a.x, b.x));
  const float ih = fmaxf(0.f, fminf(a.w, b.w) - fmaxf(a.y, b.y));
  const float inter = iw * ih;
  return inter / (aa + ab - inter) > thr;   // 0/0 = NaN never suppresses (as torchvision)
}

constexpr int kRpnMax = 1024;
constexpr int kRpnSmem = kRpnMax * 32 * 4 + kRpnMax * 16 + kRpnMax * 8 + kRpnMax * 2;

__global__ void __launch_bounds__(1024) rpn_level_kernel(const RpnTask* __restrict__ tasks, int n_tasks) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint32_t* mask = reinterpret_cast<uint32_t*>(smem);                                   // [W32][K]
  float4* bx = reinterpret_cast<float4*>(smem + kRpnMax * 32 * 4);                      // [K]
  unsigned long long* sk = reinterpret_cast<unsigned long long*>(smem + kRpnMax * 32 * 4 + kRpnMax * 16);
  uint8_t* ok = smem + kRpnMax * 32 * 4 + kRpnMax * 24;
  uint8_t* keep = ok + kRpnMax;
  __shared__ int hist[256];
  __shared__ int warp_tot[33];
  __shared__ int sel_idx[kRpnMax];
  __shared__ uint32_t s_prefix;
  __shared__ int s_remaining;
  __shared__ int s_cnt, s_eq;
  __shared__ int eq_idx[kRpnMax];
  int ti = 0;
  while (ti + 1 < n_tasks && int(blockIdx.x) >= tasks[ti + 1].block_begin) ++ti;
  const RpnTask& T = tasks[ti];
  const int frame = blockIdx.x - T.block_begin, tid = threadIdx.x;
  const int HW = T.h * T.w, A = T.A, N = HW * A, K = T.K;
  const float* cls = T.cls + int64_t(frame) * HW * T.cpc;
  const float* box = T.box + int64_t(frame) * HW * T.cpb;
  auto logit = [&](int i) { return cls[int64_t(i / A) * T.cpc + i % A]; };

  // 1. radix select: the K-th largest key and how many keys equal to it are taken
  if (tid == 0) { s_prefix = 0; s_remaining = K; }
  __syncthreads();
  uint32_t msk = 0;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int i = tid; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    const uint32_t prefix = s_prefix;
    // warp-aggregated histogram: logits cluster in a few top-byte bins, so lanes with
    // the same bin add once (__match_any) instead of serialising on one smem address
    for (int base = 0; base < N; base += blockDim.x) {
      const int i = base + tid;
      const uint32_t key = i < N ? okey(logit(i)) : 0u;
      const int bin = (i < N && (key & msk) == prefix) ? int((key >> shift) & 255) : 256;
      const unsigned peers = __match_any_sync(0xffffffffu, bin);
      if (bin < 256 && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&hist[bin], __popc(peers));
    }
    __syncthreads();
    if (tid == 0) {
      int cum = 0;
      const int rem = s_remaining;
      for (int d = 255; d >= 0; --d) {
        if (cum + hist[d] >= rem) { s_prefix = prefix | (uint32_t(d) << shift); s_remaining = rem - cum; break; }
        cum += hist[d];
      }
    }
    msk |= 255u << shift;
    __syncthreads();
  }
  const uint32_t thr = s_prefix;
  const int need_eq = s_remaining;
  // 2. compaction: keys above the threshold in any order (warp-aggregated smem atomics,
  //    no block-wide scans: the survivors are sorted next), then the need_eq keys equal
  //    to the threshold with the lowest indices (ties by lower index)
  if (tid == 0) { s_cnt = 0; s_eq = 0; }
  __syncthreads();
  const int lane = tid & 31;
  for (int base = 0; base < N; base += blockDim.x) {
    const int i = base + tid;
    const uint32_t key = i < N ? okey(logit(i)) : 0u;
    const bool above = i < N && key > thr, eq = i < N && key == thr;
    const unsigned ma = __ballot_sync(0xffffffffu, above), me = __ballot_sync(0xffffffffu, eq);
    int ba = 0, be = 0;
    if (lane == 0) {
      if (ma) ba = atomicAdd(&s_cnt, __popc(ma));
      if (me) be = atomicAdd(&s_eq, __popc(me));
    }
    ba = __shfl_sync(0xffffffffu, ba, 0);
    be = __shfl_sync(0xffffffffu, be, 0);
    const unsigned lt = (1u << lane) - 1u;
    if (above) sel_idx[ba + __popc(ma & lt)] = i;
    if (eq && be + __popc(me & lt) < kRpnMax) eq_idx[be + __popc(me & lt)] = i;
  }
  __syncthreads();
  const int n_above = s_cnt, n_eq = s_eq;
  if (n_eq <= kRpnMax) {
    // rank of each equal key by index (counting); the need_eq lowest are taken
    if (tid < n_eq) {
      const int me_i = eq_idx[tid];
      int rank = 0;
      for (int j = 0; j < n_eq; ++j) rank += eq_idx[j] < me_i;
      if (rank < need_eq) sel_idx[n_above + rank] = me_i;
    }
  } else {
    // more than kRpnMax equal keys (degenerate heads): index-ordered scan of the equal ones
    int eq_seen = 0;
    for (int base = 0; base < N && eq_seen < need_eq; base += blockDim.x) {
      const int i = base + tid;
      const bool eq = i < N && okey(logit(i)) == thr;
      int eq_rank;
      const int eq_tot = scan1024(eq, warp_tot, eq_rank);
      if (eq && eq_seen + eq_rank < need_eq) sel_idx[n_above + eq_seen + eq_rank] = i;
      eq_seen += eq_tot;
    }
  }
  __syncthreads();
  // 3. order the survivors: logit descending, anchor index ascending
  sk[tid] = tid < K ? (uint64_t(~okey(logit(sel_idx[tid]))) << 32) | uint32_t(sel_idx[tid]) : ~0ull;
  bitonic_sort(sk, kRpnMax);
  // 4. decode (BoxCoder(1,1,1,1)), clip, small-box test; rows written with keep = 0
  const float one[4] = {1.f, 1.f, 1.f, 1.f};
  float* out = T.dst + int64_t(frame) * T.dst_pitch;
  if (tid < K) {
    const int i = int(sk[tid] & 0xffffffffu), pix = i / A, a = i % A;
    const float sx = float((pix % T.w) * T.stride_x), sy = float((pix / T.w) * T.stride_y);
    const float4 an = make_float4(sx + T.base[a][0], sy + T.base[a][1], sx + T.base[a][2], sy + T.base[a][3]);
    const float* d = box + int64_t(pix) * T.cpb + a * 4;
    const float4 b = clip(decode(an, d[0], d[1], d[2], d[3], one), T.img_w, T.img_h);
    bx[tid] = b;
    ok[tid] = (b.z - b.x) >= T.min_size && (b.w - b.y) >= T.min_size;
    keep[tid] = 0;
    out[tid * 6 + 0] = b.x; out[tid * 6 + 1] = b.y; out[tid * 6 + 2] = b.z; out[tid * 6 + 3] = b.w;
    out[tid * 6 + 4] = logit(i);
  }
  __syncthreads();
  // 5. suppression bitmask, stored word-major (mask[wd*K + i]): bit b of word wd of row i
  //    is set iff j = 32 wd + b > i, box j valid and IoU(i, j) > nms.  Lanes of a warp
  //    take consecutive rows i of one word, so every bx[j] read is a broadcast and the
  //    word stores are consecutive; words wholly left of the diagonal are zero.
  const int W32 = (K + 31) >> 5;
  for (int it = tid; it < K * W32; it += blockDim.x) {
    const int wd = it / K, i = it - wd * K;
    const int j0 = wd * 32;
    uint32_t bits = 0;
    if (j0 + 31 > i) {
      const float4 bi = bx[i];
      for (int b = 0; b < 32; ++b) {
        const int j = j0 + b;
        if (j > i && j < K && ok[j] && iou_above(bi, bx[j], T.nms)) bits |= 1u << b;
      }
    }
    mask[wd * K + i] = bits;
  }
  __syncthreads();
  // 6. greedy scan in score order by warp 0 (lane w holds removed-word w)
  if (tid < 32) {
    uint32_t removed = 0;
    for (int i = 0; i < K; ++i) {
      const uint32_t r = __shfl_sync(0xffffffffu, removed, i >> 5);
      if (ok[i] && !((r >> (i & 31)) & 1u)) {
        if (tid == 0) keep[i] = 1;
        if (tid < W32) removed |= mask[tid * K + i];
      }
    }
  }
  __syncthreads();
  if (tid < K) out[tid * 6 + 5] = keep[tid] ? 1.f : 0.f;
}

__global__ void __launch_bounds__(1024) rpn_merge_kernel(const RpnMergeTask* __restrict__ tasks, int n_tasks) {
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned long long* sk = reinterpret_cast<unsigned long long*>(smem);
  int ti = 0;
  while (ti + 1 < n_tasks && int(blockIdx.x) >= tasks[ti + 1].block_begin) ++ti;
  const RpnMergeTask& T = tasks[ti];
  const int frame = blockIdx.x - T.block_begin;
  int total = 0;
  for (int l = 0; l < T.n_levels; ++l) total += T.k[l];
  int P = 1;
  while (P < total) P <<= 1;
  auto row = [&](int i) {
    int l = 0;
    while (i >= T.k[l]) i -= T.k[l++];
    return T.src[l] + int64_t(frame) * T.src_pitch[l] + int64_t(i) * 6;
  };
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    unsigned long long key = ~0ull;
    if (i < total) {
      const float* r = row(i);
      if (r[5] > 0.5f) key = (uint64_t(~okey(r[4])) << 32) | uint32_t(i);
    }
    sk[i] = key;
  }
  bitonic_sort(sk, P);
  float* out = T.dst + int64_t(frame) * T.dst_pitch;
  for (int t = threadIdx.x; t < T.post_n; t += blockDim.x) {
    const unsigned long long key = t < P ? sk[t] : ~0ull;
    if (key != ~0ull) {
      const float* r = row(int(key & 0xffffffffu));
      out[t * 5 + 0] = r[0]; out[t * 5 + 1] = r[1]; out[t * 5 + 2] = r[2]; out[t * 5 + 3] = r[3];
      out[t * 5 + 4] = 1.f;
    } else {
      for (int f = 0; f < 5; ++f) out[t * 5 + f] = 0.f;
    }
  }
}

// One CTA per proposal: its 7x7 bins x C/8 channel groups loop over the CTA's threads,
// so the proposal's footprint on its pyramid level (the bins' shared bilinear taps) is
// fetched from L2 once into this SM's L1 instead of once per bin on scattered SMs.
__global__ void __launch_bounds__(256) roi_align_kernel(const RoiTask* __restrict__ tasks, int n_tasks) {
  const int64_t g = blockIdx.x;   // proposal index over all tasks
  int ti = 0;
  while (ti + 1 < n_tasks && g >= tasks[ti + 1].work_begin) ++ti;
  const RoiTask& T = tasks[ti];
  const int64_t roi = g - T.work_begin;
  const int nv = T.C >> 3;
  const int per = T.out * T.out * nv;
  for (int l0 = int(threadIdx.x); l0 < per; l0 += int(blockDim.x)) {
    int l = l0;
    const int v = l % nv;
    l /= nv;
    const int pw = l % T.out;
    const int ph = l / T.out;
    const int frame = int(roi / T.R), r = int(roi % T.R);
    const float* p = T.props + int64_t(frame) * T.props_pitch + int64_t(r) * 5;
    const float x1 = p[0], y1 = p[1], x2 = p[2], y2 = p[3];
    // LevelMapper: floor(lvl0 + log2(sqrt(area) / s0) + 1e-6), clamped (area 0 -> k_min)
    const float area = (x2 - x1) * (y2 - y1);
    float lv = floorf(T.canon_level + log2f(sqrtf(area) / T.canon_scale) + 1e-6f);
    lv = fminf(fmaxf(lv, float(T.k_min)), float(T.k_min + T.n_maps - 1));
    const int li = int(lv) - T.k_min;
    const int H = T.mh[li], W = T.mw[li];
    const float sc = T.scale[li];
    const float sw = x1 * sc, sh = y1 * sc;
    const float rw = fmaxf(x2 * sc - sw, 1.f), rh = fmaxf(y2 * sc - sh, 1.f);
    const float bw = rw / float(T.out), bh = rh / float(T.out);
    const __nv_bfloat16* fm = static_cast<const __nv_bfloat16*>(T.map[li]) + int64_t(frame) * H * W * T.cp + v * 8;
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    auto tap = [&](int yy, int xx, float wgt) {
      const uint4 q = *reinterpret_cast<const uint4*>(fm + (int64_t(yy) * W + xx) * T.cp);
      const uint32_t u[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        acc[2 * k] += wgt * __uint_as_float(u[k] << 16);
        acc[2 * k + 1] += wgt * __uint_as_float(u[k] & 0xFFFF0000u);
      }
    };
    if (T.sampling == 2) {
      // torchvision's default: the 16 taps' offsets and weights first, then 16 independent
      // 16-byte loads in flight (a sample outside the map contributes weight 0)
      int64_t off[16];
      float wt[16];
#pragma unroll
      for (int iy = 0; iy < 2; ++iy)
#pragma unroll
        for (int ix = 0; ix < 2; ++ix) {
          const int t = 4 * (2 * iy + ix);
          const float y = sh + float(ph) * bh + (float(iy) + .5f) * bh / 2.f;
          const float x = sw + float(pw) * bw + (float(ix) + .5f) * bw / 2.f;
          const bool in = !(y < -1.f || y > float(H) || x < -1.f || x > float(W));
          float yy = fmaxf(y, 0.f), xx = fmaxf(x, 0.f);
          int y0 = in ? int(yy) : 0, x0 = in ? int(xx) : 0, y1i, x1i;
          if (y0 >= H - 1) { y0 = y1i = H - 1; yy = float(y0); } else { y1i = y0 + 1; }
          if (x0 >= W - 1) { x0 = x1i = W - 1; xx = float(x0); } else { x1i = x0 + 1; }
          const float ly = yy - float(y0), lx = xx - float(x0), hy = 1.f - ly, hx = 1.f - lx;
          off[t + 0] = (int64_t(y0) * W + x0) * T.cp;  wt[t + 0] = in ? hy * hx : 0.f;
          off[t + 1] = (int64_t(y0) * W + x1i) * T.cp; wt[t + 1] = in ? hy * lx : 0.f;
          off[t + 2] = (int64_t(y1i) * W + x0) * T.cp; wt[t + 2] = in ? ly * hx : 0.f;
          off[t + 3] = (int64_t(y1i) * W + x1i) * T.cp; wt[t + 3] = in ? ly * lx : 0.f;
        }
      uint4 q[16];
#pragma unroll
      for (int t = 0; t < 16; ++t) q[t] = __ldg(reinterpret_cast<const uint4*>(fm + off[t]));
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        const uint32_t u[4] = {q[t].x, q[t].y, q[t].z, q[t].w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          acc[2 * k] += wt[t] * __uint_as_float(u[k] << 16);
          acc[2 * k + 1] += wt[t] * __uint_as_float(u[k] & 0xFFFF0000u);
        }
      }
    } else {
      for (int iy = 0; iy < T.sampling; ++iy) {
        float y = sh + float(ph) * bh + (float(iy) + .5f) * bh / float(T.sampling);
        for (int ix = 0; ix < T.sampling; ++ix) {
          float x = sw + float(pw) * bw + (float(ix) + .5f) * bw / float(T.sampling);
          if (y < -1.f || y > float(H) || x < -1.f || x > float(W)) continue;
          float yy = fmaxf(y, 0.f), xx = fmaxf(x, 0.f);
          int y0 = int(yy), x0 = int(xx), y1i, x1i;
          if (y0 >= H - 1) { y0 = y1i = H - 1; yy = float(y0); } else { y1i = y0 + 1; }
          if (x0 >= W - 1) { x0 = x1i = W - 1; xx = float(x0); } else { x1i = x0 + 1; }
          const float ly = yy - float(y0), lx = xx - float(x0), hy = 1.f - ly, hx = 1.f - lx;
          tap(y0, x0, hy * hx);
          tap(y0, x1i, hy * lx);
          tap(y1i, x0, ly * hx);
          tap(y1i, x1i, ly * lx);
        }
      }
    }
    const float inv = 1.f / float(T.sampling * T.sampling);
    uint4 o;
    uint32_t* ou = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      __nv_bfloat162 h2 = __floats2bfloat162_rn(acc[2 * k] * inv, acc[2 * k + 1] * inv);
      ou[k] = *reinterpret_cast<uint32_t*>(&h2);
    }
    *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(T.dst) +
                              ((roi * T.out + ph) * T.out + pw) * T.cpd + v * 8) = o;
  }
}

__global__ void box_post_kernel(const BoxPostTask* __restrict__ tasks, int n_tasks, int64_t total_warps) {
  const int lane = threadIdx.x & 31;
  for (int64_t wi = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5; wi < total_warps;
       wi += (int64_t(gridDim.x) * blockDim.x) >> 5) {
    int ti = 0;
    while (ti + 1 < n_tasks && wi >= tasks[ti + 1].work_begin) ++ti;
    const BoxPostTask& T = tasks[ti];
    const int64_t roi = wi - T.work_begin;
    const int frame = int(roi / T.R), r = int(roi % T.R);
    const float* lg = T.cls + roi * T.cpc;
    float mx = -INFINITY;
    for (int j = lane; j < T.classes; j += 32) mx = fmaxf(mx, lg[j]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float sum = 0.f;
    for (int j = lane; j < T.classes; j += 32) sum += expf(lg[j] - mx);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    const float* p = T.props + int64_t(frame) * T.props_pitch + int64_t(r) * 5;
    const float4 pb = make_float4(p[0], p[1], p[2], p[3]);
    const bool valid = p[4] > 0.5f;
    float* out = T.dst + int64_t(frame) * T.dst_pitch + int64_t(r) * (T.classes - 1) * 6;
    const float* d = T.box + roi * T.cpb;
    for (int j = 1 + lane; j < T.classes; j += 32) {
      const float4 b = clip(decode(pb, d[4 * j], d[4 * j + 1], d[4 * j + 2], d[4 * j + 3], T.wts), T.img_w, T.img_h);
      float* o = out + (j - 1) * 6;
      o[0] = b.x; o[1] = b.y; o[2] = b.z; o[3] = b.w;
      o[4] = valid ? expf(lg[j] - mx) / sum : -1.f;
      o[5] = float(j);
    }
  }
}

int grid_for(int64_t work, int threads) {
  int64_t g = (work + threads - 1) / threads;
  const int64_t cap = int64_t(device_sm_count()) * 16;
  if (g > cap) g = cap;
  return int(g < 1 ? 1 : g);
}

}  // namespace

int launch_rpn_level(const RpnTask* tasks, int n, int blocks, void* stream) {
  cudaError_t e = cudaFuncSetAttribute(rpn_level_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kRpnSmem);
  if (e != cudaSuccess) return int(e);
  rpn_level_kernel<<<blocks, 1024, kRpnSmem, static_cast<cudaStream_t>(stream)>>>(tasks, n);
  return int(cudaGetLastError());
}

int launch_rpn_merge(const RpnMergeTask* tasks, int n, int blocks, void* stream) {
  const int smem = 8192 * 8;
  cudaError_t e = cudaFuncSetAttribute(rpn_merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return int(e);
  rpn_merge_kernel<<<blocks, 1024, smem, static_cast<cudaStream_t>(stream)>>>(tasks, n);
  return int(cudaGetLastError());
}

int launch_roi_align(const RoiTask* tasks, int n, int64_t total_rois, void* stream) {
  roi_align_kernel<<<unsigned(total_rois), 256, 0, static_cast<cudaStream_t>(stream)>>>(tasks, n);
  return int(cudaGetLastError());
}

// Final detections: greedy batched NMS over one frame's
// score-ranked candidates, one 1024-thread CTA per frame, one candidate per thread
// (box, label and a removed flag in registers).  Each round takes the first candidate
// not yet removed (a block-wide min over warp ballots), keeps it, and every later
// candidate of the same label tests its IoU against it in parallel -- so a frame costs
// one round per KEPT row (<= max_det), not per visited candidate.  Rows with index -1
// or a negative score (dropped candidates) rank last and start removed.
constexpr int kNmsMax = 1024;

__global__ void __launch_bounds__(1024) det_nms_kernel(const NmsTask* __restrict__ tasks, int n_tasks) {
  __shared__ int s_first[32];
  __shared__ float4 s_box;
  __shared__ float s_lab;
  __shared__ int kept_idx[kNmsMax];
  int ti = 0;
  while (ti + 1 < n_tasks && int(blockIdx.x) >= tasks[ti + 1].block_begin) ++ti;
  const NmsTask& T = tasks[ti];
  const int f = int(blockIdx.x) - T.block_begin;
  const int tid = int(threadIdx.x), lane = tid & 31, wid = tid >> 5;
  const float* src = T.src + int64_t(f) * T.src_pitch;
  float* dst = T.dst + int64_t(f) * T.dst_pitch;
  const int K = min(T.k_in, kNmsMax);
  float4 b = make_float4(0.f, 0.f, 0.f, 0.f);
  float lab = 0.f, score = -1.f;
  bool removed = true;
  if (tid < K) {
    const float* r = src + int64_t(tid) * 7;
    b = make_float4(r[1], r[2], r[3], r[4]);
    score = r[5];
    lab = r[6];
    removed = r[0] < 0.f || score < 0.f;
  }
  int n_kept = 0, cur = 0;
  while (n_kept < T.max_det) {
    // the first candidate >= cur not removed: per-warp ballot, then the min over warps
    const unsigned live = __ballot_sync(0xffffffffu, !removed && tid >= cur);
    if (lane == 0) s_first[wid] = live ? wid * 32 + __ffs(live) - 1 : 0x7fffffff;
    __syncthreads();
    int first = s_first[lane];
    first = min(first, __shfl_xor_sync(0xffffffffu, first, 16));
    first = min(first, __shfl_xor_sync(0xffffffffu, first, 8));
    first = min(first, __shfl_xor_sync(0xffffffffu, first, 4));
    first = min(first, __shfl_xor_sync(0xffffffffu, first, 2));
    first = min(first, __shfl_xor_sync(0xffffffffu, first, 1));
    if (first == 0x7fffffff) break;                 // block-uniform
    if (tid == first) { s_box = b; s_lab = lab; kept_idx[n_kept] = tid; }
    __syncthreads();
    const float4 kb = s_box;
    if (!removed && tid > first && lab == s_lab && iou_above(kb, b, T.iou)) removed = true;
    ++n_kept;
    cur = first + 1;
    __syncthreads();                                // s_first / s_box reused next round
  }
  for (int e = tid; e < T.max_det * 6; e += blockDim.x) {
    const int q = e / 6, c = e - q * 6;
    dst[e] = q < n_kept ? src[int64_t(kept_idx[q]) * 7 + 1 + c] : (c == 4 ? -1.f : 0.f);
  }
}

int launch_det_nms(const NmsTask* tasks, int n, int blocks, void* stream) {
  det_nms_kernel<<<blocks, 1024, 0, static_cast<cudaStream_t>(stream)>>>(tasks, n);
  return int(cudaGetLastError());
}

int launch_box_post(const BoxPostTask* tasks, int n, int64_t total_warps, void* stream) {
  box_post_kernel<<<grid_for(total_warps * 32, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(tasks, n,
                                                                                                   total_warps);
  return int(cudaGetLastError());
}

}  // namespace gemel
