// Memory-bound kernels: frame preprocessing, max /
// adaptive-average pooling and standalone residual add (a9).  Grouped: one
// launch covers every task of a scheduler wave through a task table; each
// thread handles one 16-byte vector (8 bf16 channels) of one output pixel.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "gemm.h"
#include "memops.h"
#include "smem_attr.cuh"
#include "select.cuh"

namespace gemel {
namespace {

__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ float lo(uint32_t u) { return __uint_as_float(u << 16); }
__device__ __forceinline__ float hi(uint32_t u) { return __uint_as_float(u & 0xFFFF0000u); }

// task of work item i, searched forward from k (a grid-stride loop visits increasing i,
// so the search is amortised O(1) instead of a scan of the task table per item)
template <typename T>
__device__ __forceinline__ int find_task(const T* t, int n, int64_t i, int k = 0) {
  while (k + 1 < n && i >= t[k + 1].work_begin) ++k;
  return k;
}

__global__ void preprocess_kernel(const PreTask* __restrict__ tasks, int n_tasks, int64_t total) {
  // ImageNet normalisation (x/255 - mean) / std, written as x * a + b in fp32.
  const float A[3] = {1.f / (255.f * 0.229f), 1.f / (255.f * 0.224f), 1.f / (255.f * 0.225f)};
  const float Bc[3] = {-0.485f / 0.229f, -0.456f / 0.224f, -0.406f / 0.225f};
  int ti = 0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    ti = find_task(tasks, n_tasks, i, ti);
    const PreTask& T = tasks[ti];
    const int64_t p = i - T.work_begin;
    if (T.mode == 0) {
      const uint8_t* s = T.src + 3 * p;
      const float r = fmaf(float(s[0]), A[0], Bc[0]), g = fmaf(float(s[1]), A[1], Bc[1]),
                  b = fmaf(float(s[2]), A[2], Bc[2]);
      reinterpret_cast<uint4*>(T.dst)[p] = make_uint4(pack2(r, g), pack2(b, 0.f), 0u, 0u);
    } else {
      // im2col row m = (img, oh, ow), columns k = (r * kw + s) * 3 + c; zero padding
      const int kv = T.Kp / 8;
      const int g8 = int(p % kv);
      const int64_t m = p / kv;
      const int ow = int(m % T.wo);
      const int64_t t2 = m / T.wo;
      const int oh = int(t2 % T.ho);
      const int64_t img = t2 / T.ho;
      float v[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int k = g8 * 8 + e;
        float x = 0.f;
        if (k < T.K) {
          const int tap = k / 3, c = k - tap * 3;
          const int r = tap / T.kw, s = tap - r * T.kw;
          const int ih = oh * T.sh - T.ph + r * T.dh, iw = ow * T.sw - T.pw + s * T.dw;
          if (ih >= 0 && ih < T.h && iw >= 0 && iw < T.w)
            x = fmaf(float(T.src[((img * T.h + ih) * T.w + iw) * 3 + c]), A[c], Bc[c]);
        }
        v[e] = x;
      }
      reinterpret_cast<uint4*>(T.dst)[p] =
          make_uint4(pack2(v[0], v[1]), pack2(v[2], v[3]), pack2(v[4], v[5]), pack2(v[6], v[7]));
    }
  }
}

// im2col rows of the first conv, one block per (image, output row): the
// receptive-field input rows are normalised once into shared memory, then every
// (output pixel, 8-column group) of the row is assembled from smem and written
// as one 16-byte vector.  Column k = (r * kw + s) * 3 + c; zero padding.
__global__ void ingest_cols_kernel(const PreTask* __restrict__ tasks, int n_tasks) {
  extern __shared__ float xs[];   // [Kp] column offsets (as int), then [kh_eff][wspan][3]
  const float A[3] = {1.f / (255.f * 0.229f), 1.f / (255.f * 0.224f), 1.f / (255.f * 0.225f)};
  const float Bc[3] = {-0.485f / 0.229f, -0.456f / 0.224f, -0.406f / 0.225f};
  const PreTask& T = tasks[find_task(tasks, n_tasks, int64_t(blockIdx.x))];
  const int64_t row = int64_t(blockIdx.x) - T.work_begin;   // (img, oh)
  const int oh = int(row % T.ho);
  const int64_t img = row / T.ho;
  const int kh_eff = (T.kh - 1) * T.dh + 1;
  const int wspan = (T.wo - 1) * T.sw + (T.kw - 1) * T.dw + 1;
  const int ih0 = oh * T.sh - T.ph, iw0 = -T.pw;
  const uint8_t* src = T.src + img * int64_t(T.h) * T.w * 3;
  int* koff = reinterpret_cast<int*>(xs);
  float* xt = xs + T.Kp;
  for (int k = threadIdx.x; k < T.Kp; k += blockDim.x) {   // column -> smem offset (-1: zero pad)
    int o = -1;
    if (k < T.K) {
      const int tap = k / 3, c = k - tap * 3, r = tap / T.kw, s = tap - r * T.kw;
      o = ((r * T.dh) * wspan + s * T.dw) * 3 + c;
    }
    koff[k] = o;
  }
  for (int i = threadIdx.x; i < kh_eff * wspan * 3; i += blockDim.x) {
    const int c = i % 3, t = i / 3, x = t % wspan, y = t / wspan;
    const int ih = ih0 + y, iw = iw0 + x;
    float v = 0.f;
    if (ih >= 0 && ih < T.h && iw >= 0 && iw < T.w) v = fmaf(float(src[(int64_t(ih) * T.w + iw) * 3 + c]), A[c], Bc[c]);
    xt[i] = v;
  }
  __syncthreads();
  const int kv = T.Kp / 8;
  const int step = T.sw * 3;
  uint4* dst = reinterpret_cast<uint4*>(T.dst) + row * int64_t(T.wo) * kv;
  // each thread keeps one 8-column group g8 (its 8 smem offsets in registers) and
  // walks output pixels ow = tid / kv, + per, ...: 8 smem reads per 16-byte vector
  const int per = int(blockDim.x) / kv;        // pixels covered per sweep of the block
  if (int(threadIdx.x) < per * kv) {
    const int g8 = int(threadIdx.x) % kv;
    int o[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) o[e] = koff[g8 * 8 + e];
    for (int ow = int(threadIdx.x) / kv; ow < T.wo; ow += per) {
      const float* base = xt + ow * step;
      float v[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) v[e] = o[e] >= 0 ? base[o[e]] : 0.f;
      dst[int64_t(ow) * kv + g8] = make_uint4(pack2(v[0], v[1]), pack2(v[2], v[3]), pack2(v[4], v[5]), pack2(v[6], v[7]));
    }
  }
}

__global__ void pool_kernel(const PoolTask* __restrict__ tasks, int n_tasks, int64_t total) {
  int ti = 0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    ti = find_task(tasks, n_tasks, i, ti);
    const PoolTask& T = tasks[ti];
    uint32_t r = uint32_t(i - T.work_begin);   // task-local work < 2^31: 32-bit index arithmetic
    const uint32_t cv = uint32_t(T.cp) / 8u;
    const int v = int(r % cv);
    r /= cv;
    const int ow = int(r % uint32_t(T.wo));
    r /= uint32_t(T.wo);
    const int oh = int(r % uint32_t(T.ho));
    const int n = int(r / uint32_t(T.ho));
    const uint4* src = reinterpret_cast<const uint4*>(T.src);
    float acc[8];
    int h0, h1, w0, w1;
    if (T.kind == 0 && T.kh * T.kw <= 9) {
      // the common windows (3x3, 2x2, 1x1): every tap's 16-byte load issued before the
      // max, out-of-window taps predicated off (-inf), instead of a branchy load chain
      uint4 q[9];
      bool ok[9];
#pragma unroll
      for (int t = 0; t < 9; ++t) {
        const int a = t / 3, b = t - 3 * (t / 3);
        const int ih = oh * T.sh - T.ph + a * T.dh, iw = ow * T.sw - T.pw + b * T.dw;
        ok[t] = a < T.kh && b < T.kw && ih >= 0 && ih < T.h && iw >= 0 && iw < T.w;
        q[t] = ok[t] ? __ldg(src + ((int64_t(n) * T.h + ih) * T.w + iw) * cv + v) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = -INFINITY;
#pragma unroll
      for (int t = 0; t < 9; ++t) {
        if (!ok[t]) continue;
        const uint4 x = q[t];
        acc[0] = fmaxf(acc[0], lo(x.x)); acc[1] = fmaxf(acc[1], hi(x.x));
        acc[2] = fmaxf(acc[2], lo(x.y)); acc[3] = fmaxf(acc[3], hi(x.y));
        acc[4] = fmaxf(acc[4], lo(x.z)); acc[5] = fmaxf(acc[5], hi(x.z));
        acc[6] = fmaxf(acc[6], lo(x.w)); acc[7] = fmaxf(acc[7], hi(x.w));
      }
    } else if (T.kind == 0) {
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = -INFINITY;
      for (int a = 0; a < T.kh; ++a) {
        const int ih = oh * T.sh - T.ph + a * T.dh;
        if (ih < 0 || ih >= T.h) continue;
        for (int b = 0; b < T.kw; ++b) {
          const int iw = ow * T.sw - T.pw + b * T.dw;
          if (iw < 0 || iw >= T.w) continue;
          const uint4 x = src[((int64_t(n) * T.h + ih) * T.w + iw) * cv + v];
          acc[0] = fmaxf(acc[0], lo(x.x)); acc[1] = fmaxf(acc[1], hi(x.x));
          acc[2] = fmaxf(acc[2], lo(x.y)); acc[3] = fmaxf(acc[3], hi(x.y));
          acc[4] = fmaxf(acc[4], lo(x.z)); acc[5] = fmaxf(acc[5], hi(x.z));
          acc[6] = fmaxf(acc[6], lo(x.w)); acc[7] = fmaxf(acc[7], hi(x.w));
        }
      }
    } else {
      // adaptive average: bin [floor(i*H/oh), ceil((i+1)*H/oh))
      h0 = (oh * T.h) / T.ho; h1 = ((oh + 1) * T.h + T.ho - 1) / T.ho;
      w0 = (ow * T.w) / T.wo; w1 = ((ow + 1) * T.w + T.wo - 1) / T.wo;
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = 0.f;
      for (int ih = h0; ih < h1; ++ih)
        for (int iw = w0; iw < w1; ++iw) {
          const uint4 x = src[((int64_t(n) * T.h + ih) * T.w + iw) * cv + v];
          acc[0] += lo(x.x); acc[1] += hi(x.x); acc[2] += lo(x.y); acc[3] += hi(x.y);
          acc[4] += lo(x.z); acc[5] += hi(x.z); acc[6] += lo(x.w); acc[7] += hi(x.w);
        }
      const float inv = 1.f / float((h1 - h0) * (w1 - w0));
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] *= inv;
    }
    reinterpret_cast<uint4*>(T.dst)[((int64_t(n) * T.ho + oh) * T.wo + ow) * cv + v] =
        make_uint4(pack2(acc[0], acc[1]), pack2(acc[2], acc[3]), pack2(acc[4], acc[5]), pack2(acc[6], acc[7]));
  }
}

__device__ __forceinline__ float actf(float y, int act, float slope) {
  if (act == ACT_RELU) return fmaxf(y, 0.f);
  if (act == ACT_LEAKY) return y >= 0.f ? y : y * slope;
  return y;
}

__global__ void add_kernel(const AddTask* __restrict__ tasks, int n_tasks, int64_t total) {
  int ti = 0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    ti = find_task(tasks, n_tasks, i, ti);
    const AddTask& T = tasks[ti];
    const int64_t r = i - T.work_begin;
    const uint4 a = reinterpret_cast<const uint4*>(T.a)[r];
    const uint4 b = reinterpret_cast<const uint4*>(T.b)[r];
    uint4 o;
    o.x = pack2(actf(lo(a.x) + lo(b.x), T.act, T.slope), actf(hi(a.x) + hi(b.x), T.act, T.slope));
    o.y = pack2(actf(lo(a.y) + lo(b.y), T.act, T.slope), actf(hi(a.y) + hi(b.y), T.act, T.slope));
    o.z = pack2(actf(lo(a.z) + lo(b.z), T.act, T.slope), actf(hi(a.z) + hi(b.z), T.act, T.slope));
    o.w = pack2(actf(lo(a.w) + lo(b.w), T.act, T.slope), actf(hi(a.w) + hi(b.w), T.act, T.slope));
    reinterpret_cast<uint4*>(T.out)[r] = o;
  }
}

// Concat piece: 8 channels (16 B) per thread, read from the nearest-upsampled
// source pixel and written at the piece's channel window of the concat slab.
// YOLO decode: one output element per thread, (anchor, cy, cx, field) order, so
// consecutive threads read consecutive channels of one pixel (darknet yolo
// layer; oracle/ops.py yolo_decode).
__global__ void misc_kernel(const MiscTask* __restrict__ tasks, int n_tasks, int64_t total) {
  // every task's work_begin / work is a multiple of 32, so a warp never straddles tasks
  int ti = 0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    ti = find_task(tasks, n_tasks, i, ti);
    const MiscTask& T = tasks[ti];
    const int64_t r64 = i - T.work_begin;
    if (r64 >= T.work) continue;   // padding to the next multiple of 32
    uint32_t r = uint32_t(r64);    // task-local work < 2^31: 32-bit index arithmetic
    if (T.kind == 0) {
      const uint32_t cv = uint32_t(T.c) / 8u;
      const int v = int(r % cv);
      r /= cv;
      const int x = int(r % uint32_t(T.w));
      r /= uint32_t(T.w);
      const int y = int(r % uint32_t(T.h));
      const int n = int(r / uint32_t(T.h));
      const int hs = T.h / T.scale, ws = T.w / T.scale;
      const uint4 val = reinterpret_cast<const uint4*>(T.src)[((int64_t(n) * hs + y / T.scale) * ws + x / T.scale) *
                                                                  (T.cps / 8) + v];
      reinterpret_cast<uint4*>(T.dst)[((int64_t(n) * T.h + y) * T.w + x) * (T.cpd / 8) + T.c_off / 8 + v] = val;
    } else if (T.kind == 4) {   // detection candidates (N2): a thread per row -> (x1, y1, x2, y2, score, label)
      // (a warp per YOLO/SSD row, lanes over the classes, measured 3x slower: 127 vs 47 us)
      const int64_t n = int64_t(r) / T.rows, row = int64_t(r) - n * T.rows;
      const float* x = reinterpret_cast<const float*>(T.src) + n * T.cps + row * T.c;
      float* o = reinterpret_cast<float*>(T.dst) + n * T.cpd + row * 6;
      float b0, b1, b2, b3, sc, lab;
      if (T.det_fmt == 0) {            // Fast R-CNN box_post rows, as they are
        b0 = x[0]; b1 = x[1]; b2 = x[2]; b3 = x[3]; sc = x[4]; lab = x[5];
      } else if (T.det_fmt == 1) {     // YOLO: corners, obj * best class, first argmax
        float best = x[5];
        int k = 0;
        for (int j = 1; j < T.c - 5; ++j)
          if (x[5 + j] > best) { best = x[5 + j]; k = j; }
        b0 = x[0] - x[2] / 2.f; b1 = x[1] - x[3] / 2.f; b2 = x[0] + x[2] / 2.f; b3 = x[1] + x[3] / 2.f;
        sc = x[4] * best; lab = float(k);
      } else {                         // SSD: best foreground class (>= 1), first argmax
        float best = x[6];
        int k = 1;
        for (int j = 2; j < T.c - 5; ++j)
          if (x[5 + j] > best) { best = x[5 + j]; k = j; }
        b0 = x[0]; b1 = x[1]; b2 = x[2]; b3 = x[3]; sc = best; lab = float(k);
      }
      const bool keep = sc > T.det_thresh && (b2 - b0) >= T.eps && (b3 - b1) >= T.eps;
      o[0] = b0; o[1] = b1; o[2] = b2; o[3] = b3; o[4] = keep ? sc : -1.f; o[5] = lab;
    } else if (T.kind == 2) {   // L2Norm: warp per pixel (work_begin and work are multiples of 32)
      const int lane = int(r & 31u);
      const int64_t pix = r >> 5;
      if (pix >= int64_t(T.n) * T.h * T.w) continue;   // padding lanes (whole warp)
      const uint4* src = reinterpret_cast<const uint4*>(T.src) + pix * (T.cps / 8);
      uint4* dst = reinterpret_cast<uint4*>(T.dst) + pix * (T.cpd / 8);
      const int cv = T.c / 8;
      float ss = 0.f;
      for (int v = lane; v < cv; v += 32) {
        const uint4 x = src[v];
        const float a[8] = {lo(x.x), hi(x.x), lo(x.y), hi(x.y), lo(x.z), hi(x.z), lo(x.w), hi(x.w)};
#pragma unroll
        for (int j = 0; j < 8; ++j) ss = fmaf(a[j], a[j], ss);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      const float inv = 1.f / fmaxf(sqrtf(ss), T.eps);
      for (int v = lane; v < cv; v += 32) {
        const uint4 x = src[v];
        const float* sc = T.vec + v * 8;
        uint4 y;
        y.x = pack2(lo(x.x) * inv * sc[0], hi(x.x) * inv * sc[1]);
        y.y = pack2(lo(x.y) * inv * sc[2], hi(x.y) * inv * sc[3]);
        y.z = pack2(lo(x.z) * inv * sc[4], hi(x.z) * inv * sc[5]);
        y.w = pack2(lo(x.w) * inv * sc[6], hi(x.w) * inv * sc[7]);
        dst[v] = y;
      }
    } else if (T.kind == 3) {   // SSD: a warp per default box, (n, cy, cx, a) order; lanes over classes
      const int lane = int(r & 31u);
      const uint32_t bx = r >> 5;
      if (bx >= uint32_t(T.n) * T.h * T.w * T.A) continue;   // padding (whole warp)
      const int a = int(bx % uint32_t(T.A));
      uint32_t q = bx / uint32_t(T.A);
      const int x = int(q % uint32_t(T.w));
      q /= uint32_t(T.w);
      const int y = int(q % uint32_t(T.h));
      const int n = int(q / uint32_t(T.h));
      const int64_t pix = (int64_t(n) * T.h + y) * T.w + x;
      const float* lc = reinterpret_cast<const float*>(T.src) + pix * T.cps + a * 4;
      const float* cf = reinterpret_cast<const float*>(T.src2) + pix * T.cps2 + a * T.c;
      float* o = reinterpret_cast<float*>(T.dst) + int64_t(n) * T.dst_pitch + T.dst_off +
                 (int64_t(bx) - int64_t(n) * T.h * T.w * T.A) * (5 + T.c);
      if (lane < 4) {
        // default box (xyxy in pixels, as torchvision builds it), then BoxCoder.decode_single
        const float acx = (float(x) + 0.5f) * T.stride_w, acy = (float(y) + 0.5f) * T.stride_h;
        const float aw = T.anchors[2 * a] * T.img_w, ah = T.anchors[2 * a + 1] * T.img_h;
        const float x1 = acx - 0.5f * aw, x2 = acx + 0.5f * aw, y1 = acy - 0.5f * ah, y2 = acy + 0.5f * ah;
        const float wd = x2 - x1, ht = y2 - y1, cx = x1 + 0.5f * wd, cy = y1 + 0.5f * ht;
        const float clampv = 4.135166556742356f;   // log(1000 / 16)
        const float dx = lc[0] / T.wts[0], dy = lc[1] / T.wts[1];
        const float dw = fminf(lc[2] / T.wts[2], clampv), dh = fminf(lc[3] / T.wts[3], clampv);
        const float pcx = dx * wd + cx, pcy = dy * ht + cy, pw = expf(dw) * wd, ph = expf(dh) * ht;
        const float v = lane == 0 ? pcx - 0.5f * pw : lane == 1 ? pcy - 0.5f * ph : lane == 2 ? pcx + 0.5f * pw
                                                                                        : pcy + 0.5f * ph;
        o[lane] = fminf(fmaxf(v, 0.f), (lane & 1) ? T.img_h : T.img_w);
      }
      float m = -INFINITY;
      for (int k = lane; k < T.c; k += 32) m = fmaxf(m, cf[k]);
#pragma unroll
      for (int s2 = 16; s2 > 0; s2 >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, s2));
      float sum = 0.f;
      for (int k = lane; k < T.c; k += 32) sum += expf(cf[k] - m);
#pragma unroll
      for (int s2 = 16; s2 > 0; s2 >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, s2);
      const float inv = 1.f / sum;
      float best = 0.f;
      for (int k = lane; k < T.c; k += 32) {
        const float pk = expf(cf[k] - m) * inv;
        o[5 + k] = pk;
        if (k > 0) best = fmaxf(best, pk);
      }
#pragma unroll
      for (int s2 = 16; s2 > 0; s2 >>= 1) best = fmaxf(best, __shfl_xor_sync(0xffffffffu, best, s2));
      if (lane == 0) o[4] = best;
    } else {   // YOLO decode: a half-warp per box (n, a, y, x), lanes over its fields (coalesced rows)
      const int lane = int(r & 15u);
      const uint32_t bx = r >> 4, per = uint32_t(T.A) * T.h * T.w;   // boxes per frame of this head
      const int n = int(bx / per);
      const uint32_t qb = bx - uint32_t(n) * per;                     // box index within the frame
      uint32_t q = qb;
      const int x = int(q % uint32_t(T.w));
      q /= uint32_t(T.w);
      const int y = int(q % uint32_t(T.h));
      const int a = int(q / uint32_t(T.h));
      const float* srow = reinterpret_cast<const float*>(T.src) + ((int64_t(n) * T.h + y) * T.w + x) * T.cps + a * T.c;
      float* drow = reinterpret_cast<float*>(T.dst) + int64_t(n) * T.dst_pitch + T.dst_off + int64_t(qb) * T.c;
      // every load of the box first (one round trip, up to 8 per lane), then the math and stores
      float tv[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) tv[i] = lane + 16 * i < T.c ? srow[lane + 16 * i] : 0.f;
      auto field = [&](int f, float t) {
        if (f == 0) return (1.f / (1.f + __expf(-t)) + float(x)) * T.stride_w;
        if (f == 1) return (1.f / (1.f + __expf(-t)) + float(y)) * T.stride_h;
        if (f == 2) return T.anchors[2 * a] * expf(t);
        if (f == 3) return T.anchors[2 * a + 1] * expf(t);
        return 1.f / (1.f + expf(-t));
      };
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (lane + 16 * i < T.c) drow[lane + 16 * i] = field(lane + 16 * i, tv[i]);
      for (int f = lane + 128; f < T.c; f += 16) drow[f] = field(f, srow[f]);   // more than 128 fields
    }
  }
}

// Top-k rows per frame: a cluster of sel::SEL_CS CTAs per frame
// (select.cuh: cluster-wide radix select over DSMEM, index-ordered ties, the leader's
// bitonic sort); the leader then writes the k rows in rank order (index, fields...),
// rows past the frame's row count as (-1, 0...).  Integer selection: bit-exact against
// the oracle.
__global__ void __cluster_dims__(sel::SEL_CS, 1, 1) __launch_bounds__(sel::SEL_THREADS)
    topk_kernel(const TopkTask* __restrict__ tasks, int n_tasks) {
  extern __shared__ uint32_t keys[];
  __shared__ sel::Shared S;
  const int fb = int(blockIdx.x) / sel::SEL_CS;   // frame over all tasks
  int ti = 0;
  while (ti + 1 < n_tasks && fb >= tasks[ti + 1].block_begin) ++ti;
  const TopkTask& T = tasks[ti];
  const int frame = fb - T.block_begin;
  const float* row = T.src + frame * T.src_pitch;
  float* out = T.dst + frame * T.dst_pitch;
  const int F = T.fields, sc = T.score;
  const int kt = sel::cluster_select([&](int i) { return sel::order_key(row[int64_t(i) * F + sc]); }, T.rows, T.k,
                                     S, keys);
  if (kt < 0) return;
  const int Fo = F + 1;
  for (int e = threadIdx.x; e < T.k * Fo; e += sel::SEL_THREADS) {
    const int t = e / Fo, f = e - t * Fo;
    float v;
    if (t < kt) {
      const int me = int(S.out[t] & 0xffffffffu);
      v = f == 0 ? float(me) : row[int64_t(me) * F + f - 1];
    } else {
      v = f == 0 ? -1.f : 0.f;
    }
    out[int64_t(t) * Fo + f] = v;
  }
}

int grid_for(int64_t work, int threads) {
  int64_t g = (work + threads - 1) / threads;
  const int64_t cap = int64_t(device_sm_count()) * 16;   // 16 resident 256-thread CTAs per SM, grid-stride beyond
  if (g > cap) g = cap;
  return int(g < 1 ? 1 : g);
}

}  // namespace

int device_sm_count() {
  static const int n = [] {
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      return 148;
    return sms > 0 ? sms : 148;
  }();
  return n;
}

int launch_preprocess(const PreTask* tasks, int n, int64_t total, void* stream) {
  preprocess_kernel<<<grid_for(total, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(tasks, n, total);
  return int(cudaGetLastError());
}
int launch_ingest_cols(const PreTask* tasks, int n, int64_t blocks, int smem_bytes, void* stream) {
  if (smem_bytes > 48 * 1024) {
    cudaError_t e = allow_max_dyn_smem(ingest_cols_kernel);
    if (e != cudaSuccess) return int(e);
  }
  ingest_cols_kernel<<<unsigned(blocks), 256, smem_bytes, static_cast<cudaStream_t>(stream)>>>(tasks, n);
  return int(cudaGetLastError());
}
int launch_pool(const PoolTask* tasks, int n, int64_t total, void* stream) {
  pool_kernel<<<grid_for(total, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(tasks, n, total);
  return int(cudaGetLastError());
}
int launch_misc(const MiscTask* tasks, int n, int64_t total, void* stream) {
  misc_kernel<<<grid_for(total, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(tasks, n, total);
  return int(cudaGetLastError());
}
int launch_topk(const TopkTask* tasks, int n, int blocks, int max_rows, void* stream) {
  const size_t smem = sel::stage_bytes(max_rows);
  cudaError_t e = allow_max_dyn_smem(topk_kernel);
  if (e != cudaSuccess) return int(e);
  topk_kernel<<<unsigned(blocks) * sel::SEL_CS, sel::SEL_THREADS, smem, static_cast<cudaStream_t>(stream)>>>(tasks, n);
  return int(cudaGetLastError());
}
int launch_add(const AddTask* tasks, int n, int64_t total, void* stream) {
  add_kernel<<<grid_for(total, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(tasks, n, total);
  return int(cudaGetLastError());
}

}  // namespace gemel
