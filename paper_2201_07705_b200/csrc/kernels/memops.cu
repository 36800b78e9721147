// Memory-bound kernels: frame preprocessing, max /
// adaptive-average pooling and standalone residual add (a9).  Grouped: one
// launch covers every task of a scheduler wave through a task table; each
// thread handles one 16-byte vector (8 bf16 channels) of one output pixel.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "gemm.h"
#include "memops.h"

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
    } else {
      const uint32_t per = uint32_t(T.A) * T.h * T.w * T.c;   // elements per frame of this head
      const int n = int(r / per);
      uint32_t q = r - uint32_t(n) * per;
      const int f = int(q % uint32_t(T.c));
      q /= uint32_t(T.c);
      const int x = int(q % uint32_t(T.w));
      q /= uint32_t(T.w);
      const int y = int(q % uint32_t(T.h));
      const int a = int(q / uint32_t(T.h));
      const float t = reinterpret_cast<const float*>(T.src)[((int64_t(n) * T.h + y) * T.w + x) * T.cps + a * T.c + f];
      float o;
      if (f == 0) o = (1.f / (1.f + __expf(-t)) + float(x)) * T.stride_w;
      else if (f == 1) o = (1.f / (1.f + __expf(-t)) + float(y)) * T.stride_h;
      else if (f == 2) o = T.anchors[2 * a] * expf(t);
      else if (f == 3) o = T.anchors[2 * a + 1] * expf(t);
      else o = 1.f / (1.f + expf(-t));
      reinterpret_cast<float*>(T.dst)[int64_t(n) * T.dst_pitch + T.dst_off + (r - uint32_t(n) * per)] = o;
    }
  }
}

// Top-k rows per frame, one CTA of 1024 threads per frame:
//  1. scores -> order-preserving uint32 keys in smem;
//  2. radix select (4 passes of 8 bits, smem histograms) finds T, the k-th largest key,
//     and how many rows equal to T are taken;
//  3. an index-ordered compaction (warp ballots + a block scan per 1024-row chunk)
//     keeps rows with key > T and the first rows with key == T -- ties by lower index;
//  4. the k survivors are placed by counting rank (score desc, index asc) and their
//     fields copied.  Integer selection: bit-exact against the oracle.
constexpr int kTopkSmemRows = 50000;

__device__ __forceinline__ uint32_t order_key(float f) {
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// exclusive prefix of a per-thread flag over the 1024-thread block; returns the block total
__device__ __forceinline__ int block_excl_scan(bool flag, int* warp_tot, int& excl) {
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
    warp_tot[lane] = incl - v;   // exclusive warp offsets
    if (lane == 31) warp_tot[32] = incl;
  }
  __syncthreads();
  excl = warp_tot[wid] + in_warp;
  return warp_tot[32];
}

__global__ void __launch_bounds__(1024) topk_kernel(const TopkTask* __restrict__ tasks, int n_tasks) {
  extern __shared__ uint32_t keys[];
  __shared__ int hist[256];
  __shared__ int warp_tot[33];
  __shared__ int sel_idx[1024];
  __shared__ int eq_idx[1024];
  __shared__ int s_cnt, s_eq;
  __shared__ uint32_t s_prefix;
  __shared__ int s_remaining;
  int ti = 0;
  while (ti + 1 < n_tasks && int(blockIdx.x) >= tasks[ti + 1].block_begin) ++ti;
  const TopkTask& T = tasks[ti];
  const int frame = blockIdx.x - T.block_begin;
  const float* row = T.src + frame * T.src_pitch;
  float* out = T.dst + frame * T.dst_pitch;
  const int n = T.rows, F = T.fields, tid = threadIdx.x;
  const int kt = min(T.k, n);
  // keys staged in shared memory when they fit (<= kTopkSmemRows), else re-derived from
  // the row (L2-resident) on every pass -- e.g. Faster R-CNN's 90 000 (proposal, class) rows
  const bool staged = n <= kTopkSmemRows;
  auto key_of = [&](int i) { return staged ? keys[i] : order_key(row[int64_t(i) * F + T.score]); };
  if (staged)
    for (int i = tid; i < n; i += blockDim.x) keys[i] = order_key(row[int64_t(i) * F + T.score]);
  if (tid == 0) { s_prefix = 0; s_remaining = kt; }
  __syncthreads();
  uint32_t mask = 0;
  for (int shift = 24; shift >= 0 && kt > 0; shift -= 8) {
    for (int i = tid; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    const uint32_t prefix = s_prefix;
    for (int i = tid; i < n; i += blockDim.x) {
      const uint32_t key = key_of(i);
      if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255], 1);
    }
    __syncthreads();
    if (tid == 0) {
      int cum = 0, rem = s_remaining;
      for (int d = 255; d >= 0; --d) {
        if (cum + hist[d] >= rem) {
          s_prefix = prefix | (uint32_t(d) << shift);
          s_remaining = rem - cum;
          break;
        }
        cum += hist[d];
      }
    }
    mask |= 255u << shift;
    __syncthreads();
  }
  const uint32_t thr = s_prefix;
  const int need_eq = s_remaining;   // rows equal to the threshold key that are taken
  // compaction: rows above the threshold in any order (warp-aggregated smem atomics, no
  // block-wide scans -- the survivors are ranked below), then the need_eq equal rows with
  // the lowest indices
  if (tid == 0) { s_cnt = 0; s_eq = 0; }
  __syncthreads();
  const int lane = tid & 31;
  for (int base = 0; base < n && kt > 0; base += blockDim.x) {
    const int i = base + tid;
    const uint32_t key = i < n ? key_of(i) : 0u;
    const bool above = i < n && key > thr, eq = i < n && key == thr;
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
    if (eq && be + __popc(me & lt) < 1024) eq_idx[be + __popc(me & lt)] = i;
  }
  __syncthreads();
  const int n_above = s_cnt, n_eq = s_eq;
  if (kt > 0 && n_eq <= 1024) {
    if (tid < n_eq) {   // rank of each equal row by index; the need_eq lowest are taken
      const int me_i = eq_idx[tid];
      int rank = 0;
      for (int j = 0; j < n_eq; ++j) rank += eq_idx[j] < me_i;
      if (rank < need_eq) sel_idx[n_above + rank] = me_i;
    }
  } else if (kt > 0) {   // more than 1024 equal rows: index-ordered scan of the equal ones
    int eq_seen = 0;
    for (int base = 0; base < n && eq_seen < need_eq; base += blockDim.x) {
      const int i = base + tid;
      const bool eq = i < n && key_of(i) == thr;
      int eq_rank;
      const int eq_tot = block_excl_scan(eq, warp_tot, eq_rank);
      if (eq && eq_seen + eq_rank < need_eq) sel_idx[n_above + eq_seen + eq_rank] = i;
      eq_seen += eq_tot;
    }
  }
  __syncthreads();
  const int Fo = F + 1;
  if (tid < kt) {   // counting rank among the survivors: score desc, index asc
    const int me = sel_idx[tid];
    const uint32_t mk = key_of(me);
    int rank = 0;
    for (int j = 0; j < kt; ++j) {
      const int o = sel_idx[j];
      const uint32_t ok = key_of(o);
      rank += (ok > mk) || (ok == mk && o < me);
    }
    out[int64_t(rank) * Fo] = float(me);
    for (int f = 0; f < F; ++f) out[int64_t(rank) * Fo + 1 + f] = row[int64_t(me) * F + f];
  } else if (tid < T.k) {
    out[int64_t(tid) * Fo] = -1.f;
    for (int f = 0; f < F; ++f) out[int64_t(tid) * Fo + 1 + f] = 0.f;
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
    cudaError_t e = cudaFuncSetAttribute(ingest_cols_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
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
  const size_t smem = size_t(max_rows < kTopkSmemRows ? max_rows : kTopkSmemRows) * 4;
  cudaError_t e = cudaFuncSetAttribute(topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  if (e != cudaSuccess) return int(e);
  topk_kernel<<<blocks, 1024, smem, static_cast<cudaStream_t>(stream)>>>(tasks, n);
  return int(cudaGetLastError());
}
int launch_add(const AddTask* tasks, int n, int64_t total, void* stream) {
  add_kernel<<<grid_for(total, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(tasks, n, total);
  return int(cudaGetLastError());
}

}  // namespace gemel
