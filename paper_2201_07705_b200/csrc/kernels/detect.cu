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
//  rpn_merge_kernel  one CTA per frame: every level's kept rows compacted in rank order,
//                    final ranks by binary searches across levels (a k-way merge), the
//                    first post_n written as proposals.
//  roi_align_kernel  a CTA per proposal, a thread per (bin, 8 channels): level from the
//                    box area, 4 bilinear samples of 16-byte NHWC bf16 vectors, fp32 average.
//  box_post_kernel   a warp per proposal: softmax over the class logits (warp
//                    reductions), BoxCoder(10,10,5,5) decode + clip per class.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "memops.h"
#include "smem_attr.cuh"
#include "select.cuh"

namespace gemel {
namespace {

constexpr float kXformClip = 4.135166556742356f;   // log(1000 / 16)

__device__ __forceinline__ uint32_t okey(float f) {   // order-preserving float -> uint32
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
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
  // disjoint: 0 / union = 0 (0/0 = NaN for two empty boxes) never suppresses (as
  // torchvision, thr >= 0); skipping the division also avoids its 0/0 slow path
  return inter > 0.f && inter / (aa + ab - inter) > thr;
}

constexpr int kRpnMax = 1024;
constexpr int kRpnMaskBytes = (kRpnMax + 1) * 32 * 4;   // [W32][Kp] words, Kp = K rounded up to odd
constexpr int kRpnSmem = kRpnMaskBytes + kRpnMax * 16 + kRpnMax * 4;

// RPN pre-NMS selection: a cluster of sel::SEL_CS CTAs per (model level, frame) selects
// the K highest objectness logits (ties by lower anchor index) straight from the fp32
// head; the leader writes rows t < K as (logit in field 4, anchor index bit-cast into
// field 5) in rank order -- rpn_nms_kernel decodes them and overwrites every field.
__global__ void __cluster_dims__(sel::SEL_CS, 1, 1) __launch_bounds__(sel::SEL_THREADS)
    rpn_select_kernel(const RpnTask* __restrict__ tasks, int n_tasks) {
  extern __shared__ uint32_t keys[];
  __shared__ sel::Shared S;
  const int fb = int(blockIdx.x) / sel::SEL_CS;
  int ti = 0;
  while (ti + 1 < n_tasks && fb >= tasks[ti + 1].block_begin) ++ti;
  const RpnTask& T = tasks[ti];
  const int frame = fb - T.block_begin;
  const int HW = T.h * T.w, A = T.A, cpc = T.cpc;
  const float* cls = T.cls + int64_t(frame) * HW * cpc;
  auto logit = [&](int i) { return cls[int64_t(i / A) * cpc + i % A]; };
  const int kt = sel::cluster_select([&](int i) { return sel::order_key(logit(i)); }, HW * A, T.K, S, keys);
  if (kt < 0) return;
  float* out = T.dst + int64_t(frame) * T.dst_pitch;
  for (int t = threadIdx.x; t < kt; t += sel::SEL_THREADS) {
    const int i = int(S.out[t] & 0xffffffffu);
    out[t * 6 + 4] = logit(i);
    out[t * 6 + 5] = __int_as_float(i);
  }
}

// RPN per level, after the selection: one CTA (1024 threads) per (model level, frame):
// BoxCoder decode + clip of the K ranked anchors, the IoU bitmask in shared memory and
// a blocked greedy scan by one warp.
__global__ void __launch_bounds__(1024) rpn_nms_kernel(const RpnTask* __restrict__ tasks, int n_tasks) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint32_t* mask = reinterpret_cast<uint32_t*>(smem);                                   // [W32][K]
  float4* bx = reinterpret_cast<float4*>(smem + kRpnMaskBytes);                         // [K]
  float* area = reinterpret_cast<float*>(smem + kRpnMaskBytes + kRpnMax * 16);          // [K]
  __shared__ uint32_t okw[32], keepw[32];
  int ti = 0;
  while (ti + 1 < n_tasks && int(blockIdx.x) >= tasks[ti + 1].block_begin) ++ti;
  const RpnTask& T = tasks[ti];
  const int frame = blockIdx.x - T.block_begin, tid = threadIdx.x, lane = tid & 31;
  const int HW = T.h * T.w, A = T.A, K = min(T.K, HW * A);
  const float* box = T.box + int64_t(frame) * HW * T.cpb;
  // 1. decode (BoxCoder(1,1,1,1)), clip, small-box test (one bit per row in okw)
  const float one[4] = {1.f, 1.f, 1.f, 1.f};
  float* out = T.dst + int64_t(frame) * T.dst_pitch;   // rows hold (logit, index) from the selection
  bool ok = false;
  if (tid < K) {
    const int i = __float_as_int(out[tid * 6 + 5]), pix = i / A, a = i % A;
    const float sx = float((pix % T.w) * T.stride_x), sy = float((pix / T.w) * T.stride_y);
    const float4 an = make_float4(sx + T.base[a][0], sy + T.base[a][1], sx + T.base[a][2], sy + T.base[a][3]);
    const float* d = box + int64_t(pix) * T.cpb + a * 4;
    const float4 b = clip(decode(an, d[0], d[1], d[2], d[3], one), T.img_w, T.img_h);
    bx[tid] = b;
    area[tid] = (b.z - b.x) * (b.w - b.y);
    ok = (b.z - b.x) >= T.min_size && (b.w - b.y) >= T.min_size;
    out[tid * 6 + 0] = b.x; out[tid * 6 + 1] = b.y; out[tid * 6 + 2] = b.z; out[tid * 6 + 3] = b.w;
  }
  const uint32_t okb = __ballot_sync(0xffffffffu, ok);   // blockDim 1024: warp w = rows 32w..32w+31
  if (lane == 0) okw[tid >> 5] = okb;
  __syncthreads();
  // 2. IoU bitmask, word-major (mask[wd*Kp + i], Kp = K | 1: the scan's lanes read one word
  //    per word row, lane * Kp apart -- an odd stride, so no bank conflicts): bit b of word wd of row i is set iff
  //    j = 32 wd + b < K, j != i and IoU(i, j) > nms.  Words right of row i's block hold
  //    the later rows; the diagonal word holds both sides (IoU is symmetric bit for bit:
  //    min/max and the area sum commute), which the blocked scan reads as "suppressed by
  //    an earlier row".  Branch-free over the 32 columns; words left of the diagonal are
  //    never read.  A warp = 32 consecutive rows of one word: the bx[j] reads broadcast.
  const int W32 = (K + 31) >> 5;
  const int Kp = K | 1;
  // the work is the upper triangle of (32-row block rb, word wd >= rb) pairs: one warp
  // task each, dealt round-robin over the warps so every warp gets the same number of
  // IoU words (a flat (word, row) loop gave the low-row warps ~30x the work of the
  // high-row ones)
  const int n_tasks_mask = W32 * (W32 + 1) / 2;
  for (int task = tid >> 5; task < n_tasks_mask; task += int(blockDim.x) >> 5) {
    int rb = 0, rest = task;
    while (rest >= W32 - rb) { rest -= W32 - rb; ++rb; }
    const int wd = rb + rest, i = rb * 32 + lane;
    const int j0 = wd * 32;
    if (i >= K) continue;   // past the last row (a partial last block)
    const float4 bi = bx[i];
    const float ai = area[i];
    uint32_t bits = 0;
#pragma unroll 8
    for (int b = 0; b < 32; ++b) {
      const float4 bj = bx[j0 + b];
      const float iw = fmaxf(0.f, fminf(bi.z, bj.z) - fmaxf(bi.x, bj.x));
      const float ih = fmaxf(0.f, fminf(bi.w, bj.w) - fmaxf(bi.y, bj.y));
      const float inter = iw * ih;
      // disjoint boxes (most pairs) skip the division: 0 / union = 0 (or NaN for two
      // empty boxes) never exceeds the threshold -- and 0/0 would take the slow path
      bool sup = false;
      if (inter > 0.f) sup = inter / (ai + area[j0 + b] - inter) > T.nms;
      bits |= uint32_t(sup) << b;
    }
    const int valid = K - j0;   // columns j < K
    if (valid < 32) bits &= (1u << valid) - 1u;
    if (j0 == i - (i & 31)) bits &= ~(1u << (i & 31));   // not itself
    mask[wd * Kp + i] = bits;
  }
  __syncthreads();
  // 3. greedy scan in score order by warp 0, 32 rows at a time (lane w holds removed-word
  //    w).  Within block b the kept set is the unique fixed point of
  //    kept = {j in cand : no kept l < j suppresses j}, reached by iterating from cand
  //    (row l's value is final after l + 1 iterations, so <= 32 rounds, usually 2-3);
  //    then every kept row's mask row is OR-ed into the later removed words.
  if (tid < 32) {
    uint32_t removed = 0;
    for (int b = 0; b < W32; ++b) {
      const uint32_t cand = okw[b] & ~__shfl_sync(0xffffffffu, removed, b);
      const int row = 32 * b + lane;
      const uint32_t before = row < K ? mask[b * Kp + row] & ((1u << lane) - 1u) : 0u;
      const bool mine = (cand >> lane) & 1u;
      uint32_t kept = cand;
      for (;;) {
        const uint32_t nk = __ballot_sync(0xffffffffu, mine && (before & kept) == 0u);
        if (nk == kept) break;
        kept = nk;
      }
      for (uint32_t k2 = kept; k2; k2 &= k2 - 1u) {
        const int l = __ffs(k2) - 1;
        if (lane > b && lane < W32) removed |= mask[lane * Kp + 32 * b + l];
      }
      if (lane == 0) keepw[b] = kept;
    }
  }
  __syncthreads();
  if (tid < K) out[tid * 6 + 5] = (keepw[tid >> 5] >> (tid & 31)) & 1u ? 1.f : 0.f;
}

// A frame's proposals across levels, one CTA (1024 threads) per frame.  Each level's rows
// are already in rank order (score descending, anchor index ascending), so its KEPT rows,
// compacted by a block scan, form a sorted list of packed keys (~okey(score) << 32 |
// level-concatenated index).  A kept row's final rank is its position in its own list
// plus, for every other level, the number of keys below its own (a binary search): a
// k-way merge by ranks, no sort; rows ranked < post_n are written, the rest of the
// post_n rows are zero.
__global__ void __launch_bounds__(1024) rpn_merge_kernel(const RpnMergeTask* __restrict__ tasks, int n_tasks) {
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned long long* lk = reinterpret_cast<unsigned long long*>(smem);   // [8][kRpnMax] kept keys per level
  __shared__ int warp_tot[33];
  __shared__ int s_cnt[8];
  int ti = 0;
  while (ti + 1 < n_tasks && int(blockIdx.x) >= tasks[ti + 1].block_begin) ++ti;
  const RpnMergeTask& T = tasks[ti];
  const int frame = blockIdx.x - T.block_begin, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  int off = 0;
  for (int l = 0; l < T.n_levels; ++l) {   // compaction of level l's kept rows, rank order kept
    const float* src = T.src[l] + int64_t(frame) * T.src_pitch[l];
    const int kl = T.k[l];
    const bool kept = tid < kl && src[tid * 6 + 5] > 0.5f;
    const unsigned b = __ballot_sync(0xffffffffu, kept);
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
      if (lane == 31) s_cnt[l] = incl;
    }
    __syncthreads();
    if (kept)
      lk[l * kRpnMax + warp_tot[wid] + __popc(b & ((1u << lane) - 1u))] =
          (uint64_t(~okey(src[tid * 6 + 4])) << 32) | uint32_t(off + tid);
    off += kl;
  }
  __syncthreads();
  int total = 0;
  for (int l = 0; l < T.n_levels; ++l) total += s_cnt[l];
  float* out = T.dst + int64_t(frame) * T.dst_pitch;
  for (int l = 0; l < T.n_levels; ++l) {
    const float* src = T.src[l] + int64_t(frame) * T.src_pitch[l];
    for (int r = tid; r < s_cnt[l]; r += blockDim.x) {
      const unsigned long long key = lk[l * kRpnMax + r];
      int rank = r;
      for (int l2 = 0; l2 < T.n_levels; ++l2) {   // keys of level l2 below this one
        if (l2 == l) continue;
        const unsigned long long* a2 = lk + l2 * kRpnMax;
        int lo = 0, hi = s_cnt[l2];
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (a2[mid] < key) lo = mid + 1; else hi = mid;
        }
        rank += lo;
      }
      if (rank < T.post_n) {
        int row = int(key & 0xffffffffu);
        for (int l3 = 0; l3 < l; ++l3) row -= T.k[l3];
        const float* sr = src + row * 6;
        out[rank * 5 + 0] = sr[0]; out[rank * 5 + 1] = sr[1]; out[rank * 5 + 2] = sr[2]; out[rank * 5 + 3] = sr[3];
        out[rank * 5 + 4] = 1.f;
      }
    }
  }
  for (int t = total + tid; t < T.post_n; t += blockDim.x)
    for (int f = 0; f < 5; ++f) out[t * 5 + f] = 0.f;
}

// One CTA per proposal: its out x out bins x C/8 channel groups loop over the CTA's
// threads (consecutive threads = consecutive 8-channel groups of one bin: 512-byte
// coalesced tap loads and output stores), so the proposal's footprint on its pyramid
// level (the bins' shared bilinear taps) is fetched from L2 once into this SM's L1.
// The proposal's level, its 2*out y-samples and 2*out x-samples (tap rows / columns,
// bilinear weights, the beyond-the-map test) are computed ONCE per CTA into shared
// memory (torchvision's sample positions and weight products, same float expressions);
// a (bin, channel group) item then issues its 16 tap loads straight from the tables.
constexpr int kRoiMaxSamples = 32;   // 2 * out (out <= 16) for the tabulated sampling = 2 path
constexpr int kRoiTableOut = 8;      // per-bin tap tables for out <= 8 (7x7 RoIAlign)

struct RoiSample {   // one sample coordinate along y or x
  int32_t i0, i1;    // tap rows / columns (clamped exactly as bilinear_interpolate)
  float l, h;        // weights of i1 and i0
  int32_t in;        // 0: the sample lies beyond [-1, size]: weight 0
};

// a0 += lo(v) * w, a1 += hi(v) * w (v: two bf16 values): one packed fp32x2 fma (sm_100
// FFMA2) after the two unpacks -- each lane an IEEE fma, the same value as two FFMAs
__device__ __forceinline__ void fma_bf16x2(float& a0, float& a1, uint32_t v, float w) {
  const float lo = __uint_as_float(v << 16), hi = __uint_as_float(v & 0xFFFF0000u);
  asm("{\n\t.reg .b64 x, y, a;\n\tmov.b64 x, {%2, %3};\n\tmov.b64 y, {%4, %4};\n\t"
      "mov.b64 a, {%0, %1};\n\tfma.rn.f32x2 a, x, y, a;\n\tmov.b64 {%0, %1}, a;\n\t}"
      : "+f"(a0), "+f"(a1)
      : "f"(lo), "f"(hi), "f"(w));
}

__device__ __forceinline__ RoiSample roi_sample(float v, int size) {
  RoiSample q;
  q.in = !(v < -1.f || v > float(size));
  float vv = fmaxf(v, 0.f);
  int i0 = q.in ? int(vv) : 0, i1;
  if (i0 >= size - 1) { i0 = i1 = size - 1; vv = float(i0); } else { i1 = i0 + 1; }
  q.i0 = i0; q.i1 = i1;
  q.l = vv - float(i0);
  q.h = 1.f - q.l;
  return q;
}

__global__ void __launch_bounds__(256, 4) roi_align_kernel(const RoiTask* __restrict__ tasks, int n_tasks) {
  __shared__ RoiSample sy[kRoiMaxSamples], sx[kRoiMaxSamples];
  __shared__ uint4 s_toff[kRoiTableOut * kRoiTableOut][4];    // per bin: 16 tap offsets (elements)
  __shared__ float4 s_twt[kRoiTableOut * kRoiTableOut][4];    // per bin: 16 tap weights
  const int64_t g = blockIdx.x;   // proposal index over all tasks
  int ti = 0;
  while (ti + 1 < n_tasks && g >= tasks[ti + 1].work_begin) ++ti;
  const RoiTask& T = tasks[ti];
  const int64_t roi = g - T.work_begin;
  const int nv = T.C >> 3;
  const int per = T.out * T.out * nv;
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
  const __nv_bfloat16* fm = static_cast<const __nv_bfloat16*>(T.map[li]) + int64_t(frame) * H * W * T.cp;
  __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(T.dst) + roi * T.out * T.out * T.cpd;
  const int cp = T.cp;

  if (T.sampling == 2 && 2 * T.out <= kRoiMaxSamples) {
    const int tid = threadIdx.x;
    if (tid < 2 * T.out) {   // y-sample tid = 2 ph + iy
      const int ph = tid >> 1, iy = tid & 1;
      sy[tid] = roi_sample(sh + float(ph) * bh + (float(iy) + .5f) * bh / 2.f, H);
    } else if (tid >= 64 && tid < 64 + 2 * T.out) {   // x-sample 2 pw + ix
      const int pw = (tid - 64) >> 1, ix = tid & 1;
      sx[tid - 64] = roi_sample(sw + float(pw) * bw + (float(ix) + .5f) * bw / 2.f, W);
    }
    __syncthreads();
    // per-bin tap tables (out <= 8): the 16 (offset, weight) pairs of every bin are the
    // same for the bin's 32 channel groups, so they are computed once per CTA here and each
    // item reads them as 8 broadcast 16-byte loads (the kernel is issue-bound)
    const bool tables = T.out <= kRoiTableOut;
    if (tables) {
      uint32_t* toff = reinterpret_cast<uint32_t*>(s_toff);
      float* twt = reinterpret_cast<float*>(s_twt);
      for (int e = tid; e < T.out * T.out * 16; e += int(blockDim.x)) {
        const int b2 = e >> 4, tap = e & 15, iy = tap >> 3, ix = (tap >> 2) & 1, corner = tap & 3;
        const int ph2 = b2 / T.out, pw2 = b2 - ph2 * T.out;
        const RoiSample a = sy[2 * ph2 + iy], b = sx[2 * pw2 + ix];
        const bool in = a.in && b.in;
        const uint32_t r = uint32_t(in ? ((corner & 2) ? a.i1 : a.i0) : 0) * uint32_t(W);
        const uint32_t cc = in ? ((corner & 1) ? b.i1 : b.i0) : 0;
        toff[e] = (r + cc) * cp;
        twt[e] = in ? ((corner & 2) ? a.l : a.h) * ((corner & 1) ? b.l : b.h) : 0.f;
      }
      __syncthreads();
    }
    // item l0 = bin * nv + v; with blockDim a multiple of nv (C = 256: nv = 32) a thread keeps
    // its channel group v and steps its bin (ph, pw) incrementally -- no divisions per item
    const bool fixed_v = int(blockDim.x) % nv == 0;
    const int bstep = int(blockDim.x) / nv;
    int bin = tid / nv, v = tid - bin * nv;
    int ph = bin / T.out, pw = bin - ph * T.out;
    for (int l0 = tid; l0 < per; l0 += int(blockDim.x)) {
      if (!fixed_v) {
        bin = l0 / nv; v = l0 - bin * nv;
        ph = bin / T.out; pw = bin - ph * T.out;
      }
      const __nv_bfloat16* fv = fm + v * 8;
      uint32_t off[16];
      float wt[16];
      if (tables) {
        const int b2 = ph * T.out + pw;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint4 o4 = s_toff[b2][k];
          const float4 w4 = s_twt[b2][k];
          off[4 * k] = o4.x; off[4 * k + 1] = o4.y; off[4 * k + 2] = o4.z; off[4 * k + 3] = o4.w;
          wt[4 * k] = w4.x; wt[4 * k + 1] = w4.y; wt[4 * k + 2] = w4.z; wt[4 * k + 3] = w4.w;
        }
      } else
#pragma unroll
      for (int iy = 0; iy < 2; ++iy)
#pragma unroll
        for (int ix = 0; ix < 2; ++ix) {
          const RoiSample a = sy[2 * ph + iy], b = sx[2 * pw + ix];
          const bool in = a.in && b.in;
          const int t = 4 * (2 * iy + ix);
          const uint32_t r0 = uint32_t(in ? a.i0 : 0) * uint32_t(W), r1 = uint32_t(in ? a.i1 : 0) * uint32_t(W);
          const uint32_t c0 = in ? b.i0 : 0, c1 = in ? b.i1 : 0;
          off[t + 0] = (r0 + c0) * cp; wt[t + 0] = in ? a.h * b.h : 0.f;
          off[t + 1] = (r0 + c1) * cp; wt[t + 1] = in ? a.h * b.l : 0.f;
          off[t + 2] = (r1 + c0) * cp; wt[t + 2] = in ? a.l * b.h : 0.f;
          off[t + 3] = (r1 + c1) * cp; wt[t + 3] = in ? a.l * b.l : 0.f;
        }
      uint4 q[16];
#pragma unroll
      for (int t = 0; t < 16; ++t) q[t] = __ldg(reinterpret_cast<const uint4*>(fv + off[t]));
      // fp32 weights and accumulation, channel pairs through packed fp32x2 fmas (the
      // kernel is issue-bound: ncu issue-active 84%)
      float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        fma_bf16x2(acc[0], acc[1], q[t].x, wt[t]);
        fma_bf16x2(acc[2], acc[3], q[t].y, wt[t]);
        fma_bf16x2(acc[4], acc[5], q[t].z, wt[t]);
        fma_bf16x2(acc[6], acc[7], q[t].w, wt[t]);
      }
      uint4 o;
      uint32_t* ou = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        __nv_bfloat162 h2 = __floats2bfloat162_rn(acc[2 * k] * .25f, acc[2 * k + 1] * .25f);
        ou[k] = *reinterpret_cast<uint32_t*>(&h2);
      }
      *reinterpret_cast<uint4*>(dst + (int64_t(ph) * T.out + pw) * T.cpd + v * 8) = o;
      if (fixed_v) {   // next bin of this thread
        pw += bstep;
        while (pw >= T.out) { pw -= T.out; ++ph; }
      }
    }
    return;
  }

  // general sampling ratio: samples evaluated per item
  for (int l0 = int(threadIdx.x); l0 < per; l0 += int(blockDim.x)) {
    const int bin = l0 / nv, v = l0 - bin * nv;
    const int ph = bin / T.out, pw = bin - ph * T.out;
    const __nv_bfloat16* fv = fm + v * 8;
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    auto tap = [&](int yy, int xx, float wgt) {
      const uint4 q = __ldg(reinterpret_cast<const uint4*>(fv + (int64_t(yy) * W + xx) * cp));
      const uint32_t u[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        acc[2 * k] += wgt * __uint_as_float(u[k] << 16);
        acc[2 * k + 1] += wgt * __uint_as_float(u[k] & 0xFFFF0000u);
      }
    };
    for (int iy = 0; iy < T.sampling; ++iy) {
      const RoiSample a = roi_sample(sh + float(ph) * bh + (float(iy) + .5f) * bh / float(T.sampling), H);
      for (int ix = 0; ix < T.sampling; ++ix) {
        const RoiSample b = roi_sample(sw + float(pw) * bw + (float(ix) + .5f) * bw / float(T.sampling), W);
        if (!a.in || !b.in) continue;
        tap(a.i0, b.i0, a.h * b.h);
        tap(a.i0, b.i1, a.h * b.l);
        tap(a.i1, b.i0, a.l * b.h);
        tap(a.i1, b.i1, a.l * b.l);
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
    *reinterpret_cast<uint4*>(dst + (int64_t(ph) * T.out + pw) * T.cpd + v * 8) = o;
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

int launch_rpn_level(const RpnTask* tasks, int n, int blocks, int max_anchors, void* stream) {
  const size_t sel_smem = sel::stage_bytes(max_anchors);
  cudaError_t e = allow_max_dyn_smem(rpn_select_kernel);
  if (e == cudaSuccess) e = allow_max_dyn_smem(rpn_nms_kernel);
  if (e != cudaSuccess) return int(e);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  rpn_select_kernel<<<unsigned(blocks) * sel::SEL_CS, sel::SEL_THREADS, sel_smem, st>>>(tasks, n);
  e = cudaGetLastError();
  if (e != cudaSuccess) return int(e);
  rpn_nms_kernel<<<blocks, 1024, kRpnSmem, st>>>(tasks, n);
  return int(cudaGetLastError());
}

int launch_rpn_merge(const RpnMergeTask* tasks, int n, int blocks, void* stream) {
  const int smem = 8 * kRpnMax * 8;
  cudaError_t e = allow_max_dyn_smem(rpn_merge_kernel);
  if (e != cudaSuccess) return int(e);
  rpn_merge_kernel<<<blocks, 1024, smem, static_cast<cudaStream_t>(stream)>>>(tasks, n);
  return int(cudaGetLastError());
}

int launch_roi_align(const RoiTask* tasks, int n, int64_t total_rois, void* stream) {
  roi_align_kernel<<<unsigned(total_rois), 256, 0, static_cast<cudaStream_t>(stream)>>>(tasks, n);
  return int(cudaGetLastError());
}

// Final detections: greedy batched NMS over one frame's
// score-ranked candidates, one 1024-thread CTA per frame, visited in blocks of 32:
//   A. every thread tests (candidate c of the block, kept rows slice) pairs -- a candidate
//      is suppressed by an already kept row of the same label with IoU > thr (smem
//      atomicOr into one 32-bit word);
//   B. warp 0 resolves the block in order: lane c's earlier same-label overlaps within
//      the block ("before" bits), the kept set as the unique fixed point of
//      kept = {c alive : no kept l < c in before(c)} (ballots, usually 2-3 rounds), cut to
//      the max_det - n_kept first, appended to the kept list.
// So a frame costs a few barriers per 32 visited candidates instead of per kept row.
// Rows with index -1 or a negative score (dropped candidates) start removed.
constexpr int kNmsMax = 1024;

__global__ void __launch_bounds__(1024) det_nms_kernel(const NmsTask* __restrict__ tasks, int n_tasks) {
  __shared__ float4 s_box[kNmsMax];
  __shared__ float s_lab[kNmsMax];
  __shared__ uint32_t s_alive[kNmsMax / 32];
  __shared__ int kept_idx[kNmsMax];
  __shared__ uint32_t s_sup;
  __shared__ int s_nkept;
  int ti = 0;
  while (ti + 1 < n_tasks && int(blockIdx.x) >= tasks[ti + 1].block_begin) ++ti;
  const NmsTask& T = tasks[ti];
  const int f = int(blockIdx.x) - T.block_begin;
  const int tid = int(threadIdx.x), lane = tid & 31, wid = tid >> 5;
  const float* src = T.src + int64_t(f) * T.src_pitch;
  float* dst = T.dst + int64_t(f) * T.dst_pitch;
  const int K = min(T.k_in, kNmsMax), max_det = min(T.max_det, kNmsMax);
  bool alive = false;
  if (tid < K) {
    const float* r = src + int64_t(tid) * 7;
    s_box[tid] = make_float4(r[1], r[2], r[3], r[4]);
    s_lab[tid] = r[6];
    alive = !(r[0] < 0.f || r[5] < 0.f);
  }
  const uint32_t aw = __ballot_sync(0xffffffffu, alive);
  if (lane == 0) s_alive[wid] = aw;
  if (tid == 0) { s_nkept = 0; s_sup = 0u; }
  __syncthreads();
  for (int base = 0; base < K; base += 32) {
    const int n_kept = s_nkept;                     // block-uniform (read after a barrier)
    if (n_kept >= max_det) break;
    const uint32_t blk_alive = s_alive[base >> 5];
    if (blk_alive) {
      // A. candidates of this block vs the kept rows: thread = (candidate c, slice)
      const int c = tid & 31, slice = tid >> 5;
      if ((blk_alive >> c) & 1u) {
        const float4 bc = s_box[base + c];
        const float lc = s_lab[base + c];
        bool sup = false;
        for (int k = slice; k < n_kept && !sup; k += 32) {
          const int j = kept_idx[k];
          sup = s_lab[j] == lc && iou_above(s_box[j], bc, T.iou);
        }
        if (sup) atomicOr(&s_sup, 1u << c);
      }
      __syncthreads();
      // B. in-order resolution of the block by warp 0
      if (wid == 0) {
        const uint32_t cand = blk_alive & ~s_sup;
        const int i = base + lane;
        uint32_t before = 0;
        if ((cand >> lane) & 1u) {
          const float4 bi = s_box[i];
          const float li = s_lab[i];
          for (int l = 0; l < lane; ++l)
            if (((cand >> l) & 1u) && s_lab[base + l] == li && iou_above(s_box[base + l], bi, T.iou)) before |= 1u << l;
        }
        const bool mine = (cand >> lane) & 1u;
        uint32_t kept = cand;
        for (;;) {
          const uint32_t nk = __ballot_sync(0xffffffffu, mine && (before & kept) == 0u);
          if (nk == kept) break;
          kept = nk;
        }
        const int room = max_det - n_kept;          // keep the first `room` of them
        while (__popc(kept) > room) kept &= ~(1u << (31 - __clz(kept)));
        if ((kept >> lane) & 1u) kept_idx[n_kept + __popc(kept & ((1u << lane) - 1u))] = i;
        if (lane == 0) { s_nkept = n_kept + __popc(kept); s_sup = 0u; }
      }
      __syncthreads();
    }
  }
  const int n_kept = s_nkept;
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
