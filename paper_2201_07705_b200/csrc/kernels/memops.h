// Memory-bound kernels: frame ingest, pooling,
// standalone residual add, concat / nearest upsample, YOLO box decode.
// NHWC bf16, 16-byte vectors (8 channels) per thread.
#pragma once
#include <cstdint>

namespace gemel {

struct PreTask {            // uint8 RGB HWC frames -> normalised bf16
  const uint8_t* src;
  void* dst;
  int64_t work;             // mode 0: pixels; mode 1: rows * (Kp / 8)
  int64_t work_begin;       // prefix over tasks
  int32_t mode;             // 0: NHWC, C padded to 8; 1: im2col matrix of the first conv
  int32_t h, w, ho, wo;     // input / conv output size (mode 1)
  int32_t kh, kw, sh, sw, ph, pw, dh, dw;
  int32_t K, Kp;            // K = kh*kw*3 columns (r, s, c), row pitch Kp (zero padded)
};

struct PoolTask {           // NHWC bf16 [n, h, w, cp] -> [n, ho, wo, cp]
  const void* src;
  void* dst;
  int32_t n, h, w, cp, ho, wo;
  int32_t kh, kw, sh, sw, ph, pw, dh, dw;
  int32_t kind;             // 0 max (PyTorch, -inf pad), 1 adaptive average
  int32_t pad_;
  int64_t work_begin;       // prefix over tasks of n*ho*wo*(cp/8)
};

struct AddTask {            // out = act(a + b), bf16 vectors
  const void* a;
  const void* b;
  void* out;
  int64_t vecs;             // number of 8-element vectors
  int32_t act;
  float slope;
  int64_t work_begin;
};

struct MiscTask {           // one concat piece (bf16) or one YOLO head decode (fp32)
  const void* src;
  void* dst;
  int32_t kind;             // 0: concat piece with nearest upsample by `scale`, 1: YOLO decode,
                            // 2: L2Norm (a warp per pixel), 3: SSD decode (a warp per box)
  int32_t n, h, w;          // output spatial size (concat) / feature size (YOLO)
  int32_t c;                // concat: channels copied (multiple of 8); YOLO: fields per box (5 + classes)
  int32_t cps, cpd;         // channel pitch of src / dst (elements)
  int32_t c_off;            // concat: first destination channel (multiple of 8)
  int32_t scale;            // concat: nearest-upsample factor (1 = plain copy)
  int32_t A;                // YOLO: anchors
  float stride_w, stride_h; // YOLO: input pixels per cell
  float anchors[16];        // YOLO: (w, h) pixels per anchor; SSD: (w, h) relative to the image
  int64_t dst_pitch;        // YOLO/SSD: elements per frame of the detection row
  int64_t dst_off;          // YOLO/SSD: element offset of this head within the row
  int64_t work_begin;       // concat: 8-channel vectors; YOLO: 16 per box (a half-warp per box); L2Norm: 32 per
                            // pixel (multiple of 32); SSD: 32 per box (a warp per box)
  const void* src2;         // SSD: conf head (fp32 [n, h, w, cps2])
  const float* vec;         // L2Norm: per-channel scale (fp32, weight arena)
  int32_t cps2;             // SSD: conf channel pitch
  float eps;                // L2Norm
  float wts[4];             // SSD box-coder weights
  float img_w, img_h;       // SSD: image size in pixels
  int64_t work;             // real work items of this task (work_begin spacing is padded to 32)
  int32_t det_fmt;          // detection candidates (kind 4): 0 Fast R-CNN rows, 1 YOLO, 2 SSD
  float det_thresh;         // detection candidates: score threshold (kept iff score > it); eps = min side
  int64_t rows;             // detection candidates: rows per frame (c = fields per row)
};

struct NmsTask {            // greedy batched NMS over one model's top-k candidate rows (N2)
  const float* src;         // [n][k_in * 7] (index, x1, y1, x2, y2, score, label), score-ranked
  float* dst;               // [n][max_det * 6]
  int32_t n, k_in, max_det;
  float iou;
  int64_t src_pitch, dst_pitch;   // elements per frame
  int32_t block_begin;      // first CTA (one CTA of 32 threads per frame)
  int32_t pad_;
};

struct TopkTask {           // per frame: the k highest-scoring rows of a flat fp32 row set
  const float* src;
  float* dst;
  int32_t n;                // frames
  int32_t rows, fields, k, score;
  int32_t block_begin;      // prefix over tasks of frames (one CTA per frame)
  int64_t src_pitch, dst_pitch;   // elements per frame
};

// ---- Faster R-CNN stages (RPN top-k + NMS, MultiScaleRoIAlign;
// a11: box decode).  detect.cu.
struct RpnTask {            // one FPN level of one model: proposals per frame (one CTA per frame)
  const float* cls;         // objectness head, fp32 NHWC [n, h, w, cpc], channel a
  const float* box;         // box-delta head, fp32 NHWC [n, h, w, cpb], channel a*4+j
  float* dst;               // fp32 [n, dst_pitch]: K rows (x1, y1, x2, y2, logit, keep)
  int32_t n, h, w, A, cpc, cpb;
  int32_t K;                // min(pre_n, h*w*A) <= 1024
  int32_t stride_y, stride_x;   // image // feature (integer division, torchvision)
  float base[8][4];         // rounded base anchors (x1, y1, x2, y2), ratio-major
  float nms, min_size, img_w, img_h;
  int64_t dst_pitch;
  int32_t block_begin;      // prefix over tasks of frames
  int32_t pad_;
};

struct RpnMergeTask {       // a frame's proposals across levels (one CTA per frame)
  const float* src[8];      // RpnTask outputs
  int64_t src_pitch[8];
  int32_t k[8];             // rows per level
  int32_t n_levels, n, post_n, block_begin;
  float* dst;               // fp32 [n, dst_pitch]: post_n rows (x1, y1, x2, y2, valid)
  int64_t dst_pitch;
};

struct RoiTask {            // MultiScaleRoIAlign of one model: a CTA per proposal, a thread per (bin, 8 channels)
  const float* props;       // RpnMergeTask output
  int64_t props_pitch;
  const void* map[4];       // bf16 NHWC [n, mh, mw, cp] finest first
  int32_t mh[4], mw[4];
  float scale[4];
  int32_t n_maps, k_min, cp, C;
  int32_t n, R, out, sampling;
  float canon_scale, canon_level;
  void* dst;                // bf16 NHWC [n*R, out, out, cpd]
  int32_t cpd, pad_;
  int64_t work_begin, work;   // first proposal (over all tasks) and proposals of this task
};

struct BoxPostTask {        // Fast R-CNN decode of one model: a warp per (frame, roi)
  const float* cls;         // fp32 [n*R, cpc] logits
  const float* box;         // fp32 [n*R, cpb] deltas (class j at 4j)
  const float* props;       // RpnMergeTask output
  float* dst;               // fp32 [n, dst_pitch]: R*(classes-1) rows of 6
  int32_t n, R, classes, cpc, cpb, pad_;
  int64_t props_pitch, dst_pitch;
  float wts[4];
  float img_w, img_h;
  int64_t work_begin;       // prefix over tasks of warps (n*R)
};

// SM count of the current device (queried once per process; one context per GPU).
int device_sm_count();

// two launches: the cluster top-K selection per (level, frame), then decode + NMS
int launch_rpn_level(const RpnTask* tasks_dev, int n_tasks, int blocks, int max_anchors, void* stream);
int launch_rpn_merge(const RpnMergeTask* tasks_dev, int n_tasks, int blocks, void* stream);
int launch_roi_align(const RoiTask* tasks_dev, int n_tasks, int64_t total_work, void* stream);
int launch_box_post(const BoxPostTask* tasks_dev, int n_tasks, int64_t total_warps, void* stream);

int launch_preprocess(const PreTask* tasks_dev, int n_tasks, int64_t total_pixels, void* stream);
// tasks: mode-1 (im2col) tasks only, work_begin = block prefix (blocks = images * out rows)
int launch_ingest_cols(const PreTask* tasks_dev, int n_tasks, int64_t blocks, int smem_bytes, void* stream);
int launch_pool(const PoolTask* tasks_dev, int n_tasks, int64_t total_work, void* stream);
int launch_add(const AddTask* tasks_dev, int n_tasks, int64_t total_work, void* stream);
int launch_misc(const MiscTask* tasks_dev, int n_tasks, int64_t total_work, void* stream);
int launch_topk(const TopkTask* tasks_dev, int n_tasks, int blocks, int max_rows, void* stream);
int launch_det_nms(const NmsTask* tasks_dev, int n_tasks, int blocks, void* stream);

}  // namespace gemel
