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
                            // 2: L2Norm (a warp per pixel), 3: SSD decode (a thread per box)
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
  int64_t work_begin;       // concat: 8-channel vectors; YOLO: output elements; L2Norm: 32 per
                            // pixel (multiple of 32); SSD: boxes
  const void* src2;         // SSD: conf head (fp32 [n, h, w, cps2])
  const float* vec;         // L2Norm: per-channel scale (fp32, weight arena)
  int32_t cps2;             // SSD: conf channel pitch
  float eps;                // L2Norm
  float wts[4];             // SSD box-coder weights
  float img_w, img_h;       // SSD: image size in pixels
  int64_t work;             // real work items of this task (work_begin spacing is padded to 32)
};

struct TopkTask {           // per frame: the k highest-scoring rows of a flat fp32 row set
  const float* src;
  float* dst;
  int32_t n;                // frames
  int32_t rows, fields, k, score;
  int32_t block_begin;      // prefix over tasks of frames (one CTA per frame)
  int64_t src_pitch, dst_pitch;   // elements per frame
};

int launch_preprocess(const PreTask* tasks_dev, int n_tasks, int64_t total_pixels, void* stream);
// tasks: mode-1 (im2col) tasks only, work_begin = block prefix (blocks = images * out rows)
int launch_ingest_cols(const PreTask* tasks_dev, int n_tasks, int64_t blocks, int smem_bytes, void* stream);
int launch_pool(const PoolTask* tasks_dev, int n_tasks, int64_t total_work, void* stream);
int launch_add(const AddTask* tasks_dev, int n_tasks, int64_t total_work, void* stream);
int launch_misc(const MiscTask* tasks_dev, int n_tasks, int64_t total_work, void* stream);
int launch_topk(const TopkTask* tasks_dev, int n_tasks, int blocks, int max_rows, void* stream);

}  // namespace gemel
