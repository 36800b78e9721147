/*
 * gemel.h -- C ABI of the B200-native GEMEL merged multi-model inference path.
 *
 * The library implements the data-parallel hot path of model merging from
 * Padmanabhan et al., "GEMEL: Model Merging for Memory-Efficient, Real-Time
 * Video Analytics at the Edge" (arXiv 2201.07705; PAPER.md = its LaTeX source):
 *
 *   gemel_register_model  -- a query's DNN as a layer list
 *   gemel_find_shareable  -- groups of architecturally identical
 *                            layers, memory-sorted
 *   gemel_apply_merge     -- bind each group to ONE weight copy,
 *                            return the weight bytes saved
 *   gemel_infer           -- one frame batch per camera stream through every
 *                            (merged) model; each shared layer runs once over
 *                            the concatenated batches of the models sharing it
 *                            (SURVEY.md §8(a) a5-a11).  Merging never shares
 *                            intermediates: models see their own frames.
 *
 * Conventions
 *   - Every call returns gemel_status: GEMEL_OK (0) or a negative error.  No
 *     exception crosses the ABI.  gemel_last_error(ctx) gives a message naming
 *     the model id, op position and failed invariant.
 *   - A context is not thread-safe; use one context per GPU / process.
 *   - Host-side calls (create, register_model, find_shareable, apply_merge,
 *     stats, last_error, destroy) never touch the GPU; gemel_plan and later
 *     require a CUDA device.
 *   - Tensors: activations are NHWC bf16 with the channel pitch padded to a
 *     multiple of 8 (pad channels hold zeros); final-layer outputs are fp32
 *     [batch, features].  Weights are registered as fp32 host arrays in PyTorch
 *     layout (conv [cout, cin/groups, kh, kw], linear [fout, fin]); the library
 *     stores conv/linear weights in bf16 (values are expected to be bf16-exact,
 *     they are rounded to nearest-even otherwise) and BN statistics in fp32.
 *   - Byte accounting (bytes saved, group bytes) is exact integer arithmetic in
 *     the registered dtype: bf16 = 2 bytes per parameter element, BN counting
 *     gamma, beta, running mean and running var (reading R4).
 */
#ifndef GEMEL_H
#define GEMEL_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t gemel_status;
typedef struct gemel_ctx_s* gemel_ctx;

enum {
  GEMEL_OK = 0,
  GEMEL_E_ARG = -1,         /* null pointer, bad id, bad size                      */
  GEMEL_E_SCHEMA = -2,      /* layer list violates its op schema                   */
  GEMEL_E_MERGE = -3,       /* invalid merge group (signature mismatch, reuse...) */
  GEMEL_E_STATE = -4,       /* call out of order (e.g. register after plan)        */
  GEMEL_E_NOMEM = -5,       /* arena too small / allocation failed                 */
  GEMEL_E_CUDA = -6,        /* CUDA runtime / driver error (message has details)   */
  GEMEL_E_SMALLBUF = -7,    /* caller buffer too small; required count returned    */
  GEMEL_E_UNSUPPORTED = -8  /* layer configuration the CUDA path does not support  */
};

/* Layer types: the paper's "layer type". */
enum gemel_op {
  GEMEL_OP_CONV2D = 1,
  GEMEL_OP_LINEAR = 2,
  GEMEL_OP_BATCHNORM2D = 3,
  GEMEL_OP_RELU = 4,
  GEMEL_OP_LEAKY_RELU = 5,
  GEMEL_OP_MAXPOOL2D = 6,
  GEMEL_OP_ADAPTIVE_AVGPOOL2D = 7,
  GEMEL_OP_ADD = 8,
  GEMEL_OP_FLATTEN = 9,
  GEMEL_OP_CONCAT = 10,
  GEMEL_OP_UPSAMPLE_NEAREST = 11,
  GEMEL_OP_YOLO_DECODE = 12,
  GEMEL_OP_TOPK = 13,
  GEMEL_OP_L2NORM = 14,
  GEMEL_OP_SSD_DECODE = 15,
  GEMEL_OP_RPN_LEVEL = 16,
  GEMEL_OP_RPN_MERGE = 17,
  GEMEL_OP_ROI_ALIGN = 18,
  GEMEL_OP_BOX_POST = 19,
  GEMEL_OP_DET_CANDIDATES = 20,
  GEMEL_OP_DET_NMS = 21
};

/*
 * One layer.  in[] are producer op positions within the same model (-1 = the
 * model input, i.e. the preprocessed frame); the list must be topologically
 * ordered.  Fields used per op (others must be 0):
 *   CONV2D      cin, cout, kh, kw, sh, sw, ph, pw, dh, dw, groups (=1), bias;
 *               param[0] = weight [cout, cin, kh, kw], param[1] = bias [cout] or NULL
 *   LINEAR      cin = in_features, cout = out_features, bias;
 *               param[0] = weight [cout, cin], param[1] = bias or NULL
 *   BATCHNORM2D cin = channels, eps, momentum, affine (=1), track_stats (=1);
 *               param[0..3] = gamma, beta, running_mean, running_var
 *   LEAKY_RELU  neg_slope
 *   MAXPOOL2D   kh, kw, sh, sw, ph, pw, dh, dw, ceil_mode (0 floor, 1 PyTorch ceil_mode,
 *               2 darknet: windows [i*s, i*s+k) with out-of-range taps ignored,
 *               out = (H-1)/s + 1 -- Tiny-YOLOv3's 2x2 stride-1 pool)
 *   ADAPTIVE_AVGPOOL2D out_h, out_w
 *   ADD         n_in = 2
 *   CONCAT      n_in = 2..8 along channels (equal H x W), or along features when
 *               every input is flat (a YOLO decode): darknet "route" / detection output
 *   UPSAMPLE_NEAREST sh = sw = integer scale factor
 *   YOLO_DECODE kh = anchors A, cout = classes, cin = A*(5+classes) (= producer channels);
 *               param[0] = anchors [A][2] (w, h in input pixels).  Output flat fp32
 *               [A*H*W*(5+classes)] per frame in (anchor, cy, cx, field) order:
 *               bx = (sigmoid(t0)+cx)*in_w/W, by = (sigmoid(t1)+cy)*in_h/H,
 *               bw = aw*exp(t2), bh = ah*exp(t3), objectness/classes = sigmoid
 *               (darknet yolo layer).  Not a param layer.
 *   TOPK        cin = fields per candidate row, cout = k, kh = score column; input flat
 *               (e.g. a concat of YOLO decodes).  Output flat fp32 [k*(fields+1)] per frame:
 *               the k rows with the highest score, descending, ties by lower row index,
 *               each as (row index, fields...); missing rows are (-1, 0...).
 *   L2NORM      cin = channels, eps; param[0] = scale [cin]:  x / max(||x||_c, eps) * scale
 *               (SSD conv4_3).  Not a param layer (R2); the scale stays resident.
 *   SSD_DECODE  n_in = 2 (loc head [A*4 ch], conf head [A*cout ch], same H x W); kh = A,
 *               cout = classes, sh = step (pixels per default-box cell); param[0] = (w, h)
 *               per anchor relative to the image [A][2], param[1] = box-coder weights [4].
 *               Output flat fp32 [H*W*A*(5+classes)] in (cy, cx, anchor) order: x1, y1, x2, y2
 *               (torchvision BoxCoder decode of the default box, dw/dh clamped at
 *               log(1000/16), clipped to the image), best foreground probability, softmax.
 *   RPN_LEVEL   Faster R-CNN region proposals of one FPN level (torchvision RPN, eval):
 *               n_in = 2 (objectness head [A ch], box-delta head [4A ch, channel a*4+j],
 *               both conv heads, same H x W); kh = A anchors, cout = pre_n (1..1024),
 *               neg_slope = NMS IoU threshold, eps = min box size; param[0] = [A][2]
 *               (size, aspect ratio).  Anchors round([-w,-h,w,h]/2), h = size*sqrt(r),
 *               w = size/sqrt(r), shifted by (x, y) * (image / feature, integer division),
 *               order (y, x, a); BoxCoder(1,1,1,1) decode (dw, dh <= log(1000/16)); the
 *               K = min(pre_n, H*W*A) highest logits (ties by lower anchor index), in that
 *               order; clipped to the image; keep = w, h >= eps and not suppressed by greedy
 *               NMS (IoU > neg_slope) among this level's kept boxes.  Output flat fp32
 *               [K*6] per frame: rows (x1, y1, x2, y2, logit, keep 0/1).
 *   RPN_MERGE   n_in = 1..8 RPN_LEVEL outputs of one frame; cout = post_n.  Output flat fp32
 *               [post_n*5]: the kept rows of all levels by logit descending (ties by lower
 *               level-concatenated index), first post_n, as (x1, y1, x2, y2, 1); missing
 *               rows (0, 0, 0, 0, 0).
 *   ROI_ALIGN   MultiScaleRoIAlign: n_in = 1 + L, in[0] = RPN_MERGE proposals, in[1..L] =
 *               feature maps finest first (bf16, equal C); out_h = out_w = output size,
 *               kh = sampling ratio, sh = canonical scale (224), sw = canonical level (4).
 *               Map l's scale = 2^round(log2(H_l / in_h)); proposal level = floor(sw +
 *               log2(sqrt(area) / sh) + 1e-6) clamped to the maps' levels; roi_align with
 *               aligned = false.  Output: one [C, out_h, out_w] value PER PROPOSAL (the
 *               value's batch is frames * post_n), stored NHWC bf16 like any activation.
 *   BOX_POST    Fast R-CNN box decode: n_in = 3 (class logits [cout] and box deltas
 *               [4*cout] per proposal -- linear outputs over ROI_ALIGN rows -- then the
 *               RPN_MERGE proposals); cout = classes; param[0] = box-coder weights [4].
 *               Output flat fp32 [post_n*(cout-1)*6] per frame: rows (x1, y1, x2, y2,
 *               softmax probability, class) for classes 1.. in (proposal, class) order,
 *               boxes decoded against the proposal and clipped; a missing proposal's rows
 *               score -1.
 *   DET_CANDIDATES  final detection candidates (R22): n_in = 1
 *               flat input of rows of cin fields; kh = format: 0 Fast R-CNN BOX_POST rows
 *               (x1, y1, x2, y2, p, label) as they are (cin = 6); 1 YOLO decode rows (cx, cy,
 *               w, h, obj, classes...): corners, score obj * max class, label the first
 *               argmax; 2 SSD decode rows (x1, y1, x2, y2, best, softmax...): score max over
 *               classes >= 1, label its first argmax.  neg_slope = score threshold (kept iff
 *               score > it), eps = min box side (kept iff w, h >= eps).  Output flat fp32
 *               [rows*6] per frame (x1, y1, x2, y2, score, label), dropped rows score -1.
 *   DET_NMS     greedy batched NMS (torchvision batched_nms): n_in = 1, a TOPK (score
 *               column 4) over DET_CANDIDATES rows; cout = max detections (1..1024),
 *               neg_slope = IoU threshold.  Rows are visited in the TOPK order, skipping
 *               index -1 / negative scores; a row is kept unless a kept row of the same
 *               label overlaps it with IoU > neg_slope.  Output flat fp32 [cout*6]: the
 *               first cout kept rows (x1, y1, x2, y2, score, label); missing rows score -1.
 * tie (CONV2D only): 0 = the layer owns its parameters; j+1 = it applies op j's
 *   parameters (same hyperparameters; param[] ignored).  A tied conv is not a separate
 *   layer: no parameter bytes, never in a shareable group (the Faster R-CNN RPN head is
 *   one weight set run on every FPN level).
 * Architectural signature: op + every field above except in[],
 * param[] and the input H x W.
 */
typedef struct {
  int32_t op;
  int32_t n_in;
  int32_t in[8];
  int32_t cin, cout;
  int32_t kh, kw, sh, sw, ph, pw, dh, dw;
  int32_t groups, bias, ceil_mode, tie;
  int32_t out_h, out_w;
  float eps, momentum, neg_slope;
  int32_t affine, track_stats;
  const float* param[4]; /* host, fp32, copied by register_model (caller keeps ownership) */
} gemel_layer;

enum { GEMEL_FLAG_DRY_PLAN = 1 }; /* gemel_plan without a device (host-side planner tests); no bind/infer */

typedef struct {
  int32_t device;                /* CUDA device ordinal used from gemel_plan on */
  int32_t flags;                 /* GEMEL_FLAG_* */
  void* compute_stream;          /* cudaStream_t for all kernels (NULL = legacy default) */
  uint64_t weight_budget_bytes;  /* 0 = unlimited (weights fully resident) */
  int32_t weight_source;         /* where weights above the budget are paged from every step:
                                    GEMEL_SOURCE_HOST (pinned host memory over PCIe) or
                                    GEMEL_SOURCE_PEER (the HBM of device `source_device`, a
                                    peer GPU over NVLink -- SURVEY.md §8(f) N4; the same
                                    device is allowed and pages within HBM) */
  int32_t source_device;         /* CUDA ordinal holding the paged weights (GEMEL_SOURCE_PEER) */
} gemel_options;

enum { GEMEL_SOURCE_HOST = 0, GEMEL_SOURCE_PEER = 1 };

/* A group of architecturally identical layers across the workload. */
typedef struct {
  int32_t op;             /* gemel_op of the layers in the group */
  int32_t n_apps;         /* appearances (>= 2) */
  int32_t app_offset;     /* index of the first appearance in the appearance array */
  int32_t reserved;
  uint64_t per_bytes;     /* parameter bytes of one appearance (bf16) */
  uint64_t total_bytes;   /* per_bytes * n_apps: the sort key */
  uint64_t reclaimable;   /* per_bytes * (n_apps - 1): saved if fully merged */
} gemel_group;

typedef struct {
  int32_t model_id;
  int32_t op_pos;
} gemel_appearance;

/* A merge group: members bound to the weights of members[source]. */
typedef struct {
  const gemel_appearance* members;
  int32_t n_members;
  int32_t source;
} gemel_merge_group;

typedef struct {
  uint64_t weight_arena_bytes;    /* device bytes the weight arena must hold */
  uint64_t act_arena_bytes;       /* device bytes the activation arena must hold */
  uint64_t meta_bytes;            /* device bytes of launch tables (library-allocated) */
  uint64_t unique_weight_bytes;   /* bf16 bytes of distinct (merged) weight tensors */
  uint64_t unmerged_weight_bytes; /* bf16 bytes if nothing were merged */
  int32_t n_levels;               /* scheduler waves */
  int32_t n_launches;             /* kernel launches per gemel_infer */
  int32_t n_gemm_problems;        /* GEMM problems per step */
  int32_t n_union_problems;       /* of which run over >1 model's frames (batch union) */
  int32_t frames_per_step;
  int32_t n_swapped;              /* weight tensors streamed every step (budget mode, a10) */
  double gemm_flops_per_step;     /* algorithmic conv+linear FLOPs (2*MAC) per step */
  uint64_t pinned_weight_bytes;   /* resident weight bytes (all of them without a budget) */
  uint64_t swap_ring_bytes;       /* ring of swap slots in the weight arena (0 = no swap) */
  uint64_t swap_bytes_per_step;   /* host->device weight bytes copied every step */
} gemel_plan_info;

typedef struct {
  int32_t stream_id;
  int32_t n_frames;     /* must equal the planned batch of this stream */
  const uint8_t* frames;/* uint8 [n_frames, in_h, in_w, 3] RGB, HWC */
  int32_t on_host;      /* 1: host memory (pinned for async copies), 0: device.  Device frames
                           may still be in production on the compute stream: the library's
                           ingest copy is ordered after all work already enqueued there. */
  int32_t reserved;
} gemel_stream_batch;

typedef struct {
  int32_t model_id;
  int32_t on_host;      /* 1: host destination, 0: device destination */
  float* out;           /* fp32 [batch, out_features] of the model's last layer */
  uint64_t out_bytes;
} gemel_result;

typedef struct {
  int32_t n_models;
  int32_t n_param_layers;
  int32_t n_merged_layers;      /* param layers bound to another layer's weights */
  int32_t planned;
  uint64_t registered_bytes;    /* bf16 param bytes of all registered layers */
  uint64_t bytes_saved;         /* cumulative over apply_merge calls */
} gemel_stats_t;

typedef struct {
  int32_t dtype;                /* 0 = bf16, 1 = fp32 */
  int32_t n, h, w, c, c_pitch;  /* NHWC, c_pitch >= c elements */
} gemel_value_desc;

typedef struct {
  int32_t kind;                 /* 0 preprocess, 1 gemm, 2 maxpool, 3 avgpool, 4 add, 5 concat/YOLO decode, 6 top-k,
                                   7 rpn level, 8 rpn merge, 9 roi align, 10 box post, 11 det nms,
                                   12 fused frame ingest + first conv (stem) */
  int32_t level;
  int32_t n_problems;
  int32_t reserved;
  double flops;                 /* algorithmic FLOPs of the launch (gemm) */
  double bytes;                 /* algorithmic HBM bytes (activations read+written, weights once) */
} gemel_launch_info;

/* Context lifetime.  create never touches the GPU. */
gemel_status gemel_create(const gemel_options* opt, gemel_ctx* out);
void gemel_destroy(gemel_ctx ctx);
const char* gemel_last_error(gemel_ctx ctx);

/* Validate and copy a model (PAPER.md:292 query registration).  Output shapes
 * are inferred for an in_h x in_w RGB input.  Returns its id (0, 1, ...).
 * GEMEL_E_SCHEMA names the offending op position.  GEMEL_E_STATE after plan. */
gemel_status gemel_register_model(gemel_ctx ctx, const gemel_layer* ops, int32_t n_ops, int32_t stream_id,
                                  int32_t in_h, int32_t in_w, int32_t* model_id);

/* Workload-wide groups of architecturally identical param layers (conv, linear,
 * BN) with >= 2 appearances, sorted by total bytes desc, then per-appearance
 * bytes desc, then first appearance (model, pos) asc.  Appearances of a group
 * are contiguous in apps[] in (model, pos) order.  Two-call sizing: pass
 * cap = 0 to get *n_groups / *n_apps; GEMEL_E_SMALLBUF if a buffer is short. */
gemel_status gemel_find_shareable(gemel_ctx ctx, gemel_group* groups, int32_t cap, int32_t* n_groups,
                                  gemel_appearance* apps, int32_t app_cap, int32_t* n_apps);

/* Bind every member of each group to the weights of its source member.  All or
 * nothing: validation (same signature, n >= 2, valid ids, no member in two
 * groups, no member already merged) precedes any state change.  Merges are
 * cumulative.  *bytes_saved = sum over groups of (n - 1) * per-appearance bytes
 * ("parameter reduction").  GEMEL_E_STATE after plan. */
gemel_status gemel_apply_merge(gemel_ctx ctx, const gemel_merge_group* groups, int32_t n, uint64_t* bytes_saved);

/* Incremental merging planner (§4.2 "Merging Heuristic"; SURVEY.md
 * §8(f) N3).  The pluggable retraining oracle is called with the running merge
 * configuration plus one candidate group (last entry; source 0 = weights of its first
 * member) and returns 1 if every merged model meets its accuracy target within
 * the retraining budget, 0 if not, < 0 to abort (GEMEL_E_ARG).  No training happens
 * in the library. */
typedef int32_t (*gemel_retrain_fn)(void* user, const gemel_merge_group* running, int32_t n_groups);

typedef struct {
  int32_t group;        /* index in gemel_find_shareable's memory-sorted order */
  int32_t n_members;    /* appearances tried: the first n_members of the group's (model, pos)-sorted list */
  int32_t ok;           /* retraining met the accuracy targets: the candidate was bound */
  int32_t reserved;
  uint64_t bytes;       /* per-appearance bytes x n_members */
} gemel_merge_attempt;

/* Run the heuristic on an unmerged workload (GEMEL_E_STATE if any layer is already
 * merged or after plan): groups in find_shareable order, each first with ALL its
 * appearances; on success the candidate is bound through gemel_apply_merge
 * (merges are cumulative) and the next group is tried; on failure the
 * candidate is halved -- its first ceil(n/2) appearances, reading R21 -- and retried
 * if >= 2 appearances remain whose bytes exceed the next group's total, else the
 * group is dropped.  Every retraining attempt is written to log[] (up to
 * log_cap; GEMEL_E_SMALLBUF after the run if it was short); *n_attempts = attempts,
 * *bytes_saved = bytes saved by the accepted groups. */
gemel_status gemel_incremental_merge(gemel_ctx ctx, gemel_retrain_fn retrain, void* user, gemel_merge_attempt* log,
                                     int32_t log_cap, int32_t* n_attempts, uint64_t* bytes_saved);

/* Build the execution plan for a per-stream batch (batch_per_stream[s] frames
 * for stream id s): layer fusion, batch union of shared layers, waves, arena
 * layout.  Requires a CUDA device.  Fills *info (may be NULL). */
gemel_status gemel_plan(gemel_ctx ctx, const int32_t* batch_per_stream, int32_t n_streams, gemel_plan_info* info);

/* Hand the library its device arenas (caller-owned, e.g. torch tensors; at
 * least the planned sizes, 256-byte aligned).  Uploads the merged weights,
 * encodes TMA descriptors, uploads launch tables and captures the step's CUDA
 * graph.  The library never allocates on the hot path. */
gemel_status gemel_bind_arenas(gemel_ctx ctx, void* w_dev, uint64_t w_bytes, void* act_dev, uint64_t act_bytes);

/* Device view of the whole weight arena (for an NCCL broadcast from rank 0,
 * SURVEY.md §8(e)).  Valid after bind. */
gemel_status gemel_weight_view(gemel_ctx ctx, void** dev, uint64_t* bytes);

/* One step: copy each stream's frames in, run every model, copy each model's
 * result out.  Asynchronous on the compute stream (synchronise before reading
 * host results).  n_in must cover every planned stream.  Frames are staged in one
 * of two device buffers, alternating per call, and copied on a library-owned
 * ingest stream as soon as the last step that read that buffer has finished: the
 * copy of step k+1 overlaps the compute of step k.  Frame buffers must stay valid
 * until the compute stream has completed the step. */
gemel_status gemel_infer(gemel_ctx ctx, const gemel_stream_batch* in, int32_t n_in, gemel_result* out, int32_t n_out);

/* Inspection (tests): copy a stored intermediate value -- the output of op
 * op_pos of a model, as the device stores it -- to host memory (synchronous).
 * Values fused into a producer's epilogue are not stored: GEMEL_E_ARG. */
gemel_status gemel_read_value(gemel_ctx ctx, int32_t model_id, int32_t op_pos, void* host_dst, uint64_t bytes,
                              gemel_value_desc* desc);

/* Per-launch CUDA-event timing of the next gemel_infer calls (no graph). */
gemel_status gemel_set_profiling(gemel_ctx ctx, int32_t enable);
/* Launch list of the plan and the last profiled step's per-launch times (ms). */
gemel_status gemel_launch_list(gemel_ctx ctx, gemel_launch_info* info, float* ms, int32_t cap, int32_t* n);

gemel_status gemel_stats(gemel_ctx ctx, gemel_stats_t* out);

/* The plan as JSON text: scheduler levels, launches with their GEMM problems
 * (members as [model, op], M, N, K, tile shape) and nodes (layers each node
 * covers, input values, level) -- for inspection and the oracle's plan
 * validator.  Two-call sizing: buf = NULL returns the size (incl. NUL) in *len. */
gemel_status gemel_plan_dump(gemel_ctx ctx, char* buf, uint64_t cap, uint64_t* len);

#ifdef __cplusplus
}
#endif
#endif /* GEMEL_H */
