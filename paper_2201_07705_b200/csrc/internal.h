// Internal state of a gemel context (host side).
#pragma once
#include <cstdint>
#include <functional>
#include <map>
#include <string>
#include <vector>

#include "../../include/gemel.h"
#include "kernels/gemm.h"
#include "kernels/memops.h"
#include "kernels/stem.h"

namespace gemel {

struct Layer {
  gemel_layer d{};          // hyperparameters (param pointers cleared)
  int C = 0, H = 0, W = 0;  // output shape per image (linear/flatten: C features, H = W = 1)
  int inC = 0, inH = 0, inW = 0;  // input shape of in[0]
  int param_id = -1;        // index into Ctx::params (conv/linear/bn)
  bool flat = false;        // output is a flat feature vector (linear, flatten, YOLO decode)
  int rows = 1;             // values per frame (ROI_ALIGN and its consumers: one per proposal)
  int tie = -1;             // CONV2D applying op `tie`'s parameters (-1: its own)
  std::vector<float> anchors;  // YOLO_DECODE: [A][2] (w, h) pixels
};

struct Model {
  std::vector<Layer> layers;
  int stream_id = 0, in_h = 0, in_w = 0;
};

// Host copy of one param layer's parameters (fp32, as registered).
struct ParamLayer {
  int model = 0, pos = 0, op = 0;
  std::vector<float> w, b;                  // conv/linear
  std::vector<float> gamma, beta, mean, var;  // bn
  uint64_t bytes = 0;                       // bf16 accounting bytes
  int bound_to = -1;                        // merged: param id of the source (-1: itself)
  int merge_group = -1;
};

// ---------------------------------------------------------------- plan
struct Value {
  int model = -1, pos = -1;     // pos -1: preprocessed model input
  int C = 0, H = 0, W = 0, Cp = 0, B = 0;
  bool fp32 = false;
  bool virt = false;            // never materialised: the im2col input of a fused first conv (stem launch)
  uint64_t bytes = 0;
  int slab = -1;                // slab id (contiguous group) or -1 (singleton)
  uint64_t offset = 0;          // byte offset in the activation arena
  int producer = -1;            // node id
};

enum NodeKind { NK_PRE = 0, NK_GEMM = 1, NK_MAXPOOL = 2, NK_AVGPOOL = 3, NK_ADD = 4, NK_MISC = 5, NK_TOPK = 6,
                NK_RPN = 7, NK_RPNM = 8, NK_ROI = 9, NK_BOXP = 10,   // Faster R-CNN stages (detect.cu)
                NK_NMS = 11 };                                        // final detection NMS (detect.cu)
enum MiscKind { MISC_CONCAT = 0, MISC_YOLO = 1, MISC_L2NORM = 2, MISC_SSD = 3, MISC_DETC = 4 };

struct Node {
  int kind = NK_GEMM;
  int model = -1;
  int layer = -1;               // conv/linear (gemm), pool/add layer, -1 for PRE
  int bn = -1, add = -1, act_layer = -1;
  int res_post = 0;             // gemm: residual added after the activation (darknet shortcut)
  int res_up = 1;               // gemm: residual read nearest-upsampled by this factor (FPN)
  int up_layer = -1;            // gemm: the UPSAMPLE layer fused into that residual read
  int act = ACT_NONE;
  float slope = 0.f;
  int in_value = -1, in_value2 = -1, res_value = -1, out_value = -1;
  int wkey = -1;                // device weight tensor id (gemm)
  // gemm geometry
  int Cin = 0, Cp_in = 0, H = 0, W = 0, Cout = 0, Ho = 0, Wo = 0;
  int kh = 1, kw = 1, sh = 1, sw = 1, ph = 0, pw = 0, dh = 1, dw = 1;
  int B = 0;
  int cols = 0;                 // gemm: input is the im2col matrix of the model input (first conv)
  int stem = 0;                 // gemm (cols): fused ingest + conv in a stem launch (stem_sm100.cu);
                                // PRE: the im2col node of such a conv (no work, its value is virtual)
  int problem = -1;             // problem id
  int level = -1;
  double flops = 0;
  uint64_t scale_off = 0, shift_off = 0;   // weight-arena offsets of epilogue vectors
  // NK_MISC: concat pieces (value, nearest-upsample factor) or one YOLO decode
  int misc = MISC_CONCAT;
  std::vector<int> ins, in_scale;
  int64_t out_off = 0;          // YOLO: element offset of this head in the output row
};

struct DevWeight {              // one device weight matrix [N, Ktot] bf16 (merged: shared)
  int param_id = -1;            // source param layer
  int flatC = 0, flatH = 1, flatW = 1, flatCp = 0;  // linear: pre-flatten shape (NHWC permutation)
  int N = 0, Ktot = 0, cin_k = 0, chunk = 64, kh = 1, kw = 1, Cin = 0;
  bool linear = false;
  bool cols = false;            // K = (r, s, c) over the 3 frame channels, dense
  uint64_t offset = 0, bytes = 0;
  // weight residency under a budget: swapped tensors live in a
  // ring slot of the weight arena and are copied from pinned host memory every step
  bool swapped = false;
  int first_launch = -1, last_launch = -1;   // launches that read it
  int wait_launch = -1;         // its copy waits for this launch (previous slot occupant's last use)
  int copy_order = -1;
};

struct Problem {                // one GEMM problem (possibly a batch union)
  std::vector<int> members;     // gemm node ids, model order
  int wkey = -1;
  int level = -1;
  int in_value_first = -1;      // first member's input value (slab start)
  int n_img = 0;
  int bn = 0;
  int ksplit = 1, kst_split = 0;  // split-K (deterministic fixed-order reduction)
  int run = 1;                  // consecutive tiles per tile-queue grab (cheap tiles, many waves)
  int msub = 1;                 // 128-row sub-tiles per tile (skinny problems)
  uint64_t ws_off = 0;          // activation-arena offset of the split-K partials
  int tcnt_idx = 0;             // index of its per-(m, n) tile counters in the launch counter block
  int cnt_off = 0;              // index of its per-m-tile completion counters in the launch counter block
  int m_tiles = 0;
  uint64_t dep_idx = 0;         // first int32 of its [m_tiles][n_deps][lo, hi] dependency ranges
};

struct Launch {
  int kind = NK_GEMM;
  int level = 0;
  std::vector<int> items;       // problem ids (gemm) or node ids (others)
  double flops = 0, bytes = 0;
  // device tables
  uint64_t meta_off = 0;        // offset of problem table in meta buffer
  uint64_t seg_off = 0;
  uint64_t cnt_off = 0;         // scheduler counters: [0] next tile, then per problem one completion
                                // counter per m-tile, then split-K per-tile arrival counters
  uint64_t dep_off = 0;         // per-m-tile dependency ranges of the launch's problems
  int n_counters = 0;
  std::vector<std::vector<int>> deps;   // per problem (launch-local indices)
  int n_probs = 0, total_tiles = 0, total_items = 0, bn_max = 0, stages = 0, grid = 0;
  int cg = 1;                   // GEMM: 2 = CTA-pair kernel (256-row tiles, cta_group::2)
  int stem = 0;                 // GEMM: fused first-conv launch (stem_kernel over StemTasks, no GemmProblems)
  int stem_tasks = 0, stem_n_max = 0, stem_kp_max = 0;
  int64_t stem_tiles = 0;
  uint64_t stem_off = 0;        // meta offset of the stem launch's StemTask tables (one per staging buffer)
  int acc_w = 256;              // GEMM: TMEM columns per accumulator (max msub x bn)
  int epi_flags = 0;            // GEMM: GemmLaunch::epi_flags
  // frame ingest: im2col tasks first (block prefix), then NHWC tasks (pixel prefix)
  int n_cols = 0, cols_smem = 0, n_pre_tasks = 0;
  int64_t cols_blocks = 0, pre_pixels = 0;
  // concat / YOLO decode (NK_MISC): task count and total work items
  int misc_tasks = 0;
  int64_t misc_work = 0;
  int topk_blocks = 0, topk_rows = 0;   // NK_TOPK: frames and the largest row count (NK_RPN: anchors)
  int det_blocks = 0;                   // NK_RPN / NK_RPNM: CTAs (frames)
  int64_t det_work = 0;                 // NK_ROI: threads; NK_BOXP: warps
};

struct Ctx {
  gemel_options opt{};
  std::string err;
  std::vector<Model> models;
  std::vector<ParamLayer> params;
  uint64_t bytes_saved = 0;
  int n_merge_groups = 0;
  bool planned = false, bound = false;
  // plan
  std::vector<int> batch;                 // per stream
  std::vector<Value> values;
  std::map<std::pair<int, int>, int> value_of;   // (model, pos) -> value id
  std::vector<Node> nodes;
  std::vector<DevWeight> dweights;
  std::vector<Problem> problems;
  std::vector<Launch> launches;
  std::vector<int64_t> frame_off;         // per stream: u8 staging offset in act arena (buffer 0)
  std::vector<int64_t> frame_off2;        // per stream: the second staging buffer (double-buffered ingest)
  int n_levels = 0;
  // weight swap (budget mode)
  uint64_t pinned_bytes = 0, ring_off = 0, ring_bytes = 0, swap_bytes = 0;
  std::vector<int> swap_order;            // swapped dweight ids in copy order
  std::vector<void*> host_w;              // bound: paging source per swapped dweight (pinned host,
                                          // or device memory on opt.source_device for GEMEL_SOURCE_PEER)
  void* copy_stream = nullptr;            // bound: cudaStream_t for swap copies
  std::vector<void*> swap_events;         // bound: per launch: done, ready (+1 start)
  uint64_t w_bytes = 0, act_bytes = 0, meta_bytes = 0;
  uint64_t unique_weight_bytes = 0, unmerged_weight_bytes = 0;
  double gemm_flops = 0;
  // bound
  uint8_t* w_dev = nullptr;
  uint8_t* act_dev = nullptr;
  uint8_t* meta_dev = nullptr;
  void* graph_exec = nullptr;             // cudaGraphExec_t reading staging buffer 0
  void* graph_exec2 = nullptr;            // the same step reading staging buffer 1
  void* in_stream = nullptr;              // frame copies of the next step overlap this step's compute
  void* in_ready[2] = {nullptr, nullptr}; // frames of buffer b landed
  void* buf_free[2] = {nullptr, nullptr}; // the last step reading buffer b finished
  void* dev_frames_ready = nullptr;       // caller's compute-stream work before device-resident frames
  int parity = 0;
  bool profiling = false;
  int sm_count = 148;                     // SMs of the device (queried at plan; 148 for a dry plan)
  bool sync_each = false;                 // developer: synchronise after every profiled launch
  int gemm_dbg = 0;                       // developer probes (GEMEL_GEMM_DBG at bind; needs -DGEMEL_DEV_PROBES)
  std::vector<float> launch_ms;
  std::vector<void*> events;              // cudaEvent_t pairs
  std::vector<void*> trace_dev;           // GEMEL_TRACE_DIR: per-launch tile timestamp buffers
  std::string trace_path;
};

int set_err(Ctx* c, int code, const std::string& msg);
int plan_swap(Ctx* c, const std::function<void(Launch&, int)>& gemm_cost);
int build_plan(Ctx* c);
int bind(Ctx* c, void* w, uint64_t wb, void* a, uint64_t ab);
int run_step(Ctx* c, const gemel_stream_batch* in, int n_in, gemel_result* out, int n_out);
void release_device(Ctx* c);

inline uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }
inline int round_up(int x, int a) { return (x + a - 1) / a * a; }

}  // namespace gemel
