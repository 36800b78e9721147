// Step planner: layer fusion, batch union of merged
// layers, scheduler waves, arena layout.  Host-only, integer work.
//
//  * Fusion: conv|linear -> [bn] -> [add (as first operand)] -> [relu|leaky]
//    becomes ONE GEMM node whose epilogue applies the member's folded BN,
//    residual and activation (reading R7).
//  * Batch union: GEMM nodes of different models bound to the same merged
//    weight (gemel_apply_merge) with the same input geometry are aligned by an
//    order-preserving weighted LCS (progressive over models: a common
//    supersequence, so the contracted graph stays acyclic) and run as one
//    problem over the concatenation of their input slabs.  PAPER.md:399 asks
//    that models sharing layers be adjacent in the load order; on B200 the
//    shared layer's members are fused into one launch instead.
//  * Waves: ASAP levels of the contracted DAG; per level one grouped GEMM
//    launch plus one grouped launch per memory-bound op kind.
//  * Layout: every stored value gets its own region in the activation arena
//    (union inputs/outputs as contiguous slabs in model order); merged weights
//    are stored once in the weight arena.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <functional>
#include <map>
#include <sstream>
#include <tuple>

#include "internal.h"

namespace gemel {

namespace {

int chunk_for(int cp) {
  if (cp >= 64) return 64;
  int c = 8;
  while (c < cp) c <<= 1;
  return c;
}

struct Col {
  int wkey;
  std::tuple<int, int, int> geom;
  std::vector<int> nodes;   // node ids (one per model at most)
};

}  // namespace

int build_plan(Ctx* c) {
  c->values.clear();
  c->value_of.clear();
  c->nodes.clear();
  c->dweights.clear();
  c->problems.clear();
  c->launches.clear();
  c->frame_off.clear();
  std::ostringstream err;

  // ------------------------------------------------------------ 1. fusion
  // First convolutions over the 3-channel frame run fused with the frame ingest
  // (stem_sm100.cu: im2col rows built in shared memory, never in HBM) when their
  // output fits one tcgen05 N tile and the padded K <= 256 (GEMEL_STEM=0: the unfused
  // ingest-written im2col + grouped GEMM path)
  // GEMEL_STEM: 1 (default) fused stem kernel, 0 ingest-written im2col + grouped GEMM, 2 NHWC8 frame +
  // TMA im2col in the grouped GEMM (8-channel boxes)
  const int stem_mode = std::getenv("GEMEL_STEM") ? std::atoi(std::getenv("GEMEL_STEM")) : 1;
  const bool stem_fuse = stem_mode == 1;
  std::vector<std::vector<int>> gemm_seq(c->models.size());
  std::vector<int> model_out_value(c->models.size(), -1);
  for (int mi = 0; mi < int(c->models.size()); ++mi) {
    const Model& M = c->models[mi];
    if (M.stream_id >= int(c->batch.size()) || c->batch[M.stream_id] <= 0)
      return set_err(c, GEMEL_E_ARG, "plan: no batch for stream of model " + std::to_string(mi));
    const int B = c->batch[M.stream_id];
    const int n = int(M.layers.size());
    std::vector<std::vector<int>> cons(n);
    for (int i = 0; i < n; ++i)
      for (int k = 0; k < M.layers[i].d.n_in; ++k)
        if (M.layers[i].d.in[k] >= 0) cons[M.layers[i].d.in[k]].push_back(i);
    auto sole = [&](int i) { return cons[i].size() == 1 ? cons[i][0] : -1; };

    // Frame ingest.  When only convolutions read the frame, the ingest kernel
    // writes each such conv's im2col matrix directly (K = kh*kw*3 is far too
    // narrow for efficient TMA im2col boxes); otherwise NHWC with C padded to 8.
    bool input_cols = stem_mode != 2;
    for (int i = 0; i < n; ++i)
      for (int k = 0; k < M.layers[i].d.n_in; ++k)
        if (M.layers[i].d.in[k] == -1 && M.layers[i].d.op != GEMEL_OP_CONV2D) input_cols = false;
    int vin_id = -1;
    if (!input_cols) {
      Value vin;
      vin.model = mi; vin.pos = -1; vin.C = 3; vin.H = M.in_h; vin.W = M.in_w; vin.Cp = 8; vin.B = B;
      vin.bytes = uint64_t(B) * vin.H * vin.W * vin.Cp * 2;
      vin_id = int(c->values.size());
      c->values.push_back(vin);
      c->value_of[{mi, -1}] = vin_id;
      Node pre;
      pre.kind = NK_PRE; pre.model = mi; pre.out_value = vin_id; pre.B = B;
      c->values[vin_id].producer = int(c->nodes.size());
      c->nodes.push_back(pre);
    }

    std::map<int, int> alias;   // flatten pos -> value id
    auto val = [&](int pos) -> int {
      if (pos < 0) return vin_id;
      auto a = alias.find(pos);
      if (a != alias.end()) return a->second;
      auto it = c->value_of.find({mi, pos});
      return it == c->value_of.end() ? -1 : it->second;
    };
    auto new_value = [&](int pos, int C, int H, int W, bool fp32) {
      Value v;
      v.model = mi; v.pos = pos; v.C = C; v.H = H; v.W = W; v.Cp = round_up(C, 8); v.fp32 = fp32;
      v.B = B * (pos >= 0 ? M.layers[pos].rows : 1);   // ROI_ALIGN and after: one value per proposal
      v.bytes = uint64_t(v.B) * H * W * v.Cp * (fp32 ? 4 : 2);
      const int id = int(c->values.size());
      c->values.push_back(v);
      c->value_of[{mi, pos}] = id;
      return id;
    };

    std::vector<char> covered(n, 0);
    // A model whose last layer concatenates YOLO decodes: every decode writes its
    // boxes straight into that fp32 detection row at its own offset (no copy).
    std::map<int, std::pair<int, int64_t>> yolo_dst;   // yolo pos -> (value, element offset)
    auto is_decode = [&](int j) {
      return j >= 0 && (M.layers[j].d.op == GEMEL_OP_YOLO_DECODE || M.layers[j].d.op == GEMEL_OP_SSD_DECODE ||
                        M.layers[j].d.op == GEMEL_OP_RPN_LEVEL || M.layers[j].d.op == GEMEL_OP_BOX_POST);
    };
    for (int ci = 0; ci < n; ++ci) {
      const Layer& Ll = M.layers[ci];
      bool all_yolo = Ll.d.op == GEMEL_OP_CONCAT;
      for (int k = 0; all_yolo && k < Ll.d.n_in; ++k)
        all_yolo = is_decode(Ll.d.in[k]) && cons[Ll.d.in[k]].size() == 1;
      if (!all_yolo) continue;
      const int ov = new_value(ci, Ll.C, 1, 1, true);
      int64_t off = 0;
      for (int k = 0; k < Ll.d.n_in; ++k) {
        yolo_dst[Ll.d.in[k]] = {ov, off};
        off += M.layers[Ll.d.in[k]].C;
      }
      covered[ci] = 1;
    }
    auto feeds_only_yolo = [&](int i) {   // a detector head: stored fp32 for its decode
      if (cons[i].empty()) return false;
      for (int j : cons[i])
        if (!is_decode(j)) return false;
      return true;
    };
    for (int i = 0; i < n; ++i) {
      if (covered[i]) continue;
      const Layer& L = M.layers[i];
      const int op = L.d.op;
      const std::string at = "plan: model " + std::to_string(mi) + " op " + std::to_string(i) + ": ";
      if (op == GEMEL_OP_FLATTEN) {
        const int v = val(L.d.in[0]);
        alias[i] = v;
        covered[i] = 1;
        continue;
      }
      if (op == GEMEL_OP_CONV2D || op == GEMEL_OP_LINEAR) {
        Node g;
        g.kind = NK_GEMM; g.model = mi; g.layer = i; g.B = B * L.rows;
        int cur = i;
        covered[i] = 1;
        int j = sole(cur);
        if (j >= 0 && M.layers[j].d.op == GEMEL_OP_BATCHNORM2D) { g.bn = j; cur = j; covered[j] = 1; j = sole(cur); }
        auto is_residual_add = [&](int a, int x) {
          if (a < 0 || covered[a] || M.layers[a].d.op != GEMEL_OP_ADD) return false;
          const int* in = M.layers[a].d.in;
          return (in[0] == x) != (in[1] == x);   // x is exactly one operand
        };
        if (is_residual_add(j, cur)) {
          g.add = j; cur = j; covered[j] = 1;
          // the residual's producer may come later in the list (e.g. a downsample
          // branch): resolved after all of this model's values exist
          j = sole(cur);
        }
        if (j >= 0 && (M.layers[j].d.op == GEMEL_OP_RELU || M.layers[j].d.op == GEMEL_OP_LEAKY_RELU)) {
          g.act_layer = j; cur = j; covered[j] = 1;
          g.act = M.layers[j].d.op == GEMEL_OP_RELU ? ACT_RELU : ACT_LEAKY;
          g.slope = M.layers[j].d.neg_slope;
          // darknet shortcut: conv -> bn -> leaky -> add, the residual after the activation
          const int a = sole(cur);
          if (g.add < 0 && is_residual_add(a, cur)) {
            g.add = a; g.res_post = 1; cur = a; covered[a] = 1;
          }
        }
        g.Cout = L.d.cout;
        if (op == GEMEL_OP_CONV2D && L.d.in[0] == -1 && input_cols) {
          // im2col matrix written by the ingest kernel: a dense [B*Ho*Wo, K] GEMM
          Value cv;
          cv.model = mi; cv.pos = -2 - i; cv.C = L.d.kh * L.d.kw * L.d.cin; cv.H = L.H; cv.W = L.W;
          cv.Cp = round_up(cv.C, 8); cv.B = B;
          const bool fuse = stem_fuse && L.d.cin == 3 && L.d.cout % 16 == 0 && L.d.cout <= 128 &&
                            stem_kp(L.d.kh, L.d.kw) <= 256 && L.d.dh == 1 && L.d.dw == 1;
          cv.virt = fuse;
          cv.bytes = fuse ? 0 : uint64_t(B) * cv.H * cv.W * cv.Cp * 2;
          const int cid = int(c->values.size());
          c->values.push_back(cv);
          c->value_of[{mi, -2 - i}] = cid;
          if (!c->value_of.count({mi, -1})) c->value_of[{mi, -1}] = cid;
          Node pre;
          pre.kind = NK_PRE; pre.model = mi; pre.layer = i; pre.out_value = cid; pre.B = B;
          pre.stem = fuse ? 1 : 0;
          c->values[cid].producer = int(c->nodes.size());
          c->nodes.push_back(pre);
          g.in_value = cid;
          g.cols = 1;
          g.stem = fuse ? 1 : 0;
          g.Cin = cv.C; g.Cp_in = cv.Cp; g.H = 1; g.W = 1;
          g.Ho = L.H; g.Wo = L.W;
          g.flops = 2.0 * B * g.Ho * g.Wo * double(g.Cout) * g.Cin;
          const bool last = (cur == n - 1) || feeds_only_yolo(cur);
          const Layer& Lc = M.layers[cur];
          g.out_value = new_value(cur, Lc.C, Lc.H, Lc.W, last);
          c->values[g.out_value].producer = int(c->nodes.size());
          gemm_seq[mi].push_back(int(c->nodes.size()));
          c->nodes.push_back(g);
          continue;
        }
        g.in_value = val(L.d.in[0]);
        if (g.in_value < 0) return set_err(c, GEMEL_E_UNSUPPORTED, at + "input not materialised");
        const Value& vi = c->values[g.in_value];
        if (op == GEMEL_OP_CONV2D) {
          g.Cin = L.d.cin; g.Cp_in = vi.Cp; g.H = vi.H; g.W = vi.W;
          g.kh = L.d.kh; g.kw = L.d.kw; g.sh = L.d.sh; g.sw = L.d.sw; g.ph = L.d.ph; g.pw = L.d.pw;
          g.dh = L.d.dh; g.dw = L.d.dw;
          g.Ho = L.H; g.Wo = L.W;
          if (vi.fp32) return set_err(c, GEMEL_E_UNSUPPORTED, at + "fp32 input to conv");
        } else {
          // linear over a (possibly flattened) NHWC value: K = H*W*Cp in NHWC order
          g.Cin = L.d.cin; g.Cp_in = vi.H * vi.W * vi.Cp; g.H = 1; g.W = 1; g.Ho = 1; g.Wo = 1;
          if (vi.fp32) return set_err(c, GEMEL_E_UNSUPPORTED, at + "fp32 input to linear");
        }
        if (g.ph > 127 || g.pw > 127 || (g.kh - 1) * g.dh > 127 || (g.kw - 1) * g.dw > 127 || g.sh > 8 || g.sw > 8)
          return set_err(c, GEMEL_E_UNSUPPORTED, at + "conv geometry outside TMA im2col limits");
        g.flops = 2.0 * B * g.Ho * g.Wo * double(g.Cout) * g.kh * g.kw * g.Cin;
        const bool last = (cur == n - 1) || feeds_only_yolo(cur);
        const Layer& Lc = M.layers[cur];
        g.out_value = new_value(cur, Lc.C, Lc.H, Lc.W, last);
        c->values[g.out_value].producer = int(c->nodes.size());
        gemm_seq[mi].push_back(int(c->nodes.size()));
        c->nodes.push_back(g);
        continue;
      }
      if (op == GEMEL_OP_UPSAMPLE_NEAREST) {
        // fused into its consumer concat (the piece is read with the scale factor);
        // standalone it becomes a one-piece concat
        const int u = sole(i);
        if (u >= 0 && M.layers[u].d.op == GEMEL_OP_CONCAT && !M.layers[u].flat) { covered[i] = 1; continue; }
        // read nearest-upsampled by a GEMM whose epilogue adds it as the residual (FPN
        // top-down: lateral conv + up(coarser level)); the add was fused when its conv
        // (an earlier op) was planned
        if (u >= 0 && M.layers[u].d.op == GEMEL_OP_ADD && covered[u] && !M.layers[L.d.in[0]].flat) {
          covered[i] = 1;
          continue;
        }
      }
      if (op == GEMEL_OP_UPSAMPLE_NEAREST || (op == GEMEL_OP_CONCAT && !L.flat)) {
        Node m;
        m.kind = NK_MISC; m.misc = MISC_CONCAT; m.model = mi; m.layer = i; m.B = B;
        const int npieces = op == GEMEL_OP_CONCAT ? L.d.n_in : 1;
        for (int k = 0; k < npieces; ++k) {
          int src = op == GEMEL_OP_CONCAT ? L.d.in[k] : i, scale = 1;
          if (src >= 0 && M.layers[src].d.op == GEMEL_OP_UPSAMPLE_NEAREST) {
            scale = M.layers[src].d.sh;
            src = M.layers[src].d.in[0];
          }
          const int v = val(src);
          if (v < 0 || c->values[v].fp32 || c->values[v].C % 8)
            return set_err(c, GEMEL_E_UNSUPPORTED, at + "concat piece must be a stored bf16 value with C % 8 == 0");
          m.ins.push_back(v);
          m.in_scale.push_back(scale);
        }
        m.in_value = m.ins[0];
        if (i == n - 1) return set_err(c, GEMEL_E_UNSUPPORTED, at + "model must end in a conv/linear chain");
        m.out_value = new_value(i, L.C, L.H, L.W, false);
        c->values[m.out_value].producer = int(c->nodes.size());
        covered[i] = 1;
        c->nodes.push_back(m);
        continue;
      }
      if (op == GEMEL_OP_L2NORM) {
        Node m;
        m.kind = NK_MISC; m.misc = MISC_L2NORM; m.model = mi; m.layer = i; m.B = B;
        m.in_value = val(L.d.in[0]);
        if (m.in_value < 0 || c->values[m.in_value].fp32 || c->values[m.in_value].C % 8)
          return set_err(c, GEMEL_E_UNSUPPORTED, at + "l2norm input must be a stored bf16 value with C % 8 == 0");
        m.ins = {m.in_value};
        m.in_scale = {1};
        m.Cout = L.C;
        m.out_value = new_value(i, L.C, L.H, L.W, false);
        c->values[m.out_value].producer = int(c->nodes.size());
        covered[i] = 1;
        c->nodes.push_back(m);
        continue;
      }
      if (op == GEMEL_OP_SSD_DECODE) {
        Node m;
        m.kind = NK_MISC; m.misc = MISC_SSD; m.model = mi; m.layer = i; m.B = B;
        const int vl = val(L.d.in[0]), vc = val(L.d.in[1]);
        if (vl < 0 || vc < 0 || !c->values[vl].fp32 || !c->values[vc].fp32)
          return set_err(c, GEMEL_E_UNSUPPORTED, at + "ssd decode inputs must be conv heads (fp32)");
        m.in_value = vl;
        m.ins = {vl, vc};
        m.in_scale = {1, 1};
        auto d = yolo_dst.find(i);
        if (d != yolo_dst.end()) {
          m.out_value = d->second.first;
          m.out_off = d->second.second;
        } else {
          if (i != n - 1) return set_err(c, GEMEL_E_UNSUPPORTED, at + "ssd decode must feed the detection output");
          m.out_value = new_value(i, L.C, 1, 1, true);
        }
        c->values[m.out_value].producer = int(c->nodes.size());
        covered[i] = 1;
        c->nodes.push_back(m);
        continue;
      }
      if (op == GEMEL_OP_RPN_LEVEL || op == GEMEL_OP_RPN_MERGE || op == GEMEL_OP_ROI_ALIGN || op == GEMEL_OP_BOX_POST) {
        Node m;
        m.kind = op == GEMEL_OP_RPN_LEVEL ? NK_RPN : op == GEMEL_OP_RPN_MERGE ? NK_RPNM : op == GEMEL_OP_ROI_ALIGN ? NK_ROI
                                                                                                       : NK_BOXP;
        m.model = mi; m.layer = i; m.B = B;
        for (int k = 0; k < L.d.n_in; ++k) {
          const int v = val(L.d.in[k]);
          if (v < 0) return set_err(c, GEMEL_E_UNSUPPORTED, at + "detector stage input not materialised");
          // heads / proposals / class rows are fp32; ROI_ALIGN's feature maps bf16
          const bool want32 = !(op == GEMEL_OP_ROI_ALIGN && k > 0);
          if (c->values[v].fp32 != want32)
            return set_err(c, GEMEL_E_UNSUPPORTED, at + "detector stage input has the wrong storage type");
          m.ins.push_back(v);
          m.in_scale.push_back(1);
        }
        m.in_value = m.ins[0];
        if (i == n - 1) return set_err(c, GEMEL_E_UNSUPPORTED, at + "model must end in a conv/linear chain or top-k");
        m.out_value = new_value(i, L.C, L.H, L.W, op != GEMEL_OP_ROI_ALIGN);
        c->values[m.out_value].producer = int(c->nodes.size());
        covered[i] = 1;
        c->nodes.push_back(m);
        continue;
      }
      if (op == GEMEL_OP_DET_CANDIDATES || op == GEMEL_OP_DET_NMS) {   // final detections (N2, detect.cu)
        Node m;
        m.kind = op == GEMEL_OP_DET_NMS ? NK_NMS : NK_MISC;
        m.misc = MISC_DETC;
        m.model = mi; m.layer = i; m.B = B;
        m.in_value = val(L.d.in[0]);
        if (m.in_value < 0 || !c->values[m.in_value].fp32)
          return set_err(c, GEMEL_E_UNSUPPORTED, at + "detection post-processing input must be fp32 rows");
        m.ins.push_back(m.in_value);
        m.in_scale.push_back(1);
        m.out_value = new_value(i, L.C, 1, 1, true);
        c->values[m.out_value].producer = int(c->nodes.size());
        covered[i] = 1;
        c->nodes.push_back(m);
        continue;
      }
      if (op == GEMEL_OP_TOPK) {
        Node m;
        m.kind = NK_TOPK; m.model = mi; m.layer = i; m.B = B;
        m.in_value = val(L.d.in[0]);
        if (m.in_value < 0 || !c->values[m.in_value].fp32)
          return set_err(c, GEMEL_E_UNSUPPORTED, at + "topk input must be an fp32 detection row");
        if (c->values[m.in_value].C / L.d.cin > (1 << 24))
          return set_err(c, GEMEL_E_UNSUPPORTED, at + "topk over more than 2^24 rows per frame");
        m.out_value = new_value(i, L.C, 1, 1, true);
        c->values[m.out_value].producer = int(c->nodes.size());
        covered[i] = 1;
        c->nodes.push_back(m);
        continue;
      }
      if (op == GEMEL_OP_YOLO_DECODE) {
        Node m;
        m.kind = NK_MISC; m.misc = MISC_YOLO; m.model = mi; m.layer = i; m.B = B;
        m.in_value = val(L.d.in[0]);
        if (m.in_value < 0 || !c->values[m.in_value].fp32)
          return set_err(c, GEMEL_E_UNSUPPORTED, at + "yolo decode input must be a conv head (fp32)");
        m.ins = {m.in_value};
        m.in_scale = {1};
        auto d = yolo_dst.find(i);
        if (d != yolo_dst.end()) {
          m.out_value = d->second.first;
          m.out_off = d->second.second;
        } else {
          if (i != n - 1) return set_err(c, GEMEL_E_UNSUPPORTED, at + "yolo decode must feed the detection output");
          m.out_value = new_value(i, L.C, 1, 1, true);
        }
        c->values[m.out_value].producer = int(c->nodes.size());
        covered[i] = 1;
        c->nodes.push_back(m);
        continue;
      }
      if (op == GEMEL_OP_MAXPOOL2D || op == GEMEL_OP_ADAPTIVE_AVGPOOL2D) {
        Node p;
        p.kind = op == GEMEL_OP_MAXPOOL2D ? NK_MAXPOOL : NK_AVGPOOL;
        p.model = mi; p.layer = i; p.B = B;
        p.in_value = val(L.d.in[0]);
        if (p.in_value < 0 || c->values[p.in_value].fp32)
          return set_err(c, GEMEL_E_UNSUPPORTED, at + "pool input not a stored bf16 value");
        if (i == n - 1) return set_err(c, GEMEL_E_UNSUPPORTED, at + "model must end in a conv/linear chain");
        p.out_value = new_value(i, L.C, L.H, L.W, false);
        c->values[p.out_value].producer = int(c->nodes.size());
        covered[i] = 1;
        c->nodes.push_back(p);
        continue;
      }
      if (op == GEMEL_OP_ADD) {
        Node a;
        a.kind = NK_ADD; a.model = mi; a.layer = i; a.B = B;
        a.in_value = val(L.d.in[0]);
        a.in_value2 = val(L.d.in[1]);
        if (a.in_value < 0 || a.in_value2 < 0) return set_err(c, GEMEL_E_UNSUPPORTED, at + "add operand not stored");
        covered[i] = 1;
        int cur = i, j = sole(i);
        if (j >= 0 && (M.layers[j].d.op == GEMEL_OP_RELU || M.layers[j].d.op == GEMEL_OP_LEAKY_RELU)) {
          a.act = M.layers[j].d.op == GEMEL_OP_RELU ? ACT_RELU : ACT_LEAKY;
          a.slope = M.layers[j].d.neg_slope;
          covered[j] = 1;
          cur = j;
        }
        if (cur == n - 1) return set_err(c, GEMEL_E_UNSUPPORTED, at + "model must end in a conv/linear chain");
        a.out_value = new_value(cur, L.C, L.H, L.W, false);
        c->values[a.out_value].producer = int(c->nodes.size());
        c->nodes.push_back(a);
        continue;
      }
      return set_err(c, GEMEL_E_UNSUPPORTED, at + "op not fusable into a supported kernel (standalone BN/activation)");
    }
    for (int nid : gemm_seq[mi]) {
      Node& g = c->nodes[nid];
      if (g.add < 0) continue;
      const int* ain = M.layers[g.add].d.in;
      const int chain_end = g.res_post ? g.act_layer : (g.bn >= 0 ? g.bn : g.layer);
      const int other = ain[0] == chain_end ? ain[1] : ain[0];
      if (other >= 0 && M.layers[other].d.op == GEMEL_OP_UPSAMPLE_NEAREST && val(other) < 0) {
        g.res_value = val(M.layers[other].d.in[0]);   // fused nearest upsample of the residual
        g.res_up = M.layers[other].d.sh;
        g.up_layer = other;
      } else {
        g.res_value = val(other);
      }
      if (g.res_value < 0)
        return set_err(c, GEMEL_E_UNSUPPORTED, "plan: model " + std::to_string(mi) + " op " +
                                                   std::to_string(g.add) + ": residual operand not materialised");
    }
    // chain ends are after all their inputs (incl. residuals): ordering by
    // output position gives a topological order of the model's GEMM nodes
    std::sort(gemm_seq[mi].begin(), gemm_seq[mi].end(),
              [&](int a, int b) { return c->values[c->nodes[a].out_value].pos < c->values[c->nodes[b].out_value].pos; });
    model_out_value[mi] = val(n - 1);
    if (model_out_value[mi] < 0 || !c->values[model_out_value[mi]].fp32)
      return set_err(c, GEMEL_E_UNSUPPORTED, "plan: model " + std::to_string(mi) + " must end in a conv/linear chain");
  }

  // ------------------------------------------------------------ 2. device weights (merged: one copy)
  std::map<std::tuple<int, int, int, int, int>, int> wkey_of;
  for (auto& g : c->nodes) {
    if (g.kind != NK_GEMM) continue;
    const Layer& L = c->models[g.model].layers[g.layer];
    const ParamLayer& P = c->params[L.param_id];
    const int src = P.bound_to >= 0 ? P.bound_to : L.param_id;
    const Value& vi = c->values[g.in_value];
    const bool lin = L.d.op == GEMEL_OP_LINEAR;
    auto key = lin ? std::make_tuple(src, vi.C, vi.H, vi.W, vi.Cp)
                   : std::make_tuple(src, vi.Cp, g.cols ? -1 : 0, 0, 0);
    auto it = wkey_of.find(key);
    if (it == wkey_of.end()) {
      DevWeight w;
      w.param_id = src;
      w.linear = lin;
      w.N = L.d.cout;
      w.Cin = g.cols ? g.Cin : L.d.cin;
      w.cols = g.cols != 0;
      w.chunk = chunk_for(g.Cp_in);
      w.cin_k = round_up(g.Cp_in, w.chunk);
      w.kh = g.kh; w.kw = g.kw;
      w.Ktot = w.kh * w.kw * w.cin_k;
      if (lin) { w.flatC = vi.C; w.flatH = vi.H; w.flatW = vi.W; w.flatCp = vi.Cp; }
      w.bytes = uint64_t(w.N) * w.Ktot * 2;
      it = wkey_of.emplace(key, int(c->dweights.size())).first;
      c->dweights.push_back(w);
    }
    g.wkey = it->second;
  }

  // ------------------------------------------------------------ 3. batch union by progressive weighted LCS
  std::vector<Col> prof;
  for (int mi = 0; mi < int(c->models.size()); ++mi) {
    const auto& seq = gemm_seq[mi];
    auto geom = [&](int nid) {
      const Node& g = c->nodes[nid];
      return std::make_tuple(g.H, g.W, g.Cp_in);
    };
    if (prof.empty()) {
      for (int nid : seq) prof.push_back({c->nodes[nid].wkey, geom(nid), {nid}});
      continue;
    }
    const int P = int(prof.size()), S = int(seq.size());
    std::vector<std::vector<double>> dp(P + 1, std::vector<double>(S + 1, 0.0));
    auto match = [&](int p, int s) {
      const Node& g = c->nodes[seq[s]];
      return prof[p].wkey == g.wkey && prof[p].geom == geom(seq[s]);
    };
    for (int p = 1; p <= P; ++p)
      for (int s = 1; s <= S; ++s) {
        double best = std::max(dp[p - 1][s], dp[p][s - 1]);
        if (match(p - 1, s - 1)) best = std::max(best, dp[p - 1][s - 1] + c->nodes[seq[s - 1]].flops / c->nodes[seq[s - 1]].B + 1.0);
        dp[p][s] = best;
      }
    std::vector<Col> merged;
    int p = P, s = S;
    while (p > 0 || s > 0) {
      if (p > 0 && s > 0 && match(p - 1, s - 1) &&
          dp[p][s] == dp[p - 1][s - 1] + c->nodes[seq[s - 1]].flops / c->nodes[seq[s - 1]].B + 1.0) {
        Col col = prof[p - 1];
        col.nodes.push_back(seq[s - 1]);
        merged.push_back(col);
        --p; --s;
      } else if (p > 0 && (s == 0 || dp[p][s] == dp[p - 1][s])) {
        merged.push_back(prof[p - 1]);
        --p;
      } else {
        merged.push_back({c->nodes[seq[s - 1]].wkey, geom(seq[s - 1]), {seq[s - 1]}});
        --s;
      }
    }
    std::reverse(merged.begin(), merged.end());
    prof.swap(merged);
  }

  // ------------------------------------------------------------ 4. slabs + problems
  std::vector<std::vector<int>> slabs;   // value ids, contiguous in order
  auto consecutive_in_slab = [&](const std::vector<int>& vs) {
    const int sl = c->values[vs[0]].slab;
    if (sl < 0) return false;
    const auto& S = slabs[sl];
    auto it = std::find(S.begin(), S.end(), vs[0]);
    for (size_t k = 0; k < vs.size(); ++k, ++it)
      if (it == S.end() || *it != vs[k]) return false;
    return true;
  };
  for (auto& col : prof) {
    std::vector<int> mem = col.nodes;
    std::sort(mem.begin(), mem.end(), [&](int a, int b) { return c->nodes[a].model < c->nodes[b].model; });
    bool unioned = false;
    if (mem.size() >= 2) {
      std::vector<int> ins;
      for (int nid : mem) ins.push_back(c->nodes[nid].in_value);
      bool floating = true;
      for (int v : ins) floating = floating && c->values[v].slab < 0;
      std::vector<int> uniq(ins);
      std::sort(uniq.begin(), uniq.end());
      const bool distinct = std::unique(uniq.begin(), uniq.end()) == uniq.end();
      if (distinct && floating) {
        for (int v : ins) c->values[v].slab = int(slabs.size());
        slabs.push_back(ins);
        unioned = true;
      } else if (distinct && consecutive_in_slab(ins)) {
        unioned = true;
      }
      if (unioned) {
        std::vector<int> outs;
        for (int nid : mem) outs.push_back(c->nodes[nid].out_value);
        for (int v : outs) c->values[v].slab = int(slabs.size());
        slabs.push_back(outs);
        Problem pr;
        pr.members = mem;
        pr.wkey = col.wkey;
        for (int nid : mem) {
          c->nodes[nid].problem = int(c->problems.size());
          pr.n_img += c->nodes[nid].B;
        }
        c->problems.push_back(pr);
      }
    }
    if (!unioned)
      for (int nid : mem) {
        Problem pr;
        pr.members = {nid};
        pr.wkey = col.wkey;
        pr.n_img = c->nodes[nid].B;
        c->nodes[nid].problem = int(c->problems.size());
        c->problems.push_back(pr);
      }
  }

  // ------------------------------------------------------------ 5. levels (ASAP on the contracted DAG)
  // unit = problem (gemm) or node (others); dependencies through value producers
  const int NN = int(c->nodes.size());
  std::vector<int> unit_level_node(NN, -1), prob_level(c->problems.size(), -1), state(NN, 0);
  std::vector<int> pstate(c->problems.size(), 0);
  bool cycle = false;
  std::function<int(int)> node_level;
  std::function<int(int)> problem_level = [&](int pid) -> int {
    if (prob_level[pid] >= 0) return prob_level[pid];
    if (pstate[pid] == 1) { cycle = true; return 0; }
    pstate[pid] = 1;
    int lv = 0;
    for (int nid : c->problems[pid].members) {
      const Node& g = c->nodes[nid];
      for (int v : {g.in_value, g.res_value})
        if (v >= 0) lv = std::max(lv, node_level(c->values[v].producer) + 1);
    }
    pstate[pid] = 2;
    return prob_level[pid] = lv;
  };
  node_level = [&](int nid) -> int {
    const Node& g = c->nodes[nid];
    if (g.kind == NK_GEMM) return problem_level(g.problem);
    if (unit_level_node[nid] >= 0) return unit_level_node[nid];
    if (state[nid] == 1) { cycle = true; return 0; }
    state[nid] = 1;
    int lv = 0;
    for (int v : {g.in_value, g.in_value2, g.res_value})
      if (v >= 0) lv = std::max(lv, node_level(c->values[v].producer) + 1);
    for (int v : g.ins) lv = std::max(lv, node_level(c->values[v].producer) + 1);
    state[nid] = 2;
    return unit_level_node[nid] = lv;
  };
  int max_level = 0;
  for (int nid = 0; nid < NN; ++nid) {
    c->nodes[nid].level = node_level(nid);
    max_level = std::max(max_level, c->nodes[nid].level);
  }
  if (cycle) return set_err(c, GEMEL_E_STATE, "plan: batch union produced a cyclic schedule");
  // RPN levels as late as possible (just before their consumer, the proposal merge):
  // every FPN level of every model then shares one launch of (levels x frames) CTAs
  // instead of one latency-bound launch per level
  for (int nid = 0; nid < NN; ++nid) {
    Node& g = c->nodes[nid];
    if (g.kind != NK_RPN) continue;
    int lim = max_level + 1;
    for (const Node& h : c->nodes)
      for (int v : h.ins)
        if (v == g.out_value) lim = std::min(lim, h.level);
    if (lim - 1 > g.level) g.level = lim - 1;
  }
  for (size_t pid = 0; pid < c->problems.size(); ++pid) c->problems[pid].level = prob_level[pid];
  c->n_levels = max_level + 1;

  // ------------------------------------------------------------ 6. launches
  // Consecutive GEMM-only levels form ONE persistent GEMM launch whose
  // problems carry in-launch dependencies (the kernel waits on per-problem
  // completion counters), so dependent layers and independent models overlap.
  // A level with memory-bound nodes closes the segment after its own GEMMs.
  auto gemm_cost = [&](Launch& L, int pid) {
    const Problem& pr = c->problems[pid];
    const DevWeight& w = c->dweights[pr.wkey];
    L.bytes += double(w.N) * w.kh * w.kw * w.Cin * 2;
    for (int nid : pr.members) {
      const Node& g = c->nodes[nid];
      L.flops += g.flops;
      // fused first conv: reads the uint8 frames (3 B per pixel), not an im2col matrix
      L.bytes += (g.stem ? double(g.B) * c->models[g.model].in_h * c->models[g.model].in_w * 3
                         : double(g.B) * g.H * g.W * g.Cin * 2) +
                 double(c->values[g.out_value].B) * g.Ho * g.Wo * g.Cout * (c->values[g.out_value].fp32 ? 4 : 2);
      if (g.res_value >= 0) L.bytes += double(g.B) * g.Ho * g.Wo * g.Cout * 2;
    }
  };
  Launch seg;
  seg.kind = NK_GEMM;
  auto close_seg = [&]() {
    if (seg.items.empty()) return;
    c->launches.push_back(seg);
    seg = Launch();
    seg.kind = NK_GEMM;
  };
  for (int lv = 0; lv <= max_level; ++lv) {
    Launch pre, mp, ap, ad, ms, tk, rp, rm, ro, bp, nm;
    pre.kind = NK_PRE; mp.kind = NK_MAXPOOL; ap.kind = NK_AVGPOOL; ad.kind = NK_ADD; ms.kind = NK_MISC;
    tk.kind = NK_TOPK; rp.kind = NK_RPN; rm.kind = NK_RPNM; ro.kind = NK_ROI; bp.kind = NK_BOXP; nm.kind = NK_NMS;
    bool mem_nodes = false;
    for (int nid = 0; nid < NN; ++nid) {
      const Node& g = c->nodes[nid];
      if (g.level != lv || g.kind == NK_GEMM) continue;
      mem_nodes = true;
      Launch& L = g.kind == NK_PRE ? pre : g.kind == NK_MAXPOOL ? mp : g.kind == NK_AVGPOOL ? ap :
                  g.kind == NK_MISC ? ms : g.kind == NK_TOPK ? tk : g.kind == NK_RPN ? rp : g.kind == NK_RPNM ? rm :
                  g.kind == NK_ROI ? ro : g.kind == NK_BOXP ? bp : g.kind == NK_NMS ? nm : ad;
      L.items.push_back(nid);
      if (g.kind == NK_PRE && g.stem) continue;   // fused into the stem launch: no work here
      const Value& vo = c->values[g.out_value];
      if (g.kind >= NK_RPN) {   // algorithmic bytes: the output once, inputs once (ROI_ALIGN: taps, not maps)
        L.bytes += double(vo.bytes);
        if (g.kind == NK_ROI) L.bytes += double(vo.bytes) * 4.0;   // 4 bilinear taps per sample, L2-served
        else for (int v : g.ins) L.bytes += double(c->values[v].bytes);
        continue;
      }
      if (g.kind == NK_MISC) {   // pieces read once; concat output / decoded boxes written once
        for (int v : g.ins) L.bytes += double(c->values[v].bytes);
        L.bytes += g.misc == MISC_CONCAT ? double(vo.bytes) : double(c->values[g.in_value].bytes);
        continue;
      }
      const Value& vi = c->values[g.kind == NK_PRE ? g.out_value : g.in_value];
      L.bytes += double(vo.bytes) + (g.kind == NK_PRE ? double(vo.B) * vo.H * vo.W * 3 : double(vi.bytes));
      if (g.kind == NK_ADD) L.bytes += double(c->values[g.in_value2].bytes);
    }
    std::vector<int> lvl_probs;
    for (size_t pid = 0; pid < c->problems.size(); ++pid)
      if (c->problems[pid].level == lv) lvl_probs.push_back(int(pid));
    // biggest problems of a level first (better packing of the dynamic queue)
    std::stable_sort(lvl_probs.begin(), lvl_probs.end(), [&](int a, int b) {
      double fa = 0, fb = 0;
      for (int n : c->problems[a].members) fa += c->nodes[n].flops;
      for (int n : c->problems[b].members) fb += c->nodes[n].flops;
      return fa > fb;
    });
    // fused first convs: their own launch (stem kernel), ahead of this level's GEMMs
    Launch stem;
    stem.kind = NK_GEMM;
    stem.stem = 1;
    stem.level = lv;
    for (int pid : lvl_probs)
      if (c->nodes[c->problems[pid].members[0]].stem) {
        stem.items.push_back(pid);
        gemm_cost(stem, pid);
      }
    if (!stem.items.empty()) {
      close_seg();
      c->launches.push_back(stem);
    }
    for (int pid : lvl_probs) {
      if (c->nodes[c->problems[pid].members[0]].stem) continue;
      if (seg.items.empty()) seg.level = lv;
      seg.items.push_back(pid);
      gemm_cost(seg, pid);
    }
    if (mem_nodes) {
      close_seg();
      for (Launch* L : {&pre, &mp, &ap, &ad, &ms, &tk, &rp, &rm, &ro, &bp, &nm})
        if (!L->items.empty()) {
          L->level = lv;
          c->launches.push_back(*L);
        }
    }
  }
  close_seg();

  // weight budget: pinned set, swap ring, GEMM launches split so each one's
  // swapped weights fit half the ring (the other half fills for the next launch)
  {
    const int rc = plan_swap(c, [&](Launch& L, int pid) { gemm_cost(L, pid); });
    if (rc) return rc;
  }

  // N tile per problem: largest of {256, 128, 64} that still gives the problem
  // >= 64 tiles (chain latency vs. operand reuse); whole-launch fallback when
  // a launch cannot fill the machine.
  for (auto& L : c->launches) {
    if (L.kind != NK_GEMM) continue;
    if (L.stem) {   // stem launch: one tile = 128 consecutive output pixels of a member, all N columns
      L.stem_tasks = 0; L.stem_n_max = 16; L.stem_kp_max = 16; L.stem_tiles = 0;
      for (int pid : L.items) {
        Problem& pr = c->problems[pid];
        const DevWeight& w = c->dweights[pr.wkey];
        pr.bn = w.N; pr.msub = 1; pr.ksplit = 1; pr.kst_split = 1; pr.run = 1;
        for (int nid : pr.members) {
          const Node& g = c->nodes[nid];
          const gemel_layer& d = c->models[g.model].layers[g.layer].d;
          ++L.stem_tasks;
          L.stem_n_max = std::max(L.stem_n_max, w.N);
          L.stem_kp_max = std::max(L.stem_kp_max, stem_kp(d.kh, d.kw));
          L.stem_tiles += stem_tile_count(g.B, g.Ho, g.Wo, stem_sub(stem_kp(d.kh, d.kw)));
        }
      }
      L.total_tiles = L.total_items = int(std::min<int64_t>(L.stem_tiles, INT32_MAX));
      L.bn_max = L.stem_n_max; L.stages = 1; L.grid = 0; L.cg = 1; L.acc_w = 0;
      continue;
    }
    int cap = std::getenv("GEMEL_BN_CAP") ? std::atoi(std::getenv("GEMEL_BN_CAP")) : 256;
    const int min_tiles = std::getenv("GEMEL_MIN_TILES") ? std::atoi(std::getenv("GEMEL_MIN_TILES")) : 64;
    // split-K: off for convolution chains (the fp32 partial round trip lengthens the
    // dependency chain more than the parallelism gains, profiles/), on for weight-streaming
    // problems -- a few m-tiles over a long K (the classifiers' FC layers at small batch,
    // VGG fc6: M = 48, K = 25 088, 205 MB of weights) whose tiles would otherwise leave
    // most SMs idle while the weights stream (GEMEL_MAX_SPLIT overrides both)
    const char* split_env = std::getenv("GEMEL_MAX_SPLIT");
    const int max_split = split_env ? std::atoi(split_env) : 1;
    const int max_split_stream = split_env ? std::atoi(split_env) : 8;
    for (;;) {
      int tiles = 0, bn_max = 16;
      for (int pid : L.items) {
        Problem& pr = c->problems[pid];
        const DevWeight& w = c->dweights[pr.wkey];
        int64_t M = 0;
        for (int nid : pr.members) M += int64_t(c->nodes[nid].B) * c->nodes[nid].Ho * c->nodes[nid].Wo;
        const int64_t mt = (M + GEMM_BM - 1) / GEMM_BM;
        int bcap = cap;
        while (bcap > 64 && mt * ((w.N + bcap - 1) / bcap) < min_tiles) bcap /= 2;
        const int nt = (w.N + bcap - 1) / bcap;
        pr.bn = std::min(bcap, round_up((w.N + nt - 1) / nt, 16));
        const int ntiles = (w.N + pr.bn - 1) / pr.bn;
        // split-K for problems too small to occupy the machine (late layers at small batch):
        // double the split while the split tiles still fit in about one wave and every
        // split keeps >= 4 K stages; partials are reduced in a fixed order (deterministic)
        const int n_sub = w.kh * w.kw * (w.cin_k / w.chunk), R = GEMM_BK / w.chunk;
        const int n_kst = (n_sub + R - 1) / R;
        int ks = 1;
        const int cap_split = (w.linear && mt <= 2 && n_kst >= 64) ? max_split_stream : max_split;
        while (ks < cap_split && mt * ntiles * ks * 2 <= c->sm_count && n_kst / (ks * 2) >= 4) ks *= 2;
        pr.ksplit = ks;
        pr.kst_split = (n_kst + ks - 1) / ks;
        tiles += int(mt) * ntiles * ks;
        bn_max = std::max(bn_max, pr.bn);
      }
      L.total_tiles = tiles;
      L.bn_max = bn_max;
      if (tiles >= c->sm_count || cap <= 64) break;
      cap /= 2;
    }
    L.n_probs = int(L.items.size());
    auto rows_of = [&](const Problem& pr) {
      int64_t M = 0;
      for (int nid : pr.members) M += int64_t(c->nodes[nid].B) * c->nodes[nid].Ho * c->nodes[nid].Wo;
      return M;
    };
    // CTA pairs (cta_group::2, 256-row tiles): every launch with enough tiles for two waves
    // of pairs and no split-K (GEMEL_PAIR=0 disables -- the default, see DESIGN.md §6 --
    // 1 forces where legal)
    {
      const int pair_env = std::getenv("GEMEL_PAIR") ? std::atoi(std::getenv("GEMEL_PAIR")) : 0;
      bool legal = true;
      int64_t pair_tiles = 0;
      for (int pid : L.items) {
        const Problem& pr = c->problems[pid];
        legal &= pr.ksplit == 1;
        pair_tiles += ((rows_of(pr) + GEMM_BM - 1) / GEMM_BM + 1) / 2 * ((c->dweights[pr.wkey].N + pr.bn - 1) / pr.bn);
      }
      L.cg = legal && (pair_env == 1 || (pair_env != 0 && pair_tiles >= c->sm_count)) ? 2 : 1;
    }
    // Sub-tiles: a skinny problem (bn <= 128) runs tiles of msub consecutive 128-row
    // m-tiles (one accumulator of msub x bn TMEM columns, one scheduling / epilogue pass),
    // which amortises the per-tile fixed latencies that bound small tiles, while >= 2
    // waves of tiles remain.  The launch's accumulator width acc_w = max msub x bn <= 256.
    const int max_ms = std::getenv("GEMEL_MAX_MSUB") ? std::atoi(std::getenv("GEMEL_MAX_MSUB")) : 4;
    L.acc_w = 16;
    for (int pid : L.items) {
      Problem& pr = c->problems[pid];
      const int64_t mt = (rows_of(pr) + GEMM_BM - 1) / GEMM_BM;
      const int64_t nt = (c->dweights[pr.wkey].N + pr.bn - 1) / pr.bn;
      pr.msub = 1;
      if (L.cg == 1 && pr.ksplit == 1)
        while (pr.msub * 2 <= max_ms && pr.msub * 2 * pr.bn <= 256 &&
               (mt + pr.msub * 2 - 1) / (pr.msub * 2) * nt >= 2 * c->sm_count)
          pr.msub *= 2;
      L.acc_w = std::max(L.acc_w, pr.msub * pr.bn);
    }
    // Output chunks through TMA stores (bulk async; their completion is awaited before a
    // tile publishes) or through the LSU transpose path (GEMEL_TMA_STORE, default on)
    L.epi_flags = (std::getenv("GEMEL_TMA_STORE") ? std::atoi(std::getenv("GEMEL_TMA_STORE")) : 1) ? 1 : 0;
    // Tile-queue grabs: a problem of short-K tiles spread over many waves hands out runs
    // of consecutive tiles per atomic, keeping >= 2 waves of grabs.
    // (measured: off by default -- cfg4 GEMM 9.08 ms with runs of up to 8, 8.92 ms without)
    const int max_run = std::getenv("GEMEL_MAX_RUN") ? std::atoi(std::getenv("GEMEL_MAX_RUN")) : 1;
    L.total_tiles = 0;
    L.total_items = 0;
    for (int pid : L.items) {
      Problem& pr = c->problems[pid];
      const int m_step = L.cg * pr.msub;
      const int64_t tp = ((rows_of(pr) + GEMM_BM - 1) / GEMM_BM + m_step - 1) / m_step *
                         ((c->dweights[pr.wkey].N + pr.bn - 1) / pr.bn) * pr.ksplit;
      pr.run = 1;
      if (pr.ksplit == 1 && pr.kst_split * pr.msub <= 8)
        while (pr.run < max_run && tp / (2 * pr.run) >= 2 * c->sm_count / L.cg) pr.run *= 2;
      L.total_tiles += int(tp);
      L.total_items += int((tp + pr.run - 1) / pr.run);
    }
    L.stages = gemm_pick_stages(L.bn_max, L.cg);
    if (const char* e = std::getenv("GEMEL_STAGES"))   // developer probe: fewer pipeline stages
      L.stages = std::max(2, std::min(L.stages, std::atoi(e)));
    L.grid = L.cg == 2 ? 2 * std::min(L.total_tiles, c->sm_count / 2) : std::min(L.total_tiles, c->sm_count);
  }
  // in-launch dependencies (problem indices local to the launch)
  for (size_t li = 0; li < c->launches.size(); ++li) {
    Launch& L = c->launches[li];
    if (L.kind != NK_GEMM) continue;
    std::map<int, int> local;
    for (size_t k = 0; k < L.items.size(); ++k) local[L.items[k]] = int(k);
    L.deps.assign(L.items.size(), {});
    for (size_t k = 0; k < L.items.size(); ++k) {
      std::vector<int>& d = L.deps[k];
      for (int nid : c->problems[L.items[k]].members) {
        const Node& g = c->nodes[nid];
        for (int v : {g.in_value, g.res_value}) {
          if (v < 0) continue;
          const Node& pn = c->nodes[c->values[v].producer];
          if (pn.kind != NK_GEMM) continue;
          auto it = local.find(pn.problem);
          if (it == local.end()) continue;
          if (it->second >= int(k))
            return set_err(c, GEMEL_E_STATE, "plan: dependency does not precede its consumer in a launch");
          if (std::find(d.begin(), d.end(), it->second) == d.end()) d.push_back(it->second);
        }
      }
      if (int(d.size()) > GEMM_MAX_DEPS) return set_err(c, GEMEL_E_UNSUPPORTED, "plan: too many producer problems");
    }
  }

  // ------------------------------------------------------------ 7. arena layout
  // pinned weights, then the swap ring (swapped weights at their slots), then the
  // always-resident epilogue vectors
  uint64_t off = 0;
  for (auto& w : c->dweights) {
    if (w.swapped) continue;
    w.offset = off;
    off = align_up(off + w.bytes, 256);
  }
  c->ring_off = off;
  for (auto& w : c->dweights)
    if (w.swapped) w.offset += c->ring_off;   // plan_swap stored the slot offset within the ring
  off += c->ring_bytes;
  for (auto& g : c->nodes)
    if (g.kind == NK_GEMM) {
      g.scale_off = off;
      off = align_up(off + uint64_t(g.Cout) * 4, 256);
      g.shift_off = off;
      off = align_up(off + uint64_t(g.Cout) * 4, 256);
    } else if (g.kind == NK_MISC && g.misc == MISC_L2NORM) {   // the L2Norm scale, resident
      g.scale_off = off;
      off = align_up(off + uint64_t(g.Cout) * 4, 256);
    }
  c->w_bytes = off;

  off = 0;
  int max_stream = 0;
  for (auto& M : c->models) max_stream = std::max(max_stream, M.stream_id);
  c->frame_off.assign(max_stream + 1, -1);
  std::vector<int> stream_hw(2 * (max_stream + 1), 0);
  for (auto& M : c->models) {
    const int s = M.stream_id;
    if (c->frame_off[s] >= 0) {
      if (stream_hw[2 * s] != M.in_h || stream_hw[2 * s + 1] != M.in_w)
        return set_err(c, GEMEL_E_ARG, "plan: models on one stream must share the input resolution");
      continue;
    }
    stream_hw[2 * s] = M.in_h;
    stream_hw[2 * s + 1] = M.in_w;
    c->frame_off[s] = int64_t(off);
    off = align_up(off + uint64_t(c->batch[s]) * M.in_h * M.in_w * 3, 256);
  }
  // second staging buffer: step k+1's frames are copied while step k computes
  const uint64_t stage_bytes = off;
  c->frame_off2.assign(c->frame_off.size(), -1);
  for (size_t s = 0; s < c->frame_off.size(); ++s)
    if (c->frame_off[s] >= 0) c->frame_off2[s] = int64_t(c->frame_off[s] + stage_bytes);
  off += stage_bytes;
  for (auto& S : slabs) {
    for (int v : S) {
      c->values[v].offset = off;
      off += c->values[v].bytes;
    }
    off = align_up(off, 256);
  }
  for (auto& v : c->values)
    if (v.slab < 0) {
      v.offset = off;
      off = align_up(off + v.bytes, 256);
    }
  // split-K partial workspaces and per-launch counter blocks
  for (auto& L : c->launches) {
    if (L.kind != NK_GEMM) continue;
    int ncnt = 1;
    uint64_t dep_idx = 0;
    for (size_t k = 0; k < L.items.size(); ++k) {   // per-m-tile completion counters + dependency ranges
      Problem& pr = c->problems[L.items[k]];
      int64_t M = 0;
      for (int nid : pr.members) M += int64_t(c->nodes[nid].B) * c->nodes[nid].Ho * c->nodes[nid].Wo;
      pr.m_tiles = int((M + GEMM_BM - 1) / GEMM_BM);
      pr.cnt_off = ncnt;
      ncnt += pr.m_tiles;
      pr.dep_idx = dep_idx;
      dep_idx += uint64_t(pr.m_tiles) * L.deps[k].size() * 2;
    }
    L.dep_off = dep_idx;   // (int32 count; turned into a meta offset below)
    for (int pid : L.items) {
      Problem& pr = c->problems[pid];
      if (pr.ksplit <= 1) continue;
      const DevWeight& w = c->dweights[pr.wkey];
      const int64_t mn = int64_t(pr.m_tiles) * ((w.N + pr.bn - 1) / pr.bn);
      pr.ws_off = off;
      off = align_up(off + uint64_t(mn) * pr.ksplit * GEMM_BM * round_up(pr.bn, 32) * 4, 256);
      pr.tcnt_idx = ncnt;
      ncnt += int(mn);
    }
    L.n_counters = ncnt;
  }
  c->act_bytes = off;

  // accounting
  c->unique_weight_bytes = c->unmerged_weight_bytes = 0;
  for (auto& p : c->params) {
    c->unmerged_weight_bytes += p.bytes;
    if (p.bound_to < 0) c->unique_weight_bytes += p.bytes;
  }
  c->gemm_flops = 0;
  for (auto& g : c->nodes)
    if (g.kind == NK_GEMM) c->gemm_flops += g.flops;
  // meta (launch tables) sizes
  uint64_t meta = 0;
  for (auto& L : c->launches) {
    L.meta_off = meta;
    if (L.kind == NK_GEMM) {
      int nseg = 0;
      for (int pid : L.items) nseg += int(c->problems[pid].members.size());
      meta = align_up(meta + uint64_t(L.items.size()) * sizeof(GemmProblem), 256);
      L.seg_off = meta;
      meta = align_up(meta + uint64_t(nseg) * sizeof(GemmSeg), 256);
      L.cnt_off = meta;
      meta = align_up(meta + uint64_t(L.n_counters) * 4, 256);
      const uint64_t n_dep_ints = L.dep_off;
      L.dep_off = meta;
      meta = align_up(meta + n_dep_ints * 4, 256);
      if (L.stem) {
        L.stem_off = meta;
        meta = align_up(meta + 2 * uint64_t(L.stem_tasks) * sizeof(StemTask), 256);
      }
    } else if (L.kind == NK_PRE) {   // one task table per staging buffer
      meta = align_up(meta + 2 * L.items.size() * sizeof(PreTask), 256);
    } else if (L.kind == NK_ADD) {
      meta = align_up(meta + L.items.size() * sizeof(AddTask), 256);
    } else if (L.kind == NK_TOPK) {
      meta = align_up(meta + L.items.size() * sizeof(TopkTask), 256);
    } else if (L.kind == NK_RPN) {
      meta = align_up(meta + L.items.size() * sizeof(RpnTask), 256);
    } else if (L.kind == NK_RPNM) {
      meta = align_up(meta + L.items.size() * sizeof(RpnMergeTask), 256);
    } else if (L.kind == NK_ROI) {
      meta = align_up(meta + L.items.size() * sizeof(RoiTask), 256);
    } else if (L.kind == NK_BOXP) {
      meta = align_up(meta + L.items.size() * sizeof(BoxPostTask), 256);
    } else if (L.kind == NK_NMS) {
      meta = align_up(meta + L.items.size() * sizeof(NmsTask), 256);
    } else if (L.kind == NK_MISC) {
      size_t nt = 0;
      for (int nid : L.items) nt += c->nodes[nid].ins.size();
      meta = align_up(meta + nt * sizeof(MiscTask), 256);
    } else {
      meta = align_up(meta + L.items.size() * sizeof(PoolTask), 256);
    }
  }
  c->meta_bytes = meta;
  return GEMEL_OK;
}

std::string plan_json(const Ctx* c) {
  std::ostringstream o;
  // algorithmic bytes of a GEMM problem (the gemm_cost rule): the weight once, every
  // member's input and output once (fp32 outputs 4 B), its residual once
  auto problem_bytes = [&](const Problem& pr) {
    const DevWeight& w = c->dweights[pr.wkey];
    double b = double(w.N) * w.kh * w.kw * w.Cin * 2;
    for (int nid : pr.members) {
      const Node& g = c->nodes[nid];
      b += (g.stem ? double(g.B) * c->models[g.model].in_h * c->models[g.model].in_w * 3
                   : double(g.B) * g.H * g.W * g.Cin * 2) +
           double(c->values[g.out_value].B) * g.Ho * g.Wo * g.Cout * (c->values[g.out_value].fp32 ? 4 : 2);
      if (g.res_value >= 0) b += double(g.B) * g.Ho * g.Wo * g.Cout * 2;
    }
    return b;
  };
  auto kind = [](int k) {
    switch (k) {
      case NK_PRE: return "preprocess";
      case NK_GEMM: return "gemm";
      case NK_MAXPOOL: return "maxpool";
      case NK_AVGPOOL: return "avgpool";
      case NK_MISC: return "concat_yolo";
      case NK_TOPK: return "topk";
      case NK_RPN: return "rpn_level";
      case NK_RPNM: return "rpn_merge";
      case NK_ROI: return "roi_align";
      case NK_BOXP: return "box_post";
      case NK_NMS: return "det_nms";
      default: return "add";
    }
  };
  auto vref = [&](int v) {
    std::ostringstream t;
    if (v < 0) { t << "null"; return t.str(); }
    t << "[" << c->values[v].model << "," << c->values[v].pos << "]";
    return t.str();
  };
  o << "{\"levels\":" << c->n_levels << ",\"swap\":{\"budget\":" << c->opt.weight_budget_bytes
    << ",\"weight_arena_bytes\":" << c->w_bytes << ",\"pinned_bytes\":" << c->pinned_bytes
    << ",\"ring_off\":" << c->ring_off << ",\"ring_bytes\":" << c->ring_bytes << ",\"swap_bytes\":" << c->swap_bytes
    << ",\"weights\":[";
  for (size_t i = 0; i < c->dweights.size(); ++i) {
    const DevWeight& w = c->dweights[i];
    o << (i ? "," : "") << "{\"param\":[" << c->params[w.param_id].model << "," << c->params[w.param_id].pos
      << "],\"bytes\":" << w.bytes << ",\"offset\":" << w.offset << ",\"swapped\":" << (w.swapped ? 1 : 0)
      << ",\"first_launch\":" << w.first_launch << ",\"last_launch\":" << w.last_launch
      << ",\"wait_launch\":" << w.wait_launch << ",\"copy_order\":" << w.copy_order << "}";
  }
  o << "]},\"nodes\":[";
  for (size_t i = 0; i < c->nodes.size(); ++i) {
    const Node& g = c->nodes[i];
    if (i) o << ",";
    o << "{\"kind\":\"" << kind(g.kind) << "\",\"model\":" << g.model << ",\"level\":" << g.level
      << ",\"layers\":[";
    bool first = true;
    if (g.kind != NK_PRE)
      for (int l : {g.layer, g.bn, g.add, g.act_layer, g.kind == NK_GEMM ? g.up_layer : -1})
        if (l >= 0) { o << (first ? "" : ",") << l; first = false; }
    if (g.kind == NK_MISC) {
      const auto& M = c->models[g.model];
      const gemel_layer& d = M.layers[g.layer].d;
      if (g.misc == MISC_CONCAT && d.op == GEMEL_OP_CONCAT)   // upsample layers fused into the pieces
        for (int k = 0; k < d.n_in; ++k)
          if (d.in[k] >= 0 && M.layers[d.in[k]].d.op == GEMEL_OP_UPSAMPLE_NEAREST) o << "," << d.in[k];
      if ((g.misc == MISC_YOLO || g.misc == MISC_SSD) && g.out_off == 0)   // the detection concat it writes into
        for (int j = g.layer + 1; j < int(M.layers.size()); ++j)
          if (M.layers[j].d.op == GEMEL_OP_CONCAT &&
              std::find(M.layers[j].d.in, M.layers[j].d.in + M.layers[j].d.n_in, g.layer) != M.layers[j].d.in + M.layers[j].d.n_in) {
            o << "," << j;
            break;
          }
    }
    if (g.kind == NK_ADD && g.act != ACT_NONE) {
      const auto& M = c->models[g.model];
      for (int j = g.layer + 1; j < int(M.layers.size()); ++j)
        if (M.layers[j].d.n_in == 1 && M.layers[j].d.in[0] == g.layer &&
            (M.layers[j].d.op == GEMEL_OP_RELU || M.layers[j].d.op == GEMEL_OP_LEAKY_RELU)) {
          o << "," << j;
          break;
        }
    }
    o << "],\"inputs\":[";
    if (g.kind == NK_MISC || g.kind >= NK_RPN)
      for (size_t k = 0; k < g.ins.size(); ++k) o << (k ? "," : "") << vref(g.ins[k]);
    else
      o << vref(g.in_value) << "," << vref(g.in_value2) << "," << vref(g.res_value);
    o << "],\"output\":" << vref(g.out_value) << ",\"problem\":" << g.problem << "}";
  }
  o << "],\"launches\":[";
  for (size_t li = 0; li < c->launches.size(); ++li) {
    const Launch& L = c->launches[li];
    if (li) o << ",";
    o << "{\"kind\":\"" << kind(L.kind) << "\",\"level\":" << L.level << ",\"flops\":" << L.flops
      << ",\"bytes\":" << L.bytes;
    if (L.kind == NK_GEMM) {
      o << ",\"stem\":" << L.stem << ",\"tiles\":" << L.total_tiles << ",\"cg\":" << L.cg << ",\"acc_w\":" << L.acc_w << ",\"grid\":" << L.grid << ",\"bn_max\":" << L.bn_max
        << ",\"stages\":" << L.stages << ",\"problems\":[";
      for (size_t k = 0; k < L.items.size(); ++k) {
        const Problem& pr = c->problems[L.items[k]];
        const DevWeight& w = c->dweights[pr.wkey];
        const Node& g0 = c->nodes[pr.members[0]];
        int64_t M = 0;
        for (int nid : pr.members) M += int64_t(c->nodes[nid].B) * c->nodes[nid].Ho * c->nodes[nid].Wo;
        if (k) o << ",";
        o << "{\"members\":[";
        for (size_t m = 0; m < pr.members.size(); ++m)
          o << (m ? "," : "") << "[" << c->nodes[pr.members[m]].model << "," << c->nodes[pr.members[m]].layer << "]";
        o << "],\"M\":" << M << ",\"N\":" << w.N << ",\"K\":" << w.kh * w.kw * w.Cin << ",\"Ktot\":" << w.Ktot
          << ",\"bn\":" << pr.bn << ",\"ksplit\":" << pr.ksplit << ",\"run\":" << pr.run << ",\"msub\":" << pr.msub << ",\"chunk\":" << w.chunk << ",\"kh\":" << w.kh
          << ",\"kw\":" << w.kw << ",\"sh\":" << g0.sh << ",\"cols\":" << (w.cols ? 1 : 0) << ",\"linear\":" << (w.linear ? 1 : 0)
          << ",\"Ho\":" << g0.Ho << ",\"Wo\":" << g0.Wo
          << ",\"wkey\":" << pr.wkey << ",\"bytes\":" << problem_bytes(pr)
          << ",\"weight_param\":[" << c->params[w.param_id].model << "," << c->params[w.param_id].pos << "]}";
      }
      o << "]";
    } else {
      o << ",\"nodes\":[";
      for (size_t k = 0; k < L.items.size(); ++k)
        o << (k ? "," : "") << "[" << c->nodes[L.items[k]].model << "," << c->nodes[L.items[k]].layer << "]";
      o << "]";
    }
    o << "}";
  }
  o << "]}";
  return o.str();
}

}  // namespace gemel

using namespace gemel;

extern "C" gemel_status gemel_plan_dump(gemel_ctx ctx, char* buf, uint64_t cap, uint64_t* len) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c || !len) return GEMEL_E_ARG;
  if (!c->planned) return set_err(c, GEMEL_E_STATE, "plan_dump before plan");
  const std::string s = plan_json(c);
  *len = s.size() + 1;
  if (!buf) return GEMEL_OK;
  if (cap < s.size() + 1) return set_err(c, GEMEL_E_SMALLBUF, "plan_dump: buffer too small");
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return GEMEL_OK;
}
