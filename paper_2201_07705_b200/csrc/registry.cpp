// Host-side, integer-only part of the C ABI: context, model registration,
// shareable-group enumeration and merge accounting.  Never touches the GPU.
//
//   register_model  PAPER.md:292 (a query's DNN), schema per layer type
//   find_shareable  PAPER.md:209-213 (architectural equivalence: same type and
//                   identical type-specific properties, weights excluded),
//                   PAPER.md:374 (groups = every appearance, memory-sorted)
//   apply_merge     PAPER.md:376-378 (running merge configuration, weights from
//                   one member), PAPER.md:443 (parameter-memory reduction)
#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <sstream>
#include <tuple>

#include "internal.h"

namespace gemel {

int set_err(Ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  return code;
}

namespace {

bool is_param_op(int op) { return op == GEMEL_OP_CONV2D || op == GEMEL_OP_LINEAR || op == GEMEL_OP_BATCHNORM2D; }

uint32_t fbits(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  return u;
}

// Architectural signature: op + every defining hyperparameter (no weights,
// no position, no input H x W).
std::vector<int64_t> signature(const gemel_layer& d) {
  switch (d.op) {
    case GEMEL_OP_CONV2D:
      return {d.op, d.cin, d.cout, d.kh, d.kw, d.sh, d.sw, d.ph, d.pw, d.dh, d.dw, d.groups, d.bias ? 1 : 0};
    case GEMEL_OP_LINEAR:
      return {d.op, d.cin, d.cout, d.bias ? 1 : 0};
    case GEMEL_OP_BATCHNORM2D:
      return {d.op, d.cin, fbits(d.eps), fbits(d.momentum), d.affine ? 1 : 0, d.track_stats ? 1 : 0};
    default:
      return {};
  }
}

uint64_t param_elems(const gemel_layer& d) {
  switch (d.op) {
    case GEMEL_OP_CONV2D:
      return uint64_t(d.cout) * (d.cin / std::max(d.groups, 1)) * d.kh * d.kw + (d.bias ? d.cout : 0);
    case GEMEL_OP_LINEAR:
      return uint64_t(d.cout) * d.cin + (d.bias ? d.cout : 0);
    case GEMEL_OP_BATCHNORM2D:
      return 4ull * d.cin;
    default:
      return 0;
  }
}

int conv_out(int h, int k, int s, int p, int d) { return (h + 2 * p - d * (k - 1) - 1) / s + 1; }

int pool_out(int h, int k, int s, int p, int d, bool ceil_mode) {
  int num = h + 2 * p - d * (k - 1) - 1;
  if (!ceil_mode) return num / s + 1;
  int o = (num + s - 1) / s + 1;
  if ((o - 1) * s >= h + p) --o;
  return o;
}

std::string where(int model, int pos) {
  std::ostringstream o;
  o << "model " << model << " op " << pos << ": ";
  return o.str();
}

}  // namespace
}  // namespace gemel

using namespace gemel;

extern "C" {

gemel_status gemel_create(const gemel_options* opt, gemel_ctx* out) {
  if (!out) return GEMEL_E_ARG;
  if (opt && (opt->weight_source < GEMEL_SOURCE_HOST || opt->weight_source > GEMEL_SOURCE_PEER)) return GEMEL_E_ARG;
  Ctx* c = new Ctx();
  if (opt) c->opt = *opt;
  *out = reinterpret_cast<gemel_ctx>(c);
  return GEMEL_OK;
}

void gemel_destroy(gemel_ctx ctx) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c) return;
  release_device(c);
  delete c;
}

const char* gemel_last_error(gemel_ctx ctx) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  return c ? c->err.c_str() : "null context";
}

gemel_status gemel_register_model(gemel_ctx ctx, const gemel_layer* ops, int32_t n_ops, int32_t stream_id,
                                  int32_t in_h, int32_t in_w, int32_t* model_id) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c) return GEMEL_E_ARG;
  if (c->planned) return set_err(c, GEMEL_E_STATE, "register_model after plan");
  if (!ops || n_ops <= 0 || in_h <= 0 || in_w <= 0 || stream_id < 0)
    return set_err(c, GEMEL_E_ARG, "register_model: bad arguments");
  const int mid = int(c->models.size());
  Model m;
  m.stream_id = stream_id;
  m.in_h = in_h;
  m.in_w = in_w;
  std::vector<ParamLayer> newp;
  for (int i = 0; i < n_ops; ++i) {
    const gemel_layer& d = ops[i];
    Layer L;
    L.d = d;
    for (auto& p : L.d.param) p = nullptr;
    const std::string at = where(mid, i);
    if (d.n_in < 1 || d.n_in > 8) return set_err(c, GEMEL_E_SCHEMA, at + "n_in out of range");
    for (int k = 0; k < d.n_in; ++k)
      if (d.in[k] < -1 || d.in[k] >= i) return set_err(c, GEMEL_E_SCHEMA, at + "input index not topological");
    auto in_shape = [&](int k, int& C, int& H, int& W) {
      int j = d.in[k];
      if (j < 0) { C = 3; H = in_h; W = in_w; }
      else { C = m.layers[j].C; H = m.layers[j].H; W = m.layers[j].W; }
    };
    int C, H, W;
    in_shape(0, C, H, W);
    L.inC = C; L.inH = H; L.inW = W;
    L.rows = d.in[0] >= 0 ? m.layers[d.in[0]].rows : 1;
    if (d.tie != 0) {   // tied conv: op (tie-1)'s parameters, identical hyperparameters
      const int j = d.tie - 1;
      if (d.op != GEMEL_OP_CONV2D || j < 0 || j >= i || m.layers[j].d.op != GEMEL_OP_CONV2D || m.layers[j].tie >= 0)
        return set_err(c, GEMEL_E_SCHEMA, at + "tie must name an earlier untied conv");
      gemel_layer a = d, b = m.layers[j].d;
      a.tie = b.tie = 0;
      for (int k = 0; k < 8; ++k) a.in[k] = b.in[k] = 0;
      for (auto& q : a.param) q = nullptr;
      for (auto& q : b.param) q = nullptr;
      a.out_h = b.out_h = a.out_w = b.out_w = 0;
      if (signature(a) != signature(b)) return set_err(c, GEMEL_E_SCHEMA, at + "tied conv hyperparameters differ");
      L.tie = j;
    }
    switch (d.op) {
      case GEMEL_OP_CONV2D: {
        if (d.n_in != 1) return set_err(c, GEMEL_E_SCHEMA, at + "conv takes one input");
        if (d.cin != C) return set_err(c, GEMEL_E_SCHEMA, at + "conv cin != producer channels");
        if (d.cout <= 0 || d.kh <= 0 || d.kw <= 0 || d.sh <= 0 || d.sw <= 0 || d.ph < 0 || d.pw < 0 || d.dh <= 0 ||
            d.dw <= 0)
          return set_err(c, GEMEL_E_SCHEMA, at + "conv hyperparameters out of range");
        if (d.groups != 1) return set_err(c, GEMEL_E_UNSUPPORTED, at + "grouped convolution not supported");
        if (L.tie < 0 && (!d.param[0] || (d.bias && !d.param[1])))
          return set_err(c, GEMEL_E_SCHEMA, at + "conv params missing");
        L.C = d.cout;
        L.H = conv_out(H, d.kh, d.sh, d.ph, d.dh);
        L.W = conv_out(W, d.kw, d.sw, d.pw, d.dw);
        if (L.H <= 0 || L.W <= 0) return set_err(c, GEMEL_E_SCHEMA, at + "conv output is empty");
        break;
      }
      case GEMEL_OP_LINEAR: {
        if (d.n_in != 1) return set_err(c, GEMEL_E_SCHEMA, at + "linear takes one input");
        if (d.cin != C * H * W) return set_err(c, GEMEL_E_SCHEMA, at + "linear in_features != producer features");
        if (d.cout <= 0 || !d.param[0] || (d.bias && !d.param[1]))
          return set_err(c, GEMEL_E_SCHEMA, at + "linear params missing");
        L.C = d.cout; L.H = 1; L.W = 1; L.flat = true;
        break;
      }
      case GEMEL_OP_BATCHNORM2D: {
        if (d.n_in != 1 || d.cin != C) return set_err(c, GEMEL_E_SCHEMA, at + "bn channels != producer channels");
        if (!(d.eps > 0.f) || !d.affine || !d.track_stats)
          return set_err(c, GEMEL_E_UNSUPPORTED, at + "bn needs eps > 0, affine and running stats");
        for (int k = 0; k < 4; ++k)
          if (!d.param[k]) return set_err(c, GEMEL_E_SCHEMA, at + "bn params missing");
        L.C = C; L.H = H; L.W = W;
        break;
      }
      case GEMEL_OP_RELU:
      case GEMEL_OP_LEAKY_RELU:
        if (d.n_in != 1) return set_err(c, GEMEL_E_SCHEMA, at + "activation takes one input");
        L.C = C; L.H = H; L.W = W;
        break;
      case GEMEL_OP_MAXPOOL2D: {
        if (d.n_in != 1 || d.kh <= 0 || d.kw <= 0 || d.sh <= 0 || d.sw <= 0 || d.ph < 0 || d.pw < 0 ||
            d.dh <= 0 || d.dw <= 0 || 2 * d.ph > d.kh || 2 * d.pw > d.kw || d.ceil_mode < 0 || d.ceil_mode > 2)
          return set_err(c, GEMEL_E_SCHEMA, at + "maxpool hyperparameters out of range");
        L.C = C;
        if (d.ceil_mode == 2) {   // darknet: out-of-range taps ignored, out = (H-1)/s + 1
          if (d.ph || d.pw || d.dh != 1 || d.dw != 1)
            return set_err(c, GEMEL_E_SCHEMA, at + "darknet maxpool takes no padding or dilation");
          L.H = (H - 1) / d.sh + 1;
          L.W = (W - 1) / d.sw + 1;
          break;
        }
        L.H = pool_out(H, d.kh, d.sh, d.ph, d.dh, d.ceil_mode != 0);
        L.W = pool_out(W, d.kw, d.sw, d.pw, d.dw, d.ceil_mode != 0);
        if (L.H <= 0 || L.W <= 0) return set_err(c, GEMEL_E_SCHEMA, at + "maxpool output is empty");
        break;
      }
      case GEMEL_OP_ADAPTIVE_AVGPOOL2D:
        if (d.n_in != 1 || d.out_h <= 0 || d.out_w <= 0)
          return set_err(c, GEMEL_E_SCHEMA, at + "adaptive avgpool needs out_h, out_w > 0");
        L.C = C; L.H = d.out_h; L.W = d.out_w;
        break;
      case GEMEL_OP_ADD: {
        if (d.n_in != 2) return set_err(c, GEMEL_E_SCHEMA, at + "add takes two inputs");
        int C2, H2, W2;
        in_shape(1, C2, H2, W2);
        if (C2 != C || H2 != H || W2 != W) return set_err(c, GEMEL_E_SCHEMA, at + "add operand shapes differ");
        L.C = C; L.H = H; L.W = W;
        break;
      }
      case GEMEL_OP_FLATTEN:
        if (d.n_in != 1) return set_err(c, GEMEL_E_SCHEMA, at + "flatten takes one input");
        L.C = C * H * W; L.H = 1; L.W = 1; L.flat = true;
        break;
      case GEMEL_OP_CONCAT: {
        if (d.n_in < 2) return set_err(c, GEMEL_E_SCHEMA, at + "concat takes 2..8 inputs");
        const bool flat0 = d.in[0] >= 0 && m.layers[d.in[0]].flat;
        int Ct = 0;
        for (int k = 0; k < d.n_in; ++k) {
          int Ck, Hk, Wk;
          in_shape(k, Ck, Hk, Wk);
          const bool fk = d.in[k] >= 0 && m.layers[d.in[k]].flat;
          if (fk != flat0 || (!flat0 && (Hk != H || Wk != W)))
            return set_err(c, GEMEL_E_SCHEMA, at + "concat operands differ in spatial size or kind");
          Ct += Ck;
        }
        L.C = Ct; L.H = H; L.W = W; L.flat = flat0;
        break;
      }
      case GEMEL_OP_UPSAMPLE_NEAREST:
        if (d.n_in != 1 || d.sh < 1 || d.sw < 1 || d.sh != d.sw)
          return set_err(c, GEMEL_E_SCHEMA, at + "upsample needs sh = sw >= 1");
        L.C = C; L.H = H * d.sh; L.W = W * d.sw;
        break;
      case GEMEL_OP_L2NORM:
        if (d.n_in != 1 || d.cin != C || !(d.eps > 0.f) || !d.param[0])
          return set_err(c, GEMEL_E_SCHEMA, at + "l2norm needs cin = producer channels, eps > 0 and a scale");
        L.anchors.assign(d.param[0], d.param[0] + C);   // the per-channel scale
        L.C = C; L.H = H; L.W = W;
        break;
      case GEMEL_OP_SSD_DECODE: {
        int C2, H2, W2;
        if (d.n_in != 2 || d.kh < 1 || d.kh > 8 || d.cout < 2 || d.sh < 1 || !d.param[0] || !d.param[1])
          return set_err(c, GEMEL_E_SCHEMA, at + "ssd decode needs (loc, conf), 1..8 anchors, classes, step");
        in_shape(1, C2, H2, W2);
        if (C != d.kh * 4 || C2 != d.kh * d.cout || H2 != H || W2 != W)
          return set_err(c, GEMEL_E_SCHEMA, at + "ssd decode: loc = A*4, conf = A*classes channels, same H x W");
        L.anchors.assign(d.param[0], d.param[0] + 2 * d.kh);
        L.anchors.insert(L.anchors.end(), d.param[1], d.param[1] + 4);   // then the coder weights
        L.C = d.kh * H * W * (5 + d.cout); L.H = 1; L.W = 1; L.flat = true;
        break;
      }
      case GEMEL_OP_RPN_LEVEL: {
        int C2, H2, W2;
        if (d.n_in != 2 || d.kh < 1 || d.kh > 8 || d.cout < 1 || d.cout > 1024 || !(d.neg_slope >= 0.f) ||
            !(d.eps >= 0.f) || !d.param[0])
          return set_err(c, GEMEL_E_SCHEMA, at + "rpn level needs (objectness, deltas), 1..8 anchors, pre_n 1..1024");
        in_shape(1, C2, H2, W2);
        if (C != d.kh || C2 != 4 * d.kh || H2 != H || W2 != W || L.rows != 1)
          return set_err(c, GEMEL_E_SCHEMA, at + "rpn level: objectness = A, deltas = 4A channels, same H x W");
        L.anchors.assign(d.param[0], d.param[0] + 2 * d.kh);   // (size, ratio) per anchor
        L.C = std::min(d.cout, d.kh * H * W) * 6; L.H = 1; L.W = 1; L.flat = true;
        break;
      }
      case GEMEL_OP_RPN_MERGE: {
        if (d.cout < 1 || d.cout > 4096) return set_err(c, GEMEL_E_SCHEMA, at + "rpn merge needs post_n 1..4096");
        int tot = 0;
        for (int k = 0; k < d.n_in; ++k) {
          if (d.in[k] < 0 || m.layers[d.in[k]].d.op != GEMEL_OP_RPN_LEVEL)
            return set_err(c, GEMEL_E_SCHEMA, at + "rpn merge inputs must be rpn levels");
          tot += m.layers[d.in[k]].C / 6;
        }
        if (tot > 8192) return set_err(c, GEMEL_E_UNSUPPORTED, at + "rpn merge over more than 8192 candidates");
        L.C = d.cout * 5; L.H = 1; L.W = 1; L.flat = true;
        break;
      }
      case GEMEL_OP_ROI_ALIGN: {
        if (d.n_in < 2 || d.n_in > 5 || d.in[0] < 0 || m.layers[d.in[0]].d.op != GEMEL_OP_RPN_MERGE ||
            d.out_h < 1 || d.out_h != d.out_w || d.kh < 1 || d.sh < 1)
          return set_err(c, GEMEL_E_SCHEMA, at + "roi align needs (proposals, 1..4 maps), square output, sampling");
        int Cf = -1;
        for (int k = 1; k < d.n_in; ++k) {
          int Ck, Hk, Wk;
          in_shape(k, Ck, Hk, Wk);
          if (d.in[k] < 0 || m.layers[d.in[k]].flat || m.layers[d.in[k]].rows != 1 || (Cf >= 0 && Ck != Cf) || Ck % 8)
            return set_err(c, GEMEL_E_SCHEMA, at + "roi align maps must be spatial, equal C (multiple of 8)");
          Cf = Ck;
        }
        L.C = Cf; L.H = d.out_h; L.W = d.out_w;
        L.rows = m.layers[d.in[0]].C / 5;
        break;
      }
      case GEMEL_OP_BOX_POST: {
        int C1, H1, W1, C2, H2, W2;
        in_shape(1, C1, H1, W1);
        in_shape(2, C2, H2, W2);
        if (d.n_in != 3 || d.cout < 2 || !d.param[0] || d.in[2] < 0 || m.layers[d.in[2]].d.op != GEMEL_OP_RPN_MERGE ||
            C != d.cout || C1 != 4 * d.cout || L.rows != C2 / 5 || m.layers[d.in[1]].rows != L.rows)
          return set_err(c, GEMEL_E_SCHEMA, at + "box post needs (logits [classes], deltas [4 classes]) per proposal");
        L.anchors.assign(d.param[0], d.param[0] + 4);   // box-coder weights
        L.C = L.rows * (d.cout - 1) * 6; L.H = 1; L.W = 1; L.flat = true;
        L.rows = 1;
        break;
      }
      case GEMEL_OP_DET_CANDIDATES: {
        const bool flat_in = d.in[0] >= 0 && m.layers[d.in[0]].flat;
        const int need = d.kh == 0 ? 6 : 7;
        if (d.n_in != 1 || !flat_in || d.kh < 0 || d.kh > 2 || d.cin < need || (d.kh == 0 && d.cin != 6) ||
            C % d.cin || !(d.neg_slope >= 0.f) || !(d.eps >= 0.f))
          return set_err(c, GEMEL_E_SCHEMA, at + "det candidates needs a flat input of rows (format 0: 6 fields, "
                                                 "1/2: >= 7), score threshold >= 0, min size >= 0");
        L.C = C / d.cin * 6; L.H = 1; L.W = 1; L.flat = true;
        break;
      }
      case GEMEL_OP_DET_NMS: {
        const int t = d.in[0];
        if (d.n_in != 1 || t < 0 || m.layers[t].d.op != GEMEL_OP_TOPK || m.layers[t].d.cin != 6 ||
            m.layers[t].d.kh != 4 || m.layers[t].d.in[0] < 0 ||
            m.layers[m.layers[t].d.in[0]].d.op != GEMEL_OP_DET_CANDIDATES || d.cout < 1 || d.cout > 1024 ||
            !(d.neg_slope >= 0.f))
          return set_err(c, GEMEL_E_SCHEMA, at + "det nms needs a topk (score column 4) over det candidates, "
                                                 "1 <= max detections <= 1024, IoU threshold >= 0");
        L.C = d.cout * 6; L.H = 1; L.W = 1; L.flat = true;
        break;
      }
      case GEMEL_OP_TOPK: {
        const bool flat_in = d.in[0] >= 0 && m.layers[d.in[0]].flat;
        if (d.n_in != 1 || !flat_in || d.cin < 1 || d.cout < 1 || d.cout > 1024 || d.kh < 0 || d.kh >= d.cin ||
            C % d.cin)
          return set_err(c, GEMEL_E_SCHEMA, at + "topk needs a flat input of rows of cin fields, k >= 1, kh < cin");
        L.C = d.cout * (d.cin + 1); L.H = 1; L.W = 1; L.flat = true;
        break;
      }
      case GEMEL_OP_YOLO_DECODE: {
        if (d.n_in != 1 || d.kh < 1 || d.kh > 4 || d.cout < 0 || d.cin != d.kh * (5 + d.cout) || d.cin != C)
          return set_err(c, GEMEL_E_SCHEMA, at + "yolo decode needs cin = anchors*(5+classes) = producer channels");
        if (!d.param[0]) return set_err(c, GEMEL_E_SCHEMA, at + "yolo decode anchors missing");
        L.anchors.assign(d.param[0], d.param[0] + 2 * d.kh);
        L.C = d.kh * H * W * (5 + d.cout); L.H = 1; L.W = 1; L.flat = true;
        break;
      }
      default:
        return set_err(c, GEMEL_E_SCHEMA, at + "unknown op");
    }
    if (is_param_op(d.op) && L.tie >= 0) {
      L.param_id = m.layers[L.tie].param_id;   // applies the tied layer's parameters
    } else if (is_param_op(d.op)) {
      ParamLayer p;
      p.model = mid; p.pos = i; p.op = d.op;
      p.bytes = param_elems(d) * 2;
      if (d.op == GEMEL_OP_BATCHNORM2D) {
        p.gamma.assign(d.param[0], d.param[0] + d.cin);
        p.beta.assign(d.param[1], d.param[1] + d.cin);
        p.mean.assign(d.param[2], d.param[2] + d.cin);
        p.var.assign(d.param[3], d.param[3] + d.cin);
      } else {
        const uint64_t nw = param_elems(d) - (d.bias ? d.cout : 0);
        p.w.assign(d.param[0], d.param[0] + nw);
        if (d.bias) p.b.assign(d.param[1], d.param[1] + d.cout);
      }
      L.param_id = int(c->params.size() + newp.size());
      newp.push_back(std::move(p));
    }
    m.layers.push_back(L);
  }
  for (auto& p : newp) c->params.push_back(std::move(p));
  c->models.push_back(std::move(m));
  if (model_id) *model_id = mid;
  return GEMEL_OK;
}

gemel_status gemel_find_shareable(gemel_ctx ctx, gemel_group* groups, int32_t cap, int32_t* n_groups,
                                  gemel_appearance* apps, int32_t app_cap, int32_t* n_apps) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c || !n_groups || !n_apps) return GEMEL_E_ARG;
  std::map<std::vector<int64_t>, std::vector<std::pair<int, int>>> classes;
  for (int mi = 0; mi < int(c->models.size()); ++mi)
    for (int pos = 0; pos < int(c->models[mi].layers.size()); ++pos) {
      const auto& d = c->models[mi].layers[pos].d;
      if (is_param_op(d.op) && c->models[mi].layers[pos].tie < 0) classes[signature(d)].push_back({mi, pos});
    }
  struct G { std::vector<std::pair<int, int>> apps; uint64_t per; int op; };
  std::vector<G> gs;
  for (auto& kv : classes) {
    if (kv.second.size() < 2) continue;
    G g;
    g.apps = kv.second;
    std::sort(g.apps.begin(), g.apps.end());
    const auto& d = c->models[g.apps[0].first].layers[g.apps[0].second].d;
    g.per = param_elems(d) * 2;
    g.op = d.op;
    gs.push_back(std::move(g));
  }
  std::sort(gs.begin(), gs.end(), [](const G& a, const G& b) {
    const uint64_t ta = a.per * a.apps.size(), tb = b.per * b.apps.size();
    if (ta != tb) return ta > tb;
    if (a.per != b.per) return a.per > b.per;
    return a.apps[0] < b.apps[0];
  });
  int total_apps = 0;
  for (auto& g : gs) total_apps += int(g.apps.size());
  *n_groups = int(gs.size());
  *n_apps = total_apps;
  if (cap == 0 && app_cap == 0) return GEMEL_OK;
  if (cap < int(gs.size()) || app_cap < total_apps || !groups || !apps)
    return set_err(c, GEMEL_E_SMALLBUF, "find_shareable: buffers too small");
  int off = 0;
  for (size_t i = 0; i < gs.size(); ++i) {
    gemel_group& o = groups[i];
    std::memset(&o, 0, sizeof(o));
    o.op = gs[i].op;
    o.n_apps = int(gs[i].apps.size());
    o.app_offset = off;
    o.per_bytes = gs[i].per;
    o.total_bytes = gs[i].per * gs[i].apps.size();
    o.reclaimable = gs[i].per * (gs[i].apps.size() - 1);
    for (auto& a : gs[i].apps) apps[off++] = {a.first, a.second};
  }
  return GEMEL_OK;
}

gemel_status gemel_apply_merge(gemel_ctx ctx, const gemel_merge_group* groups, int32_t n, uint64_t* bytes_saved) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c || n < 0 || (n > 0 && !groups)) return GEMEL_E_ARG;
  if (c->planned) return set_err(c, GEMEL_E_STATE, "apply_merge after plan");
  // validate everything first (all or nothing)
  std::map<std::pair<int, int>, int> seen;
  uint64_t saved = 0;
  for (int gi = 0; gi < n; ++gi) {
    const gemel_merge_group& g = groups[gi];
    std::ostringstream pre;
    pre << "merge group " << gi << ": ";
    if (g.n_members < 2 || !g.members) return set_err(c, GEMEL_E_MERGE, pre.str() + "fewer than 2 members");
    if (g.source < 0 || g.source >= g.n_members) return set_err(c, GEMEL_E_MERGE, pre.str() + "bad source index");
    std::vector<int64_t> sig0;
    uint64_t per = 0;
    for (int k = 0; k < g.n_members; ++k) {
      const int mi = g.members[k].model_id, pos = g.members[k].op_pos;
      if (mi < 0 || mi >= int(c->models.size()) || pos < 0 || pos >= int(c->models[mi].layers.size()))
        return set_err(c, GEMEL_E_MERGE, pre.str() + "member id out of range");
      const auto& L = c->models[mi].layers[pos];
      if (!is_param_op(L.d.op) || L.tie >= 0)
        return set_err(c, GEMEL_E_MERGE, pre.str() + where(mi, pos) + "layer has no weights of its own");
      auto s = signature(L.d);
      if (k == 0) { sig0 = s; per = param_elems(L.d) * 2; }
      else if (s != sig0) return set_err(c, GEMEL_E_MERGE, pre.str() + where(mi, pos) + "signature mismatch");
      if (c->params[L.param_id].merge_group >= 0)
        return set_err(c, GEMEL_E_MERGE, pre.str() + where(mi, pos) + "already merged");
      if (seen.count({mi, pos})) return set_err(c, GEMEL_E_MERGE, pre.str() + where(mi, pos) + "member in two groups");
      seen[{mi, pos}] = gi;
    }
    saved += per * uint64_t(g.n_members - 1);
  }
  for (int gi = 0; gi < n; ++gi) {
    const gemel_merge_group& g = groups[gi];
    const int gid = c->n_merge_groups++;
    const auto& sm = g.members[g.source];
    const int src = c->models[sm.model_id].layers[sm.op_pos].param_id;
    for (int k = 0; k < g.n_members; ++k) {
      const int pid = c->models[g.members[k].model_id].layers[g.members[k].op_pos].param_id;
      c->params[pid].merge_group = gid;
      c->params[pid].bound_to = (pid == src) ? -1 : src;
    }
  }
  c->bytes_saved += saved;
  if (bytes_saved) *bytes_saved = saved;
  return GEMEL_OK;
}

gemel_status gemel_incremental_merge(gemel_ctx ctx, gemel_retrain_fn retrain, void* user, gemel_merge_attempt* log,
                                     int32_t log_cap, int32_t* n_attempts, uint64_t* bytes_saved) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c || !retrain || !n_attempts || (log_cap > 0 && !log)) return GEMEL_E_ARG;
  if (c->planned) return set_err(c, GEMEL_E_STATE, "incremental_merge after plan");
  for (const auto& p : c->params)
    if (p.merge_group >= 0) return set_err(c, GEMEL_E_STATE, "incremental_merge needs an unmerged workload");
  int32_t ng = 0, na = 0;
  gemel_status rc = gemel_find_shareable(ctx, nullptr, 0, &ng, nullptr, 0, &na);
  if (rc) return rc;
  std::vector<gemel_group> groups(ng);
  std::vector<gemel_appearance> apps(na);
  if (ng > 0) {
    rc = gemel_find_shareable(ctx, groups.data(), ng, &ng, apps.data(), na, &na);
    if (rc) return rc;
  }
  // running configuration: accepted groups (members = a prefix of the group's sorted
  // appearances: halving keeps the first ceil(n/2), reading R21) + the candidate
  std::vector<std::vector<gemel_appearance>> running;
  std::vector<gemel_merge_group> view;
  uint64_t saved = 0;
  int attempts = 0;
  int i = 0, cur = ng > 0 ? groups[0].n_apps : 0;
  while (i < ng) {
    const gemel_group& G = groups[i];
    running.emplace_back(apps.begin() + G.app_offset, apps.begin() + G.app_offset + cur);
    view.clear();
    for (auto& r : running) view.push_back({r.data(), int32_t(r.size()), 0});
    const int32_t ok = retrain(user, view.data(), int32_t(view.size()));
    if (ok < 0) return set_err(c, GEMEL_E_ARG, "incremental_merge: retraining oracle reported an error");
    if (attempts < log_cap) {
      gemel_merge_attempt& a = log[attempts];
      std::memset(&a, 0, sizeof(a));
      a.group = i;
      a.n_members = cur;
      a.ok = ok ? 1 : 0;
      a.bytes = G.per_bytes * uint64_t(cur);
    }
    ++attempts;
    if (ok) {   // accepted: bind it now (merges are cumulative)
      uint64_t b = 0;
      rc = gemel_apply_merge(ctx, &view.back(), 1, &b);
      if (rc) return rc;
      saved += b;
      ++i;
      cur = i < ng ? groups[i].n_apps : 0;
      continue;
    }
    running.pop_back();
    const int half = (cur + 1) / 2;   // halve; keep it if it still outweighs the next group
    const uint64_t next = i + 1 < ng ? groups[i + 1].total_bytes : 0;
    if (half >= 2 && G.per_bytes * uint64_t(half) > next) {
      cur = half;
    } else {
      ++i;
      cur = i < ng ? groups[i].n_apps : 0;
    }
  }
  *n_attempts = attempts;
  if (bytes_saved) *bytes_saved = saved;
  if (attempts > log_cap && log_cap > 0) return set_err(c, GEMEL_E_SMALLBUF, "incremental_merge: log buffer too small");
  return GEMEL_OK;
}

gemel_status gemel_stats(gemel_ctx ctx, gemel_stats_t* out) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c || !out) return GEMEL_E_ARG;
  std::memset(out, 0, sizeof(*out));
  out->n_models = int(c->models.size());
  out->n_param_layers = int(c->params.size());
  for (auto& p : c->params) {
    out->registered_bytes += p.bytes;
    if (p.bound_to >= 0) out->n_merged_layers++;
  }
  out->planned = c->planned ? 1 : 0;
  out->bytes_saved = c->bytes_saved;
  return GEMEL_OK;
}

}  // extern "C"
