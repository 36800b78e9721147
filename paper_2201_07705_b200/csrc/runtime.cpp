// Device side of the C ABI: arena binding (weight upload, TMA descriptors,
// launch tables, CUDA-graph capture) and the per-step executor.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <sstream>

#include "internal.h"
#include "tmap.h"

namespace gemel {

namespace {

int cuda_err(Ctx* c, cudaError_t e, const char* what) {
  std::ostringstream o;
  o << what << ": " << cudaGetErrorString(e);
  return set_err(c, GEMEL_E_CUDA, o.str());
}

#define CUDA_TRY(expr, what)                       \
  do {                                             \
    cudaError_t e_ = (expr);                       \
    if (e_ != cudaSuccess) return cuda_err(c, e_, what); \
  } while (0)

uint16_t f2bf(float f) {   // round to nearest even
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7F800000u) == 0x7F800000u) return uint16_t(u >> 16);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return uint16_t(u >> 16);
}

const ParamLayer& src_param(const Ctx* c, int pid) {
  const ParamLayer& p = c->params[pid];
  return p.bound_to >= 0 ? c->params[p.bound_to] : p;
}

// Device weight [N, Ktot] bf16, K = (tap, channel) with channels padded to cin_k.
// Linear: columns permuted from PyTorch's NCHW flatten order (c, h, w) to the
// NHWC storage order (h, w, c) of the input value -- an exact reordering.
void build_weight(const Ctx* c, const DevWeight& w, std::vector<uint16_t>& out) {
  const ParamLayer& P = c->params[w.param_id];
  out.assign(size_t(w.N) * w.Ktot, 0);
  if (w.cols) {
    // im2col columns k = (r * kw + s) * Cf + c over the Cf frame channels
    const Layer* L = nullptr;
    for (const auto& l : c->models[P.model].layers)
      if (l.param_id == w.param_id) L = &l;
    const int Cf = L->d.cin, taps = L->d.kh * L->d.kw;
    for (int n = 0; n < w.N; ++n)
      for (int ci = 0; ci < Cf; ++ci)
        for (int t = 0; t < taps; ++t)
          out[size_t(n) * w.Ktot + size_t(t) * Cf + ci] = f2bf(P.w[(size_t(n) * Cf + ci) * taps + t]);
  } else if (!w.linear) {
    const int taps = w.kh * w.kw;
    for (int n = 0; n < w.N; ++n)
      for (int ci = 0; ci < w.Cin; ++ci)
        for (int t = 0; t < taps; ++t)
          out[size_t(n) * w.Ktot + size_t(t) * w.cin_k + ci] = f2bf(P.w[(size_t(n) * w.Cin + ci) * taps + t]);
  } else {
    const int C = w.flatC, H = w.flatH, W = w.flatW, Cp = w.flatCp;
    for (int n = 0; n < w.N; ++n)
      for (int ci = 0; ci < C; ++ci)
        for (int h = 0; h < H; ++h)
          for (int x = 0; x < W; ++x)
            out[size_t(n) * w.Ktot + (size_t(h) * W + x) * Cp + ci] =
                f2bf(P.w[size_t(n) * w.Cin + (size_t(ci) * H + h) * W + x]);
  }
}

// Folded epilogue of a GEMM node: y = acc * scale + shift, with
// scale = gamma / sqrt(var + eps), shift = beta - mean * scale + bias * scale
// (no BN: scale = 1, shift = bias).  Uses the merged (source) weights.
void build_epilogue(const Ctx* c, const Node& g, std::vector<float>& sc, std::vector<float>& sh) {
  const Model& M = c->models[g.model];
  const ParamLayer& W = src_param(c, M.layers[g.layer].param_id);
  sc.assign(g.Cout, 1.f);
  sh.assign(g.Cout, 0.f);
  std::vector<double> bias(g.Cout, 0.0);
  if (!W.b.empty())
    for (int i = 0; i < g.Cout; ++i) bias[i] = W.b[i];
  if (g.bn >= 0) {
    const ParamLayer& B = src_param(c, M.layers[g.bn].param_id);
    const double eps = M.layers[g.bn].d.eps;
    for (int i = 0; i < g.Cout; ++i) {
      const double s = double(B.gamma[i]) / std::sqrt(double(B.var[i]) + eps);
      sc[i] = float(s);
      sh[i] = float(double(B.beta[i]) - double(B.mean[i]) * s + bias[i] * s);
    }
  } else {
    for (int i = 0; i < g.Cout; ++i) sh[i] = float(bias[i]);
  }
}

// Swap copies of the weights first read by launch `li`, on the copy stream, each
// after the launch that last read the ring slot it overwrites; then `ready[li]`.
int issue_swap_copies(Ctx* c, size_t li) {
  cudaStream_t cs = static_cast<cudaStream_t>(c->copy_stream);
  const size_t nl = c->launches.size();
  bool any = false;
  for (int wk : c->swap_order) {
    const DevWeight& w = c->dweights[wk];
    if (w.first_launch != int(li)) continue;
    if (w.wait_launch >= 0)
      CUDA_TRY(cudaStreamWaitEvent(cs, static_cast<cudaEvent_t>(c->swap_events[w.wait_launch]), 0), "swap wait");
    if (c->opt.weight_source == GEMEL_SOURCE_PEER && c->opt.source_device != c->opt.device)   // NVLink peer read
      CUDA_TRY(cudaMemcpyPeerAsync(c->w_dev + w.offset, c->opt.device, c->host_w[wk], c->opt.source_device, w.bytes, cs),
               "peer swap copy");
    else
      CUDA_TRY(cudaMemcpyAsync(c->w_dev + w.offset, c->host_w[wk], w.bytes,
                               c->opt.weight_source == GEMEL_SOURCE_PEER ? cudaMemcpyDeviceToDevice
                                                                         : cudaMemcpyHostToDevice, cs),
               "swap copy");
    any = true;
  }
  if (any) CUDA_TRY(cudaEventRecord(static_cast<cudaEvent_t>(c->swap_events[nl + li]), cs), "swap ready");
  return GEMEL_OK;
}

bool launch_has_copies(const Ctx* c, size_t li) {
  for (int wk : c->swap_order)
    if (c->dweights[wk].first_launch == int(li)) return true;
  return false;
}

// Per consumer m-tile and dependency: the band [lo, hi] of producer m-tiles holding
// the rows it reads -- the receptive field of its output pixels in the producer's
// output (conv input), all pixels of its images (linear over a flattened value),
// or the same pixels (residual).  A producer row is (member's segment start in
// the producer problem) + pixel index in that member's value.
int build_dep_ranges(Ctx* c, const Launch& L, const GemmProblem* probs, uint8_t* meta) {
  std::map<int, std::pair<int, int64_t>> src;   // value -> (local problem, first row)
  for (size_t k = 0; k < L.items.size(); ++k) {
    int64_t m0 = 0;
    for (int nid : c->problems[L.items[k]].members) {
      const Node& g = c->nodes[nid];
      src[g.out_value] = {int(k), m0};
      m0 += int64_t(g.B) * g.Ho * g.Wo;
    }
  }
  int32_t* tab = reinterpret_cast<int32_t*>(meta + L.dep_off);
  for (size_t k = 0; k < L.items.size(); ++k) {
    const Problem& pr = c->problems[L.items[k]];
    const GemmProblem& P = probs[k];
    const int nd = P.n_deps;
    if (nd == 0) continue;
    int32_t* t = tab + pr.dep_idx;
    for (int mt = 0; mt < P.m_tiles; ++mt) {
      std::vector<int64_t> lo(nd, INT64_MAX), hi(nd, -1);
      const int64_t r0 = int64_t(mt) * GEMM_BM, r1 = std::min<int64_t>(r0 + GEMM_BM, P.M);
      int64_t mb = 0;
      for (int nid : pr.members) {
        const Node& g = c->nodes[nid];
        const int64_t me = mb + int64_t(g.B) * g.Ho * g.Wo;
        const int64_t a = std::max(r0, mb) - mb, b = std::min(r1, me) - mb;   // member rows [a, b)
        mb = me;
        if (a >= b) continue;
        auto need = [&](int v, int64_t p0, int64_t p1) {
          auto it = src.find(v);
          if (it == src.end()) return;
          int d = 0;
          while (d < nd && P.deps[d] != it->second.first) ++d;
          if (d == nd) return;
          lo[d] = std::min(lo[d], (it->second.second + p0) / GEMM_BM);
          hi[d] = std::max(hi[d], (it->second.second + p1) / GEMM_BM);
        };
        if (g.in_value >= 0 && !g.cols) {
          const Value& vi = c->values[g.in_value];
          const int64_t HW = int64_t(vi.H) * vi.W;
          if (g.Ho == 1 && g.Wo == 1 && g.H == 1 && g.W == 1) {   // linear: whole images
            need(g.in_value, a * HW, b * HW - 1);
          } else {
            auto corner = [&](int64_t o, bool last) {
              const int64_t img = o / (int64_t(g.Ho) * g.Wo), r = o % (int64_t(g.Ho) * g.Wo);
              const int oh = int(r / g.Wo), ow = int(r % g.Wo);
              int ih = oh * g.sh - g.ph + (last ? (g.kh - 1) * g.dh : 0);
              int iw = ow * g.sw - g.pw + (last ? (g.kw - 1) * g.dw : 0);
              ih = std::min(std::max(ih, 0), vi.H - 1);
              iw = std::min(std::max(iw, 0), vi.W - 1);
              return img * HW + int64_t(ih) * vi.W + iw;
            };
            need(g.in_value, corner(a, false), corner(b - 1, true));
          }
        }
        if (g.res_value >= 0 && g.res_up > 1) {   // coarse rows of the nearest-upsampled residual
          // o -> coarse pixel is not monotonic within a fine row band (x / up restarts every
          // fine row), so the band covers WHOLE coarse rows: from the start of the coarse row
          // of the first fine row to the end of the coarse row of the last one.
          const Value& vr = c->values[g.res_value];
          auto coarse_row = [&](int64_t o, bool last) {
            const int64_t img = o / (int64_t(g.Ho) * g.Wo), r = o % (int64_t(g.Ho) * g.Wo);
            return img * vr.H * vr.W + (r / g.Wo) / g.res_up * vr.W + (last ? vr.W - 1 : 0);
          };
          need(g.res_value, coarse_row(a, false), coarse_row(b - 1, true));
        } else if (g.res_value >= 0) {
          need(g.res_value, a, b - 1);
        }
      }
      for (int d = 0; d < nd; ++d) {
        t[(mt * nd + d) * 2 + 0] = hi[d] < 0 ? 0 : int32_t(lo[d]);
        t[(mt * nd + d) * 2 + 1] = hi[d] < 0 ? -1 : int32_t(hi[d]);
      }
    }
  }
  return GEMEL_OK;
}

// Task tables of the Faster R-CNN stages (include/gemel.h RPN_LEVEL .. BOX_POST).
int build_detect_tasks(Ctx* c, Launch& L, uint8_t* base) {
  int blocks = 0;
  int64_t work = 0;
  L.topk_rows = 0;   // NK_RPN: the most anchors of a level (the selection's staging size)
  for (size_t k = 0; k < L.items.size(); ++k) {
    const Node& g = c->nodes[L.items[k]];
    const Model& Mo = c->models[g.model];
    const Layer& Ly = Mo.layers[g.layer];
    const Value& vo = c->values[g.out_value];
    auto ptr = [&](int v) { return c->act_dev + c->values[v].offset; };
    if (L.kind == NK_RPN) {
      RpnTask& T = reinterpret_cast<RpnTask*>(base)[k];
      std::memset(&T, 0, sizeof(T));
      const Value& vc = c->values[g.ins[0]];
      const Value& vb = c->values[g.ins[1]];
      T.cls = reinterpret_cast<const float*>(ptr(g.ins[0]));
      T.box = reinterpret_cast<const float*>(ptr(g.ins[1]));
      T.dst = reinterpret_cast<float*>(ptr(g.out_value));
      T.n = vc.B; T.h = vc.H; T.w = vc.W; T.A = Ly.d.kh; T.cpc = vc.Cp; T.cpb = vb.Cp;
      T.K = vo.C / 6;
      T.stride_y = Mo.in_h / vc.H;
      T.stride_x = Mo.in_w / vc.W;
      for (int a = 0; a < T.A; ++a) {   // AnchorGenerator.generate_anchors, float32 like torchvision
        const float size = Ly.anchors[2 * a], r = Ly.anchors[2 * a + 1];
        const float hr = std::sqrt(r), wr = 1.f / hr;
        const float ws = wr * size, hs = hr * size;
        T.base[a][0] = std::nearbyint(-ws / 2.f);
        T.base[a][1] = std::nearbyint(-hs / 2.f);
        T.base[a][2] = std::nearbyint(ws / 2.f);
        T.base[a][3] = std::nearbyint(hs / 2.f);
      }
      T.nms = Ly.d.neg_slope;
      T.min_size = Ly.d.eps;
      T.img_w = float(Mo.in_w);
      T.img_h = float(Mo.in_h);
      T.dst_pitch = vo.Cp;
      T.block_begin = blocks;
      blocks += T.n;
      L.topk_rows = std::max(L.topk_rows, T.h * T.w * T.A);
    } else if (L.kind == NK_RPNM) {
      RpnMergeTask& T = reinterpret_cast<RpnMergeTask*>(base)[k];
      std::memset(&T, 0, sizeof(T));
      T.n_levels = int(g.ins.size());
      for (int l = 0; l < T.n_levels; ++l) {
        const Value& vl = c->values[g.ins[l]];
        T.src[l] = reinterpret_cast<const float*>(ptr(g.ins[l]));
        T.src_pitch[l] = vl.Cp;
        T.k[l] = vl.C / 6;
      }
      T.dst = reinterpret_cast<float*>(ptr(g.out_value));
      T.dst_pitch = vo.Cp;
      T.n = vo.B;
      T.post_n = Ly.d.cout;
      T.block_begin = blocks;
      blocks += T.n;
    } else if (L.kind == NK_ROI) {
      RoiTask& T = reinterpret_cast<RoiTask*>(base)[k];
      std::memset(&T, 0, sizeof(T));
      const Value& vp = c->values[g.ins[0]];
      T.props = reinterpret_cast<const float*>(ptr(g.ins[0]));
      T.props_pitch = vp.Cp;
      T.n_maps = int(g.ins.size()) - 1;
      int lv0 = 0;
      for (int l = 0; l < T.n_maps; ++l) {
        const Value& vm = c->values[g.ins[1 + l]];
        T.map[l] = ptr(g.ins[1 + l]);
        T.mh[l] = vm.H; T.mw[l] = vm.W;
        // MultiScaleRoIAlign._infer_scale: 2^round(log2(feature / image))
        const int e = int(std::lround(std::log2(double(vm.H) / double(Mo.in_h))));
        T.scale[l] = float(std::ldexp(1.0, e));
        if (l == 0) lv0 = -e;
        if (vm.Cp != c->values[g.ins[1]].Cp) return set_err(c, GEMEL_E_STATE, "bind: roi maps differ in pitch");
      }
      T.k_min = lv0;
      T.cp = c->values[g.ins[1]].Cp;
      T.C = c->values[g.ins[1]].C;
      T.n = vp.B; T.R = Ly.rows; T.out = Ly.d.out_h; T.sampling = Ly.d.kh;
      T.canon_scale = float(Ly.d.sh);
      T.canon_level = float(Ly.d.sw);
      T.dst = ptr(g.out_value);
      T.cpd = vo.Cp;
      T.work_begin = work;   // first proposal of this task (one CTA per proposal)
      T.work = int64_t(vo.B);
      work += T.work;
    } else {
      BoxPostTask& T = reinterpret_cast<BoxPostTask*>(base)[k];
      std::memset(&T, 0, sizeof(T));
      const Value& vc = c->values[g.ins[0]];
      const Value& vb = c->values[g.ins[1]];
      const Value& vp = c->values[g.ins[2]];
      T.cls = reinterpret_cast<const float*>(ptr(g.ins[0]));
      T.box = reinterpret_cast<const float*>(ptr(g.ins[1]));
      T.props = reinterpret_cast<const float*>(ptr(g.ins[2]));
      T.dst = reinterpret_cast<float*>(ptr(g.out_value));
      T.n = vp.B; T.R = vp.C / 5; T.classes = Ly.d.cout; T.cpc = vc.Cp; T.cpb = vb.Cp;
      T.props_pitch = vp.Cp;
      T.dst_pitch = vo.Cp;
      for (int j = 0; j < 4; ++j) T.wts[j] = Ly.anchors[j];
      T.img_w = float(Mo.in_w);
      T.img_h = float(Mo.in_h);
      T.work_begin = work;
      work += int64_t(T.n) * T.R;
    }
  }
  L.det_blocks = blocks;
  L.det_work = work;
  return GEMEL_OK;
}

int run_launches(Ctx* c, cudaStream_t st, bool timed, int buf = 0) {
  const bool swap = !c->swap_order.empty();
  const size_t nl = c->launches.size();
  if (swap) {   // fork the copy stream off the step (joins it into a graph capture too)
    cudaEvent_t start = static_cast<cudaEvent_t>(c->swap_events[2 * nl]);
    CUDA_TRY(cudaEventRecord(start, st), "swap start");
    CUDA_TRY(cudaStreamWaitEvent(static_cast<cudaStream_t>(c->copy_stream), start, 0), "swap fork");
    int rc = issue_swap_copies(c, 0);
    if (rc) return rc;
  }
  for (size_t li = 0; li < c->launches.size(); ++li) {
    const Launch& L = c->launches[li];
    if (swap && launch_has_copies(c, li))
      CUDA_TRY(cudaStreamWaitEvent(st, static_cast<cudaEvent_t>(c->swap_events[nl + li]), 0), "swap join");
    if (timed) CUDA_TRY(cudaEventRecord(static_cast<cudaEvent_t>(c->events[2 * li]), st), "event record");
    int rc = 0;
    uint8_t* meta = c->meta_dev + L.meta_off;
    if (L.kind == NK_GEMM && L.stem) {
      // one kernel per first-conv problem: each runs with its own shared-memory footprint
      // (a 7x7/s2 stem needs ~4x the smem of a 3x3 one, which would cap the occupancy of both)
      const StemTask* tasks = reinterpret_cast<const StemTask*>(c->meta_dev + L.stem_off) + (buf ? L.stem_tasks : 0);
      int64_t t0 = 0;
      for (int pid : L.items) {
        const Problem& pr = c->problems[pid];
        const DevWeight& w = c->dweights[pr.wkey];
        const Node& g0 = c->nodes[pr.members[0]];
        int64_t tiles = 0;
        int in_slot = 0;
        bool direct = false;
        for (int nid : pr.members) {
          const Node& g = c->nodes[nid];
          const gemel_layer& d = c->models[g.model].layers[g.layer].d;
          const int sub = stem_sub(stem_kp(d.kh, d.kw));
          tiles += stem_tile_count(g.B, g.Ho, g.Wo, sub);
          const int sb = stem_in_slot_bytes(d.kh, d.sh, g.Wo, c->models[g.model].in_w, sub);
          direct = direct || sb == 0 || (c->frame_off[c->models[g.model].stream_id] % 16) ||
                   (c->frame_off2.size() > size_t(c->models[g.model].stream_id) &&
                    c->frame_off2[c->models[g.model].stream_id] % 16);
          in_slot = std::max(in_slot, sb);
        }
        const gemel_layer& d0 = c->models[g0.model].layers[g0.layer].d;
        rc = launch_stem(tasks, L.stem_tasks, t0, tiles, w.N, stem_kp(d0.kh, d0.kw), direct ? 0 : in_slot,
                         c->sm_count, st);
        if (rc) break;
        t0 += tiles;
      }
    } else if (L.kind == NK_GEMM) {
      int32_t* cnt = reinterpret_cast<int32_t*>(c->meta_dev + L.cnt_off);
      CUDA_TRY(cudaMemsetAsync(cnt, 0, size_t(L.n_counters) * 4, st), "reset scheduler counters");
      GemmLaunch G{reinterpret_cast<const GemmProblem*>(meta), reinterpret_cast<const GemmSeg*>(c->meta_dev + L.seg_off),
                   cnt, li < c->trace_dev.size() ? static_cast<unsigned long long*>(c->trace_dev[li]) : nullptr,
                   L.n_probs, L.total_tiles, L.total_items, L.bn_max, L.stages, L.cg, L.acc_w, L.epi_flags,
                   c->gemm_dbg};
      rc = gemm_launch(G, L.grid, st);
    } else if (L.kind == NK_PRE) {
      // the task table reading staging buffer `buf` (the second table follows the first)
      const PreTask* tasks = reinterpret_cast<const PreTask*>(meta) + (buf ? L.n_pre_tasks : 0);
      if (L.n_cols > 0) rc = launch_ingest_cols(tasks, L.n_cols, L.cols_blocks, L.cols_smem, st);
      if (!rc && L.n_pre_tasks > L.n_cols)
        rc = launch_preprocess(tasks + L.n_cols, L.n_pre_tasks - L.n_cols, L.pre_pixels, st);
    } else if (L.kind == NK_ADD) {
      int64_t total = 0;
      for (int nid : L.items) total += int64_t(c->values[c->nodes[nid].out_value].bytes / 16);
      rc = launch_add(reinterpret_cast<const AddTask*>(meta), int(L.items.size()), total, st);
    } else if (L.kind == NK_MISC) {
      rc = launch_misc(reinterpret_cast<const MiscTask*>(meta), L.misc_tasks, L.misc_work, st);
    } else if (L.kind == NK_TOPK) {
      rc = launch_topk(reinterpret_cast<const TopkTask*>(meta), int(L.items.size()), L.topk_blocks, L.topk_rows, st);
    } else if (L.kind == NK_RPN) {
      rc = launch_rpn_level(reinterpret_cast<const RpnTask*>(meta), int(L.items.size()), L.det_blocks, L.topk_rows, st);
    } else if (L.kind == NK_RPNM) {
      rc = launch_rpn_merge(reinterpret_cast<const RpnMergeTask*>(meta), int(L.items.size()), L.det_blocks, st);
    } else if (L.kind == NK_ROI) {
      rc = launch_roi_align(reinterpret_cast<const RoiTask*>(meta), int(L.items.size()), L.det_work, st);
    } else if (L.kind == NK_BOXP) {
      rc = launch_box_post(reinterpret_cast<const BoxPostTask*>(meta), int(L.items.size()), L.det_work, st);
    } else if (L.kind == NK_NMS) {
      rc = launch_det_nms(reinterpret_cast<const NmsTask*>(meta), int(L.items.size()), L.det_blocks, st);
    } else {
      int64_t total = 0;
      for (int nid : L.items) {
        const Value& v = c->values[c->nodes[nid].out_value];
        total += int64_t(v.B) * v.H * v.W * (v.Cp / 8);
      }
      rc = launch_pool(reinterpret_cast<const PoolTask*>(meta), int(L.items.size()), total, st);
    }
    if (rc) return cuda_err(c, cudaError_t(rc), "kernel launch");
    if (timed) CUDA_TRY(cudaEventRecord(static_cast<cudaEvent_t>(c->events[2 * li + 1]), st), "event record");
    if (timed && c->sync_each) {   // developer (GEMEL_SYNC_EACH): locate a hanging launch
      std::fprintf(stderr, "gemel: launch %zu (kind %d) issued\n", li, L.kind);
      CUDA_TRY(cudaStreamSynchronize(st), "sync each");
      std::fprintf(stderr, "gemel: launch %zu done\n", li);
    }
    if (swap) {   // this launch's slots may be refilled; prefetch the next launch's weights
      CUDA_TRY(cudaEventRecord(static_cast<cudaEvent_t>(c->swap_events[li]), st), "swap done");
      if (li + 1 < nl) {
        int rc2 = issue_swap_copies(c, li + 1);
        if (rc2) return rc2;
      }
    }
  }
  return GEMEL_OK;
}

}  // namespace

void release_device(Ctx* c) {
  if (c->graph_exec) cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(c->graph_exec));
  c->graph_exec = nullptr;
  if (c->graph_exec2) cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(c->graph_exec2));
  c->graph_exec2 = nullptr;
  for (int b = 0; b < 2; ++b) {
    if (c->in_ready[b]) cudaEventDestroy(static_cast<cudaEvent_t>(c->in_ready[b]));
    if (c->buf_free[b]) cudaEventDestroy(static_cast<cudaEvent_t>(c->buf_free[b]));
    c->in_ready[b] = c->buf_free[b] = nullptr;
  }
  if (c->dev_frames_ready) cudaEventDestroy(static_cast<cudaEvent_t>(c->dev_frames_ready));
  c->dev_frames_ready = nullptr;
  if (c->in_stream) cudaStreamDestroy(static_cast<cudaStream_t>(c->in_stream));
  c->in_stream = nullptr;
  c->parity = 0;
  if (c->meta_dev) cudaFree(c->meta_dev);
  c->meta_dev = nullptr;
  for (void* e : c->events) cudaEventDestroy(static_cast<cudaEvent_t>(e));
  c->events.clear();
  for (void* t : c->trace_dev)
    if (t) cudaFree(t);
  c->trace_dev.clear();
  for (void* e : c->swap_events) cudaEventDestroy(static_cast<cudaEvent_t>(e));
  c->swap_events.clear();
  for (void* h : c->host_w) {
    if (!h) continue;
    if (c->opt.weight_source == GEMEL_SOURCE_PEER) cudaFree(h);   // a device allocation (setup, not the hot path)
    else cudaFreeHost(h);
  }
  c->host_w.clear();
  if (c->copy_stream) cudaStreamDestroy(static_cast<cudaStream_t>(c->copy_stream));
  c->copy_stream = nullptr;
}

int bind(Ctx* c, void* wdev, uint64_t wb, void* adev, uint64_t ab) {
  if (!c->planned) return set_err(c, GEMEL_E_STATE, "bind before plan");
  if (c->opt.flags & GEMEL_FLAG_DRY_PLAN) return set_err(c, GEMEL_E_STATE, "bind on a dry-plan context");
  if (!wdev || !adev || wb < c->w_bytes || ab < c->act_bytes)
    return set_err(c, GEMEL_E_NOMEM, "bind: arenas smaller than planned");
  if ((reinterpret_cast<uintptr_t>(wdev) | reinterpret_cast<uintptr_t>(adev)) & 255)
    return set_err(c, GEMEL_E_ARG, "bind: arenas must be 256-byte aligned");
  CUDA_TRY(cudaSetDevice(c->opt.device), "cudaSetDevice");
  if (c->opt.weight_source == GEMEL_SOURCE_PEER && c->opt.source_device != c->opt.device) {
    int n_dev = 0, can = 0;
    CUDA_TRY(cudaGetDeviceCount(&n_dev), "device count");
    if (c->opt.source_device < 0 || c->opt.source_device >= n_dev)
      return set_err(c, GEMEL_E_ARG, "bind: weight source device out of range");
    CUDA_TRY(cudaDeviceCanAccessPeer(&can, c->opt.device, c->opt.source_device), "peer query");
    if (can) {   // direct NVLink reads by the copy engine
      const cudaError_t e = cudaDeviceEnablePeerAccess(c->opt.source_device, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return cuda_err(c, e, "enable peer access");
      cudaGetLastError();
    }
  }
  release_device(c);
  c->w_dev = static_cast<uint8_t*>(wdev);
  c->act_dev = static_cast<uint8_t*>(adev);
  c->gemm_dbg = std::getenv("GEMEL_GEMM_DBG") ? std::atoi(std::getenv("GEMEL_GEMM_DBG")) : 0;   // developer probes
  c->sync_each = std::getenv("GEMEL_SYNC_EACH") != nullptr;
  CUDA_TRY(cudaMemset(c->act_dev, 0, c->act_bytes), "zero activation arena");

  // weights (merged tensors once) + per-node epilogue vectors
  std::vector<uint16_t> hw;
  c->host_w.assign(c->dweights.size(), nullptr);
  for (size_t i = 0; i < c->dweights.size(); ++i) {
    const DevWeight& w = c->dweights[i];
    build_weight(c, w, hw);
    if (w.swapped && c->opt.weight_source == GEMEL_SOURCE_PEER) {
      // paged every step from a peer GPU's HBM (N4): the weight store lives on source_device
      CUDA_TRY(cudaSetDevice(c->opt.source_device), "cudaSetDevice source");
      cudaError_t e = cudaMalloc(&c->host_w[i], w.bytes);
      if (e == cudaSuccess) e = cudaMemcpy(c->host_w[i], hw.data(), w.bytes, cudaMemcpyHostToDevice);
      cudaSetDevice(c->opt.device);
      CUDA_TRY(e, "peer weight store");
    } else if (w.swapped) {   // streamed every step from pinned host memory into its ring slot
      CUDA_TRY(cudaHostAlloc(&c->host_w[i], w.bytes, cudaHostAllocDefault), "pinned swap buffer");
      std::memcpy(c->host_w[i], hw.data(), w.bytes);
    } else {
      CUDA_TRY(cudaMemcpy(c->w_dev + w.offset, hw.data(), w.bytes, cudaMemcpyHostToDevice), "upload weights");
    }
  }
  if (!c->swap_order.empty()) {
    cudaStream_t cs;
    CUDA_TRY(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking), "copy stream");
    c->copy_stream = cs;
    for (size_t i = 0; i < 2 * c->launches.size() + 1; ++i) {
      cudaEvent_t e;
      CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "swap event");
      c->swap_events.push_back(e);
    }
  }
  std::vector<float> sc, sh;
  for (auto& g : c->nodes)
    if (g.kind == NK_GEMM) {
      build_epilogue(c, g, sc, sh);
      CUDA_TRY(cudaMemcpy(c->w_dev + g.scale_off, sc.data(), sc.size() * 4, cudaMemcpyHostToDevice), "upload scale");
      CUDA_TRY(cudaMemcpy(c->w_dev + g.shift_off, sh.data(), sh.size() * 4, cudaMemcpyHostToDevice), "upload shift");
    } else if (g.kind == NK_MISC && g.misc == MISC_L2NORM) {
      const std::vector<float>& scale = c->models[g.model].layers[g.layer].anchors;
      CUDA_TRY(cudaMemcpy(c->w_dev + g.scale_off, scale.data(), scale.size() * 4, cudaMemcpyHostToDevice),
               "upload l2norm scale");
    }

  // launch tables
  std::vector<uint8_t> meta(c->meta_bytes, 0);
  void* mdev = nullptr;
  CUDA_TRY(cudaMalloc(&mdev, std::max<uint64_t>(c->meta_bytes, 256)), "cudaMalloc meta");
  c->meta_dev = static_cast<uint8_t*>(mdev);
  for (auto& L : c->launches) {
    uint8_t* base = meta.data() + L.meta_off;
    if (L.kind == NK_GEMM && L.stem) {
      // fused first convs: one StemTask per member, one table per staging buffer
      StemTask* t = reinterpret_cast<StemTask*>(meta.data() + L.stem_off);
      int k = 0;
      int64_t tiles = 0;
      for (int pid : L.items) {
        const Problem& pr = c->problems[pid];
        const DevWeight& w = c->dweights[pr.wkey];
        for (int nid : pr.members) {
          const Node& g = c->nodes[nid];
          const Value& vo = c->values[g.out_value];
          const Model& Mo = c->models[g.model];
          const gemel_layer& d = Mo.layers[g.layer].d;
          if (vo.fp32 || vo.Cp != w.N || w.N % 16 || w.Ktot % 8)
            return set_err(c, GEMEL_E_STATE, "bind: stem output must be bf16 with channel pitch == N");
          if (int64_t(g.B) * std::max<int64_t>(int64_t(g.Ho) * g.Wo, int64_t(Mo.in_h) * Mo.in_w) >= (int64_t(1) << 30))
            return set_err(c, GEMEL_E_UNSUPPORTED, "bind: fused stem member over 2^30 pixels (32-bit tile indexing)");
          StemTask& T = t[k++];
          std::memset(&T, 0, sizeof(T));
          T.src = c->act_dev + c->frame_off[Mo.stream_id];
          T.wgt = c->w_dev + w.offset;
          T.scale = reinterpret_cast<const float*>(c->w_dev + g.scale_off);
          T.shift = reinterpret_cast<const float*>(c->w_dev + g.shift_off);
          T.out = c->act_dev + vo.offset;
          T.tile_begin = tiles;
          T.n_img = g.B; T.h = Mo.in_h; T.w = Mo.in_w; T.ho = g.Ho; T.wo = g.Wo;
          T.kh = d.kh; T.kw = d.kw; T.sh = d.sh; T.sw = d.sw; T.ph = d.ph; T.pw = d.pw;
          T.K = g.Cin; T.ldw = w.Ktot; T.N = w.N;
          T.act = g.act; T.slope = g.slope;
          tiles += stem_tile_count(g.B, g.Ho, g.Wo, stem_sub(stem_kp(d.kh, d.kw)));
        }
      }
      if (k != L.stem_tasks || tiles != L.stem_tiles) return set_err(c, GEMEL_E_STATE, "bind: stem task table mismatch");
      for (int j = 0; j < k; ++j) {   // the same tasks reading staging buffer 1
        StemTask& T2 = t[k + j];
        T2 = t[j];
        const int64_t off0 = static_cast<const uint8_t*>(t[j].src) - c->act_dev;
        for (size_t s2 = 0; s2 < c->frame_off.size(); ++s2)
          if (c->frame_off[s2] == off0) T2.src = c->act_dev + c->frame_off2[s2];
      }
      continue;
    }
    if (L.kind == NK_GEMM) {
      GemmProblem* probs = reinterpret_cast<GemmProblem*>(base);
      GemmSeg* segs = reinterpret_cast<GemmSeg*>(meta.data() + L.seg_off);
      int tile = 0, seg = 0, item = 0;
      for (size_t k = 0; k < L.items.size(); ++k) {
        const Problem& pr = c->problems[L.items[k]];
        const DevWeight& w = c->dweights[pr.wkey];
        const Node& g0 = c->nodes[pr.members[0]];
        const Value& vin = c->values[g0.in_value];
        GemmProblem& P = probs[k];
        std::memset(&P, 0, sizeof(P));
        int64_t M = 0;
        for (int nid : pr.members) M += int64_t(c->nodes[nid].B) * c->nodes[nid].Ho * c->nodes[nid].Wo;
        if (M >= (int64_t(1) << 31)) return set_err(c, GEMEL_E_UNSUPPORTED, "bind: GEMM M exceeds 2^31");
        int rc;
        // A operand: a plain 2-D tiled map whenever A is already a row-major [M, K] matrix
        // (ingest-written im2col rows, flattened linear input, 1x1 stride-1 unpadded conv
        // over the NHWC slab); TMA im2col mode for every other conv.
        const bool pointwise = !w.cols && !w.linear && g0.kh == 1 && g0.kw == 1 && g0.sh == 1 && g0.sw == 1 &&
                               g0.ph == 0 && g0.pw == 0;
        if (w.cols || w.linear) {
          const int K = g0.Cp_in;   // im2col row width / H*W*Cp of the flattened input
          rc = tmap_encode_2d(&P.tmap_a, c->act_dev + vin.offset, uint64_t(K), uint64_t(M), uint64_t(K) * 2, w.chunk,
                              GEMM_BM, w.chunk * 2);
          P.a_tiled = 1;
        } else if (pointwise) {
          rc = tmap_encode_2d(&P.tmap_a, c->act_dev + vin.offset, uint64_t(vin.Cp), uint64_t(M), uint64_t(vin.Cp) * 2,
                              w.chunk, GEMM_BM, w.chunk * 2);
          P.a_tiled = 1;
        } else {
          const int up_w = g0.pw - (g0.kw - 1) * g0.dw, up_h = g0.ph - (g0.kh - 1) * g0.dh;
          rc = tmap_encode_im2col(&P.tmap_a, c->act_dev + vin.offset, pr.n_img, g0.H, g0.W, vin.Cp, vin.Cp, -g0.pw,
                                  -g0.ph, up_w, up_h, w.chunk, GEMM_BM, g0.sw, g0.sh);
        }
        if (rc) return set_err(c, GEMEL_E_CUDA, "bind: im2col tensor map encode failed (" + std::to_string(rc) + ")");
        rc = tmap_encode_2d(&P.tmap_b, c->w_dev + w.offset, w.Ktot, w.N, uint64_t(w.Ktot) * 2, w.chunk, pr.bn / L.cg,
                            w.chunk * 2);   // a CTA pair loads half of the N tile per CTA
        if (rc) return set_err(c, GEMEL_E_CUDA, "bind: weight tensor map encode failed (" + std::to_string(rc) + ")");
        P.M = int(M); P.N = w.N; P.Ktot = w.Ktot;
        P.HoWo = w.cols ? 1 : g0.Ho * g0.Wo;
        P.Wo = w.cols ? 1 : g0.Wo;
        P.sh = g0.sh; P.sw = g0.sw; P.ph = g0.ph; P.pw = g0.pw;
        P.kw = g0.kw; P.dh = g0.dh; P.dw = g0.dw;
        P.cin_k = w.cin_k; P.chunk = w.chunk;
        P.n_sub = w.kh * w.kw * (w.cin_k / w.chunk);
        P.n_kstages = (P.n_sub + GEMM_BK / w.chunk - 1) / (GEMM_BK / w.chunk);
        P.c_oob = (w.linear || w.cols) ? g0.Cp_in : vin.Cp;
        P.bn = pr.bn;
        P.m_tiles = int((M + GEMM_BM - 1) / GEMM_BM);
        P.n_tiles = (w.N + pr.bn - 1) / pr.bn;
        P.tile_begin = tile;
        P.item_begin = item;
        P.run = pr.run;
        P.msub = pr.msub;
        P.ksplit = pr.ksplit;
        P.kst_split = pr.kst_split;
        if (pr.ksplit > 1) {
          P.ws = reinterpret_cast<float*>(c->act_dev + pr.ws_off);
          P.tcnt = reinterpret_cast<int32_t*>(c->meta_dev + L.cnt_off) + pr.tcnt_idx;
        }
        const int m_step = L.cg * P.msub;   // a tile: msub sub-tiles, or a CTA pair's 256 rows
        const int tiles_p = (P.m_tiles + m_step - 1) / m_step * P.n_tiles * P.ksplit;
        tile += tiles_p;
        item += (tiles_p + P.run - 1) / P.run;
        P.seg_begin = seg;
        P.n_seg = int(pr.members.size());
        P.n_deps = int(L.deps[k].size());
        for (int d = 0; d < P.n_deps; ++d) P.deps[d] = L.deps[k][d];
        P.cnt_off = pr.cnt_off;
        P.dep_rng = reinterpret_cast<const int32_t*>(c->meta_dev + L.dep_off) + pr.dep_idx;
        int64_t m0 = 0;
        for (int nid : pr.members) {
          const Node& g = c->nodes[nid];
          const Value& vo = c->values[g.out_value];
          GemmSeg& S = segs[seg++];
          std::memset(&S, 0, sizeof(S));
          S.m_begin = int(m0);
          m0 += int64_t(g.B) * g.Ho * g.Wo;
          S.m_end = int(m0);
          S.act = g.act; S.slope = g.slope; S.res_post = g.res_post;
          S.scale = reinterpret_cast<const float*>(c->w_dev + g.scale_off);
          S.shift = reinterpret_cast<const float*>(c->w_dev + g.shift_off);
          S.out = c->act_dev + vo.offset;
          S.ldo = vo.Cp;
          S.out_fp32 = vo.fp32 ? 1 : 0;
          const uint64_t rows = uint64_t(S.m_end - S.m_begin);
          if (!vo.fp32) {
            rc = tmap_encode_2d(&S.out_map, S.out, uint64_t(g.Cout), rows, uint64_t(vo.Cp) * 2, 32, 32, 64);
            if (rc) return set_err(c, GEMEL_E_CUDA, "bind: output tensor map encode failed");
          }
          if (g.res_value >= 0) {
            const Value& vr = c->values[g.res_value];
            S.res = c->act_dev + vr.offset;
            S.ldr = vr.Cp;
            S.res_up = g.res_up;
            S.res_w = vr.W; S.res_hw = vr.H * vr.W;
            S.out_w = g.Wo; S.out_hw = g.Ho * g.Wo;
            if (g.res_up > 1 && (vr.H * g.res_up != g.Ho || vr.W * g.res_up != g.Wo))
              return set_err(c, GEMEL_E_STATE, "bind: upsampled residual size mismatch");
            rc = tmap_encode_2d(&S.res_map, S.res, uint64_t(g.Cout), uint64_t(vr.B) * vr.H * vr.W,
                                uint64_t(S.ldr) * 2, 32, 32, 64);
            if (rc) return set_err(c, GEMEL_E_CUDA, "bind: residual tensor map encode failed");
          }
        }
      }
      int rc2 = build_dep_ranges(c, L, probs, meta.data());
      if (rc2) return rc2;
    } else if (L.kind == NK_PRE) {
      PreTask* t = reinterpret_cast<PreTask*>(base);
      int64_t blocks = 0, pix = 0;
      int k = 0;
      L.cols_smem = 0;
      for (int pass = 0; pass < 2; ++pass)        // im2col tasks first, then NHWC tasks
        for (int nid : L.items) {
          const Node& g = c->nodes[nid];
          if (g.stem) continue;   // fused into the stem launch
          if ((g.layer >= 0) != (pass == 0)) continue;
          const Value& v = c->values[g.out_value];
          const Model& Mo = c->models[g.model];
          PreTask& T = t[k++];
          std::memset(&T, 0, sizeof(T));
          T.src = c->act_dev + c->frame_off[Mo.stream_id];
          T.dst = c->act_dev + v.offset;
          T.h = Mo.in_h; T.w = Mo.in_w;
          if (g.layer >= 0) {   // im2col matrix of the first conv: one block per (image, output row)
            const gemel_layer& d = Mo.layers[g.layer].d;
            T.mode = 1;
            T.ho = v.H; T.wo = v.W;
            T.kh = d.kh; T.kw = d.kw; T.sh = d.sh; T.sw = d.sw; T.ph = d.ph; T.pw = d.pw; T.dh = d.dh; T.dw = d.dw;
            T.K = v.C; T.Kp = v.Cp;
            if (T.Kp / 8 > 256) return set_err(c, GEMEL_E_UNSUPPORTED, "bind: first-conv im2col row wider than 2048");
            T.work = int64_t(v.B) * v.H;
            T.work_begin = blocks;
            blocks += T.work;
            const int smem = ((d.kh - 1) * d.dh + 1) * ((v.W - 1) * d.sw + (d.kw - 1) * d.dw + 1) * 3 * 4 + v.Cp * 4;
            L.cols_smem = std::max(L.cols_smem, smem);
            L.n_cols = k;
          } else {
            T.work = int64_t(v.B) * v.H * v.W;
            T.work_begin = pix;
            pix += T.work;
          }
        }
      L.cols_blocks = blocks;
      L.pre_pixels = pix;
      L.n_pre_tasks = k;
      // the same tasks reading staging buffer 1 (double-buffered ingest)
      for (int j = 0; j < k; ++j) {
        PreTask& T2 = t[k + j];
        T2 = t[j];
        const int64_t off0 = static_cast<const uint8_t*>(t[j].src) - c->act_dev;  // staging offsets are 64-bit
        for (size_t s2 = 0; s2 < c->frame_off.size(); ++s2)
          if (c->frame_off[s2] == off0) T2.src = c->act_dev + c->frame_off2[s2];
      }
      if (L.cols_smem > 200 * 1024) return set_err(c, GEMEL_E_UNSUPPORTED, "bind: first-conv receptive rows too wide");
    } else if (L.kind == NK_TOPK) {
      TopkTask* t = reinterpret_cast<TopkTask*>(base);
      int blocks = 0;
      L.topk_rows = 0;
      for (size_t k = 0; k < L.items.size(); ++k) {
        const Node& g = c->nodes[L.items[k]];
        const Value& vi = c->values[g.in_value];
        const Value& vo = c->values[g.out_value];
        const gemel_layer& d = c->models[g.model].layers[g.layer].d;
        TopkTask& T = t[k];
        std::memset(&T, 0, sizeof(T));
        T.src = reinterpret_cast<const float*>(c->act_dev + vi.offset);
        T.dst = reinterpret_cast<float*>(c->act_dev + vo.offset);
        T.n = vi.B; T.rows = vi.C / d.cin; T.fields = d.cin; T.k = d.cout; T.score = d.kh;
        T.src_pitch = vi.Cp; T.dst_pitch = vo.Cp;
        T.block_begin = blocks;
        blocks += T.n;
        L.topk_rows = std::max(L.topk_rows, T.rows);
      }
      L.topk_blocks = blocks;
    } else if (L.kind == NK_NMS) {   // final detection NMS: one 32-thread CTA per frame
      NmsTask* t = reinterpret_cast<NmsTask*>(base);
      int blocks = 0;
      for (size_t k = 0; k < L.items.size(); ++k) {
        const Node& g = c->nodes[L.items[k]];
        const Value& vi = c->values[g.in_value];
        const Value& vo = c->values[g.out_value];
        const gemel_layer& d = c->models[g.model].layers[g.layer].d;
        NmsTask& T = t[k];
        std::memset(&T, 0, sizeof(T));
        T.src = reinterpret_cast<const float*>(c->act_dev + vi.offset);
        T.dst = reinterpret_cast<float*>(c->act_dev + vo.offset);
        T.n = vi.B; T.k_in = vi.C / 7; T.max_det = d.cout; T.iou = d.neg_slope;
        T.src_pitch = vi.Cp; T.dst_pitch = vo.Cp;
        T.block_begin = blocks;
        blocks += T.n;
      }
      L.det_blocks = blocks;
    } else if (L.kind >= NK_RPN) {
      int rc = build_detect_tasks(c, L, base);
      if (rc) return rc;
    } else if (L.kind == NK_MISC) {
      MiscTask* t = reinterpret_cast<MiscTask*>(base);
      int64_t work = 0;
      int k = 0;
      auto place = [&](MiscTask& T, int64_t w) {   // every task starts on a multiple of 32
        T.work_begin = work;
        T.work = w;
        work += (w + 31) / 32 * 32;
      };
      for (int nid : L.items) {
        const Node& g = c->nodes[nid];
        const Value& vo = c->values[g.out_value];
        const Layer& Ly = c->models[g.model].layers[g.layer];
        const Model& Mm = c->models[g.model];
        if (g.misc == MISC_CONCAT) {
          int c_off = 0;
          for (size_t p = 0; p < g.ins.size(); ++p, ++k) {
            const Value& vp = c->values[g.ins[p]];
            MiscTask& T = t[k];
            std::memset(&T, 0, sizeof(T));
            T.kind = 0;
            T.src = c->act_dev + vp.offset;
            T.dst = c->act_dev + vo.offset;
            T.n = vo.B; T.h = vo.H; T.w = vo.W; T.c = vp.C; T.cps = vp.Cp; T.cpd = vo.Cp;
            T.c_off = c_off; T.scale = g.in_scale[p];
            if (vp.H * T.scale != vo.H || vp.W * T.scale != vo.W)
              return set_err(c, GEMEL_E_STATE, "bind: concat piece size mismatch");
            place(T, int64_t(T.n) * T.h * T.w * (T.c / 8));
            c_off += vp.C;
          }
        } else if (g.misc == MISC_L2NORM) {
          const Value& vi = c->values[g.in_value];
          MiscTask& T = t[k++];
          std::memset(&T, 0, sizeof(T));
          T.kind = 2;
          T.src = c->act_dev + vi.offset;
          T.dst = c->act_dev + vo.offset;
          T.n = vi.B; T.h = vi.H; T.w = vi.W; T.c = vi.C; T.cps = vi.Cp; T.cpd = vo.Cp;
          T.vec = reinterpret_cast<const float*>(c->w_dev + g.scale_off);
          T.eps = Ly.d.eps;
          place(T, int64_t(T.n) * T.h * T.w * 32);
        } else if (g.misc == MISC_DETC) {   // detection candidates: a thread per row
          const Value& vi = c->values[g.in_value];
          MiscTask& T = t[k++];
          std::memset(&T, 0, sizeof(T));
          T.kind = 4;
          T.src = c->act_dev + vi.offset;
          T.dst = c->act_dev + vo.offset;
          T.n = vi.B; T.c = Ly.d.cin; T.cps = vi.Cp; T.cpd = vo.Cp;
          T.rows = vi.C / Ly.d.cin;
          T.det_fmt = Ly.d.kh; T.det_thresh = Ly.d.neg_slope; T.eps = Ly.d.eps;
          place(T, int64_t(T.n) * T.rows);
        } else if (g.misc == MISC_SSD) {
          const Value& vl = c->values[g.ins[0]];
          const Value& vc = c->values[g.ins[1]];
          MiscTask& T = t[k++];
          std::memset(&T, 0, sizeof(T));
          T.kind = 3;
          T.src = c->act_dev + vl.offset;
          T.src2 = c->act_dev + vc.offset;
          T.dst = c->act_dev + vo.offset;
          T.n = vl.B; T.h = vl.H; T.w = vl.W; T.c = Ly.d.cout; T.cps = vl.Cp; T.cps2 = vc.Cp; T.A = Ly.d.kh;
          // torchvision's default-box centres: (j + 0.5) / (image / step) of the image = (j + 0.5) * step
          T.stride_w = float(Ly.d.sh);
          T.stride_h = float(Ly.d.sh);
          T.img_w = float(Mm.in_w);
          T.img_h = float(Mm.in_h);
          for (int a = 0; a < 2 * T.A; ++a) T.anchors[a] = Ly.anchors[a];
          for (int j = 0; j < 4; ++j) T.wts[j] = Ly.anchors[2 * T.A + j];
          T.dst_pitch = vo.Cp;
          T.dst_off = g.out_off;
          place(T, int64_t(T.n) * T.h * T.w * T.A * 32);   // a warp per default box
        } else {
          const Value& vi = c->values[g.in_value];
          MiscTask& T = t[k++];
          std::memset(&T, 0, sizeof(T));
          T.kind = 1;
          T.src = c->act_dev + vi.offset;
          T.dst = c->act_dev + vo.offset;
          T.n = vi.B; T.h = vi.H; T.w = vi.W; T.c = 5 + Ly.d.cout; T.cps = vi.Cp; T.A = Ly.d.kh;
          T.stride_w = float(Mm.in_w) / float(vi.W);
          T.stride_h = float(Mm.in_h) / float(vi.H);
          for (int a = 0; a < 2 * T.A; ++a) T.anchors[a] = Ly.anchors[a];
          T.dst_pitch = vo.Cp;
          T.dst_off = g.out_off;
          place(T, int64_t(T.n) * T.A * T.h * T.w * 16);   // a half-warp per box
        }
      }
      L.misc_tasks = k;
      L.misc_work = work;
    } else if (L.kind == NK_ADD) {
      AddTask* t = reinterpret_cast<AddTask*>(base);
      int64_t work = 0;
      for (size_t k = 0; k < L.items.size(); ++k) {
        const Node& g = c->nodes[L.items[k]];
        t[k].a = c->act_dev + c->values[g.in_value].offset;
        t[k].b = c->act_dev + c->values[g.in_value2].offset;
        t[k].out = c->act_dev + c->values[g.out_value].offset;
        t[k].vecs = int64_t(c->values[g.out_value].bytes / 16);
        t[k].act = g.act;
        t[k].slope = g.slope;
        t[k].work_begin = work;
        work += t[k].vecs;
      }
    } else {
      PoolTask* t = reinterpret_cast<PoolTask*>(base);
      int64_t work = 0;
      for (size_t k = 0; k < L.items.size(); ++k) {
        const Node& g = c->nodes[L.items[k]];
        const Value& vi = c->values[g.in_value];
        const Value& vo = c->values[g.out_value];
        const gemel_layer& d = c->models[g.model].layers[g.layer].d;
        PoolTask& T = t[k];
        T.src = c->act_dev + vi.offset;
        T.dst = c->act_dev + vo.offset;
        T.n = vi.B; T.h = vi.H; T.w = vi.W; T.cp = vi.Cp; T.ho = vo.H; T.wo = vo.W;
        T.kh = d.kh; T.kw = d.kw; T.sh = d.sh; T.sw = d.sw; T.ph = d.ph; T.pw = d.pw; T.dh = d.dh; T.dw = d.dw;
        T.kind = L.kind == NK_MAXPOOL ? 0 : 1;
        T.work_begin = work;
        work += int64_t(vo.B) * vo.H * vo.W * (vo.Cp / 8);
      }
    }
  }
  CUDA_TRY(cudaMemcpy(c->meta_dev, meta.data(), c->meta_bytes, cudaMemcpyHostToDevice), "upload launch tables");

  for (size_t i = 0; i < 2 * c->launches.size(); ++i) {
    cudaEvent_t e;
    CUDA_TRY(cudaEventCreate(&e), "event create");
    c->events.push_back(e);
  }
  c->launch_ms.assign(c->launches.size(), 0.f);
  // developer tracing (GEMEL_TRACE_DIR): per-tile timestamps of every GEMM launch
  if (const char* td = std::getenv("GEMEL_TRACE_DIR")) {
    c->trace_path = td;
    c->trace_dev.assign(c->launches.size(), nullptr);
    for (size_t li = 0; li < c->launches.size(); ++li)
      if (c->launches[li].kind == NK_GEMM && !c->launches[li].stem)
        CUDA_TRY(cudaMalloc(&c->trace_dev[li], size_t(c->launches[li].total_tiles) * 128), "trace alloc");
  }

  // capture the whole step as one CUDA graph on a private stream, once per staging buffer
  for (int buf = 0; buf < 2; ++buf) {
    cudaStream_t cap;
    CUDA_TRY(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking), "stream create");
    cudaGraph_t graph;
    CUDA_TRY(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal), "begin capture");
    int rc = run_launches(c, cap, false, buf);
    cudaError_t ce = cudaStreamEndCapture(cap, &graph);
    if (rc) { cudaStreamDestroy(cap); return rc; }
    if (ce != cudaSuccess) { cudaStreamDestroy(cap); return cuda_err(c, ce, "end capture"); }
    cudaGraphExec_t exec;
    ce = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    cudaStreamDestroy(cap);
    if (ce != cudaSuccess) return cuda_err(c, ce, "graph instantiate");
    (buf ? c->graph_exec2 : c->graph_exec) = exec;
  }
  {
    cudaStream_t is;
    CUDA_TRY(cudaStreamCreateWithFlags(&is, cudaStreamNonBlocking), "ingest stream");
    c->in_stream = is;
    for (int b = 0; b < 2; ++b) {
      cudaEvent_t e1, e2;
      CUDA_TRY(cudaEventCreateWithFlags(&e1, cudaEventDisableTiming), "ingest event");
      CUDA_TRY(cudaEventCreateWithFlags(&e2, cudaEventDisableTiming), "ingest event");
      c->in_ready[b] = e1;
      c->buf_free[b] = e2;
    }
    cudaEvent_t e3;
    CUDA_TRY(cudaEventCreateWithFlags(&e3, cudaEventDisableTiming), "ingest event");
    c->dev_frames_ready = e3;
  }
  CUDA_TRY(cudaDeviceSynchronize(), "bind sync");
  c->bound = true;
  return GEMEL_OK;
}

int run_step(Ctx* c, const gemel_stream_batch* in, int n_in, gemel_result* out, int n_out) {
  if (!c->bound) return set_err(c, GEMEL_E_STATE, "infer before bind");
  cudaStream_t st = static_cast<cudaStream_t>(c->opt.compute_stream);
  // Double-buffered ingest (graph mode): this step's frames go to staging buffer `buf`
  // on the ingest stream once the last step that read `buf` has finished, so they
  // overlap the previous step's compute; the compute stream waits for them.
  const int buf = c->profiling ? 0 : c->parity;
  cudaStream_t cs = c->profiling ? st : static_cast<cudaStream_t>(c->in_stream);
  if (!c->profiling) {
    CUDA_TRY(cudaStreamWaitEvent(cs, static_cast<cudaEvent_t>(c->buf_free[buf]), 0), "ingest wait");
    // device-resident frames may be produced by the caller's earlier work on the compute
    // stream (decode, preprocessing): the ingest stream's D2D copies are ordered after it
    bool dev_frames = false;
    for (int i = 0; i < n_in; ++i) dev_frames |= in[i].on_host == 0;
    if (dev_frames) {
      CUDA_TRY(cudaEventRecord(static_cast<cudaEvent_t>(c->dev_frames_ready), st), "frames ready record");
      CUDA_TRY(cudaStreamWaitEvent(cs, static_cast<cudaEvent_t>(c->dev_frames_ready), 0), "frames ready wait");
    }
  }
  const std::vector<int64_t>& stage = buf ? c->frame_off2 : c->frame_off;
  std::vector<char> fed(c->frame_off.size(), 0);
  for (int i = 0; i < n_in; ++i) {
    const gemel_stream_batch& b = in[i];
    if (b.stream_id < 0 || b.stream_id >= int(c->frame_off.size()) || c->frame_off[b.stream_id] < 0 || !b.frames)
      return set_err(c, GEMEL_E_ARG, "infer: unknown stream " + std::to_string(b.stream_id));
    if (b.n_frames != c->batch[b.stream_id])
      return set_err(c, GEMEL_E_ARG, "infer: stream " + std::to_string(b.stream_id) + " batch differs from plan");
    int h = 0, w = 0;
    for (auto& M : c->models)
      if (M.stream_id == b.stream_id) { h = M.in_h; w = M.in_w; }
    const uint64_t bytes = uint64_t(b.n_frames) * h * w * 3;
    CUDA_TRY(cudaMemcpyAsync(c->act_dev + stage[b.stream_id], b.frames, bytes,
                             b.on_host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, cs),
             "frame copy");
    fed[b.stream_id] = 1;
  }
  for (size_t s = 0; s < c->frame_off.size(); ++s)
    if (c->frame_off[s] >= 0 && !fed[s]) return set_err(c, GEMEL_E_ARG, "infer: stream " + std::to_string(s) + " missing");
  if (c->profiling) {
    int rc = run_launches(c, st, true);
    if (rc) return rc;
  } else {
    CUDA_TRY(cudaEventRecord(static_cast<cudaEvent_t>(c->in_ready[buf]), cs), "ingest record");
    CUDA_TRY(cudaStreamWaitEvent(st, static_cast<cudaEvent_t>(c->in_ready[buf]), 0), "ingest join");
    CUDA_TRY(cudaGraphLaunch(static_cast<cudaGraphExec_t>(buf ? c->graph_exec2 : c->graph_exec), st), "graph launch");
    CUDA_TRY(cudaEventRecord(static_cast<cudaEvent_t>(c->buf_free[buf]), st), "buffer free record");
    c->parity ^= 1;
  }
  for (int i = 0; i < n_out; ++i) {
    const gemel_result& r = out[i];
    if (r.model_id < 0 || r.model_id >= int(c->models.size()) || !r.out)
      return set_err(c, GEMEL_E_ARG, "infer: bad result model id");
    const Model& M = c->models[r.model_id];
    const Value& v = c->values[c->value_of.at({r.model_id, int(M.layers.size()) - 1})];
    const uint64_t need = uint64_t(v.B) * v.C * 4;
    if (r.out_bytes < need) return set_err(c, GEMEL_E_SMALLBUF, "infer: result buffer too small");
    CUDA_TRY(cudaMemcpy2DAsync(r.out, size_t(v.C) * 4, c->act_dev + v.offset, size_t(v.Cp) * 4, size_t(v.C) * 4, v.B,
                               r.on_host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, st),
             "result copy");
  }
  if (c->profiling) {
    CUDA_TRY(cudaStreamSynchronize(st), "profiling sync");
    for (size_t li = 0; li < c->launches.size(); ++li)
      cudaEventElapsedTime(&c->launch_ms[li], static_cast<cudaEvent_t>(c->events[2 * li]),
                           static_cast<cudaEvent_t>(c->events[2 * li + 1]));
    for (size_t li = 0; li < c->trace_dev.size(); ++li) {
      if (!c->trace_dev[li]) continue;
      std::vector<unsigned long long> h(size_t(c->launches[li].total_tiles) * 16);
      CUDA_TRY(cudaMemcpy(h.data(), c->trace_dev[li], h.size() * 8, cudaMemcpyDeviceToHost), "trace copy");
      const std::string path = c->trace_path + "/launch" + std::to_string(li) + ".bin";
      if (FILE* f = std::fopen(path.c_str(), "wb")) {
        std::fwrite(h.data(), 8, h.size(), f);
        std::fclose(f);
      }
    }
  }
  return GEMEL_OK;
}

}  // namespace gemel

using namespace gemel;

extern "C" {

gemel_status gemel_plan(gemel_ctx ctx, const int32_t* batch, int32_t n_streams, gemel_plan_info* info) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c || !batch || n_streams <= 0) return GEMEL_E_ARG;
  if (c->models.empty()) return set_err(c, GEMEL_E_STATE, "plan: no models registered");
  int ndev = 0;
  if (!(c->opt.flags & GEMEL_FLAG_DRY_PLAN) && (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= c->opt.device))
    return set_err(c, GEMEL_E_CUDA, "plan: no CUDA device (the B200 path has no CPU fallback)");
  c->batch.assign(batch, batch + n_streams);
  c->sm_count = 148;
  if (!(c->opt.flags & GEMEL_FLAG_DRY_PLAN)) {
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->opt.device) == cudaSuccess && sms > 0)
      c->sm_count = sms;
  }
  int rc = build_plan(c);
  if (rc) return rc;
  c->planned = true;
  if (info) {
    std::memset(info, 0, sizeof(*info));
    info->weight_arena_bytes = c->w_bytes;
    info->act_arena_bytes = c->act_bytes;
    info->meta_bytes = c->meta_bytes;
    info->unique_weight_bytes = c->unique_weight_bytes;
    info->unmerged_weight_bytes = c->unmerged_weight_bytes;
    info->n_levels = c->n_levels;
    for (const Launch& L : c->launches) {   // kernels, not plan launches
      if (L.kind == NK_GEMM && L.stem) {
        info->n_launches += int(L.items.size());   // one fused stem kernel per first-conv problem
      } else if (L.kind == NK_RPN) {
        info->n_launches += 2;   // cluster top-K selection, then decode + NMS
      } else if (L.kind == NK_PRE) {
        bool cols = false, nhwc = false;
        for (int nid : L.items) {
          const Node& g = c->nodes[nid];
          if (g.stem) continue;
          (g.layer >= 0 ? cols : nhwc) = true;
        }
        info->n_launches += int(cols) + int(nhwc);
      } else {
        info->n_launches += 1;
      }
    }
    for (auto& p : c->problems) {
      info->n_gemm_problems++;
      if (p.members.size() > 1) info->n_union_problems++;
    }
    for (auto& M : c->models) info->frames_per_step += c->batch[M.stream_id];
    info->gemm_flops_per_step = c->gemm_flops;
    info->pinned_weight_bytes = c->pinned_bytes;
    info->swap_ring_bytes = c->ring_bytes;
    info->swap_bytes_per_step = c->swap_bytes;
    info->n_swapped = int32_t(c->swap_order.size());
  }
  return GEMEL_OK;
}

gemel_status gemel_bind_arenas(gemel_ctx ctx, void* w, uint64_t wb, void* a, uint64_t ab) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c) return GEMEL_E_ARG;
  return bind(c, w, wb, a, ab);
}

gemel_status gemel_weight_view(gemel_ctx ctx, void** dev, uint64_t* bytes) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c || !dev || !bytes) return GEMEL_E_ARG;
  if (!c->bound) return set_err(c, GEMEL_E_STATE, "weight_view before bind");
  *dev = c->w_dev;
  *bytes = c->w_bytes;
  return GEMEL_OK;
}

gemel_status gemel_infer(gemel_ctx ctx, const gemel_stream_batch* in, int32_t n_in, gemel_result* out, int32_t n_out) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c || (n_in > 0 && !in) || (n_out > 0 && !out)) return GEMEL_E_ARG;
  return run_step(c, in, n_in, out, n_out);
}

gemel_status gemel_read_value(gemel_ctx ctx, int32_t model_id, int32_t op_pos, void* host_dst, uint64_t bytes,
                              gemel_value_desc* desc) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c) return GEMEL_E_ARG;
  if (!c->bound) return set_err(c, GEMEL_E_STATE, "read_value before bind");
  auto it = c->value_of.find({model_id, op_pos});
  if (it == c->value_of.end()) return set_err(c, GEMEL_E_ARG, "read_value: value not stored (fused or unknown)");
  const Value& v = c->values[it->second];
  if (v.virt) return set_err(c, GEMEL_E_ARG, "read_value: value not stored (fused into the first-conv stem launch)");
  if (desc) {
    desc->dtype = v.fp32 ? 1 : 0;
    desc->n = v.B; desc->h = v.H; desc->w = v.W; desc->c = v.C; desc->c_pitch = v.Cp;
  }
  if (!host_dst) return GEMEL_OK;
  if (bytes < v.bytes) return set_err(c, GEMEL_E_SMALLBUF, "read_value: buffer too small");
  CUDA_TRY(cudaDeviceSynchronize(), "read_value sync");
  CUDA_TRY(cudaMemcpy(host_dst, c->act_dev + v.offset, v.bytes, cudaMemcpyDeviceToHost), "read_value copy");
  return GEMEL_OK;
}

gemel_status gemel_set_profiling(gemel_ctx ctx, int32_t enable) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c) return GEMEL_E_ARG;
  c->profiling = enable != 0;
  return GEMEL_OK;
}

gemel_status gemel_launch_list(gemel_ctx ctx, gemel_launch_info* info, float* ms, int32_t cap, int32_t* n) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c || !n) return GEMEL_E_ARG;
  *n = int(c->launches.size());
  if (cap == 0) return GEMEL_OK;
  if (cap < *n) return set_err(c, GEMEL_E_SMALLBUF, "launch_list: buffer too small");
  for (int i = 0; i < *n; ++i) {
    const Launch& L = c->launches[i];
    if (info) {
      std::memset(&info[i], 0, sizeof(info[i]));
      info[i].kind = L.kind == NK_GEMM && L.stem ? 12 : L.kind == NK_PRE ? 0 : L.kind == NK_GEMM ? 1 : L.kind == NK_MAXPOOL ? 2 : L.kind == NK_AVGPOOL ? 3 :
                     L.kind == NK_ADD ? 4 : L.kind == NK_MISC ? 5 : L.kind;
      info[i].level = L.level;
      info[i].n_problems = int(L.items.size());
      info[i].flops = L.flops;
      info[i].bytes = L.bytes;
    }
    if (ms) ms[i] = i < int(c->launch_ms.size()) ? c->launch_ms[i] : 0.f;
  }
  return GEMEL_OK;
}

}  // extern "C"
