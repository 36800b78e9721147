"""Thin ctypes binding of the C ABI in include/gemel.h (argument marshalling only).

Every function here has the C name and forwards to libgemel.so; all compute
runs in the library's CUDA kernels.  There is no fallback: if the shared
library is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libgemel.so")
if not os.path.exists(_LIB_PATH):
    raise ImportError(f"{_LIB_PATH} not built: run `python -m paper_2201_07705_b200.build` "
                      "(the B200 path has no CPU fallback)")
_lib = C.CDLL(_LIB_PATH)

OK, E_ARG, E_SCHEMA, E_MERGE, E_STATE, E_NOMEM, E_CUDA, E_SMALLBUF, E_UNSUPPORTED = 0, -1, -2, -3, -4, -5, -6, -7, -8
OP = {"conv": 1, "linear": 2, "bn": 3, "relu": 4, "leaky": 5, "maxpool": 6, "gap": 7, "add": 8, "flatten": 9,
      "concat": 10, "upsample": 11, "yolo": 12, "topk": 13, "l2norm": 14, "ssd_decode": 15,
      "rpn_level": 16, "rpn_merge": 17, "roi_align": 18, "box_post": 19, "det_cand": 20, "det_nms": 21}
OP_NAME = {v: k for k, v in OP.items()}


class GemelLayer(C.Structure):
    _fields_ = [("op", C.c_int32), ("n_in", C.c_int32), ("in_", C.c_int32 * 8),
                ("cin", C.c_int32), ("cout", C.c_int32),
                ("kh", C.c_int32), ("kw", C.c_int32), ("sh", C.c_int32), ("sw", C.c_int32),
                ("ph", C.c_int32), ("pw", C.c_int32), ("dh", C.c_int32), ("dw", C.c_int32),
                ("groups", C.c_int32), ("bias", C.c_int32), ("ceil_mode", C.c_int32), ("tie", C.c_int32),
                ("out_h", C.c_int32), ("out_w", C.c_int32),
                ("eps", C.c_float), ("momentum", C.c_float), ("neg_slope", C.c_float),
                ("affine", C.c_int32), ("track_stats", C.c_int32),
                ("param", C.POINTER(C.c_float) * 4)]


class GemelOptions(C.Structure):
    _fields_ = [("device", C.c_int32), ("flags", C.c_int32), ("compute_stream", C.c_void_p),
                ("weight_budget_bytes", C.c_uint64), ("weight_source", C.c_int32), ("source_device", C.c_int32)]


class GemelGroup(C.Structure):
    _fields_ = [("op", C.c_int32), ("n_apps", C.c_int32), ("app_offset", C.c_int32), ("reserved", C.c_int32),
                ("per_bytes", C.c_uint64), ("total_bytes", C.c_uint64), ("reclaimable", C.c_uint64)]


class GemelAppearance(C.Structure):
    _fields_ = [("model_id", C.c_int32), ("op_pos", C.c_int32)]


class GemelMergeGroup(C.Structure):
    _fields_ = [("members", C.POINTER(GemelAppearance)), ("n_members", C.c_int32), ("source", C.c_int32)]


class GemelPlanInfo(C.Structure):
    _fields_ = [("weight_arena_bytes", C.c_uint64), ("act_arena_bytes", C.c_uint64), ("meta_bytes", C.c_uint64),
                ("unique_weight_bytes", C.c_uint64), ("unmerged_weight_bytes", C.c_uint64),
                ("n_levels", C.c_int32), ("n_launches", C.c_int32), ("n_gemm_problems", C.c_int32),
                ("n_union_problems", C.c_int32), ("frames_per_step", C.c_int32), ("n_swapped", C.c_int32),
                ("gemm_flops_per_step", C.c_double), ("pinned_weight_bytes", C.c_uint64),
                ("swap_ring_bytes", C.c_uint64), ("swap_bytes_per_step", C.c_uint64)]


class GemelStreamBatch(C.Structure):
    _fields_ = [("stream_id", C.c_int32), ("n_frames", C.c_int32), ("frames", C.c_void_p),
                ("on_host", C.c_int32), ("reserved", C.c_int32)]


class GemelResult(C.Structure):
    _fields_ = [("model_id", C.c_int32), ("on_host", C.c_int32), ("out", C.c_void_p), ("out_bytes", C.c_uint64)]


class GemelStats(C.Structure):
    _fields_ = [("n_models", C.c_int32), ("n_param_layers", C.c_int32), ("n_merged_layers", C.c_int32),
                ("planned", C.c_int32), ("registered_bytes", C.c_uint64), ("bytes_saved", C.c_uint64)]


class GemelValueDesc(C.Structure):
    _fields_ = [("dtype", C.c_int32), ("n", C.c_int32), ("h", C.c_int32), ("w", C.c_int32), ("c", C.c_int32),
                ("c_pitch", C.c_int32)]


class GemelLaunchInfo(C.Structure):
    _fields_ = [("kind", C.c_int32), ("level", C.c_int32), ("n_problems", C.c_int32), ("reserved", C.c_int32),
                ("flops", C.c_double), ("bytes", C.c_double)]


class GemelMergeAttempt(C.Structure):
    _fields_ = [("group", C.c_int32), ("n_members", C.c_int32), ("ok", C.c_int32), ("reserved", C.c_int32),
                ("bytes", C.c_uint64)]


RETRAIN_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.POINTER(GemelMergeGroup), C.c_int32)

_ctx_t = C.c_void_p
_sig = {
    "gemel_create": ([C.POINTER(GemelOptions), C.POINTER(_ctx_t)], C.c_int32),
    "gemel_destroy": ([_ctx_t], None),
    "gemel_last_error": ([_ctx_t], C.c_char_p),
    "gemel_register_model": ([_ctx_t, C.POINTER(GemelLayer), C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                              C.POINTER(C.c_int32)], C.c_int32),
    "gemel_find_shareable": ([_ctx_t, C.POINTER(GemelGroup), C.c_int32, C.POINTER(C.c_int32),
                              C.POINTER(GemelAppearance), C.c_int32, C.POINTER(C.c_int32)], C.c_int32),
    "gemel_apply_merge": ([_ctx_t, C.POINTER(GemelMergeGroup), C.c_int32, C.POINTER(C.c_uint64)], C.c_int32),
    "gemel_incremental_merge": ([_ctx_t, RETRAIN_FN, C.c_void_p, C.POINTER(GemelMergeAttempt), C.c_int32,
                                 C.POINTER(C.c_int32), C.POINTER(C.c_uint64)], C.c_int32),
    "gemel_plan": ([_ctx_t, C.POINTER(C.c_int32), C.c_int32, C.POINTER(GemelPlanInfo)], C.c_int32),
    "gemel_bind_arenas": ([_ctx_t, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64], C.c_int32),
    "gemel_weight_view": ([_ctx_t, C.POINTER(C.c_void_p), C.POINTER(C.c_uint64)], C.c_int32),
    "gemel_infer": ([_ctx_t, C.POINTER(GemelStreamBatch), C.c_int32, C.POINTER(GemelResult), C.c_int32], C.c_int32),
    "gemel_read_value": ([_ctx_t, C.c_int32, C.c_int32, C.c_void_p, C.c_uint64, C.POINTER(GemelValueDesc)],
                         C.c_int32),
    "gemel_set_profiling": ([_ctx_t, C.c_int32], C.c_int32),
    "gemel_launch_list": ([_ctx_t, C.POINTER(GemelLaunchInfo), C.POINTER(C.c_float), C.c_int32,
                           C.POINTER(C.c_int32)], C.c_int32),
    "gemel_stats": ([_ctx_t, C.POINTER(GemelStats)], C.c_int32),
    "gemel_plan_dump": ([_ctx_t, C.c_char_p, C.c_uint64, C.POINTER(C.c_uint64)], C.c_int32),
}
for _n, (_a, _r) in _sig.items():
    _f = getattr(_lib, _n)
    _f.argtypes = _a
    _f.restype = _r

EXPORTED = tuple(_sig)


class GemelError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"gemel error {code}: {msg}")
        self.code = code


def _check(ctx, rc):
    if rc != OK:
        raise GemelError(rc, gemel_last_error(ctx))


def gemel_last_error(ctx):
    s = _lib.gemel_last_error(ctx)
    return s.decode() if s else ""


FLAG_DRY_PLAN = 1


SOURCE_HOST, SOURCE_PEER = 0, 1


def gemel_create(device=0, compute_stream=0, weight_budget_bytes=0, flags=0, weight_source=SOURCE_HOST,
                 source_device=0):
    opt = GemelOptions(device, flags, C.c_void_p(compute_stream or None), weight_budget_bytes, weight_source,
                       source_device)
    ctx = _ctx_t()
    rc = _lib.gemel_create(C.byref(opt), C.byref(ctx))
    if rc != OK:
        raise GemelError(rc, "create failed")
    return ctx


def gemel_destroy(ctx):
    _lib.gemel_destroy(ctx)


def _pair(v):
    return tuple(v) if isinstance(v, (tuple, list)) else (v, v)


def layer_struct(l, p, keep):
    """Marshal one zoo layer dict + its params into a GemelLayer (keeps arrays alive in `keep`)."""
    s = GemelLayer()
    op = l["op"]
    if op not in OP:
        raise GemelError(E_UNSUPPORTED, f"op {op} not in the C ABI")
    s.op = OP[op]
    s.n_in = len(l["in"])
    for i, x in enumerate(l["in"]):
        s.in_[i] = x
    if op == "conv":
        s.cin, s.cout = l["cin"], l["cout"]
        (s.kh, s.kw), (s.sh, s.sw), (s.ph, s.pw), (s.dh, s.dw) = l["k"], l["s"], l["p"], l["d"]
        s.groups, s.bias = l["groups"], int(l["bias"])
        s.tie = l["tie"] + 1 if "tie" in l else 0
    elif op == "linear":
        s.cin, s.cout, s.bias = l["fin"], l["fout"], int(l["bias"])
    elif op == "bn":
        s.cin, s.eps, s.momentum, s.affine, s.track_stats = l["c"], l["eps"], l["momentum"], int(l["affine"]), int(l["track"])
    elif op == "leaky":
        s.neg_slope = l["slope"]
    elif op == "maxpool":
        (s.kh, s.kw), (s.sh, s.sw), (s.ph, s.pw), (s.dh, s.dw) = l["k"], l["s"], l["p"], l["d"]
        s.ceil_mode = 2 if l.get("darknet") else int(l["ceil"])
    elif op == "upsample":
        s.sh = s.sw = int(l["scale"])
    elif op == "yolo":
        s.kh = len(l["anchors"])
        s.cout = l["classes"]
        s.cin = s.kh * (5 + l["classes"])
        a = np.ascontiguousarray(np.asarray(l["anchors"], np.float32).reshape(-1))
        keep.append(a)
        s.param[0] = a.ctypes.data_as(C.POINTER(C.c_float))
    elif op == "topk":
        s.cin, s.cout, s.kh = l["fields"], l["k"], l["score"]
    elif op == "det_cand":
        s.cin, s.kh, s.neg_slope, s.eps = l["fields"], l["fmt"], l["score_thresh"], l["min_size"]
    elif op == "det_nms":
        s.cout, s.neg_slope = l["max_det"], l["iou"]
    elif op == "l2norm":
        s.cin, s.eps = l["c"], l["eps"]
        a = np.ascontiguousarray(p["scale"], dtype=np.float32)
        keep.append(a)
        s.param[0] = a.ctypes.data_as(C.POINTER(C.c_float))
    elif op == "ssd_decode":
        s.kh, s.cout, s.sh = len(l["wh"]), l["classes"], int(l["step"])
        for i, v in enumerate((np.asarray(l["wh"], np.float32).reshape(-1), np.asarray(l["weights"], np.float32))):
            a = np.ascontiguousarray(v)
            keep.append(a)
            s.param[i] = a.ctypes.data_as(C.POINTER(C.c_float))
    elif op == "gap":
        s.out_h, s.out_w = l["out"]
    elif op == "rpn_level":
        s.kh, s.cout, s.neg_slope, s.eps = len(l["ratios"]), l["pre_n"], l["nms"], l["min_size"]
        a = np.ascontiguousarray(np.asarray([(l["size"], r) for r in l["ratios"]], np.float32).reshape(-1))
        keep.append(a)
        s.param[0] = a.ctypes.data_as(C.POINTER(C.c_float))
    elif op == "rpn_merge":
        s.cout = l["post_n"]
    elif op == "roi_align":
        s.out_h = s.out_w = l["out"]
        s.kh = l["sampling"]
        s.sh, s.sw = l["canonical"]
    elif op == "box_post":
        s.cout = l["classes"]
        a = np.ascontiguousarray(np.asarray(l["weights"], np.float32))
        keep.append(a)
        s.param[0] = a.ctypes.data_as(C.POINTER(C.c_float))
    names = {"conv": ("w", "b"), "linear": ("w", "b"), "bn": ("gamma", "beta", "mean", "var")}.get(op, ())
    for i, k in enumerate(names):
        if k in p:
            a = np.ascontiguousarray(p[k], dtype=np.float32)
            keep.append(a)
            s.param[i] = a.ctypes.data_as(C.POINTER(C.c_float))
    return s


def gemel_register_model(ctx, layers, params, stream_id, in_h, in_w):
    keep = []
    arr = (GemelLayer * len(layers))(*[layer_struct(l, p, keep) for l, p in zip(layers, params)])
    mid = C.c_int32()
    _check(ctx, _lib.gemel_register_model(ctx, arr, len(layers), stream_id, in_h, in_w, C.byref(mid)))
    return mid.value


def gemel_find_shareable(ctx):
    ng, na = C.c_int32(), C.c_int32()
    _check(ctx, _lib.gemel_find_shareable(ctx, None, 0, C.byref(ng), None, 0, C.byref(na)))
    groups = (GemelGroup * max(ng.value, 1))()
    apps = (GemelAppearance * max(na.value, 1))()
    _check(ctx, _lib.gemel_find_shareable(ctx, groups, ng.value, C.byref(ng), apps, na.value, C.byref(na)))
    out = []
    for g in groups[:ng.value]:
        out.append({"op": OP_NAME[g.op], "per_bytes": g.per_bytes, "total_bytes": g.total_bytes,
                    "reclaimable": g.reclaimable,
                    "apps": [(a.model_id, a.op_pos) for a in apps[g.app_offset:g.app_offset + g.n_apps]]})
    return out


def gemel_apply_merge(ctx, groups):
    keep = []
    arr = (GemelMergeGroup * max(len(groups), 1))()
    for i, g in enumerate(groups):
        mem = (GemelAppearance * len(g["members"]))(*[GemelAppearance(m, p) for m, p in g["members"]])
        keep.append(mem)
        arr[i] = GemelMergeGroup(mem, len(g["members"]), g.get("source", 0))
    saved = C.c_uint64()
    _check(ctx, _lib.gemel_apply_merge(ctx, arr, len(groups), C.byref(saved)))
    return saved.value


def gemel_incremental_merge(ctx, retrain, log_cap=4096):
    """retrain(config) -> bool, config = [{"members": [(model, pos), ...], "source": 0}, ...]
    (the running configuration, candidate last).  Returns (attempts, bytes_saved) with
    attempts = [{"group", "n_members", "ok", "bytes"}, ...]."""
    err = []

    def cb(_user, groups, n):
        try:
            cfg = [{"members": [(groups[i].members[k].model_id, groups[i].members[k].op_pos)
                                for k in range(groups[i].n_members)], "source": groups[i].source} for i in range(n)]
            return 1 if retrain(cfg) else 0
        except Exception as e:   # never unwind through the C frame
            err.append(e)
            return -1
    fn = RETRAIN_FN(cb)
    log = (GemelMergeAttempt * log_cap)()
    n = C.c_int32()
    saved = C.c_uint64()
    rc = _lib.gemel_incremental_merge(ctx, fn, None, log, log_cap, C.byref(n), C.byref(saved))
    if err:
        raise err[0]
    _check(ctx, rc)
    return [{"group": log[i].group, "n_members": log[i].n_members, "ok": bool(log[i].ok), "bytes": log[i].bytes}
            for i in range(n.value)], saved.value


def gemel_plan(ctx, batch_per_stream):
    b = (C.c_int32 * len(batch_per_stream))(*batch_per_stream)
    info = GemelPlanInfo()
    _check(ctx, _lib.gemel_plan(ctx, b, len(batch_per_stream), C.byref(info)))
    return {k: getattr(info, k) for k, _ in GemelPlanInfo._fields_ if k != "reserved"}


def gemel_bind_arenas(ctx, w_ptr, w_bytes, a_ptr, a_bytes):
    _check(ctx, _lib.gemel_bind_arenas(ctx, C.c_void_p(w_ptr), w_bytes, C.c_void_p(a_ptr), a_bytes))


def gemel_weight_view(ctx):
    p, n = C.c_void_p(), C.c_uint64()
    _check(ctx, _lib.gemel_weight_view(ctx, C.byref(p), C.byref(n)))
    return p.value, n.value


def gemel_infer(ctx, inputs, outputs):
    """inputs: [(stream_id, ptr, n_frames, on_host)], outputs: [(model_id, ptr, bytes, on_host)]."""
    ins = (GemelStreamBatch * max(len(inputs), 1))(*[GemelStreamBatch(s, n, C.c_void_p(p), int(h), 0)
                                                      for s, p, n, h in inputs])
    outs = (GemelResult * max(len(outputs), 1))(*[GemelResult(m, int(h), C.c_void_p(p), b) for m, p, b, h in outputs])
    _check(ctx, _lib.gemel_infer(ctx, ins, len(inputs), outs, len(outputs)))


def gemel_value_desc(ctx, model_id, op_pos):
    """Shape / dtype of a stored value (no copy): dict n, h, w, c, c_pitch, dtype (0 bf16, 1 fp32)."""
    d = GemelValueDesc()
    _check(ctx, _lib.gemel_read_value(ctx, model_id, op_pos, None, 0, C.byref(d)))
    return {"n": d.n, "h": d.h, "w": d.w, "c": d.c, "c_pitch": d.c_pitch, "dtype": d.dtype}


def gemel_read_value(ctx, model_id, op_pos):
    """Stored intermediate as float32 NHWC [n, h, w, c] (bf16 values widened exactly)."""
    d = GemelValueDesc()
    _check(ctx, _lib.gemel_read_value(ctx, model_id, op_pos, None, 0, C.byref(d)))
    if d.dtype == 0:
        buf = np.empty((d.n, d.h, d.w, d.c_pitch), dtype=np.uint16)
        _check(ctx, _lib.gemel_read_value(ctx, model_id, op_pos, buf.ctypes.data, buf.nbytes, C.byref(d)))
        out = (buf.astype(np.uint32) << 16).view(np.float32)
    else:
        out = np.empty((d.n, d.h, d.w, d.c_pitch), dtype=np.float32)
        _check(ctx, _lib.gemel_read_value(ctx, model_id, op_pos, out.ctypes.data, out.nbytes, C.byref(d)))
    return out[..., :d.c]


def gemel_set_profiling(ctx, enable):
    _check(ctx, _lib.gemel_set_profiling(ctx, int(enable)))


def gemel_launch_list(ctx):
    n = C.c_int32()
    _check(ctx, _lib.gemel_launch_list(ctx, None, None, 0, C.byref(n)))
    info = (GemelLaunchInfo * max(n.value, 1))()
    ms = (C.c_float * max(n.value, 1))()
    _check(ctx, _lib.gemel_launch_list(ctx, info, ms, n.value, C.byref(n)))
    kinds = {0: "preprocess", 1: "gemm", 2: "maxpool", 3: "avgpool", 4: "add", 5: "concat_yolo", 6: "topk",
             7: "rpn_level", 8: "rpn_merge", 9: "roi_align", 10: "box_post", 11: "det_nms",
             12: "stem_conv"}
    return [{"kind": kinds[i.kind], "level": i.level, "n_problems": i.n_problems, "flops": i.flops,
             "bytes": i.bytes, "ms": m} for i, m in zip(info[:n.value], ms[:n.value])]


def gemel_stats(ctx):
    s = GemelStats()
    _check(ctx, _lib.gemel_stats(ctx, C.byref(s)))
    return {k: getattr(s, k) for k, _ in GemelStats._fields_}


def gemel_plan_dump(ctx):
    import json
    n = C.c_uint64()
    _check(ctx, _lib.gemel_plan_dump(ctx, None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value)
    _check(ctx, _lib.gemel_plan_dump(ctx, buf, n.value, C.byref(n)))
    return json.loads(buf.value.decode())
