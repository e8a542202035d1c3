"""Thin Python binding of libmt.so (include/mt.h): argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; this module converts Python
objects (workload graphs, torch device tensors, pointer matrices) into the C ABI's plain arrays
and pointers.  PyTorch provides device memory and streams only.  There is no CPU fallback: if
the shared library is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os
import re

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MT_LIB_PATH") or os.path.join(HERE, "libmt.so")   # override: A/B builds (tools/ab.py)
HEADER = os.path.join(HERE, "..", "include", "mt.h")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
lib = C.CDLL(LIB_PATH)

MT_OK, MT_ERR_INTERNAL, MT_ERR_VALIDATION, MT_ERR_REFUSED, MT_ERR_CUDA, MT_ERR_ARG, MT_ERR_STATE = range(7)
MT_MAX_INPUTS = 8
MT_MAX_TENANTS = 16
MT_OPT_STEAL, MT_OPT_NUM_SMS, MT_OPT_TIMEOUT_MS, MT_OPT_PARTITION, MT_OPT_CLAIM_DEPTH, MT_OPT_STAGE_SPLIT = 1, 2, 3, 5, 6, 7
MT_OPT_CTAS_PER_SM = 4
BASE_MODES = {"seq": 1, "ms_dfs": 2, "ms_bfs": 3, "seq_graph": 4, "ms_graph": 5, "stage_events": 6}


class mt_node(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n_inputs", C.c_int32), ("inputs", C.c_int32 * MT_MAX_INPUTS),
                ("out_c", C.c_int32), ("out_h", C.c_int32), ("out_w", C.c_int32),
                ("kh", C.c_int32), ("kw", C.c_int32), ("sh", C.c_int32), ("sw", C.c_int32),
                ("ph", C.c_int32), ("pw", C.c_int32), ("groups", C.c_int32),
                ("ceil_mode", C.c_int32), ("count_include_pad", C.c_int32), ("act", C.c_int32),
                ("residual", C.c_int32), ("weight", C.c_void_p), ("scale", C.c_void_p),
                ("shift", C.c_void_p)]


class mt_graph(C.Structure):
    _fields_ = [("n_nodes", C.c_int32), ("nodes", C.POINTER(mt_node)), ("batch", C.c_int32),
                ("in_c", C.c_int32), ("in_h", C.c_int32), ("in_w", C.c_int32), ("precision", C.c_int32)]


class mt_cost_params(C.Structure):
    _fields_ = [("peak_flops", C.c_double), ("mem_bw", C.c_double), ("op_latency_us", C.c_double),
                ("sync_us", C.c_double), ("c_compute", C.c_double), ("c_memory", C.c_double),
                ("max_concurrency", C.c_int32)]


class mt_error_info(C.Structure):
    _fields_ = [("code", C.c_int32), ("stage", C.c_int32), ("tenant", C.c_int32), ("op", C.c_int32)]


P = C.c_void_p
I32P = C.POINTER(C.c_int32)
F32P = C.POINTER(C.c_float)
_sig = {
    "mt_create": (C.c_int, [C.c_int, C.POINTER(P)]),
    "mt_destroy": (C.c_int, [P]),
    "mt_set_option": (C.c_int, [P, C.c_int32, C.c_int64]),
    "mt_load_graphs": (C.c_int, [P, C.c_int32, C.POINTER(mt_graph)]),
    "mt_op_count": (C.c_int, [P, C.c_int32, I32P]),
    "mt_op_cost": (C.c_int, [P, C.c_int32, C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "mt_op_tiles": (C.c_int, [P, C.c_int32, C.c_int32, I32P]),
    "mt_op_plan": (C.c_int, [P, C.c_int32, C.c_int32, I32P]),
    "mt_op_work": (C.c_int, [P, C.c_int32, C.c_int32, I32P, C.POINTER(C.c_int64)]),
    "mt_estimate_batch_pointers": (C.c_int, [P, C.POINTER(mt_cost_params), C.c_int32, I32P, I32P,
                                             C.POINTER(C.c_double), I32P]),
    "mt_workspace_size": (C.c_int, [P, C.POINTER(C.c_size_t)]),
    "mt_bind_workspace": (C.c_int, [P, P, C.c_size_t]),
    "mt_set_schedule": (C.c_int, [P, C.c_int32, I32P]),
    "mt_set_schedule_pointers": (C.c_int, [P, C.c_int32, I32P]),
    "mt_num_stages": (C.c_int, [P, I32P]),
    "mt_get_schedule": (C.c_int, [P, I32P]),
    "mt_stage_assignment": (C.c_int, [P, I32P]),
    "mt_sm_partition": (C.c_int, [P, I32P]),
    "mt_stage_homes": (C.c_int, [P, I32P, I32P]),
    "mt_run": (C.c_int, [P, C.POINTER(P), C.POINTER(P), F32P, F32P, P]),
    "mt_run_async": (C.c_int, [P, C.POINTER(P), C.POINTER(P), P]),
    "mt_run_host": (C.c_int, [P, C.POINTER(P), C.POINTER(P), F32P, P]),
    "mt_run_baseline": (C.c_int, [P, C.c_int32, C.POINTER(P), C.POINTER(P), F32P, P]),
    "mt_profile_batch": (C.c_int, [P, C.c_int32, I32P, I32P, C.POINTER(P), C.POINTER(P), C.c_int32,
                                   C.c_int32, F32P, I32P, P]),
    "mt_profile_batch_pointers": (C.c_int, [P, C.c_int32, I32P, I32P, C.POINTER(P), C.POINTER(P),
                                            C.c_int32, C.c_int32, F32P, I32P, P]),
    "mt_get_activation": (C.c_int, [P, C.c_int32, C.c_int32, P, C.c_size_t]),
    "mt_set_trace": (C.c_int, [P, P, C.c_int64]),
    "mt_trace_count": (C.c_int, [P, C.POINTER(C.c_int64)]),
    "mt_last_error_info": (C.c_int, [P, C.POINTER(mt_error_info)]),
    "mt_last_error": (C.c_char_p, [P]),
    "mt_version": (C.c_char_p, []),
}
for _name, (_res, _args) in _sig.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args
    globals()[_name] = _f


def declared_functions():
    """Function names declared in include/mt.h (for the export check)."""
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:mt_status|const char \*)\s*(mt_[a-z_]+)\s*\(", txt, re.M)))


class MTError(RuntimeError):
    def __init__(self, status, msg, info=None):
        super().__init__(f"mt status {status}: {msg} {info or ''}")
        self.status = status
        self.info = info


def _i32(a):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.int32))
    return a, a.ctypes.data_as(I32P)


def _ptrs(lst):
    arr = (P * len(lst))(*[int(x) for x in lst])
    return arr


class Context:
    """Owns one mt_ctx.  device=-1 gives a host-only plan context (no CUDA calls)."""

    def __init__(self, device=0):
        self.h = P()
        st = mt_create(device, C.byref(self.h))
        if st != MT_OK:
            raise MTError(st, "mt_create failed")
        self.device = device
        self._keep = []
        self.ws = None
        self.n_tenants = 0

    def close(self):
        if self.h:
            mt_destroy(self.h)
            self.h = P()

    __del__ = close

    def check(self, st):
        if st != MT_OK:
            info = None
            if st == MT_ERR_VALIDATION:
                e = mt_error_info()
                mt_last_error_info(self.h, C.byref(e))
                info = (e.code, e.stage, e.tenant, e.op)
            raise MTError(st, mt_last_error(self.h).decode(), info)

    def set_option(self, opt, value):
        self.check(mt_set_option(self.h, opt, int(value)))

    # ---- graphs ------------------------------------------------------------------------
    def load_graphs(self, graphs, param_ptrs=None):
        """graphs: workloads.zoo.Graph list.  param_ptrs[t][j] = (weight, scale, shift) device
        addresses (ints) or None; host-only contexts may pass placeholders."""
        gs = (mt_graph * len(graphs))()
        keep = []
        for t, g in enumerate(graphs):
            nodes = (mt_node * g.n_ops)()
            for j, nd in enumerate(g.nodes):
                n = nodes[j]
                n.kind = nd["kind"]
                n.n_inputs = len(nd["inputs"])
                for q, i in enumerate(nd["inputs"]):
                    n.inputs[q] = i
                for f in ("out_c", "out_h", "out_w", "kh", "kw", "sh", "sw", "ph", "pw", "groups",
                          "ceil_mode", "count_include_pad", "act", "residual"):
                    setattr(n, f, int(nd[f]))
                if param_ptrs is not None and param_ptrs[t][j] is not None:
                    w, s, b = param_ptrs[t][j]
                    n.weight, n.scale, n.shift = w, s, b
            keep.append(nodes)
            gs[t].n_nodes = g.n_ops
            gs[t].nodes = C.cast(nodes, C.POINTER(mt_node))
            gs[t].batch, gs[t].in_c, gs[t].in_h, gs[t].in_w = g.batch, g.in_c, g.in_h, g.in_w
            gs[t].precision = g.precision
        self.check(mt_load_graphs(self.h, len(graphs), gs))
        self.n_tenants = len(graphs)
        self.lengths = [g.n_ops for g in graphs]

    def op_cost(self, t, j):
        f, b = C.c_int64(), C.c_int64()
        self.check(mt_op_cost(self.h, t, j, C.byref(f), C.byref(b)))
        return f.value, b.value

    def op_tiles(self, t, j):
        v = C.c_int32()
        self.check(mt_op_tiles(self.h, t, j, C.byref(v)))
        return v.value

    PLAN_KEYS = ("kind", "path", "bn", "splits", "tiles_m", "tiles_n", "stages", "tiles", "segments")
    PLAN_KINDS = ("conv_tc", "conv_simt", "dw", "pool", "gap", "fc", "elt")

    def op_plan(self, t, j):
        v = (C.c_int32 * len(self.PLAN_KEYS))()
        self.check(mt_op_plan(self.h, t, j, v))
        d = dict(zip(self.PLAN_KEYS, list(v)))
        d["kind"] = self.PLAN_KINDS[d["kind"]]
        return d

    def op_work(self, t, j):
        """[(tiles, ns per tile)] work items of op j (mt_op_work; split-K reduce tiles second)."""
        tiles = (C.c_int32 * 2)()
        ns = (C.c_int64 * 2)()
        self.check(mt_op_work(self.h, t, j, tiles, ns))
        return [(int(tiles[q]), int(ns[q])) for q in range(2) if tiles[q] > 0]

    def workspace_size(self):
        v = C.c_size_t()
        self.check(mt_workspace_size(self.h, C.byref(v)))
        return v.value

    def bind_workspace(self, ptr, nbytes):
        self.check(mt_bind_workspace(self.h, P(int(ptr)), nbytes))

    # ---- schedules ---------------------------------------------------------------------
    def set_schedule(self, ranges):
        """ranges: [S][N][2] (begin, end)"""
        arr = np.asarray(ranges, dtype=np.int32).reshape(-1, self.n_tenants, 2) if len(ranges) else \
            np.zeros((0, self.n_tenants, 2), np.int32)
        a, p = _i32(arr)
        self.check(mt_set_schedule(self.h, arr.shape[0], p))

    def set_schedule_pointers(self, rho):
        P_ = len(rho[0]) if len(rho) else 0
        if any(len(r) != P_ for r in rho) or len(rho) != self.n_tenants:
            raise MTError(MT_ERR_ARG, "rho must be [N][P]")
        a, p = _i32(np.asarray(rho, dtype=np.int32).reshape(-1) if P_ else np.zeros(1, np.int32))
        self.check(mt_set_schedule_pointers(self.h, P_, p))

    def num_stages(self):
        v = C.c_int32()
        self.check(mt_num_stages(self.h, C.byref(v)))
        return v.value

    def get_schedule(self):
        S = self.num_stages()
        out = np.zeros((S, self.n_tenants, 2), np.int32)
        self.check(mt_get_schedule(self.h, out.ctypes.data_as(I32P)))
        return out

    def stage_assignment(self):
        out = np.zeros(sum(self.lengths), np.int32)
        self.check(mt_stage_assignment(self.h, out.ctypes.data_as(I32P)))
        res, o = [], 0
        for L in self.lengths:
            res.append(out[o:o + L].tolist())
            o += L
        return res

    def sm_partition(self):
        S = self.num_stages()
        out = np.zeros((S, self.n_tenants), np.int32)
        self.check(mt_sm_partition(self.h, out.ctypes.data_as(I32P)))
        return out

    def stage_homes(self):
        """[S][grid] home tenant of every executor CTA per stage (mt_stage_homes)"""
        g = C.c_int32(0)
        self.check(mt_stage_homes(self.h, C.byref(g), None))
        out = np.zeros((self.num_stages(), g.value), np.int32)
        self.check(mt_stage_homes(self.h, C.byref(g), out.ctypes.data_as(I32P)))
        return out

    # ---- execution ---------------------------------------------------------------------
    def run(self, in_ptrs, out_ptrs, stream=0, timing=True):
        S = self.num_stages()
        stage = (C.c_float * S)()
        total = C.c_float()
        self.check(mt_run(self.h, _ptrs(in_ptrs), _ptrs(out_ptrs), stage, C.byref(total), P(stream)))
        return total.value, list(stage)

    def run_async(self, in_ptrs, out_ptrs, stream=0):
        self.check(mt_run_async(self.h, _ptrs(in_ptrs), _ptrs(out_ptrs), P(stream)))

    def run_host(self, host_in_ptrs, host_out_ptrs, stream=0):
        total = C.c_float()
        self.check(mt_run_host(self.h, _ptrs(host_in_ptrs), _ptrs(host_out_ptrs), C.byref(total), P(stream)))
        return total.value

    def run_baseline(self, mode, in_ptrs, out_ptrs, stream=0):
        total = C.c_float()
        self.check(mt_run_baseline(self.h, BASE_MODES[mode], _ptrs(in_ptrs), _ptrs(out_ptrs),
                                   C.byref(total), P(stream)))
        return total.value

    def profile_batch_pointers(self, cands, in_ptrs, out_ptrs, warmup=2, iters=10, stream=0):
        n = len(cands)
        Ps = np.array([len(r[0]) if len(r) else 0 for r in cands], np.int32)
        flat = np.concatenate([np.asarray(r, np.int32).reshape(-1) for r in cands] + [np.zeros(1, np.int32)])
        lat = np.zeros(n, np.float32)
        st = np.zeros(n, np.int32)
        self.check(mt_profile_batch_pointers(self.h, n, Ps.ctypes.data_as(I32P), flat.ctypes.data_as(I32P),
                                             _ptrs(in_ptrs), _ptrs(out_ptrs), warmup, iters,
                                             lat.ctypes.data_as(F32P), st.ctypes.data_as(I32P), P(stream)))
        return lat, st

    def estimate_batch_pointers(self, cands, peak_flops, mem_bw, op_latency_us, sync_us, c_compute=0.0,
                                c_memory=0.0, max_concurrency=1):
        """analytic pre-filter estimate (us) per candidate (include/mt.h); host-only"""
        n = len(cands)
        Ps = np.array([len(r[0]) if len(r) else 0 for r in cands], np.int32)
        flat = np.concatenate([np.asarray(r, np.int32).reshape(-1) for r in cands] + [np.zeros(1, np.int32)])
        est = np.zeros(n, np.float64)
        st = np.zeros(n, np.int32)
        prm = mt_cost_params(peak_flops, mem_bw, op_latency_us, sync_us, c_compute, c_memory, max_concurrency)
        self.check(mt_estimate_batch_pointers(self.h, C.byref(prm), n, Ps.ctypes.data_as(I32P),
                                              flat.ctypes.data_as(I32P),
                                              est.ctypes.data_as(C.POINTER(C.c_double)), st.ctypes.data_as(I32P)))
        return est, st

    def profile_batch(self, cand_ranges, in_ptrs, out_ptrs, warmup=2, iters=10, stream=0):
        n = len(cand_ranges)
        Ss = np.array([len(r) for r in cand_ranges], np.int32)
        flat = np.concatenate([np.asarray(r, np.int32).reshape(-1) for r in cand_ranges] + [np.zeros(1, np.int32)])
        lat = np.zeros(n, np.float32)
        st = np.zeros(n, np.int32)
        self.check(mt_profile_batch(self.h, n, Ss.ctypes.data_as(I32P), flat.ctypes.data_as(I32P),
                                    _ptrs(in_ptrs), _ptrs(out_ptrs), warmup, iters,
                                    lat.ctypes.data_as(F32P), st.ctypes.data_as(I32P), P(stream)))
        return lat, st

    def set_trace(self, dev_ptr, capacity):
        self.check(mt_set_trace(self.h, P(int(dev_ptr) if dev_ptr else 0), int(capacity)))

    def trace_count(self):
        v = C.c_int64()
        self.check(mt_trace_count(self.h, C.byref(v)))
        return v.value

    def get_activation(self, t, j, shape_nhwc, dtype):
        buf = np.zeros(shape_nhwc, dtype=dtype)
        self.check(mt_get_activation(self.h, t, j, P(buf.ctypes.data), buf.nbytes))
        return buf
