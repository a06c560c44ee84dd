"""Thin ctypes binding of libgbe.so (include/gbe.h): argument marshalling only.

Every computation runs in libgbe (C++ host planner + sm_100a CUDA kernels).
There is no CPU fallback: if libgbe.so is missing, or a solve is requested
without a CUDA device, the call raises.
"""
from __future__ import annotations

import ctypes
import json
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GBE_LIB") or os.path.join(_HERE, "libgbe.so")  # GBE_LIB: A/B builds

INF_I32 = 1 << 30
MAX_SEP = 40
MAX_INPUTS = 32

MINSUM_I32, MINSUM_F64, SUMPROD_F64 = 0, 1, 2
ORDER_MINFILL, ORDER_PAPER_DEGREE, ORDER_GIVEN = 0, 1, 2

STATUS = {0: "OK", 1: "INVALID", 2: "PARSE", 3: "BUDGET", 4: "CUDA", 5: "COMM", 6: "INTERNAL"}

EXPORTED = [
    "gbe_problem_create", "gbe_problem_load_wcsp", "gbe_problem_load_uai", "gbe_generate",
    "gbe_problem_info", "gbe_problem_destroy", "gbe_evaluate", "gbe_order", "gbe_pseudotree",
    "gbe_plan_create", "gbe_plan_info", "gbe_plan_destroy", "gbe_solve_be", "gbe_solve_mbe",
    "gbe_dpop_util", "gbe_dpop_value", "gbe_run_stats", "gbe_run_table", "gbe_run_destroy",
    "gbe_bucket_kernel", "gbe_set_allocator", "gbe_set_allgather", "gbe_last_error",
    "gbe_version", "gbe_bucket_kernel_variant", "gbe_comm_nccl_id", "gbe_comm_nccl_init",
    "gbe_comm_finalize", "gbe_solve_count", "gbe_run_count", "gbe_run_count_table",
    "gbe_set_table_hook", "gbe_bucket_kernel_ex",
]


class GbeError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"gbe {STATUS.get(status, status)}: {msg}")
        self.status = status


class Value(ctypes.Structure):
    _fields_ = [("is_inf", ctypes.c_int32), ("i", ctypes.c_int64), ("f", ctypes.c_double)]


class BucketDesc(ctypes.Structure):
    """Mirror of gbe_bucket_desc (include/gbe.h)."""
    _fields_ = [
        ("semiring", ctypes.c_int32), ("nsep", ctypes.c_int32), ("d", ctypes.c_int32),
        ("ninputs", ctypes.c_int32), ("rows", ctypes.c_int64),
        ("radix", ctypes.c_int32 * MAX_SEP),
        ("stride", (ctypes.c_int64 * MAX_SEP) * MAX_INPUTS),
        ("shift", ctypes.c_int64 * MAX_INPUTS),
    ]


AG_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                         ctypes.c_void_p, ctypes.c_void_p)
ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p)
FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p)
HOOK_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                           ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p)

_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with `make -C {os.path.dirname(_HERE)} gbe` "
                               "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        vp, i32, i64, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
        P = ctypes.POINTER
        pv = P(vp)
        L.gbe_problem_create.argtypes = [i32, vp, i32, vp, vp, i32, vp, pv]
        L.gbe_problem_load_wcsp.argtypes = [ctypes.c_char_p, pv]
        L.gbe_problem_load_uai.argtypes = [ctypes.c_char_p, ctypes.c_char_p, pv]
        L.gbe_generate.argtypes = [ctypes.c_char_p, pv]
        L.gbe_problem_info.argtypes = [vp, P(i32), P(i32), P(i32)]
        L.gbe_problem_destroy.argtypes = [vp]
        L.gbe_problem_destroy.restype = None
        L.gbe_evaluate.argtypes = [vp, vp, P(Value)]
        L.gbe_order.argtypes = [vp, i32, vp, vp, P(i32)]
        L.gbe_pseudotree.argtypes = [vp, vp, vp, vp]
        L.gbe_plan_create.argtypes = [vp, vp, i32, ctypes.c_char_p, pv]
        L.gbe_plan_info.argtypes = [vp, ctypes.c_char_p, sz]
        L.gbe_plan_destroy.argtypes = [vp]
        L.gbe_plan_destroy.restype = None
        L.gbe_solve_be.argtypes = [vp, vp, P(Value), vp, ctypes.c_char_p, sz]
        L.gbe_solve_mbe.argtypes = [vp, vp, P(Value), P(Value), vp, ctypes.c_char_p, sz]
        L.gbe_dpop_util.argtypes = [vp, vp, pv, P(Value)]
        L.gbe_dpop_value.argtypes = [vp, vp]
        L.gbe_run_stats.argtypes = [vp, ctypes.c_char_p, sz]
        L.gbe_run_table.argtypes = [vp, i32, vp, vp]
        L.gbe_solve_count.argtypes = [vp, vp, P(Value), P(ctypes.c_double)]
        L.gbe_run_count.argtypes = [vp, P(ctypes.c_double)]
        L.gbe_run_count_table.argtypes = [vp, i32, vp]
        L.gbe_run_destroy.argtypes = [vp]
        L.gbe_run_destroy.restype = None
        L.gbe_bucket_kernel.argtypes = [vp, vp, vp, vp, i64, i64, vp]
        L.gbe_bucket_kernel_ex.argtypes = [vp, vp, vp, vp, i64, i64, vp, i32]
        L.gbe_bucket_kernel_variant.argtypes = [vp, i64, i64]
        L.gbe_bucket_kernel_variant.restype = i32
        L.gbe_set_allocator.argtypes = [ALLOC_FN, FREE_FN, vp]
        L.gbe_set_allgather.argtypes = [AG_FN, vp]
        L.gbe_set_table_hook.argtypes = [HOOK_FN, vp]
        L.gbe_comm_nccl_id.argtypes = [vp]
        L.gbe_comm_nccl_init.argtypes = [vp, i32, i32, i32]
        L.gbe_comm_finalize.argtypes = []
        L.gbe_last_error.restype = ctypes.c_char_p
        L.gbe_version.restype = ctypes.c_char_p
        for name in EXPORTED:
            fn = getattr(L, name)
            if fn.restype is ctypes.c_int:  # default restype: gbe_status
                fn.restype = ctypes.c_int
        _LIB = L
    return _LIB


def _check(st):
    if st != 0:
        raise GbeError(st, lib().gbe_last_error().decode())


def _ptr(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else None


def _val(v: Value, f64: bool):
    if f64:
        return float(v.f)
    return int(v.i)


def _stream_ptr(stream):
    if stream is None:
        return None
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


class Problem:
    """gbe_problem: a WCSP / DCOP / MPE instance."""

    def __init__(self, handle):
        self._h = ctypes.c_void_p(handle)
        n, nf, sr = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        _check(lib().gbe_problem_info(self._h, ctypes.byref(n), ctypes.byref(nf), ctypes.byref(sr)))
        self.n, self.nf, self.is_f64 = n.value, nf.value, sr.value == MINSUM_F64

    @classmethod
    def create(cls, dom, arity, scopes, costs, f64=False):
        dom = np.ascontiguousarray(dom, dtype=np.int32)
        arity = np.ascontiguousarray(arity, dtype=np.int32)
        scopes = np.ascontiguousarray(scopes, dtype=np.int32)
        costs = np.ascontiguousarray(costs, dtype=np.float64 if f64 else np.int32)
        h = ctypes.c_void_p()
        _check(lib().gbe_problem_create(len(dom), _ptr(dom), len(arity), _ptr(arity),
                                        _ptr(scopes) if scopes.size else None,
                                        MINSUM_F64 if f64 else MINSUM_I32,
                                        _ptr(costs) if costs.size else None, ctypes.byref(h)))
        return cls(h.value)

    @classmethod
    def from_instance(cls, inst):
        """From a gen.Instance-like object (dom, arity, scopes, costs, is_f64)."""
        return cls.create(inst.dom, inst.arity, inst.scopes, inst.costs, bool(inst.is_f64))

    @classmethod
    def load_wcsp(cls, path):
        h = ctypes.c_void_p()
        _check(lib().gbe_problem_load_wcsp(path.encode(), ctypes.byref(h)))
        return cls(h.value)

    @classmethod
    def load_uai(cls, model, evid=None):
        h = ctypes.c_void_p()
        _check(lib().gbe_problem_load_uai(model.encode(), evid.encode() if evid else None, ctypes.byref(h)))
        return cls(h.value)

    @classmethod
    def generate(cls, **cfg):
        h = ctypes.c_void_p()
        _check(lib().gbe_generate(json.dumps(cfg).encode(), ctypes.byref(h)))
        return cls(h.value)

    def __del__(self):
        if getattr(self, "_h", None) and _LIB is not None:
            _LIB.gbe_problem_destroy(self._h)
            self._h = None

    def evaluate(self, assign):
        a = np.ascontiguousarray(assign, dtype=np.int32)
        v = Value()
        _check(lib().gbe_evaluate(self._h, _ptr(a), ctypes.byref(v)))
        return _val(v, self.is_f64)

    def order(self, kind=ORDER_MINFILL, given=None):
        out = np.zeros(max(self.n, 1), dtype=np.int32)
        w = ctypes.c_int32()
        g = np.ascontiguousarray(given, dtype=np.int32) if given is not None else None
        _check(lib().gbe_order(self._h, kind, _ptr(g), _ptr(out), ctypes.byref(w)))
        return out[:self.n], w.value

    def pseudotree(self, order):
        o = np.ascontiguousarray(order, dtype=np.int32)
        par = np.zeros(max(self.n, 1), dtype=np.int32)
        ss = np.zeros(max(self.n, 1), dtype=np.int32)
        _check(lib().gbe_pseudotree(self._h, _ptr(o), _ptr(par), _ptr(ss)))
        return par[:self.n], ss[:self.n]


class Plan:
    """gbe_plan: BE (ibound < 0) or MBE(ibound) over an ordering."""

    def __init__(self, problem: Problem, order, ibound=-1, **exec_opts):
        self.problem = problem
        self.order = np.ascontiguousarray(order, dtype=np.int32)
        self.ibound = ibound
        h = ctypes.c_void_p()
        _check(lib().gbe_plan_create(problem._h, _ptr(self.order), int(ibound),
                                     json.dumps(exec_opts).encode(), ctypes.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None) and _LIB is not None:
            _LIB.gbe_plan_destroy(self._h)
            self._h = None

    def info(self):
        cap = 1 << 16
        while True:
            buf = ctypes.create_string_buffer(cap)
            st = lib().gbe_plan_info(self._h, buf, cap)
            if st == 0:
                return json.loads(buf.value.decode())
            if cap > (1 << 30):
                _check(st)
            cap *= 4

    def solve_be(self, stream=None, stats=False, assignment=True):
        """(optimum, assignment[, stats]); assignment=False runs a value-only
        solve (no value phase; works with retain="none")."""
        v = Value()
        a = np.zeros(max(self.problem.n, 1), dtype=np.int32)
        cap = (1 << 22) if stats else 0
        buf = ctypes.create_string_buffer(cap) if stats else None
        _check(lib().gbe_solve_be(self._h, _stream_ptr(stream), ctypes.byref(v),
                                  _ptr(a) if assignment else None, buf, cap))
        out = (_val(v, self.problem.is_f64), a[:self.problem.n] if assignment else None)
        return out + (json.loads(buf.value.decode()),) if stats else out

    def log_z(self, stream=None):
        """log Z of a plan made with semiring="sumprod" (natural log of the
        partition function; -log P(E) for a belief network with evidence is
        -log_z()).  One value-only solve: -(gbe_solve_be's optimum)."""
        return -self.solve_be(stream, assignment=False)[0]

    def solve_count(self, stream=None):
        """(optimum, count) of a plan made with count="optimal" (number of
        optimal assignments) or count="consistent" (number of assignments of
        finite cost; optimum 0 or INF): solution counting."""
        v, c = Value(), ctypes.c_double()
        _check(lib().gbe_solve_count(self._h, _stream_ptr(stream), ctypes.byref(v), ctypes.byref(c)))
        return _val(v, self.problem.is_f64), c.value

    def solve_mbe(self, stream=None, stats=False, assignment=True):
        """(lower, upper, assignment[, stats]); assignment=False: lower bound
        only (no value phase; messages freed once consumed with retain="none")."""
        lo, up = Value(), Value()
        a = np.zeros(max(self.problem.n, 1), dtype=np.int32)
        cap = (1 << 22) if stats else 0
        buf = ctypes.create_string_buffer(cap) if stats else None
        _check(lib().gbe_solve_mbe(self._h, _stream_ptr(stream), ctypes.byref(lo),
                                   ctypes.byref(up) if assignment else None,
                                   _ptr(a) if assignment else None, buf, cap))
        f = self.problem.is_f64
        out = (_val(lo, f), _val(up, f) if assignment else None, a[:self.problem.n] if assignment else None)
        return out + (json.loads(buf.value.decode()),) if stats else out

    def dpop_util(self, stream=None):
        h = ctypes.c_void_p()
        v = Value()
        _check(lib().gbe_dpop_util(self._h, _stream_ptr(stream), ctypes.byref(h), ctypes.byref(v)))
        return Run(h, self), _val(v, self.problem.is_f64)


class Run:
    """gbe_run: device-resident UTIL messages / argmins of one UTIL phase."""

    def __init__(self, h, plan):
        self._h = h
        self.plan = plan  # the plan must outlive the run

    def __del__(self):
        self.close()

    def close(self):
        if getattr(self, "_h", None) and _LIB is not None:
            _LIB.gbe_run_destroy(self._h)
            self._h = None

    def value(self):
        a = np.zeros(max(self.plan.problem.n, 1), dtype=np.int32)
        _check(lib().gbe_dpop_value(self._h, _ptr(a)))
        return a[:self.plan.problem.n]

    def stats(self):
        cap = 1 << 22
        buf = ctypes.create_string_buffer(cap)
        _check(lib().gbe_run_stats(self._h, buf, cap))
        return json.loads(buf.value.decode())

    def table(self, t, rows, want_out=True, want_arg=True):
        f64 = self.plan.problem.is_f64
        out = np.zeros(max(rows, 1), dtype=np.float64 if f64 else np.int32) if want_out else None
        arg = np.zeros(max(rows, 1), dtype=np.uint8) if want_arg else None
        _check(lib().gbe_run_table(self._h, int(t), _ptr(out), _ptr(arg)))
        return (out[:rows] if out is not None else None), (arg[:rows] if arg is not None else None)


    def count(self):
        """number of optimal / consistent solutions (counting plans)"""
        c = ctypes.c_double()
        _check(lib().gbe_run_count(self._h, ctypes.byref(c)))
        return c.value

    def count_table(self, t, rows):
        """count table of table t (counting plans with retain="all")"""
        out = np.zeros(max(rows, 1), dtype=np.float64)
        _check(lib().gbe_run_count_table(self._h, int(t), _ptr(out)))
        return out[:rows]


def bucket_kernel(desc: BucketDesc, inputs, out, arg, row_begin, row_end, stream=None, variant=-1):
    """The hot primitive on device pointers (ints) or torch tensors; variant
    -1 auto, 0 generic, 1 tiled TMA, 2 streaming, 3 streaming staged
    (gbe_bucket_kernel_ex)."""
    def p(x):
        if x is None:
            return None
        return ctypes.c_void_p(x if isinstance(x, int) else x.data_ptr())
    arr = (ctypes.c_void_p * max(len(inputs), 1))(*[p(x) for x in inputs])
    if variant < 0:
        _check(lib().gbe_bucket_kernel(ctypes.byref(desc), arr, p(out), p(arg), int(row_begin),
                                       int(row_end), _stream_ptr(stream)))
    else:
        _check(lib().gbe_bucket_kernel_ex(ctypes.byref(desc), arr, p(out), p(arg), int(row_begin),
                                          int(row_end), _stream_ptr(stream), int(variant)))


def bucket_kernel_variant(desc: BucketDesc, row_begin, row_end):
    """0 = generic kernel, 1 = tiled TMA kernel, -1 = invalid descriptor."""
    return int(lib().gbe_bucket_kernel_variant(ctypes.byref(desc), int(row_begin), int(row_end)))


_HOOKS = {}


def set_allgather(fn):
    """fn(send_ptr, recv_ptr, nbytes, stream_ptr) -> 0 on success; None clears."""
    if fn is None:
        _check(lib().gbe_set_allgather(AG_FN(), None))
        _HOOKS.pop("ag", None)
        return
    cb = AG_FN(lambda s, r, n, st, u: int(fn(s, r, n, st)))
    _HOOKS["ag"] = cb
    _check(lib().gbe_set_allgather(cb, None))


def set_table_hook(fn):
    """fn(task, dev_out_ptr, dev_arg_ptr, row_begin, rows, stream_ptr) -> 0, called
    after every bucket of a solve (gbe_set_table_hook); None removes it.  An
    exception inside fn aborts the solve (GBE_E_INTERNAL)."""
    if fn is None:
        _check(lib().gbe_set_table_hook(HOOK_FN(), None))
        _HOOKS.pop("table", None)
        return

    def cb(t, o, a, rb, n, st, u):
        try:
            return int(fn(int(t), o, a, int(rb), int(n), st) or 0)
        except Exception as e:  # noqa: BLE001 -- reported through the status
            _HOOKS["table_error"] = e
            return 1
    h = HOOK_FN(cb)
    _HOOKS["table"] = h
    _HOOKS.pop("table_error", None)
    _check(lib().gbe_set_table_hook(h, None))


def table_hook_error():
    """The exception raised inside the last failing table hook (or None)."""
    return _HOOKS.get("table_error")


def set_allocator(alloc, free):
    """alloc(nbytes, stream_ptr) -> device ptr; free(ptr). None restores the default."""
    if alloc is None:
        _check(lib().gbe_set_allocator(ALLOC_FN(), FREE_FN(), None))
        _HOOKS.pop("alloc", None)
        return
    a = ALLOC_FN(lambda n, st, u: alloc(n, st))
    f = FREE_FN(lambda p, u: free(p))
    _HOOKS["alloc"] = (a, f)
    _check(lib().gbe_set_allocator(a, f, None))


def comm_nccl_id() -> bytes:
    """128-byte NCCL unique id (rank 0)."""
    buf = ctypes.create_string_buffer(128)
    _check(lib().gbe_comm_nccl_id(buf))
    return buf.raw


def comm_nccl_init(uid: bytes, nranks: int, rank: int, device: int):
    """Built-in NCCL all-gather for row-sharded plans (all ranks)."""
    buf = ctypes.create_string_buffer(bytes(uid), 128)
    _check(lib().gbe_comm_nccl_init(buf, int(nranks), int(rank), int(device)))


def comm_finalize():
    _check(lib().gbe_comm_finalize())


def version():
    return lib().gbe_version().decode()
