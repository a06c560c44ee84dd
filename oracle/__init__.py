"""CPU oracle for the BE / MBE / DPOP bucket computation.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package.  The product
path (paper_1608_05288_b200) never imports it and shares no code with it.

The arithmetic lives in oracle/oracle.c (plain C, every function citing the
PAPER.md passage it restates); oracle/brute.py is a pure-Python brute force
for tiny instances.  Pins: tests/test_oracle_pins.py.  Parity unpinned:
Examples 3/4 numeric values (Fig. 1(b) tables are missing from PAPER.md).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

INF_I32 = 1 << 30
I32P = ctypes.POINTER(ctypes.c_int32)
I64P = ctypes.POINTER(ctypes.c_int64)
F64P = ctypes.POINTER(ctypes.c_double)
U8P = ctypes.POINTER(ctypes.c_uint8)


class OrProblem(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int32), ("nf", ctypes.c_int32), ("is_f64", ctypes.c_int32),
        ("dom", I32P), ("arity", I32P), ("scope_off", I64P), ("scopes", I32P),
        ("table_off", I64P), ("icost", I32P), ("fcost", F64P),
    ]


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make -C {os.path.dirname(_HERE)} oracle`")
        L = ctypes.CDLL(path)
        PP = ctypes.POINTER(OrProblem)
        L.or_primal_graph.argtypes = [PP, U8P]
        L.or_induced_width.argtypes = [PP, I32P]
        L.or_induced_width.restype = ctypes.c_int32
        L.or_minfill_order.argtypes = [PP, I32P]
        L.or_degree_order.argtypes = [PP, I32P]
        L.or_elim_tree.argtypes = [PP, I32P, I32P]
        L.or_bucket_rows.argtypes = [I32P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                     ctypes.c_int32, I32P, I64P, I32P,
                                     ctypes.POINTER(I32P), ctypes.POINTER(F64P),
                                     ctypes.c_int32, I32P, ctypes.c_int64, ctypes.c_int64,
                                     I32P, F64P, U8P, ctypes.c_int32]
        L.or_solve.argtypes = [PP, I32P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32]
        L.or_solve.restype = ctypes.c_void_p
        L.or_bucket_row_sums.argtypes = [I32P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                         ctypes.c_int32, I32P, I64P, I32P,
                                         ctypes.POINTER(I32P), ctypes.POINTER(F64P),
                                         ctypes.c_int32, I32P, ctypes.c_int64, I64P, I64P, F64P]
        L.or_bucket_rows_sp.argtypes = [I32P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                        I32P, I64P, I32P, ctypes.POINTER(F64P), ctypes.c_int32,
                                        I32P, ctypes.c_int64, ctypes.c_int64, F64P, ctypes.c_int32]
        L.or_solve_sumprod.argtypes = [PP, I32P, ctypes.c_int32, ctypes.c_int32]
        L.or_solve_sumprod.restype = ctypes.c_void_p
        L.or_solve_count.argtypes = [PP, I32P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32]
        L.or_solve_count.restype = ctypes.c_void_p
        L.or_run_count.argtypes = [ctypes.c_void_p]
        L.or_run_count.restype = ctypes.c_double
        L.or_run_table_count.argtypes = [ctypes.c_void_p, ctypes.c_int32, F64P]
        L.or_run_table_count.restype = ctypes.c_int32
        L.or_run_status.argtypes = [ctypes.c_void_p]
        L.or_run_status.restype = ctypes.c_int32
        L.or_run_ntables.argtypes = [ctypes.c_void_p]
        L.or_run_ntables.restype = ctypes.c_int32
        L.or_run_table_meta.argtypes = [ctypes.c_void_p, ctypes.c_int32, I32P, I32P, I32P,
                                        I64P, I32P, I32P]
        L.or_run_table_sep.argtypes = [ctypes.c_void_p, ctypes.c_int32, I32P]
        L.or_run_table_members.argtypes = [ctypes.c_void_p, ctypes.c_int32, I32P, I32P]
        L.or_run_table_out.argtypes = [ctypes.c_void_p, ctypes.c_int32, I32P, F64P, U8P]
        L.or_run_table_out.restype = ctypes.c_int32
        L.or_run_table_digest.argtypes = [ctypes.c_void_p, ctypes.c_int32]
        L.or_run_table_digest.restype = ctypes.c_uint64
        for nm, rt in [("or_run_value_i", ctypes.c_int64), ("or_run_value_f", ctypes.c_double),
                       ("or_run_upper_i", ctypes.c_int64), ("or_run_upper_f", ctypes.c_double)]:
            getattr(L, nm).argtypes = [ctypes.c_void_p]
            getattr(L, nm).restype = rt
        L.or_run_assignment.argtypes = [ctypes.c_void_p, I32P]
        L.or_run_assignment.restype = ctypes.c_int32
        L.or_run_free.argtypes = [ctypes.c_void_p]
        L.or_evaluate_i.argtypes = [PP, I32P]
        L.or_evaluate_i.restype = ctypes.c_int64
        L.or_evaluate_f.argtypes = [PP, I32P]
        L.or_evaluate_f.restype = ctypes.c_double
        L.or_fnv1a.argtypes = [ctypes.c_uint64, ctypes.c_void_p, ctypes.c_int64]
        L.or_fnv1a.restype = ctypes.c_uint64
        L.or_mixsum.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64,
                                ctypes.c_int32]
        L.or_mixsum.restype = ctypes.c_uint64
        L.or_set_digest_kind.argtypes = [ctypes.c_int32]
        L.or_set_digest_kind.restype = None
        _LIB = L
    return _LIB


def _p(a, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


class Problem:
    """Keeps the numpy arrays alive and exposes the C struct."""

    def __init__(self, inst):
        self.inst = inst
        self.dom = np.ascontiguousarray(inst.dom, dtype=np.int32)
        self.arity = np.ascontiguousarray(inst.arity, dtype=np.int32)
        self.scope_off = np.ascontiguousarray(inst.scope_off, dtype=np.int64)
        self.scopes = np.ascontiguousarray(inst.scopes, dtype=np.int32)
        self.table_off = np.ascontiguousarray(inst.table_off, dtype=np.int64)
        self.is_f64 = bool(inst.is_f64)
        if self.is_f64:
            self.fcost = np.ascontiguousarray(inst.costs, dtype=np.float64)
            self.icost = None
        else:
            self.icost = np.ascontiguousarray(inst.costs, dtype=np.int32)
            self.fcost = None
        if self.scopes.size == 0:
            self.scopes = np.zeros(1, np.int32)
        self.s = OrProblem(inst.n, inst.nf, int(self.is_f64), _p(self.dom, ctypes.c_int32),
                           _p(self.arity, ctypes.c_int32), _p(self.scope_off, ctypes.c_int64),
                           _p(self.scopes, ctypes.c_int32), _p(self.table_off, ctypes.c_int64),
                           _p(self.icost, ctypes.c_int32) if self.icost is not None else None,
                           _p(self.fcost, ctypes.c_double) if self.fcost is not None else None)

    @property
    def ref(self):
        return ctypes.byref(self.s)


def primal_graph(inst) -> np.ndarray:
    P = Problem(inst)
    adj = np.zeros((inst.n, inst.n), dtype=np.uint8)
    lib().or_primal_graph(P.ref, _p(adj, ctypes.c_uint8))
    return adj


def induced_width(inst, order) -> int:
    P = Problem(inst)
    o = np.ascontiguousarray(order, dtype=np.int32)
    return int(lib().or_induced_width(P.ref, _p(o, ctypes.c_int32)))


def minfill_order(inst) -> np.ndarray:
    P = Problem(inst)
    o = np.zeros(max(inst.n, 1), dtype=np.int32)
    lib().or_minfill_order(P.ref, _p(o, ctypes.c_int32))
    return o[:inst.n]


def degree_order(inst) -> np.ndarray:
    P = Problem(inst)
    o = np.zeros(max(inst.n, 1), dtype=np.int32)
    lib().or_degree_order(P.ref, _p(o, ctypes.c_int32))
    return o[:inst.n]


def elim_tree(inst, order) -> np.ndarray:
    P = Problem(inst)
    o = np.ascontiguousarray(order, dtype=np.int32)
    par = np.zeros(max(inst.n, 1), dtype=np.int32)
    lib().or_elim_tree(P.ref, _p(o, ctypes.c_int32), _p(par, ctypes.c_int32))
    return par[:inst.n]


def evaluate(inst, assign):
    P = Problem(inst)
    a = np.ascontiguousarray(assign, dtype=np.int32)
    if inst.is_f64:
        return float(lib().or_evaluate_f(P.ref, _p(a, ctypes.c_int32)))
    return int(lib().or_evaluate_i(P.ref, _p(a, ctypes.c_int32)))


def fnv1a(*arrays) -> int:
    h = 0xcbf29ce484222325
    for a in arrays:
        a = np.ascontiguousarray(a)
        h = lib().or_fnv1a(h, a.ctypes.data, a.nbytes)
    return int(h)


def mixsum(a, salt, nthreads=0) -> int:
    """or_mixsum: position-keyed sum checksum of a 1/4/8-byte array (mod 2^64)."""
    a = np.ascontiguousarray(a)
    return int(lib().or_mixsum(a.ctypes.data, a.itemsize, a.size, salt, nthreads))


def mix_digest(out, arg, nthreads=0) -> int:
    """Table digest of digest kind 1: mixsum(out, 1) + mixsum(arg, 2) mod 2^64."""
    return (mixsum(out, 1, nthreads) + mixsum(arg, 2, nthreads)) & ((1 << 64) - 1)


def set_digest_kind(kind: int):
    """Digest or_solve records per table: 0 FNV-1a (default), 1 mix_digest."""
    lib().or_set_digest_kind(int(kind))


def bucket_eval(dom, is_f64, x, members, sep, row_begin=0, row_end=None, nthreads=0):
    """Rows [row_begin, row_end) of pi_{-x}(sum members); sep most significant
    first.  members = [(scope, flat table in that scope order)]."""
    dom = np.ascontiguousarray(dom, dtype=np.int32)
    sep = [int(v) for v in sep]
    if row_end is None:
        row_end = int(np.prod([dom[v] for v in sep], dtype=np.int64)) if sep else 1
    nm = len(members)
    mar = np.array([len(s) for s, _ in members] + [0], dtype=np.int32)
    moff = np.zeros(nm + 1, dtype=np.int64)
    moff[1:] = np.cumsum(mar[:nm]) if nm else []
    flat = [int(v) for s, _ in members for v in s]
    msc = np.array(flat + [0], dtype=np.int32)
    tabs = [np.ascontiguousarray(t, dtype=np.float64 if is_f64 else np.int32) for _, t in members]
    it = (I32P * (nm + 1))()
    ft = (F64P * (nm + 1))()
    for k, t in enumerate(tabs):
        if is_f64:
            ft[k] = _p(t, ctypes.c_double)
        else:
            it[k] = _p(t, ctypes.c_int32)
    sepa = np.array(sep + [0], dtype=np.int32)
    nrows = row_end - row_begin
    out = np.zeros(max(nrows, 1), dtype=np.float64 if is_f64 else np.int32)
    arg = np.zeros(max(nrows, 1), dtype=np.uint8)
    lib().or_bucket_rows(_p(dom, ctypes.c_int32), len(dom), int(is_f64), int(x), nm,
                         _p(mar, ctypes.c_int32), _p(moff, ctypes.c_int64), _p(msc, ctypes.c_int32),
                         it, ft, len(sep), _p(sepa, ctypes.c_int32), row_begin, row_end,
                         _p(out, ctypes.c_int32) if not is_f64 else None,
                         _p(out, ctypes.c_double) if is_f64 else None,
                         _p(arg, ctypes.c_uint8), nthreads)
    return out[:nrows], arg[:nrows]


def _members_c(members, is_f64):
    nm = len(members)
    mar = np.array([len(s) for s, _ in members] + [0], dtype=np.int32)
    moff = np.zeros(nm + 1, dtype=np.int64)
    moff[1:] = np.cumsum(mar[:nm]) if nm else []
    msc = np.array([int(v) for s, _ in members for v in s] + [0], dtype=np.int32)
    tabs = [np.ascontiguousarray(t, dtype=np.float64 if is_f64 else np.int32) for _, t in members]
    it = (I32P * (nm + 1))()
    ft = (F64P * (nm + 1))()
    for k, t in enumerate(tabs):
        if is_f64:
            ft[k] = _p(t, ctypes.c_double)
        else:
            it[k] = _p(t, ctypes.c_int32)
    return nm, mar, moff, msc, tabs, it, ft


def bucket_row_sums(dom, is_f64, x, members, sep, rows):
    """Aggregated sums (before the min over x) of the given output rows:
    array [len(rows), d] -- or_bucket_row_sums."""
    dom = np.ascontiguousarray(dom, dtype=np.int32)
    sep = [int(v) for v in sep]
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    nm, mar, moff, msc, tabs, it, ft = _members_c(members, is_f64)
    sepa = np.array(sep + [0], dtype=np.int32)
    d = int(dom[x])
    si = np.zeros(max(rows.size * d, 1), dtype=np.int64)
    sf = np.zeros(max(rows.size * d, 1), dtype=np.float64)
    lib().or_bucket_row_sums(_p(dom, ctypes.c_int32), len(dom), int(is_f64), int(x), nm,
                             _p(mar, ctypes.c_int32), _p(moff, ctypes.c_int64), _p(msc, ctypes.c_int32),
                             it, ft, len(sep), _p(sepa, ctypes.c_int32), rows.size, _p(rows, ctypes.c_int64),
                             _p(si, ctypes.c_int64), _p(sf, ctypes.c_double))
    s = sf if is_f64 else si
    return s[:rows.size * d].reshape(rows.size, d)


def bucket_eval_sp(dom, x, members, sep, row_begin=0, row_end=None, nthreads=0):
    """Sum-product bucket (or_bucket_rows_sp): rows [row_begin, row_end) of
    -log sum_x exp(-sum members); f64 members [(scope, table)]."""
    dom = np.ascontiguousarray(dom, dtype=np.int32)
    sep = [int(v) for v in sep]
    if row_end is None:
        row_end = int(np.prod([dom[v] for v in sep], dtype=np.int64)) if sep else 1
    nm = len(members)
    mar = np.array([len(s) for s, _ in members] + [0], dtype=np.int32)
    moff = np.zeros(nm + 1, dtype=np.int64)
    moff[1:] = np.cumsum(mar[:nm]) if nm else []
    msc = np.array([int(v) for s, _ in members for v in s] + [0], dtype=np.int32)
    tabs = [np.ascontiguousarray(t, dtype=np.float64) for _, t in members]
    ft = (F64P * (nm + 1))()
    for k, t in enumerate(tabs):
        ft[k] = _p(t, ctypes.c_double)
    sepa = np.array(sep + [0], dtype=np.int32)
    nrows = row_end - row_begin
    out = np.zeros(max(nrows, 1), dtype=np.float64)
    lib().or_bucket_rows_sp(_p(dom, ctypes.c_int32), len(dom), int(x), nm, _p(mar, ctypes.c_int32),
                            _p(moff, ctypes.c_int64), _p(msc, ctypes.c_int32), ft, len(sep),
                            _p(sepa, ctypes.c_int32), row_begin, row_end, _p(out, ctypes.c_double),
                            nthreads)
    return out[:nrows]


class Table:
    __slots__ = ("var", "mb", "sep", "rows", "dest", "members", "out", "arg", "digest", "count")


class Run:
    """Result of or_solve: tables in creation order, optimum / bounds,
    assignment."""

    def __init__(self, inst, order, ibound=-1, keep_tables=True, nthreads=0, table_fn=None,
                 sumprod=False, count=None):
        """table_fn(t, table, out, arg), if given, receives each kept table
        instead of the Run storing a copy (bounded memory for big runs).
        sumprod: exact BE in the sum-product semiring (f64; value = -log Z).
        count: "optimal" / "consistent" -- exact BE in the (min, count)
        semiring; .count = number of optimal / consistent solutions and every
        kept table gets .count (doubles)."""
        self.inst = inst
        self._P = Problem(inst)
        self.order = np.ascontiguousarray(order, dtype=np.int32)
        L = lib()
        if count is not None:
            if ibound >= 0 or count not in ("optimal", "consistent"):
                raise ValueError("counting oracle: exact BE, count = 'optimal' or 'consistent'")
            h = L.or_solve_count(self._P.ref, _p(self.order, ctypes.c_int32), int(count == "consistent"),
                                 int(bool(keep_tables)), int(nthreads))
        elif sumprod:
            if not inst.is_f64 or ibound >= 0:
                raise ValueError("sum-product oracle: f64 problems, exact BE only")
            h = L.or_solve_sumprod(self._P.ref, _p(self.order, ctypes.c_int32),
                                   int(bool(keep_tables)), int(nthreads))
        else:
            h = L.or_solve(self._P.ref, _p(self.order, ctypes.c_int32), int(ibound),
                           int(bool(keep_tables)), int(nthreads))
        try:
            self.status = int(L.or_run_status(h))
            self.tables = []
            if self.status == 0:
                for t in range(L.or_run_ntables(h)):
                    var, mb, nsep, dest, nmem = (ctypes.c_int32() for _ in range(5))
                    rows = ctypes.c_int64()
                    L.or_run_table_meta(h, t, ctypes.byref(var), ctypes.byref(mb), ctypes.byref(nsep),
                                        ctypes.byref(rows), ctypes.byref(dest), ctypes.byref(nmem))
                    T = Table()
                    T.var, T.mb, T.rows, T.dest = var.value, mb.value, rows.value, dest.value
                    sep = np.zeros(max(nsep.value, 1), dtype=np.int32)
                    L.or_run_table_sep(h, t, _p(sep, ctypes.c_int32))
                    T.sep = sep[:nsep.value].copy()
                    kind = np.zeros(max(nmem.value, 1), dtype=np.int32)
                    idx = np.zeros(max(nmem.value, 1), dtype=np.int32)
                    L.or_run_table_members(h, t, _p(kind, ctypes.c_int32), _p(idx, ctypes.c_int32))
                    T.members = [(int(kind[k]), int(idx[k])) for k in range(nmem.value)]
                    T.digest = int(L.or_run_table_digest(h, t))
                    T.out, T.arg, T.count = None, None, None
                    if keep_tables and count is not None:
                        c = np.zeros(T.rows, dtype=np.float64)
                        if L.or_run_table_count(h, t, _p(c, ctypes.c_double)):
                            T.count = c
                    if keep_tables:
                        out = np.zeros(T.rows, dtype=np.float64 if inst.is_f64 else np.int32)
                        arg = np.zeros(T.rows, dtype=np.uint8)
                        ok = L.or_run_table_out(h, t, None if inst.is_f64 else _p(out, ctypes.c_int32),
                                                _p(out, ctypes.c_double) if inst.is_f64 else None,
                                                _p(arg, ctypes.c_uint8))
                        if ok:
                            if table_fn is not None:
                                table_fn(t, T, out, arg)
                            else:
                                T.out, T.arg = out, arg
                        del out, arg
                    self.tables.append(T)
                if inst.is_f64:
                    self.value = float(L.or_run_value_f(h))
                    self.upper = float(L.or_run_upper_f(h))
                else:
                    self.value = int(L.or_run_value_i(h))
                    self.upper = int(L.or_run_upper_i(h))
                self.count = float(L.or_run_count(h)) if count is not None else None
                a = np.zeros(max(inst.n, 1), dtype=np.int32)
                self.assignment = a[:inst.n].copy() if L.or_run_assignment(h, _p(a, ctypes.c_int32)) else None
                if self.assignment is not None:
                    self.assignment = a[:inst.n].copy()
        finally:
            L.or_run_free(h)


def solve_be(inst, order, keep_tables=True, nthreads=0) -> Run:
    return Run(inst, order, -1, keep_tables, nthreads)


def solve_mbe(inst, order, ibound, keep_tables=True, nthreads=0) -> Run:
    return Run(inst, order, ibound, keep_tables, nthreads)


def solve_sumprod(inst, order, keep_tables=True, nthreads=0) -> Run:
    """Exact BE in the sum-product semiring: .value = -log Z."""
    return Run(inst, order, -1, keep_tables, nthreads, sumprod=True)


def solve_count(inst, order, count="optimal", keep_tables=True, nthreads=0) -> Run:
    """Exact BE in the (min, count) semiring:
    .count = number of optimal (count="optimal") or consistent
    (count="consistent") solutions."""
    return Run(inst, order, -1, keep_tables, nthreads, count=count)
