"""Seeded synthetic instance generators shared by the oracle and the CUDA path.

This package holds none of the method's arithmetic: it draws graphs and cost
tables (gen/gen.c, splitmix64) and writes/reads nothing but plain arrays and
the WCSP / UAI text formats.  See gen/gen.h for the topology definitions
(§8.1) and DESIGN.md §4 for the input recipe.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

INF_I32 = 1 << 30


class _GenInstance(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int32),
        ("nf", ctypes.c_int32),
        ("is_f64", ctypes.c_int32),
        ("dom", ctypes.POINTER(ctypes.c_int32)),
        ("arity", ctypes.POINTER(ctypes.c_int32)),
        ("scope_off", ctypes.POINTER(ctypes.c_int64)),
        ("scopes", ctypes.POINTER(ctypes.c_int32)),
        ("table_off", ctypes.POINTER(ctypes.c_int64)),
        ("icost", ctypes.POINTER(ctypes.c_int32)),
        ("fcost", ctypes.POINTER(ctypes.c_double)),
    ]


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "libgbegen.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make -C {os.path.dirname(_HERE)} gen`")
        L = ctypes.CDLL(path)
        P = ctypes.POINTER(_GenInstance)
        L.gen_random_graph.restype = P
        L.gen_random_graph.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_int64,
                                       ctypes.c_int32, ctypes.c_double, ctypes.c_uint64]
        L.gen_scalefree.restype = P
        L.gen_scalefree.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_double, ctypes.c_uint64]
        L.gen_grid.restype = P
        L.gen_grid.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_double,
                               ctypes.c_uint64]
        L.gen_belief_net.restype = P
        L.gen_belief_net.argtypes = [ctypes.c_int32] * 5 + [ctypes.c_uint64]
        L.gen_random_network.restype = P
        L.gen_random_network.argtypes = [ctypes.c_int32] * 7 + [ctypes.c_double, ctypes.c_uint64]
        L.gen_random_network_f64.restype = P
        L.gen_random_network_f64.argtypes = [ctypes.c_int32] * 6 + [ctypes.c_double, ctypes.c_double,
                                                                  ctypes.c_uint64]
        L.gen_free.argtypes = [P]
        L.gen_free.restype = None
        L.gen_splitmix64.argtypes = [ctypes.POINTER(ctypes.c_uint64)]
        L.gen_splitmix64.restype = ctypes.c_uint64
        _LIB = L
    return _LIB


@dataclass
class Instance:
    """A cost network: domains, function scopes (declared order) and flat
    tables (lexicographic, first scope variable most significant).
    is_f64: float64 costs (MPE as -log p), else int32 with INF = 2^30."""

    dom: np.ndarray
    arity: np.ndarray
    scope_off: np.ndarray
    scopes: np.ndarray
    table_off: np.ndarray
    costs: np.ndarray
    is_f64: bool
    name: str = ""
    meta: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return int(self.dom.shape[0])

    @property
    def nf(self) -> int:
        return int(self.arity.shape[0])

    def scope(self, f: int) -> np.ndarray:
        return self.scopes[self.scope_off[f]:self.scope_off[f + 1]]

    def table(self, f: int) -> np.ndarray:
        return self.costs[self.table_off[f]:self.table_off[f + 1]]

    def edges(self):
        """Primal-graph edge set as sorted (u, v) pairs, u < v."""
        es = set()
        for f in range(self.nf):
            s = [int(v) for v in self.scope(f)]
            for a in s:
                for b in s:
                    if a < b:
                        es.add((a, b))
        return sorted(es)

    @staticmethod
    def from_functions(dom, functions, is_f64=False, name=""):
        """Build from a list of (scope list, flat table) pairs."""
        dom = np.ascontiguousarray(dom, dtype=np.int32)
        arity = np.array([len(s) for s, _ in functions], dtype=np.int32)
        scope_off = np.zeros(len(functions) + 1, dtype=np.int64)
        scope_off[1:] = np.cumsum(arity)
        table_off = np.zeros(len(functions) + 1, dtype=np.int64)
        sizes = []
        for s, t in functions:
            cells = int(np.prod([dom[v] for v in s], dtype=np.int64)) if len(s) else 1
            if len(t) != cells:
                raise ValueError("table size does not match scope domains")
            sizes.append(cells)
        table_off[1:] = np.cumsum(sizes) if sizes else []
        scopes = (np.concatenate([np.asarray(s, dtype=np.int32) for s, _ in functions])
                  if int(arity.sum()) else np.zeros(0, dtype=np.int32))
        dt = np.float64 if is_f64 else np.int32
        costs = (np.concatenate([np.asarray(t, dtype=dt) for _, t in functions])
                 if functions else np.zeros(0, dtype=dt))
        return Instance(dom, arity, scope_off, scopes.astype(np.int32), table_off,
                        np.ascontiguousarray(costs), bool(is_f64), name)


def _take(ptr) -> Instance:
    if not ptr:
        raise RuntimeError("generator failed (parameters infeasible)")
    g = ptr.contents
    n, nf = g.n, g.nf
    dom = np.ctypeslib.as_array(g.dom, shape=(n,)).copy()
    arity = np.ctypeslib.as_array(g.arity, shape=(nf,)).copy() if nf else np.zeros(0, np.int32)
    scope_off = np.ctypeslib.as_array(g.scope_off, shape=(nf + 1,)).copy()
    table_off = np.ctypeslib.as_array(g.table_off, shape=(nf + 1,)).copy()
    ns, nt = int(scope_off[-1]), int(table_off[-1])
    scopes = np.ctypeslib.as_array(g.scopes, shape=(ns,)).copy() if ns else np.zeros(0, np.int32)
    if g.is_f64:
        costs = np.ctypeslib.as_array(g.fcost, shape=(nt,)).copy()
    else:
        costs = np.ctypeslib.as_array(g.icost, shape=(nt,)).copy()
    inst = Instance(dom, arity, scope_off, scopes, table_off, costs, bool(g.is_f64))
    lib().gen_free(ptr)
    return inst


def random_graph(n, d, nedges, mode=0, p2=0.0, seed=0) -> Instance:
    """Random topology: mode 0 = `nedges` uniform pairs resampled until
    connected; mode 1 = uniform spanning tree + uniform extra edges."""
    inst = _take(lib().gen_random_graph(n, d, nedges, mode, p2, seed))
    inst.name = f"random(n={n},d={d},e={nedges},mode={mode},p2={p2},seed={seed})"
    return inst


def scalefree(n, d, p2=0.0, seed=0) -> Instance:
    """Barabasi-Albert, 2(n-2)+1 edges."""
    inst = _take(lib().gen_scalefree(n, d, p2, seed))
    inst.name = f"scalefree(n={n},d={d},p2={p2},seed={seed})"
    return inst


def grid(rows, cols, d, p2=0.0, seed=0) -> Instance:
    """rows x cols lattice."""
    inst = _take(lib().gen_grid(rows, cols, d, p2, seed))
    inst.name = f"grid({rows}x{cols},d={d},p2={p2},seed={seed})"
    return inst


def belief_net(n, dmin=2, dmax=4, maxpar=3, window=20, seed=0) -> Instance:
    """Belief network, CPTs ~ Dirichlet(1) stored as -log p."""
    inst = _take(lib().gen_belief_net(n, dmin, dmax, maxpar, window, seed))
    inst.name = f"bn(n={n},d={dmin}-{dmax},par={maxpar},win={window},seed={seed})"
    return inst


def random_network(n, dmin, dmax, nf, amin, amax, cmax=100, p2=0.0, seed=0) -> Instance:
    inst = _take(lib().gen_random_network(n, dmin, dmax, nf, amin, amax, cmax, p2, seed))
    inst.name = f"net(n={n},d={dmin}-{dmax},nf={nf},a={amin}-{amax},p2={p2},seed={seed})"
    return inst


def random_network_f64(n, dmin, dmax, nf, amin, amax, fmax=10.0, p2=0.0, seed=0) -> Instance:
    inst = _take(lib().gen_random_network_f64(n, dmin, dmax, nf, amin, amax, fmax, p2, seed))
    inst.name = f"netf(n={n},d={dmin}-{dmax},nf={nf},a={amin}-{amax},p2={p2},seed={seed})"
    return inst


def splitmix_stream(seed: int, count: int) -> np.ndarray:
    """`count` raw splitmix64 outputs from `seed` (same generator as gen.c)."""
    s = ctypes.c_uint64(seed)
    return np.array([lib().gen_splitmix64(ctypes.byref(s)) for _ in range(count)], dtype=np.uint64)


# ---------------------------------------------------------------------------
# text formats (SPEC.md S:507-525 layouts)

def write_wcsp(inst: Instance, path: str, ub: int = INF_I32) -> None:
    """WCSP text: `name n maxdom nf ub`, domains, then per function
    `arity vars... default ntuples` and one `values... cost` line per tuple.
    Costs >= ub mean infinity.  Every cell is listed explicitly (default 0)."""
    assert not inst.is_f64
    lines = [f"{inst.name or 'gbe'} {inst.n} {int(inst.dom.max()) if inst.n else 0} {inst.nf} {ub}",
             " ".join(str(int(d)) for d in inst.dom)]
    for f in range(inst.nf):
        sc = [int(v) for v in inst.scope(f)]
        t = inst.table(f)
        lines.append(" ".join([str(len(sc))] + [str(v) for v in sc] + ["0", str(len(t))]))
        dims = [int(inst.dom[v]) for v in sc]
        for idx, c in enumerate(t):
            tup = np.unravel_index(idx, dims) if dims else ()
            cost = ub if int(c) >= INF_I32 else int(c)
            lines.append(" ".join([str(int(x)) for x in tup] + [str(cost)]))
    with open(path, "w") as fh:
        fh.write("\n".join(lines) + "\n")


def write_uai(inst: Instance, path: str) -> None:
    """UAI BAYES text with probabilities p = exp(-cost)."""
    assert inst.is_f64
    lines = ["BAYES", str(inst.n), " ".join(str(int(d)) for d in inst.dom), str(inst.nf)]
    for f in range(inst.nf):
        sc = [int(v) for v in inst.scope(f)]
        lines.append(" ".join([str(len(sc))] + [str(v) for v in sc]))
    lines.append("")
    for f in range(inst.nf):
        t = inst.table(f)
        lines.append(str(len(t)))
        lines.append(" ".join(repr(float(np.exp(-c))) for c in t))
        lines.append("")
    with open(path, "w") as fh:
        fh.write("\n".join(lines) + "\n")
