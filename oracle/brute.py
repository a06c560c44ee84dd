"""Pure-Python brute force for tiny instances (TEST INFRASTRUCTURE ONLY).

Enumerates the whole state space Sigma of Eq. (1) (MPE Eq. (2),
P:388-391, as min-sum over -log p) in lexicographic order of a given ordering
(order[0] most significant) and returns the optimum together with the
lexicographically smallest optimal assignment under that ordering.  No
elimination, no tables: the plain definition of the optimum.
"""
from __future__ import annotations

import itertools

INF_I32 = 1 << 30


def _cost(inst, assign):
    if inst.is_f64:
        s = 0.0
        for f in range(inst.nf):
            sc = inst.scope(f)
            idx = 0
            for v in sc:
                idx = idx * int(inst.dom[v]) + assign[int(v)]
            s = s + float(inst.costs[inst.table_off[f] + idx])
        return s
    s = 0
    for f in range(inst.nf):
        sc = inst.scope(f)
        idx = 0
        for v in sc:
            idx = idx * int(inst.dom[v]) + assign[int(v)]
        s = min(s + int(inst.costs[inst.table_off[f] + idx]), INF_I32)
    return s


def brute_force(inst, order=None, limit=2_000_000):
    """Returns (optimum, assignment).  Ties: the first optimum met in
    lexicographic order of `order` (default: identity)."""
    n = inst.n
    order = list(range(n)) if order is None else [int(v) for v in order]
    space = 1
    for v in order:
        space *= int(inst.dom[v])
    if space > limit:
        raise ValueError(f"state space {space} exceeds brute-force limit {limit}")
    best, best_a = None, None
    assign = [0] * n
    for vals in itertools.product(*[range(int(inst.dom[v])) for v in order]):
        for v, val in zip(order, vals):
            assign[v] = val
        c = _cost(inst, assign)
        if best is None or c < best:
            best, best_a = c, list(assign)
    if best is None:  # n == 0
        best, best_a = (0.0 if inst.is_f64 else 0), []
        best = _cost(inst, [])
    return best, best_a


def mpe_linear(inst, order=None, limit=2_000_000):
    """MPE in the linear domain: max over Sigma of prod_f exp(-cost) (Eq. 2),
    computed as a product of probabilities (not a log-sum)."""
    import math
    n = inst.n
    order = list(range(n)) if order is None else [int(v) for v in order]
    best = -1.0
    assign = [0] * n
    for vals in itertools.product(*[range(int(inst.dom[v])) for v in order]):
        for v, val in zip(order, vals):
            assign[v] = val
        p = 1.0
        for f in range(inst.nf):
            idx = 0
            for v in inst.scope(f):
                idx = idx * int(inst.dom[v]) + assign[int(v)]
            p *= math.exp(-float(inst.costs[inst.table_off[f] + idx]))
        if p > best:
            best = p
    return best


def brute_force_np(inst, order=None, limit=50_000_000):
    """Vectorised brute force (same definition as brute_force): enumerates
    every assignment in lexicographic order of `order`, sums every function
    (int: clamp at 2^30; f64: in function-index order), returns the first
    minimum."""
    import numpy as np
    n = inst.n
    order = list(range(n)) if order is None else [int(v) for v in order]
    dims = [int(inst.dom[v]) for v in order]
    space = int(np.prod(dims, dtype=np.int64)) if dims else 1
    if space > limit:
        raise ValueError(f"state space {space} exceeds limit {limit}")
    idx = np.arange(space, dtype=np.int64)
    vals = np.zeros((n, space), dtype=np.int64)
    rem = idx.copy()
    for pos in range(n - 1, -1, -1):
        vals[order[pos]] = rem % dims[pos]
        rem //= dims[pos]
    total = np.zeros(space, dtype=np.float64 if inst.is_f64 else np.int64)
    for f in range(inst.nf):
        sc = [int(v) for v in inst.scope(f)]
        k = np.zeros(space, dtype=np.int64)
        for v in sc:
            k = k * int(inst.dom[v]) + vals[v]
        t = inst.table(f)[k]
        if inst.is_f64:
            total = total + t
        else:
            total = np.minimum(total + t.astype(np.int64), INF_I32)
    best = int(np.argmin(total))  # first occurrence = lexicographically smallest
    return (float(total[best]) if inst.is_f64 else int(total[best])), [int(vals[v][best]) for v in range(n)]


def neg_log_z(inst, limit=2_000_000):
    """-log Z by enumeration, Z = sum over the whole state space of
    exp(-cost(assignment)) (the partition function; cost = Eq. (1) summed
    in f64).  Accumulated with math.fsum over exp(m - cost), m = min cost."""
    import math
    n = inst.n
    space = 1
    for v in range(n):
        space *= int(inst.dom[v])
    if space > limit:
        raise ValueError(f"state space {space} exceeds brute-force limit {limit}")
    costs = []
    assign = [0] * n
    for vals in itertools.product(*[range(int(inst.dom[v])) for v in range(n)]):
        assign[:] = vals
        costs.append(_cost(inst, assign))
    m = min(costs)
    if math.isinf(m):
        return math.inf
    return m - math.log(math.fsum(math.exp(m - c) for c in costs))


def count_solutions(inst, limit=50_000_000):
    """Counting by enumeration (P:245's "number of consistent solutions";
    SURVEY §8(f) row 4): returns (optimum, number of assignments whose cost
    equals the optimum, number of assignments of finite cost), the cost
    being Eq. (1) computed as in brute_force_np.  An infeasible problem has
    no optimal and no consistent assignment (counts 0, 0).  Exact Python
    integers."""
    import numpy as np
    n = inst.n
    dims = [int(inst.dom[v]) for v in range(n)]
    space = int(np.prod(dims, dtype=np.int64)) if dims else 1
    if space > limit:
        raise ValueError(f"state space {space} exceeds limit {limit}")
    idx = np.arange(space, dtype=np.int64)
    vals = np.zeros((n, space), dtype=np.int64)
    rem = idx.copy()
    for pos in range(n - 1, -1, -1):
        vals[pos] = rem % dims[pos]
        rem //= dims[pos]
    total = np.zeros(space, dtype=np.float64 if inst.is_f64 else np.int64)
    for f in range(inst.nf):
        k = np.zeros(space, dtype=np.int64)
        for v in (int(x) for x in inst.scope(f)):
            k = k * int(inst.dom[v]) + vals[v]
        t = inst.table(f)[k]
        total = total + t if inst.is_f64 else np.minimum(total + t.astype(np.int64), INF_I32)
    finite = np.isfinite(total) if inst.is_f64 else total < INF_I32
    opt = total.min()
    n_cons = int(finite.sum())
    n_opt = int((total == opt).sum()) if n_cons else 0
    return (float(opt) if inst.is_f64 else int(opt)), n_opt, n_cons
