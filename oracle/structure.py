"""Bucket structure of BE along an ordering, in plain Python (scopes only).

TEST / BASELINE INFRASTRUCTURE (see oracle/__init__.py): used by bench.py's
--impl reference arm to find the workload's largest bucket without loading
the product library.  Restates Alg. 1 lines 2-5 symbolically:
membership by the latest-ordered scope variable (reading A1), the
message scope = union of the member scopes minus x, ascending by order
position (A2), routed to the bucket of its latest variable.  Pinned against
the oracle's own tables (tests/test_oracle_pins.py).
"""
from __future__ import annotations

import numpy as np


def bucket_structure(inst, order):
    """[{var, sep, members: [(kind, index)], scopes: [member scope]}] in
    creation order (kind 0 = original function, 1 = earlier table)."""
    order = [int(v) for v in order]
    pos = {v: i for i, v in enumerate(order)}
    bucket = {v: [] for v in order}
    for f in range(inst.nf):
        sc = [int(v) for v in inst.scope(f)]
        if sc:
            bucket[max(sc, key=lambda v: pos[v])].append((0, f, sc))
    tables = []
    for x in reversed(order):
        mem = bucket[x]
        U = set()
        for _, _, sc in mem:
            U |= set(sc)
        U.discard(x)
        sep = sorted(U, key=lambda v: pos[v])
        tables.append({"var": x, "sep": sep, "members": [(k, i) for k, i, _ in mem],
                       "scopes": [sc for _, _, sc in mem],
                       "rows": int(np.prod([int(inst.dom[v]) for v in sep], dtype=np.int64)) if sep else 1,
                       "d": int(inst.dom[x])})
        if sep:
            bucket[sep[-1]].append((1, len(tables) - 1, sep))
    return tables
