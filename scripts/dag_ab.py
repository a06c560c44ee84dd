"""A/B of the UTIL-phase graph: task DAG (concurrent subtrees) vs the serial
chain.  Median wall time of a value-only solve (graph replay, resident inputs)
per config.  python scripts/dag_ab.py [c2 c4 c5 c3]"""
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402  (orderings only)
import paper_1608_05288_b200 as G  # noqa: E402
from gen import configs  # noqa: E402


def ab(name, inst, order, ib=-1, reps=15):
    P = G.Problem.from_instance(inst)
    res = {}
    for conc in (False, True, False, True):
        plan = G.Plan(P, order, ib, retain="none", resident_inputs=True, concurrent=conc)
        f = (lambda: plan.solve_mbe(assignment=False)) if ib >= 0 else (lambda: plan.solve_be(assignment=False))
        for _ in range(3):
            v = f()
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            f()
            ts.append((time.perf_counter() - t0) * 1e3)
        res.setdefault(conc, []).append(statistics.median(ts))
        del plan
    print(f"{name:10s} i={ib:3d} serial {min(res[False]):8.3f} ms  dag {min(res[True]):8.3f} ms  "
          f"value {v[0]}", flush=True)


which = sys.argv[1:] or ["c2", "c4", "c5", "c3"]
if "c2" in which:
    inst = configs.c2()
    ab("C2", inst, oracle.minfill_order(inst))
if "c4" in which:
    inst = configs.c4()
    ab("C4", inst, oracle.minfill_order(inst))
if "c5" in which:
    inst = configs.c5()
    o = oracle.minfill_order(inst)
    ab("C5", inst, o)
    ab("C5", inst, o, configs.C5_IBOUND)
if "c3" in which:
    inst = configs.c3()
    for ib in (8, 12, 16):
        ab("C3", inst, configs.c3_order(), ib, reps=5)
