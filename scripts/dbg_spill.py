"""Debug: spill plan, repeated solves vs the oracle (development tool)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import gen, oracle
import paper_1608_05288_b200 as G
inst = gen.scalefree(90, 3, 0.0, 4)
P = G.Problem.from_instance(inst)
order, _ = P.order()
orun = oracle.solve_be(inst, order)
peak = G.Plan(P, order, retain="all").info()["peak_bytes"]
for kernel in (-1, 0, 1, 2):
    plan = G.Plan(P, order, retain="all", spill=True, budget_bytes=peak // 2, stage_bytes=peak // 64, kernel=kernel)
    info = plan.info()
    res = []
    for rep in range(4):
        if rep % 2 == 0:
            run, root = plan.dpop_util()
            a = run.value()
            bad = []
            for t, (ti, ot) in enumerate(zip(info["tables"], orun.tables)):
                out, arg = run.table(t, ti["rows"])
                if not (np.array_equal(out, ot.out) and np.array_equal(arg, ot.arg)):
                    bad.append((t, ti["host"], int((out != ot.out).sum()), int((arg != ot.arg).sum())))
            run.close()
        else:
            root, a = plan.solve_be()
            bad = None
        res.append((root == orun.value, list(a) == list(orun.assignment), bad))
    print(kernel, orun.value, res, flush=True)
