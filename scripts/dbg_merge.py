import sys, os, numpy as np
sys.path.insert(0, os.getcwd())
import gen, oracle
import paper_1608_05288_b200 as G
n, d, seed = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
inst = gen.scalefree(n, d, 0.0, seed)
P = G.Problem.from_instance(inst)
order, w = P.order()
plan = G.Plan(P, order, retain="all")
info = plan.info()
print("w*", w, "max rows", max(t["rows"] for t in info["tables"]), flush=True)
run, root = plan.dpop_util()
orun = oracle.solve_be(inst, order)
bad = 0
for t, (ti, ot) in enumerate(zip(info["tables"], orun.tables)):
    out, arg = run.table(t, ti["rows"])
    if not (np.array_equal(out, ot.out) and np.array_equal(arg, ot.arg)):
        bad += 1
        if bad < 4: print("table", t, "differs", ti["rows"], ti["kernel"].get("classes") if isinstance(ti.get("kernel"), dict) else None)
print("root", root, orun.value, "bad", bad)
