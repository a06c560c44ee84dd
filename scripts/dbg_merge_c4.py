import sys, os
sys.path.insert(0, os.getcwd())
import paper_1608_05288_b200 as G
from gen import configs
inst = configs.c4()
P = G.Problem.from_instance(inst)
order, w = P.order()
plan = G.Plan(P, order, timing=len(sys.argv) > 1)
run, root = plan.dpop_util()
print("root", root, flush=True)
a = run.value()
print("ok", flush=True)
