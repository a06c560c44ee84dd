"""Per-bucket kernel times of one workload under the current environment
(knob sweeps: run once per setting; development tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1608_05288_b200 as G
from gen import configs

wl = sys.argv[1]
tag = sys.argv[2] if len(sys.argv) > 2 else ""
inst = {"c4": configs.c4, "c5": configs.c5, "c3": configs.c3, "c4d4": configs.c4d4}[wl]()
P = G.Problem.from_instance(inst)
order = configs.c3_order() if wl == "c3" else P.order()[0]
ib = int(os.environ.get("SWEEP_IB", "-1"))
plan = G.Plan(P, order, ib, resident_inputs=True, timing=True)
best = None
for i in range(20):
    run, root = plan.dpop_util(); run.value(); st = run.stats(); run.close()
    if i >= 16:
        ks = sum(t["ms"] for t in st["tasks"])
        if best is None or ks < best[0]:
            best = (ks, st["tasks"])
ks, tasks = best
top = sorted(tasks, key=lambda t: -t["ms"])[:10]
print(f"{wl} [{tag}] sum {ks:.2f} ms | " + " ".join(
    f"x{t['var']}={t['ms']:.3f}{('S' if t.get('staged') else 's') if t['variant'] == 2 else ''}{'/' + str(t.get('tile_rows')) if t.get('tile_rows') else ''}{'D' + str(t['stages']) if t.get('direct_stores') else ''}" for t in top), flush=True)
