"""One exact DPOP solve of a BASELINE workload (for ncu launch lists /
captures; the profiled steps follow --warm unprofiled solves: run ncu with
--profile-from-start off).  --which-fast prints the index, among tiled-kernel launches, of
the largest bucket (use it as ncu -k regex:bk_fast -s IDX -c 1)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1608_05288_b200 as G
from gen import configs

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c4")
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--which-fast", action="store_true")
ap.add_argument("--var", type=int, default=-1)
ap.add_argument("--warm", type=int, default=24)
ap.add_argument("--no-autotune", action="store_true")  # default variants (ncu -s indices then count from the start)
a = ap.parse_args()
inst = {"c4": configs.c4, "c2": configs.c2, "c5": configs.c5, "c5sp": configs.c5, "c4d4": configs.c4d4}[a.workload]()
sp = a.workload == "c5sp"
P = G.Problem.from_instance(inst)
order, w = P.order()
plan = G.Plan(P, order, timing=True, **({"semiring": "sumprod"} if sp else {}),
              **({"autotune": False} if a.no_autotune else {}))
import torch
for _ in range(a.warm):  # past the plan's autotuning solves (not profiled under --profile-from-start off)
    run, root = plan.dpop_util()
    if not sp:
        run.value()
    run.close()
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _ in range(a.steps):
    run, root = plan.dpop_util()
    if not sp:
        assign = run.value()
    st = run.stats()
    run.close()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
want = int(os.environ.get("PROF_VARIANT", "1"))  # 1 tiled (bk_fast), 2 streaming (bk_stream)
fast = [t for t in st["tasks"] if t["variant"] == want]
big = max(range(len(fast)), key=lambda i: fast[i]["cells"]) if a.var < 0 else [i for i, t in enumerate(fast) if t["var"] == a.var][0]
sel = fast[big]
if want == 2:  # input merges also launch bk_stream, just before their bucket (serial chain in timing mode)
    idx = 0
    for t in st["tasks"]:
        idx += t.get("merges", 0)
        if t is sel:
            break
        idx += 1 if t["variant"] == 2 else 0
    big = idx
if a.which_fast:
    print(big)
else:
    print(json.dumps({"root": root, "fast_launches": len(fast), "largest_fast_index": big,
                      "largest": sel}))
