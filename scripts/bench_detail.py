"""Per-bucket timing breakdown of one workload (development tool)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1608_05288_b200 as G
from gen import configs

wl = sys.argv[1] if len(sys.argv) > 1 else "c4"
ib = int(sys.argv[2]) if len(sys.argv) > 2 else -1
inst = {"c4": configs.c4, "c2": configs.c2, "c5": configs.c5, "c3": configs.c3,
        "c4alt": lambda: configs.c4(seed=configs.C4_ALT_SEED), "c4d4": configs.c4d4}[wl]()
P = G.Problem.from_instance(inst)
order = configs.c3_order() if wl == "c3" else P.order()[0]
info = G.Plan(P, order, ib).info()
for label, opts in [("resident", dict(resident_inputs=True, timing=True)), ("e2e", dict(timing=True)),
                    ("e2e-notiming", dict())]:
    plan = G.Plan(P, order, ib, **opts)
    for _ in range(20):  # past the autotuning solves and the graph capture
        run, root = plan.dpop_util(); run.value(); run.close()
    s = torch.cuda.current_stream()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    run, root = plan.dpop_util(s)
    t1 = time.perf_counter()
    a = run.value()
    t2 = time.perf_counter()
    st = run.stats() if opts.get("timing") else None
    run.close()
    e1.record(s)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"[{label}] events {e0.elapsed_time(e1):.2f} ms; util wall {1e3*(t1-t0):.2f} value wall {1e3*(t2-t1):.2f} close {1e3*(t3-t2):.2f}")
    if st and os.environ.get("DETAIL_JSON") and label == "resident":
        json.dump(st["tasks"], open(os.environ["DETAIL_JSON"], "w"))
    if st:
        tasks = st["tasks"]
        ksum = sum(t["ms"] for t in tasks)
        print(f"   kernel sum {ksum:.2f} ms over {len(tasks)} launches; cells {st['total_cells']:.3e}")
        for t in sorted(tasks, key=lambda t: -t["ms"])[:12]:
            ti = info["tables"][[i for i, x in enumerate(info["tables"]) if x["var"] == t["var"] and x["mb"] == t["mb"]][0]]
            print(f"   x{t['var']:<4d} k={t['k']:<3d} rows={t['rows']:.3e} ms={t['ms']:.3f} "
                  f"cells/s={t['cells']/t['ms']*1e3:.3e} GB/s={t['bytes']/t['ms']/1e6:.0f} var={t['variant']} in/C={ti['in_cells']/(t['cells']):.3f}"
                  f" merge_ms={t.get('merge_ms', 0):.3f} k_eff={t.get('k_eff')} PL={t.get('tile_rows')} st={t.get('stages')} nob={t.get('staging_bufs')} cls={t.get('classes')}")
