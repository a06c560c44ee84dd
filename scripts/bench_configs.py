"""Measure every BASELINE config on one GPU (fills BASELINE.md "Results").

For each config: kernel cells/s and HBM fraction over all bucket launches and
over the buckets with >= 1e8 cells (CUDA events per launch), end-to-end solve
time through the C ABI (median of 5 after 1 warm-up, inputs from pinned host
memory, optimum + assignment back), and the CPU oracle's time on the same
instance where it finishes quickly (C1, C2: 1 thread and all cores).
Prints one JSON line per (config, i-bound).
"""
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1608_05288_b200 as G  # noqa: E402
from gen import configs  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0


def measure(name, inst, order, ib, exact_value_only=False, oracle_threads=(), **extra):
    P = G.Problem.from_instance(inst)
    opts = dict(retain="none") if exact_value_only else {}
    opts.update(extra)
    plan_t = G.Plan(P, order, ib, timing=True, **opts)
    mbe = ib >= 0

    def solve(pl, stats=False):
        if mbe:
            return pl.solve_mbe(stats=stats, assignment=not exact_value_only)
        return pl.solve_be(stats=stats, assignment=not exact_value_only)

    for _ in range(18):  # warm-up: lazy module loading, the autotuning solves
        solve(plan_t)
    r = solve(plan_t, stats=True)
    st = r[-1]
    tasks = st["tasks"]
    ms = sum(t["ms"] for t in tasks)
    by = sum(t["bytes"] for t in tasks)
    big = [t for t in tasks if t["cells"] >= 1e8]
    del plan_t
    plan = G.Plan(P, order, ib, **opts)
    for _ in range(18):  # autotuning solves, graph capture
        solve(plan)
    walls = []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = solve(plan)
        walls.append((time.perf_counter() - t0) * 1e3)
    del plan
    rec = {"config": name, "ibound": ib, "cells": st["total_cells"], "launches": len(tasks),
           "kernel_ms": ms, "kernel_cells_per_s": st["total_cells"] / (ms * 1e-3),
           "hbm_frac": by / (ms * 1e-3) / 1e9 / PEAK, "e2e_solve_ms_median": statistics.median(walls),
           "value": res[0], "upper": res[1] if mbe else None}
    if big:
        bms = sum(t["ms"] for t in big)
        rec["big_buckets"] = {"n": len(big), "cells_per_s": sum(t["cells"] for t in big) / (bms * 1e-3),
                              "hbm_frac": sum(t["bytes"] for t in big) / (bms * 1e-3) / 1e9 / PEAK}
    for th in oracle_threads:
        t0 = time.perf_counter()
        orun = oracle.Run(inst, order, ib, keep_tables=True, nthreads=th)
        rec[f"oracle_s_{th}t"] = time.perf_counter() - t0
        rec["oracle_value"] = orun.value
    print(json.dumps(rec), flush=True)
    return rec


def measure_count(name, inst, order, mode):
    """Solution counting: kernel cells/s and HBM fraction
    of the counting bucket kernel (algorithmic bytes include the float64
    count tables), one-shot solve time, oracle time at all cores."""
    P = G.Problem.from_instance(inst)
    plan_t = G.Plan(P, order, count=mode, timing=True)
    for _ in range(2):
        run, root = plan_t.dpop_util()
        st = run.stats()
        cnt = run.count()
        run.close()
    tasks = st["tasks"]
    ms = sum(t["ms"] for t in tasks)
    by = sum(t["bytes"] for t in tasks)
    del plan_t
    plan = G.Plan(P, order, count=mode)
    plan.solve_count()
    walls = []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        v, c = plan.solve_count()
        walls.append((time.perf_counter() - t0) * 1e3)
    t0 = time.perf_counter()
    orun = oracle.solve_count(inst, order, mode, keep_tables=False)
    rec = {"config": name, "count": mode, "cells": st["total_cells"], "kernel_ms": ms,
           "kernel_cells_per_s": st["total_cells"] / (ms * 1e-3), "hbm_frac": by / (ms * 1e-3) / 1e9 / PEAK,
           "e2e_solve_ms_median": statistics.median(walls), "value": v, "n_solutions": c,
           "oracle_n_solutions": orun.count, "oracle_s_all_cores": time.perf_counter() - t0}
    print(json.dumps(rec), flush=True)
    return rec


def main(which):
    cores = os.cpu_count()
    if "c1" in which:
        inst = configs.c1(0)
        measure("C1", inst, oracle.minfill_order(inst), -1, oracle_threads=(1, cores))
    if "c2" in which:
        inst = configs.c2()
        measure("C2", inst, oracle.minfill_order(inst), -1, oracle_threads=(1, cores))
    if "count" in which:  # solution counting on C2 and C4
        inst = configs.c2()
        for mode in ("optimal", "consistent"):
            measure_count("C2", inst, oracle.minfill_order(inst), mode)
    if "c4count" in which:
        inst = configs.c4()
        measure_count("C4", inst, oracle.minfill_order(inst), "optimal")
    if "c4host" in which:  # argmin spill: argmins streamed to pinned host memory
        inst = configs.c4()
        measure("C4-hostargs", inst, oracle.minfill_order(inst), -1, retain="host")
    if "c4spill" in which:  # out-of-core plan, messages streamed under a 12 GB budget
        inst = configs.c4()
        measure("C4-spill-12GB", inst, oracle.minfill_order(inst), -1, spill=True, budget_bytes=12 * 10**9)
    if "c3" in which:
        inst = configs.c3()
        order = configs.c3_order()
        for ib in configs.C3_IBOUNDS:
            measure("C3", inst, order, ib, exact_value_only=(ib == 18))
        measure("C3-exact", inst, order, -1, exact_value_only=True)
    if "c4" in which:
        inst = configs.c4()
        measure("C4", inst, oracle.minfill_order(inst), -1)
    if "c4d4" in which:  # SURVEY's alternative C4: n=150, d=4, w*=16
        inst = configs.c4d4()
        measure("C4-d4", inst, oracle.minfill_order(inst), -1)
    if "c5" in which:
        inst = configs.c5()
        order = oracle.minfill_order(inst)
        measure("C5", inst, order, -1)
        measure("C5", inst, order, configs.C5_IBOUND)
    if "c5sp" in which:  # the same network, sum-product (-log Z)
        inst = configs.c5()
        measure("C5-sumprod", inst, oracle.minfill_order(inst), -1, exact_value_only=True,
                semiring="sumprod")


if __name__ == "__main__":
    main(sys.argv[1:] or ["c1", "c2", "c3", "c4", "c4d4", "c5"])
