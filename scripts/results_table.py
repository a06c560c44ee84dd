"""BASELINE.md "Results" table from a bench_configs.py JSONL file."""
import json
import sys

rows = [json.loads(l) for l in open(sys.argv[1]) if l.startswith("{")]
print("| Config | GPUs | Cells | Kernel cells/s | HBM fraction | End-to-end solve | Oracle | Result |")
print("|---|---|---|---|---|---|---|---|")
for r in rows:
    name = r["config"]
    if "count" in r:
        name = f"{name} count {r['count']}"
    elif r.get("ibound", -1) >= 0:
        name = f"{name} i={r['ibound']}"
    elif name in ("C5",):
        name = "C5 exact"
    frac = f"{100 * r['hbm_frac']:.1f} %"
    if "big_buckets" in r:
        b = r["big_buckets"]
        frac += f" ({100 * b['hbm_frac']:.1f} % on {b['n']} buckets ≥1e8 cells)"
    orc = ""
    if "oracle_s_1t" in r:
        orc = f"{1e3 * r['oracle_s_1t']:.1f} ms (1 thread) / {1e3 * r[[k for k in r if k.startswith('oracle_s_') and not k.endswith('_1t')][0]]:.1f} ms (all cores)"
    elif "oracle_s_all_cores" in r:
        orc = f"{1e3 * r['oracle_s_all_cores']:.1f} ms (all cores)"
    if "n_solutions" in r:
        res = f"value {r['value']}, {r['n_solutions']:.6g} solutions (oracle {r['oracle_n_solutions']:.6g})"
    else:
        res = f"value {r['value']}" + (f", upper {r['upper']}" if r.get("upper") is not None else "")
    print(f"| {name} | 1 | {r['cells']:.3g} | {r['kernel_cells_per_s']:.3g} | {frac} | "
          f"{r['e2e_solve_ms_median']:.2f} ms | {orc} | {res} |")
