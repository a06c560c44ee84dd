"""Summarise an ncu report (details + instruction mix + top stalls)."""
import csv, io, subprocess, sys
from collections import Counter
rep = sys.argv[1]
def run(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout
det = list(csv.reader(io.StringIO(run("--page", "details", "--csv"))))
keep = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread",
        "Dynamic Shared Memory Per Block", "Grid Size", "Block Size", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction", "Executed Instructions",
        "Avg. Active Threads Per Warp", "Block Limit Registers", "Block Limit Shared Mem"]
h0 = det[0]
iN, iU, iV = h0.index("Metric Name"), h0.index("Metric Unit"), h0.index("Metric Value")
seen = set()
for row in det[1:]:
    if len(row) > iV and row[iN] in keep and row[iN] not in seen:
        seen.add(row[iN])
        print(f"{row[iN]:40s} {row[iV]} {row[iU]}")
raw = list(csv.reader(io.StringIO(run("--page", "raw", "--csv"))))
hdr, vals = raw[0], raw[2]
for h, v in zip(hdr, vals):
    if h in ("dram__bytes_read.sum", "dram__bytes_write.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
             "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "smsp__sass_inst_executed_op_shared_ld.sum",
             "smsp__sass_inst_executed_op_global_st.sum") or h.endswith("pct_of_peak_sustained_elapsed") and (
                 h.startswith("l1tex__") or h.startswith("lts__") or h.startswith("dram__") or h.startswith("gpu__compute_memory")) or h in (
             "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
             "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_st.sum",
             "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts.sum",
             "l1tex__data_pipe_lsu_wavefronts_mem_lg.sum", "lts__t_sectors_op_read.sum", "lts__t_sectors_op_write.sum") or (h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued")):
        if v not in ("0", ""):
            print(f"{h:70s} {v} {raw[1][hdr.index(h)]}")
src = list(csv.reader(io.StringIO(run("--page", "source", "--csv", "--print-source", "sass"))))
h = src[1]; data = src[2:]
iS, iW, iE = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
te = sum(int(r[iE] or 0) for r in data); tw = sum(int(r[iW] or 0) for r in data)
ce, cw = Counter(), Counter()
for r in data:
    toks = r[iS].strip().split()
    if not toks: continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    op = op.split(".")[0]
    ce[op] += int(r[iE] or 0); cw[op] += int(r[iW] or 0)
print("instructions executed:", te)
for op, c in ce.most_common(18):
    print(f"  {op:10s} exec {c / te * 100:5.1f}%  stall-samples {cw[op] / max(tw,1) * 100:5.1f}%")
print("top stalled instructions:")
for r in sorted(data, key=lambda r: -int(r[iW] or 0))[:12]:
    print("  ", r[iW], r[iE], r[iS].strip()[:80])
