"""Group the SASS of an ncu source-page CSV by execution count (hot regions)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; data = rows[2:]
iE = hdr.index("Instructions Executed"); iS = hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[iE] or 0) for r in data); tots = sum(int(r[iS] or 0) for r in data)
groups = []
for i, r in enumerate(data):
    e = int(r[iE] or 0); st = int(r[iS] or 0)
    if groups and groups[-1][2] == e: groups[-1][1] = i; groups[-1][3] += e; groups[-1][4] += st
    else: groups.append([i, i, e, e, st])
print("total warp inst", tot, "samples", tots)
for g in sorted(groups, key=lambda g: -g[3])[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"lines {g[0]}-{g[1]} n={g[1]-g[0]+1} exec={g[2]} total={100*g[3]/tot:.1f}% stall={100*g[4]/tots:.1f}%")
if len(sys.argv) > 4:
    for i in range(int(sys.argv[3]), int(sys.argv[4])):
        print(i, data[i][1].strip()[:80], data[i][iE], data[i][iS])
