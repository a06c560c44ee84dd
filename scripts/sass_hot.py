"""Print the SASS around the most-stalled instructions of an ncu source CSV
(ncu -i rep --page source --csv --print-source sass): address, stall
samples, executions, instruction (development tool)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
iA, iS, iW, iE = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
ins = [(r[iA], r[iS].strip(), int(r[iW] or 0), int(r[iE] or 0)) for r in rows[2:] if len(r) > iE]
tot = sum(x[2] for x in ins)
print("total samples", tot)
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 6
top = sorted(range(len(ins)), key=lambda i: -ins[i][2])[: int(sys.argv[2]) if len(sys.argv) > 2 else 5]
for i in sorted(top):
    print("----")
    for j in range(max(0, i - ctx), min(len(ins), i + 3)):
        a, s, w, e = ins[j]
        print(f"{'>>' if j == i else '  '} {j:5d} {a[-5:]} {w:7d} {e:10d}  {s}")
