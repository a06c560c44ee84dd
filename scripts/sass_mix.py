"""Opcode mix of the instructions executed exactly N times (a loop body) in
an ncu source CSV (development tool).  usage: sass_mix.py CSV [N]"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
iS, iE, iW = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
ins = [(r[iS].strip(), int(r[iE] or 0), int(r[iW] or 0)) for r in rows[2:] if len(r) > iE]
cnt = collections.Counter(e for _, e, _ in ins if e)
print("most common exec counts:", cnt.most_common(8))
N = int(sys.argv[2]) if len(sys.argv) > 2 else cnt.most_common(1)[0][0]
body = [(s, w) for s, e, w in ins if e == N]
ops = collections.Counter()
for s, w in body:
    t = s.split()
    op = t[1] if t[0].startswith("@") else t[0]
    ops[op.split(".")[0]] += 1
print(f"N={N}: {len(body)} instructions, {sum(w for _, w in body)} stall samples")
for op, c in ops.most_common():
    print(f"  {op:10s} {c}")
