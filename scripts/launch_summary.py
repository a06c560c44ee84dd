"""Summarise an ncu launch list (gpu__time_duration per launch) by kernel."""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]; iK, iN, iV = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
tot = defaultdict(float); cnt = defaultdict(int)
for r in rows[hdr + 1:]:
    if len(r) > iV and r[iN] == "gpu__time_duration.sum":
        k = r[iK].split("(")[0].replace("void ", "")
        k = k.split("<")[0] + ("<" + r[iK].split("<")[1].split(">")[0] + ">" if "<" in r[iK] else "")
        tot[k] += float(r[iV].replace(",", "")); cnt[k] += 1
s = sum(tot.values())
print(f"{'kernel':60s} {'launches':>8s} {'total ms':>10s} {'share':>7s}")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{k[:60]:60s} {cnt[k]:8d} {v/1e6:10.3f} {v/s*100:6.1f}%")
print(f"{'TOTAL':60s} {sum(cnt.values()):8d} {s/1e6:10.3f}")
