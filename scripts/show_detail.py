"""Print the post-merge structure of the largest buckets from a DETAIL_JSON
dump of scripts/bench_detail.py (development tool)."""
import json, sys
tasks = json.load(open(sys.argv[1]))
for t in sorted(tasks, key=lambda t: -t["ms"])[: int(sys.argv[2]) if len(sys.argv) > 2 else 8]:
    print(f"x{t['var']} rows {t['rows']:.3g} ms {t['ms']:.3f} k_eff {t['k_eff']} tile {t.get('tile_rows')} "
          f"st {t.get('stages')} g {t.get('g')} classes {t.get('classes')}")
    for q, s in enumerate(t.get("in_scope", [])):
        sl = t.get("slen", [None] * 64)[q]
        print(f"     {s}  slice {sl}")
