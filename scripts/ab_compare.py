"""Compare per-bucket times of two A/B JSON task dumps (development tool)."""
import json, sys
a = json.load(open(sys.argv[1])); b = json.load(open(sys.argv[2]))
n = int(sys.argv[3]) if len(sys.argv) > 3 else 15
ta = sum(t["ms"] for t in a); tb = sum(t["ms"] for t in b)
best = sum(min(x["ms"], y["ms"]) for x, y in zip(a, b))
by = sum(x["bytes"] for x in a)
print(f"A {ta:.3f} ms ({by/ta/1e6/6457.1:.3f})  B {tb:.3f} ms ({by/tb/1e6/6457.1:.3f})  best-of {best:.3f} ms ({by/best/1e6/6457.1:.3f})")
big = [(x, y) for x, y in zip(a, b) if x["cells"] >= 1e8]
if big:
    ba = sum(x["ms"] for x, _ in big); bb = sum(y["ms"] for _, y in big); bbest = sum(min(x["ms"], y["ms"]) for x, y in big)
    byb = sum(x["bytes"] for x, _ in big)
    print(f">=1e8 cells ({len(big)}): A {byb/ba/1e6/6457.1:.3f} B {byb/bb/1e6/6457.1:.3f} best {byb/bbest/1e6/6457.1:.3f}")
for x, y in sorted(zip(a, b), key=lambda p: -max(p[0]["ms"], p[1]["ms"]))[:n]:
    print(f"  x{x['var']:<4} k={x['k']} keff={x['k_eff']} d={x['d']} rows={x['rows']:.2e} A {x['ms']:.3f} ({x['bytes']/x['ms']/1e6:.0f} GB/s) B {y['ms']:.3f} ({y['bytes']/y['ms']/1e6:.0f} GB/s) PL={x.get('tile_rows')} st={x.get('stages')}")
