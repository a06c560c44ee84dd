"""Pin generator seeds for the BASELINE configs by min-fill induced width.

Calls only gen/ and the oracle's min-fill/induced width (the oracle is test
infrastructure; this script is a development tool, not product code).
Output: seed -> w* tables; the chosen seeds are constants in gen/configs.py.
"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen, oracle

def widths(make, seeds):
    out = []
    for s in seeds:
        i = make(s)
        out.append((s, oracle.induced_width(i, oracle.minfill_order(i))))
    return out

if __name__ == "__main__":
    print("C2 random tree+45 (n=100,d=5):", widths(lambda s: gen.random_graph(100, 5, 144, 1, 0.0, s), range(10)))
    print("C4 BA (n=200,d=3):", widths(lambda s: gen.scalefree(200, 3, 0.0, s), range(12)))
    print("C5 BN (n=150):", widths(lambda s: gen.belief_net(150, 2, 4, 3, 20, s), range(6)))
