"""Large-domain buckets (the paper's Table 1 domains d = 10, 25, 50, 100,
P:929, plus 6 and 256) through the streaming kernel: cells/s and
the HBM fraction of each launch (CUDA events, warm-up, median of 10).

Bucket shape (a random-graph DCOP bucket): one message over every output
digit (the dominant read) and two binary constraints (x, y_q), int32 and
float64; d^m rows for the largest m with d^(m+1) <= 4.3e9 cells.
Algorithmic bytes = b * sum_j |T_j| + b * R + R.  One JSON line per (d, dtype).
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1608_05288_b200 as G  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]


def bucket(d, f64, seed):
    m = 1
    while d ** (m + 2) <= 4_300_000_000:
        m += 1
    rows = d ** m
    D = G.BucketDesc()
    D.semiring = G.MINSUM_F64 if f64 else G.MINSUM_I32
    D.nsep, D.d, D.ninputs, D.rows = m, d, 3, rows
    for q in range(m):
        D.radix[q] = d
    st = d
    for q in range(m - 1, -1, -1):  # input 0: the message over every digit (+ x)
        D.stride[0][q] = st
        st *= d
    D.stride[1][0] = d               # input 1: constraint (y_0, x)
    D.stride[2][m - 1] = d           # input 2: constraint (y_{m-1}, x)
    g = torch.Generator(device="cuda").manual_seed(seed)
    dt = torch.float64 if f64 else torch.int32
    mk = (lambda n: torch.rand(n, generator=g, device="cuda", dtype=dt) * 100) if f64 else \
        (lambda n: torch.randint(0, 100, (n,), generator=g, device="cuda", dtype=dt))
    ins = [mk(rows * d), mk(d * d), mk(d * d)]
    return D, rows, ins


def main():
    for d in (6, 10, 25, 50, 100, 256):
        for f64 in (False, True):
            D, rows, ins = bucket(d, f64, d)
            dt = torch.float64 if f64 else torch.int32
            out = torch.empty(rows, dtype=dt, device="cuda")
            arg = torch.empty(rows, dtype=torch.uint8, device="cuda")
            assert G.bucket_kernel_variant(D, 0, rows) == 2
            ms = []
            for it in range(13):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                G.bucket_kernel(D, ins, out, arg, 0, rows)
                e1.record()
                torch.cuda.synchronize()
                if it >= 3:
                    ms.append(e0.elapsed_time(e1))
            t = statistics.median(ms)
            b = 8 if f64 else 4
            by = b * sum(x.numel() for x in ins) + b * rows + rows
            cells = rows * d
            print(json.dumps({"d": d, "dtype": "f64" if f64 else "int32", "rows": rows, "cells": cells,
                              "ms": t, "cells_per_s": cells / (t * 1e-3), "gbs": by / (t * 1e-3) / 1e9,
                              "hbm_frac": by / (t * 1e-3) / 1e9 / PEAK, "bytes_per_cell": by / cells}), flush=True)
            del ins, out, arg


if __name__ == "__main__":
    main()
