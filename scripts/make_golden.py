"""Write tests/golden/*.json from the CPU oracle at the BASELINE full sizes.

Calls only oracle/ and gen/ (the oracle is test infrastructure; this script
is how its stored values are produced, so no expected value ever comes from
the CUDA path).  Per table: the FNV-1a digest of (out, argmin) for int32
configs; for the f64 config (C5) the f64 sum / min / max of the finite
entries and the count of infinite ones (the tiled kernel's f64 summation order
differs from the oracle's canonical order, so digests would not be stable).

  python scripts/make_golden.py [c2] [c4] [c4d4] [c3] [c5] [c3i18]

c3i18 (MBE i = 18 on the 20x20 grid, 3.8e11 cells, value-only) records
digests of kind 1 (oracle.mix_digest) instead of FNV-1a.
"""
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
from gen import configs  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def run(inst, order, ib, keep):
    t0 = time.time()
    r = oracle.Run(inst, order, ib, keep_tables=keep, nthreads=0)
    return r, time.time() - t0


def int_record(name, inst, order, ib, keep):
    r, dt = run(inst, order, ib, keep)
    assert r.status == 0
    rec = {"config": name, "ibound": ib, "order": [int(v) for v in order], "value": r.value,
           "upper": r.upper if keep else None,
           "assignment": [int(v) for v in r.assignment] if r.assignment is not None else None,
           "tables": [{"var": t.var, "mb": t.mb, "rows": t.rows, "digest": f"{t.digest:016x}"} for t in r.tables],
           "oracle_seconds": dt}
    print(f"{name} i={ib}: value {r.value} upper {rec['upper']} tables {len(r.tables)} in {dt:.1f}s", flush=True)
    return rec


def mix_record(name, inst, order, ib, nthreads):
    """Value-only oracle run (messages freed once consumed, no forward pass)
    recording per-table digests of kind 1 (oracle.mix_digest: a parallel
    position-keyed sum, which a GPU test can form on the device)."""
    oracle.set_digest_kind(1)
    t0 = time.time()
    r = oracle.Run(inst, order, ib, keep_tables=False, nthreads=nthreads)
    dt = time.time() - t0
    oracle.set_digest_kind(0)
    assert r.status == 0
    rec = {"config": name, "ibound": ib, "order": [int(v) for v in order], "value": r.value,
           "digest_kind": "mix",
           "tables": [{"var": t.var, "mb": t.mb, "rows": t.rows, "digest": f"{t.digest:016x}"} for t in r.tables],
           "oracle_seconds": dt, "oracle_threads": nthreads}
    print(f"{name} i={ib}: value {r.value} tables {len(r.tables)} in {dt:.1f}s", flush=True)
    return rec


def f64_record(name, inst, order, ib):
    stats = {}

    def keep(t, T, out, arg):
        fin = np.isfinite(out)
        stats[t] = {"n_inf": int((~fin).sum()),
                    "sum": float(np.sum(out[fin], dtype=np.float64)) if fin.any() else 0.0,
                    "min": float(out[fin].min()) if fin.any() else None,
                    "max": float(out[fin].max()) if fin.any() else None}

    t0 = time.time()
    r = oracle.Run(inst, order, ib, keep_tables=True, nthreads=0, table_fn=keep)
    dt = time.time() - t0
    assert r.status == 0
    tabs = [dict(var=t.var, mb=t.mb, rows=t.rows, **stats[i]) for i, t in enumerate(r.tables)]
    rec = {"config": name, "ibound": ib, "order": [int(v) for v in order], "value": r.value,
           "upper": r.upper, "assignment": [int(v) for v in r.assignment], "tables": tabs,
           "oracle_seconds": dt}
    print(f"{name} i={ib}: value {r.value} upper {r.upper} tables {len(tabs)} in {dt:.1f}s", flush=True)
    return rec


def main(which):
    os.makedirs(OUT, exist_ok=True)
    if "c2" in which:
        inst = configs.c2()
        order = oracle.minfill_order(inst)
        json.dump(int_record("C2", inst, order, -1, True), open(os.path.join(OUT, "c2.json"), "w"))
    if "c4" in which:
        inst = configs.c4()
        order = oracle.minfill_order(inst)
        json.dump(int_record("C4", inst, order, -1, False), open(os.path.join(OUT, "c4.json"), "w"))
    if "c4d4" in which:  # SURVEY's alternative C4 (n=150, d=4, w*=16): 3.4e10 cells
        inst = configs.c4d4()
        order = oracle.minfill_order(inst)
        json.dump(int_record("C4-d4", inst, order, -1, False), open(os.path.join(OUT, "c4d4.json"), "w"))
    if "c3" in which:
        inst = configs.c3()
        order = configs.c3_order()
        recs = []
        for ib in (8, 10, 12, 14):
            recs.append(int_record("C3", inst, order, ib, True))
        recs.append(int_record("C3", inst, order, 16, False))
        json.dump(recs, open(os.path.join(OUT, "c3.json"), "w"))
    if "c3i18" in which:  # ~3.8e11 cells: hours of oracle time
        inst = configs.c3()
        order = configs.c3_order()
        nthreads = int(os.environ.get("ORACLE_THREADS", "0"))
        json.dump(mix_record("C3", inst, order, 18, nthreads), open(os.path.join(OUT, "c3_i18.json"), "w"))
    if "c5" in which:
        inst = configs.c5()
        order = oracle.minfill_order(inst)
        recs = [f64_record("C5", inst, order, configs.C5_IBOUND), f64_record("C5", inst, order, -1)]
        json.dump(recs, open(os.path.join(OUT, "c5.json"), "w"))


if __name__ == "__main__":
    main(sys.argv[1:] or ["c2", "c4", "c3", "c5"])
