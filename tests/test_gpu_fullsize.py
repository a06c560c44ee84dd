"""Element-wise / digest parity at the BASELINE full sizes (-m gpu).

Every bucket of the run is inspected through the table hook
(gbe_set_table_hook): the executor calls back after each (mini-)bucket,
before its message can be freed, with device pointers to the bucket's output
rows and argmins.

* C3 MBE(18) (grid 20x20, 419 tables, 3.8e11 cells): every table's checksum
  (oracle.mix_digest: out and argmin) formed on the device equals the one the
  oracle recorded in tests/golden/c3_i18.json (scripts/make_golden.py c3i18,
  which calls only oracle/ and gen/); the lower bound equals the oracle's.
* C3 exact (400 tables, 3.8e12 cells; the oracle would need ~1 day): every
  bucket is checked on sampled BLOCKS of rows -- the leading output digits
  fixed, all values of the trailing ones (up to 2^21 rows, whole tiles and the
  ragged end) -- against oracle.bucket_eval run on the same block of the
  bucket's own inputs (originals from the instance, messages read back from
  the device slice by slice).  Composed over the whole elimination this
  checks every step of the path; the value lies inside every MBE bracket.
* C5 (BN MPE, f64, exact and MBE(16)): every table element-wise against an
  in-test oracle run: values within 1e-9 relative, the same infinite cells,
  argmins equal except where the oracle's own sums of the two choices are a
  near-tie (reading A10, oracle.bucket_row_sums).
"""
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle
import paper_1608_05288_b200 as G
from gen import configs
from tests import devtools

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


class Hook:
    """Installs fn as the table hook for the duration of a with-block."""

    def __init__(self, fn):
        self.fn = fn

    def __enter__(self):
        G.set_table_hook(self.fn)
        return self

    def __exit__(self, et, ev, tb):
        G.set_table_hook(None)
        err = G.table_hook_error()
        if et is not None and issubclass(et, G.GbeError) and err is not None:
            raise err  # the assertion that failed inside the hook


def _member_scope_table(inst, info, m):
    kind, idx = m
    if kind == 0:
        return [int(v) for v in inst.scope(idx)], inst.table(idx)
    return info["tables"][idx]["sep"], None


def test_c3_mbe18_table_digests():
    p = os.path.join(GOLD, "c3_i18.json")
    if not os.path.exists(p):
        pytest.skip("tests/golden/c3_i18.json not generated (python scripts/make_golden.py c3i18)")
    g = json.load(open(p))
    inst = configs.c3()
    order = configs.c3_order()
    assert list(order) == g["order"]
    P = G.Problem.from_instance(inst)
    plan = G.Plan(P, order, 18, retain="none")
    info = plan.info()
    assert [(t["var"], t["mb"], t["rows"]) for t in info["tables"]] == \
        [(t["var"], t["mb"], t["rows"]) for t in g["tables"]]
    got = {}

    def fn(t, o, a, rb, n, st):
        assert rb == 0 and n == info["tables"][t]["rows"]
        got[t] = devtools.mix_digest(devtools.dev_view(o, n, torch.int32), devtools.dev_view(a, n, torch.uint8))
        torch.cuda.synchronize()
        return 0

    with Hook(fn):
        lo, _, _ = plan.solve_mbe(assignment=False)
    assert lo == g["value"]
    assert len(got) == len(g["tables"])
    bad = [t for t in range(len(got)) if f"{got[t]:016x}" != g["tables"][t]["digest"]]
    assert not bad, f"{len(bad)} of {len(got)} tables differ, first {bad[:5]}"


def _blocks(radix, max_rows, rng, nrand):
    """Leading digits to fix (h) and a list of blocks (values of those digits):
    nrand random ones and the last one (the ragged end of the table)."""
    h = 0
    while h < len(radix) and int(np.prod(radix[h:], dtype=np.int64)) > max_rows:
        h += 1
    if h == 0:
        return 0, [()]
    out = [tuple(int(r) - 1 for r in radix[:h])]
    for _ in range(nrand):
        out.append(tuple(int(rng.integers(0, r)) for r in radix[:h]))
    return h, out


def test_c3_exact_block_sampled_every_bucket():
    inst = configs.c3()
    order = configs.c3_order()
    dom = [int(v) for v in inst.dom]
    P = G.Problem.from_instance(inst)
    plan = G.Plan(P, order, retain="none")
    info = plan.info()
    T = info["tables"]
    rng = np.random.default_rng(20)
    ptr = {}
    checked = {"buckets": 0, "rows": 0}

    def fn(t, o, a, rb, n, st):
        tb = T[t]
        assert rb == 0 and n == tb["rows"]
        ptr[t] = o
        sep, x = tb["sep"], tb["var"]
        radix = [dom[v] for v in sep]
        h, blocks = _blocks(radix, 1 << 21, rng, 1)
        out_v = devtools.dev_view(o, n, torch.int32).view(*radix) if sep else devtools.dev_view(o, 1, torch.int32)
        arg_v = devtools.dev_view(a, n, torch.uint8).view(*radix) if sep else devtools.dev_view(a, 1, torch.uint8)
        for blk in blocks:
            fixed = dict(zip(sep[:h], blk))
            mem = []
            for m in tb["members"]:
                sc, tab = _member_scope_table(inst, info, m)
                shape = [dom[v] for v in sc]
                idx = tuple(fixed[v] if v in fixed else slice(None) for v in sc)
                if tab is not None:
                    sl = np.ascontiguousarray(np.asarray(tab).reshape(shape)[idx])
                else:
                    src = devtools.dev_view(ptr[m[1]], int(np.prod(shape, dtype=np.int64)), torch.int32)
                    sl = src.view(*shape)[idx].contiguous().cpu().numpy()
                mem.append(([v for v in sc if v not in fixed], sl.reshape(-1)))
            eo, ea = oracle.bucket_eval(dom, False, x, mem, sep[h:])
            go = out_v[blk].reshape(-1).cpu().numpy() if sep else out_v.cpu().numpy()
            ga = arg_v[blk].reshape(-1).cpu().numpy() if sep else arg_v.cpu().numpy()
            assert np.array_equal(go, eo), (t, blk)
            assert np.array_equal(ga, ea), (t, blk)
            checked["rows"] += go.size
        checked["buckets"] += 1
        torch.cuda.synchronize()
        return 0

    with Hook(fn):
        exact, _ = plan.solve_be(assignment=False)
    assert checked["buckets"] == len(T)
    # every MBE lower bound <= exact <= its upper bound (golden c3.json)
    for g in json.load(open(os.path.join(GOLD, "c3.json"))):
        assert g["value"] <= exact
        if g["upper"] is not None:
            assert exact <= g["upper"]
    p18 = os.path.join(GOLD, "c3_i18.json")
    if os.path.exists(p18):
        assert json.load(open(p18))["value"] <= exact
    print(f"C3 exact = {exact}: {checked['buckets']} buckets, {checked['rows']} rows checked")


def _f64_tables_against_oracle(inst, order, ib, run, info, orun):
    dom = [int(v) for v in inst.dom]
    n_near = 0
    for t, (ti, ot) in enumerate(zip(info["tables"], orun.tables)):
        assert (ti["var"], ti["mb"], ti["rows"]) == (ot.var, ot.mb, ot.rows)
        o, a = run.table(t, ti["rows"])
        fin = np.isfinite(ot.out)
        assert np.array_equal(np.isfinite(o), fin), t
        assert np.array_equal(o[~fin], ot.out[~fin]), t
        err = np.abs(o[fin] - ot.out[fin])
        assert np.all(err <= 1e-9 * np.maximum(1.0, np.abs(ot.out[fin]))), (t, float(err.max()))
        bad = np.nonzero(a != ot.arg)[0]
        if bad.size:
            assert bad.size <= max(10, ti["rows"] // 1000), (t, bad.size)
            mem = []
            for kind, idx in ot.members:
                if kind == 0:
                    mem.append(([int(v) for v in inst.scope(idx)], inst.table(idx)))
                else:
                    mem.append((list(orun.tables[idx].sep), orun.tables[idx].out))
            sums = oracle.bucket_row_sums(dom, True, ot.var, mem, ot.sep, bad)
            ok = devtools.near_tie_ok(sums, a[bad].astype(np.int64), ot.arg[bad].astype(np.int64))
            assert ok.all(), (t, bad[~ok][:5])
            n_near += bad.size
    return n_near


@pytest.mark.parametrize("ib", [-1, configs.C5_IBOUND])
def test_c5_every_table_elementwise(ib):
    inst = configs.c5()
    P = G.Problem.from_instance(inst)
    order, _ = P.order()
    plan = G.Plan(P, order, ib, retain="all")
    info = plan.info()
    run, val = plan.dpop_util()  # exact DPOP, or ADPOP = MBE(16) elimination
    orun = oracle.Run(inst, order, ib, keep_tables=True, nthreads=0)
    assert orun.status == 0
    assert math.isclose(val, orun.value, rel_tol=1e-9), (val, orun.value)
    n_near = _f64_tables_against_oracle(inst, order, ib, run, info, orun)
    assign = run.value()
    run.close()
    if ib < 0:
        assert math.isclose(oracle.evaluate(inst, assign), orun.value, rel_tol=1e-9)
    else:
        assert math.isclose(oracle.evaluate(inst, assign), orun.upper, rel_tol=1e-9) or n_near > 0
    print(f"C5 i={ib}: {len(info['tables'])} tables, {n_near} near-tie argmins")
