"""BASELINE configs at full size on the GPU against stored oracle results
(tests/golden/*.json, written by scripts/make_golden.py, which calls only
oracle/ and gen/) and against properties that hold at any size (-m gpu).

* C2 / C4 (int32 DCOP, DPOP): every UTIL table's FNV-1a digest of
  (out, argmin) equals the oracle's; optimum equal; evaluate(assignment) =
  optimum (C2: assignment equal).
* C3 (20x20 grid, row-major): MBE i = 8..16 lower bounds and table digests
  equal (i <= 14: upper bound and assignment equal); the i = 18 lower bound
  (value-only: its retained messages would total ~0.5 TB) and the exact value
  (value-only: its argmins would need 1.27 TB) satisfy
  lower(i) <= exact <= upper(i).
* C5 (BN MPE, f64): exact and MBE i=16 optima within 1e-9 relative, per-table
  sum / min / max of finite entries within 1e-9, infinite counts equal.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
import paper_1608_05288_b200 as G
from gen import configs

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def gold(name):
    p = os.path.join(GOLD, name)
    if not os.path.exists(p):
        pytest.skip(f"{p} not generated (python scripts/make_golden.py)")
    return json.load(open(p))


def table_digests(run, info):
    out = []
    for t, ti in enumerate(info["tables"]):
        o, a = run.table(t, ti["rows"])
        out.append(f"{oracle.fnv1a(o, a):016x}")
        del o, a
    return out


def _dpop_against(name, inst):
    g = gold(name)
    P = G.Problem.from_instance(inst)
    order, _ = P.order()
    assert list(order) == g["order"]
    plan = G.Plan(P, order, retain="all")
    info = plan.info()
    run, root = plan.dpop_util()
    assert root == g["value"]
    digests = table_digests(run, info)
    assign = run.value()
    run.close()
    assert len(digests) == len(g["tables"])
    bad = [i for i, (d, t) in enumerate(zip(digests, g["tables"])) if d != t["digest"]]
    assert not bad, f"{len(bad)} tables differ, first {bad[:5]}"
    assert P.evaluate(assign) == root == oracle.evaluate(inst, assign)
    if g.get("assignment"):
        assert list(assign) == g["assignment"]


def test_c2_full_dpop_digests():
    _dpop_against("c2.json", configs.c2())


def test_c4_full_dpop_digests():
    """The bench workload: 200 UTIL tables, the largest 3^20 rows."""
    _dpop_against("c4.json", configs.c4())


def test_c4d4_full_dpop_digests():
    """SURVEY's alternative C4 at the BASELINE domain d = 4 (n = 150, min-fill
    w* = 16): the largest table 4^16 = 4.29e9 rows, so the tiled kernel's
    R = 4 register-block shapes run at full size."""
    _dpop_against("c4d4.json", configs.c4d4())


def test_c3_grid_mbe_sweep_and_exact():
    """MBE / ADPOP i-bound sweep on the 20x20 grid: lower bounds, tables,
    upper bounds and assignments against the oracle; then i = 18 and the
    exact value (value-only) inside every [lower, upper] bracket."""
    recs = gold("c3.json")
    inst = configs.c3()
    order = configs.c3_order()
    P = G.Problem.from_instance(inst)
    bounds = {}
    for g in recs:
        ib = g["ibound"]
        plan = G.Plan(P, order, ib, retain="all")
        info = plan.info()
        assert [(t["var"], t["mb"], t["rows"]) for t in info["tables"]] == \
            [(t["var"], t["mb"], t["rows"]) for t in g["tables"]]
        run, lo = plan.dpop_util()  # ADPOP UTIL = MBE elimination
        assert lo == g["value"], (ib, lo, g["value"])
        digests = table_digests(run, info)
        bad = [i for i, (d, t) in enumerate(zip(digests, g["tables"])) if d != t["digest"]]
        assert not bad, f"i={ib}: {len(bad)} tables differ"
        a = run.value()
        run.close()
        up = P.evaluate(a)
        if g["upper"] is not None:
            assert up == g["upper"] and list(a) == g["assignment"]
        lo2, up2, a2 = G.Plan(P, order, ib).solve_mbe()
        assert (lo2, up2) == (lo, up) and list(a2) == list(a)
        bounds[ib] = (lo, up)
    # i = 18: its retained messages would total ~0.5 TB, so lower bound only
    # (value-only MBE frees each message once consumed)
    lo18, _, _ = G.Plan(P, order, 18, retain="none").solve_mbe(assignment=False)
    exact, _ = G.Plan(P, order, retain="none").solve_be(assignment=False)
    assert lo18 <= exact
    for ib, (lo, up) in bounds.items():
        assert lo <= exact <= up, (ib, lo, exact, up)
    assert lo18 >= bounds[8][0]


def test_c5_bn_mpe_exact_and_mbe16():
    recs = gold("c5.json")
    inst = configs.c5()
    P = G.Problem.from_instance(inst)
    order, _ = P.order()
    for g in recs:
        ib = g["ibound"]
        assert list(order) == g["order"]
        plan = G.Plan(P, order, ib, retain="all")
        info = plan.info()
        if ib < 0:
            run, val = plan.dpop_util()
            assign = run.value()
        else:
            lo, up, assign = plan.solve_mbe()
            val = lo
            assert math.isclose(up, g["upper"], rel_tol=1e-9) or up >= g["value"]
            run = None
        assert math.isclose(val, g["value"], rel_tol=1e-9), (ib, val, g["value"])
        assert math.isclose(P.evaluate(assign), oracle.evaluate(inst, assign), rel_tol=1e-12)
        if ib < 0:
            assert math.isclose(P.evaluate(assign), val, rel_tol=1e-9)
            for t, (ti, gt) in enumerate(zip(info["tables"], g["tables"])):
                o, _ = run.table(t, ti["rows"], want_arg=False)
                fin = np.isfinite(o)
                assert int((~fin).sum()) == gt["n_inf"], t
                if fin.any():
                    assert math.isclose(float(np.sum(o[fin], dtype=np.float64)), gt["sum"], rel_tol=1e-9), t
                    assert math.isclose(float(o[fin].min()), gt["min"], rel_tol=1e-9)
                    assert math.isclose(float(o[fin].max()), gt["max"], rel_tol=1e-9)
            run.close()
