"""The streaming bucket kernel (bk_stream.cu, variant 2) against the oracle (-m gpu).

* Large domains (d = 6 .. 256, the paper's Table 1 range d = 10..100,
  P:929): the lanes of a row split the eliminated domain and a
  warp-shuffle (value, index) min picks the first minimiser (A8) -- int32 with
  INF cells (A9) and f64 (A10), several warp-tiles per warp, ragged row ranges.
* d <= 5 through the same kernel (forced with exec option kernel = 2 and the
  GBE_KERNEL_POLICY=stream knob for the bare primitive): random descriptors,
  sum-product (A18), and whole solves (tables, argmins, optimum, assignment).
int32 bit-exact; f64 within 1e-9 relative, argmins equal except on
oracle-confirmed near-ties.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

import gen
import oracle
import paper_1608_05288_b200 as G
from gen import configs
from tests import devtools

pytestmark = pytest.mark.gpu
INF = G.INF_I32
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def bucket(rng, dom_sep, d, k, f64, p_inf=0.08):
    m = len(dom_sep)
    dom = list(dom_sep) + [d]
    members = []
    for j in range(k):
        sub = list(range(m)) if j == 0 else sorted(q for q in range(m) if rng.random() < 0.6)
        scope = sub + [m]
        cells = int(np.prod([dom[v] for v in scope]))
        if f64:
            t = rng.uniform(0, 10, cells)
            t[rng.random(cells) < p_inf] = np.inf
        else:
            t = rng.integers(0, 60, cells).astype(np.int64)  # small range: many ties
            t[rng.random(cells) < p_inf] = INF
        members.append((scope, t))
    return dom, list(range(m)), m, members


def desc_for(dom, sep, x, members, semiring):
    D = G.BucketDesc()
    D.semiring = semiring
    D.nsep = len(sep)
    D.d = dom[x]
    D.ninputs = len(members)
    rows = 1
    for q, v in enumerate(sep):
        D.radix[q] = dom[v]
        rows *= dom[v]
    D.rows = rows
    for j, (scope, _) in enumerate(members):
        st, s = {}, 1
        for v in reversed(scope):
            st[v] = s
            s *= dom[v]
        for q, v in enumerate(sep):
            D.stride[j][q] = st.get(v, 0)
    return D, rows


def run(D, members, f64, rb, re):
    dt = torch.float64 if f64 else torch.int32
    ins = [torch.tensor(np.asarray(t), dtype=dt, device="cuda") for _, t in members]
    out = torch.empty(max(re - rb, 1), dtype=dt, device="cuda")
    arg = torch.empty(max(re - rb, 1), dtype=torch.uint8, device="cuda")
    G.bucket_kernel(D, ins, out, arg, rb, re)
    torch.cuda.synchronize()
    return out.cpu().numpy()[:re - rb], arg.cpu().numpy()[:re - rb]


def check(got, ga, exp, ea, f64, dom=None, x=None, members=None, sep=None, rb=0):
    if not f64:
        np.testing.assert_array_equal(got, exp)
        np.testing.assert_array_equal(ga, ea)
        return
    assert np.array_equal(np.isinf(got), np.isinf(exp))
    f = np.isfinite(exp)
    assert np.all(np.abs(got[f] - exp[f]) <= 1e-9 * np.maximum(1.0, np.abs(exp[f])))
    bad = np.nonzero(ga != ea)[0]
    if bad.size:
        sums = oracle.bucket_row_sums(dom, True, x, members, sep, bad + rb)
        assert devtools.near_tie_ok(sums, ga[bad].astype(np.int64), ea[bad].astype(np.int64)).all()


@pytest.mark.parametrize("d", [6, 7, 8, 10, 16, 25, 33, 64, 100, 129, 200, 256])
@pytest.mark.parametrize("f64", [False, True])
def test_large_domain_lane_split(d, f64):
    rng = np.random.default_rng(d * 7 + int(f64))
    # sep radices: enough rows for several warp-tiles per warp
    dom_sep = [3, 2, 4, 3, 2, 3, 4, 3, 5] if d <= 33 else [3, 2, 4, 3, 2, 3, 4, 5]
    dom, sep, x, members = bucket(rng, dom_sep, d, 4, f64)
    D, rows = desc_for(dom, sep, x, members, G.MINSUM_F64 if f64 else G.MINSUM_I32)
    assert G.bucket_kernel_variant(D, 0, rows) == 2
    exp, ea = oracle.bucket_eval(dom, f64, x, members, sep)
    got, ga = run(D, members, f64, 0, rows)
    check(got, ga, exp, ea, f64, dom, x, members, sep)
    # a ragged row range (not tile aligned)
    rb, re = rows // 7 + 3, rows - rows // 5 - 1
    got, ga = run(D, members, f64, rb, re)
    check(got, ga, exp[rb:re], ea[rb:re], f64, dom, x, members, sep, rb)


def test_large_domain_all_inf_rows_and_ties():
    """Rows that are INF everywhere keep argmin 0; rows whose minimum is
    attained by several v keep the smallest v (A8) across lane boundaries."""
    d = 40
    dom = [5, d]
    t = np.full(5 * d, 7, dtype=np.int64)
    t[:d] = INF                      # row 0: all INF
    t[d + 33] = 3; t[d + 38] = 3    # row 1: tie at v = 33, 38 -> 33
    t[2 * d + 1] = 0; t[2 * d + 17] = 0  # row 2: tie across lanes -> 1
    members = [([0, 1], t)]
    D, rows = desc_for(dom, [0], 1, members, G.MINSUM_I32)
    got, ga = run(D, members, False, 0, rows)
    assert list(got[:3]) == [INF, 3, 0] and list(ga[:3]) == [0, 33, 1]
    assert list(ga[3:]) == [0, 0]


SCRIPT = r"""
import json, sys, numpy as np
sys.path.insert(0, sys.argv[1])
from tests import test_gpu_stream as T
import oracle, paper_1608_05288_b200 as G
res = []
for seed in range(24):
    rng = np.random.default_rng(900 + seed)
    f64 = seed % 3 == 1
    sp = seed % 6 == 4
    m = int(rng.integers(0, 9))
    dom_sep = [int(v) for v in rng.integers(1, 5, m)]
    d = int(rng.integers(1, 6))
    dom, sep, x, members = T.bucket(rng, dom_sep, d, int(rng.integers(1, 7)), f64 or sp)
    sr = G.SUMPROD_F64 if sp else (G.MINSUM_F64 if f64 else G.MINSUM_I32)
    D, rows = T.desc_for(dom, sep, x, members, sr)
    rb = int(rng.integers(0, rows)) if seed % 2 else 0
    re = int(rng.integers(rb + 1, rows + 1)) if seed % 2 else rows
    var = G.bucket_kernel_variant(D, rb, re)
    got, ga = T.run(D, members, f64 or sp, rb, re)
    if sp:
        exp = oracle.bucket_eval_sp(dom, x, members, sep, rb, re)
        ok = bool(np.array_equal(np.isinf(got), np.isinf(exp)) and np.all(np.abs(got - exp)[np.isfinite(exp)] <= 1e-9 * (1 + np.abs(exp[np.isfinite(exp)]))))
    else:
        exp, ea = oracle.bucket_eval(dom, f64, x, members, sep, rb, re)
        try:
            T.check(got, ga, exp, ea, f64, dom, x, members, sep, rb); ok = True
        except AssertionError:
            ok = False
    res.append({"seed": seed, "var": var, "ok": ok})
print(json.dumps(res))
"""


def test_small_domain_random_descriptors_forced_stream():
    env = dict(os.environ, GBE_KERNEL_POLICY="stream")
    r = subprocess.run([sys.executable, "-c", SCRIPT, ROOT], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    assert all(x["var"] == 2 for x in res), res
    assert all(x["ok"] for x in res), [x for x in res if not x["ok"]]


@pytest.mark.parametrize("name", ["c2", "bn", "sf_inf"])
def test_whole_solve_stream_kernel(name):
    if name == "c2":
        inst = configs.c2()
    elif name == "bn":
        inst = gen.belief_net(40, 2, 4, 3, 10, 3)
    else:
        inst = gen.scalefree(60, 3, 0.1, 4)
    P = G.Problem.from_instance(inst)
    order, _ = P.order()
    plan = G.Plan(P, order, retain="all", kernel=2)
    info = plan.info()
    run_, root = plan.dpop_util()
    st = run_.stats()
    assert all(t["variant"] == 2 for t in st["tasks"])
    ref = oracle.solve_be(inst, order)
    dom = [int(v) for v in inst.dom]
    for t, (ti, ot) in enumerate(zip(info["tables"], ref.tables)):
        o, a = run_.table(t, ti["rows"])
        if inst.is_f64:
            mem = [([int(v) for v in inst.scope(i)], inst.table(i)) if kd == 0 else (list(ref.tables[i].sep), ref.tables[i].out)
                   for kd, i in ot.members]
            check(o, a, ot.out, ot.arg, True, dom, ot.var, mem, ot.sep)
        else:
            check(o, a, ot.out, ot.arg, False)
    assign = run_.value()
    run_.close()
    if inst.is_f64:
        assert abs(root - ref.value) <= 1e-9 * max(1.0, abs(ref.value))
    else:
        assert root == ref.value and list(assign) == list(ref.assignment)


def bd_bucket(rng, dom_sep, d, k, f64, lack):
    """The largest input spans every output digit but `lack` (an in-tile
    digit): the streaming kernel's broadcast-digit mode loads it once for the
    rows that differ only in that digit."""
    m = len(dom_sep)
    dom = list(dom_sep) + [d]
    members = []
    for j in range(k):
        if j == 0:
            sub = [q for q in range(m) if q != lack]
        else:
            sub = sorted(q for q in range(m) if rng.random() < 0.5)
        scope = sub + [m]
        cells = int(np.prod([dom[v] for v in scope]))
        if f64:
            t = rng.uniform(0, 10, cells)
            t[rng.random(cells) < 0.05] = np.inf
        else:
            t = rng.integers(0, 60, cells).astype(np.int64)
            t[rng.random(cells) < 0.05] = INF
        members.append((scope, t))
    return dom, list(range(m)), m, members


@pytest.mark.parametrize("dom_sep,lack", [([3] * 10, 9), ([3] * 10, 8), ([4, 2, 4, 3, 4, 4, 2, 4], 7),
                                          ([4, 2, 4, 3, 4, 4, 2, 4], 5), ([2] * 14, 12), ([4] * 7, 6),
                                          # high digits (outside the warp-tile): placed on top of it
                                          ([3] * 10, 1), ([3] * 11, 0), ([4, 2, 4, 3, 4, 4, 2, 4], 1),
                                          ([2] * 14, 0), ([4] * 7, 0)])
@pytest.mark.parametrize("d", [2, 3, 4, 5])
@pytest.mark.parametrize("f64", [False, True])
def test_stream_broadcast_digit(dom_sep, lack, d, f64):
    """Broadcast-digit rows (the lane's rows differ only in a digit the
    largest input lacks; inputs without it loaded once), the digit inside
    the warp-tile or (full-range launches) a high digit on top of it: full
    range and ragged partial ranges, INF cells and ties, against the oracle."""
    os.environ["GBE_STREAM_BD"] = "1"  # the mode is opt-in; read per descriptor build
    rng = np.random.default_rng(hash((tuple(dom_sep), lack, d, f64)) % (1 << 32))
    k = int(rng.integers(2, 5))
    dom, sep, x, members = bd_bucket(rng, dom_sep, d, k, f64, lack)
    D, rows = desc_for(dom, sep, x, members, G.MINSUM_F64 if f64 else G.MINSUM_I32)
    exp, ea = oracle.bucket_eval(dom, f64, x, members, sep)
    for rb, re in [(0, rows), (7, rows - 5), (rows // 3 + 1, rows // 2 + 3)]:
        dt = torch.float64 if f64 else torch.int32
        ins = [torch.tensor(np.asarray(t), dtype=dt, device="cuda") for _, t in members]
        out = torch.empty(re - rb, dtype=dt, device="cuda")
        arg = torch.empty(re - rb, dtype=torch.uint8, device="cuda")
        G.bucket_kernel(D, ins, out, arg, rb, re, variant=2)
        torch.cuda.synchronize()
        check(out.cpu().numpy(), arg.cpu().numpy(), exp[rb:re], ea[rb:re], f64, dom, x, members, sep, rb)
    del os.environ["GBE_STREAM_BD"]


@pytest.mark.parametrize("f64", [False, True])
def test_stream_blocked_high_digits(f64):
    """Three large inputs (>= 16 MB) that lack different high digits: the
    third one's absent digits go on top of the warp-tile (its re-reads stay
    inside a tile; the tile's rows are then strided), the two largest are
    served by the tile order.  Full range through the streaming kernel,
    against the oracle."""
    rng = np.random.default_rng(77 + int(f64))
    m, d = 12, 4
    dom = [4] * m + [d]
    lacks = [(2, 5), (3, 7), (0, 1)]
    members = []
    for la in lacks:
        scope = [q for q in range(m) if q not in la] + [m]
        cells = int(np.prod([dom[v] for v in scope]))
        t = rng.uniform(0, 10, cells) if f64 else rng.integers(0, 60, cells).astype(np.int64)
        members.append((scope, t))
    small = [4, 9, m]
    members.append((small, rng.uniform(0, 10, 64) if f64 else rng.integers(0, 60, 64).astype(np.int64)))
    sep = list(range(m))
    D, rows = desc_for(dom, sep, m, members, G.MINSUM_F64 if f64 else G.MINSUM_I32)
    exp, ea = oracle.bucket_eval(dom, f64, m, members, sep)
    for hx in ("1", "0"):
        os.environ["GBE_STREAM_HX"] = hx
        dt = torch.float64 if f64 else torch.int32
        ins = [torch.tensor(np.asarray(t), dtype=dt, device="cuda") for _, t in members]
        out = torch.empty(rows, dtype=dt, device="cuda")
        arg = torch.empty(rows, dtype=torch.uint8, device="cuda")
        G.bucket_kernel(D, ins, out, arg, 0, rows, variant=2)
        torch.cuda.synchronize()
        check(out.cpu().numpy(), arg.cpu().numpy(), exp, ea, f64, dom, m, members, sep, 0)
        del ins, out, arg
    del os.environ["GBE_STREAM_HX"]


@pytest.mark.parametrize("dom_sep,lacks", [([2, 3, 2, 2, 3, 3, 3, 3, 3], (0, 2)),  # two radix-2 digits
                                           ([2, 2, 4, 3, 2, 4, 2, 4, 4], (1, 4)),
                                           ([3, 4, 3, 3, 3, 3, 3, 3, 3], (1,)),    # one radix-4 digit
                                           ([3, 2, 3, 3, 3, 3, 3, 3, 3], (0,)),    # one radix-3 digit
                                           ([2, 2, 2, 3, 3, 3, 3, 3, 3], (0, 1, 2))])
@pytest.mark.parametrize("d", [2, 3, 4, 5])
@pytest.mark.parametrize("f64", [False, True])
def test_stream_high_broadcast_digits(dom_sep, lacks, d, f64):
    """High broadcast digits (opt-in, measured slower; forced here): the largest input lacks high output digits, a lane's rows are the
    combinations of two radix-2 such digits (or the values of one of radix
    3-4) on top of the warp-tile, inputs lacking one load once per
    combination of the others.  Full range (the mode's only use) plus a
    partial range (plain streaming), INF cells and ties, against the oracle."""
    os.environ["GBE_STREAM_BD2"] = "1"
    try:
        rng = np.random.default_rng(hash((tuple(dom_sep), lacks, d, f64, "bd2")) % (1 << 32))
        m = len(dom_sep)
        dom = list(dom_sep) + [d]
        members = []
        for j in range(int(rng.integers(2, 5))):
            if j == 0:
                sub = [q for q in range(m) if q not in lacks]
            else:  # other inputs: random subsets (some lack a broadcast digit, some not)
                sub = sorted(q for q in range(m) if rng.random() < 0.5)
            scope = sub + [m]
            cells = int(np.prod([dom[v] for v in scope]))
            if f64:
                t = rng.uniform(0, 10, cells).round(1)  # ties
                t[rng.random(cells) < 0.05] = np.inf
            else:
                t = rng.integers(0, 30, cells).astype(np.int64)
                t[rng.random(cells) < 0.05] = INF
            members.append((scope, t))
        sep = list(range(m))
        D, rows = desc_for(dom, sep, m, members, G.MINSUM_F64 if f64 else G.MINSUM_I32)
        exp, ea = oracle.bucket_eval(dom, f64, m, members, sep)
        dt = torch.float64 if f64 else torch.int32
        for rb, re in [(0, rows), (5, rows - 3)]:
            ins = [torch.tensor(np.asarray(t), dtype=dt, device="cuda") for _, t in members]
            out = torch.empty(re - rb, dtype=dt, device="cuda")
            arg = torch.empty(re - rb, dtype=torch.uint8, device="cuda")
            G.bucket_kernel(D, ins, out, arg, rb, re, variant=2)
            torch.cuda.synchronize()
            check(out.cpu().numpy(), arg.cpu().numpy(), exp[rb:re], ea[rb:re], f64, dom, m, members, sep, rb)
    finally:
        del os.environ["GBE_STREAM_BD2"]


def run_variant(D, members, f64, rb, re, variant):
    dt = torch.float64 if f64 else torch.int32
    ins = [torch.tensor(np.asarray(t), dtype=dt, device="cuda") for _, t in members]
    out = torch.empty(max(re - rb, 1), dtype=dt, device="cuda")
    arg = torch.empty(max(re - rb, 1), dtype=torch.uint8, device="cuda")
    G.bucket_kernel(D, ins, out, arg, rb, re, variant=variant)
    torch.cuda.synchronize()
    return out.cpu().numpy()[:re - rb], arg.cpu().numpy()[:re - rb]


@pytest.mark.parametrize("seed", range(16))
def test_staged_random_descriptors(seed):
    """The streaming kernel's staged mode (variant 3: per-warp TMA double
    buffers of the tile's input slices, shared-memory loads): random
    canonical descriptors, d = 2..5, int32 with INF cells and f64, full and
    ragged partial row ranges, against the oracle."""
    rng = np.random.default_rng(4100 + seed)
    f64 = seed % 2 == 1
    m = int(rng.integers(1, 10))
    dom_sep = [int(v) for v in rng.integers(1, 5, m)]
    d = int(rng.integers(2, 6))
    dom, sep, x, members = bucket(rng, dom_sep, d, int(rng.integers(1, 7)), f64)
    D, rows = desc_for(dom, sep, x, members, G.MINSUM_F64 if f64 else G.MINSUM_I32)
    for rb, re in [(0, rows), (int(rng.integers(0, rows)), rows)]:
        re = max(re, rb + 1)
        got, ga = run_variant(D, members, f64, rb, re, 3)
        exp, ea = oracle.bucket_eval(dom, f64, x, members, sep, rb, re)
        check(got, ga, exp, ea, f64, dom, x, members, sep, rb)


@pytest.mark.parametrize("f64", [False, True])
def test_staged_many_tiles_per_warp(f64):
    """Staged mode over 10-25 warp-tiles per warp (both buffers of every
    warp reused many times: the mbarrier phases flip), one large input
    lacking a high digit plus small ones, full range and a ragged range, vs
    the oracle."""
    rng = np.random.default_rng(4200 + int(f64))
    if f64:
        dom_sep, d = [2, 4, 3, 4, 4, 3, 4, 4, 3, 4, 4, 2, 2], 4
    else:
        dom_sep, d = [3] * 15, 3
    m = len(dom_sep)
    dom = list(dom_sep) + [d]
    members = []
    for j, sub in enumerate([list(range(1, m)), [0, 3, m - 1], [2, m - 2], [m - 1]]):
        scope = sub + [m]
        cells = int(np.prod([dom[v] for v in scope]))
        t = rng.uniform(0, 10, cells).round(1) if f64 else rng.integers(0, 40, cells).astype(np.int64)
        if j == 1:
            t[rng.random(cells) < 0.05] = np.inf if f64 else INF
        members.append((scope, t))
    D, rows = desc_for(dom, list(range(m)), m, members, G.MINSUM_F64 if f64 else G.MINSUM_I32)
    for rb, re in [(0, rows), (12345, rows - 777)]:
        got, ga = run_variant(D, members, f64, rb, re, 3)
        exp, ea = oracle.bucket_eval(dom, f64, m, members, list(range(m)), rb, re)
        check(got, ga, exp, ea, f64, dom, m, members, list(range(m)), rb)


STAGED_SOLVE = r"""
import json, sys, numpy as np
sys.path.insert(0, sys.argv[1])
from tests import test_gpu_stream as T
import gen, oracle, paper_1608_05288_b200 as G
from gen import configs
res = []
for name in ["c2", "bn", "sf_inf"]:
    inst = configs.c2() if name == "c2" else (gen.belief_net(40, 2, 4, 3, 10, 3) if name == "bn" else gen.scalefree(60, 3, 0.1, 4))
    P = G.Problem.from_instance(inst)
    order, _ = P.order()
    plan = G.Plan(P, order, retain="all", kernel=2)
    info = plan.info()
    ok = True
    for rep in range(2):
        run_, root = plan.dpop_util()
        st = run_.stats()
        staged = sum(1 for t in st["tasks"] if t.get("staged"))
        ref = oracle.solve_be(inst, order)
        dom = [int(v) for v in inst.dom]
        try:
            for t, (ti, ot) in enumerate(zip(info["tables"], ref.tables)):
                o, a = run_.table(t, ti["rows"])
                if inst.is_f64:
                    mem = [([int(v) for v in inst.scope(i)], inst.table(i)) if kd == 0 else (list(ref.tables[i].sep), ref.tables[i].out)
                           for kd, i in ot.members]
                    T.check(o, a, ot.out, ot.arg, True, dom, ot.var, mem, ot.sep)
                else:
                    T.check(o, a, ot.out, ot.arg, False)
            assign = run_.value()
            if inst.is_f64:
                ok = ok and abs(root - ref.value) <= 1e-9 * max(1.0, abs(ref.value))
            else:
                ok = ok and root == ref.value and list(assign) == list(ref.assignment)
        except AssertionError:
            ok = False
        run_.close()
    res.append({"name": name, "staged": staged, "ok": ok})
print(json.dumps(res))
"""


def test_whole_solve_staged():
    """Whole solves with every bucket the staged mode fits staged
    (GBE_STREAM_STAGE=1, read once per process: a subprocess): tables,
    argmins, optimum and assignment against the oracle, two solves per plan
    (the second a CUDA-graph replay)."""
    env = dict(os.environ, GBE_STREAM_STAGE="1")
    r = subprocess.run([sys.executable, "-c", STAGED_SOLVE, ROOT], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    assert all(x["staged"] > 0 for x in res), res
    assert all(x["ok"] for x in res), res
