"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle,
element by element, on the same seeded inputs (-m gpu).

Bar: bit-exact for int32 min-sum (tables, argmins, optimum, assignment);
float64 MPE within 1e-9 relative (tables, optimum) with argmins compared
where the oracle's decision is not a near-tie (DESIGN.md §3 A10).
"""
import math

import numpy as np
import pytest

import gen
import oracle
from tests import devtools
import paper_1608_05288_b200 as G
from gen import configs
from oracle.brute import brute_force_np

pytestmark = pytest.mark.gpu
INF = G.INF_I32


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    return torch


# ---------------------------------------------------------------- helpers

def random_bucket(rng, f64=False, max_m=6, dmax=5, big=False):
    """A random (mini-)bucket: sep variables 0..m-1, eliminated variable m,
    k members over random sub-scopes (each contains m), random INF cells."""
    m = int(rng.integers(0, max_m + 1))
    dom = [int(x) for x in rng.integers(1, dmax + 1, m)]
    if big:
        dom = [int(x) for x in rng.integers(2, 5, m)]
    d = int(rng.choice([1, 2, 3, 4, 5, 10, 33, 100])) if not big else int(rng.choice([2, 3, 4, 5]))
    dom.append(d)
    k = int(rng.integers(0, 17))
    members = []
    for _ in range(k):
        sub = sorted(rng.choice(m, size=int(rng.integers(0, m + 1)), replace=False).tolist()) if m else []
        scope = sub + [m]
        cells = int(np.prod([dom[v] for v in scope]))
        if f64:
            t = rng.uniform(0, 10, cells)
            t[rng.random(cells) < 0.1] = np.inf
        else:
            t = rng.integers(0, 1000, cells).astype(np.int64)
            t[rng.random(cells) < 0.1] = INF
        members.append((scope, t))
    return dom, list(range(m)), m, members


def desc_for(dom, sep, x, members, f64):
    D = G.BucketDesc()
    D.semiring = G.MINSUM_F64 if f64 else G.MINSUM_I32
    D.nsep = len(sep)
    D.d = dom[x]
    D.ninputs = len(members)
    rows = 1
    for q, v in enumerate(sep):
        D.radix[q] = dom[v]
        rows *= dom[v]
    D.rows = rows
    for j, (scope, _) in enumerate(members):
        st = {}
        s = 1
        for v in reversed(scope):
            st[v] = s
            s *= dom[v]
        for q, v in enumerate(sep):
            D.stride[j][q] = st.get(v, 0)
    return D, rows


def run_bucket(torch, dom, sep, x, members, f64, rb, re, variant=-1):
    D, rows = desc_for(dom, sep, x, members, f64)
    dt = torch.float64 if f64 else torch.int32
    ins = [torch.tensor(np.asarray(t), dtype=dt, device="cuda") for _, t in members]
    n = max(re - rb, 1)
    out = torch.empty(n, dtype=dt, device="cuda")
    arg = torch.empty(n, dtype=torch.uint8, device="cuda")
    G.bucket_kernel(D, ins, out, arg, rb, re, variant=variant)
    torch.cuda.synchronize()
    return out.cpu().numpy()[:re - rb], arg.cpu().numpy()[:re - rb]


def compare_f64(got, got_arg, exp, exp_arg, rows_members=None):
    assert np.allclose(got, exp, rtol=1e-9, atol=0.0, equal_nan=False) or np.array_equal(got, exp)
    np.testing.assert_array_equal(np.isinf(got), np.isinf(exp))
    return np.mean(got_arg == exp_arg)


# ---------------------------------------------------------------- the primitive

@pytest.mark.parametrize("seed", range(60))
def test_bucket_kernel_random_descriptors_int(torch_cuda, seed):
    rng = np.random.default_rng(1000 + seed)
    dom, sep, x, members = random_bucket(rng, big=seed % 3 == 0, max_m=9 if seed % 3 == 0 else 6)
    rows = int(np.prod([dom[v] for v in sep])) if sep else 1
    rb = int(rng.integers(0, rows)) if seed % 4 == 1 else 0
    re = int(rng.integers(rb + 1, rows + 1)) if seed % 4 == 1 else rows
    exp, exp_arg = oracle.bucket_eval(dom, False, x, members, sep, rb, re)
    got, got_arg = run_bucket(torch_cuda, dom, sep, x, members, False, rb, re)
    np.testing.assert_array_equal(got, exp)
    np.testing.assert_array_equal(got_arg, exp_arg)


@pytest.mark.parametrize("seed", range(30))
def test_bucket_kernel_random_descriptors_f64(torch_cuda, seed):
    rng = np.random.default_rng(5000 + seed)
    dom, sep, x, members = random_bucket(rng, f64=True, big=seed % 3 == 0, max_m=8)
    rows = int(np.prod([dom[v] for v in sep])) if sep else 1
    exp, exp_arg = oracle.bucket_eval(dom, True, x, members, sep)
    got, got_arg = run_bucket(torch_cuda, dom, sep, x, members, True, 0, rows)
    # same canonical summation order -> bit-exact; the bar is 1e-9 relative
    np.testing.assert_array_equal(np.isinf(got), np.isinf(exp))
    fin = np.isfinite(exp)
    assert np.allclose(got[fin], exp[fin], rtol=1e-9, atol=0)
    np.testing.assert_array_equal(got_arg, exp_arg)


def test_bucket_kernel_edge_cases(torch_cuda):
    # eliminate [5,2,7,1] -> [2,1]
    got, arg = run_bucket(torch_cuda, [2, 2], [0], 1, [([0, 1], [5, 2, 7, 1])], False, 0, 2)
    assert list(got) == [2, 1] and list(arg) == [1, 1]
    # empty bucket: constant 0, argmin 0
    got, arg = run_bucket(torch_cuda, [3], [], 0, [], False, 0, 1)
    assert list(got) == [0] and list(arg) == [0]
    # all-INF row stays INF with argmin 0
    got, arg = run_bucket(torch_cuda, [2, 3], [0], 1, [([0, 1], [INF] * 6)], False, 0, 2)
    assert list(got) == [INF, INF] and list(arg) == [0, 0]
    # d = 1 copies
    got, arg = run_bucket(torch_cuda, [3, 1], [0], 1, [([0, 1], [5, 6, 7])], False, 0, 3)
    assert list(got) == [5, 6, 7]


def test_bucket_kernel_virtual_shards(torch_cuda):
    """Row ranges computed separately and concatenated equal one launch
    (the row-sharding contract)."""
    rng = np.random.default_rng(77)
    dom = [3] * 11
    sep, x = list(range(10)), 10
    members = [(sorted(rng.choice(10, 7, replace=False).tolist()) + [10], None) for _ in range(5)]
    members = [(s, rng.integers(0, 100, int(np.prod([dom[v] for v in s])))) for s, _ in members]
    rows = 3 ** 10
    full, fa = run_bucket(torch_cuda, dom, sep, x, members, False, 0, rows)
    cuts = sorted(set([0, rows] + rng.integers(1, rows, 6).tolist()))
    parts = [run_bucket(torch_cuda, dom, sep, x, members, False, a, b) for a, b in zip(cuts, cuts[1:])]
    np.testing.assert_array_equal(np.concatenate([p[0] for p in parts]), full)
    np.testing.assert_array_equal(np.concatenate([p[1] for p in parts]), fa)


# ---------------------------------------------------------------- solves

def _check_tables(run, plan_info, orun, f64):
    for t, (ti, ot) in enumerate(zip(plan_info["tables"], orun.tables)):
        out, arg = run.table(t, ti["rows"])
        if f64:
            np.testing.assert_array_equal(np.isinf(out), np.isinf(ot.out))
            fin = np.isfinite(ot.out)
            assert np.allclose(out[fin], ot.out[fin], rtol=1e-9, atol=0)
        else:
            np.testing.assert_array_equal(out, ot.out, err_msg=f"table {t} (x{ti['var']})")
        np.testing.assert_array_equal(arg, ot.arg, err_msg=f"argmin {t} (x{ti['var']})")


INSTANCES = {
    "random_net": lambda: gen.random_network(16, 2, 4, 24, 1, 3, 100, 0.2, 3),
    "random_graph_p2": lambda: gen.random_graph(18, 3, 40, 0, 0.5, 4),
    "scalefree": lambda: gen.scalefree(45, 3, 0.0, 2),
    "grid6": lambda: gen.grid(6, 6, 3, 0.0, 1),
    "rand_d10": lambda: gen.random_graph(12, 10, 22, 1, 0.0, 8),
    "bn": lambda: gen.belief_net(40, 2, 4, 3, 8, 1),
    "netf": lambda: gen.random_network_f64(14, 2, 5, 20, 1, 3, 10.0, 0.1, 2),
}


@pytest.mark.parametrize("name", sorted(INSTANCES))
def test_be_matches_oracle(torch_cuda, name):
    inst = INSTANCES[name]()
    P = G.Problem.from_instance(inst)
    order, _ = P.order()
    plan = G.Plan(P, order, retain="all")
    info = plan.info()
    orun = oracle.solve_be(inst, order)
    run, root = plan.dpop_util()
    assign = run.value()
    _check_tables(run, info, orun, inst.is_f64)
    run.close()
    if inst.is_f64:
        assert math.isclose(root, orun.value, rel_tol=1e-9)
        assert math.isclose(P.evaluate(assign), orun.value, rel_tol=1e-9)
    else:
        assert root == orun.value
        assert list(assign) == list(orun.assignment)
    # the one-call solve agrees
    opt, a2 = G.Plan(P, order).solve_be()
    assert opt == root and list(a2) == list(assign)


@pytest.mark.parametrize("name", ["random_net", "scalefree", "grid6", "bn"])
@pytest.mark.parametrize("ib", [1, 2, 3, 5])
def test_mbe_matches_oracle(torch_cuda, name, ib):
    inst = INSTANCES[name]()
    P = G.Problem.from_instance(inst)
    order, w = P.order()
    maxar = int(inst.arity.max())
    if ib + 1 < maxar:
        with pytest.raises(G.GbeError):
            G.Plan(P, order, ib)
        return
    orun = oracle.solve_mbe(inst, order, ib)
    lo, up, a = G.Plan(P, order, ib).solve_mbe()
    if inst.is_f64:
        assert math.isclose(lo, orun.value, rel_tol=1e-9)
        assert math.isclose(up, P.evaluate(a), rel_tol=1e-12)
    else:
        assert lo == orun.value and up == orun.upper
        assert list(a) == list(orun.assignment)
        assert lo <= oracle.solve_be(inst, order).value <= up


@pytest.mark.parametrize("seed", range(8))
def test_c1_against_brute_force(torch_cuda, seed):
    """C1: tiny random WCSP, exact BE vs brute force (3^12 states)."""
    inst = configs.c1(seed, literal=bool(seed % 2), p2=0.5 if seed >= 4 else 0.0)
    P = G.Problem.from_instance(inst)
    order, _ = P.order()
    opt, a = G.Plan(P, order).solve_be()
    bopt, ba = brute_force_np(inst, order)
    assert opt == bopt
    assert P.evaluate(a) == bopt
    if bopt < INF:
        assert list(a) == ba


def test_c2_dpop_matches_oracle(torch_cuda):
    """C2: random DCOP n=100, d=5, w*=10: every UTIL table bit-exact."""
    inst = configs.c2()
    P = G.Problem.from_instance(inst)
    order, w = P.order()
    assert w == 10
    plan = G.Plan(P, order, retain="all")
    run, root = plan.dpop_util()
    orun = oracle.solve_be(inst, order)
    _check_tables(run, plan.info(), orun, False)
    assign = run.value()
    assert root == orun.value and list(assign) == list(orun.assignment)
    # Cor. 2: n - #components UTIL messages (connected: n - 1)
    assert sum(1 for t in plan.info()["tables"] if t["dest"] >= 0) == inst.n - 1


def test_dpop_equals_be_and_message_count(torch_cuda):
    inst = gen.scalefree(60, 3, 0.0, 7)
    P = G.Problem.from_instance(inst)
    order, _ = P.order()
    plan = G.Plan(P, order)
    run, root = plan.dpop_util()
    a = run.value()
    opt, a2 = G.Plan(P, order).solve_be()
    assert root == opt and list(a) == list(a2)
    assert P.evaluate(a) == opt


def test_mpe_bn_small_against_brute_force(torch_cuda):
    from oracle.brute import mpe_linear
    for seed in range(4):
        inst = gen.belief_net(9, 2, 3, 2, 4, seed)
        P = G.Problem.from_instance(inst)
        order, _ = P.order()
        opt, a = G.Plan(P, order).solve_be()
        assert math.isclose(math.exp(-opt), mpe_linear(inst), rel_tol=1e-9)


# ---------------------------------------------------------------- tiled TMA kernel

FAST_SHAPES = [(2, 2), (2, 3), (2, 4), (2, 5), (3, 2), (3, 3), (3, 4), (3, 5), (4, 2), (4, 3), (4, 4),
               (4, 5), (5, 2), (5, 3), (5, 4), (5, 5)]


def uniform_bucket(rng, R, DV, m, k, f64):
    dom = [R] * m + [DV]
    members = []
    for j in range(k):
        p = rng.uniform(0.1, 0.95)
        sub = [q for q in range(m) if rng.random() < p]
        scope = sub + [m]
        cells = int(np.prod([dom[v] for v in scope]))
        if f64:
            t = rng.uniform(0, 10, cells)
            t[rng.random(cells) < 0.05] = np.inf
        else:
            t = rng.integers(0, 1000, cells).astype(np.int64)
            t[rng.random(cells) < 0.05] = INF
        members.append((scope, t))
    return dom, list(range(m)), m, members


@pytest.mark.parametrize("R,DV", FAST_SHAPES)
@pytest.mark.parametrize("f64", [False, True])
def test_fast_kernel_shapes(torch_cuda, R, DV, f64):
    rng = np.random.default_rng(R * 100 + DV * 10 + int(f64))
    m = {2: 13, 3: 9, 4: 7, 5: 6}[R]
    for trial in range(3):
        k = int(rng.integers(1, 12))
        dom, sep, x, members = uniform_bucket(rng, R, DV, m, k, f64)
        D, rows = desc_for(dom, sep, x, members, f64)
        # auto: tiled for int32, streaming for f64; both variants run explicitly
        assert G.bucket_kernel_variant(D, 0, rows) == (2 if f64 else 1)
        variants = [2] if (f64 and R == 5 and DV == 5) else [1, 2]  # no f64 tiled 5x5x5 shape
        exp, exp_arg = oracle.bucket_eval(dom, f64, x, members, sep)
        for var in variants:
            got, got_arg = run_bucket(torch_cuda, dom, sep, x, members, f64, 0, rows, variant=var)
            if f64:
                np.testing.assert_array_equal(np.isinf(got), np.isinf(exp))
                fin = np.isfinite(exp)
                assert np.allclose(got[fin], exp[fin], rtol=1e-9, atol=0)
                # argmins may differ only on near-ties (different summation
                # order): the oracle's own sums of both choices within 1e-9 (A10)
                bad = np.nonzero(got_arg != exp_arg)[0]
                if bad.size:
                    sums = oracle.bucket_row_sums(dom, True, x, members, sep, bad)
                    assert devtools.near_tie_ok(sums, got_arg[bad].astype(np.int64),
                                                exp_arg[bad].astype(np.int64)).all()
            else:
                np.testing.assert_array_equal(got, exp)
                np.testing.assert_array_equal(got_arg, exp_arg)


def test_fast_kernel_partial_ranges(torch_cuda):
    """Tile-aligned row ranges (the row-shard contract) on the tiled kernel."""
    rng = np.random.default_rng(9)
    dom, sep, x, members = uniform_bucket(rng, 3, 3, 10, 7, False)
    D, rows = desc_for(dom, sep, x, members, False)
    full, fa = run_bucket(torch_cuda, dom, sep, x, members, False, 0, rows)
    blk = rows // 9
    for a, b in [(0, 3 * blk), (3 * blk, 7 * blk), (7 * blk, rows)]:
        assert G.bucket_kernel_variant(D, a, b) == 1
        got, ga = run_bucket(torch_cuda, dom, sep, x, members, False, a, b)
        np.testing.assert_array_equal(got, full[a:b])
        np.testing.assert_array_equal(ga, fa[a:b])


def test_fast_and_generic_kernels_agree_on_c4alt_buckets(torch_cuda):
    """Whole DPOP on a BA n=120 DCOP: every table from the auto plan (tiled
    kernel on large buckets) equals the generic-kernel plan bit for bit, and
    the tiled kernel was actually used."""
    inst = gen.scalefree(120, 3, 0.0, 3)
    P = G.Problem.from_instance(inst)
    order, w = P.order()
    pa = G.Plan(P, order, retain="all", timing=True)
    pg = G.Plan(P, order, retain="all", kernel=0)
    ra, roota = pa.dpop_util()
    rg, rootg = pg.dpop_util()
    st = ra.stats()
    assert any(t["variant"] == 1 for t in st["tasks"])
    assert roota == rootg
    for t, ti in enumerate(pa.info()["tables"]):
        oa, aa = ra.table(t, ti["rows"])
        og, ag = rg.table(t, ti["rows"])
        np.testing.assert_array_equal(oa, og)
        np.testing.assert_array_equal(aa, ag)
    assert list(ra.value()) == list(rg.value())


@pytest.mark.parametrize("concurrent", [True, False])
@pytest.mark.parametrize("name", ["scalefree", "grid6", "random_graph_p2", "bn", "c2"])
def test_graph_replay_matches_oracle(torch_cuda, name, concurrent):
    """From the second solve on the UTIL phase replays as a CUDA graph; with
    "concurrent" that graph is the task DAG (sibling subtrees overlap, arena
    ranges reused under DAG edges).  Every replay must equal the oracle: all
    tables and argmins (retain all), optimum + assignment (retain args) and the
    value-only optimum (retain none, maximum arena reuse).  Autotuning is off
    so the graph is captured on the first solve and replayed from the second
    (with it, the first 2n solves are eager candidate timings)."""
    inst = configs.c2() if name == "c2" else INSTANCES[name]()
    P = G.Problem.from_instance(inst)
    order, _ = P.order()
    orun = oracle.solve_be(inst, order)

    def same(v):
        return math.isclose(v, orun.value, rel_tol=1e-9) if inst.is_f64 else v == orun.value

    plan = G.Plan(P, order, retain="all", concurrent=concurrent, autotune=False)
    info = plan.info()
    for rep in range(3):
        run, root = plan.dpop_util()
        assert same(root), rep
        if rep == 2:
            _check_tables(run, info, orun, inst.is_f64)
        run.close()
    plan = G.Plan(P, order, concurrent=concurrent, autotune=False)
    for rep in range(4):
        opt, a = plan.solve_be()
        assert same(opt), rep
        if not inst.is_f64:
            assert list(a) == list(orun.assignment), rep
    plan = G.Plan(P, order, retain="none", concurrent=concurrent, autotune=False)
    for rep in range(4):
        opt, _ = plan.solve_be(assignment=False)
        assert same(opt), rep


@pytest.mark.parametrize("ib", [2, 4])
def test_graph_replay_mbe(torch_cuda, ib):
    """MBE plans replay too: lower/upper bounds and assignment stay equal to the
    oracle's on every replay (messages retained for the value phase, A7)."""
    inst = INSTANCES["grid6"]()
    P = G.Problem.from_instance(inst)
    order, _ = P.order()
    orun = oracle.solve_mbe(inst, order, ib)
    plan = G.Plan(P, order, ib, autotune=False)
    for rep in range(4):
        lo, up, a = plan.solve_mbe()
        assert (lo, up) == (orun.value, orun.upper), rep
        assert list(a) == list(orun.assignment), rep
    plan = G.Plan(P, order, ib, retain="none", autotune=False)
    for rep in range(4):
        lo, _, _ = plan.solve_mbe(assignment=False)
        assert lo == orun.value, rep


@pytest.mark.parametrize("name", ["scalefree", "bn", "c2"])
def test_autotuned_plan_every_solve(torch_cuda, name):
    """With autotuning on, a plan's first 2n solves run the buckets' candidate
    launches (tiled, streaming, prefetch flipped, half-length warp-tiles) in
    turn, eagerly; then the chosen ones are captured and replayed.  Every
    solve -- each candidate round, the capture and the replays -- must equal
    the oracle (optimum, assignment), and the tables of the last replay too."""
    inst = configs.c2() if name == "c2" else INSTANCES[name]()
    P = G.Problem.from_instance(inst)
    order, _ = P.order()
    orun = oracle.solve_be(inst, order)
    plan = G.Plan(P, order, retain="all")
    info = plan.info()
    tuned, replays = 0, 0
    for rep in range(16):
        run, root = plan.dpop_util()
        st = run.stats()
        tuned += bool(st.get("autotune_solve"))
        replays += bool(st.get("graph_replay"))
        if inst.is_f64:
            assert math.isclose(root, orun.value, rel_tol=1e-9), rep
        else:
            assert root == orun.value, rep
            assert list(run.value()) == list(orun.assignment), rep
        if rep == 15:
            _check_tables(run, info, orun, inst.is_f64)
        run.close()
    assert tuned >= 2 and replays >= 2, (tuned, replays)
