"""GPU parity of the sum-product semiring (-m gpu).

The same bucket kernels with -log sum_v exp(-s_v) elimination
(GBE_SUMPROD_F64), compared with the oracle's or_bucket_rows_sp /
or_solve_sumprod on the same seeded inputs, plus properties that hold at any
size (a belief network's Z = 1; evidence on x0, x1 gives two CPT entries).

Tolerance: |gpu - oracle| <= 1e-9 * (1 + |oracle|), infinities at the same
places (DESIGN.md §3 A18: values may be negative or ~0, so a purely relative
bar is meaningless near 0; the kernels sum members in another order and
use an online log-sum-exp in the generic kernel).
"""
import math

import numpy as np
import pytest

import gen
import oracle
import paper_1608_05288_b200 as G
from gen import configs

from tests.test_gpu_parity import FAST_SHAPES, desc_for, random_bucket, uniform_bucket

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    return torch


def close(got, exp, tol=1e-9):
    got = np.asarray(got, dtype=np.float64)
    exp = np.asarray(exp, dtype=np.float64)
    np.testing.assert_array_equal(np.isinf(got), np.isinf(exp))
    fin = np.isfinite(exp)
    err = np.abs(got[fin] - exp[fin]) / (1 + np.abs(exp[fin]))
    assert err.size == 0 or err.max() <= tol, f"max scaled error {err.max():.3g}"


def run_sp(torch, dom, sep, x, members, rb, re, variant=-1):
    D, rows = desc_for(dom, sep, x, members, True)
    D.semiring = G.SUMPROD_F64
    ins = [torch.tensor(np.asarray(t), dtype=torch.float64, device="cuda") for _, t in members]
    n = max(re - rb, 1)
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    arg = torch.full((n,), 77, dtype=torch.uint8, device="cuda")
    G.bucket_kernel(D, ins, out, arg, rb, re, variant=variant)
    torch.cuda.synchronize()
    return D, out.cpu().numpy()[:re - rb], arg.cpu().numpy()[:re - rb]


# ---------------------------------------------------------------- primitive

@pytest.mark.parametrize("seed", range(24))
def test_sumprod_bucket_random_descriptors(torch_cuda, seed):
    """Random descriptors (generic kernel; tiled when the shape fits)."""
    rng = np.random.default_rng(9100 + seed)
    dom, sep, x, members = random_bucket(rng, f64=True, big=seed % 3 == 0, max_m=8)
    if seed % 4 == 1:  # negative values too (messages of a sum-product run are)
        members = [(s, t - 5.0) for s, t in members]
    rows = int(np.prod([dom[v] for v in sep])) if sep else 1
    exp = oracle.bucket_eval_sp(dom, x, members, sep)
    _, got, arg = run_sp(torch_cuda, dom, sep, x, members, 0, rows)
    close(got, exp)
    assert not arg.any()


@pytest.mark.parametrize("R,DV", [s for s in FAST_SHAPES if not (s[0] == 5 and s[1] == 5)])
def test_sumprod_fast_kernel_shapes(torch_cuda, R, DV):
    rng = np.random.default_rng(R * 1000 + DV)
    m = {2: 13, 3: 9, 4: 7, 5: 6}[R]
    for trial in range(2):
        k = int(rng.integers(1, 12))
        dom, sep, x, members = uniform_bucket(rng, R, DV, m, k, True)
        D, rows = desc_for(dom, sep, x, members, True)
        D.semiring = G.SUMPROD_F64
        assert G.bucket_kernel_variant(D, 0, rows) == 2  # auto: f64 streams
        exp = oracle.bucket_eval_sp(dom, x, members, sep)
        for var in (1, 2):  # the tiled and the streaming kernel, explicitly
            _, got, arg = run_sp(torch_cuda, dom, sep, x, members, 0, rows, variant=var)
            close(got, exp)
            assert not arg.any()


def test_sumprod_edge_cases(torch_cuda):
    """All-infinite rows stay +inf; d = 1 is the identity on the sum; no
    members gives -log d for every row; a partial row range."""
    dom = [3, 4, 6]
    t = np.random.default_rng(1).uniform(0, 9, 72)
    t[:6] = np.inf
    _, got, _ = run_sp(torch_cuda, dom, [0, 1], 2, [([0, 1, 2], t)], 0, 12)
    assert math.isinf(got[0]) and got[0] > 0
    close(got, oracle.bucket_eval_sp(dom, 2, [([0, 1, 2], t)], [0, 1]))
    _, got, _ = run_sp(torch_cuda, [5, 1], [0], 1, [([0, 1], np.arange(5.0))], 0, 5)
    np.testing.assert_array_equal(got, np.arange(5.0))
    _, got, _ = run_sp(torch_cuda, [2, 7], [0], 1, [], 0, 2)
    close(got, [-math.log(7)] * 2, 1e-15)
    _, got, _ = run_sp(torch_cuda, dom, [0, 1], 2, [([0, 1, 2], t)], 5, 11)
    close(got, oracle.bucket_eval_sp(dom, 2, [([0, 1, 2], t)], [0, 1], 5, 11))


# ---------------------------------------------------------------- solves

SP_INSTANCES = {
    "bn": lambda: gen.belief_net(40, 2, 4, 3, 8, 1),
    "netf": lambda: gen.random_network_f64(14, 2, 5, 20, 1, 3, 10.0, 0.1, 2),
    "netf_big": lambda: gen.random_network_f64(40, 2, 3, 70, 2, 3, 4.0, 0.05, 7),
    "netf_d6": lambda: gen.random_network_f64(16, 6, 6, 24, 2, 2, 3.0, 0.0, 3),
}


@pytest.mark.parametrize("name", sorted(SP_INSTANCES))
def test_sumprod_solve_matches_oracle(torch_cuda, name):
    """Every table (retain all) and -log Z against the oracle; graph replays
    agree; the value-only default plan agrees."""
    inst = SP_INSTANCES[name]()
    P = G.Problem.from_instance(inst)
    order, _ = P.order()
    orun = oracle.solve_sumprod(inst, order)
    plan = G.Plan(P, order, retain="all", semiring="sumprod")
    info = plan.info()
    for rep in range(3):
        run, root = plan.dpop_util()
        close([root], [orun.value])
        if rep in (0, 2):
            for t, (ti, ot) in enumerate(zip(info["tables"], orun.tables)):
                out, arg = run.table(t, ti["rows"])
                close(out, ot.out)
                assert not arg.any()
        run.close()
    plan = G.Plan(P, order, semiring="sumprod")
    for rep in range(3):
        close([-plan.log_z()], [orun.value])


def test_sumprod_brute_force_small(torch_cuda):
    from oracle.brute import neg_log_z
    for seed in range(4):
        inst = gen.random_network_f64(8, 2, 3, 12, 1, 3, 4.0, 0.3 if seed >= 2 else 0.0, seed)
        P = G.Problem.from_instance(inst)
        order, _ = P.order()
        close([-G.Plan(P, order, semiring="sumprod").log_z()], [neg_log_z(inst)], 1e-12)


def _with_evidence(bn, ev):
    funcs = [(list(bn.scope(f)), bn.table(f)) for f in range(bn.nf)]
    for v, e in ev.items():
        t = np.full(int(bn.dom[v]), np.inf)
        t[e] = 0.0
        funcs.append(([v], t))
    return gen.Instance.from_functions(bn.dom, funcs, is_f64=True)


def test_sumprod_c5_full_size_properties(torch_cuda):
    """C5 (the MPE belief network at full size): Z = 1 without evidence; with
    evidence x0 = e0, x1 = e1, -log P(E) = the two CPT entries (closed forms,
    so no oracle run is needed at this size)."""
    bn = configs.c5()
    P = G.Problem.from_instance(bn)
    order, _ = P.order()
    assert abs(G.Plan(P, order, semiring="sumprod").log_z()) < 1e-9
    f0 = [f for f in range(bn.nf) if list(bn.scope(f)) == [0]]
    f1 = [f for f in range(bn.nf) if list(bn.scope(f)) == [0, 1]]
    assert len(f0) == 1 and len(f1) == 1
    t1 = bn.table(f1[0]).reshape(int(bn.dom[0]), int(bn.dom[1]))
    e0, e1 = int(bn.dom[0]) - 1, 0
    inst = _with_evidence(bn, {0: e0, 1: e1})
    P2 = G.Problem.from_instance(inst)
    o2, _ = P2.order()
    expect = float(bn.table(f0[0])[e0]) + float(t1[e0, e1])
    close([-G.Plan(P2, o2, semiring="sumprod").log_z()], [expect])


def test_sumprod_errors(torch_cuda):
    inst = SP_INSTANCES["netf"]()
    P = G.Problem.from_instance(inst)
    order, _ = P.order()
    with pytest.raises(G.GbeError):
        G.Plan(P, order, 3, semiring="sumprod")  # exact BE only
    with pytest.raises(G.GbeError):
        G.Plan(P, order, semiring="maxprod")
    plan = G.Plan(P, order, semiring="sumprod")
    with pytest.raises(G.GbeError):
        plan.solve_be()  # no assignment in the sum-product semiring
    run, _ = plan.dpop_util()
    with pytest.raises(G.GbeError):
        run.value()
    run.close()
    Pi = G.Problem.from_instance(gen.random_graph(10, 3, 20, 0, 0.0, 1))
    oi, _ = Pi.order()
    with pytest.raises(G.GbeError):
        G.Plan(Pi, oi, semiring="sumprod")  # int32 costs are not -log values
