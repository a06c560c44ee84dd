"""GPU parity of solution counting (-m gpu).

P:245: "as a byproduct, and without additional overhead, BE can compute the
number of consistent solutions".  Plans built with "count" run the counting
bucket kernel (bk_count: the (min, count) semiring over bk_generic's tiling)
and are compared with the oracle's or_solve_count on the same seeded inputs:

* the cost tables and argmins are those of plain BE (bit-exact, both
  semirings share them);
* the count tables and the final counts are bit-exact: both sides multiply
  the member counts in member order and add the minimisers' counts in
  ascending v, in float64 (exact integers below 2^53, the same rounding
  above);
* "consistent" counts the assignments of finite cost (optimum 0 / INF).
"""
import numpy as np
import pytest

import gen
import oracle
import paper_1608_05288_b200 as G
from gen import configs

pytestmark = pytest.mark.gpu

INF = oracle.INF_I32


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    torch.cuda.set_device(0)
    return torch


def check(inst, mode, order=None, tables=True):
    P = G.Problem.from_instance(inst)
    if order is None:
        order, _ = P.order()
    plan = G.Plan(P, order, count=mode, retain="all" if tables else "args")
    run, root = plan.dpop_util()
    ref = oracle.solve_count(inst, order, mode, keep_tables=tables)
    assert root == ref.value, (root, ref.value)
    assert run.count() == ref.count, (run.count(), ref.count)
    if tables:
        info = plan.info()
        for t, (ti, ot) in enumerate(zip(info["tables"], ref.tables)):
            out, arg = run.table(t, ti["rows"])
            np.testing.assert_array_equal(out, ot.out, err_msg=f"table {t} values")
            np.testing.assert_array_equal(arg, ot.arg, err_msg=f"table {t} argmins")
            np.testing.assert_array_equal(run.count_table(t, ti["rows"]), ot.count, err_msg=f"table {t} counts")
    run.close()
    # one-shot solve (the second solve of a plan replays the CUDA graph)
    for _ in range(2):
        v, c = plan.solve_count()
        assert v == ref.value and c == ref.count
    return ref


@pytest.mark.parametrize("seed", range(24))
def test_count_random_int(torch_cuda, seed):
    """int32 problems with ties (cost ranges 1, 2, 100) and forbidden cells."""
    rng = np.random.default_rng(500 + seed)
    n = int(rng.integers(8, 16))
    d = int(rng.integers(2, 5))
    p2 = [0.0, 0.2, 0.5][seed % 3]
    cmax = [1, 2, 100][(seed // 3) % 3]
    inst = gen.random_network(n, d, d, int(rng.integers(n, 2 * n)), 1, 3, cmax, p2, seed)
    for mode in ("optimal", "consistent"):
        check(inst, mode)


@pytest.mark.parametrize("seed", range(4))
def test_count_f64(torch_cuda, seed):
    """float64 (-log p) problems, with 0-probability cells."""
    inst = gen.random_network_f64(12, 2, 4, 18, 1, 3, 4.0, 0.25, seed)
    for mode in ("optimal", "consistent"):
        check(inst, mode)


def test_count_against_brute_force(torch_cuda):
    """The GPU counts equal enumeration directly (not only the oracle)."""
    from oracle.brute import count_solutions
    for seed in range(5):
        inst = gen.random_network(8, 3, 3, 12, 1, 3, 2, 0.3, 70 + seed)
        opt, n_opt, n_cons = count_solutions(inst)
        P = G.Problem.from_instance(inst)
        order, _ = P.order()
        assert G.Plan(P, order, count="optimal").solve_count() == (opt, n_opt)
        assert G.Plan(P, order, count="consistent").solve_count()[1] == n_cons


def test_count_scalefree_tiled_sizes(torch_cuda):
    """A scale-free DCOP with 1.4e7-row buckets (several tiles per launch,
    ragged tails): every table, argmin and count equals the oracle's."""
    inst = gen.scalefree(120, 3, 0.0, 2)
    check(inst, "optimal")


def test_count_c2_full_size(torch_cuda):
    """C2 (n=100, d=5, w*=10, largest table 9.8e6 rows): the counts equal the
    oracle's; the consistent count of an INF-free problem is prod d = 5^100
    (float64, the same products in the same order on both sides)."""
    inst = configs.c2()
    ref = check(inst, "optimal", tables=False)
    assert ref.count >= 1
    P = G.Problem.from_instance(inst)
    order, _ = P.order()
    v, c = G.Plan(P, order, count="consistent").solve_count()
    assert v == 0 and c == oracle.solve_count(inst, order, "consistent", keep_tables=False).count
    assert abs(c - 5.0 ** 100) <= 1e-12 * 5.0 ** 100
