"""Run tiles of the tiled kernel (opt-in: GBE_FAST_HTILE=1; -m gpu): a bucket whose largest input
lacks a high output digit h gets tiles with h on top of the low digits
(g1 = h: the register blocks span h's values, so that input is loaded once
for all of them; the tile's output rows are radix(h) runs), with the bucket's
merged tables laid out so h sits right above the tile's low digits.
Every table, argmin, optimum and assignment against the oracle (int32
INF-free / with INF, f64), and C4's largest bucket takes such a tile.
(Opt-in: measured slower on C4.)"""
import os

import numpy as np
import pytest

import gen
import oracle
import paper_1608_05288_b200 as G
from tests.test_gpu_fullsize import _f64_tables_against_oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    torch.cuda.set_device(0)
    os.environ["GBE_FAST_HTILE"] = "1"  # read per plan / descriptor build
    yield torch
    del os.environ["GBE_FAST_HTILE"]


CASES = [("sf", 110, 3, 0.0, s) for s in (1, 2, 3, 4, 5, 6)] + [("sf", 90, 3, 0.1, 7), ("sf", 80, 4, 0.0, 8),
                                                                  ("bn", 60, 2, 4, 1), ("bn", 70, 2, 4, 3)]


@pytest.mark.parametrize("case", CASES, ids=[f"{c[0]}{c[1]}_{c[-1]}" for c in CASES])
def test_run_tiles_parity(torch_cuda, case):
    kind = case[0]
    inst = gen.scalefree(case[1], case[2], case[3], case[4]) if kind == "sf" else \
        gen.belief_net(case[1], case[2], case[3], 3, 12, case[4])
    P = G.Problem.from_instance(inst)
    order, _ = P.order()
    plan = G.Plan(P, order, retain="all", timing=True)
    for _ in range(5):  # past the autotuning solves
        r, _root = plan.dpop_util()
        r.close()
    run, root = plan.dpop_util()
    st = run.stats()
    info = plan.info()
    orun = oracle.solve_be(inst, order)
    if inst.is_f64:
        assert abs(root - orun.value) <= 1e-9 * max(1.0, abs(orun.value))
        _f64_tables_against_oracle(inst, order, -1, run, info, orun)
    else:
        assert root == orun.value
        for t, (ti, ot) in enumerate(zip(info["tables"], orun.tables)):
            out, arg = run.table(t, ti["rows"])
            np.testing.assert_array_equal(out, ot.out, err_msg=f"table {t}")
            np.testing.assert_array_equal(arg, ot.arg, err_msg=f"argmins {t}")
        assert list(run.value()) == list(orun.assignment)
    run.close()
    ht = [t for t in st["tasks"] if t.get("htile", -1) >= 0]
    print(f"{case}: {len(ht)} run-tile buckets of {len(st['tasks'])}")


def test_c4_largest_bucket_takes_a_run_tile(torch_cuda):
    from gen import configs
    P = G.Problem.from_instance(configs.c4())
    order, _ = P.order()
    plan = G.Plan(P, order, timing=True)
    for _ in range(5):
        plan.solve_be()
    _, _, st = plan.solve_be(stats=True)
    x57 = [t for t in st["tasks"] if t["var"] == 57][0]
    # the autotuner may keep the streaming kernel for it; the tiled kernel's
    # descriptor must still be the run tile
    assert x57.get("htile", -1) >= 0 or x57["variant"] == 2, x57
