"""Argmin tables in host memory ("retain":"host", the
argmin spill; -m gpu).

Each bucket runs in row chunks; the chunk's argmins go to a 2-slot device
ring and are copied to mapped pinned host memory on a second stream while
the next chunk computes (Fig. 8's host/device concurrency); the
value phase reads them in place.  Small chunks (host_arg_chunk) force many
chunks per bucket, including tiled-kernel chunks of whole tiles and ragged
final chunks.  Parity: optimum, assignment, every value table and every
argmin table equal the oracle's (bit-exact) and the device-argmin run's.
"""
import numpy as np
import pytest

import gen
import oracle
import paper_1608_05288_b200 as G
from gen import configs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    torch.cuda.set_device(0)
    return torch


@pytest.mark.parametrize("case", ["scalefree", "inf", "f64"])
@pytest.mark.parametrize("chunk", [4096, 1 << 20])
def test_host_args_parity(torch_cuda, case, chunk):
    if case == "scalefree":
        inst = gen.scalefree(90, 3, 0.0, 4)
    elif case == "inf":
        inst = gen.scalefree(70, 3, 0.2, 5)
    else:
        inst = gen.random_network_f64(40, 2, 3, 70, 1, 3, 4.0, 0.1, 6)
    P = G.Problem.from_instance(inst)
    order, _ = P.order()
    ref = oracle.solve_be(inst, order)
    plan = G.Plan(P, order, retain="host", host_arg_chunk=chunk)
    info = plan.info()
    for _ in range(2):  # the second solve reuses the plan's ring and host tables
        opt, a = plan.solve_be()
        assert opt == ref.value
        assert list(a) == list(ref.assignment)
    run, root = plan.dpop_util()
    assert root == ref.value and list(run.value()) == list(ref.assignment)
    for t, (ti, ot) in enumerate(zip(info["tables"], ref.tables)):
        _, arg = run.table(t, ti["rows"], want_out=False)
        np.testing.assert_array_equal(arg, ot.arg, err_msg=f"argmins of table {t}")
    run.close()


def test_host_args_c2_full_size(torch_cuda):
    """C2 at full size (largest table 9.8e6 rows) in 1e6-row chunks: the
    assignment equals the golden one of the device-argmin path."""
    inst = configs.c2()
    P = G.Problem.from_instance(inst)
    order, _ = P.order()
    o1, a1 = G.Plan(P, order).solve_be()
    o2, a2 = G.Plan(P, order, retain="host", host_arg_chunk=1 << 20).solve_be()
    assert o1 == o2 and list(a1) == list(a2)
