"""World-size-2 tests of the row-sharded path.

-m "not gpu": two gloo processes on CPU build the per-rank plans of C4 and
check, over the process group, that every sharded bucket's row ranges tile
its rows exactly once, block-aligned, with identical structure on both ranks.

-m gpu: two gloo processes share ONE GPU (host-staged all-gather hook) and run
a sharded DPOP; every rank's local rows of every table, the optimum and the
assignment must equal the single-GPU run bit for bit.
"""
import json
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _plan_worker(rank, world, port, out_path):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    import paper_1608_05288_b200 as G
    from gen import configs
    from paper_1608_05288_b200 import dist as gdist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    P = G.Problem.from_instance(configs.c4())
    order, _ = P.order()
    info = G.Plan(P, order, world_size=world, rank=rank, shard_min_rows=1 << 20).info()
    got = [None] * world
    dist.all_gather_object(got, info)
    t = gdist.max_over_ranks(float(rank + 1), dist.group.WORLD)
    if rank == 0:
        with open(out_path, "w") as fh:
            json.dump({"infos": got, "max": t}, fh)
    dist.barrier()
    dist.destroy_process_group()


def test_shard_plan_world2_gloo(tmp_path):
    port = _free_port()
    out = str(tmp_path / "plans.json")
    mp.start_processes(_plan_worker, args=(2, port, out), nprocs=2, start_method="spawn")
    res = json.load(open(out))
    a, b = res["infos"]
    assert res["max"] == 2.0  # max over ranks (the bench's timing reduction)
    assert len(a["tables"]) == len(b["tables"])
    nshard = 0
    for ta, tb in zip(a["tables"], b["tables"]):
        assert ta["sep"] == tb["sep"] and ta["members"] == tb["members"] and ta["rows"] == tb["rows"]
        sa, sb = ta["shard"], tb["shard"]
        assert sa["on"] == sb["on"] and sa["gather"] == sb["gather"] and sa["key_digits"] == sb["key_digits"]
        if not sa["on"]:
            assert (sa["lo"], sa["hi"]) == (0, ta["rows"]) == (sb["lo"], sb["hi"])
            continue
        nshard += 1
        # disjoint, covering, block aligned
        assert sa["lo"] == 0 and sa["hi"] == sb["lo"] and sb["hi"] == ta["rows"]
        block = ta["rows"] // sa["blocks"]
        assert sa["hi"] % block == 0
        # the row-shard contract of the tiled kernel: ranges are whole tiles
        if ta["kernel"]["variant"] == 1:
            assert sa["hi"] % ta["kernel"]["PL"] == 0
    assert nshard >= 5
    # at least one message stays sharded into its consumer (no all-gather)
    assert any(t["shard"]["on"] and not t["shard"]["gather"] for t in a["tables"])


def _gpu_worker(rank, world, port, out_dir):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    import gen
    import paper_1608_05288_b200 as G
    from paper_1608_05288_b200 import dist as gdist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    gdist.install(0, "gloo")
    inst = gen.scalefree(90, 3, 0.0, 4)
    P = G.Problem.from_instance(inst)
    order, _ = P.order()
    plan = G.Plan(P, order, world_size=world, rank=rank, shard_min_rows=2000, retain="all")
    info = plan.info()
    run, root = plan.dpop_util()
    assign = run.value()
    tabs = {}
    for t, ti in enumerate(info["tables"]):
        lo, hi = ti["shard"]["lo"], ti["shard"]["hi"]
        out, arg = run.table(t, hi - lo)
        tabs[t] = (lo, hi, out, arg)
    run.close()
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), root=root, assign=assign,
             **{f"o{t}": v[2] for t, v in tabs.items()}, **{f"a{t}": v[3] for t, v in tabs.items()},
             lohi=np.array([[v[0], v[1]] for t, v in sorted(tabs.items())]))
    gdist.uninstall()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_sharded_dpop_two_ranks_one_gpu(tmp_path):
    import gen
    import paper_1608_05288_b200 as G
    port = _free_port()
    mp.start_processes(_gpu_worker, args=(2, port, str(tmp_path)), nprocs=2, start_method="spawn")
    inst = gen.scalefree(90, 3, 0.0, 4)
    P = G.Problem.from_instance(inst)
    order, _ = P.order()
    plan = G.Plan(P, order, retain="all")
    info = plan.info()
    run, root = plan.dpop_util()
    assign = run.value()
    full = [run.table(t, ti["rows"]) for t, ti in enumerate(info["tables"])]
    run.close()
    sharded = 0
    for r in range(2):
        z = np.load(tmp_path / f"rank{r}.npz")
        assert int(z["root"]) == root
        assert list(z["assign"]) == list(assign)
        for t, (lo, hi) in enumerate(z["lohi"]):
            if hi - lo < info["tables"][t]["rows"]:
                sharded += 1
            np.testing.assert_array_equal(z[f"o{t}"], full[t][0][lo:hi], err_msg=f"rank {r} table {t}")
            np.testing.assert_array_equal(z[f"a{t}"], full[t][1][lo:hi], err_msg=f"rank {r} argmin {t}")
    assert sharded >= 4


@pytest.mark.gpu
def test_builtin_nccl_communicator_single_rank():
    """The built-in NCCL transport loads (dlopen libnccl.so.2), creates a
    communicator and tears it down (1 rank; the multi-GPU data path runs in
    the driver's scaling step)."""
    import paper_1608_05288_b200 as G
    uid = G.comm_nccl_id()
    assert len(uid) == 128
    G.comm_nccl_init(uid, 1, 0, 0)
    G.comm_finalize()


def _c4_worker(rank, world, port, out_dir):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    import paper_1608_05288_b200 as G
    from gen import configs
    from paper_1608_05288_b200 import dist as gdist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    gdist.install(0, "gloo")
    P = G.Problem.from_instance(configs.c4())
    order, _ = P.order()
    plan = G.Plan(P, order, world_size=world, rank=rank)  # bench.py's launch configuration
    info = plan.info()
    run, root = plan.dpop_util()
    assign = run.value()
    run.close()
    np.savez(os.path.join(out_dir, f"c4rank{rank}.npz"), root=root, assign=assign,
             nshard=sum(1 for t in info["tables"] if t["shard"]["on"]))
    del plan
    gdist.uninstall()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_c4_sharded_two_ranks_one_gpu(tmp_path):
    """The bench workload (C4, largest UTIL table 3^20 rows) row-sharded over 2
    ranks (sharing one GPU, host-staged all-gather): optimum and assignment
    equal the oracle's golden optimum and the 1-GPU assignment."""
    import json

    import paper_1608_05288_b200 as G
    from gen import configs
    port = _free_port()
    mp.start_processes(_c4_worker, args=(2, port, str(tmp_path)), nprocs=2, start_method="spawn")
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "c4.json")))
    P = G.Problem.from_instance(configs.c4())
    order, _ = P.order()
    opt, assign = G.Plan(P, order).solve_be()
    for r in range(2):
        z = np.load(tmp_path / f"c4rank{r}.npz")
        assert int(z["root"]) == g["value"] == opt
        assert list(z["assign"]) == list(assign)
        assert int(z["nshard"]) >= 5


def _nccl_worker(rank, world, port, out_dir):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(world), RANK=str(rank))
    import torch

    import paper_1608_05288_b200 as G
    from gen import configs
    from paper_1608_05288_b200 import dist as gdist
    torch.cuda.set_device(rank)
    pg = gdist.init(rank, "nccl")  # built-in NCCL communicator (bench.py's path)
    P = G.Problem.from_instance(configs.c4())
    order, _ = P.order()
    plan = G.Plan(P, order, device=rank, world_size=world, rank=rank)
    roots = []
    for _ in range(3):  # warm-up run, graph capture, replay
        run, root = plan.dpop_util()
        assign = run.value()
        run.close()
        roots.append(root)
    np.savez(os.path.join(out_dir, f"nccl{rank}.npz"), roots=np.array(roots), assign=assign)
    del plan
    gdist.finish(pg)


@pytest.mark.gpu
def test_c4_sharded_builtin_nccl_two_gpus(tmp_path):
    """Row-sharded C4 over 2 GPUs with the built-in NCCL all-gather inside
    the captured UTIL graph (the bench's --gpus 2 path): every run's optimum
    equals the oracle's golden value and the assignment the 1-GPU one."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    import paper_1608_05288_b200 as G
    from gen import configs
    port = _free_port()
    mp.start_processes(_nccl_worker, args=(2, port, str(tmp_path)), nprocs=2, start_method="spawn")
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "c4.json")))
    P = G.Problem.from_instance(configs.c4())
    order, _ = P.order()
    opt, assign = G.Plan(P, order).solve_be()
    for r in range(2):
        z = np.load(tmp_path / f"nccl{r}.npz")
        assert all(int(x) == g["value"] == opt for x in z["roots"])
        assert list(z["assign"]) == list(assign)
