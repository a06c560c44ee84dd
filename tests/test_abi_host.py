"""Host-side checks of libgbe (-m "not gpu"): the library loads, exports every
symbol include/gbe.h declares, and its host logic (orderings, induced width,
pseudo-tree, bucket plan, mini-bucket partition, loaders, evaluate, shard
plan) agrees with the independent oracle.  No kernel is launched here."""
import os
import re

import numpy as np
import pytest

import gen
import oracle
import paper_1608_05288_b200 as G
from gen import configs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_every_declared_symbol_is_exported():
    hdr = open(os.path.join(ROOT, "include", "gbe.h")).read()
    declared = set(re.findall(r"\b(gbe_[a-z_0-9]+)\s*\(", hdr))
    declared -= {"gbe_bucket_desc"}
    L = G.lib()
    missing = [s for s in sorted(declared) if not hasattr(L, s)]
    assert not missing, missing
    assert set(G.gbe.EXPORTED) <= declared


def test_solve_without_device_fails_loudly():
    """No CPU fallback: a solve on a box without a GPU must raise."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    inst = gen.random_graph(6, 2, 7, 0, 0.0, 1)
    P = G.Problem.from_instance(inst)
    plan = G.Plan(P, P.order()[0])
    with pytest.raises(G.GbeError) as e:
        plan.solve_be()
    assert e.value.status == 4


@pytest.mark.parametrize("seed", range(8))
def test_orderings_and_width_match_oracle(seed):
    inst = gen.scalefree(40, 3, 0.0, seed) if seed % 2 else gen.random_graph(30, 3, 60, 0, 0.0, seed)
    P = G.Problem.from_instance(inst)
    o, w = P.order(G.ORDER_MINFILL)
    assert list(o) == list(oracle.minfill_order(inst))
    assert w == oracle.induced_width(inst, o)
    o2, w2 = P.order(G.ORDER_PAPER_DEGREE)
    assert list(o2) == list(oracle.degree_order(inst))
    assert w2 == oracle.induced_width(inst, o2)
    par, ss = P.pseudotree(o)
    assert list(par) == list(oracle.elim_tree(inst, o))


def _same_structure(plan_info, run):
    tabs = plan_info["tables"]
    assert len(tabs) == len(run.tables)
    for a, b in zip(tabs, run.tables):
        assert a["var"] == b.var and a["mb"] == b.mb and a["rows"] == b.rows
        assert a["sep"] == [int(v) for v in b.sep]
        assert [tuple(m) for m in a["members"]] == list(b.members)
        assert a["dest"] == b.dest


@pytest.mark.parametrize("seed", range(6))
def test_be_plan_matches_oracle_buckets(seed):
    inst = gen.random_network(14, 2, 4, 18, 1, 3, 100, 0.2, seed)
    P = G.Problem.from_instance(inst)
    o, _ = P.order()
    _same_structure(G.Plan(P, o).info(), oracle.solve_be(inst, o))


@pytest.mark.parametrize("ib", [1, 2, 3, 4, 6])
def test_mbe_partition_matches_oracle(ib):
    inst = gen.random_graph(16, 3, 40, 0, 0.0, ib)
    P = G.Problem.from_instance(inst)
    o, _ = P.order()
    _same_structure(G.Plan(P, o, ib).info(), oracle.solve_mbe(inst, o, ib))


def test_example4_partition_through_the_abi():
    """Example 4, z = 1: B4 splits into three singletons."""
    inst = gen.Instance.from_functions([2] * 4, [((0, 1), [1, 2, 3, 4]), ((0, 3), [1, 2, 3, 4]),
                                                 ((1, 2), [1, 2, 3, 4]), ((1, 3), [1, 2, 3, 4]),
                                                 ((2, 3), [1, 2, 3, 4])])
    info = G.Plan(G.Problem.from_instance(inst), [0, 1, 2, 3], 1).info()
    b4 = [t for t in info["tables"] if t["var"] == 3]
    assert [t["members"] for t in b4] == [[[0, 1]], [[0, 3]], [[0, 4]]]
    with pytest.raises(G.GbeError) as e:
        G.Plan(G.Problem.from_instance(inst), [0, 1, 2, 3], 0)
    assert e.value.status == 1


def test_invalid_inputs_rejected():
    with pytest.raises(G.GbeError):
        G.Problem.create([2, 2], [2], [0, 0], [0, 0, 0, 0])  # duplicate scope var
    with pytest.raises(G.GbeError):
        G.Problem.create([2, 300], [1], [1], [0] * 300)  # domain > 256
    with pytest.raises(G.GbeError):
        G.Problem.create([2], [1], [0], [-1, 0])  # negative cost
    p = G.Problem.create([2, 2], [2], [0, 1], [0, 1, 2, 3])
    with pytest.raises(G.GbeError):
        G.Plan(p, [0, 0])  # not a permutation
    with pytest.raises(G.GbeError):
        G.Plan(p, [0, 1], -1, retain="sometimes")


def test_budget_error_names_the_bucket():
    """a plan that exceeds the memory budget is refused up front."""
    inst = configs.c4()
    P = G.Problem.from_instance(inst)
    o, w = P.order()
    with pytest.raises(G.GbeError) as e:
        G.Plan(P, o, budget_bytes=1 << 30)
    assert e.value.status == 3 and "rows" in str(e.value) and "bucket x" in str(e.value)


@pytest.mark.parametrize("seed", range(4))
def test_evaluate_matches_oracle(seed):
    for inst in (gen.random_network(10, 2, 4, 12, 0, 3, 100, 0.3, seed),
                 gen.belief_net(12, 2, 4, 3, 5, seed)):
        P = G.Problem.from_instance(inst)
        rng = np.random.default_rng(seed)
        for _ in range(5):
            a = np.array([rng.integers(d) for d in inst.dom], dtype=np.int32)
            assert P.evaluate(a) == oracle.evaluate(inst, a)


def test_wcsp_roundtrip(tmp_path):
    inst = gen.random_network(9, 2, 4, 11, 0, 3, 100, 0.3, 5)
    path = str(tmp_path / "x.wcsp")
    gen.write_wcsp(inst, path)
    P = G.Problem.load_wcsp(path)
    rng = np.random.default_rng(0)
    for _ in range(20):
        a = np.array([rng.integers(d) for d in inst.dom], dtype=np.int32)
        assert P.evaluate(a) == oracle.evaluate(inst, a)


def test_wcsp_parse_error_has_line(tmp_path):
    path = tmp_path / "bad.wcsp"
    path.write_text("x 2 2 1 1000\n2 2\n2 0 1 0 2\n0 0 5\n0 1\n")
    with pytest.raises(G.GbeError) as e:
        G.Problem.load_wcsp(str(path))
    assert e.value.status == 2 and "line 5" in str(e.value)


def test_uai_roundtrip_and_evidence(tmp_path):
    inst = gen.belief_net(8, 2, 3, 2, 4, 3)
    path = str(tmp_path / "x.uai")
    gen.write_uai(inst, path)
    P = G.Problem.load_uai(path)
    a = np.zeros(8, np.int32)
    assert P.evaluate(a) == pytest.approx(oracle.evaluate(inst, a), rel=1e-12)
    ev = tmp_path / "x.evid"
    ev.write_text("1 3 1\n")
    Pe = G.Problem.load_uai(path, str(ev))
    a[3] = 0
    assert Pe.evaluate(a) == float("inf")
    a[3] = 1
    assert Pe.evaluate(a) == pytest.approx(oracle.evaluate(inst, a), rel=1e-12)
    ev.write_text("1 3 7\n")
    with pytest.raises(G.GbeError) as e:
        G.Problem.load_uai(path, str(ev))
    assert e.value.status == 1


def test_generate_matches_gen_module():
    """gbe_generate uses the same seeded generator module as gen/."""
    P = G.Problem.generate(topology="scalefree", n=50, d=3, seed=4)
    inst = gen.scalefree(50, 3, 0.0, 4)
    rng = np.random.default_rng(1)
    for _ in range(10):
        a = np.array([rng.integers(3) for _ in range(50)], dtype=np.int32)
        assert P.evaluate(a) == oracle.evaluate(inst, a)


def test_c4_plan_shape():
    """BASELINE C4 (BA n=200, d=3, w*=20): largest UTIL table 3^20 rows."""
    P = G.Problem.from_instance(configs.c4())
    o, w = P.order()
    assert w == 20
    info = G.Plan(P, o).info()
    assert max(t["rows"] for t in info["tables"]) == 3 ** 20
    assert info["total_cells"] == sum(t["rows"] * t["d"] for t in info["tables"])


def test_sumprod_plan_validation_host():
    """"semiring":"sumprod" is validated at plan time (host only): float64
    problems, exact BE; unknown semirings are rejected."""
    fi = gen.random_network_f64(12, 2, 3, 18, 1, 3, 4.0, 0.0, 1)
    P = G.Problem.from_instance(fi)
    order, _ = P.order()
    G.Plan(P, order, semiring="sumprod").info()
    with pytest.raises(G.GbeError):
        G.Plan(P, order, 2, semiring="sumprod")
    with pytest.raises(G.GbeError):
        G.Plan(P, order, semiring="logsum")
    Pi = G.Problem.from_instance(gen.random_graph(10, 3, 20, 0, 0.0, 1))
    oi, _ = Pi.order()
    with pytest.raises(G.GbeError):
        G.Plan(Pi, oi, semiring="sumprod")


def test_count_plan_errors():
    """Counting plans are exact BE, one rank, min-sum:
    the planner rejects the rest on the host (GBE_E_INVALID), and a plan
    without "count" cannot be counted."""
    inst = gen.random_network(6, 2, 2, 6, 1, 2, 5, 0.0, 1)
    P = G.Problem.from_instance(inst)
    order, _ = P.order()
    for kw in (dict(count="sometimes"), dict(count="optimal", world_size=2, rank=0)):
        with pytest.raises(G.GbeError):
            G.Plan(P, order, **kw)
    with pytest.raises(G.GbeError):
        G.Plan(P, order, 2, count="optimal")  # MBE: exact BE only
    with pytest.raises(G.GbeError):
        G.Plan(P, order).solve_count()        # plan without "count"
    fp = G.Problem.from_instance(gen.random_network_f64(6, 2, 2, 6, 1, 2, 3.0, 0.0, 1))
    with pytest.raises(G.GbeError):
        G.Plan(fp, order, count="optimal", semiring="sumprod")


def test_host_args_plan_errors():
    """"retain":"host" (argmin spill) is exact BE/DPOP on
    one rank in the min-sum semiring; the planner rejects the rest."""
    inst = gen.random_network(6, 2, 2, 6, 1, 2, 5, 0.0, 1)
    P = G.Problem.from_instance(inst)
    order, _ = P.order()
    G.Plan(P, order, retain="host", host_arg_chunk=64)  # valid
    for args, kw in (((2,), dict(retain="host")),
                     ((), dict(retain="host", world_size=2, rank=0)),
                     ((), dict(retain="host", count="optimal")),
                     ((), dict(retain="host", host_arg_chunk=0))):
        with pytest.raises(G.GbeError):
            G.Plan(P, order, *args, **kw)


def _desc(radix, d, strides, semiring=0):
    D = G.BucketDesc()
    D.semiring = semiring
    D.nsep = len(radix)
    D.d = d
    D.ninputs = len(strides)
    D.rows = int(np.prod(radix, dtype=np.int64)) if radix else 1
    for q, r in enumerate(radix):
        D.radix[q] = r
    for j, st in enumerate(strides):
        for q, s in enumerate(st):
            D.stride[j][q] = s
    return D


def test_tiled_kernel_requires_contiguous_tile_slices():
    """bkf_build takes a descriptor only when every input's
    tile digits carry dense trailing strides (one contiguous slice per tile).
    A member stored with its separator digits reversed must not be tiled."""
    m, d = 10, 3
    radix = [3] * m
    canon = [d * 3 ** (m - 1 - q) for q in range(m)]         # ascending scope, x last
    rev = [d * 3 ** q for q in range(m)]                     # reversed separator order
    assert G.bucket_kernel_variant(_desc(radix, d, [canon, canon]), 0, 3 ** m) == 1
    assert G.bucket_kernel_variant(_desc(radix, d, [canon, rev]), 0, 3 ** m) != 1
    # padded strides (gaps between digits) are not contiguous either
    pad = [2 * s for s in canon]
    assert G.bucket_kernel_variant(_desc(radix, d, [canon, pad]), 0, 3 ** m) != 1


def test_domain1_digits_do_not_overflow_tile_tables():
    """radix-1 digits must not push the tiled kernel's
    middle-digit count past its 12-entry tables (the call must not corrupt
    memory; it may take either kernel)."""
    radix = [1, 3] * 15
    d = 3
    st, s = [0] * len(radix), d
    for q in reversed(range(len(radix))):
        st[q] = s
        s *= radix[q]
    v = G.bucket_kernel_variant(_desc(radix, d, [st, st]), 0, int(np.prod(radix)))
    assert v in (0, 1)


def test_spill_plan_errors():
    """"spill" (out-of-core): exact BE/DPOP on one rank,
    a positive budget; a budget no chunking can meet is GBE_E_BUDGET."""
    inst = gen.scalefree(40, 3, 0.0, 3)
    P = G.Problem.from_instance(inst)
    order, _ = P.order()
    G.Plan(P, order, spill=True, budget_bytes=1 << 30)  # valid
    for args, kw in (((2,), dict(spill=True, budget_bytes=1 << 30)),
                     ((), dict(spill=True, budget_bytes=1 << 30, world_size=2, rank=0)),
                     ((), dict(spill=True, budget_bytes=1 << 30, count="optimal")),
                     ((), dict(spill=True)),
                     ((), dict(spill=True, budget_bytes=1 << 30, stage_bytes=-1))):
        with pytest.raises(G.GbeError) as e:
            G.Plan(P, order, *args, **kw)
        assert e.value.status == 1
    with pytest.raises(G.GbeError) as e:
        G.Plan(P, order, spill=True, budget_bytes=4096)
    assert e.value.status == 3


def _input_layout(inst, info, pos, t):
    """(scope, stride per variable) of every input of table t: originals and
    messages in the canonical layout (scope ascending by order position,
    first variable most significant, P:553-554 / P:751-753)."""
    tab = info["tables"][t]
    out = []
    for kind, idx in tab["members"]:
        scope = [int(v) for v in inst.scope(idx)] if kind == 0 else list(info["tables"][idx]["sep"])
        scope = sorted(scope, key=lambda v: pos[v])
        st, s = {}, 1
        for v in reversed(scope):
            st[v] = s
            s *= int(inst.dom[v])
        out.append((kind, idx, st))
    return out


@pytest.mark.parametrize("seed,budget_frac,stage_div", [(3, 0.6, 16), (4, 0.5, 8), (5, 0.7, 64)])
def test_spill_plan_chunks_fit_their_slot(seed, budget_frac, stage_div):
    """Every chunk of an out-of-core plan fits one staging slot: its output
    rows (host message), argmins and, for each host-resident input, the
    element range the chunk's rows read -- recomputed here by enumerating the
    rows of each chunk and applying the index map (Eq. P:673-697) directly."""
    inst = gen.scalefree(60, 3, 0.0, seed)
    P = G.Problem.from_instance(inst)
    order, _ = P.order()
    pos = {int(v): i for i, v in enumerate(order)}
    peak = G.Plan(P, order).info()["peak_bytes"]
    info = G.Plan(P, order, spill=True, budget_bytes=int(peak * budget_frac),
                  stage_bytes=peak // stage_div).info()
    assert info["peak_bytes"] <= int(peak * budget_frac)
    tabs = info["tables"]
    host = [t["host"] for t in tabs]
    assert any(host)
    # greedy by size: no device message is larger than a host one
    assert min(t["rows"] for t in tabs if t["host"]) >= max([t["rows"] for t in tabs if not t["host"]] + [0])
    slot = info["slot_bytes"]
    up = lambda b: (b + 255) // 256 * 256  # noqa: E731
    nmulti = 0
    for t, tab in enumerate(tabs):
        sep, d, rows, cr = tab["sep"], tab["d"], tab["rows"], tab["chunk_rows"]
        assert 1 <= cr <= rows
        nmulti += cr < rows
        dom = [int(inst.dom[v]) for v in sep]
        layouts = _input_layout(inst, info, pos, t)
        for lo in range(0, rows, cr):
            hi = min(rows, lo + cr)
            need = (up(4 * (hi - lo)) if tab["host"] else 0) + up(hi - lo)
            r = np.arange(lo, hi, dtype=np.int64)
            digits = []
            for q in range(len(sep) - 1, -1, -1):
                digits.append(r % dom[q])
                r //= dom[q]
            digits = digits[::-1]
            for kind, idx, st in layouts:
                if kind != 1 or not host[idx]:
                    continue
                off = np.zeros(hi - lo, dtype=np.int64)
                for q, v in enumerate(sep):
                    off += digits[q] * st.get(v, 0)
                n = int(off.max() - off.min()) + d
                need += up(4 * n + 64)
            assert need <= slot, (t, lo, need, slot)
    assert nmulti > 0
