"""Pins of the CPU oracle to things other than itself (-m "not gpu").

Each test names the PAPER.md passage (P:n) or mathematical fact it checks.
A plausible mistake in the oracle (dropped term, wrong sign / index,
transposed operand, wrong bucket rule, wrong tie-break) fails at least one.
"""
import itertools
import math

import numpy as np
import pytest

import gen
import oracle
from gen import configs
from oracle.brute import brute_force, brute_force_np, mpe_linear

INF = oracle.INF_I32


def example1(costs=None):
    """Example 1: 4 binary variables x1..x4 (ids 0..3), functions
    f(x1,x2), f(x1,x4), f(x2,x3), f(x2,x4), f(x3,x4)."""
    scopes = [(0, 1), (0, 3), (1, 2), (1, 3), (2, 3)]
    rng = np.random.default_rng(7)
    if costs is None:
        costs = [rng.integers(0, 10, 4) for _ in scopes]
    return gen.Instance.from_functions([2, 2, 2, 2], list(zip(scopes, costs)))


# ---------------------------------------------------------------- structure

def test_example1_induced_width_is_3():
    """along <x1,x2,x3,x4> the induced width is 3."""
    assert oracle.induced_width(example1(), [0, 1, 2, 3]) == 3


def test_example1_primal_graph_has_5_edges():
    """P:162-163 / S:141: 5 binary constraints -> 5 edges."""
    assert int(oracle.primal_graph(example1()).sum()) == 2 * 5


def test_degree_ordering_example():
    """S:163 applying P:610 to Example 1 (degrees 2,3,2,3): <x1,x3,x2,x4>."""
    assert list(oracle.degree_order(example1())) == [0, 2, 1, 3]


def test_induced_width_closed_forms():
    """Path graph -> 1, complete graph K4 -> 3, cycle -> 2 (any ordering)."""
    path = gen.Instance.from_functions([2] * 3, [((0, 1), [0] * 4), ((1, 2), [0] * 4)])
    assert oracle.induced_width(path, [0, 1, 2]) == 1
    k4 = gen.Instance.from_functions([2] * 4, [((a, b), [0] * 4) for a in range(4) for b in range(a + 1, 4)])
    for order in itertools.permutations(range(4)):
        assert oracle.induced_width(k4, order) == 3
    cyc = gen.Instance.from_functions([2] * 6, [((i, (i + 1) % 6), [0] * 4) for i in range(6)])
    for order in [range(6), [3, 1, 5, 0, 2, 4]]:
        assert oracle.induced_width(cyc, list(order)) == 2


def test_minfill_on_trees_gives_width_1():
    """A tree has treewidth 1 and min-fill never adds fill on a tree."""
    for seed in range(5):
        t = gen.random_graph(30, 2, 29, 1, 0.0, seed)
        assert oracle.induced_width(t, oracle.minfill_order(t)) == 1


def test_example2_pseudotree():
    """Example 2: tree edges {12,23,34}; x4's pseudo-parents are x1
    and x2 (backedges (1,4), (2,4))."""
    par = oracle.elim_tree(example1(), [0, 1, 2, 3])
    assert list(par) == [-1, 0, 1, 2]
    tree = {(min(v, p), max(v, p)) for v, p in enumerate(par) if p >= 0}
    assert tree == {(0, 1), (1, 2), (2, 3)}
    back = set(example1().edges()) - tree
    assert back == {(0, 3), (1, 3)}


def test_example3_buckets():
    """Example 3: B4 = {f14, f24, f34}, B3 = {f23, f^4},
    B2 = {f12, f^3}, B1 = {f^2} (reading A1: latest-ordered variable)."""
    r = oracle.solve_be(example1(), [0, 1, 2, 3])
    by_var = {t.var: (i, t) for i, t in enumerate(r.tables)}
    assert [t.var for t in r.tables] == [3, 2, 1, 0]
    assert by_var[3][1].members == [(0, 1), (0, 3), (0, 4)]
    assert by_var[2][1].members == [(0, 2), (1, by_var[3][0])]
    assert by_var[1][1].members == [(0, 0), (1, by_var[2][0])]
    assert by_var[0][1].members == [(1, by_var[1][0])]
    assert list(by_var[3][1].sep) == [0, 1, 2]


def test_example4_minibucket_partition():
    """Example 4 with z=1 (reading A5: i bounds the generated
    arity): B4 splits into the singletons {f14}, {f24}, {f34}; then
    B3 = {f23, f^4_3}, B2 = {f12, f^4_2, f^3_1}, B1 = {f^4_1, f^2_1}."""
    r = oracle.solve_mbe(example1(), [0, 1, 2, 3], 1)
    assert r.status == 0
    tabs = r.tables
    b4 = [(i, t) for i, t in enumerate(tabs) if t.var == 3]
    assert [t.members for _, t in b4] == [[(0, 1)], [(0, 3)], [(0, 4)]]
    assert [list(t.sep) for _, t in b4] == [[0], [1], [2]]
    f41, f42, f43 = (i for i, _ in b4)
    t3 = [t for t in tabs if t.var == 2]
    assert len(t3) == 1 and t3[0].members == [(0, 2), (1, f43)]
    i31 = [i for i, t in enumerate(tabs) if t.var == 2][0]
    t2 = [t for t in tabs if t.var == 1]
    assert len(t2) == 1 and t2[0].members == [(0, 0), (1, f42), (1, i31)]
    i21 = [i for i, t in enumerate(tabs) if t.var == 1][0]
    t1 = [t for t in tabs if t.var == 0]
    assert len(t1) == 1 and t1[0].members == [(1, f41), (1, i21)]


def test_minibucket_ibound_below_arity_is_invalid():
    """a member that cannot fit the bound is an error."""
    assert oracle.solve_mbe(example1(), [0, 1, 2, 3], 0).status == 1


# ---------------------------------------------------------------- index map

def test_section63_index_map_example():
    """§6.3 example: aggregating T_j = f23 (scope x2,x3) into the
    output table over (x1,x2,x3) maps T_id 0..7 to r_j 0,1,2,3,0,1,2,3.  We
    read it through the oracle's bucket function: a selector member g(x3)
    forces the eliminated value v, so out(x1,x2) = f23[map(x1,x2,v)]."""
    dom = [2, 2, 2]
    f23 = ((1, 2), [0, 1, 2, 3])  # value = its own row index r_j
    got = []
    for v in range(2):
        sel = ((2,), [0, INF] if v == 0 else [INF, 0])
        out, arg = oracle.bucket_eval(dom, False, 2, [f23, sel], [0, 1])
        assert list(arg) == [v] * 4
        got.append(list(out))
    tid_to_rj = [got[tid % 2][tid // 2] for tid in range(8)]  # T_id = x1 x2 x3
    assert tid_to_rj == [0, 1, 2, 3, 0, 1, 2, 3]


def test_eliminate_closed_form():
    """S:279 (Proc. 5): scope (x1,x2), chi = [5,2,7,1], min over
    the last variable -> [2,1] with argmins [1,1]."""
    out, arg = oracle.bucket_eval([2, 2], False, 1, [((0, 1), [5, 2, 7, 1])], [0])
    assert list(out) == [2, 1] and list(arg) == [1, 1]


def test_transposed_scope_is_reranked():
    """A member declared as (x2, x1) must be read transposed."""
    out, _ = oracle.bucket_eval([2, 2], False, 1, [((1, 0), [5, 2, 7, 1])], [0])
    # f(x2,x1): f(x1=0,x2=0)=5, f(x1=0,x2=1)=7, f(x1=1,x2=0)=2, f(x1=1,x2=1)=1
    assert list(out) == [5, 1]


def test_one_hot_pins_each_row_mapping():
    """One-hot inputs: a single 1 in a zero table of a member over a random
    sub-scope lights exactly the output rows whose tuple projects onto that
    cell (naive tuple matching)."""
    rng = np.random.default_rng(3)
    for trial in range(40):
        m = int(rng.integers(1, 5))
        dom = [int(x) for x in rng.integers(1, 4, m + 1)]
        x = m
        sep = list(range(m))
        sub = sorted(rng.choice(m, size=int(rng.integers(0, m + 1)), replace=False).tolist())
        scope = [int(v) for v in rng.permutation(sub + [x])]
        cells = int(np.prod([dom[v] for v in scope]))
        hot = int(rng.integers(cells))
        t = np.zeros(cells, np.int64)
        t[hot] = 1
        # second member pins v: cost 0 only at v = 0
        selv = [0] + [INF] * (dom[x] - 1)
        out, _ = oracle.bucket_eval(dom, False, x, [(scope, t), ((x,), selv)], sep)
        hot_tuple = np.unravel_index(hot, [dom[v] for v in scope])
        hv = dict(zip(scope, hot_tuple))
        for r, tup in enumerate(itertools.product(*[range(dom[v]) for v in sep])):
            a = dict(zip(sep, tup))
            a[x] = 0
            expect = 1 if all(a[v] == hv[v] for v in scope) else 0
            assert out[r] == expect


# ---------------------------------------------------------------- exactness

@pytest.mark.parametrize("seed", range(200))
def test_be_equals_brute_force_small(seed):
    """Cor. 3 / S:586: BE optimum = brute-force optimum, and the
    BE assignment (smallest-index forward pass) is the lexicographically
    smallest optimum under the ordering."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(6, 10))
    d = int(rng.integers(2, 5))
    while d ** n > 70000:
        n -= 1
    p1 = float(rng.uniform(0.2, 0.9))
    p2 = [0.0, 0.3, 0.5][seed % 3]
    ne = max(n - 1, int(p1 * n * (n - 1) / 2))
    inst = gen.random_graph(n, d, ne, 0, p2, seed)
    order = oracle.minfill_order(inst) if seed % 2 else oracle.degree_order(inst)
    r = oracle.solve_be(inst, order)
    opt, a = brute_force_np(inst, order)
    assert r.value == opt
    assert oracle.evaluate(inst, r.assignment) == opt
    if opt < INF:  # an infeasible optimum (INF) has no unique assignment
        assert list(r.assignment) == a


@pytest.mark.parametrize("seed", range(6))
def test_c1_config_against_brute_force(seed):
    """C1 (n=12, d=3, 19 or 39 edges, p2 in {0, 0.5}): exact BE vs 3^12
    brute force."""
    inst = configs.c1(seed, literal=bool(seed % 2), p2=0.5 if seed >= 3 else 0.0)
    order = oracle.minfill_order(inst)
    r = oracle.solve_be(inst, order)
    opt, a = brute_force_np(inst, order)
    assert r.value == opt and oracle.evaluate(inst, r.assignment) == opt
    if opt < INF:
        assert list(r.assignment) == a


def test_pure_python_brute_force_agrees_with_vectorised():
    inst = gen.random_graph(7, 3, 10, 0, 0.3, 11)
    assert brute_force(inst, range(7)) == brute_force_np(inst, range(7))


def _tree_dp(inst, root=0):
    """Independent min-sum dynamic programme on a tree (w* = 1)."""
    n = inst.n
    nbr = {v: [] for v in range(n)}
    fn = {}
    for f in range(inst.nf):
        u, v = (int(x) for x in inst.scope(f))
        nbr[u].append(v)
        nbr[v].append(u)
        t = inst.table(f).reshape(int(inst.dom[u]), int(inst.dom[v]))
        fn[(u, v)] = t
        fn[(v, u)] = t.T

    def msg(c, p):  # min over c of f(p, c) + sum of c's children messages
        below = np.zeros(int(inst.dom[c]), np.int64)
        for g in nbr[c]:
            if g != p:
                below = np.minimum(below + msg(g, c), INF)
        tab = fn[(p, c)].astype(np.int64)
        return np.minimum(tab + below[None, :], INF).min(axis=1)

    tot = np.zeros(int(inst.dom[root]), np.int64)
    for c in nbr[root]:
        tot = np.minimum(tot + msg(c, root), INF)
    return int(tot.min())


@pytest.mark.parametrize("seed", range(10))
def test_tree_instances_match_tree_dp(seed):
    inst = gen.random_graph(40, 4, 39, 1, 0.2 if seed % 2 else 0.0, seed)
    order = oracle.minfill_order(inst)
    assert oracle.induced_width(inst, order) == 1
    assert oracle.solve_be(inst, order).value == _tree_dp(inst)


def test_special_cases():
    """S:514-style closed forms: all-zero -> 0 and all-zero assignment;
    unary-only -> sum of minima and argmins; all-INF -> INF; d = 1 copy."""
    z = gen.Instance.from_functions([3, 3, 3], [((0, 1), [0] * 9), ((1, 2), [0] * 9)])
    r = oracle.solve_be(z, [0, 1, 2])
    assert r.value == 0 and list(r.assignment) == [0, 0, 0]
    un = gen.Instance.from_functions([3, 2], [((0,), [4, 1, 9]), ((1,), [7, 3])])
    r = oracle.solve_be(un, [0, 1])
    assert r.value == 1 + 3 and list(r.assignment) == [1, 1]
    inf = gen.Instance.from_functions([2, 2], [((0, 1), [INF] * 4)])
    r = oracle.solve_be(inf, [0, 1])
    assert r.value == INF and list(r.assignment) == [0, 0]
    out, arg = oracle.bucket_eval([3, 1], False, 1, [((0, 1), [5, 6, 7])], [0])
    assert list(out) == [5, 6, 7] and list(arg) == [0, 0, 0]


def test_disconnected_components_sum():
    """disconnected graphs are solved per component and the root
    costs are summed."""
    a = gen.random_graph(6, 3, 8, 0, 0.0, 1)
    b = gen.random_graph(5, 3, 6, 0, 0.0, 2)
    fns = [(list(a.scope(f)), a.table(f)) for f in range(a.nf)]
    fns += [([int(v) + 6 for v in b.scope(f)], b.table(f)) for f in range(b.nf)]
    ab = gen.Instance.from_functions([3] * 11, fns)
    va = oracle.solve_be(a, oracle.minfill_order(a)).value
    vb = oracle.solve_be(b, oracle.minfill_order(b)).value
    assert oracle.solve_be(ab, oracle.minfill_order(ab)).value == va + vb


# ---------------------------------------------------------------- MBE

@pytest.mark.parametrize("seed", range(30))
def test_mbe_bound_sandwich_and_exactness(seed):
    """MBE lower <= BE <= evaluate(MBE assignment); with i >= w*
    there is no partition and every table equals BE's (Thm 1)."""
    inst = gen.random_graph(14, 3, 30, 0, 0.0 if seed % 2 else 0.3, seed)
    order = oracle.minfill_order(inst)
    w = oracle.induced_width(inst, order)
    be = oracle.solve_be(inst, order)
    for i in range(1, w + 1):
        r = oracle.solve_mbe(inst, order, i)
        assert r.status == 0
        assert r.value <= be.value <= r.upper
        assert r.upper == oracle.evaluate(inst, r.assignment)
        assert max(len(t.sep) for t in r.tables) <= i  # Cor. 1: arity <= i
    r = oracle.solve_mbe(inst, order, w)
    assert r.value == be.value == r.upper
    assert len(r.tables) == len(be.tables)
    for t, u in zip(r.tables, be.tables):
        assert np.array_equal(t.out, u.out) and np.array_equal(t.arg, u.arg)


# ---------------------------------------------------------------- DPOP

@pytest.mark.parametrize("seed", range(10))
def test_elimination_tree_is_a_pseudotree(seed):
    """every primal edge joins an ancestor and a descendant; Cor. 2
    (P:876-883): n - #components UTIL messages."""
    inst = gen.scalefree(25, 2, 0.0, seed)
    order = oracle.minfill_order(inst)
    par = oracle.elim_tree(inst, order)

    def anc(v):
        out = set()
        while par[v] >= 0:
            v = int(par[v])
            out.add(v)
        return out

    for u, v in inst.edges():
        assert u in anc(v) or v in anc(u)
    assert sum(1 for p in par if p >= 0) == inst.n - 1
    r = oracle.solve_be(inst, order)
    # UTIL message of v goes to parent(v): the table's destination
    for t in r.tables:
        assert t.dest == par[t.var]


# ---------------------------------------------------------------- MPE

@pytest.mark.parametrize("seed", range(12))
def test_mpe_matches_linear_domain_brute_force(seed):
    """MPE Eq. (2): exp(-BE value) = max_sigma prod Pr within
    1e-9 relative; the BE assignment attains it."""
    inst = gen.belief_net(9, 2, 3, 2, 4, seed)
    order = oracle.minfill_order(inst)
    r = oracle.solve_be(inst, order)
    best = mpe_linear(inst)
    assert math.isclose(math.exp(-r.value), best, rel_tol=1e-9)
    assert math.isclose(oracle.evaluate(inst, r.assignment), r.value, rel_tol=1e-12)


def test_mpe_chain_viterbi():
    """A chain BN (one parent each) has the closed-form Viterbi recursion."""
    inst = gen.belief_net(30, 2, 4, 1, 1, 5)
    # Viterbi in the linear domain with rescaling
    dom = [int(d) for d in inst.dom]
    p0 = np.exp(-inst.table(0))
    best = p0.copy()
    logscale = 0.0
    for v in range(1, inst.n):
        cpt = np.exp(-inst.table(v)).reshape(dom[v - 1], dom[v])
        best = (best[:, None] * cpt).max(axis=0)
        s = best.max()
        best /= s
        logscale += math.log(s)
    viterbi_log = logscale + math.log(best.max())
    r = oracle.solve_be(inst, oracle.minfill_order(inst))
    assert math.isclose(-r.value, viterbi_log, rel_tol=1e-9)


# ---------------------------------------------------------------- generators

def test_generator_laws():
    """2(n-2)+1 scale-free edges; grid degree profile 2/3/4;
    P:922 (reading A4): exact edge count, connected."""
    for n in (10, 57, 200):
        assert len(gen.scalefree(n, 2, 0.0, 1).edges()) == 2 * (n - 2) + 1
    g = gen.grid(4, 5, 2)
    adj = oracle.primal_graph(g)
    deg = adj.sum(1).reshape(4, 5)
    assert deg[0, 0] == deg[0, 4] == deg[3, 0] == deg[3, 4] == 2
    assert (deg[1:3, 1:4] == 4).all() and deg[0, 2] == 3 and deg[2, 0] == 3
    r = gen.random_graph(12, 3, 19, 0, 0.0, 4)
    assert len(r.edges()) == 19
    assert oracle.induced_width(r, oracle.minfill_order(r)) >= 1


def test_generator_tightness_exact_count():
    """P:928 / S:564: exactly floor(p2 * cells) infinite cells per function."""
    inst = gen.random_graph(10, 5, 20, 0, 0.5, 3)
    for f in range(inst.nf):
        assert int((inst.table(f) == INF).sum()) == 12


def test_pinned_config_widths():
    """BASELINE.md re-parameterisations: C2 w*=10, C4 w*=20, C5 w*=18 under
    min-fill; C3 row-major w*=20."""
    assert oracle.induced_width(configs.c2(), oracle.minfill_order(configs.c2())) == 10
    c4 = configs.c4()
    assert oracle.induced_width(c4, oracle.minfill_order(c4)) == 20
    c5 = configs.c5()
    assert oracle.induced_width(c5, oracle.minfill_order(c5)) == 18
    assert oracle.induced_width(configs.c3(), configs.c3_order()) == 20
    c4d4 = configs.c4d4()  # SURVEY's alternative C4: n=150, d=4, w*=16
    assert oracle.induced_width(c4d4, oracle.minfill_order(c4d4)) == 16
    assert len(c4d4.dom) == 150 and set(int(v) for v in c4d4.dom) == {4}


# ------------------------------------------------ sum-product (§8(f) row 3)
# The sum/product semiring (partition function = the paper's future
# work): -log Z with Z = sum over all assignments of prod exp(-f).

def _close(a, b, tol=1e-12):
    return (math.isinf(a) and math.isinf(b)) or abs(a - b) <= tol * (1 + abs(b))


@pytest.mark.parametrize("seed", range(6))
def test_sumprod_against_brute_force(seed):
    """-log Z of the oracle's sum-product BE equals enumeration of the whole
    state space (with forbidden cells for seeds >= 3)."""
    from oracle.brute import neg_log_z
    inst = gen.random_network_f64(8, 2, 3, 12, 1, 3, 4.0, 0.3 if seed >= 3 else 0.0, seed)
    for order in (oracle.minfill_order(inst), np.arange(inst.n, dtype=np.int32)):
        r = oracle.solve_sumprod(inst, order)
        assert r.assignment is None
        assert _close(r.value, neg_log_z(inst)), (r.value, neg_log_z(inst))


@pytest.mark.parametrize("n,seed", [(30, 1), (80, 2), (150, 3)])
def test_sumprod_belief_net_is_normalised(n, seed):
    """A belief network without evidence is a normalised distribution
    (CPTs sum to 1 over the child), so Z = 1 exactly and
    -log Z = 0 up to rounding, at any size."""
    bn = gen.belief_net(n, 2, 4, 3, 8, seed)
    r = oracle.solve_sumprod(bn, oracle.minfill_order(bn))
    assert abs(r.value) < 1e-12 * n


def _with_evidence(bn, ev):
    """Evidence as 0 / +inf unary functions."""
    funcs = [(list(bn.scope(f)), bn.table(f)) for f in range(bn.nf)]
    for v, e in ev.items():
        t = np.full(int(bn.dom[v]), np.inf)
        t[e] = 0.0
        funcs.append(([v], t))
    return gen.Instance.from_functions(bn.dom, funcs, is_f64=True)


def test_sumprod_root_evidence_is_the_prior():
    """Evidence on the parentless x0 and on a child x1 whose only parent is
    x0: Z = P(E) = p(x0 = e0) * p(x1 = e1 | x0 = e0), two CPT entries (the
    generator's CPT tables are -log p with the child last)."""
    bn = gen.belief_net(40, 2, 4, 3, 8, 5)
    f0 = [f for f in range(bn.nf) if list(bn.scope(f)) == [0]]
    f1 = [f for f in range(bn.nf) if list(bn.scope(f)) == [0, 1]]
    assert len(f0) == 1 and len(f1) == 1
    t1 = bn.table(f1[0]).reshape(int(bn.dom[0]), int(bn.dom[1]))
    assert np.allclose(np.exp(-t1).sum(axis=1), 1.0)  # child last: rows normalised
    e0, e1 = int(bn.dom[0]) - 1, 1
    inst = _with_evidence(bn, {0: e0})
    r = oracle.solve_sumprod(inst, oracle.minfill_order(inst))
    assert _close(r.value, float(bn.table(f0[0])[e0]), 1e-11)
    inst = _with_evidence(bn, {0: e0, 1: e1})
    r = oracle.solve_sumprod(inst, oracle.minfill_order(inst))
    expect = float(bn.table(f0[0])[e0]) + float(t1[e0, e1])
    assert _close(r.value, expect, 1e-11), (r.value, expect)


def test_sumprod_evidence_against_brute_force():
    """P(E) for evidence on non-root variables, against enumeration."""
    from oracle.brute import neg_log_z
    bn = gen.belief_net(9, 2, 3, 2, 4, 11)
    inst = _with_evidence(bn, {8: 1, 5: 0})
    r = oracle.solve_sumprod(inst, oracle.minfill_order(inst))
    assert _close(r.value, neg_log_z(inst))
    assert r.value > 0  # P(E) < 1


def test_sumprod_independent_factors_closed_form():
    """Unary factors only: Z = prod_i sum_v exp(-f_i(v)); all-zero costs give
    Z = prod d_i, i.e. negative messages (-log d) — pins the sign."""
    rng = np.random.default_rng(3)
    dom = [2, 3, 5, 4, 1]
    tabs = [rng.uniform(0, 6, d) for d in dom]
    inst = gen.Instance.from_functions(dom, [([i], t) for i, t in enumerate(tabs)], is_f64=True)
    expect = math.fsum(-math.log(math.fsum(math.exp(-c) for c in t)) for t in tabs)
    assert _close(oracle.solve_sumprod(inst, oracle.minfill_order(inst)).value, expect)
    zero = gen.Instance.from_functions(dom, [([i], np.zeros(d)) for i, d in enumerate(dom)],
                                       is_f64=True)
    assert _close(oracle.solve_sumprod(zero, np.arange(5, dtype=np.int32)).value,
                  -math.log(2 * 3 * 5 * 4 * 1))


def test_sumprod_bucket_rows_special_cases():
    """One member: each row is scipy's logsumexp of the negated slice
    (library routine); an all-infinite row stays +inf; d = 1 is the identity."""
    from scipy.special import logsumexp
    rng = np.random.default_rng(9)
    dom = [3, 4, 6]
    t = rng.uniform(-5, 20, 3 * 4 * 6)
    t[:6] = np.inf  # row (0, 0) all infinite
    t[7] = np.inf
    out = oracle.bucket_eval_sp(dom, 2, [([0, 1, 2], t)], [0, 1])
    ref = [-logsumexp(-t[r * 6:(r + 1) * 6]) for r in range(12)]
    assert math.isinf(out[0]) and out[0] > 0
    np.testing.assert_allclose(out[1:], ref[1:], rtol=1e-13)
    # two members: sum inside the exponent (aggregation P:204-205)
    u = rng.uniform(0, 3, 4 * 6)
    out2 = oracle.bucket_eval_sp(dom, 2, [([0, 1, 2], t), ([1, 2], u)], [0, 1])
    for r in range(1, 12):
        b = r % 4
        assert _close(out2[r], -logsumexp(-(t[r * 6:(r + 1) * 6] + u[b * 6:(b + 1) * 6])), 1e-13)
    one = oracle.bucket_eval_sp([3, 1], 1, [([0, 1], np.array([1.5, 2.0, 7.0]))], [0])
    np.testing.assert_array_equal(one, [1.5, 2.0, 7.0])


# ------------------------------------------ solution counting (§8(f) row 4)
# "as a byproduct ... BE can compute the number of consistent
# solutions".  The (min, count) semiring: count = number of optimal
# assignments; with every finite cost read as 0 it counts the consistent ones.

@pytest.mark.parametrize("seed", range(40))
def test_count_against_brute_force(seed):
    """Optimal and consistent counts equal enumeration (exact integers),
    with forbidden cells (p2 > 0) and small cost ranges (many ties)."""
    from oracle.brute import count_solutions
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(5, 9))
    d = int(rng.integers(2, 4))
    p2 = [0.0, 0.2, 0.4][seed % 3]
    cmax = [1, 2, 100][seed % 3 if seed % 5 else 0]
    inst = gen.random_network(n, d, d, int(rng.integers(n, 2 * n)), 1, 3, cmax, p2, seed)
    order = oracle.minfill_order(inst) if seed % 2 else oracle.degree_order(inst)
    opt, n_opt, n_cons = count_solutions(inst)
    ro = oracle.solve_count(inst, order, "optimal")
    assert ro.value == opt and ro.count == n_opt, (ro.value, opt, ro.count, n_opt)
    rc = oracle.solve_count(inst, order, "consistent")
    assert rc.count == n_cons, (rc.count, n_cons)
    assert rc.value == (0 if n_cons else INF)
    # the min-sum tables and argmins are those of plain BE
    rb = oracle.solve_be(inst, order)
    assert all(a.digest == b.digest for a, b in zip(ro.tables, rb.tables))


def test_count_f64_against_brute_force():
    """f64 (MPE-style) problems: optimal count (ties at equal doubles) and
    consistent count (p = 0 cells) by enumeration."""
    from oracle.brute import count_solutions
    for seed in range(6):
        inst = gen.random_network_f64(7, 2, 3, 10, 1, 3, 4.0, 0.3, seed)
        order = oracle.minfill_order(inst)
        opt, n_opt, n_cons = count_solutions(inst)
        assert oracle.solve_count(inst, order, "optimal").count == n_opt
        assert oracle.solve_count(inst, order, "consistent").count == n_cons


def test_count_closed_forms():
    """All-zero costs: every assignment optimal and consistent, prod d_i.
    Unary-only: prod_i (#values attaining the unary minimum).  All-INF: 0.
    Two disjoint copies of an instance: the counts multiply."""
    dom = [2, 3, 4, 3]
    z = gen.Instance.from_functions(dom, [((0, 1), [0] * 6), ((1, 2, 3), [0] * 36)])
    for mode in ("optimal", "consistent"):
        assert oracle.solve_count(z, oracle.minfill_order(z), mode).count == 2 * 3 * 4 * 3
    un = [[3, 1, 1], [0, 5], [2, 2, 2, 9]]
    u = gen.Instance.from_functions([3, 2, 4], [((i,), t) for i, t in enumerate(un)])
    r = oracle.solve_count(u, [0, 1, 2], "optimal")
    assert r.value == 1 + 0 + 2 and r.count == 2 * 1 * 3
    assert oracle.solve_count(u, [0, 1, 2], "consistent").count == 3 * 2 * 4
    ai = gen.Instance.from_functions([2, 2], [((0, 1), [INF] * 4)])
    for mode in ("optimal", "consistent"):
        assert oracle.solve_count(ai, [0, 1], mode).count == 0
    base = gen.random_network(5, 3, 3, 7, 1, 3, 2, 0.2, 4)
    funcs = [(list(base.scope(f)), base.table(f)) for f in range(base.nf)]
    two = gen.Instance.from_functions(list(base.dom) * 2, funcs + [([v + 5 for v in s], t) for s, t in funcs])
    for mode in ("optimal", "consistent"):
        c1 = oracle.solve_count(base, oracle.minfill_order(base), mode).count
        c2 = oracle.solve_count(two, oracle.minfill_order(two), mode).count
        assert c2 == c1 * c1


def test_count_tree_closed_form():
    """A chain x0 - x1 - ... - x7 with 0/1 costs f(a, b) = [a != b]: optimum
    0, attained by the d constant assignments; every assignment consistent."""
    d, n = 3, 8
    t = [0 if a == b else 1 for a in range(d) for b in range(d)]
    ch = gen.Instance.from_functions([d] * n, [((i, i + 1), t) for i in range(n - 1)])
    r = oracle.solve_count(ch, oracle.minfill_order(ch), "optimal")
    assert r.value == 0 and r.count == d
    assert oracle.solve_count(ch, oracle.minfill_order(ch), "consistent").count == d ** n


# ------------------------------------------- row sums / checksums (test tools)

@pytest.mark.parametrize("is_f64", [False, True])
def test_bucket_row_sums_against_direct_evaluation(is_f64):
    """or_bucket_row_sums = Alg. 1 line 3 before the projection:
    each sum equals the members evaluated directly at theta.v (numpy indexing
    of the member tables reshaped to their scopes), and min / first minimiser
    over v equal or_bucket_rows (A8)."""
    rng = np.random.default_rng(11)
    dom = [2, 3, 4, 3, 2]
    x = 2
    sep = [0, 1, 3, 4]
    scopes = [(0, 2), (4, 1, 2), (3, 2), (2,), (0, 1, 3, 4, 2)]
    members = []
    for sc in scopes:
        cells = int(np.prod([dom[v] for v in sc]))
        t = rng.random(cells) * 5 if is_f64 else rng.integers(0, 50, cells).astype(np.int32)
        if not is_f64:
            t[rng.random(cells) < 0.2] = INF
        members.append((list(sc), t))
    R = int(np.prod([dom[v] for v in sep]))
    rows = np.arange(R, dtype=np.int64)
    sums = oracle.bucket_row_sums(dom, is_f64, x, members, sep, rows)
    out, arg = oracle.bucket_eval(dom, is_f64, x, members, sep)
    for r in range(R):
        digits, q = {}, r
        for v in reversed(sep):
            digits[v] = q % dom[v]
            q //= dom[v]
        for val in range(dom[x]):
            digits[x] = val
            tot = 0.0 if is_f64 else 0
            for sc, t in members:
                e = t.reshape([dom[v] for v in sc])[tuple(digits[v] for v in sc)]
                tot = tot + float(e) if is_f64 else min(tot + int(e), INF)
            assert sums[r, val] == tot
        assert sums[r].min() == out[r]
        assert int(np.argmin(sums[r])) == arg[r]


def test_mixsum_checksum_properties():
    """The table checksum (not method arithmetic): equal arrays give equal
    sums, any single change, swap or shift changes it, and it is the sum of
    per-element terms (so chunks add up mod 2^64) -- what the GPU tests use
    to compare 1e10-cell tables without copying them to the host."""
    rng = np.random.default_rng(3)
    a = rng.integers(0, 1 << 30, 10001).astype(np.int32)
    h = oracle.mixsum(a, 1)
    assert h == oracle.mixsum(a.copy(), 1)
    b = a.copy(); b[17] += 1
    assert oracle.mixsum(b, 1) != h
    b = a.copy(); b[[5, 9]] = b[[9, 5]]
    assert oracle.mixsum(b, 1) != h
    assert oracle.mixsum(np.roll(a, 1), 1) != h
    assert oracle.mixsum(a, 2) != h
    # pure-Python restatement on a short prefix
    M = (1 << 64) - 1

    def term(i, x, salt):
        z = (i * 0x9E3779B97F4A7C15 + x + salt * 0xD1B54A32D192ED03) & M
        z = ((z ^ (z >> 31)) * 0xBF58476D1CE4E5B9) & M
        return z ^ (z >> 29)
    assert oracle.mixsum(a[:50], 1) == sum(term(i, int(x) & 0xFFFFFFFF, 1) for i, x in enumerate(a[:50])) & M
    u = rng.integers(0, 4, 777).astype(np.uint8)
    assert oracle.mixsum(u, 2) == sum(term(i, int(x), 2) for i, x in enumerate(u)) & M
    f = rng.random(99)
    assert oracle.mixsum(f, 1) == sum(term(i, int(x), 1) for i, x in enumerate(f.view(np.uint64))) & M


@pytest.mark.parametrize("seed", range(5))
def test_symbolic_bucket_structure_matches_oracle_tables(seed):
    """oracle/structure.py (the reference arm's planner) gives the same
    buckets, separators and canonical member lists as the oracle's own BE
    run (Alg. 1 lines 2-5, A1/A2)."""
    from oracle.structure import bucket_structure
    inst = gen.scalefree(30, 3, 0.0, seed) if seed % 2 else gen.random_graph(25, 3, 40, 1, 0.0, seed)
    order = oracle.minfill_order(inst)
    ref = oracle.solve_be(inst, order, keep_tables=False)
    tabs = bucket_structure(inst, order)
    assert len(tabs) == len(ref.tables)
    for t, rt in zip(tabs, ref.tables):
        assert t["var"] == rt.var and t["sep"] == list(rt.sep) and t["rows"] == rt.rows
        assert t["members"] == rt.members


def test_fnv1a_published_vectors():
    """The golden-file table digest (not method arithmetic) is 64-bit FNV-1a:
    pinned to the algorithm's published test vectors (offset basis for the
    empty input; "a" and "foobar"), and chaining over several arrays equals
    hashing their concatenation."""
    def b(s):
        return np.frombuffer(s, dtype=np.uint8)
    assert oracle.fnv1a(b(b"")) == 0xCBF29CE484222325
    assert oracle.fnv1a(b(b"a")) == 0xAF63DC4C8601EC8C
    assert oracle.fnv1a(b(b"foobar")) == 0x85944171F73967E8
    assert oracle.fnv1a(b(b"foo"), b(b"bar")) == oracle.fnv1a(b(b"foobar"))
