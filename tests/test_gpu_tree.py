"""Congruence tree and SAS plans on the device (sfft_tree_build) against
golden trees from the unmodified reference (tests/golden/make_golden_trees.py:
the reference test shapes of tests/test_congruence.py, random supports, a
homogeneous set and the config-3 support).  Reference: congruence.py:134-222,
sas.py:69-77."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def S():
    import paper_2211_15299_b200 as S
    return S


@pytest.fixture(scope="module")
def golden():
    return np.load(os.path.join(HERE, "golden", "golden_trees.npz"))


def _cases(g):
    return range(int(g["n_cases"]))


def test_tree_levels_bit_exact(S, golden):
    """Every level: node count, node order (ascending residue), members
    (ascending) and offsets identical to the reference's build_tree."""
    for i in _cases(golden):
        N, J, depth = int(golden[f"c{i}_N"]), golden[f"c{i}_J"], int(golden[f"c{i}_depth"])
        tree = S.build_tree(S.SupportSet(N, J), depth)
        for l in range(depth + 1):
            n = int(golden[f"c{i}_n"][l])
            assert int(tree._n[l]) == n, (i, l)
            assert np.array_equal(tree._off[l][:n + 1], golden[f"c{i}_off"][l][:n + 1]), (i, l)
            assert np.array_equal(tree._members[l], golden[f"c{i}_members"][l]), (i, l)
        assert tree.split_levels() == tuple(int(x) for x in golden[f"c{i}_split"]), i
        assert [tree.max_weight_at_level(l) for l in range(depth + 1)] == golden[f"c{i}_maxw"].tolist(), i


def test_tree_interface(S, golden):
    """The reference's TreeNode / CongruenceTree interface on the device tree:
    nodes_at_level, node, node_weight (0 when absent), children (left carries
    bit `level`), parent, root, induced_weight, levels, split_levels = pivots,
    depth checks (tests/test_congruence.py:60-200)."""
    for i in list(_cases(golden))[:20]:
        N, J, depth = int(golden[f"c{i}_N"]), golden[f"c{i}_J"], int(golden[f"c{i}_depth"])
        Js = S.SupportSet(N, J)
        tree = S.build_tree(Js, depth)
        assert tree.root.members == tuple(int(x) for x in J) and tree.root.residue == 0
        if depth == Js.M:
            assert tree.split_levels() == S.pivots(Js)
            assert all(nd.weight == 1 for nd in tree.nodes_at_level(depth))
        w = {int(j): complex(1.0 + 0.5 * t, -0.25 * t) for t, j in enumerate(J)}
        for l in range(depth + 1):
            nodes = tree.nodes_at_level(l)
            assert sum(nd.weight for nd in nodes) == len(J)
            assert [nd.residue for nd in nodes] == sorted(nd.residue for nd in nodes)
            assert tree.levels[l].keys() == {nd.residue for nd in nodes}
            for nd in nodes:
                assert all(j % (1 << l) == nd.residue for j in nd.members)
                assert tree.node(l, nd.residue) == nd
                assert abs(tree.induced_weight(l, nd.residue, w) - sum(w[j] for j in nd.members)) < 1e-12
                if l > 0:
                    assert tree.parent(nd).residue == nd.residue % (1 << (l - 1))
                if l < depth:
                    left, right = tree.children(nd)
                    kids = [c for c in (left, right) if c is not None]
                    assert sum(c.weight for c in kids) == nd.weight
                    if left is not None:
                        assert left.residue == nd.residue + (1 << l)
            missing = next((r for r in range(1 << l) if r not in tree.levels[l]), None)
            if missing is not None:
                assert tree.node(l, missing) is None and tree.node_weight(l, missing) == 0
                assert tree.induced_weight(l, missing, w) == 0j
        with pytest.raises(S.InvalidInputError):
            S.build_tree(Js, Js.M + 1)
        with pytest.raises(S.InvalidInputError):
            tree.nodes_at_level(depth + 1)
        if depth > 0:
            with pytest.raises(S.InvalidInputError):
                tree.children(tree.nodes_at_level(depth)[0])


def test_sas_plan_matches_reference(S, golden):
    """SasPlan.plan: decode level, mu*, node weights (ascending residue) and
    the predicted cost for pivot prefixes, equal to the reference's."""
    for i in _cases(golden):
        N, J = int(golden[f"c{i}_N"]), golden[f"c{i}_J"]
        Js = S.SupportSet(N, J)
        piv = S.pivots(Js)
        for row in golden[f"c{i}_plans"]:
            t, level, mu, cost = int(row[0]), int(row[1]), int(row[2]), float(row[3])
            wts = tuple(int(x) for x in row[4:] if x >= 0)
            sp = S.SasPlan.plan(Js, piv[:t])
            assert (sp.decode_level, sp.mu_star, sp.node_weights) == (level, mu, wts), (i, t)
            assert sp.predicted_cost == pytest.approx(cost, rel=1e-15)
            assert sp.shifts == range(mu)


def test_sas_plan_counts_tree_cost_and_contract(S):
    """The counter is charged |J| * level bit operations (the reference's
    build_tree cost) and a non part-homogeneous r raises ContractViolation."""
    Js = S.SupportSet(64, [3, 17, 25, 27, 35])
    c = S.OpCounter()
    sp = S.SasPlan.plan(Js, (1, 3), counter=c)
    assert sp.decode_level == 4 and c.bit_ops == len(Js) * 4
    with pytest.raises(S.ContractViolationError):
        S.SasPlan.plan(Js, (3,))
