"""Shift-and-sample with mu* > 1 on the device vs the reference's own outputs
(tests/golden/make_golden_sas.py, reference tests/test_sas.py shapes)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2211_15299_b200 as S
    return S


def rel_error(got, want, floor=1e-30):
    got = np.asarray(got, np.complex128)
    want = np.asarray(want, np.complex128)
    return float(np.max(np.abs(got - want) / np.maximum(np.abs(want), floor))) if got.size else 0.0


def _case(g, i):
    p = f"s{i}_"
    pol = bytes(g[p + "policy"]).decode().strip()
    base = tuple(int(x) for x in g[p + "base"])
    return p, pol, ({"base_pivots": base} if base else None)


def test_sas_matches_reference(S, golden_sas):
    g = golden_sas
    n_esc = 0
    for i in range(int(g["n_cases"][0])):
        p, pol, meta = _case(g, i)
        N = int(g[p + "N"][0])
        J = S.SupportSet(N, g[p + "J"])
        c = g[p + "c"]
        sig = S.BandlimitedSignal(J, c)
        src = sig.synthesize() if int(g[p + "dense"][0]) else sig
        ctr = S.OpCounter()
        res = S.sas_transform(src, J, policy=pol, family_meta=meta, counter=ctr)
        assert res.plan.pivots == tuple(int(x) for x in g[p + "pivots"]), i
        assert [res.plan.decode_level, res.plan.mu_star] == [int(x) for x in g[p + "plan"]]
        assert res.plan.node_weights == tuple(int(x) for x in g[p + "weights"])
        got = np.asarray(res.coeffs)
        assert rel_error(got, c) < 1e-8, (i, rel_error(got, c))            # tests/test_sas.py standard
        assert rel_error(got, g[p + "coeffs"], floor=1e-9) < 1e-7, i
        rep = res.report
        want = [int(x) for x in g[p + "report"]]
        mine = [rep.tree_build_bitops, rep.hidft_adds, rep.hidft_mults, rep.solve_adds, rep.solve_mults,
                rep.read_ops, rep.samples_touched, rep.escalated_nodes, rep.dense_fallbacks]
        assert mine[:7] == want[:7], (i, mine, want)
        assert rep.total <= rep.bound_alg1bnd + 1e-9 or want[8] > 0
        np.testing.assert_allclose([rep.bound_alg1bnd, rep.bound_hidft], g[p + "bounds"])
        sysw = g[p + "systems"]
        assert [(s.residue, s.size) for s in res.node_systems] == [(int(a), int(b)) for a, b, _, _ in sysw]
        n_esc += rep.escalated_nodes
    assert n_esc > 0  # the double-double path was exercised


def test_worked_example(S):
    # tests/test_sas.py: {0,1,6,7,512}: pivots (0,1), mu*=2, node sizes [1,1,1,2], 8 samples touched
    J = S.SupportSet.make(1024, [0, 1, 6, 7, 512])
    rng = np.random.default_rng(3)
    mag = 0.5 + rng.random(5)
    c = mag * np.exp(1j * rng.random(5) * 2 * np.pi)
    out = S.sas_transform(S.BandlimitedSignal(J, c), J)
    assert rel_error(out.coeffs, c) < 1e-8
    assert out.plan.pivots == (0, 1) and out.plan.mu_star == 2
    assert sorted(s.size for s in out.node_systems) == [1, 1, 1, 2]
    assert out.report.total <= out.report.bound_alg1bnd
    assert out.report.samples_touched == 2 * 4


def test_sas_batched_dense_rows(S):
    import torch
    rng = np.random.default_rng(11)
    M, B = 12, 6
    base = (0, 2, 3, 5, 7, 9)
    import structfft_oracle as O
    H = O.gen_homogeneous(base, M, 7)
    J = np.sort(H[rng.choice(H.size, size=24, replace=False)])
    Js = S.SupportSet(1 << M, J)
    coef = rng.normal(size=(B, J.size)) + 1j * rng.normal(size=(B, J.size))
    f = np.stack([O.synthesize(J, coef[b], M) for b in range(B)])
    for dt, tol in ((np.complex128, 1e-8), (np.complex64, 1e-4)):
        sig = torch.from_numpy(f.astype(dt)).cuda()
        res = S.sas_transform(sig, Js, policy="random_subset", family_meta={"base_pivots": base})
        assert res.plan.mu_star > 1
        got = res.coeffs.cpu().numpy()
        for b in range(B):
            single = S.sas_transform(f[b].astype(dt), Js, policy="random_subset", family_meta={"base_pivots": base})
            assert np.allclose(got[b], single.coeffs, rtol=0, atol=1e-12 * np.abs(single.coeffs).max())
            assert np.linalg.norm(got[b] - coef[b]) / np.linalg.norm(coef[b]) < tol


@pytest.mark.parametrize("pol", ["auto", "random_subset"])
def test_config3_reference_policies(S, golden_sas, pol):
    """Config 3 under the reference's own SAS policies (mu* = 10 / 28, the
    latter with ~90 double-double escalations), identical dense c64 input."""
    import torch
    import structfft_oracle as O
    g = golden_sas
    J, M = O.config_support(3)
    coef = O.config_coefficients(3, 0, J.size)
    f = O.synthesize(J, coef, M).astype(np.complex64)
    Js = S.SupportSet(1 << M, J)
    base = tuple(int(x) for x in g["cfg3_base_pivots"])
    res = S.sas_transform(torch.from_numpy(f).cuda(), Js, policy=pol, family_meta={"base_pivots": base})
    s, mu, esc, fb, touched = (int(x) for x in g[f"cfg3_{pol}_plan"])
    assert (len(res.plan.pivots), res.plan.mu_star, res.report.samples_touched) == (s, mu, touched)
    assert abs(res.report.escalated_nodes - esc) <= max(2, esc // 20), (res.report.escalated_nodes, esc)
    got = res.coeffs.cpu().numpy().reshape(-1)
    want = g[f"cfg3_{pol}_coeffs"]
    assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-8


def test_config3_host_rows(S, golden_sas):
    """Config 3 rows resident in host memory (pinned and pageable): the host
    pool stages the mu* shifted sample sets (sfft_host_stage) and the result
    matches the device-resident path."""
    import torch
    import structfft_oracle as O
    g = golden_sas
    J, M = O.config_support(3)
    Js = S.SupportSet(1 << M, J)
    B = 2
    coef = np.stack([O.config_coefficients(3, b, J.size) for b in range(B)])
    f = np.stack([O.synthesize(J, coef[b], M) for b in range(B)]).astype(np.complex64)
    base = tuple(int(x) for x in g["cfg3_base_pivots"])
    meta = {"base_pivots": base}
    dev = S.sas_transform(torch.from_numpy(f).cuda(), Js, policy="auto", family_meta=meta)
    want = dev.coeffs.cpu().numpy()
    for host in (torch.from_numpy(f).pin_memory(), f):
        res = S.sas_transform(host, Js, policy="auto", family_meta=meta)
        assert res.plan.mu_star == dev.plan.mu_star > 1
        got = np.asarray(res.coeffs)
        assert np.abs(got - want).max() <= 1e-13 * np.abs(want).max()
        assert res.report.escalated_nodes == dev.report.escalated_nodes
    for b in range(B):
        assert np.linalg.norm(want[b] - coef[b]) / np.linalg.norm(coef[b]) < 1e-4


def test_select_pivots_policies(S):
    # reference tests/test_sas.py TestSelectPivots
    import math
    import structfft_oracle as O
    J = S.SupportSet(32, O.gen_homogeneous((1, 3), 5, 3))
    assert S.select_pivots(J, "auto") == S.pivots(J)
    assert S.select_pivots(S.SupportSet.make(1024, [0, 1, 6, 7, 512]), "auto") == (0, 1)
    jstar = S.SupportSet.make(1 << 10, [1 << i for i in range(10)])
    r = S.select_pivots(jstar, "auto")
    assert r == tuple(range(len(r)))
    with pytest.raises(S.InvalidInputError):
        S.select_pivots(jstar, "uoh")
    with pytest.raises(S.InvalidInputError):
        S.select_pivots(jstar, "balanced")
    with pytest.raises(S.InvalidInputError):
        S.select_pivots(jstar, "nope")
    base = (0, 2, 5, 7, 9)
    K = O.gen_homogeneous(base, 12, 1)
    sub = S.SupportSet(1 << 12, K[:9])
    t = int(math.floor(math.log2(9) - math.log2(math.log2(9))))
    assert S.select_pivots(sub, "random_subset", {"base_pivots": base}) == base[:t]


def test_sas_heavy_nodes_match_reference(S):
    """Node weights above 64 (the CTA-per-node decode path, up to 1024):
    mu* = 100 (one node: the k x k Vandermonde of the submatrix method) and
    prefixes leaving nodes of weight 74-91, band-limited sources with
    double-double escalation, against the unmodified reference
    (tests/golden/make_golden_sas_big.py): plan and node weights identical,
    coefficients equal to the reference's within the accuracy the
    reference's own conditioning leaves (its error against the planted
    spectrum)."""
    import os
    g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_sas_big.npz"))
    for i in range(int(g["n_cases"][0])):
        p = f"b{i}_"
        N, J, c = int(g[p + "N"][0]), g[p + "J"], g[p + "c"]
        r = tuple(int(x) for x in g[p + "r"])
        Js = S.SupportSet(N, J)
        res = S.sas_transform(S.BandlimitedSignal(Js, c), Js, r=r, policy="balanced", family_meta={"pivots": r})
        assert (res.plan.decode_level, res.plan.mu_star) == tuple(int(x) for x in g[p + "plan"])
        assert res.plan.node_weights == tuple(int(x) for x in g[p + "weights"])
        got = res.coeffs.detach().cpu().numpy() if hasattr(res.coeffs, "detach") else np.asarray(res.coeffs)
        want = g[p + "coeffs"]
        ref_err = float(np.max(np.abs(want - c)))
        diff = float(np.max(np.abs(got - want)))
        assert diff <= max(1e-8, 2.0 * ref_err), (i, diff, ref_err)
