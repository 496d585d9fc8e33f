"""Pin the CPU oracle against golden vectors produced by the reference.

The golden files come from tests/golden/make_golden.py, which imports the
unmodified reference package; here only the committed fixtures are read.
"""

import hashlib

import numpy as np
import pytest

import structfft_oracle as O


def test_pivots_and_classify(kats):
    for case in kats["pivots"]:
        N, J = case["N"], np.asarray(case["J"], np.int64)
        M = N.bit_length() - 1
        assert O.pivots(J, M) == tuple(case["pivots"]), case
        assert O.is_homogeneous(J, M) == (case["kind"] == "homogeneous")
        if len(J) <= 64:
            assert O.pivots_pairwise(J) == tuple(case["pivots"])


def test_paper_pivot_fixtures():
    # tests/test_congruence.py:106-112
    assert O.pivots([3, 17, 25, 27], 5) == (1, 3)
    assert O.pivots([23, 187, 190, 247, 386, 731, 990, 994], 10) == (0, 2, 5)
    assert O.pivots([84, 305, 725, 992], 10) == (0, 2)
    assert O.pivots([9], 4) == ()


def test_part_homogeneity(kats):
    for case in kats["part_homogeneous"]:
        M = case["N"].bit_length() - 1
        ok = O.part_homogeneity_violation(case["J"], M, case["r"]) is None
        assert ok == case["ok"]


def test_patterns(kats):
    for case in kats["patterns"]:
        got = O.pivoted_pattern(case["r"], case["M"])
        assert got.tolist() == case["I"]


def test_pattern_edge_cases():
    assert O.pivoted_pattern((0, 2), 10).tolist() == [0, 128, 512, 640]
    assert O.pivoted_pattern((), 6).tolist() == [0]
    with pytest.raises(O.OracleError):
        O.pivoted_pattern((6,), 6)
    with pytest.raises(O.OracleError):
        O.pivoted_pattern((2, 1), 6)


def test_hidft_cases(golden_hidft):
    g = golden_hidft
    for i in range(int(g["n_cases"][0])):
        p = f"c{i}_"
        N, n, a, level, adds, mults = (int(x) for x in g[p + "meta"])
        M = N.bit_length() - 1
        J, r, f = g[p + "J"], tuple(int(x) for x in g[p + "r"]), g[p + "f"]
        out = O.hidft(f, J, M, r, n, a)
        assert out.level == level
        assert np.array_equal(out.node_residues, g[p + "node_residues"])
        assert np.array_equal(out.slot_residues, g[p + "slot_residues"])
        assert np.array_equal(out.slot_real, g[p + "slot_real"])
        assert (out.ops_adds, out.ops_mults) == (adds, mults)
        plan = O.build_plan(J, M, r[: len(r) - n])
        assert np.array_equal(plan.element_slots, g[p + "element_slots"])
        tw = np.concatenate(plan.twiddles) if plan.twiddles else np.zeros(0, complex)
        assert np.array_equal(tw, g[p + "twiddles"])
        np.testing.assert_allclose(out.node_values, g[p + "node_values"], rtol=0, atol=1e-12 * max(1.0, np.abs(g[p + "node_values"]).max()))
        np.testing.assert_allclose(out.slot_values, g[p + "slot_values"], rtol=0, atol=1e-12 * max(1.0, np.abs(g[p + "slot_values"]).max()))
        if p + "dft" in g:
            d = O.hidft_to_dft(f, J, M)
            rel = np.linalg.norm(d - g[p + "dft"]) / np.linalg.norm(g[p + "dft"])
            assert rel < 1e-13


def test_dense_oracle_agrees(golden_hidft):
    g = golden_hidft
    for i in range(0, int(g["n_cases"][0]), 3):
        p = f"c{i}_"
        N, n, a = (int(x) for x in g[p + "meta"][:3])
        M = N.bit_length() - 1
        r = tuple(int(x) for x in g[p + "r"])
        want = O.dense_submatrix(g[p + "f"], g[p + "J"], M, r, n, a)
        got = g[p + "node_values"]
        assert np.max(np.abs(got - want)) <= 1e-9 * max(1.0, np.abs(want).max())


def test_config_supports(golden_configs):
    g = golden_configs
    for c in (1, 2, 3, 5):
        J, M = O.config_support(c)
        assert np.array_equal(J, g[f"cfg{c}_J"]), c
        assert O.pivots(J, M) == tuple(int(x) for x in g[f"cfg{c}_pivots"])
    h = hashlib.sha256()
    for b in range(256):
        J, M = O.config_support(4, b)
        if b < 8:
            assert np.array_equal(J, g[f"cfg4_J{b}"])
        h.update(J.astype("<i8").tobytes())
    assert h.digest() == bytes(g["cfg4_sha256_first256"])


@pytest.mark.parametrize("c", [1, 2, 3, 4])
def test_config_outputs(golden_configs, c):
    g = golden_configs
    dt = {1: np.complex128, 2: np.complex64, 3: np.complex64, 4: np.complex64}[c]
    for b in range(2):
        J, M = O.config_support(c, b)
        coef = O.config_coefficients(c, b, len(J))
        np.testing.assert_array_equal(coef, g[f"cfg{c}_b{b}_coef"])
        f = O.synthesize(J, coef, M).astype(dt)
        got = O.sas_mu1(f, J, M) if c == 3 else O.hidft_to_dft(f, J, M)
        want = g[f"cfg{c}_b{b}_out"]
        assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-13
        # and the planted spectrum is recovered to the dtype's precision
        tol = 1e-11 if dt == np.complex128 else 1e-5
        assert np.linalg.norm(got - coef) / np.linalg.norm(coef) < tol


def test_reference_call_shapes_match():
    J, M = O.config_support(1)
    coef = O.config_coefficients(1, 0, len(J))
    f = O.synthesize(J, coef, M)
    a = O.reference_call(f, J, M)
    b = O.hidft_to_dft(f, J, M)
    assert np.array_equal(a, b)
    c = O.reference_sas_call(f, J, M)
    assert np.linalg.norm(c - b) / np.linalg.norm(b) < 1e-14


@pytest.mark.parametrize("case", ["cfg1", "cfg2", "cfg3", "cfg5", "cfg4_b0", "cfg4_b1"])
def test_plan_tables_at_config_size_match_reference_digests(plan_digests, case):
    """The oracle's plan restatement at the BASELINE config sizes (up to 2^16
    slots) against digests of the unmodified reference's own tables: supports,
    pivots, level, element_slots, slot_residues, slot_real, node_residues and
    slot-order offsets bit-exact (sha256), sampled twiddles to 1e-15."""
    from conftest import table_digest, twiddle_sample_index
    want = plan_digests[case]
    cfg = int(case[3])
    J, M = O.config_support(cfg, int(case[-1]) if "_b" in case else 0)
    assert M == want["M"] and J.size == want["k"]
    assert table_digest(J, "<i8") == want["sha256"]["J"]
    r = O.pivots(J, M)
    assert list(r) == want["pivots"]
    plan = O.build_plan(J, M, r)
    assert plan.level == want["level"]
    for name, arr, dt in (("element_slots", plan.element_slots, "<i8"), ("slot_residues", plan.slot_residues, "<i8"),
                          ("slot_real", plan.slot_real, "u1"), ("node_residues", plan.node_residues, "<i8"),
                          ("offsets", plan.offsets, "<i8")):
        assert table_digest(arr, dt) == want["sha256"][name], name
    tw = np.concatenate(plan.twiddles)
    assert tw.size == want["twiddle_count"]
    ref = np.array([complex(float.fromhex(a), float.fromhex(b)) for a, b in want["twiddle_sample"]])
    assert np.max(np.abs(tw[twiddle_sample_index(tw.size)] - ref)) < 1e-15
