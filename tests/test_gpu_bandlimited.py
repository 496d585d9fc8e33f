"""Band-limited sources synthesised on the device, and the reference's own
hidft/sas identities on them (reference tests/test_hidft.py, tests/test_sas.py)."""

import numpy as np
import pytest

import structfft_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2211_15299_b200 as S
    return S


rng = np.random.default_rng(99)


def rel_error(got, want, floor=1e-30):
    """Max entrywise relative error (reference core.py:218-223)."""
    got = np.asarray(got, np.complex128)
    want = np.asarray(want, np.complex128)
    return float(np.max(np.abs(got - want) / np.maximum(np.abs(want), floor))) if got.size else 0.0


def oracle_samples(J, c, N, loc):
    """(1/N) sum c_l exp(+2 pi i (loc*l mod N)/N), by definition (core.py:164-173)."""
    ph = np.exp(2j * np.pi * ((np.outer(loc, J) % N) / N))
    return ph @ c / N


def random_homogeneous(M_hi=12, s_hi=8):
    M = int(rng.integers(2, M_hi))
    s = int(rng.integers(1, min(M, s_hi) + 1))
    pivs = sorted(rng.choice(M, size=s, replace=False).tolist())
    return O.gen_homogeneous(pivs, M, int(rng.integers(0, 2 ** 62))), M, tuple(pivs)


def test_sample_block_matches_definition(S):
    for M, k, n in [(5, 7, 32), (12, 100, 500), (20, 1024, 2048), (26, 4096, 1000), (31, 64, 300)]:
        J = np.sort(rng.choice(1 << min(M, 20), size=k, replace=False)) << max(0, M - 20)
        c = rng.normal(size=k) + 1j * rng.normal(size=k)
        sig = S.BandlimitedSignal(S.SupportSet(1 << M, J), c)
        loc = rng.integers(0, 1 << M, size=n)
        got = sig.sample_block(loc)
        want = oracle_samples(J, c, 1 << M, loc)
        assert np.max(np.abs(got - want)) <= 1e-12 * max(1.0, np.abs(want).max()), M
    sig = S.BandlimitedSignal(S.SupportSet(16, [0, 3]), [1.0, 2.0j])
    assert np.allclose(sig.synthesize(), oracle_samples(np.array([0, 3]), np.array([1.0, 2.0j]), 16, np.arange(16)))
    with pytest.raises(S.InvalidInputError):
        S.BandlimitedSignal(S.SupportSet(16, [0, 3]), [1.0])
    with pytest.raises(S.InvalidInputError):
        sig.coeff(5)


def test_random_homogeneous_vs_planted(S):
    # tests/test_hidft.py:120-126
    for _ in range(100):
        J, M, piv = random_homogeneous()
        c = rng.normal(size=J.size) + 1j * rng.normal(size=J.size)
        sig = S.BandlimitedSignal(S.SupportSet(1 << M, J), c)
        ctr = S.OpCounter()
        Js = S.SupportSet(1 << M, J)
        rec = S.hidft_to_dft(S.hidft(sig, Js, S.pivots(Js), counter=ctr), counter=ctr)
        assert rel_error(rec, c, floor=1e-9) < 1e-9


def test_paper_eight_point_fixture(S):
    # tests/test_hidft.py:111-118
    Js = S.SupportSet.make(1024, [23, 187, 190, 247, 386, 731, 990, 994])
    assert S.classify(Js).is_homogeneous and S.pivots(Js) == (0, 2, 5)
    c = rng.normal(size=8) + 1j * rng.normal(size=8)
    sig = S.BandlimitedSignal(Js, c)
    rec = S.hidft_to_dft(S.hidft(sig, Js, (0, 2, 5)))
    assert rel_error(rec, c) < 1e-9
    full = np.fft.fft(sig.synthesize())
    assert rel_error(rec, full[list(Js.indices)]) < 1e-9


def test_tree_weight_identity(S):
    # tests/test_hidft.py:149-170: node value = (|I|/N) sum_{l in node} e^{-2 pi i a l/N} c_l
    for N, idx, r in [(64, [3, 17, 25, 27, 35], (1, 3)), (1024, [0, 1, 6, 7, 512], (0, 1))]:
        Js = S.SupportSet.make(N, idx)
        c = rng.normal(size=len(idx)) + 1j * rng.normal(size=len(idx))
        sig = S.BandlimitedSignal(Js, c)
        for n in range(len(r) + 1):
            for a in (0, 3):
                res = S.hidft(sig, Js, r, height=n, shift=a)
                scale = (1 << (len(r) - n)) / N
                mod = 1 << res.level
                for resid in res.node_residues:
                    members = [l for l in idx if l % mod == resid]
                    want = scale * sum(c[idx.index(l)] * np.exp(-2j * np.pi * a * l / N) for l in members)
                    got = res.values[resid]
                    assert abs(got - want) <= 1e-9 * max(abs(want), 1e-9)


def test_split_identity(S):
    # tests/test_hidft.py:174-186
    Js = S.SupportSet.make(32, [3, 17, 25, 27])
    c = rng.normal(size=4) + 1j * rng.normal(size=4)
    sig = S.BandlimitedSignal(Js, c)
    res1 = S.hidft(sig, Js, (1, 3), height=1)
    for sub in ([3, 17], [25, 27]):
        res0 = S.hidft(sig, S.SupportSet.make(32, sub), (1,), height=0)
        for j in sub:
            assert abs(res1.value_at_index(j) - res0.value_at_index(j)) < 1e-10


def test_elementary_equals_downsample_fft(S):
    # tests/test_hidft.py:128-139 (gen_elementary(3, 6, seed=5): one element per class mod 8)
    M, rr = 6, 3
    g = O.rng_from_seed(5, 0)
    highs = g.integers(0, 1 << (M - rr), size=1 << rr)
    J = np.sort((np.arange(1 << rr) + (highs << rr)) % (1 << M))
    Js = S.SupportSet(1 << M, J)
    c = rng.normal(size=8) + 1j * rng.normal(size=8)
    sig = S.BandlimitedSignal(Js, c)
    res = S.hidft(sig, Js, (0, 1, 2))
    down = sig.sample_block(np.arange(8) * 8)
    small = np.fft.fft(down)
    for j in J:
        assert abs(res.value_at_index(int(j)) - small[int(j) % 8]) < 1e-10
    assert rel_error(S.hidft_to_dft(res), c) < 1e-9


def test_sas_homogeneous_equals_hidft_path(S):
    # tests/test_sas.py:132-143
    for _ in range(20):
        M = int(rng.integers(2, 10))
        s = int(rng.integers(1, min(M, 6) + 1))
        pivs = sorted(rng.choice(M, size=s, replace=False).tolist())
        J = O.gen_homogeneous(pivs, M, int(rng.integers(0, 2 ** 60)))
        Js = S.SupportSet(1 << M, J)
        mag = 0.5 + rng.random(J.size)
        c = mag * np.exp(1j * rng.random(J.size) * 2 * np.pi)
        sig = S.BandlimitedSignal(Js, c)
        out = S.sas_transform(sig, Js)
        assert out.plan.mu_star == 1
        direct = S.hidft_to_dft(S.hidft(sig, Js, tuple(pivs)))
        assert rel_error(out.coeffs, direct, floor=1e-9) < 1e-12
        assert rel_error(out.coeffs, c) < 1e-8


def test_reference_style_counts(S):
    # tests/test_hidft.py:190-209: exactly 1.5 A log2 A, padding branches counted
    for _ in range(40):
        J, M, piv = random_homogeneous(M_hi=9, s_hi=6)
        Js = S.SupportSet(1 << M, J)
        c = rng.normal(size=J.size) + 1j * rng.normal(size=J.size)
        n = int(rng.integers(0, len(piv) + 1))
        ctr = S.OpCounter()
        S.hidft(S.BandlimitedSignal(Js, c), Js, piv, height=n, shift=int(rng.integers(0, 1 << M)), counter=ctr)
        A, logA = 1 << (len(piv) - n), len(piv) - n
        assert ctr.total == round(1.5 * A * logA)
    ctr = S.OpCounter()
    Js = S.SupportSet.make(8, [0, 1, 3])
    S.hidft(S.BandlimitedSignal(Js, [1.0, 2.0, 3.0]), Js, (0, 1), counter=ctr)
    assert ctr.total == round(1.5 * 4 * 2)
