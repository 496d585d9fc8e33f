"""Parity of the CUDA path against the oracle and the reference's golden vectors.

Index sets are compared bit-exactly; coefficients by relative L2 error,
||got - want|| / ||want||, with the north-star tolerances: 1e-5 for
complex64 and 1e-11 for complex128 (BASELINE.json north_star).
"""

import numpy as np
import pytest

import structfft_oracle as O

pytestmark = pytest.mark.gpu

TOL = {np.complex64: 1e-5, np.complex128: 1e-11}


@pytest.fixture(scope="module")
def S():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2211_15299_b200 as S
    return S


@pytest.fixture(scope="module")
def torch():
    import torch
    return torch


def rel_l2(got, want):
    got = np.asarray(got, np.complex128)
    want = np.asarray(want, np.complex128)
    return float(np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-300))


# --------------------------------------------------------------- indices ---

def test_pivots_kats(S, kats):
    for case in kats["pivots"]:
        J = S.SupportSet.make(case["N"], case["J"])
        assert S.pivots(J) == tuple(case["pivots"]), case
        assert S.classify(J).kind == case["kind"]


def test_paper_pivot_fixtures(S):
    assert S.pivots(S.SupportSet.make(32, [3, 17, 25, 27])) == (1, 3)
    assert S.pivots(S.SupportSet.make(1024, [23, 187, 190, 247, 386, 731, 990, 994])) == (0, 2, 5)
    assert S.pivots(S.SupportSet.make(1024, [84, 305, 725, 992])) == (0, 2)
    assert S.pivots(S.SupportSet.make(16, [9])) == ()
    J = S.SupportSet.make(64, [3, 17, 25, 27, 35])
    assert S.is_part_homogeneous(J, (1, 3)) and not S.is_part_homogeneous(J, (3,))
    with pytest.raises(S.ContractViolationError):
        S.assert_part_homogeneous(J, (3,))


def test_pivots_random_large(S):
    rng = np.random.default_rng(5)
    for M, k in [(20, 4096), (26, 65536), (31, 1000), (16, 1 << 16)]:
        J = np.sort(rng.choice(1 << M, size=k, replace=False))
        assert S.pivots(S.SupportSet(1 << M, J)) == O.pivots(J, M)
    for cfg in (1, 2, 3, 5):
        J, M = O.config_support(cfg)
        assert S.pivots(S.SupportSet(1 << M, J)) == O.pivots(J, M)


def test_patterns(S, kats):
    for case in kats["patterns"]:
        assert list(S.pivoted_pattern(case["r"], case["M"]).samples) == case["I"]
    with pytest.raises(S.InvalidInputError):
        S.pivoted_pattern((6,), 6)


def test_plan_tables_bit_exact(S, golden_hidft):
    g = golden_hidft
    for i in range(int(g["n_cases"][0])):
        p = f"c{i}_"
        N, n = int(g[p + "meta"][0]), int(g[p + "meta"][1])
        J = S.SupportSet(N, g[p + "J"])
        r = tuple(int(x) for x in g[p + "r"])
        for code in (0, 1):
            plan = S.get_plan(J, r, n, code, S._lib.require_device())
            t = plan.tables()
            assert plan.level == int(g[p + "meta"][3])
            assert np.array_equal(t["element_slots"], g[p + "element_slots"])
            assert np.array_equal(t["slot_residues"], g[p + "slot_residues"])
            assert np.array_equal(t["slot_real"], g[p + "slot_real"])
            assert np.array_equal(t["node_residues"], g[p + "node_residues"])
            used = r[: len(r) - n]
            assert np.array_equal(t["offsets"], O.slot_offsets(used, J.M))
            want_tw = g[p + "twiddles"]
            tol = 1e-15 if code == 1 else 1e-7
            if want_tw.size:
                assert np.max(np.abs(t["twiddles"] - want_tw)) < tol


# ------------------------------------------------------------ transforms ---

@pytest.mark.parametrize("dt", [np.complex128, np.complex64])
def test_hidft_golden_cases(S, golden_hidft, torch, dt):
    g = golden_hidft
    for i in range(int(g["n_cases"][0])):
        p = f"c{i}_"
        N, n, a, level, adds, mults = (int(x) for x in g[p + "meta"])
        J = S.SupportSet(N, g[p + "J"])
        r = tuple(int(x) for x in g[p + "r"])
        f = g[p + "f"].astype(dt)
        res = S.hidft(torch.from_numpy(f).cuda(), J, r, height=n, shift=a)
        assert res.node_residues == tuple(int(x) for x in g[p + "node_residues"])
        assert (res.ops_adds, res.ops_mults) == (adds, mults)
        nodes = res.node_values.cpu().numpy()
        if dt == np.complex128:
            want = g[p + "node_values"]
            want_slots = g[p + "slot_values"]
        else:  # the oracle on the identical complex64 samples
            o = O.hidft(f, g[p + "J"], N.bit_length() - 1, r, n, a)
            want, want_slots = o.node_values, o.slot_values
        assert rel_l2(nodes, want) < TOL[dt], (i, rel_l2(nodes, want))
        assert rel_l2(res.slot_values.cpu().numpy(), want_slots) < TOL[dt]
        if p + "dft" in g:
            res0 = S.hidft(torch.from_numpy(f).cuda(), J, S.pivots(J))
            d = S.hidft_to_dft(res0).cpu().numpy()
            want_d = g[p + "dft"] if dt == np.complex128 else O.hidft_to_dft(f, g[p + "J"], N.bit_length() - 1)
            assert rel_l2(d, want_d) < TOL[dt]
            fused = S.hidft_to_dft_batched(torch.from_numpy(f).cuda(), J).cpu().numpy()
            assert rel_l2(fused, want_d) < TOL[dt]


def test_numpy_and_callable_sources(S, golden_hidft):
    g = golden_hidft
    for i in range(0, int(g["n_cases"][0]), 5):
        p = f"c{i}_"
        N, n, a = (int(x) for x in g[p + "meta"][:3])
        J = S.SupportSet(N, g[p + "J"])
        r = tuple(int(x) for x in g[p + "r"])
        f = g[p + "f"]
        res = S.hidft(f, J, r, height=n, shift=a)
        assert isinstance(res.node_values, np.ndarray)
        assert rel_l2(res.node_values, g[p + "node_values"]) < 1e-11
        res2 = S.hidft(lambda loc: f[loc], J, r, height=n, shift=a)
        assert rel_l2(res2.node_values, g[p + "node_values"]) < 1e-11
        v = res.values
        assert set(v) == set(res.node_residues)


def test_top_height_is_single_sample(S, torch):
    # tests/test_hidft.py:70-77: shift a at full height reads f(-a)
    rng = np.random.default_rng(3)
    f = rng.normal(size=64) + 1j * rng.normal(size=64)
    J = S.SupportSet.make(64, [3, 17, 25, 27])
    res = S.hidft(f, J, (1, 3), height=2, shift=5)
    assert res.node_residues == (0,)
    assert abs(res.node_values[0] - f[(-5) % 64]) < 1e-12
    assert res.ops_adds == res.ops_mults == 0


@pytest.mark.parametrize("M", [1, 2, 5, 8])
def test_full_support_is_fft(S, M):
    N = 1 << M
    rng = np.random.default_rng(M)
    f = rng.normal(size=N) + 1j * rng.normal(size=N)
    Z = S.SupportSet.make(N, range(N))
    ctr = S.OpCounter()
    res = S.hidft(f, Z, tuple(range(M)), counter=ctr)
    assert rel_l2(res.values_by_index(), np.fft.fft(f)) < 1e-12
    assert ctr.total == round(1.5 * N * M)


def test_contract_errors(S):
    f = np.zeros(64, complex)
    J = S.SupportSet.make(64, [3, 17, 25, 27, 35])
    with pytest.raises(S.ContractViolationError):
        S.hidft(f, J, (3,))
    with pytest.raises(S.InvalidInputError):
        S.hidft(f, J, (1, 3), height=3)
    with pytest.raises(S.InvalidInputError):
        S.hidft(f, J, (3, 1))
    with pytest.raises(S.ContractViolationError):  # tests/test_hidft.py:141-145
        S.hidft_to_dft(S.hidft(f, J, (1, 3)))
    res = S.hidft(np.zeros(32, complex), S.SupportSet.make(32, [3, 17, 25, 27]), (1, 3), height=1)
    with pytest.raises(S.ContractViolationError):
        S.hidft_to_dft(res)
    with pytest.raises(S.InvalidInputError):
        S.hidft(np.zeros(32, complex), J, (1, 3))


def test_dc_singleton(S):
    J = S.SupportSet.make(16, [0])
    f = np.full(16, (3.0 - 2.0j) / 16)
    rec = S.hidft_to_dft(S.hidft(f, J, ()))
    assert abs(rec[0] - (3.0 - 2.0j)) < 1e-12


def _homog_batch(rng, B, M, s, per_signal):
    sup = []
    for b in range(B if per_signal else 1):
        piv = sorted(rng.choice(M, size=s, replace=False).tolist())
        sup.append(O.gen_homogeneous(piv, M, int(rng.integers(0, 2 ** 62))))
    return np.stack(sup)


@pytest.mark.parametrize("dt", [np.complex64, np.complex128])
@pytest.mark.parametrize("s", [0, 1, 3, 4, 5, 8, 10, 12])
def test_fused_random(S, torch, dt, s):
    rng = np.random.default_rng(100 + s)
    M = max(s + 2, 12)
    B = 37
    for per_signal in (False, True):
        sup = _homog_batch(rng, B, M, s, per_signal)
        coef = rng.normal(size=(B, 1 << s)) + 1j * rng.normal(size=(B, 1 << s))
        f = np.zeros((B, 1 << M), np.complex128)
        for b in range(B):
            f[b] = O.synthesize(sup[b if per_signal else 0], coef[b], M)
        f = f.astype(dt)
        Jarg = (torch.from_numpy(sup).cuda() if per_signal else S.SupportSet(1 << M, sup[0]))
        got = S.hidft_to_dft_batched(torch.from_numpy(f).cuda(), Jarg).cpu().numpy()
        for b in range(B):
            want = O.hidft_to_dft(f[b], sup[b if per_signal else 0], M)
            assert rel_l2(got[b], want) < TOL[dt], (b, per_signal)


def test_fused_status_rows(S, torch):
    rng = np.random.default_rng(9)
    M, s, B = 14, 6, 8
    sup = _homog_batch(rng, B, M, s, True)
    bad = sup.copy()
    bad[3, 5] = bad[3, 4]          # duplicate -> invalid row
    bad[5] = np.sort(rng.choice(1 << M, size=1 << s, replace=False))  # generic row
    f = torch.zeros((B, 1 << M), dtype=torch.complex64, device="cuda")
    st = torch.zeros(B, dtype=torch.int32, device="cuda")
    S.hidft_to_dft_batched(f, torch.from_numpy(bad).cuda(), status=st, check=False)
    stat = st.cpu().numpy()
    assert stat[3] == 2 and stat[5] == 3
    assert (np.delete(stat, [3, 5]) == 0).all()
    with pytest.raises(S.InvalidInputError):
        S.hidft_to_dft_batched(f, torch.from_numpy(bad).cuda())
    generic = np.stack([sup[0]] * B)
    generic[:, 0] = (generic[:, 0] + 1) % (1 << M)
    generic.sort(axis=1)
    if len(np.unique(generic[0])) == generic.shape[1]:
        with pytest.raises((S.ContractViolationError, S.InvalidInputError)):
            S.hidft_to_dft_batched(f, torch.from_numpy(generic).cuda())


def test_determinism(S, torch):
    J, M = O.config_support(2)
    coef = O.config_coefficients(2, 0, len(J))
    f = torch.from_numpy(O.synthesize(J, coef, M).astype(np.complex64)).cuda().repeat(64, 1)
    Js = S.SupportSet(1 << M, J)
    a = S.hidft_to_dft_batched(f, Js)
    b = S.hidft_to_dft_batched(f, Js)
    assert torch.equal(a, b)
    assert torch.equal(a[0], a[63])


def test_pinned_zero_copy(S, torch):
    J, M = O.config_support(2)
    coef = np.stack([O.config_coefficients(2, b, len(J)) for b in range(4)])
    f = np.stack([O.synthesize(J, coef[b], M) for b in range(4)]).astype(np.complex64)
    host = torch.from_numpy(f).pin_memory()
    Js = S.SupportSet(1 << M, J)
    got = S.hidft_to_dft_batched(host, Js)
    assert not got.is_cuda
    dev = S.hidft_to_dft_batched(host.cuda(), Js).cpu()
    assert torch.equal(got, dev)
    for b in range(4):
        assert rel_l2(got[b].numpy(), O.hidft_to_dft(f[b], J, M)) < 1e-5


def _check_stage(torch, lib, _lib, plan, f, shift, code, tdt):
    """sfft_host_stage (two shifts, pattern order) + sfft_hidft_staged equal
    the direct-gather transform at shift and shift + 1, bit for bit."""
    B, N = f.shape
    A, nn = plan.A, max(plan.n_nodes, 1)
    sp = _lib.stream_ptr(0)
    rows = torch.empty((2 * B, A), dtype=tdt, device="cuda")
    _lib.check(lib.sfft_host_stage(plan.handle, f.ctypes.data, B, N, code, shift, 2, _lib.ORDER_PATTERN, code,
                                   rows.data_ptr(), A, 3, sp))
    got = torch.empty((2 * B, nn), dtype=tdt, device="cuda")
    _lib.check(lib.sfft_hidft_staged(plan.handle, rows.data_ptr(), 2 * B, A, _lib.ORDER_PATTERN, _lib.OUT_NODES,
                                     got.data_ptr(), nn, None, 0, sp))
    d = torch.from_numpy(f).cuda()
    for j in range(2):
        want = torch.empty((B, nn), dtype=tdt, device="cuda")
        _lib.check(lib.sfft_hidft(plan.handle, d.data_ptr(), B, N, shift + j, _lib.OUT_NODES, want.data_ptr(), nn,
                                  None, 0, sp))
        assert torch.equal(got[j::2], want)


@pytest.mark.parametrize("dt,pinned", [(np.complex64, False), (np.complex128, True)])
def test_hidft_host_capi(S, torch, dt, pinned):
    """sfft_hidft_host: host rows in, host results out (pageable or pinned),
    chunked pipeline with a few workers; bit-identical to the device path."""
    from paper_2211_15299_b200 import _lib
    from paper_2211_15299_b200.hidft import get_plan
    J, M = O.config_support(1)
    N, B, shift = 1 << M, 37, 5
    rng = np.random.default_rng(7)
    f = (rng.standard_normal((B, N)) + 1j * rng.standard_normal((B, N))).astype(dt)
    Js = S.SupportSet(N, J)
    code = _lib.C64 if dt == np.complex64 else _lib.C128
    plan = get_plan(Js, S.pivots(Js), 0, code, torch.device("cuda", 0))
    lib = _lib.load()
    tdt = torch.complex64 if dt == np.complex64 else torch.complex128
    sig = torch.from_numpy(f)
    if pinned:
        sig = sig.pin_memory()
    nn = max(plan.n_nodes, 1)
    out = torch.zeros((B, nn + 3), dtype=tdt, pin_memory=pinned)
    slots = torch.zeros((B, plan.A), dtype=tdt, pin_memory=pinned)
    sp = _lib.stream_ptr(0)
    _lib.check(lib.sfft_hidft_host(plan.handle, sig.data_ptr(), B, N, shift, _lib.OUT_NODES, out.data_ptr(),
                                   nn + 3, slots.data_ptr(), plan.A, 5, 3, sp))
    d = sig.cuda()
    want = torch.zeros((B, nn), dtype=tdt, device="cuda")
    want_s = torch.zeros((B, plan.A), dtype=tdt, device="cuda")
    _lib.check(lib.sfft_hidft(plan.handle, d.data_ptr(), B, N, shift, _lib.OUT_NODES, want.data_ptr(), nn,
                              want_s.data_ptr(), plan.A, sp))
    torch.cuda.synchronize()
    assert torch.equal(out[:, :nn], want.cpu())
    assert torch.equal(out[:, nn:], torch.zeros((B, 3), dtype=tdt))
    assert torch.equal(slots, want_s.cpu())
    # DFT output kind, default chunking and threads
    coeffs = torch.zeros((B, len(J)), dtype=tdt)
    _lib.check(lib.sfft_hidft_host(plan.handle, sig.data_ptr(), B, N, 0, _lib.OUT_DFT, coeffs.data_ptr(),
                                   len(J), None, 0, 0, 0, sp))
    for b in (0, B - 1):
        assert rel_l2(coeffs[b].numpy(), O.hidft_to_dft(f[b], J, M)) < TOL[dt]
    _check_stage(torch, lib, _lib, plan, f, shift, code, tdt)


@pytest.mark.parametrize("dt,s", [(np.complex64, 15), (np.complex64, 16), (np.complex128, 14)])
def test_gathered_split_paths(S, torch, dt, s):
    """2^s beyond one CTA (two-pass split transform): host rows through
    sfft_hidft_host (sorted-order staging) and device rows pre-gathered in
    slot order through sfft_hidft_gathered match the direct-gather launch
    bit for bit."""
    from paper_2211_15299_b200 import _lib
    from paper_2211_15299_b200.hidft import get_plan
    M, B, shift = 20, 3, 11
    N = 1 << M
    J = np.arange(1 << s, dtype=np.int64) * 4 + 1  # homogeneous, pivots 2..s+1
    rng = np.random.default_rng(s)
    f = (rng.standard_normal((B, N)) + 1j * rng.standard_normal((B, N))).astype(dt)
    Js = S.SupportSet(N, J)
    code = _lib.C64 if dt == np.complex64 else _lib.C128
    tdt = torch.complex64 if dt == np.complex64 else torch.complex128
    plan = get_plan(Js, S.pivots(Js), 0, code, torch.device("cuda", 0))
    assert plan.A == 1 << s
    lib = _lib.load()
    sp = _lib.stream_ptr(0)
    d = torch.from_numpy(f).cuda()
    want = torch.empty((B, len(J)), dtype=tdt, device="cuda")
    _lib.check(lib.sfft_hidft(plan.handle, d.data_ptr(), B, N, 0, _lib.OUT_DFT, want.data_ptr(), len(J),
                              None, 0, sp))
    host = torch.empty((B, len(J)), dtype=tdt)
    _lib.check(lib.sfft_hidft_host(plan.handle, torch.from_numpy(f).data_ptr(), B, N, 0, _lib.OUT_DFT,
                                   host.data_ptr(), len(J), None, 0, 0, 0, sp))
    assert torch.equal(host, want.cpu())
    # slot-order pre-gathered rows, with a shift
    loc = torch.from_numpy((plan.tables()["offsets"] - shift) % N).cuda()
    g = d[:, loc].contiguous()
    nodes_d = torch.empty((B, plan.n_nodes), dtype=tdt, device="cuda")
    nodes_g = torch.empty_like(nodes_d)
    _lib.check(lib.sfft_hidft(plan.handle, d.data_ptr(), B, N, shift, _lib.OUT_NODES, nodes_d.data_ptr(),
                              plan.n_nodes, None, 0, sp))
    _lib.check(lib.sfft_hidft_gathered(plan.handle, g.data_ptr(), B, plan.A, _lib.OUT_NODES, nodes_g.data_ptr(),
                                       plan.n_nodes, None, 0, sp))
    torch.cuda.synchronize()
    assert torch.equal(nodes_g, nodes_d)
    b = B - 1
    assert rel_l2(want[b].cpu().numpy(), O.hidft_to_dft(f[b], J, M)) < TOL[dt]
    _check_stage(torch, lib, _lib, plan, f, shift, code, tdt)


@pytest.mark.parametrize("s", [10, 14, 16])
def test_hidft_shifts_promoted(S, torch, s):
    """sfft_hidft_shifts (the SAS shifted transforms, sas.py:343-345): a
    complex128 plan over complex64 rows, nshift shifts in one launch, equals
    per-shift transforms of the promoted rows bit for bit, on the single-CTA
    (s = 10) and split (s = 14, 16) paths."""
    from paper_2211_15299_b200 import _lib
    from paper_2211_15299_b200.hidft import get_plan
    M, B, mu, shift0 = 20, 3, 3, 5
    N = 1 << M
    J = np.arange(1 << s, dtype=np.int64) * 8 + 3
    rng = np.random.default_rng(100 + s)
    f = (rng.standard_normal((B, N)) + 1j * rng.standard_normal((B, N))).astype(np.complex64)
    Js = S.SupportSet(N, J)
    plan = get_plan(Js, S.pivots(Js), 0, _lib.C128, torch.device("cuda", 0))
    lib = _lib.load()
    sp = _lib.stream_ptr(0)
    nn = plan.n_nodes
    d64 = torch.from_numpy(f).cuda()
    d128 = d64.to(torch.complex128)
    got = torch.empty((B * mu, nn), dtype=torch.complex128, device="cuda")
    _lib.check(lib.sfft_hidft_shifts(plan.handle, d64.data_ptr(), B, N, _lib.C64, shift0, mu, _lib.OUT_NODES,
                                     got.data_ptr(), nn, sp))
    for j in range(mu):
        want = torch.empty((B, nn), dtype=torch.complex128, device="cuda")
        _lib.check(lib.sfft_hidft(plan.handle, d128.data_ptr(), B, N, shift0 + j, _lib.OUT_NODES, want.data_ptr(),
                                  nn, None, 0, sp))
        assert torch.equal(got[j::mu], want), j
    # and against the oracle for one row / shift: node values x N/k = planted DFT of the shifted row
    b, j = B - 1, mu - 1
    fs = np.roll(f[b].astype(np.complex128), shift0 + j)
    want_dft = O.hidft_to_dft(fs, J, M)
    got_dft = got[b * mu + j].cpu().numpy() * (N / len(J))
    assert rel_l2(got_dft, want_dft) < 1e-11


def test_plan_batched_capi(S, torch):
    """sfft_plan_batched (per-signal supports, config 4 shape) + sfft_hidft
    equals sfft_hidft_to_dft_fused bit for bit; the plan is rejected by every
    other entry point and bad supports come back as status 2 / 3."""
    import ctypes
    from paper_2211_15299_b200 import _lib, workloads as W
    wl = W.make_workload(4, 8)
    B, k, M = wl.B, wl.k, wl.M
    N = 1 << M
    sig = torch.empty((B, N), dtype=torch.complex64, device="cuda")
    W.synthesize_into(sig, wl.support, wl.coeffs)
    lib = _lib.load()
    sp = _lib.stream_ptr(0)
    Jh = np.ascontiguousarray(wl.support, dtype=np.int64)
    plan = ctypes.c_void_p()
    _lib.check(lib.sfft_plan_batched(Jh.ctypes.data, k, B, M, _lib.C64, sp, ctypes.byref(plan)))
    try:
        info = _lib.PlanInfo()
        _lib.check(lib.sfft_plan_get_info(plan, ctypes.byref(info)))
        assert info.per_signal == 1 and info.k == k and info.A == k
        got = torch.empty((B, k), dtype=torch.complex64, device="cuda")
        _lib.check(lib.sfft_hidft(plan, sig.data_ptr(), B, N, 0, _lib.OUT_DFT, got.data_ptr(), k, None, 0, sp))
        want = torch.empty_like(got)
        Jd = torch.from_numpy(Jh).cuda()
        _lib.check(lib.sfft_hidft_to_dft_fused(Jd.data_ptr(), k, B, M, sig.data_ptr(), B, N, _lib.C64,
                                               want.data_ptr(), k, None, sp))
        torch.cuda.synchronize()
        assert torch.equal(got, want)
        for b in (0, B - 1):
            assert rel_l2(got[b].cpu().numpy(), wl.coeffs[b]) < 1e-5
        # wrong kinds / sizes / entry points
        assert lib.sfft_hidft(plan, sig.data_ptr(), B, N, 0, _lib.OUT_NODES, got.data_ptr(), k, None, 0, sp) == 2
        assert lib.sfft_hidft(plan, sig.data_ptr(), B - 1, N, 0, _lib.OUT_DFT, got.data_ptr(), k, None, 0, sp) == 2
        assert lib.sfft_hidft_gathered(plan, sig.data_ptr(), B, N, _lib.OUT_DFT, got.data_ptr(), k, None, 0, sp) == 2
        assert lib.sfft_plan_tables(plan, None, None, None, None, None, None, sp) == 2
        assert lib.sfft_plan_nodes(plan, None, None, sp) == 2
    finally:
        lib.sfft_plan_destroy(plan)
    # a non-homogeneous row: contract status naming the support
    bad = Jh.copy()
    bad[3, 0] = (bad[3, 0] + 1) % N
    bad[3].sort()
    if len(np.unique(bad[3])) == k:
        p2 = ctypes.c_void_p()
        _lib.check(lib.sfft_plan_batched(bad.ctypes.data, k, B, M, _lib.C64, sp, ctypes.byref(p2)))
        try:
            out = torch.empty((B, k), dtype=torch.complex64, device="cuda")
            rc = lib.sfft_hidft(p2, sig.data_ptr(), B, N, 0, _lib.OUT_DFT, out.data_ptr(), k, None, 0, sp)
            assert rc in (2, 3) and b"support 3" in lib.sfft_last_error()
        finally:
            lib.sfft_plan_destroy(p2)


def test_edge_batches_strides_shifts(S, torch):
    """Empty batch, padded rows (ld > N), numpy input, and shifts outside
    [0, N) (taken mod N, as the reference's (I - a) mod N does)."""
    from paper_2211_15299_b200 import _lib
    from paper_2211_15299_b200.hidft import get_plan
    J, M = O.config_support(2)
    N = 1 << M
    Js = S.SupportSet(N, J)
    empty = torch.empty((0, N), dtype=torch.complex64, device="cuda")
    assert S.hidft_to_dft_batched(empty, Js).shape == (0, len(J))
    coef = np.stack([O.config_coefficients(2, b, len(J)) for b in range(3)])
    f = np.stack([O.synthesize(J, coef[b], M) for b in range(3)]).astype(np.complex64)
    wide = torch.zeros((3, N + 64), dtype=torch.complex64, device="cuda")
    wide[:, :N] = torch.from_numpy(f).cuda()
    got = S.hidft_to_dft_batched(wide[:, :N], Js)           # row stride N + 64, no copy
    want = S.hidft_to_dft_batched(torch.from_numpy(f).cuda(), Js)
    assert torch.equal(got, want)
    assert torch.equal(torch.as_tensor(S.hidft_to_dft_batched(f, Js)), want.cpu())  # numpy rows
    plan = get_plan(Js, S.pivots(Js), 0, _lib.C64, torch.device("cuda", 0))
    lib, sp = _lib.load(), _lib.stream_ptr(0)
    d = torch.from_numpy(f).cuda()
    outs = []
    for shift in (5, 5 - N, 5 + 3 * N, -(1 << 40) + 5 + (1 << 40) // N * N):
        o = torch.empty((3, plan.n_nodes), dtype=torch.complex64, device="cuda")
        _lib.check(lib.sfft_hidft(plan.handle, d.data_ptr(), 3, N, shift, _lib.OUT_NODES, o.data_ptr(),
                                  plan.n_nodes, None, 0, sp))
        outs.append(o)
    for o in outs[1:]:
        assert torch.equal(o, outs[0])


def test_largest_modulus(S, torch):
    """N = 2^31 (the device path's int32 index limit): one complex64 row of
    16 GiB, samples planted at the pattern offsets, planted spectrum back."""
    free = torch.cuda.mem_get_info()[0]
    if free < 20 * 2**30:
        pytest.skip("needs 20 GiB of free device memory")
    M, N = 31, 1 << 31
    J = O.gen_homogeneous((0, 5, 17, 30), M, 7)
    Js = S.SupportSet(N, J)
    rng = np.random.default_rng(31)
    c = rng.standard_normal(len(J)) + 1j * rng.standard_normal(len(J))
    pat = S.pivoted_pattern(S.pivots(Js), M).as_array()
    n = pat.astype(np.int64)
    vals = (np.exp(2j * np.pi * ((n[:, None] * J[None, :]) % N) / N) @ c) / N   # f at the samples
    sig = torch.zeros((1, N), dtype=torch.complex64, device="cuda")
    sig[0, torch.from_numpy(n).cuda()] = torch.from_numpy(vals.astype(np.complex64)).cuda()
    got = S.hidft_to_dft_batched(sig, Js)[0].cpu().numpy()
    assert rel_l2(got, c) < 1e-5
    del sig
    torch.cuda.empty_cache()


@pytest.mark.parametrize("pinned", [False, True])
def test_per_signal_host_rows(S, torch, pinned):
    """Config-4 shape with host rows: host-derived pivots + host gather +
    on-chip plans (sfft_hidft_to_dft_fused_host) equal the device-resident
    fused transform bit for bit; a non-homogeneous row raises the contract error."""
    from paper_2211_15299_b200 import workloads as W
    wl = W.make_workload(4, 40)
    sig = torch.empty((wl.B, 1 << wl.M), dtype=torch.complex64, device="cuda")
    W.synthesize_into(sig, wl.support, wl.coeffs)
    Jt = torch.from_numpy(wl.support)
    want = S.hidft_to_dft_batched(sig, Jt.cuda())
    host = sig.cpu()
    if pinned:
        host = host.pin_memory()
    got = S.hidft_to_dft_batched(host, Jt)
    assert not got.is_cuda
    assert torch.equal(got, want.cpu())
    got_np = S.hidft_to_dft_batched(host.numpy(), wl.support)   # numpy rows and supports
    assert torch.equal(torch.as_tensor(got_np), want.cpu())
    bad = wl.support.copy()
    bad[7, 0] = (bad[7, 0] + 1) % (1 << wl.M)
    bad[7].sort()
    if len(np.unique(bad[7])) == bad.shape[1]:
        with pytest.raises((S.ContractViolationError, S.InvalidInputError)):
            S.hidft_to_dft_batched(host, torch.from_numpy(bad))


# ------------------------------------------------- configs at full size ---

def _synth(torch, S, cfg, B, per_signal_rows=None):
    from paper_2211_15299_b200 import workloads as W
    wl = W.make_workload(cfg, B)
    dt = torch.complex64 if wl.dtype == "complex64" else torch.complex128
    sig = torch.empty((B, wl.N), dtype=dt, device="cuda")
    W.synthesize_into(sig, wl.support, wl.coeffs)
    return wl, sig


def _check_rows(wl, sig, got, rows, oracle_fn, tol):
    for b in rows:
        f = sig[b].cpu().numpy()
        J = wl.support if wl.support.ndim == 1 else wl.support[b]
        want = oracle_fn(f, J, wl.M)
        assert rel_l2(got[b], want) < tol, (wl.cfg, b, rel_l2(got[b], want))


@pytest.mark.parametrize("cfg", [1, 2, 4])
def test_config_full_batch(S, torch, golden_configs, cfg):
    from paper_2211_15299_b200 import workloads as W
    B = W.CONFIGS[cfg]["B"]
    wl, sig = _synth(torch, S, cfg, B)
    Jarg = (S.SupportSet(wl.N, wl.support) if wl.support.ndim == 1
            else torch.from_numpy(wl.support).cuda())
    got = S.hidft_to_dft_batched(sig, Jarg).cpu().numpy()
    tol = TOL[np.complex64 if wl.dtype == "complex64" else np.complex128]
    # size-independent property over the whole batch: planted spectrum recovered
    err = np.linalg.norm(got - wl.coeffs, axis=1) / np.linalg.norm(wl.coeffs, axis=1)
    assert err.max() < tol
    # oracle parity on a seeded subset of rows, golden rows pinned to the reference
    rows = sorted(set(np.random.default_rng(cfg).choice(B, size=min(B, 8), replace=False).tolist()) | {0, 1})
    _check_rows(wl, sig, got, rows, O.hidft_to_dft, tol)
    for b in (0, 1):
        ref = golden_configs[f"cfg{cfg}_b{b}_out"]
        assert rel_l2(got[b], ref) < max(tol, 1e-6 if wl.dtype == "complex64" else 1e-12)


def test_config3_sas(S, torch, golden_configs):
    from paper_2211_15299_b200 import workloads as W
    B = W.CONFIGS[3]["B"]
    wl, sig = _synth(torch, S, 3, B)
    J = S.SupportSet(wl.N, wl.support)
    r = S.pivots(J)
    assert len(r) == 14 and not S.classify(J).is_homogeneous
    out = S.sas_transform(sig, J, r=r)
    got = out.coeffs.cpu().numpy()
    assert out.plan.mu_star == 1
    err = np.linalg.norm(got - wl.coeffs, axis=1) / np.linalg.norm(wl.coeffs, axis=1)
    assert err.max() < 1e-5
    _check_rows(wl, sig, got, [0, 1, 7, 300, 511], O.sas_mu1, 1e-5)
    for b in (0, 1):
        assert rel_l2(got[b], golden_configs[f"cfg3_b{b}_out"]) < 1e-5


# ------------------------------------------------- split path (large A) ---

@pytest.mark.parametrize("dt,s", [(np.complex64, 15), (np.complex64, 16), (np.complex64, 17),
                                  (np.complex128, 14), (np.complex128, 15), (np.complex128, 16)])
def test_split_homogeneous(S, torch, dt, s):
    rng = np.random.default_rng(1000 + s)
    M, B = 22, 3
    piv = sorted(rng.choice(M, size=s, replace=False).tolist())
    J = O.gen_homogeneous(piv, M, int(rng.integers(0, 2 ** 62)))
    coef = rng.normal(size=(B, J.size)) + 1j * rng.normal(size=(B, J.size))
    f = np.stack([O.synthesize(J, coef[b], M) for b in range(B)]).astype(dt)
    Js = S.SupportSet(1 << M, J)
    got = S.hidft_to_dft_batched(torch.from_numpy(f).cuda(), Js).cpu().numpy()
    for b in range(B):
        want = O.hidft_to_dft(f[b], J, M)
        assert rel_l2(got[b], want) < TOL[dt], (b, rel_l2(got[b], want))
    # node / slot outputs with a shift through the generic hidft entry
    res = S.hidft(torch.from_numpy(f[:1]).cuda(), Js, tuple(piv), shift=12345)
    o = O.hidft(f[0], J, M, piv, 0, 12345)
    assert res.node_residues == tuple(int(x) for x in o.node_residues)
    assert rel_l2(res.node_values[0].cpu().numpy(), o.node_values) < TOL[dt]
    assert rel_l2(res.slot_values[0].cpu().numpy(), o.slot_values) < TOL[dt]


def test_split_part_homogeneous_sas(S, torch):
    # config-3 shape at larger scale: a 2^13 subset of a 2^16 homogeneous set
    rng = np.random.default_rng(77)
    M = 24
    piv = sorted(rng.choice(M, size=16, replace=False).tolist())
    H = O.gen_homogeneous(piv, M, 5)
    J = np.sort(H[rng.choice(H.size, size=1 << 13, replace=False)])
    r = O.pivots(J, M)
    coef = rng.normal(size=J.size) + 1j * rng.normal(size=J.size)
    f = O.synthesize(J, coef, M).astype(np.complex64)
    Js = S.SupportSet(1 << M, J)
    assert S.pivots(Js) == r
    out = S.sas_transform(torch.from_numpy(f).cuda(), Js, r=r)
    want = O.sas_mu1(f, J, M)
    if len(r) > 14:
        assert S.get_plan(Js, r, 0, 0, S._lib.require_device()).A == 1 << len(r)
    assert rel_l2(out.coeffs.cpu().numpy(), want) < 1e-5
    assert rel_l2(out.coeffs.cpu().numpy(), coef) < 1e-5
    res = S.hidft(torch.from_numpy(f).cuda(), Js, r, height=1)
    o = O.hidft(f, J, M, r, 1, 0)
    assert res.node_residues == tuple(int(x) for x in o.node_residues)
    assert rel_l2(res.node_values.cpu().numpy(), o.node_values) < 1e-5


@pytest.mark.parametrize("cfg", [5, 6])
def test_config5_full_batch(S, torch, golden_configs, cfg):
    from paper_2211_15299_b200 import workloads as W
    B = W.CONFIGS[cfg]["B"]
    wl, sig = _synth(torch, S, cfg, B)
    J = S.SupportSet(wl.N, wl.support)
    got = S.hidft_to_dft_batched(sig, J).cpu().numpy()
    tol = TOL[np.complex64 if wl.dtype == "complex64" else np.complex128]
    err = np.linalg.norm(got - wl.coeffs, axis=1) / np.linalg.norm(wl.coeffs, axis=1)
    assert err.max() < tol
    # oracle parity on the first and last row and on both sides of the row-chunk boundary (128-row chunks)
    _check_rows(wl, sig, got, sorted({0, B // 2 - 1, B // 2, B - 1}), O.hidft_to_dft, tol)
    head = golden_configs["cfg5_b0_head"]
    assert rel_l2(got[0][: head.size], head) < max(tol, 1e-6)
    del sig
    torch.cuda.empty_cache()


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_plan_tables_at_config_size(S, cfg):
    """Index tables of the device plan bit-exact with the oracle's _build_plan
    restatement at the BASELINE configs' sizes (s up to 16)."""
    J, M = O.config_support(cfg)
    r = O.pivots(J, M)
    Js = S.SupportSet(1 << M, J)
    assert S.pivots(Js) == r
    assert S.classify(Js).is_homogeneous == O.is_homogeneous(J, M)
    plan = S.get_plan(Js, r, 0, 1, S._lib.require_device())
    t = plan.tables()
    o = O.build_plan(J, M, r)
    assert plan.level == o.level and plan.mu_star == int(o.slot_count.max())
    for name, want in (("element_slots", o.element_slots), ("slot_residues", o.slot_residues),
                       ("slot_real", o.slot_real), ("node_residues", o.node_residues), ("offsets", o.offsets)):
        assert np.array_equal(t[name], want), name
    tw = np.concatenate(o.twiddles)
    assert np.max(np.abs(t["twiddles"] - tw)) < 1e-15
    assert np.array_equal(S.pivoted_pattern(r, M).as_array(), O.pivoted_pattern(r, M))


@pytest.mark.parametrize("case", ["cfg1", "cfg2", "cfg3", "cfg5", "cfg4_b0", "cfg4_b1"])
def test_plan_tables_match_reference_digests(S, plan_digests, case):
    """The device plan at the BASELINE config sizes against digests of the
    UNMODIFIED reference's own tables (tests/golden/make_golden_plan_digests.py):
    pivots, level and every index table bit-exact by sha256, sampled twiddles
    to 1e-15 -- the full-size pin that does not pass through the oracle."""
    from conftest import table_digest, twiddle_sample_index
    want = plan_digests[case]
    cfg = int(case[3])
    J, M = O.config_support(cfg, int(case[-1]) if "_b" in case else 0)
    assert table_digest(J, "<i8") == want["sha256"]["J"]
    Js = S.SupportSet(1 << M, J)
    r = S.pivots(Js)
    assert list(r) == want["pivots"]
    plan = S.get_plan(Js, r, 0, 1, S._lib.require_device())
    assert plan.level == want["level"]
    t = plan.tables()
    for name, dt in (("element_slots", "<i8"), ("slot_residues", "<i8"), ("slot_real", "u1"),
                     ("node_residues", "<i8"), ("offsets", "<i8")):
        assert table_digest(t[name], dt) == want["sha256"][name], name
    tw = np.asarray(t["twiddles"])
    assert tw.size == want["twiddle_count"]
    ref = np.array([complex(float.fromhex(a), float.fromhex(b)) for a, b in want["twiddle_sample"]])
    assert np.max(np.abs(tw[twiddle_sample_index(tw.size)] - ref)) < 1e-15


_ALT_SPLIT = r"""
import sys
import numpy as np
import torch
import structfft_oracle as O
import paper_2211_15299_b200 as S
ok = True
for dt, s, top in [(np.complex64, 16, 0), (np.complex64, 17, 0), (np.complex128, 16, 0), (np.complex128, 14, 0),
                   (np.complex64, 16, 4), (np.complex64, 16, 2)]:
    rng = np.random.default_rng(3000 + s + top)
    M, B = 22, 3
    # top > 0: the `top` largest levels are pivots (head-pass eligible; top = 4: blocked output map)
    piv = sorted(rng.choice(M - top, size=s - top, replace=False).tolist()) + list(range(M - top, M))
    J = O.gen_homogeneous(piv, M, int(rng.integers(0, 2 ** 62)))
    coef = rng.normal(size=(B, J.size)) + 1j * rng.normal(size=(B, J.size))
    f = np.stack([O.synthesize(J, coef[b], M) for b in range(B)]).astype(dt)
    got = S.hidft_to_dft_batched(torch.from_numpy(f).cuda(), S.SupportSet(1 << M, J)).cpu().numpy()
    tol = 1e-5 if dt == np.complex64 else 1e-11
    for b in range(B):
        want = O.hidft_to_dft(f[b], J, M)
        err = np.linalg.norm(got[b] - want) / np.linalg.norm(want)
        print(dt.__name__, s, b, err)
        ok &= bool(err < tol)
sys.exit(0 if ok else 1)
"""


@pytest.mark.parametrize("env", [{"SFFT_SPLIT_PASSES": "2"}, {"SFFT_TRI_SCRATCH_MB": "1"}, {"SFFT_HEAD_BULK": "0"},
                                 {"SFFT_FIN_TMA": "0"}, {"SFFT_FIN3": "0"}, {"SFFT_HEAD": "0"}])
def test_alternate_split_configurations(S, env):
    """The two-pass split (SFFT_SPLIT_PASSES=2, kept for A/B measurements),
    the three-pass split with many small row chunks (a 1 MiB scratch
    budget: 1-4 rows per chunk, the PDL chain across chunks), the head pass
    with its register epilogue (SFFT_HEAD_BULK=0) or the final pass with
    per-thread stores (SFFT_FIN_TMA=0) or per-thread loads (SFFT_FIN3=0:
    k_fin2 with the tensor store) and head-eligible patterns on the
    three-pass split (SFFT_HEAD=0), against the oracle.  Each runs in a
    fresh process: the settings are read once."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    e = dict(os.environ, PYTHONPATH=os.pathsep.join([root, os.path.join(root, "oracle")]), **env)
    out = subprocess.run([sys.executable, "-c", _ALT_SPLIT], env=e, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr


@pytest.mark.parametrize("M,B", [(10, 64), (15, 6)])
def test_back_to_back_calls_chain(S, torch, M, B):
    """Consecutive launches overlap through programmatic dependent launch
    (sfft_hidft.cu, pdl_join; M = 15 runs the three-pass split, whose first
    pass joins the chain).  A call whose signals are the previous call's
    output must still see that output (the host keeps it out of the PDL
    chain), and calls writing the same output buffer keep stream order.
    J = Z_N so a result row is a valid signal row."""
    N = 1 << M
    Js = S.SupportSet(N, np.arange(N))
    rng = np.random.default_rng(5)
    f = torch.from_numpy((rng.standard_normal((B, N)) + 1j * rng.standard_normal((B, N))).astype(np.complex64)).cuda()
    # reference: each call synchronised
    ref = [f]
    for _ in range(3):
        ref.append(S.hidft_to_dft_batched(ref[-1], Js))
        torch.cuda.synchronize()
    ref = [r.clone() for r in ref]
    bufs = [torch.empty_like(f) for _ in range(3)]
    other = torch.from_numpy((rng.standard_normal((B, N)) + 1j * rng.standard_normal((B, N))).astype(np.complex64)).cuda()
    for _ in range(20):
        with S.stream_chain():  # consecutive library calls may overlap (PDL chain scope)
            x = f
            for i in range(3):  # each call reads the previous call's output: fully ordered launches
                S.hidft_to_dft_batched(x, Js, out=bufs[i])
                x = bufs[i]
            # independent calls into one output buffer (PDL chain, write-after-write)
            S.hidft_to_dft_batched(other, Js, out=bufs[0])
            S.hidft_to_dft_batched(f, Js, out=bufs[0])
        torch.cuda.synchronize()
        assert torch.equal(bufs[0], ref[1])
        assert torch.equal(bufs[1], ref[2])
        assert torch.equal(bufs[2], ref[3])
    # planted check of the first transform: the DFT of f
    want = np.fft.fft(f.cpu().numpy().astype(np.complex128), axis=1)
    assert rel_l2(ref[1].cpu().numpy(), want) < 1e-5


def test_back_to_back_fused_chain(S, torch):
    """The per-signal fused kernel joins the PDL chain too: chained calls
    (signals = the previous call's output) and calls sharing one output and
    status buffer stay ordered."""
    M, B = 9, 48
    N = 1 << M
    Jt = torch.arange(N, dtype=torch.int64).repeat(B, 1).cuda()
    rng = np.random.default_rng(6)
    f = torch.from_numpy((rng.standard_normal((B, N)) + 1j * rng.standard_normal((B, N))).astype(np.complex64)).cuda()
    other = torch.from_numpy((rng.standard_normal((B, N)) + 1j * rng.standard_normal((B, N))).astype(np.complex64)).cuda()
    st = torch.zeros(B, dtype=torch.int32, device="cuda")
    ref = [f]
    for _ in range(3):
        ref.append(S.hidft_to_dft_batched(ref[-1], Jt, status=st, check=False).clone())
        torch.cuda.synchronize()
    bufs = [torch.empty_like(f) for _ in range(3)]
    for _ in range(20):
        with S.stream_chain():
            x = f
            for i in range(3):
                S.hidft_to_dft_batched(x, Jt, out=bufs[i], status=st, check=False)
                x = bufs[i]
            S.hidft_to_dft_batched(other, Jt, out=bufs[0], status=st, check=False)
            S.hidft_to_dft_batched(f, Jt, out=bufs[0], status=st, check=False)
        torch.cuda.synchronize()
        for i in range(3):
            assert torch.equal(bufs[i], ref[i + 1])
        assert int(st.max()) == 0
    want = np.fft.fft(f.cpu().numpy().astype(np.complex128), axis=1)
    assert rel_l2(ref[1].cpu().numpy(), want) < 1e-5


_PDL_RUN = r"""
import sys
import numpy as np
import torch
import paper_2211_15299_b200 as S
from paper_2211_15299_b200 import workloads as W
outs = []
for cfg, B in ((2, 64), (4, 48), (5, 3)):
    wl = W.make_workload(cfg, B=B)
    sig = torch.empty((wl.B, wl.N), dtype=torch.complex64, device="cuda")
    W.synthesize_into(sig, wl.support, wl.coeffs)
    J = S.SupportSet(wl.N, wl.support) if wl.support.ndim == 1 else torch.from_numpy(wl.support).cuda()
    out = torch.empty((wl.B, wl.k), dtype=torch.complex64, device="cuda")
    with S.stream_chain():
        for _ in range(8):  # back-to-back calls into one output buffer
            S.hidft_to_dft_batched(sig, J, out=out)
    torch.cuda.synchronize()
    outs.append(out.cpu().numpy())
np.savez(sys.argv[1], *outs)
"""


def test_pdl_on_off_bitwise(S, tmp_path):
    """The PDL overlap between consecutive calls changes timing only: the
    results with SFFT_PDL=0 (every launch fully stream-ordered) are bitwise
    identical (configs 2, 4, 5 shapes, back-to-back calls)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for pdl in ("1", "0"):
        path = str(tmp_path / f"pdl{pdl}.npz")
        env = dict(os.environ, PYTHONPATH=root, SFFT_PDL=pdl, SFFT_TRI_PDL=pdl)
        out = subprocess.run([sys.executable, "-c", _PDL_RUN, path], env=env, capture_output=True, text=True,
                             timeout=600)
        assert out.returncode == 0, out.stderr
        res[pdl] = np.load(path)
    for key in res["1"].files:
        assert np.array_equal(res["1"][key], res["0"][key]), key


@pytest.mark.parametrize("cfg,B", [(2, 64), (4, 32), (5, 3)])
def test_foreign_producer_early_trigger(S, torch, cfg, B):
    """A foreign kernel that produces the signals and lets its dependents
    launch early (griddepcontrol.launch_dependents at entry, then a spin, then
    the stores; tests/csrc/early_producer.cu) must never race the library's
    loads: outside a stream_chain scope every call's first kernel is fully
    stream-ordered (pdl_join)."""
    import ctypes
    import os
    from paper_2211_15299_b200 import workloads as W
    lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libsfft_test_producer.so"))
    lib.sfft_test_early_producer.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                             ctypes.c_void_p]
    wl = W.make_workload(cfg, B=B)
    src = torch.empty((wl.B, wl.N), dtype=torch.complex64, device="cuda")
    W.synthesize_into(src, wl.support, wl.coeffs)
    J = S.SupportSet(wl.N, wl.support) if wl.support.ndim == 1 else torch.from_numpy(wl.support).cuda()
    want = S.hidft_to_dft_batched(src, J).clone()
    dst = torch.empty_like(src)
    out = torch.empty_like(want)
    stream = torch.cuda.current_stream().cuda_stream
    for _ in range(5):
        dst.zero_()
        S.hidft_to_dft_batched(src, J, out=out)  # a library launch right before the producer
        assert lib.sfft_test_early_producer(dst.data_ptr(), src.data_ptr(), dst.numel(), 2_000_000, stream) == 0
        S.hidft_to_dft_batched(dst, J, out=out)
        torch.cuda.synchronize()
        assert torch.equal(out, want)


def test_out_buffer_validation(S, torch):
    """A caller-supplied out / status buffer is checked before any device
    write (hidft.py passed only data_ptr and stride(0))."""
    from paper_2211_15299_b200 import workloads as W
    wl = W.make_workload(2, B=4)
    sig = torch.empty((wl.B, wl.N), dtype=torch.complex64, device="cuda")
    W.synthesize_into(sig, wl.support, wl.coeffs)
    J = S.SupportSet(wl.N, wl.support)
    bad = [torch.empty((wl.B, wl.k), dtype=torch.complex128, device="cuda"),   # dtype
           torch.empty((wl.B - 1, wl.k), dtype=torch.complex64, device="cuda"),  # rows
           torch.empty((wl.B, wl.k), dtype=torch.complex64),                   # device
           torch.empty((wl.B, 2 * wl.k), dtype=torch.complex64, device="cuda")[:, ::2]]  # inner stride
    for o in bad:
        with pytest.raises(S.InvalidInputError):
            S.hidft_to_dft_batched(sig, J, out=o)
    Jt = torch.from_numpy(np.stack([wl.support] * wl.B)).cuda()
    for st in (torch.zeros(wl.B - 1, dtype=torch.int32, device="cuda"), torch.zeros(wl.B, dtype=torch.int64,
                                                                                     device="cuda")):
        with pytest.raises(S.InvalidInputError):
            S.hidft_to_dft_batched(sig, Jt, status=st)
    ok = torch.empty((wl.B, wl.k), dtype=torch.complex64, device="cuda")
    assert S.hidft_to_dft_batched(sig, J, out=ok) is not None


_CANARY = 12345.5


def _guarded(torch, B, k, dtype):
    """(interior view, whole buffer): rows 1..B, columns 8..8+k of a
    (B+2, k+24) buffer whose every element holds a sentinel."""
    big = torch.full((B + 2, k + 24), complex(_CANARY, -_CANARY), dtype=dtype, device="cuda")
    return big[1:B + 1, 8:8 + k], big


def _assert_guard_intact(torch, big, B, k):
    mask = torch.ones(big.shape, dtype=torch.bool, device=big.device)
    mask[1:B + 1, 8:8 + k] = False
    outside = big[mask]
    assert bool((outside.real == _CANARY).all()) and bool((outside.imag == -_CANARY).all()), \
        "a kernel wrote outside its output rows"


@pytest.mark.parametrize("case", ["plan_c128", "plan_c64", "fused", "tri", "head", "tri_c128"])
def test_output_guard_regions(S, torch, case):
    """Out-of-bounds write check (compute-sanitizer is closed on this GPU pool):
    every transform family writes into the interior of a sentinel-filled
    buffer (row stride > k) and must leave the guard rows / columns intact,
    with the interior matching the oracle-checked result."""
    rng = np.random.default_rng(11)
    if case.startswith("plan"):
        M, piv = 14, (0, 2, 3, 5, 7, 9)
    elif case == "fused":
        M, piv = 14, None
    elif case == "head":
        M, piv = 20, tuple(sorted(rng.choice(18, size=14, replace=False).tolist()) + [18, 19])
    elif case == "tri_c128":
        M, piv = 20, tuple(range(2, 18))
    else:
        M, piv = 20, tuple(range(2, 18))  # top pivot 17 < M-1: not head-eligible, three-pass split
    N = 1 << M
    dt = torch.complex128 if case.endswith("c128") else torch.complex64
    B = 3
    sig = torch.randn(B, N, dtype=dt, device="cuda")
    if case == "fused":
        sup = np.stack([O.gen_homogeneous(sorted(rng.choice(14, size=6, replace=False).tolist()), M, 40 + b)
                        for b in range(B)])
        J = torch.from_numpy(sup).cuda()
        k = sup.shape[1]
    else:
        Jn = O.gen_homogeneous(piv, M, 9)
        J = S.SupportSet(N, Jn)
        k = Jn.size
    want = S.hidft_to_dft_batched(sig, J).clone()
    inner, big = _guarded(torch, B, k, dt)
    S.hidft_to_dft_batched(sig, J, out=inner)
    torch.cuda.synchronize()
    _assert_guard_intact(torch, big, B, k)
    assert torch.equal(inner, want)
    row = sig[0].cpu().numpy()
    ref = O.hidft_to_dft(row, J[0].cpu().numpy() if torch.is_tensor(J) else J.as_array(), M)
    assert rel_l2(want[0].cpu().numpy(), ref) < (1e-5 if dt == torch.complex64 else 1e-11)


@pytest.mark.parametrize("M,piv,B,dt,pad", [(20, (0, 1, 2, 4, 5, 7, 8, 11, 12, 14), 37, "c64", 0),
                                             (16, (2, 3, 6, 9, 12, 13, 14, 15), 16, "c128", 3),
                                             (14, tuple(range(12)), 9, "c64", 5),
                                             (13, tuple(range(11)), 6, "c128", 0),
                                             (10, (1, 4), 3, "c64", 1)])
def test_interleaved_layout_matches_row_major(S, torch, M, piv, B, dt, pad):
    """sfft_hidft_interleaved on an (N, B) sample-major batch (row stride
    B + pad) gives bitwise the coefficients of the row-major call on the same
    signals (same plan, same butterfly), and the oracle's."""
    N = 1 << M
    cdt = torch.complex64 if dt == "c64" else torch.complex128
    Jn = O.gen_homogeneous(piv, M, 21)
    J = S.SupportSet(N, Jn)
    rows = torch.randn(B, N, dtype=cdt, device="cuda")
    store = torch.zeros(N, B + pad, dtype=cdt, device="cuda")
    store[:, :B] = rows.T
    got = S.hidft_to_dft_interleaved(store[:, :B], J)
    want = S.hidft_to_dft_batched(rows, J)
    torch.cuda.synchronize()
    assert torch.equal(got, want)
    ref = O.hidft_to_dft(rows[B - 1].cpu().numpy(), Jn, M)
    assert rel_l2(got[B - 1].cpu().numpy(), ref) < (1e-5 if dt == "c64" else 1e-11)


@pytest.mark.parametrize("dt", ["c64", "c128"])
def test_s13_single_cta_plan_kernel(S, torch, dt):
    """2^13 slots on one CTA (complex128: 16 slots per thread, 512 threads)
    against the oracle, with a shift and at height 0."""
    M, piv = 16, tuple(range(2, 15))
    N = 1 << M
    cdt = torch.complex64 if dt == "c64" else torch.complex128
    Jn = O.gen_homogeneous(piv, M, 8)
    J = S.SupportSet(N, Jn)
    sig = torch.randn(3, N, dtype=cdt, device="cuda")
    got = S.hidft_to_dft_batched(sig, J).cpu().numpy()
    for b in range(3):
        want = O.hidft_to_dft(sig[b].cpu().numpy(), Jn, M)
        assert rel_l2(got[b], want) < (1e-5 if dt == "c64" else 1e-11)
    res = S.hidft(sig[1], J, S.pivots(J), shift=123)
    ref = O.hidft(sig[1].cpu().numpy()[None, :], Jn, M, S.pivots(J), shift=123)
    vals = res.node_values.cpu().numpy() if hasattr(res.node_values, "cpu") else res.node_values
    assert rel_l2(np.asarray(vals).reshape(-1), np.asarray(ref.node_values).reshape(-1)) < (1e-5 if dt == "c64" else 1e-11)


@pytest.mark.parametrize("top", [4, 0])
def test_graph_capture_with_growing_scratch(S, torch, top):
    """The large-transform paths inside CUDA graph captures: the first
    capture on a stream sees a small batch, the second a larger one, so the
    per-stream scratch grows while the stream captures (a plain allocation
    with the capture mode relaxed; the outgrown buffer stays alive for the
    first graph).  Both graphs replay, in either order, to the eager result
    (top = 4: head pass with the tensor-store final pass; 0: three-pass split)."""
    M, s = 21, 16
    rng = np.random.default_rng(77 + top)
    piv = sorted(rng.choice(M - top, size=s - top, replace=False).tolist()) + list(range(M - top, M))
    Jn = O.gen_homogeneous(piv, M, 5)
    J = S.SupportSet(1 << M, Jn)
    sig = torch.randn(5, 1 << M, dtype=torch.complex64, device="cuda")
    want = S.hidft_to_dft_batched(sig, J).clone()
    torch.cuda.synchronize()
    outs = [torch.zeros(1, Jn.size, dtype=torch.complex64, device="cuda"),
            torch.zeros(5, Jn.size, dtype=torch.complex64, device="cuda")]
    graphs = []
    for o in outs:  # torch.cuda.graph captures on its own side stream: first use of that stream's scratch
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            S.hidft_to_dft_batched(sig[: o.shape[0]], J, out=o, check=False)
        graphs.append(g)
    for order in ((0, 1), (1, 0), (0, 1)):
        for o in outs:
            o.zero_()
        for i in order:
            graphs[i].replay()
        torch.cuda.synchronize()
        assert torch.equal(outs[0], want[:1])
        assert torch.equal(outs[1], want)
    ref = O.hidft_to_dft(sig[4].cpu().numpy(), Jn, M)
    assert rel_l2(want[4].cpu().numpy(), ref) < 1e-5


@pytest.mark.parametrize("M,top,B,seed", [(20, 4, 131, 1), (21, 2, 5, 2), (22, 4, 2, 3), (20, 3, 67, 4)])
def test_head_path_patterns_and_chunk_boundaries(S, torch, M, top, B, seed):
    """2^16-slot supports whose `top` largest levels are pivots (the TMA head
    pass; top = 4: blocked output map, tensor-copy final pass), random other
    pivots and multipliers, batches that cross the 128-row scratch chunk
    (131 rows: chunks of 128 + 3) or stay far below it: every row against
    the planted spectrum, seeded rows and both sides of the chunk boundary
    against the oracle."""
    rng = np.random.default_rng(9000 + seed)
    s = 16
    piv = sorted(rng.choice(M - top, size=s - top, replace=False).tolist()) + list(range(M - top, M))
    Jn = O.gen_homogeneous(piv, M, int(rng.integers(0, 2 ** 62)))
    N = 1 << M
    coef = (rng.normal(size=(B, Jn.size)) + 1j * rng.normal(size=(B, Jn.size))).astype(np.complex128)
    sig = torch.empty((B, N), dtype=torch.complex64, device="cuda")
    from paper_2211_15299_b200 import workloads as W
    W.synthesize_into(sig, Jn, coef)
    J = S.SupportSet(N, Jn)
    got = S.hidft_to_dft_batched(sig, J).cpu().numpy()
    err = np.linalg.norm(got - coef, axis=1) / np.linalg.norm(coef, axis=1)
    assert err.max() < 1e-5
    rows = sorted({0, B - 1} | ({127, 128} if B > 128 else set()) | {int(rng.integers(0, B))})
    for b in rows:
        want = O.hidft_to_dft(sig[b].cpu().numpy(), Jn, M)
        assert rel_l2(got[b], want) < 1e-5, b
