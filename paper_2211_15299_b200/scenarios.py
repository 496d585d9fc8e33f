"""Seeded Monte-Carlo scenarios behind `structfft bench` (reference
bench.py:65-336), with every trial's transform on the GPU.

A scenario file {"name", "seed", "tolerance", "scenarios": [{"kind",
"trials", "params", "id"}]} lists experiments over the support families;
each trial draws a family instance and a planted nonzero spectrum from the
(seed, scenario, trial) stream, picks the pivot vector with the family's
policy, runs the device shift-and-sample and records the exact operation
counts (identical to the reference's) and the max relative error.  The
"antipodal" kind only measures how often a Bernoulli(k/N) subset of Z_N holds
a pair j, j + N/2.  Harness code around the transform.
"""

from __future__ import annotations

import math

import numpy as np

from .congruence import SupportSet
from .counting import OpCounter
from .errors import InvalidInputError
from .families import build_family, draw_coefficients
from .sas import C1, C2, sas_transform, select_pivots
from .signals import BandlimitedSignal
from .workloads import rng_from_seed

CSV_COLUMNS = ("trial", "family", "N", "k", "size_r", "mu_star", "ops_hidft", "ops_solve", "ops_total",
               "bound_total", "samples", "correct", "max_rel_err")
C_MU_STAR = 4.0 + 3.0 * math.log(2.0)
FIXTURES = {  # named supports of the paper's worked examples
    "paper_sas": (1024, (0, 1, 6, 7, 512)),
    "uoe_union": (1024, (0, 1, 2, 3, 4, 8, 9, 10, 13, 22, 23, 31)),
    "uoe_adversarial": (1024, tuple(sorted({(1 << (4 + i)) + j for i in range(5) for j in range(1 << i)}))),
}


def _pick(rng, v) -> int:
    """A constant, or an inclusive [lo, hi] range drawn from rng."""
    if isinstance(v, (list, tuple)):
        return int(rng.integers(v[0], v[1] + 1))
    return int(v)


def _subset(rng, M: int, s: int) -> list:
    return sorted(rng.choice(M, size=min(s, M), replace=False).tolist())


def _etas(rng, a_n: int, cap: int) -> list:
    e = [int(rng.integers(0, cap + 1)) for _ in range(a_n + 1)]
    e[a_n] = max(1, e[a_n])  # the largest constituent present
    return e


def _trial_family(kind: str, p: dict, rng, seed: int):
    """(family kind, params) of one trial, drawn in the reference's order."""
    if kind == "homogeneous":
        M = _pick(rng, p["M"])
        s = _pick(rng, p.get("s", [1, max(M // 2, 1)]))
        return "homogeneous", {"pivots": _subset(rng, M, s), "M": M}
    if kind == "elementary":
        M = _pick(rng, p["M"])
        return "elementary", {"r": min(_pick(rng, p.get("r", [1, max(M // 2, 1)])), M), "M": M}
    if kind == "consecutive":
        N = 1 << _pick(rng, p["M"])
        k = min(_pick(rng, p.get("k", [2, 64])), N)
        return "consecutive", {"a": int(rng.integers(0, N)), "k": k, "N": N}
    if kind == "ap":
        M = _pick(rng, p["M"])
        N = 1 << M
        k = min(_pick(rng, p.get("k", [2, 64])), N // 2)
        alpha = _pick(rng, p.get("alpha", [0, max(M - k.bit_length() - 1, 0)]))
        s = ((2 * int(rng.integers(0, max(N >> (alpha + 2), 1))) + 1) << alpha) % N
        a = int(rng.integers(0, N))
        try:
            build_family("ap", {"a": a, "s": s, "k": k, "N": N}, seed)
        except InvalidInputError:
            s = 1 << alpha  # collision-free with the same 2-adic valuation
        return "ap", {"a": a, "s": s, "k": k, "N": N}
    if kind == "gap":
        M = _pick(rng, p["M"])
        N = 1 << M
        d = _pick(rng, p.get("d", [1, 3]))
        cap = int(p.get("volume_cap", 1 << 12))
        lengths, vol = [], 1
        for _ in range(d):
            n = int(rng.integers(2, min(max(cap // vol, 2), 64) + 1))
            lengths.append(n)
            vol *= n
        steps = [int(rng.integers(1, N)) for _ in range(d)]
        return "gap", {"a": int(rng.integers(0, N)), "steps": steps, "lengths": lengths, "N": N}
    if kind == "uoe":
        M = _pick(rng, p["M"])
        a_n = _pick(rng, p.get("a_n", [1, max(M // 2, 1)]))
        return "uoe", {"a_n": a_n, "etas": _etas(rng, a_n, int(p.get("eta_cap", 2))), "M": M}
    if kind == "uoh":
        M = _pick(rng, p["M"])
        base = _subset(rng, M, _pick(rng, p.get("s", [2, max(M // 2, 2)])))
        a_n = min(_pick(rng, p.get("a_n", [1, len(base)])), len(base))
        return "uoh", {"base_pivots": base, "a_n": a_n, "etas": _etas(rng, a_n, int(p.get("eta_cap", 2))), "M": M}
    if kind == "random_subset":
        M = _pick(rng, p["M"])
        sp = {"M": M, "k": _pick(rng, p["k"]), "base": p.get("base", "zn")}
        if sp["base"] == "homogeneous":
            sp["base_pivots"] = _subset(rng, M, _pick(rng, p.get("base_s", max(M // 2, 1))))
        return "random_subset", sp
    if kind == "jstar":
        return "jstar", {"M": _pick(rng, p["M"])}
    raise InvalidInputError(f"unknown trial kind {kind!r}")


def run_trial(kind: str, params: dict, seed: int, sidx: int, trial: int, tol: float) -> tuple:
    rng = rng_from_seed(seed, sidx, trial)
    tseed = int(rng.integers(0, 2 ** 63 - 1))
    if kind == "fixture":
        N, idx = FIXTURES[params["name"]]
        J, meta, label = SupportSet.make(N, idx), {"policy": "auto"}, f"fixture:{params['name']}"
    else:
        fk, fp = _trial_family(kind, params, rng, tseed)
        fam = build_family(fk, fp, tseed)
        J, meta, label = fam.support, fam.meta, kind
    c = draw_coefficients(len(J), rng, nonzero=True)
    r = select_pivots(J, params.get("policy", meta.get("policy", "auto")), meta)
    out = sas_transform(BandlimitedSignal(J, c), J, r=r, counter=OpCounter(), tolerance=tol)
    got = out.coeffs.detach().cpu().numpy() if hasattr(out.coeffs, "detach") else np.asarray(out.coeffs)
    err = float(np.max(np.abs(got - c) / np.abs(c))) if len(J) else 0.0
    rep = out.report
    return (trial, label, J.N, len(J), len(out.plan.pivots), out.plan.mu_star, rep.ops_hidft, rep.ops_solve,
            rep.total, rep.bound_alg1bnd, rep.samples_touched, bool(err <= tol), err)


def antipodal(params: dict, seed: int, sidx: int, trials: int) -> dict:
    M = int(params["M"])
    N = 1 << M
    k = int(params.get("k", math.isqrt(N) * int(params.get("k_factor", 4))))
    hits, sizes = 0, []
    for t in range(trials):
        keep = rng_from_seed(seed, sidx, t).random(N) < k / N
        sizes.append(int(keep.sum()))
        hits += bool(np.any(keep[:N // 2] & keep[N // 2:]))
    return {"kind": "antipodal", "trials": trials, "N": N, "k": k, "antipodal_fraction": hits / trials,
            "mean_size": float(np.mean(sizes))}


def summarize(rows: list) -> dict:
    n = len(rows)
    if not n:
        return {"trials": 0}
    col = {c: i for i, c in enumerate(CSV_COLUMNS)}
    g = lambda r, c: r[col[c]]  # noqa: E731
    big = [r for r in rows if g(r, "k") >= 2]
    ratios = [g(r, "ops_total") / (g(r, "k") * math.log2(g(r, "k"))) for r in big]
    env = C_MU_STAR * (C1 + C2 * C_MU_STAR)
    return {
        "trials": n,
        "all_correct": all(g(r, "correct") for r in rows),
        "frac_correct": sum(g(r, "correct") for r in rows) / n,
        "max_rel_err": max(g(r, "max_rel_err") for r in rows),
        "pr_mu_star_ge_c_logk": sum(g(r, "mu_star") >= C_MU_STAR * math.log2(g(r, "k")) for r in big) / n,
        "c_mu_star": C_MU_STAR,
        "hidft_exact_frac": sum(g(r, "ops_hidft") == round(C1 * g(r, "size_r") * (1 << g(r, "size_r")))
                                * g(r, "mu_star") for r in rows) / n,
        "bound_ok_frac": sum(g(r, "ops_total") <= g(r, "bound_total") for r in rows) / n,
        "lower_bound_ok_frac": sum(g(r, "ops_total") >= g(r, "k") * math.log2(g(r, "k")) for r in rows) / n,
        "proof_envelope_ok_frac": sum(g(r, "k") < 2 or g(r, "ops_total") <= env * g(r, "k") * math.log2(g(r, "k"))
                                      for r in rows) / n,
        "ops_over_klogk_max": max(ratios) if ratios else 0.0,
        "ops_over_klogk_mean": float(np.mean(ratios)) if ratios else 0.0,
    }


def run_scenarios(cfg: dict) -> tuple[list, dict]:
    if "scenarios" not in cfg:
        raise InvalidInputError("scenario file needs a 'scenarios' list")
    seed, tol = int(cfg.get("seed", 0)), float(cfg.get("tolerance", 1e-8))
    rows, sums = [], []
    for sidx, sc in enumerate(cfg["scenarios"]):
        kind, trials, params = sc["kind"], int(sc["trials"]), dict(sc.get("params", {}))
        sid = sc.get("id", f"{kind}-{sidx}")
        if kind == "antipodal":
            sums.append({**antipodal(params, seed, sidx, trials), "id": sid})
            continue
        recs = [run_trial(kind, params, seed, sidx, t, tol) for t in range(trials)]
        base = len(rows)
        rows.extend((base + r[0],) + r[1:] for r in recs)
        sums.append({**summarize(recs), "id": sid, "kind": kind})
    return rows, {"name": cfg.get("name", "bench"), "seed": seed, "tolerance": tol, "scenarios": sums}
