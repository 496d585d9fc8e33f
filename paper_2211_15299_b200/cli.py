"""`structfft` command line on the B200 path: analyze, transform, gen, bench.

Same commands, options, file formats and exit codes as the reference CLI
(reference cli.py:1-11, 316-378): support files {"N", "indices"}, signal and
spectrum files {"N", "support", "coeffs": [[re, im], ...]}; output JSON with
sorted keys, indent 2, floats rounded to 17 significant digits; exit codes 0
ok, 2 input error, 3 contract violation, 4 budget exceeded.  Every transform
runs on the GPU: hidft / sas through the Hi-DFT and node-decode kernels,
`submatrix` as the device node decoder on the single node of pivot vector
() (the k x k Vandermonde of the reference's submatrix_method), `fft` as the
device FFT of the synthesised signal and `oracle` as the dense DFT rows
F(J, Z_N) applied on the device.  `bench` runs a reference scenario file
(reference bench.py:250-336) with the device shift-and-sample per trial.
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import math
import os
import sys

import numpy as np

from .congruence import SupportSet, build_tree, classify, pivots
from .counting import OpCounter
from .errors import BudgetExceededError, ContractViolationError, InvalidInputError, StructFFTError
from .sas import CostReport
from .signals import BandlimitedSignal

LIMITS = {"oracle": 1 << 12, "fft": 1 << 22, "submatrix": 1 << 10}
EXIT = ((InvalidInputError, 2, "input error"), (ContractViolationError, 3, "contract violation"),
        (BudgetExceededError, 4, "budget exceeded"))


# ------------------------------------------------------------ JSON files ---

def _plain(v):
    """JSON-ready copy: floats at 17 significant digits (finite only), numpy
    scalars as Python scalars, tuples as lists, keys as strings."""
    if isinstance(v, (bool, np.bool_)):
        return bool(v)
    if isinstance(v, (int, np.integer)):
        return int(v)
    if isinstance(v, (float, np.floating)):
        x = float(v)
        if not math.isfinite(x):
            raise InvalidInputError("non-finite float in output")
        return float(f"{x:.17g}")
    if isinstance(v, dict):
        return {str(k): _plain(x) for k, x in v.items()}
    if isinstance(v, (list, tuple)):
        return [_plain(x) for x in v]
    return v


def write_json(obj, path=None) -> str:
    text = json.dumps(_plain(obj), sort_keys=True, indent=2) + "\n"
    if path and path != "-":
        with open(path, "w") as fh:
            fh.write(text)
    return text


def read_json(path: str) -> dict:
    if not os.path.exists(path):
        raise InvalidInputError(f"no such file: {path}")
    try:
        with open(path) as fh:
            return json.load(fh)
    except json.JSONDecodeError as e:
        raise InvalidInputError(f"malformed JSON in {path}: {e}") from None


def _field(obj, key, path, kind):
    try:
        return obj[key]
    except (KeyError, TypeError) as e:
        raise InvalidInputError(f"bad {kind} file {path}: {e}") from None


def read_support(path: str) -> SupportSet:
    obj = read_json(path)
    idx = _field(obj, "indices", path, "support")
    try:
        return SupportSet.make(int(_field(obj, "N", path, "support")), [int(j) for j in idx])
    except TypeError as e:
        raise InvalidInputError(f"bad support file {path}: {e}") from None


def read_signal(path: str) -> BandlimitedSignal:
    obj = read_json(path)
    try:
        J = SupportSet.make(int(_field(obj, "N", path, "signal")), [int(j) for j in _field(obj, "support", path,
                                                                                            "signal")])
        c = np.array([complex(float(p[0]), float(p[1])) for p in _field(obj, "coeffs", path, "signal")])
    except (TypeError, ValueError, IndexError) as e:
        raise InvalidInputError(f"bad signal file {path}: {e}") from None
    return BandlimitedSignal(J, c)


def spectrum_json(J: SupportSet, coeffs) -> dict:
    c = np.asarray(coeffs.detach().cpu().numpy() if hasattr(coeffs, "detach") else coeffs, dtype=np.complex128)
    return {"N": J.N, "support": [int(j) for j in J.indices], "coeffs": [[float(z.real), float(z.imag)] for z in c]}


def _emit(obj, out=None) -> int:
    text = write_json(obj, out)
    if not out:
        sys.stdout.write(text)
    return 0


def _int_list(text):
    if text is None:
        return None
    try:
        return tuple(int(t) for t in text.split(",") if t.strip())
    except ValueError:
        raise InvalidInputError(f"bad --pivots value {text!r}") from None


# ---------------------------------------------------------------- analyze ---

def cmd_analyze(args) -> int:
    from .families import doubling
    J = read_support(args.support)
    cls = classify(J)
    depth = min(cls.pivots[-1] + 1 if cls.pivots else 0, J.M)
    tree = build_tree(J, depth)
    rep = {"N": J.N, "k": len(J), "pivots": list(cls.pivots), "classification": cls.kind,
           "mu_star_profile": [tree.max_weight_at_level(l) for l in range(depth + 1)],
           "doubling": doubling(J) if len(J) <= 1 << 12 else None}
    if args.binary:
        rep["indices_binary"] = [np.binary_repr(j, width=J.M) for j in J.indices]
    if args.tree == "ascii":
        rep["tree"] = [f"{'  ' * l}L{l} res={nd.residue} weight={nd.weight} members={list(nd.members)}"
                       for l in range(depth + 1) for nd in tree.nodes_at_level(l)]
    elif args.tree == "dot":
        lines = ["digraph congruence_tree {"]
        for l in range(depth + 1):
            for nd in tree.nodes_at_level(l):
                lines.append(f'  n{l}_{nd.residue} [label="{nd.residue} mod 2^{l}\\nw={nd.weight}"];')
                if l:
                    lines.append(f"  n{l - 1}_{tree.parent(nd).residue} -> n{l}_{nd.residue};")
        rep["tree_dot"] = "\n".join(lines + ["}"])
    return _emit(rep, args.out)


# -------------------------------------------------------------- transform ---

def _device_signal(sig: BandlimitedSignal):
    """The length-N signal synthesised on the device (complex128, sfft_synthesize)."""
    import torch
    from . import _lib
    dev = _lib.require_device()
    return sig.sample_block_tensor(torch.arange(sig.N, dtype=torch.int64, device=dev))


def _algo_oracle(sig, J, args):
    """Dense DFT rows F(J, Z_N) f on the device (reference dft_direct, O(N^2));
    the counter is charged N^2 mults and N(N-1) adds outside the reported phases."""
    import torch
    if J.N > LIMITS["oracle"]:
        raise BudgetExceededError(f"oracle transform capped at N <= {LIMITS['oracle']}")
    f = _device_signal(sig)
    n = torch.arange(J.N, device=f.device, dtype=torch.int64)
    jj = torch.as_tensor(J.as_array(), device=f.device)
    ang = (-2.0 * math.pi / J.N) * ((jj[:, None] * n[None, :]) % J.N).to(torch.float64)
    coeffs = torch.polar(torch.ones_like(ang), ang) @ f
    ctr = OpCounter()
    ctr.mul(J.N * J.N)
    ctr.add(J.N * (J.N - 1))
    return coeffs, CostReport.from_counter(ctr, samples_touched=J.N)


def _algo_fft(sig, J, args):
    """Full FFT of the synthesised signal on the device, read at J; the
    radix-2 count 1.5 N log2 N in the hidft phase (reference fft_radix2)."""
    import torch
    if J.N > LIMITS["fft"]:
        raise BudgetExceededError(f"fft transform capped at N <= {LIMITS['fft']}")
    full = torch.fft.fft(_device_signal(sig))
    M = J.M
    ctr = OpCounter()
    ctr.mul((J.N // 2) * M, phase="hidft")
    ctr.add(J.N * M, phase="hidft")
    return full[torch.as_tensor(J.as_array(), device=full.device)], CostReport.from_counter(ctr, samples_touched=J.N)


def _algo_submatrix(sig, J, args):
    """The k x k Vandermonde of the first k samples (reference
    submatrix_method): the device decoder on the single node of the empty
    pivot vector, with the reference's counts (k read mults plus the
    Leja-ordered Bjorck-Pereyra cost, vandermonde_solve)."""
    from .sas import sas_transform
    k = len(J)
    if k > LIMITS["submatrix"]:
        raise InvalidInputError(f"submatrix baseline capped at k <= {LIMITS['submatrix']} on the device")
    res = sas_transform(sig, J, r=(), tolerance=args.tolerance)
    ctr = OpCounter()
    ctr.mul(k, phase="solve")
    if k > 1:
        half = k * (k - 1) // 2
        ctr.mul(k * (k - 1) + (half if k >= 3 else 0), phase="solve")
        ctr.add(3 * half + (half if k >= 3 else 0), phase="solve")
    return res.coeffs, CostReport.from_counter(ctr, samples_touched=k)


def _algo_sas(sig, J, args):
    from .sas import sas_transform, select_pivots
    meta = {}
    if args.base_pivots:
        meta["base_pivots"] = meta["pivots"] = _int_list(args.base_pivots)
    r = _int_list(args.pivots)
    if r is None and args.policy != "auto":
        r = select_pivots(J, args.policy, meta)
    out = sas_transform(sig, J, r=r, policy=args.policy, family_meta=meta, counter=OpCounter(),
                        tolerance=args.tolerance)
    return out.coeffs, out.report


def _algo_hidft(sig, J, args):
    from .hidft import hidft, hidft_to_dft
    ctr = OpCounter()
    r = _int_list(args.pivots)
    r = pivots(J) if r is None else r
    res = hidft(sig, J, r, height=args.height or 0, counter=ctr)
    if args.height is not None:  # node values at that height, no coefficients
        return None, {"N": J.N, "level": res.level, "height": res.height,
                      "nodes": {str(key): [v.real, v.imag] for key, v in res.values.items()},
                      "cost": CostReport.from_counter(ctr, samples_touched=1 << (len(r) - args.height)).as_dict()}
    coeffs = hidft_to_dft(res, ctr)
    return coeffs, CostReport.from_counter(ctr, samples_touched=len(res.slot_values))


ALGOS = {"oracle": _algo_oracle, "fft": _algo_fft, "submatrix": _algo_submatrix, "hidft": _algo_hidft,
         "sas": _algo_sas}


def cmd_transform(args) -> int:
    sig = read_signal(args.signal)
    J = sig.support
    coeffs, cost = ALGOS[args.algo](sig, J, args)
    if coeffs is None:  # --height report
        return _emit(cost, args.out)
    spec = spectrum_json(J, coeffs)
    if args.out:
        write_json(spec, args.out)
    payload = {"algo": args.algo, "cost": cost.as_dict()}
    if not args.out:
        payload["spectrum"] = spec
    sys.stdout.write(write_json(payload))
    return 0


# -------------------------------------------------------------------- gen ---

def cmd_gen(args) -> int:
    from .families import build_family, draw_coefficients
    from .workloads import rng_from_seed
    try:
        params = json.loads(args.params)
    except json.JSONDecodeError as e:
        raise InvalidInputError(f"bad --params JSON: {e}") from None
    fam = build_family(args.kind, params, args.seed)
    J = fam.support
    write_json({"N": J.N, "indices": [int(j) for j in J.indices]}, args.out)
    res = {"kind": args.kind, "N": J.N, "k": len(J), "pivots": list(pivots(J)), "classification": classify(J).kind,
           "out": args.out}
    if args.signal:
        c = draw_coefficients(len(J), rng_from_seed(args.seed, 100), nonzero=args.nonzero)
        write_json(spectrum_json(J, c), args.signal)
        res["signal"] = args.signal
    sys.stdout.write(write_json(res))
    return 0


# ------------------------------------------------------------------ bench ---

def cmd_bench(args) -> int:
    from .scenarios import CSV_COLUMNS, run_scenarios
    cfg = read_json(args.scenario)
    if args.seed is not None:
        cfg["seed"] = args.seed
    if args.tolerance is not None:
        cfg["tolerance"] = args.tolerance
    records, summary = run_scenarios(cfg)
    if args.csv:
        buf = io.StringIO()
        w = csv.writer(buf, lineterminator="\n")
        w.writerow(CSV_COLUMNS)
        for rec in records:
            w.writerow([f"{x:.17g}" if isinstance(x, float) else (int(x) if isinstance(x, bool) else x)
                        for x in rec])
        with open(args.csv, "w") as fh:
            fh.write(buf.getvalue())
    return _emit(summary, args.summary)


# ------------------------------------------------------------ entry point ---

def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="structfft", description="structured-support DFT toolkit (B200)")
    sub = ap.add_subparsers(dest="command", required=True)
    a = sub.add_parser("analyze", help="pivots, classification, weights of a support set")
    a.add_argument("support")
    a.add_argument("--binary", action="store_true")
    a.add_argument("--tree", choices=["none", "ascii", "dot"], default="none")
    a.add_argument("--out", default=None)
    a.set_defaults(func=cmd_analyze)
    t = sub.add_parser("transform", help="DFT coefficients on the support")
    t.add_argument("--signal", required=True)
    t.add_argument("--algo", required=True, choices=list(ALGOS))
    t.add_argument("--policy", default="auto", choices=["auto", "balanced", "uoe", "uoh", "random_subset"])
    t.add_argument("--pivots", default=None)
    t.add_argument("--base-pivots", default=None)
    t.add_argument("--height", type=int, default=None)
    t.add_argument("--tolerance", type=float, default=1e-8)
    t.add_argument("--out", default=None)
    t.set_defaults(func=cmd_transform)
    b = sub.add_parser("bench", help="run a seeded scenario file")
    b.add_argument("scenario")
    b.add_argument("--csv", default=None)
    b.add_argument("--summary", default=None)
    b.add_argument("--seed", type=int, default=None)
    b.add_argument("--tolerance", type=float, default=None)
    b.add_argument("--threads", type=int, default=None, help="accepted for compatibility: trials run on the GPU")
    b.set_defaults(func=cmd_bench)
    g = sub.add_parser("gen", help="generate a support (and optionally a signal)")
    g.add_argument("--kind", required=True)
    g.add_argument("--params", required=True)
    g.add_argument("--seed", type=int, default=0)
    g.add_argument("--out", required=True)
    g.add_argument("--signal", default=None)
    g.add_argument("--nonzero", action="store_true")
    g.set_defaults(func=cmd_gen)
    return ap


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except StructFFTError as e:
        for cls, code, label in EXIT:
            if isinstance(e, cls):
                print(f"{label}: {e}", file=sys.stderr)
                return code
        raise


if __name__ == "__main__":
    sys.exit(main())
