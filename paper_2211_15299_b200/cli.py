"""Command-line front end with the reference's file formats (cli.py:1-11).

    python -m paper_2211_15299_b200 transform --signal S.json --algo hidft|sas [...]
    python -m paper_2211_15299_b200 analyze SUPPORT.json [--binary]

support file  {"N": int, "indices": [int, ...]}
signal file   {"N": int, "support": [...], "coeffs": [[re, im], ...]}
Output is canonical JSON (sorted keys, floats at 17 significant digits);
exit codes 0 ok, 2 input error, 3 contract violation, 4 budget exceeded.
The transforms run on the B200 (hidft, sas); the reference's host oracles
(--algo oracle/fft/submatrix) are not part of this package.
"""

from __future__ import annotations

import argparse
import json
import sys

import numpy as np

from .congruence import SupportSet, classify, pivots
from .counting import OpCounter
from .errors import BudgetExceededError, ContractViolationError, InvalidInputError
from .hidft import hidft, hidft_to_dft
from .sas import CostReport, _prefix_profile, sas_transform, select_pivots
from .signals import BandlimitedSignal


def _canonical(obj):
    if isinstance(obj, float):
        if obj != obj or obj in (float("inf"), float("-inf")):
            raise InvalidInputError("non-finite float in output")
        return float(format(obj, ".17g"))
    if isinstance(obj, dict):
        return {str(k): _canonical(v) for k, v in obj.items()}
    if isinstance(obj, (list, tuple)):
        return [_canonical(v) for v in obj]
    if isinstance(obj, np.integer):
        return int(obj)
    if isinstance(obj, np.floating):
        return _canonical(float(obj))
    if isinstance(obj, np.bool_):
        return bool(obj)
    return obj


def dump_json(obj, path: str | None) -> str:
    text = json.dumps(_canonical(obj), sort_keys=True, indent=2) + "\n"
    if path and path != "-":
        with open(path, "w") as fh:
            fh.write(text)
    return text


def _load_json(path: str) -> dict:
    try:
        with open(path) as fh:
            return json.load(fh)
    except FileNotFoundError:
        raise InvalidInputError(f"no such file: {path}") from None
    except json.JSONDecodeError as e:
        raise InvalidInputError(f"malformed JSON in {path}: {e}") from None


def load_support(path: str) -> SupportSet:
    obj = _load_json(path)
    try:
        return SupportSet.make(int(obj["N"]), [int(j) for j in obj["indices"]])
    except (KeyError, TypeError) as e:
        raise InvalidInputError(f"bad support file {path}: {e}") from None


def load_signal(path: str) -> BandlimitedSignal:
    obj = _load_json(path)
    try:
        J = SupportSet.make(int(obj["N"]), [int(j) for j in obj["support"]])
        coeffs = np.asarray([complex(re, im) for re, im in obj["coeffs"]])
    except (KeyError, TypeError, ValueError) as e:
        raise InvalidInputError(f"bad signal file {path}: {e}") from None
    return BandlimitedSignal(J, coeffs)


def signal_to_json(J: SupportSet, coeffs) -> dict:
    c = np.asarray(coeffs.detach().cpu().numpy() if hasattr(coeffs, "detach") else coeffs).reshape(-1)
    return {"N": J.N, "support": list(J.indices), "coeffs": [[float(x.real), float(x.imag)] for x in c]}


def _parse_pivots(text):
    if text is None:
        return None
    try:
        return tuple(int(x) for x in text.split(",") if x.strip() != "")
    except ValueError:
        raise InvalidInputError(f"bad --pivots value {text!r}") from None


def cmd_analyze(args) -> int:
    J = load_support(args.support)
    cls = classify(J)
    p = cls.pivots
    depth = min((p[-1] + 1) if p else 0, J.M)
    mu, _ = _prefix_profile(J, p)  # weights change only at pivot levels
    profile = [int(mu[sum(1 for x in p if x < level)]) for level in range(depth + 1)]
    report = {"N": J.N, "k": len(J), "pivots": list(p), "classification": cls.kind,
              "mu_star_profile": profile, "doubling": None}
    if args.binary:
        report["indices_binary"] = [format(j, f"0{J.M}b") for j in J.indices]
    text = dump_json(report, args.out)
    if not args.out:
        sys.stdout.write(text)
    return 0


def cmd_transform(args) -> int:
    sig = load_signal(args.signal)
    J = sig.support
    counter = OpCounter()
    explicit_r = _parse_pivots(args.pivots)
    if args.algo == "hidft":
        r = explicit_r if explicit_r is not None else pivots(J)
        height = args.height if args.height is not None else 0
        res = hidft(sig, J, r, height=height, counter=counter)
        if args.height is not None:
            report = {"N": J.N, "level": res.level, "height": res.height,
                      "nodes": {str(k): [v.real, v.imag] for k, v in res.values.items()},
                      "cost": CostReport.from_counter(counter, samples_touched=1 << (len(r) - height)).as_dict()}
            text = dump_json(report, args.out)
            if not args.out:
                sys.stdout.write(text)
            return 0
        coeffs = hidft_to_dft(res, counter)
        cost = CostReport.from_counter(counter, samples_touched=len(res.slot_values))
    elif args.algo == "sas":
        meta = {}
        if args.base_pivots:
            meta["base_pivots"] = _parse_pivots(args.base_pivots)
            meta["pivots"] = meta["base_pivots"]
        r = explicit_r
        if r is None and args.policy != "auto":
            r = select_pivots(J, args.policy, meta)
        out = sas_transform(sig, J, r=r, policy=args.policy, family_meta=meta, counter=counter,
                            tolerance=args.tolerance)
        coeffs = out.coeffs
        cost = out.report
    else:
        raise InvalidInputError(f"--algo {args.algo} is a host oracle of the reference, not on the device path")
    spectrum = signal_to_json(J, coeffs)
    if args.out:
        dump_json(spectrum, args.out)
    payload = {"algo": args.algo, "cost": cost.as_dict()}
    if not args.out:
        payload["spectrum"] = spectrum
    sys.stdout.write(dump_json(payload, None))
    return 0


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="structfft-b200", description="structured-support DFT on B200")
    sub = ap.add_subparsers(dest="command", required=True)
    a = sub.add_parser("analyze", help="pivots, classification, node-weight profile of a support set")
    a.add_argument("support")
    a.add_argument("--binary", action="store_true")
    a.add_argument("--out", default=None)
    a.set_defaults(func=cmd_analyze)
    t = sub.add_parser("transform", help="compute DFT coefficients on the support")
    t.add_argument("--signal", required=True)
    t.add_argument("--algo", required=True, choices=["oracle", "fft", "submatrix", "hidft", "sas"])
    t.add_argument("--policy", default="auto", choices=["auto", "balanced", "uoe", "uoh", "random_subset"])
    t.add_argument("--pivots", default=None)
    t.add_argument("--base-pivots", default=None)
    t.add_argument("--height", type=int, default=None)
    t.add_argument("--tolerance", type=float, default=1e-8)
    t.add_argument("--out", default=None)
    t.set_defaults(func=cmd_transform)
    return ap


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except InvalidInputError as e:
        print(f"input error: {e}", file=sys.stderr)
        return 2
    except ContractViolationError as e:
        print(f"contract violation: {e}", file=sys.stderr)
        return 3
    except BudgetExceededError as e:
        print(f"budget exceeded: {e}", file=sys.stderr)
        return 4
