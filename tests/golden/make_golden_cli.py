"""Reference CLI outputs for the CLI parity test (run where /root/reference exists).

Writes tests/golden/cli/{signal_*.json, support_*.json, scenario.json,
ref_*.json} from the UNMODIFIED reference `structfft` CLI (cli.py) on small
seeded inputs: analyze (with --binary / --tree), transform with every
--algo, gen for every family kind, and bench on a small scenario file.
Output files a command writes are stored in its ref_*.json under "files";
argv paths use {DIR} (this directory) and {OUT} (the test's temp directory).
"""

import io
import json
import os
import sys
import tempfile
from contextlib import redirect_stdout

import numpy as np

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cli")


def main():
    sys.path.insert(0, "/root/reference/pkg/src")
    import structfft as R
    from structfft import cli
    os.makedirs(HERE, exist_ok=True)
    rng = np.random.default_rng(7)
    cases = {
        "homog": R.gen_homogeneous((0, 2, 5, 7), 12, 3),
        "paper": R.SupportSet.make(1024, [0, 1, 6, 7, 512]),
        "subset": R.SupportSet.make(1 << 12, sorted(rng.choice(1 << 12, size=40, replace=False).tolist())),
    }
    runs = {}
    for name, J in cases.items():
        c = rng.normal(size=len(J)) + 1j * rng.normal(size=len(J))
        sp = os.path.join(HERE, f"signal_{name}.json")
        cli.dump_json(cli.signal_to_json(J, c), sp)
        su = os.path.join(HERE, f"support_{name}.json")
        cli.dump_json(cli.support_to_json(J), su)
        runs[f"{name}_sas"] = ["transform", "--signal", sp, "--algo", "sas"]
        runs[f"{name}_analyze"] = ["analyze", su, "--binary"]
        for algo in ("oracle", "fft", "submatrix"):
            runs[f"{name}_{algo}"] = ["transform", "--signal", sp, "--algo", algo]
        if R.classify(J).is_homogeneous:
            runs[f"{name}_hidft"] = ["transform", "--signal", sp, "--algo", "hidft"]
            runs[f"{name}_hidft_h1"] = ["transform", "--signal", sp, "--algo", "hidft", "--height", "1"]
    runs["paper_tree_ascii"] = ["analyze", os.path.join(HERE, "support_paper.json"), "--tree", "ascii"]
    runs["homog_tree_dot"] = ["analyze", os.path.join(HERE, "support_homog.json"), "--tree", "dot"]
    runs["paper_sas_pivots"] = ["transform", "--signal", os.path.join(HERE, "signal_paper.json"), "--algo", "sas",
                                "--pivots", "0,1"]
    gens = {
        "homogeneous": {"pivots": [0, 2, 5], "M": 10},
        "elementary": {"r": 3, "M": 8},
        "consecutive": {"a": 5, "k": 9, "N": 64},
        "ap": {"a": 3, "s": 6, "k": 7, "N": 128},
        "gap": {"a": 1, "steps": [3, 10], "lengths": [4, 5], "N": 256},
        "uoe": {"a_n": 3, "etas": [1, 1, 0, 1], "M": 9},
        "uoh": {"base_pivots": [0, 1, 3, 6], "a_n": 2, "etas": [0, 1, 1], "M": 9},
        "random_subset": {"M": 8, "k": 20},
        "jstar": {"M": 6},
    }
    for kind, params in gens.items():
        argv = ["gen", "--kind", kind, "--params", json.dumps(params), "--seed", "11", "--out",
                "{OUT}/gen_%s.json" % kind]
        if kind in ("homogeneous", "random_subset"):
            argv += ["--signal", "{OUT}/gen_%s_signal.json" % kind]
        if kind == "random_subset":
            argv += ["--nonzero"]
        runs[f"gen_{kind}"] = argv
    runs["gen_rs_homogeneous"] = ["gen", "--kind", "random_subset", "--params",
                                  json.dumps({"M": 10, "k": 12, "base": "homogeneous",
                                              "base_pivots": [0, 2, 3, 5, 7]}), "--seed", "4", "--out",
                                  "{OUT}/gen_rsh.json"]
    scen = {"name": "parity", "seed": 5, "tolerance": 1e-8, "scenarios": [
        {"kind": "homogeneous", "trials": 3, "params": {"M": [6, 9]}},
        {"kind": "fixture", "trials": 1, "params": {"name": "paper_sas"}},
        {"kind": "random_subset", "trials": 3, "params": {"M": 8, "k": [8, 20]}},
        {"kind": "elementary", "trials": 2, "params": {"M": 8}},
        {"kind": "consecutive", "trials": 2, "params": {"M": 8, "k": [3, 12]}},
        {"kind": "ap", "trials": 2, "params": {"M": 9, "k": [3, 10]}},
        {"kind": "uoe", "trials": 2, "params": {"M": 8, "a_n": [1, 3]}},
        {"kind": "uoh", "trials": 2, "params": {"M": 9, "s": [3, 5]}},
        {"kind": "gap", "trials": 2, "params": {"M": 9, "d": [1, 2], "volume_cap": 64}},
        {"kind": "jstar", "trials": 1, "params": {"M": 6}},
        {"kind": "antipodal", "trials": 5, "params": {"M": 8}},
    ]}
    with open(os.path.join(HERE, "scenario.json"), "w") as fh:
        json.dump(scen, fh)
    runs["bench"] = ["bench", os.path.join(HERE, "scenario.json"), "--csv", "{OUT}/bench.csv"]
    for tag, argv in runs.items():
        with tempfile.TemporaryDirectory() as tmp:
            real = [a.replace("{OUT}", tmp) for a in argv]
            buf = io.StringIO()
            with redirect_stdout(buf):
                rc = cli.main(real)
            files = {}
            for a in argv:
                if a.startswith("{OUT}/"):
                    p = a.replace("{OUT}", tmp)
                    if os.path.exists(p):
                        files[os.path.basename(p)] = open(p).read()
            stdout = buf.getvalue().replace(tmp, "{OUT}")
        with open(os.path.join(HERE, f"ref_{tag}.json"), "w") as fh:
            json.dump({"argv": argv[:1] + [a.replace(HERE, "{DIR}") for a in argv[1:]], "rc": rc, "stdout": stdout,
                       "files": files}, fh)
    print(len(runs), "runs")


if __name__ == "__main__":
    main()
