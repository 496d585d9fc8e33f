"""Reference CLI outputs for the CLI parity test (run where /root/reference exists).

Writes tests/golden/cli/{signal_*.json, support_*.json, ref_*.json} from the
UNMODIFIED reference `structfft` CLI (cli.py) on small seeded inputs.
"""

import io
import json
import os
import sys
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
    for name, J in cases.items():
        c = rng.normal(size=len(J)) + 1j * rng.normal(size=len(J))
        sp = os.path.join(HERE, f"signal_{name}.json")
        cli.dump_json(cli.signal_to_json(J, c), sp)
        cli.dump_json(cli.support_to_json(J), os.path.join(HERE, f"support_{name}.json"))
        runs = {"sas": ["transform", "--signal", sp, "--algo", "sas"],
                "analyze": ["analyze", os.path.join(HERE, f"support_{name}.json"), "--binary"]}
        if R.classify(J).is_homogeneous:
            runs["hidft"] = ["transform", "--signal", sp, "--algo", "hidft"]
            runs["hidft_h1"] = ["transform", "--signal", sp, "--algo", "hidft", "--height", "1"]
        for tag, argv in runs.items():
            buf = io.StringIO()
            with redirect_stdout(buf):
                rc = cli.main(argv)
            with open(os.path.join(HERE, f"ref_{name}_{tag}.json"), "w") as fh:
                json.dump({"argv": argv[:1] + [a.replace(HERE, "{DIR}") for a in argv[1:]], "rc": rc,
                           "stdout": buf.getvalue()}, fh)
    print(sorted(os.listdir(HERE)))


if __name__ == "__main__":
    main()
