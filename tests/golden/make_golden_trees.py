"""Golden congruence trees and SAS plans from the UNMODIFIED reference.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden_trees.py

Writes tests/golden/golden_trees.npz: for each case the support, the tree
depth, and per level the members in the reference's node order (nodes
ascending by residue, members ascending -- congruence.py:134-161) with the
node offsets; the reference's split_levels() and max_weight_at_level(); and
SasPlan.plan (sas.py:69-77) for pivot prefixes.  Nothing at test time reads
/root/reference.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def main() -> None:
    sys.path.insert(0, REF)
    sys.path.insert(0, os.path.dirname(HERE))
    import structfft as R
    out = {}
    cases = [(32, [3, 17, 25, 27]), (1024, [23, 187, 190, 247, 386, 731, 990, 994]), (1024, [84, 305, 725, 992]),
             (16, [9]), (64, [3, 17, 25, 27, 35]), (64, [1, 2, 4, 8, 16, 32]), (8, [0, 1, 3]),
             (1024, [0, 1, 6, 7, 512]), (8, [0, 4]), (16, list(range(16)))]
    rng = np.random.default_rng(777)
    for _ in range(30):
        M = int(rng.integers(1, 13))
        N = 1 << M
        k = int(rng.integers(1, min(N, 200) + 1))
        cases.append((N, sorted(rng.choice(N, size=k, replace=False).tolist())))
    # a homogeneous set and the config-3 support (k = 4096 of N = 2^22)
    cases.append((1 << 12, sorted(R.gen_homogeneous((0, 3, 5, 6, 9), 12, 5).indices)))
    sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
    from paper_2211_15299_b200 import workloads as W
    J3, M3 = W.config_support(3)
    cases.append((1 << M3, J3.tolist()))
    for i, (N, idx) in enumerate(cases):
        J = R.SupportSet.make(N, idx)
        depth = J.M if i != len(cases) - 1 else 15  # config 3: up to the decode level of pivots(J)
        tree = R.build_tree(J, depth)
        k = len(J)
        mem = np.zeros((depth + 1, k), np.int64)
        off = np.zeros((depth + 1, k + 1), np.int32)
        nn = np.zeros(depth + 1, np.int32)
        for l in range(depth + 1):
            nodes = tree.nodes_at_level(l)
            nn[l] = len(nodes)
            p = 0
            for t, nd in enumerate(nodes):
                off[l, t] = p
                mem[l, p:p + nd.weight] = nd.members
                p += nd.weight
            off[l, len(nodes)] = p
        out[f"c{i}_N"] = np.int64(N)
        out[f"c{i}_J"] = np.asarray(J.indices, np.int64)
        out[f"c{i}_depth"] = np.int64(depth)
        out[f"c{i}_members"] = mem
        out[f"c{i}_off"] = off
        out[f"c{i}_n"] = nn
        out[f"c{i}_split"] = np.asarray(tree.split_levels(), np.int64)
        out[f"c{i}_maxw"] = np.asarray([tree.max_weight_at_level(l) for l in range(depth + 1)], np.int64)
        piv = R.pivots(J)
        plans = []
        for t in sorted({0, len(piv) // 2, len(piv)}):
            sp = R.SasPlan.plan(J, piv[:t])
            plans.append([t, sp.decode_level, sp.mu_star, sp.predicted_cost] + list(sp.node_weights))
        width = max(len(p) for p in plans)
        out[f"c{i}_plans"] = np.asarray([p + [-1] * (width - len(p)) for p in plans], np.float64)
    out["n_cases"] = np.int64(len(cases))
    np.savez_compressed(os.path.join(HERE, "golden_trees.npz"), **out)
    print("wrote", len(cases), "tree cases")


if __name__ == "__main__":
    main()
