"""The reference's own iteration band for every small golden solve
(tests/golden/solve_*.npz): the reference re-solved with 6 noise seeds, each
SpMV output x (1 + 2.2e-16 N(0,1)) (the model of GPU
summation reordering).  Writes tests/golden/noise_bands.json:
{case: [nominal, min, max]}.  Build container only (imports /root/reference).

    python tests/golden/make_noise_bands.py
"""

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))

from golden_io import SOLVE_CASES, load, options, problem  # noqa: E402
from make_golden_scale import ref_solve  # noqa: E402


def main():
    out = {}
    for case in SOLVE_CASES:
        d = load("solve_" + case)
        p, o = problem(d), options(d)
        its = [int(ref_solve(p, o, noise_seed=s)[0].iterations) for s in (1, 2, 3, 4, 5, 6)]
        nominal = int(d["iterations"])
        out[case] = [nominal, min(its + [nominal]), max(its + [nominal])]
        print(case, out[case], flush=True)
    with open(os.path.join(HERE, "noise_bands.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
