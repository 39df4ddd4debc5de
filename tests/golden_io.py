"""Load the golden fixtures (tests/golden/*.npz, made by make_golden.py)."""

import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name: str) -> dict:
    with np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def problem(d: dict):
    from paper_2603_15504_b200.linalg import SparseMatrix
    from paper_2603_15504_b200.model import Cone, ConeSpec, ConicProblem

    shape = tuple(int(s) for s in d["shape"])
    G = SparseMatrix.from_csr_arrays(d["indptr"], d["indices"], d["data"], shape)
    pk = json.loads(str(d["pkinds"]))
    dk = json.loads(str(d["dkinds"]))
    return ConicProblem(
        c=d["c"], G=G, h=d["h"], l=d["l"], u=d["u"], num_box=int(d["num_box"]),
        primal_cones=tuple(ConeSpec(Cone(k), int(n)) for k, n in zip(pk, d["pdims"])),
        dual_cones=tuple(ConeSpec(Cone(k), int(n)) for k, n in zip(dk, d["ddims"])))


def options(d: dict) -> dict:
    return json.loads(str(d["opts_json"]))


SOLVE_CASES = ["tiny", "ball", "expc", "dexp", "rsoc", "prim", "infeas", "unbnd", "maxit", "plain",
               "c1s", "c1s_avg", "c1s_kkt", "c2s", "c3s", "c4s", "c5s"]
