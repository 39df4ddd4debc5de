"""Every launch variant of the step kernels against the CPU oracle.

The engine picks its step kernels per instance (lane-mapped / tiled / split /
class-split SpMV passes, vectorised epilogues, the persistent cooperative
kernel); the default choice only exercises some of them on each golden case.
`PDCS_TUNE` forces each variant on small instances of the shapes it is built
for, and the early iterates must match the oracle's (the same 1e-10 bar as
the default path's trajectory tests).
"""

import numpy as np
import pytest

from oracle import pdcs_oracle as O

pytestmark = pytest.mark.gpu


def _trajectory(P, p, opts, kbars, tune, monkeypatch):
    dev, orc = {}, {}

    def cb(s):
        if s.k_bar in kbars:
            dev[s.k_bar] = (s.z.x.copy(), s.z.y.copy())

    def ocb(st, loop):
        if st.k_bar in kbars:
            orc[st.k_bar] = (st.x.copy(), st.y.copy())

    monkeypatch.setenv("PDCS_TUNE", tune)
    try:
        P.solve(p, P.SolverOptions(**opts, iteration_callback=cb))
    finally:
        monkeypatch.delenv("PDCS_TUNE")
    O.solve(p, O.options_from(None, **opts), callback=ocb)
    return dev, orc


def _mixed():
    from paper_2603_15504_b200 import instances

    # rows of 1-2 entries (cone rows, epigraph) and of ~40 (the data rows)
    return instances.group_robust_regression(ngroups=300, gsize=10, q=400, nnz_per_row=40, seed=5)


def _primal_soc():
    from paper_2603_15504_b200 import instances

    # primal SOC(11) blocks past the box: G^T rows of the cone columns are short
    return instances.group_regression_primal(ngroups=200, gsize=10, q=300, nnz_per_row=30, seed=4)


def _primal_exp():
    from paper_2603_15504_b200 import instances

    return instances.entropy_max_primal(nblk=3000, p=40, nnz_per_col=3, seed=3)


def _exp():
    from paper_2603_15504_b200 import instances

    return instances.entropy_max(nblk=3000, p=40, nnz_per_col=3, seed=3)


def _rsoc():
    from paper_2603_15504_b200 import instances

    # C4's structure: dense factor columns give G^T rows a leading run of consecutive columns
    return instances.markowitz_rsoc(N=20_000, k=20, seed=4)


def _lp():
    from paper_2603_15504_b200 import instances

    return instances.lp_large(m=20_000, n=40_000, nnz_per_row=5, eq_frac=0.3, seed=2)


CASES = [
    ("mixed", "cls_nnz=0,cls_frac=0"),   # class split: short rows thread/row, long rows 8/32 lanes
    ("mixed", "cls_nnz=0,cls_frac=0,yblkfuse=1"),  # class split, SOC blocks inside the epilogue
    ("mixed", "halfw=16"),               # dual SOC(11) blocks on 16-lane groups (default 4)
    ("mixed", "thread_max=16"),          # ... a thread per block
    ("mixed", "halfw=8"),
    ("primal_soc", "xhalfw=16"),         # primal rescaled SOC blocks on 16-lane groups
    ("mixed", "cls=0"),                  # tiled / 8-lane step kernels
    ("mixed", "cls_nnz=0,cls_frac=0,cls_vw=32"),    # class split, 32 lanes per long row
    ("primal_soc", "cls_nnz=0,cls_frac=0"),  # class split with primal cone columns after the box
    ("primal_exp", "cls_nnz=0,cls_frac=0"),
    ("primal_exp", "xexpfuse=0"),        # x-step kernel over all coordinates + k_blk_exp<OP_STEP_X>
    ("primal_exp", "texpfuse=0"),        # fused x-step, lane t-step over all rows + k_blk_exp<OP_TLAM>
    ("primal_soc", "cls=0"),
    ("lp", "cls_nnz=0,cls_frac=0"),       # class split on uniform short rows (all in the epilogue)
    ("mixed", "cls=0,tile=1"),           # tiled step kernels forced
    ("mixed", "cls=0,tile=0"),           # lane-mapped step kernels
    ("mixed", "cls_nnz=0,cls_frac=0,vec=0"),        # class split with scalar epilogues
    ("exp", ""),                         # exp rows' y-step inside the exp block kernel
    ("exp", "expfuse=0"),                # lane y-step over all rows + k_blk_exp
    ("rsoc", "cls_nnz=0"),                # class split of G^T rows of one length (C4's structure)
    ("lp", "py=3,pt=2,split=1"),         # column panels: gather-only passes + streaming epilogues
    ("lp", "py=3,pt=2,split=0"),         # column panels, fused step kernels
    ("lp", "py=3,pt=2,split=1,hs=0,vec=0"),  # split without L2 hints / double2 epilogues
    ("lp", "persist=0"),                 # graph path
    ("lp", "persist=1"),                 # persistent cooperative kernel (if eligible)
]


@pytest.mark.parametrize("shape,tune", CASES)
def test_variant_trajectory_matches_oracle(shape, tune, monkeypatch):
    import paper_2603_15504_b200 as P

    p = {"mixed": _mixed, "lp": _lp, "primal_soc": _primal_soc, "primal_exp": _primal_exp, "exp": _exp,
         "rsoc": _rsoc}[shape]()
    kb = (1, 2, 5, 10)
    dev, orc = _trajectory(P, p, dict(max_iter=10, rel_tol=1e-14, abs_tol=1e-14), kb, tune, monkeypatch)
    assert sorted(dev) == sorted(orc) and dev, (sorted(dev), sorted(orc))
    for k in dev:
        for a, b in zip(dev[k], orc[k]):
            scale = max(1.0, float(np.max(np.abs(b))))
            assert np.max(np.abs(a - b)) <= 1e-10 * scale, (shape, tune, k, np.max(np.abs(a - b)))
