"""CPU emulation of the row-sharded PDHG iteration (test infrastructure).

Each process holds the row slice `paper_2603_15504_b200.distributed` assigns
to it and runs the adaptive-step reflected-Halpern iteration with the oracle's
numpy kernels.  Cross-rank communication follows exactly the exchange plan of
the sharded CUDA graph (libpdcs `launch_slot` with a communicator): each rank
steps its x-slice only (other ranks' entries are NaN-poisoned), x~ is
all-gathered, the x- and y-space sums are all-reduced and the G^T y_hat
partial sums are reduced onto the owning slices (gloo here, NCCL on GPUs).
"""

import math
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def sharded_run(rank, world, make_problem, iters, port, out_path):
    import torch
    import torch.distributed as dist

    from oracle import pdcs_oracle as O
    from paper_2603_15504_b200.distributed import partition_cols, partition_rows, slice_problem
    from paper_2603_15504_b200.model import rsoc_to_soc

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)

    def ar(v):
        t = torch.tensor(np.atleast_1d(np.asarray(v, dtype=np.float64)))
        dist.all_reduce(t)
        return t.numpy()

    problem = make_problem()
    work = rsoc_to_soc(problem)
    Ow = O.as_oproblem(work)
    d1, d2 = O.build_scaling(Ow)
    full = O.rescale(Ow, d1, d2)
    r0, r1 = partition_rows(work, world)[rank]
    S = O.rescale(O.as_oproblem(slice_problem(work, r0, r1)), d1[r0:r1], d2)

    eta_hat = 1.0 / float(np.max(np.abs(full.G.data)))
    nc, nh = float(np.linalg.norm(full.c)), float(np.linalg.norm(full.h))
    omega = nc / nh if (nc > 1e-10 and nh > 1e-10) else 1.0
    h1, c1 = float(np.sum(np.abs(full.h))), float(np.sum(np.abs(full.c)))

    # x-split: this rank steps x-slice [c0, c1); outside it the x-space state
    # is poisoned with NaN, so any use of another rank's entries shows up in
    # the result.  Exchanged per trial exactly as the sharded CUDA graph does:
    # all-gather of x~, all-reduce of the x- and y-space sums, reduce of the
    # G^T y_hat partials onto the owner's slice.
    cuts = partition_cols(work, world)
    c0, c1 = cuts[rank], cuts[rank + 1]
    own = np.zeros(S.n, dtype=bool)
    own[c0:c1] = True

    def poison(v):
        v = np.array(v, dtype=np.float64)
        v[~own] = np.nan
        return v

    def allgather_x(v):
        parts = [None] * world
        dist.all_gather_object(parts, v[c0:c1])
        return np.concatenate(parts)

    def xdot(a, b):  # x-space sum over the slice, then over the ranks
        return float(ar(np.dot(a[own], b[own]))[0])

    nbox = S.nbox
    bown = own[:nbox]
    x, y = poison(np.zeros(S.n)), np.zeros(S.m)
    xa, ya = x.copy(), y.copy()
    xb = yb = None
    W = 0.0
    gx, gty = S.mv(np.zeros(S.n)), poison(ar(S.rmv(y)))
    gxa, gtya = gx.copy(), gty.copy()
    k = k_bar = 0
    lf, uf = np.isfinite(S.l), np.isfinite(S.u)
    for _ in range(iters):
        k_bar += 1
        grad = S.c - gty
        yy = float(ar(np.dot(y, y))[0])
        floor = 1e-14 * (1.0 + math.sqrt(omega * xdot(x, x) + yy / omega))
        eta = eta_hat
        while True:
            tau, sigma = eta / omega, eta * omega
            xh = poison(O.proj_X(S, np.where(own, x - tau * grad, 0.0)))
            xt = allgather_x(2.0 * xh - x)
            w = S.mv(xt)
            yh = O.proj_Y(S, y + sigma * (S.h - w))
            dx, dy = xh - x, yh - y
            loc = ar([np.dot(dy, dy), np.dot(dy, w - gx)])
            mv = omega * xdot(dx, dx) + loc[0] / omega
            it = abs(loc[1]) / 2.0
            bar = math.inf if (it == 0.0 or math.sqrt(mv) <= floor) else mv / (2.0 * it)
            shrink, grow = 1.0 - (k_bar + 1.0) ** -0.3, 1.0 + (k_bar + 1.0) ** -0.6
            cand = (math.inf if shrink > 0.0 else 0.0) if math.isinf(bar) else shrink * bar
            nxt = min(max(1e-12, min(cand, grow * eta)), 1e14)
            if eta < bar:
                break
            eta, k_bar = nxt, k_bar + 1
        eta_used, eta_hat = eta, nxt
        gxh = 0.5 * (w + gx)
        gtyh = poison(ar(S.rmv(yh)))  # reduce onto the owners' slices
        res = gxh - S.h
        viol = res - O.proj_residual(S, res)
        ysum = ar([np.dot(viol, viol), np.dot(yh, S.h)])
        lam = np.where(own, S.c - gtyh, 0.0)
        l1 = lam[:nbox]
        v1 = l1 - O.proj_lambda(S.l, S.u, l1)
        v2 = lam[nbox:] - O.proj_pcone_dual(S, lam[nbox:])
        p = xdot(S.c, xh)
        lsum = float(ar(np.dot(S.l[lf & bown], np.maximum(l1, 0.0)[lf & bown]))[0])
        usum = float(ar(np.dot(S.u[uf & bown], np.maximum(-l1, 0.0)[uf & bown]))[0])
        d = ysum[1] + lsum - usum
        rd2 = float(ar(np.dot(v1[bown], v1[bown]) + np.dot(v2[own[nbox:]], v2[own[nbox:]]))[0])
        e = max(math.sqrt(ysum[0]) / (1.0 + h1), math.sqrt(rd2) / (1.0 + c1),
                abs(p - d) / (1.0 + abs(p) + abs(d)))
        beta = 1.0 if e <= 0.0 else min(max(-0.1 * math.log10(e) + 0.2, 0.0), 1.0)
        a, b = (k + 1.0) / (k + 2.0), 1.0 / (k + 2.0)
        x = a * ((1.0 + beta) * xh - beta * x) + b * xa
        y = a * ((1.0 + beta) * yh - beta * y) + b * ya
        gx = a * ((1.0 + beta) * gxh - beta * gx) + b * gxa
        gty = a * ((1.0 + beta) * gtyh - beta * gty) + b * gtya
        if xb is None:
            xb, yb, W = x.copy(), y.copy(), eta_used
        else:
            tot = W + eta_used
            xb, yb, W = (W * xb + eta_used * x) / tot, (W * yb + eta_used * y) / tot, tot
        k += 1
    x = allgather_x(x)
    parts = [None] * world
    dist.all_gather_object(parts, y)
    if rank == 0:
        np.savez(out_path, x=x, y=np.concatenate(parts), k_bar=k_bar, rows=np.array([r0, r1]))
    dist.barrier()
    dist.destroy_process_group()
