"""CPU emulation of the row-sharded PDHG iteration (test infrastructure).

Each process holds the row slice `paper_2603_15504_b200.distributed` assigns
to it and runs the adaptive-step reflected-Halpern iteration with the oracle's
numpy kernels.  Cross-rank communication follows exactly the reduction plan of
the sharded CUDA graph (libpdcs `launch_slot` with a communicator): y-space
line-search / beta sums and the G^T y_hat partial sums are all-reduced
(gloo here, NCCL on GPUs); all x-space work is replicated.
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
    from paper_2603_15504_b200.distributed import partition_rows, slice_problem
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
    x, y = np.zeros(S.n), np.zeros(S.m)
    xa, ya = x.copy(), y.copy()
    xb = yb = None
    W = 0.0
    gx, gty = S.mv(x), ar(S.rmv(y))
    gxa, gtya = gx.copy(), gty.copy()
    k = k_bar = 0
    lf, uf = np.isfinite(S.l), np.isfinite(S.u)
    for _ in range(iters):
        k_bar += 1
        grad = S.c - gty
        yy = float(ar(np.dot(y, y))[0])
        floor = 1e-14 * (1.0 + math.sqrt(omega * float(np.dot(x, x)) + yy / omega))
        eta = eta_hat
        while True:
            tau, sigma = eta / omega, eta * omega
            xh = O.proj_X(S, x - tau * grad)
            w = S.mv(2.0 * xh - x)
            yh = O.proj_Y(S, y + sigma * (S.h - w))
            dx, dy = xh - x, yh - y
            loc = ar([np.dot(dy, dy), np.dot(dy, w - gx)])
            mv = omega * float(np.dot(dx, dx)) + loc[0] / omega
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
        gtyh = ar(S.rmv(yh))
        # beta on the scaled problem: y-space sums all-reduced, x-space replicated
        res = gxh - S.h
        viol = res - O.proj_residual(S, res)
        ysum = ar([np.dot(viol, viol), np.dot(yh, S.h)])
        lam = S.c - gtyh
        l1 = lam[:S.nbox]
        v1 = l1 - O.proj_lambda(S.l, S.u, l1)
        v2 = lam[S.nbox:] - O.proj_pcone_dual(S, lam[S.nbox:])
        p = float(np.dot(S.c, xh))
        d = ysum[1] + float(np.dot(S.l[lf], np.maximum(l1, 0.0)[lf])) - float(
            np.dot(S.u[uf], np.maximum(-l1, 0.0)[uf]))
        e = max(math.sqrt(ysum[0]) / (1.0 + h1),
                math.sqrt(float(np.dot(v1, v1)) + float(np.dot(v2, v2))) / (1.0 + c1),
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
    parts = [None] * world
    dist.all_gather_object(parts, y)
    if rank == 0:
        np.savez(out_path, x=x, y=np.concatenate(parts), k_bar=k_bar, rows=np.array([r0, r1]))
    dist.barrier()
    dist.destroy_process_group()
