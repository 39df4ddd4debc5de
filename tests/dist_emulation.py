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


def _gap_dist(x, y, b1, b2, r, tau, sigma, px, py, xdot, ydot, t0=1.0, eps_rel=1e-8):
    """The oracle's normalized_gap (S/restart.py:80-132) with every dot
    product combined across the ranks: x-space dots over the rank's x-slice,
    y-space dots over its rows, both all-reduced (the check-path reductions
    ShardedDevice combines on GPUs).  Same probe sequence and stopping rules."""
    from oracle import pdcs_oracle as O

    if r <= O.GAP_TINY_R:
        return 0.0

    def zt(t):
        return px(x + (t * tau) * b1), py(y + (t * sigma) * b2)

    def dist(zx, zy):
        dx, dy = x - zx, y - zy
        return math.sqrt(xdot(dx, dx) / tau + ydot(dy, dy) / sigma)

    def value(zx, zy):
        return (xdot(b1, zx - x) + ydot(b2, zy - y)) / r

    tl, tr = 0.0, t0
    tk = t0
    zx, zy = zt(tk)
    d = dist(zx, zy)
    if not d > r:
        prev, stalls, found = d, 0, False
        for _ in range(O.GAP_MAX_DOUBLE):
            tk *= 2.0
            zx, zy = zt(tk)
            d = dist(zx, zy)
            if d > r:
                tr, tl, found = tk, tk / 2.0, True
                break
            if d <= prev * (1.0 + 1e-13):
                stalls += 1
                if stalls >= 2:
                    return value(zx, zy)
            else:
                stalls = 0
            prev = d
        if not found:
            raise O.OracleGapError("no bracket")
    eps = eps_rel * max(1.0, tr)
    zx, zy = zt(0.5 * (tl + tr))
    while tr - tl > eps:
        tm = 0.5 * (tl + tr)
        zx, zy = zt(tm)
        d = dist(zx, zy)
        if d < r:
            tl = tm
        else:
            tr = tm
    return value(zx, zy)


def sharded_run(rank, world, make_problem, iters, port, out_path, restart_freq=None):
    """restart_freq: None = restarts off; else duality-gap restarts checked
    every restart_freq k_bar (products refreshed, candidate z vs z_bar by the
    cross-rank normalized gap, restart criteria and primal-weight update of
    S/engine.py:467-544, S/restart.py:148-211)."""
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

    # x-split: this rank steps x-slice [xc0, xc1); outside it the x-space state
    # is poisoned with NaN, so any use of another rank's entries shows up in
    # the result.  Exchanged per trial exactly as the sharded CUDA graph does:
    # all-gather of x~, all-reduce of the x- and y-space sums, reduce of the
    # G^T y_hat partials onto the owner's slice.
    cuts = partition_cols(work, world)
    xc0, xc1 = cuts[rank], cuts[rank + 1]
    own = np.zeros(S.n, dtype=bool)
    own[xc0:xc1] = True

    def poison(v):
        v = np.array(v, dtype=np.float64)
        v[~own] = np.nan
        return v

    def allgather_x(v):
        parts = [None] * world
        dist.all_gather_object(parts, v[xc0:xc1])
        return np.concatenate(parts)

    def xdot(a, b):  # x-space sum over the slice, then over the ranks
        return float(ar(np.dot(a[own], b[own]))[0])

    nbox = S.nbox
    bown = own[:nbox]
    x, y = poison(np.zeros(S.n)), np.zeros(S.m)
    xa, ya = x.copy(), y.copy()
    xpa = ypa = None
    xb = yb = None
    W = 0.0
    gx, gty = S.mv(np.zeros(S.n)), poison(ar(S.rmv(y)))
    gxa, gtya = gx.copy(), gty.copy()
    k = k_bar = 0
    lf, uf = np.isfinite(S.l), np.isfinite(S.u)

    def ydot(a, b):
        return float(ar(np.dot(a, b))[0])

    def px(v):
        return poison(O.proj_X(S, np.where(own, v, 0.0)))

    def py(v):
        return O.proj_Y(S, v)

    def products(xv, yv):  # G^ x (local rows, x all-gathered) and G^T y (reduced onto owners)
        return S.mv(allgather_x(xv)), poison(ar(S.rmv(yv)))

    def gap_at(xv, yv, r, om, et):
        gxv, gtyv = products(xv, yv)
        return _gap_dist(xv, yv, gtyv - S.c, S.h - gxv, r, et / om, et * om, px, py, xdot, ydot)

    def nnorm(dx, dy, om, et):
        return math.sqrt(xdot(dx, dx) / (et / om) + ydot(dy, dy) / (et * om))

    omega0 = omega
    restarts, gap0, prev_cand = 0, None, math.inf
    if restart_freq:
        # baseline gap at z0 with the radius of one plain PDHG step at eta_hat (S/engine.py:380-391)
        tau, sigma = eta_hat / omega, eta_hat * omega
        xr = px(x - tau * (S.c - gty))
        w0 = S.mv(allgather_x(2.0 * xr - x))
        yr = py(y + sigma * (S.h - w0))
        gap0 = gap_at(x, y, nnorm(x - xr, y - yr, omega, eta_hat), omega, eta_hat)
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
        if restart_freq and k_bar % restart_freq == 0 and k >= 1:
            gx, gty = products(x, y)  # product refresh at every check (S/engine.py:631)

            def gm(xv, yv):
                return gap_at(xv, yv, nnorm(xv - xa, yv - ya, omega, eta_used), omega, eta_used)

            g1, g2 = gm(x, y), gm(xb, yb)
            (pxk, pyk), val = ((x, y), g1) if g1 <= g2 else ((xb, yb), g2)
            assert val >= -1e-12 and gap0 >= -1e-12, "KKT-mode fallback is not emulated"
            fire = (val <= O.R_SUFF * gap0 or (val > prev_cand and val <= O.R_NEC * gap0)
                    or k >= O.R_ART * k_bar)
            if not fire:
                prev_cand = val
            else:
                xpa, ypa = xa, ya
                xa, ya = pxk.copy(), pyk.copy()
                x, y = pxk.copy(), pyk.copy()
                dxn, dyn = math.sqrt(xdot(xa - xpa, xa - xpa)), math.sqrt(ydot(ya - ypa, ya - ypa))
                wn = omega
                if dxn > 1e-10 and dyn > 1e-10:
                    wn = math.exp(O.THETA * math.log(dyn / dxn) + (1.0 - O.THETA) * math.log(omega))
                omega = omega0 if (wn > O.W_MAX or wn < O.W_MIN) else wn
                restarts += 1
                k, xb, yb, W, prev_cand, gap0 = 0, None, None, 0.0, math.inf, val
                gx, gty = products(x, y)
                gxa, gtya = gx.copy(), gty.copy()
    x = allgather_x(x)
    parts = [None] * world
    dist.all_gather_object(parts, y)
    if rank == 0:
        np.savez(out_path, x=x, y=np.concatenate(parts), k_bar=k_bar, rows=np.array([r0, r1]),
                 restarts=restarts)
    dist.barrier()
    dist.destroy_process_group()
