"""TEST INFRASTRUCTURE ONLY — plain restarted PDHG for the LP relaxation (the oracle of the streamed
LP iterates, NEXT f4; same import rules as oracle/__init__.py).

PAPER.md:379-387 (§3.3 "Streaming LP Iterates"): PDHG iterates are streamed at checkpoints after
10^2, 10^3, 10^4 (and 10^5) iterations, warm-starting each phase from the previous iterate, and are
used to initialise the heuristics. The PDHG internals are the paper's cited method family, stated
here as SPEC.md:339-374 fixes them (R19):

    x+ = proj_[l,u](x - eta (c + A^T y))                 (primal step)
    y+ = max(0, y + tau (A (2 x+ - x) - b))               (dual step, one y_i >= 0 per <= row)

with running averages of x+ and y+, a restart to the averages every R iterations, and at each
checkpoint a snapshot of the current averages. A is the matrix of the normalised rows (PAPER.md:345:
every finite side of a row as a <= row, upper side first); the cutoff row is not part of the LP.
Written as the formulas above with scipy.sparse products, in fp64, no reordering.
"""
from __future__ import annotations

import math

import numpy as np
import scipy.sparse as sp


def normalized_lp(inst):
    """(A, b, c, l, u) of min c.x s.t. A x <= b, l <= x <= u: each finite side of every nonempty row as
    a <= row, the upper side (a x <= rhs) first, then the lower side (-a x <= -lhs);
    integer bounds rounded inward."""
    rows, cols, vals, b = [], [], [], []
    r = 0
    for i in range(inst.m):
        s, e = int(inst.row_ptr[i]), int(inst.row_ptr[i + 1])
        cj, av = inst.col_idx[s:e], inst.val[s:e]
        keep = av != 0
        cj, av = cj[keep], av[keep]
        if cj.size == 0:
            continue
        for side, bb in ((1.0, inst.rhs[i]), (-1.0, -inst.lhs[i])):
            if math.isfinite(bb):
                rows.extend([r] * cj.size)
                cols.extend(cj.tolist())
                vals.extend((side * av).tolist())
                b.append(bb)
                r += 1
    A = sp.csr_matrix((np.array(vals, float), (np.array(rows, int), np.array(cols, int))), shape=(r, inst.n))
    l = np.where(inst.is_int.astype(bool), np.ceil(inst.lb), inst.lb)
    u = np.where(inst.is_int.astype(bool), np.floor(inst.ub), inst.ub)
    return A, np.array(b, float), inst.c.astype(float), l, u


def operator_norm(A, iters: int = 200, seed: int = 0):
    """||A||_2 by power iteration on A^T A."""
    if A.nnz == 0:
        return 0.0
    v = np.random.default_rng(seed).standard_normal(A.shape[1])
    v /= np.linalg.norm(v)
    s = 0.0
    for _ in range(iters):
        w = A.T @ (A @ v)
        s = math.sqrt(np.linalg.norm(w))
        v = w / np.linalg.norm(w)
    return s


def pdhg(inst, checkpoints, step, restart_period=400, x0=None, y0=None):
    """Restarted PDHG with eta = tau = step; returns [(iteration, x_avg, y_avg)] at the checkpoints
    (the averages since the last restart) and the final iterates (x, y)."""
    A, b, c, l, u = normalized_lp(inst)
    AT = A.T.tocsr()
    x = np.clip(np.zeros(inst.n) if x0 is None else np.asarray(x0, float), l, u)
    y = np.zeros(A.shape[0]) if y0 is None else np.asarray(y0, float).copy()
    xs, ys, cnt = np.zeros_like(x), np.zeros_like(y), 0
    snaps = []
    cps = sorted(checkpoints)
    k = 0
    for cp in cps:
        while k < cp:
            xn = np.clip(x - step * (c + AT @ y), l, u)
            y = np.maximum(0.0, y + step * (A @ (2.0 * xn - x) - b))
            x = xn
            xs += x
            ys += y
            cnt += 1
            k += 1
            if cnt == restart_period:   # restart to the average
                x, y = xs / cnt, ys / cnt
                xs, ys, cnt = np.zeros_like(x), np.zeros_like(y), 0
        snaps.append((k, xs / cnt if cnt else x.copy(), ys / cnt if cnt else y.copy()))
    return snaps, (x, y)


def round_point(inst, x):
    """An LP point to a tabu start point: integer variables to the nearest integer
    (half away from zero), everything clamped to the bounds."""
    l = np.where(inst.is_int.astype(bool), np.ceil(inst.lb), inst.lb)
    u = np.where(inst.is_int.astype(bool), np.floor(inst.ub), inst.ub)
    r = np.where(inst.is_int.astype(bool), np.sign(x) * np.floor(np.abs(x) + 0.5), x)
    return np.clip(r, l, u)
