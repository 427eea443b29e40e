"""Exact-rational (fractions.Fraction) re-derivations used to PIN the oracle, test side only.

These are deliberately different algorithms from the oracle's brute force over the candidate
set: (1) a full-domain enumeration of Eq. (1) and (2) Algorithm 1 of the paper
(emit / sort / scan / argmax) executed verbatim in exact arithmetic. Neither
imports oracle/ or the CUDA path.
"""
from __future__ import annotations

import math
from fractions import Fraction as F

import numpy as np


def rows_from_json(case):
    """Build a synth-style Instance from the json 'rows' description of a golden case."""
    import synth
    n = case["n"]
    rows, cols, vals = [], [], []
    lhs, rhs = [], []
    for i, r in enumerate(case["rows"]):
        for j, a in r["a"].items():
            rows.append(i); cols.append(int(j)); vals.append(float(a))
        lhs.append(-math.inf if r["lhs"] is None else float(r["lhs"]))
        rhs.append(math.inf if r["rhs"] is None else float(r["rhs"]))
    m = len(case["rows"])
    row_ptr, col_idx, val = synth._csr_from_coo(m, n, np.array(rows, np.int64), np.array(cols, np.int64),
                                                np.array(vals, np.float64))
    return synth.Instance(case.get("name", "case"), n, m, row_ptr, col_idx, val, np.array(lhs), np.array(rhs),
                          np.array(case["lb"], np.float64), np.array(case["ub"], np.float64),
                          np.array(case["is_int"], np.uint8), np.array(case["c"], np.float64))


def normalized_rows(inst):
    """PAPER.md:345 normalisation with the documented order (upper side, then lower side)."""
    out = []
    for i in range(inst.m):
        a = {}
        for e in range(int(inst.row_ptr[i]), int(inst.row_ptr[i + 1])):
            if inst.val[e] != 0:
                a[int(inst.col_idx[e])] = F(inst.val[e])
        if not a:
            continue
        if math.isfinite(inst.rhs[i]):
            out.append((a, F(inst.rhs[i]), i, +1))
        if math.isfinite(inst.lhs[i]):
            out.append(({j: -v for j, v in a.items()}, F(-inst.lhs[i]), i, -1))
    return out


def bounds(inst):
    lb, ub = [], []
    for j in range(inst.n):
        l, u = inst.lb[j], inst.ub[j]
        if inst.is_int[j]:
            l, u = math.ceil(l) if math.isfinite(l) else l, math.floor(u) if math.isfinite(u) else u
        lb.append(l); ub.append(u)
    return lb, ub


def p(w, r_old, r_new):
    """PAPER.md:277-285 on residuals (r <= 0 = satisfied)."""
    if r_old <= 0 and r_new > 0:
        return -w
    if r_old > 0 and r_new <= 0:
        return w
    if r_old > 0 and r_new > 0 and r_new < r_old:
        return w / 2
    if r_old > 0 and r_new > 0 and r_new > r_old:
        return -w / 2
    return F(0)


def residuals(rows, x):
    return [sum(a[j] * F(x[j]) for j in a) - b for (a, b, _, _) in rows]


def column(rows, j):
    return [(i, r[0][j]) for i, r in enumerate(rows) if j in r[0]]


def score(rows, r, x, w, j, v):
    """s_j(v, x̄) = sum_i p_ij, exact."""
    return sum((p(F(float(w[i])), r[i], r[i] + a * (F(v) - F(x[j]))) for i, a in column(rows, j)), F(0))


def full_domain_best(rows, r, x, w, j, l, u):
    """max over every integer v in [l,u] minus x̄_j of s_j(v) (Eq. (1) by enumeration)."""
    best = None
    for v in range(int(l), int(u) + 1):
        if v == x[j]:
            continue
        s = score(rows, r, x, w, j, v)
        if best is None or s > best:
            best = s
    return best


def alg1(rows, r, x, w, j, l, u, is_integer):
    """Algorithm 1 verbatim in exact arithmetic, with DESIGN.md readings:
    R1 (σ uses the entry's own value, strict >), R2 (incumbent excluded), R3 (marker −1 entries
    are the candidates), R4 (tie: smallest |v−x̄|, then smallest v), R9 (infinite bound entries
    dropped). Returns (x̂, s) or (x̄, None) if no candidate."""
    xb = F(x[j])
    beta = F(0)
    alpha = F(0)
    B = []
    for q in (l, u):
        if math.isfinite(q):
            B.append((F(q), -1, F(0)))
    for i, a in column(rows, j):
        wi = F(float(w[i]))
        t = xb - r[i] / a                        # (b_i - sum_{k!=j} a_ik x̄_k) / a_ij
        if is_integer:
            t = F(math.floor(t)) if a > 0 else F(math.ceil(t))
        if a < 0:
            if xb < t:
                beta -= wi / 2; alpha += wi; B.append((t, -1, wi / 2))
            elif xb > t:
                beta -= wi; B.append((t, -1, wi))
            else:
                beta -= wi; alpha += wi
        else:
            if xb > t:
                beta += wi; alpha -= wi; B.append((t, -1, F(0))); B.append((t, +1, -wi / 2))
            elif xb < t:
                B.append((t, -1, F(0))); B.append((t, +1, -wi))
            else:
                alpha -= wi
    B.sort()                                     # lexicographic (value, marker, delta)
    P = F(0)
    best = None
    for (v, mk, d) in B:
        P += d
        sigma = beta + P + (alpha if v > xb else 0)
        if mk != -1 or v == xb or not (F(l) <= v if math.isfinite(l) else True) or \
                not (v <= F(u) if math.isfinite(u) else True):
            continue
        key = (sigma, -abs(v - xb), -v)
        if best is None or key > best[0]:
            best = (key, v, sigma)
    if best is None:
        return xb, None
    return best[1], best[2]


def rounding_ambiguous(rows, r, x, j, col_rows, values, is_integer, l, u, eps=1e-9):
    """True when Algorithm 1's result for column j is decided by a quantity within rounding distance
    of a threshold, so that an fp64 evaluation (residuals summed in any order) may legitimately take
    the other branch of a `r <= 0` test or merge two distinct breakpoints (tolerance
    mode). Checked, per row i of the column whose terms are not all integers (an all-integer row is
    exact in fp64): |r_i| and |r_i + a_ij (v - x̄_j)| for the given candidate values v against
    eps * (|b_i| + Σ_k |a_ik x̄_k|); on a continuous column also two distinct breakpoints, or a
    breakpoint and a finite bound, closer than eps * (1 + |t|)."""
    xb = F(x[j])
    ts = []
    for i in col_rows:
        a_row, b, _, _ = rows[i]
        terms = [a_row[k] * F(x[k]) for k in a_row]
        exact_row = b.denominator == 1 and all(t.denominator == 1 for t in terms)
        scale = abs(b) + sum(abs(t) for t in terms)
        a = a_row[j]
        if not is_integer:
            ts.append(xb - r[i] / a)
        if exact_row:
            continue
        if abs(r[i]) <= eps * scale:
            return True
        for v in values:
            q = r[i] + a * (F(v) - xb)
            # on a continuous column a row whose own breakpoint is v is tight there by construction
            # (Algorithm 1 orders it by its marker, not by a residual test)
            if abs(q) <= eps * scale and (is_integer or q != 0):
                return True
    if not is_integer:
        pts = sorted(set(ts) | {F(q) for q in (l, u) if math.isfinite(q)})
        for p0, p1 in zip(pts, pts[1:]):
            if p1 - p0 <= eps * (1 + abs(p1)):
                return True
    return False
