"""CPU check of the reduced candidate set the general-column kernels score.

gen32_tile (csrc/eval.cuh) scores only the positive steps of a column plus the nearest candidate on
each side of x̄, in integer offsets d = t - x̄ computed as -ceil(r/a) (a > 0) / -floor(r/a) (a < 0).
This test restates that formulation in plain Python on the same per-entry table and checks it
against the oracle's brute force over the whole candidate set (oracle/, R4,
R5) on random tiny instances: the same (x̂_j, s_j) for every variable. It pins the derivation, not
the kernel (the GPU parity tests do that)."""
import math

import numpy as np

import oracle
import synth
from tests import exact


def _model_column(entries, xb, l, u, w):
    """entries: [(r_i, a_ij, w_i)] of column j at the point; returns (x̂, s) or (xb, -inf)."""
    lo = -math.inf if not math.isfinite(l) else l - xb
    hi = math.inf if not math.isfinite(u) else u - xb
    table = []   # (key, F, code) ; F = 2 delta
    b2 = a2 = 0.0
    for r, a, wi in entries:
        if r == -math.inf:
            continue
        q = r / a if r != 0 else 0.0
        d = -math.ceil(q) if a > 0 else -math.floor(q)
        if d == 0:
            if a < 0:
                b2 -= 2 * wi; a2 += 2 * wi
            else:
                a2 -= 2 * wi
            continue
        if a < 0 and d > 0:
            table.append((d, wi, 6)); b2 -= wi; a2 += 2 * wi
        elif a < 0:
            table.append((d, 2 * wi, 0)); b2 -= 2 * wi
        elif d < 0:
            table.append((d + 1, -wi, 5)); b2 += 2 * wi; a2 -= 2 * wi
        else:
            table.append((d + 1, -2 * wi, 3))
    vup = hi if (math.isfinite(u) and hi > 0) else None
    vdn = lo if (math.isfinite(l) and lo < 0) else None
    pos = []
    for key, F, code in table:
        v = key - (code & 1)
        up = code & 2
        if (up and v > hi) or (not up and v < lo):
            continue
        if up:
            vup = v if vup is None else min(vup, v)
        else:
            vdn = v if vdn is None else max(vdn, v)
        if code & 4:
            pos.append(v)
    cands = [v for v in [vup, vdn] + pos if v is not None]
    if not cands:
        return xb, -math.inf
    best = None
    for v in cands:
        s2 = b2 + (a2 if v > 0 else 0) + sum(F for key, F, _ in table if key <= v)
        k = (s2, -abs(v), -v)
        if best is None or k > best[0]:
            best = (k, v, s2)
    return xb + best[1], 0.5 * best[2]


def test_reduced_candidate_set_equals_oracle_brute_force():
    n_cols = 0
    for seed in range(600):
        kw = [{}, {"p_inf_bound": 0.4}, {"coef": 6, "bound": 9}, {"p_binary": 0.0, "coef": 4}][seed % 4]
        inst = synth.random_tiny(seed, **kw)
        try:
            O = oracle.Problem.from_instance(inst)
        except oracle.OracleError:
            continue
        lb, ub = exact.bounds(inst)
        x = np.clip(synth.random_point_tiny(inst, seed), lb, ub)
        rng = np.random.default_rng(seed)
        w = rng.integers(0, 5, O.m_norm).astype(np.float32)
        cut = math.inf if seed % 3 else float(inst.c @ x) - 2.0
        oxhat, oscore, _ = O.best_shift(x, w, cut)
        rows = exact.normalized_rows(inst)
        r = O.residuals(x, cut)
        cols = {j: [] for j in range(inst.n)}
        for i, (a, _, _, _) in enumerate(rows):
            for j, v in a.items():
                cols[j].append((r[i], float(v), float(w[i])))
        if math.isfinite(cut):
            for j in range(inst.n):
                if inst.c[j] != 0:
                    cols[j].append((r[-1], float(inst.c[j]), float(w[-1])))
        _, _, vc = O.vars()
        for j in range(inst.n):
            if vc[j] in (0, 1):   # fixed; binaries take the flip path
                continue
            v, s = _model_column(cols[j], x[j], lb[j], ub[j], w)
            assert (v, s) == (oxhat[j], oscore[j]), (inst.name, j, v, s, oxhat[j], oscore[j])
            n_cols += 1
    assert n_cols > 500
