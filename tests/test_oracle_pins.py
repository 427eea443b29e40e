"""Pins for the CPU oracle (oracle/), independent of the oracle's own code (CPU only).

Each test checks the oracle against something the paper or mathematics fixes: the penalty
table's case rows, the breakpoint formula's worked values, hand-worked columns, a full-domain
enumeration of Eq. (1), and Algorithm 1 executed verbatim in exact rationals (tests/exact.py).
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
import synth
from tests import exact

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


@pytest.mark.parametrize("case", _load("penalty_cases.json")["cases"], ids=lambda c: c["cite"][:40])
def test_penalty_table(case):
    assert oracle.penalty(case["w"], case["r_old"], case["r_new"]) == case["p"]


def test_penalty_antisymmetry_and_scaling():
    # reward/penalty equal to the weight on sat<->unsat transitions
    rng = np.random.default_rng(0)
    for _ in range(2000):
        w = float(rng.integers(0, 9))
        a, b = sorted(rng.integers(-5, 6, 2).astype(float))
        r_sat, r_vio = min(a, 0.0), max(b, 0.5)
        assert oracle.penalty(w, r_sat, r_vio) == -w
        assert oracle.penalty(w, r_vio, r_sat) == w
        # both violated: sign of the half-weight follows the direction of the change
        r1, r2 = 1.0 + abs(a), 1.0 + abs(b)
        expect = 0.0 if r1 == r2 else (0.5 * w if r2 < r1 else -0.5 * w)
        assert oracle.penalty(w, r1, r2) == expect


@pytest.mark.parametrize("case", _load("breakpoints.json")["cases"], ids=lambda c: c["cite"][:30])
def test_breakpoint_worked(case):
    # row "2x1 + x2 <= 4" -> a=2, r = 2*0 + 1 - 4 = -3 ; row "-x1 <= -1" -> a=-1, r = 0 + 1 = 1
    if case["row"] == "2 x1 + x2 <= 4":
        a, r = 2.0, 2.0 * case["xbar"][0] + case["xbar"][1] - 4.0
    else:
        a, r = -1.0, -case["xbar"][0] + 1.0
    assert oracle.breakpoint(case["xbar"][case["j"]], r, a, case["is_integer"]) == case["t"]


@pytest.mark.parametrize("case", _load("alg1_worked.json")["cases"], ids=lambda c: c["name"])
def test_alg1_worked_cases(case):
    inst = exact.rows_from_json(case)
    P = oracle.Problem.from_instance(inst)
    xhat, score, best = P.best_shift(np.array(case["x"], float))
    assert list(xhat) == case["xhat"]
    assert [None if s == -math.inf else s for s in score] == case["score"]
    bj, bv, bs = best
    assert bj == case["best"][0]
    if bj >= 0:
        assert (bv, bs) == (case["best"][1], case["best"][2])


def test_normalisation_examples():
    # "x1 + x2 >= 3" -> "-x1 - x2 <= -3"; "x1 = 2" -> "x1 <= 2", "-x1 <= -2"
    case = {"n": 2, "rows": [{"a": {"0": 1, "1": 1}, "lhs": 3, "rhs": None},
                             {"a": {"0": 1}, "lhs": 2, "rhs": 2},
                             {"a": {"1": 0}, "lhs": -1, "rhs": 1},       # empty row dropped
                             {"a": {"0": 2}, "lhs": None, "rhs": None}],  # free row dropped
            "lb": [0, 0], "ub": [5, 5], "is_int": [1, 1], "c": [1, 0]}
    inst = exact.rows_from_json(case)
    P = oracle.Problem.from_instance(inst)
    assert P.m_norm == 3 + 1 and P.nnz_norm == 4 and P.nnz_cut == 1
    orig, side = P.row_map()
    assert list(orig) == [0, 1, 1] and list(side) == [-1, 1, -1]
    # residuals at x = (1, 1): -2 - (-3) = 1 ; 1 - 2 = -1 ; -1 - (-2) = 1
    r = P.residuals(np.array([1.0, 1.0]))
    assert list(r[:3]) == [1.0, -1.0, 1.0] and r[3] == -math.inf
    r = P.residuals(np.array([1.0, 1.0]), cutoff_rhs=0.5)
    assert r[3] == 0.5


def test_error_paths():
    base = {"n": 1, "rows": [{"a": {"0": 1}, "lhs": None, "rhs": 1}], "lb": [0], "ub": [1], "is_int": [1], "c": [0]}
    inst = exact.rows_from_json(base)
    # l > u after inward rounding of integer bounds
    with pytest.raises(oracle.OracleError) as e:
        oracle.Problem(1, 1, inst.row_ptr, inst.col_idx, inst.val, inst.lhs, inst.rhs,
                       np.array([0.2]), np.array([0.8]), inst.is_int, inst.c)
    assert e.value.code == oracle.ORC_ERR_INFEASIBLE_BOUNDS
    # duplicate (i, j)
    with pytest.raises(oracle.OracleError) as e:
        oracle.Problem(1, 1, np.array([0, 2]), np.array([0, 0]), np.array([1.0, 1.0]), inst.lhs, inst.rhs,
                       inst.lb, inst.ub, inst.is_int, inst.c)
    assert e.value.code == oracle.ORC_ERR_INVALID_ARG
    # NaN coefficient
    with pytest.raises(oracle.OracleError):
        oracle.Problem(1, 1, inst.row_ptr, inst.col_idx, np.array([math.nan]), inst.lhs, inst.rhs,
                       inst.lb, inst.ub, inst.is_int, inst.c)
    # empty row that excludes 0
    with pytest.raises(oracle.OracleError) as e:
        oracle.Problem(1, 1, np.array([0, 0]), np.zeros(0, np.int32), np.zeros(0), np.array([1.0]),
                       np.array([2.0]), inst.lb, inst.ub, inst.is_int, inst.c)
    assert e.value.code == oracle.ORC_ERR_INFEASIBLE_BOUNDS


def _tiny_cases(n_cases, **kw):
    for seed in range(n_cases):
        inst = synth.random_tiny(seed, **kw)
        try:
            P = oracle.Problem.from_instance(inst)
        except oracle.OracleError:
            continue
        x = synth.random_point_tiny(inst, seed)
        lb, ub = exact.bounds(inst)
        x = np.clip(x, lb, ub)
        rng = np.random.default_rng(seed)
        w = rng.integers(0, 5, P.m_norm).astype(np.float32)   # weights >= 0 (zero allowed)
        yield inst, P, x, w, lb, ub


def test_full_domain_max_equals_oracle():
    """s_j(., x̄) is a step function with steps only at breakpoints and bounds, so
    the maximum over the oracle's finite candidate set equals the maximum over all of D_j."""
    checked = 0
    for inst, P, x, w, lb, ub in _tiny_cases(2500):
        rows = exact.normalized_rows(inst)
        r = exact.residuals(rows, x)
        xhat, score, _ = P.best_shift(x, w)
        for j in range(inst.n):
            if lb[j] == ub[j]:
                assert score[j] == -math.inf and xhat[j] == x[j]
                continue
            m = exact.full_domain_best(rows, r, x, w, j, lb[j], ub[j])
            assert score[j] == float(m), (inst.name, j)
            # the returned shift attains the returned score (exact recompute)
            assert exact.score(rows, r, x, w, j, xhat[j]) == m
            assert xhat[j] != x[j] and lb[j] <= xhat[j] <= ub[j] and xhat[j] == math.floor(xhat[j])
            checked += 1
    assert checked > 5000


def test_alg1_exact_equals_oracle():
    """Algorithm 1 (sort-scan-argmax) in exact rationals selects the same
    (x̂_j, s_j) as the oracle's candidate brute force, under readings R1-R5, R9."""
    checked = 0
    for kw in ({}, {"p_inf_bound": 0.3}, {"coef": 6, "bound": 9}):
        for inst, P, x, w, lb, ub in _tiny_cases(1500, **kw):
            rows = exact.normalized_rows(inst)
            r = exact.residuals(rows, x)
            xhat, score, best = P.best_shift(x, w)
            for j in range(inst.n):
                if lb[j] == ub[j]:
                    continue
                v, s = exact.alg1(rows, r, x, w, j, lb[j], ub[j], True)
                if s is None:
                    assert score[j] == -math.inf and xhat[j] == x[j]
                else:
                    assert (xhat[j], score[j]) == (float(v), float(s)), (inst.name, j)
                checked += 1
            # best move: max positive score, lowest j (R6)
            pos = [(score[j], -j) for j in range(inst.n) if score[j] > 0]
            if pos:
                s_, mj = max(pos)
                assert best[0] == -mj and best[2] == s_ and best[1] == xhat[-mj]
            else:
                assert best[0] == -1
    assert checked > 8000


def test_binary_flip_closed_form():
    """a binary's only move is the flip; its score is sum_i p(w, r, r + a(1-2x̄))."""
    for seed in range(200):
        inst = synth.random_tiny(seed, p_binary=1.0, n_max=8)
        try:
            P = oracle.Problem.from_instance(inst)
        except oracle.OracleError:
            continue
        rows = exact.normalized_rows(inst)
        x = synth.random_point_tiny(inst, seed)
        w = np.ones(P.m_norm, np.float32)
        r = exact.residuals(rows, x)
        xhat, score, _ = P.best_shift(x, w)
        for j in range(inst.n):
            s = sum((exact.p(1, r[i], r[i] + a * (1 - 2 * int(x[j]))) for i, a in exact.column(rows, j)),
                    exact.F(0))
            assert xhat[j] == 1 - x[j] and score[j] == float(s)


def test_cutoff_row_scored_like_any_row():
    """the cutoff c.x <= z* - δ is one more row; with it active the scores equal
    those of the same instance with that row appended explicitly."""
    for seed in range(60):
        inst = synth.random_tiny(seed)
        try:
            P = oracle.Problem.from_instance(inst)
        except oracle.OracleError:
            continue
        x = np.clip(synth.random_point_tiny(inst, seed), *exact.bounds(inst))
        z = float(inst.c @ x)
        cut = z - 1.0
        xhat, score, _ = P.best_shift(x, None, cutoff_rhs=cut)
        # explicit row appended
        nzc = np.nonzero(inst.c)[0]
        rp = np.concatenate([inst.row_ptr, [inst.row_ptr[-1] + nzc.size]])
        ci = np.concatenate([inst.col_idx, nzc.astype(np.int32)])
        va = np.concatenate([inst.val, inst.c[nzc]])
        P2 = oracle.Problem(inst.n, inst.m + 1, rp, ci, va, np.concatenate([inst.lhs, [-math.inf]]),
                            np.concatenate([inst.rhs, [cut]]), inst.lb, inst.ub, inst.is_int, inst.c)
        xhat2, score2, _ = P2.best_shift(x, None)
        assert np.array_equal(xhat, xhat2) and np.array_equal(score, score2)


def test_best_shift_range_equals_full_slice():
    """orc_best_shift_range (bench.py's bounded reference sample) is orc_best_shift restricted to
    [j0, j1): same per-variable values, best move = the best within the slice."""
    inst = synth.mixed(seed=5, n=3000, m=600, n_long=2, long_lo=200, long_hi=2000)
    O = oracle.Problem.from_instance(inst)
    x = synth.x_random(inst, 4)
    w = synth.weights_random(O.m_norm, 4)
    fx, fs, _ = O.best_shift(x, w)
    for j0, j1 in [(0, 3000), (100, 900), (2999, 3000), (500, 500)]:
        rx, rs, (bj, bv, bs) = O.best_shift_range(x, j0, j1, w)
        assert np.array_equal(rx[j0:j1], fx[j0:j1]) and np.array_equal(rs[j0:j1], fs[j0:j1])
        pos = [j for j in range(j0, j1) if fs[j] > 0]
        if pos:
            jb = min(pos, key=lambda j: (-fs[j], j))
            assert (bj, bv, bs) == (jb, fx[jb], fs[jb])
        else:
            assert bj == -1
