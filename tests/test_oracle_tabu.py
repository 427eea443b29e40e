"""Pins for the oracle's tabu walk (CPU only).

The selection / tenure / weight-bump / cutoff rules are NOT stated by the paper (DESIGN.md
R6, R12-R15: "parity unpinned by the paper"); they are pinned here by the hand-worked
trajectory, by an exact-rational replay of every logged step whose per-variable best shifts are
recomputed with Algorithm 1 (tests/exact.py — a different algorithm from the oracle's), by
invariants, and by the optimum of config T from HiGHS (scipy.optimize.milp).
"""
import json
import math
import os
from fractions import Fraction as F

import numpy as np
import pytest

import oracle
import synth
from tests import exact

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_trajectory_2var_golden():
    g = json.load(open(os.path.join(GOLD, "trajectory_2var.json")))
    inst = exact.rows_from_json(g)
    P = oracle.Problem.from_instance(inst)
    W = oracle.TabuWalker(P, np.array(g["x0"], float), oracle.TabuParams(tenure=g["tenure"]))
    log = W.run(len(g["records"]))
    for rec, exp in zip(log, g["records"]):
        assert rec["k"] == exp["k"] and rec["j"] == exp["j"]
        if exp["j"] >= 0:
            assert rec["v"] == exp["v"]
        else:
            assert math.isnan(rec["v"])
        assert rec["s"] == exp["s"] and rec["violated"] == exp["violated"] and rec["obj"] == exp["obj"]
    assert list(W.w) == g["final_w"]
    assert W.best_obj == g["best_obj"]


def _replay(inst, P, x0, log, params, check_alg1=True):
    """Replay a logged walk in exact arithmetic and check every step."""
    rows = exact.normalized_rows(inst)
    lb, ub = exact.bounds(inst)
    n = inst.n
    x = [F(v) for v in x0]
    w = [F(1)] * (len(rows) + 1)
    tabu = [0] * n
    c = [F(v) for v in inst.c]
    cut = None           # cutoff rhs (Fraction) or None
    best_obj = None
    delta = F(1)         # config T: integral c on integer vars -> auto delta = 1 (R14)

    def resid():
        r = exact.residuals(rows, x)
        if cut is not None:
            r.append(sum(ci * xi for ci, xi in zip(c, x)) - cut)
        return r

    def all_rows():
        rr = list(rows)
        if cut is not None:
            rr.append(({j: c[j] for j in range(n) if c[j] != 0}, cut, -1, 0))
        return rr

    n_asp = [0]          # moves admitted by aspiration
    # k = 0 incumbent check (R15)
    r = resid()
    if all(v <= 0 for v in r):
        best_obj = sum(ci * xi for ci, xi in zip(c, x)); cut = best_obj - delta
    objs = []
    for rec in log:
        k = int(rec["k"])
        rr = all_rows()
        r = resid()
        xf = [float(v) for v in x]
        # admissible argmax by Algorithm 1 in exact arithmetic
        def feasible_after(j, v):   # aspiration (R18): no active row violated after x_j <- v
            keep = x[j]
            x[j] = F(v)
            ok = all(q <= 0 for q in resid())
            x[j] = keep
            return ok

        if check_alg1:
            best = None
            for j in range(n):
                if lb[j] == ub[j]:
                    continue
                v, s = exact.alg1(rr, r, xf, [float(q) for q in w], j, lb[j], ub[j], True)
                s = s if s is not None else -math.inf
                if tabu[j] > k and not (getattr(params, "aspiration", 0) and s > 0 and feasible_after(j, v)):
                    continue
                if best is None or s > best[0]:
                    best = (s, j, v)
            exp_s = best[0] if best else -math.inf
            assert rec["s"] == float(exp_s), k
            if best and best[0] > 0:
                assert rec["j"] == best[1] and rec["v"] == float(best[2]), k
            else:
                assert rec["j"] == -1, k
        if rec["j"] >= 0:
            j, v = int(rec["j"]), F(rec["v"])
            if tabu[j] > k:                         # admissible only by aspiration (R18)
                assert getattr(params, "aspiration", 0) and feasible_after(j, v), k
                n_asp[0] += 1
            assert lb[j] <= v <= ub[j] and v != x[j] and v.denominator == 1
            # chosen score == recomputed sum of penalties (north star invariant)
            s = exact.score(rr, r, xf, [float(q) for q in w], j, v)
            assert float(s) == rec["s"] and s > 0
            x[j] = v
            tabu[j] = k + 1 + params.tenure
        else:
            for i, ri in enumerate(r):
                if ri > 0:
                    w[i] = min(w[i] + 1, F(params.weight_cap))
        r = resid()
        if all(v <= 0 for v in r):
            z = sum(ci * xi for ci, xi in zip(c, x))
            assert best_obj is None or z < best_obj    # strictly improving incumbents
            best_obj = z; cut = z - delta
            r = resid()
        assert rec["violated"] == sum(1 for v in r if v > 0)
        assert rec["obj"] == float(sum(ci * xi for ci, xi in zip(c, x)))
        assert all(1 <= q <= params.weight_cap for q in w)
        objs.append(best_obj)
    _replay.n_asp = n_asp[0]
    return best_obj


@pytest.mark.parametrize("seed", range(6))
def test_tabu_replay_config_T(seed):
    inst = synth.tiny(seed)
    P = oracle.Problem.from_instance(inst)
    prm = oracle.TabuParams(tenure=10)
    x0 = synth.x_lower(inst)
    W = oracle.TabuWalker(P, x0, prm)
    log = W.run(150)
    best = _replay(inst, P, x0, log, prm)
    assert (best is None and not W.has_incumbent) or float(best) == W.best_obj


def test_tabu_determinism_and_resume():
    inst = synth.tiny(7)
    P = oracle.Problem.from_instance(inst)
    x0 = synth.x_lower(inst)
    a = oracle.TabuWalker(P, x0).run(400)
    b = oracle.TabuWalker(P, x0).run(400)
    assert a.tobytes() == b.tobytes()
    W = oracle.TabuWalker(P, x0)
    c = np.concatenate([W.run(150), W.run(250)])
    assert a.tobytes() == c.tobytes()


def test_tabu_never_beats_highs_optimum():
    """Quality check on config T (not parity): incumbents are feasible, so the best found can
    never be below the MIP optimum computed by HiGHS."""
    from scipy.optimize import LinearConstraint, Bounds, milp
    from scipy.sparse import csr_matrix
    found = 0
    for seed in range(8):
        inst = synth.tiny(seed)
        A = csr_matrix((inst.val, inst.col_idx, inst.row_ptr), shape=(inst.m, inst.n))
        res = milp(inst.c, constraints=LinearConstraint(A, inst.lhs, inst.rhs), integrality=inst.is_int,
                   bounds=Bounds(inst.lb, inst.ub))
        assert res.status == 0
        P = oracle.Problem.from_instance(inst)
        W = oracle.TabuWalker(P, synth.x_lower(inst))
        W.run(2000)
        if W.has_incumbent:
            found += 1
            assert W.best_obj >= res.fun - 1e-9
            # the incumbent is feasible (exact check)
            rows = exact.normalized_rows(inst)
            assert all(v <= 0 for v in exact.residuals(rows, list(W.best_x)))
            assert float(inst.c @ W.best_x) == W.best_obj
    assert found >= 6


def _check_records(log, exp_records):
    for rec, exp in zip(log, exp_records):
        assert rec["k"] == exp["k"] and rec["j"] == exp["j"], (rec, exp)
        if exp["j"] >= 0:
            assert rec["v"] == exp["v"]
        else:
            assert math.isnan(rec["v"])
        s = -math.inf if exp["s"] == "-inf" else exp["s"]
        assert rec["s"] == s and rec["violated"] == exp["violated"] and rec["obj"] == exp["obj"], (rec, exp)


def test_trajectory_2var_weight_cap_golden():
    """The weight-cap clamp w <- min(w + 1, cap) (R12): a hand-worked 16-step trajectory with cap 3
    in which the cutoff row's weight (k = 3) and then the row's weight (k = 14) reach the cap."""
    g = json.load(open(os.path.join(GOLD, "trajectory_2var_cap3.json")))
    inst = exact.rows_from_json(g)
    P = oracle.Problem.from_instance(inst)
    W = oracle.TabuWalker(P, np.array(g["x0"], float),
                          oracle.TabuParams(tenure=g["tenure"], weight_cap=g["weight_cap"]))
    recs = g["records"]
    log = W.run(4)
    _check_records(log, recs[:4])
    assert list(W.w) == [1.0, 3.0]          # cutoff weight at the cap after k = 3
    log = np.concatenate([log, W.run(len(recs) - 4)])
    _check_records(log, recs)
    assert list(W.w) == g["final_w"] and W.best_obj == g["best_obj"]


def test_cutoff_delta_fractional_objective_golden():
    """The non-integral cutoff delta (R14): 1e-6 * max(1, |z|), both branches of the max (z = 0 at
    the start, z = -2.5 after the first move), hand-derived."""
    g = json.load(open(os.path.join(GOLD, "cutoff_delta_fractional.json")))
    inst = exact.rows_from_json(g)
    P = oracle.Problem.from_instance(inst)
    assert math.isnan(P.auto_delta)
    W = oracle.TabuWalker(P, np.array(g["x0"], float), oracle.TabuParams(tenure=g["tenure"]))
    st = g["steps"]
    assert W.has_incumbent and W.best_obj == 0.0
    assert abs(W.cutoff_rhs - st[0]["cutoff_rhs"]) <= 1e-15
    for exp in st[1:]:
        rec = W.run(1)[0]
        _check_records([rec], [dict(exp, k=int(exp["after"][2:]))])
        assert abs(W.cutoff_rhs - exp["cutoff_rhs"]) <= 1e-15 * abs(exp["cutoff_rhs"])
        if "w_cut" in exp:
            assert W.w[-1] == exp["w_cut"]
    assert W.best_obj == -2.5


def test_summary_and_restart_golden():
    """orc_walker_summary / orc_walker_restart against hand-derived values: violated counts (cutoff
    included), the violation sum over non-cutoff rows, and the incumbent taken by a restart to a
    feasible point; the restart keeps the weights and k and clears the tabu list."""
    g = json.load(open(os.path.join(GOLD, "summary_restart.json")))
    inst = exact.rows_from_json(g)
    P = oracle.Problem.from_instance(inst)
    W = oracle.TabuWalker(P, np.array(g["x0"], float), oracle.TabuParams(tenure=g["tenure"]))
    for exp in g["steps"]:
        if exp["op"] == "restart":
            w_before, k_before = W.w.copy(), W.k
            W.tabu_until[:] = 7
            W.restart(np.array(exp["x"], float))
            assert np.array_equal(W.w, w_before) and W.k == k_before
            assert not W.tabu_until[: inst.n].any()
        assert W.summary() == (exp["violated"], exp["sumviol"]), exp
        assert W.has_incumbent == bool(exp["has_incumbent"])
        if exp["has_incumbent"]:
            assert W.best_obj == exp["best_obj"] and W.cutoff_rhs == exp["cutoff_rhs"]


@pytest.mark.parametrize("seed", range(6))
def test_tabu_replay_aspiration(seed):
    """NEXT f1, R18 (incumbent aspiration): every logged step of an oracle walk with aspiration on is
    recomputed in exact arithmetic — Algorithm 1 for every variable, tabu variables admitted only
    when the exact residuals after their move leave no active row violated — and the walk takes
    aspiration moves (config T, tenure 10)."""
    inst = synth.tiny(seed)
    P = oracle.Problem.from_instance(inst)
    prm = oracle.TabuParams(tenure=10, aspiration=1)
    x0 = synth.x_lower(inst)
    W = oracle.TabuWalker(P, x0, prm)
    log = W.run(120)
    best = _replay(inst, P, x0, log, prm)
    assert (best is None and not W.has_incumbent) or float(best) == W.best_obj
    assert _replay.n_asp > 0, "no aspiration move in this walk"
