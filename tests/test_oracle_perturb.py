"""CPU pins of the oracle's perturbation (NEXT f1, R21; "perturb").

The draw H(seed, a, b, c) = g(g(g(g(seed) ^ a) ^ b) ^ c) is built on SplitMix64's output function g,
pinned to the published SplitMix64 test vector. The walk-level pins are SPEC.md's examples
(binary-only instance -> the perturbation flips exactly one bit; the cutoff row is eligible when it
is the only violated row; seeded runs replay byte-identically) and distribution checks of the row
and value draws through whole oracle walks (chi-square against uniform), so a wrong index in the
row/entry/value draw or a dropped exclusion of x̄ fails one of them.
"""
import math

import numpy as np
import pytest

import oracle
from synth import Instance

GAMMA = 0x9E3779B97F4A7C15
M64 = 2**64 - 1


def test_splitmix64_published_vector():
    # SplitMix64 seeded with 1234567 (Vigna's reference splitmix64.c): the n-th output is g applied
    # to the state after n - 1 increments of the golden gamma
    expect = [6457827717110365317, 3203168211198807973, 9817491932198370423, 4593380528125082431,
              16408922859458223821]
    got = [oracle.splitmix64((1234567 + n * GAMMA) & M64) for n in range(5)]
    assert got == expect
    assert oracle.splitmix64(0) == 0xE220A8397B1DCDAF


def test_draw_is_counter_based():
    # every argument enters the draw; equal arguments give equal draws
    base = oracle.draw(7, 3, 11, 5)
    assert base == oracle.draw(7, 3, 11, 5)
    assert len({base, oracle.draw(8, 3, 11, 5), oracle.draw(7, 4, 11, 5), oracle.draw(7, 3, 12, 5),
                oracle.draw(7, 3, 11, 6)}) == 5
    # the top 32 bits of draws over consecutive c are uniform (chi-square, 16 bins, 15 dof)
    h = np.array([oracle.draw(1, 0, 0, c) >> 60 for c in range(8000)])
    cnt = np.bincount(h, minlength=16)
    chi2 = float(((cnt - 500.0) ** 2 / 500.0).sum())
    assert chi2 < 37.7   # p = 0.001


def _inst(name, rows, n, lb, ub, is_int, c=None):
    """rows: list of (cols, vals, lhs, rhs)."""
    rp, ci, va, lhs, rhs = [0], [], [], [], []
    for cols, vals, lo, hi in rows:
        ci += list(cols)
        va += list(vals)
        rp.append(len(ci))
        lhs.append(lo)
        rhs.append(hi)
    return Instance(name=name, n=n, m=len(rows), row_ptr=np.array(rp, np.int64), col_idx=np.array(ci, np.int32),
                    val=np.array(va, np.float64), lhs=np.array(lhs, np.float64), rhs=np.array(rhs, np.float64),
                    lb=np.array(lb, np.float64), ub=np.array(ub, np.float64), is_int=np.array(is_int, np.uint8),
                    c=np.zeros(n) if c is None else np.array(c, np.float64))


def _always_violated(n):
    """n binaries, row i: x_i >= 2 (violated at every point), tenure beyond the walk: after the n
    improving flips every iteration is stuck or a perturbation."""
    return _inst("always_violated", [([i], [1.0], 2.0, math.inf) for i in range(n)], n, [0] * n, [1] * n, [1] * n)


def _replay(inst, log, x0):
    x = np.array(x0, float)
    pts = [x.copy()]
    for rec in log:
        if rec["j"] >= 0:
            x[rec["j"]] = rec["v"]
        pts.append(x.copy())
    return pts


def test_binary_perturbation_flips_exactly_one_bit_uniform_rows():
    n = 10
    inst = _always_violated(n)
    O = oracle.Problem.from_instance(inst)
    prm = oracle.TabuParams(tenure=10**8, perturb=1, rng_seed=12345)
    x0 = np.zeros(n)
    ow = oracle.TabuWalker(O, x0, prm)
    log = ow.run(6000)
    # the first n iterations are the improving flips 0 -> 1
    assert list(log["j"][:n]) == list(range(n)) and not log["flags"][:n].any()
    body = log[n:]
    stuck = body["j"] < 0
    pert = body["flags"] == 1
    # stuck and perturbation alternate: every stuck iteration is followed by a perturbation
    assert stuck[0] and np.array_equal(stuck[0::2], np.ones_like(stuck[0::2])) and pert[1::2].all()
    assert np.isnan(body["s"][pert]).all()
    pts = _replay(inst, log, x0)
    for k in np.nonzero(log["flags"] == 1)[0]:
        d = np.nonzero(pts[k + 1] != pts[k])[0]
        assert d.size == 1 and pts[k + 1][d[0]] == 1.0 - pts[k][d[0]]
    # every row is violated at every stuck iteration: the drawn row (= variable) is uniform
    cnt = np.bincount(body["j"][pert], minlength=n)
    e = cnt.sum() / n
    chi2 = float(((cnt - e) ** 2 / e).sum())
    assert chi2 < 27.9   # 9 dof, p = 0.001


def test_row_draw_is_uniform_over_the_violated_rows_only():
    # 12 binaries; rows 0..5 are x_i >= 2 (always violated), rows 6..11 are x_i <= 1 (never
    # violated): the perturbed variable is always one of 0..5, uniformly
    n = 12
    rows = [([i], [1.0], 2.0, math.inf) for i in range(6)] + [([i], [1.0], -math.inf, 1.0) for i in range(6, 12)]
    inst = _inst("half_violated", rows, n, [0] * n, [1] * n, [1] * n)
    O = oracle.Problem.from_instance(inst)
    ow = oracle.TabuWalker(O, np.zeros(n), oracle.TabuParams(tenure=10**8, perturb=1, rng_seed=99))
    log = ow.run(5000)
    pj = log["j"][log["flags"] == 1]
    assert pj.size > 2000 and pj.max() < 6
    cnt = np.bincount(pj, minlength=6)
    e = cnt.sum() / 6
    assert float(((cnt - e) ** 2 / e).sum()) < 20.5   # 5 dof, p = 0.001


def test_cutoff_row_is_eligible():
    # "no violated rows and cutoff row violated -> cutoff row eligible". Two binaries,
    # no constraint rows besides x_0 + x_1 <= 2 (never violated), c = (1, 1): the start (0, 0) is
    # feasible, the cutoff row c.x <= -1 is then the only violated row and no move can repair it
    # (stuck); the perturbation draws the cutoff row, i.e. a variable with c_j != 0
    inst = _inst("cutoff_only", [([0, 1], [1.0, 1.0], -math.inf, 2.0)], 2, [0, 0], [1, 1], [1, 1], c=[1.0, 1.0])
    O = oracle.Problem.from_instance(inst)
    ow = oracle.TabuWalker(O, np.zeros(2), oracle.TabuParams(tenure=3, perturb=1, rng_seed=5))
    assert ow.has_incumbent and ow.best_obj == 0.0
    log = ow.run(40)
    assert log["j"][0] == -1 and log["flags"][1] == 1
    assert set(log["j"][log["flags"] == 1]) <= {0, 1} and (log["flags"] == 1).sum() > 5


def test_integer_values_uniform_excluding_current():
    # one integer in [0, 4], row x_0 >= 10 (always violated): after the improving move to 4 every
    # perturbation draws uniformly from {0..4} minus the current value
    inst = _inst("int_dom", [([0], [1.0], 10.0, math.inf)], 1, [0], [4], [1])
    O = oracle.Problem.from_instance(inst)
    ow = oracle.TabuWalker(O, np.zeros(1), oracle.TabuParams(tenure=10**8, perturb=1, rng_seed=3))
    log = ow.run(8001)
    pts = _replay(inst, log, np.zeros(1))
    pairs = np.zeros((5, 5), int)
    for k in np.nonzero(log["flags"] == 1)[0]:
        pairs[int(pts[k][0]), int(pts[k + 1][0])] += 1
    assert np.trace(pairs) == 0   # never the current value
    for a in range(5):
        row = np.delete(pairs[a], a)
        if row.sum() < 200:
            continue
        e = row.sum() / 4
        assert float(((row - e) ** 2 / e).sum()) < 16.3   # 3 dof, p = 0.001


def test_unbounded_and_continuous_windows():
    # integer in [0, +inf): values in [0, x̄ + R] minus x̄; continuous in (-inf, +inf): [x̄ - R, x̄ + R]
    R = 5
    # rows x_0 <= -1 and x_1 >= 1, x_1 <= -1: some row of each variable is violated at every point
    inst = _inst("windows", [([0], [1.0], -math.inf, -1.0), ([1], [1.0], 1.0, math.inf), ([1], [1.0], -math.inf, -1.0)],
                 2, [0, -math.inf], [math.inf, math.inf], [1, 0])
    O = oracle.Problem.from_instance(inst)
    ow = oracle.TabuWalker(O, np.zeros(2), oracle.TabuParams(tenure=10**8, perturb=1, perturb_radius=R,
                                                             rng_seed=17))
    log = ow.run(3000)
    pts = _replay(inst, log, np.zeros(2))
    ks = np.nonzero(log["flags"] == 1)[0]
    assert ks.size > 500
    seen_int = seen_cont = 0
    for k in ks:
        j = int(log["j"][k])
        a, b = pts[k][j], pts[k + 1][j]
        if j == 0:
            assert b != a and b == math.floor(b) and 0 <= b <= a + R
            seen_int += 1
        else:
            assert a - R <= b <= a + R
            seen_cont += 1
    assert seen_int > 100 and seen_cont > 100


def test_seeded_replay_and_restart_clears_pending():
    inst = _always_violated(6)
    O = oracle.Problem.from_instance(inst)
    logs = []
    for seed in (1, 1, 2):
        ow = oracle.TabuWalker(O, np.zeros(6), oracle.TabuParams(tenure=10**8, perturb=1, rng_seed=seed))
        logs.append(ow.run(400))
    assert logs[0].tobytes() == logs[1].tobytes()
    assert not np.array_equal(logs[0]["j"], logs[2]["j"])
    # walker ids are draw arguments: two walkers of one set walk differently
    ow2 = oracle.TabuWalker(O, np.zeros(6), oracle.TabuParams(tenure=10**8, perturb=1, rng_seed=1),
                            walker_id=1)
    assert not np.array_equal(ow2.run(400)["j"], logs[0]["j"])
    # a stuck last iteration leaves a pending perturbation; a restart drops it
    ow = oracle.TabuWalker(O, np.zeros(6), oracle.TabuParams(tenure=10**8, perturb=1, rng_seed=1))
    lg = ow.run(7)    # 6 flips, then stuck
    assert lg["j"][6] == -1 and ow.S.force_j >= 0
    ow.restart(np.ones(6))
    assert ow.S.force_j == -1
    assert ow.run(1)["flags"][0] == 0


def test_perturb_off_is_the_plain_walk():
    inst = _always_violated(5)
    O = oracle.Problem.from_instance(inst)
    a = oracle.TabuWalker(O, np.zeros(5), oracle.TabuParams(tenure=10**8)).run(50)
    assert (a["flags"] == 0).all() and (a["j"][5:] == -1).all()


def test_weight_smoothing_rule():
    """R22: every stuck iteration either bumps the violated rows (+1, capped) or, when its draw falls
    below smooth_prob, lowers the satisfied rows with w > 1 by one; never both, nothing else changes;
    the smoothing share is binomial(p); p = 1 never bumps, p = 0 never smooths."""
    # rows: x_0 >= 2 (always violated), x_1 <= 1 (always satisfied), x_0 + x_1 <= 1 (flips)
    n = 2
    rows = [([0], [1.0], 2.0, math.inf), ([1], [1.0], -math.inf, 1.0), ([0, 1], [1.0, 1.0], -math.inf, 1.0)]
    inst = _inst("smooth", rows, n, [0, 0], [1, 1], [1, 1])
    O = oracle.Problem.from_instance(inst)
    for p, lo, hi in ((0.5, 0.4, 0.6), (1.0, 1.0, 1.0), (0.0, 0.0, 0.0)):
        ow = oracle.TabuWalker(O, np.zeros(n), oracle.TabuParams(tenure=2, smooth_prob=p, rng_seed=77, weight_cap=1e6))
        n_smooth = n_bump = 0
        for _ in range(3000):
            w0 = ow.w.copy()
            x0 = ow.x[:n].copy()
            r0 = O.residuals(x0, ow.cutoff_rhs)
            rec = ow.run(1)[0]
            dw = ow.w - w0
            if rec["j"] >= 0:
                assert not dw.any()
                continue
            viol = r0 > 0
            act = np.isfinite(r0)
            bump = np.where(viol & act, 1.0, 0)   # row 0 is always violated: a bump is never empty
            smooth = np.where(~viol & act & (w0 > 1), -1.0, 0)
            if np.array_equal(dw, bump) and bump.any():
                n_bump += 1
            elif np.array_equal(dw, smooth):
                n_smooth += 1
            else:
                raise AssertionError((rec, w0, ow.w, r0))
        assert (ow.w >= 1).all()
        frac = n_smooth / max(1, n_smooth + n_bump)
        assert n_smooth + n_bump > 1000 and lo - 0.05 <= frac <= hi + 0.05, (p, n_smooth, n_bump)
