"""Pins for the LP oracle (oracle/lp.py: restarted PDHG whose streamed iterates seed tabu walkers,
NEXT f4; CPU only): a 1-D LP with a known optimum, the operator norm against a
dense SVD, random feasible LPs against HiGHS (scipy.optimize.linprog, exact simplex optimum), the
normalisation against the C oracle's row count, and the rounding of LP points."""
import math

import numpy as np
from scipy.optimize import linprog

import oracle
import synth
from oracle import lp


def _inst(n, m, A, lhs, rhs, lb, ub, c, is_int=None):
    rows, cols = np.nonzero(A)
    rp = np.searchsorted(rows, np.arange(m + 1)).astype(np.int64)
    return synth.Instance("lp", n, m, rp, cols.astype(np.int32), A[rows, cols].astype(float), np.asarray(lhs, float),
                          np.asarray(rhs, float), np.asarray(lb, float), np.asarray(ub, float),
                          np.zeros(n, np.uint8) if is_int is None else np.asarray(is_int, np.uint8), np.asarray(c, float))


def _rand_lp(seed, n=12, m=10):
    rng = np.random.default_rng([0x1F, seed])
    A = rng.integers(-5, 6, (m, n)).astype(float)
    A[rng.random((m, n)) < 0.5] = 0
    xs = rng.uniform(0, 5, n)
    rhs = A @ xs + rng.uniform(0, 3, m)   # x* is strictly feasible
    return _inst(n, m, A, np.full(m, -np.inf), rhs, np.zeros(n), np.full(n, 5.0), rng.integers(-10, 11, n))


def test_one_dimensional_lp():
    """min x s.t. x >= 1, x in [0, 10]: the snapshots converge to x = 1 (SPEC.md:345 example)."""
    inst = _inst(1, 1, np.array([[1.0]]), [1.0], [np.inf], [0.0], [10.0], [1.0])
    A, b, c, l, u = lp.normalized_lp(inst)
    assert A.shape == (1, 1) and A[0, 0] == -1.0 and b[0] == -1.0   # the lower side as a <= row
    snaps, _ = lp.pdhg(inst, [100, 1000, 10000], 0.9 / lp.operator_norm(A))
    assert [k for k, _, _ in snaps] == [100, 1000, 10000]
    assert abs(snaps[-1][1][0] - 1.0) <= 1e-4 and abs(snaps[1][1][0] - 1.0) <= 1e-4


def test_operator_norm_matches_svd():
    rng = np.random.default_rng(5)
    for _ in range(5):
        inst = _rand_lp(int(rng.integers(1000)))
        A = lp.normalized_lp(inst)[0]
        s = np.linalg.svd(A.toarray(), compute_uv=False)[0]
        assert abs(lp.operator_norm(A) - s) <= 1e-2 * s


def test_random_lps_against_highs():
    """10 random feasible LPs: after 10^4 iterations the streamed average is optimal to 1e-9 relative
    (objective against HiGHS' simplex optimum) and feasible to 1e-9."""
    for seed in range(10):
        inst = _rand_lp(seed)
        A, b, c, l, u = lp.normalized_lp(inst)
        ref = linprog(c, A_ub=A.toarray(), b_ub=b, bounds=list(zip(l, u)), method="highs")
        assert ref.status == 0
        snaps, _ = lp.pdhg(inst, [10000], 0.9 / lp.operator_norm(A))
        x = snaps[-1][1]
        assert abs(c @ x - ref.fun) <= 1e-9 * max(1.0, abs(ref.fun)), seed
        assert (A @ x - b).max() <= 1e-9 and (x >= l).all() and (x <= u).all()


def test_normalisation_row_count_matches_c_oracle():
    """oracle/lp.py and oracle/chap_oracle.c normalise independently: same rows."""
    for seed in range(3):
        inst = synth.tiny(seed)
        A, b, _, _, _ = lp.normalized_lp(inst)
        assert A.shape[0] == oracle.Problem.from_instance(inst).m_norm - 1   # the C oracle adds the cutoff row


def test_round_point():
    inst = _inst(4, 1, np.ones((1, 4)), [-np.inf], [10.0], [0, -5, 0, 0], [3, 5, 3.7, 9], [0, 0, 0, 0], [1, 1, 1, 0])
    x = lp.round_point(inst, np.array([2.5, -2.5, 3.6, 1.25]))
    assert list(x) == [3.0, -3.0, 3.0, 1.25]   # half away from zero; u = 3.7 rounds inward to 3; continuous kept
