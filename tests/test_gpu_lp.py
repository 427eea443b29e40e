"""GPU: chap_lp_pdhg (streamed PDHG iterates of the LP relaxation, NEXT f4)
against the plain PDHG oracle (oracle/lp.py) with the same step, chap_lp_round against the oracle's
rounding, and LP-seeded tabu walkers (a start point and a restart from a rounded LP snapshot)
whose trajectories are bit-exact against the oracle walker from the same point."""
import numpy as np
import pytest

import oracle
import synth
from oracle import lp
from tests.test_oracle_lp import _rand_lp

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no GPU", allow_module_level=True)

import paper_2605_05086_b200 as chap  # noqa: E402


@pytest.mark.parametrize("which", ["rand0", "rand3", "T1", "mixed"])
def test_pdhg_snapshots_match_oracle(which):
    """Same step, same restart period: the snapshots at 100 and 1000 iterations agree to 1e-9
    (summation order differs: A^T y by CSC warps on the GPU, by scipy's CSR transpose here)."""
    inst = {"rand0": lambda: _rand_lp(0), "rand3": lambda: _rand_lp(3), "T1": lambda: synth.tiny(1),
            "mixed": lambda: synth.mixed(seed=5, n=3000, m=600, n_long=2, long_lo=200, long_hi=2000)}[which]()
    A = lp.normalized_lp(inst)[0]
    step = 0.9 / lp.operator_norm(A)
    snaps, _ = lp.pdhg(inst, [100, 1000], step)
    P = chap.Problem.from_instance(inst)
    x, info = chap.lp_pdhg(P, [100, 1000], step)
    x = x.cpu().numpy()
    for q, (k, xo, _) in enumerate(snaps):
        assert info[q, 0] == k and info[q, 3] == step
        assert np.abs(x[q] - xo).max() <= 1e-9 * max(1.0, np.abs(xo).max()), (which, k, np.abs(x[q] - xo).max())
        assert abs(info[q, 1] - inst.c @ xo) <= 1e-7 * max(1.0, abs(inst.c @ xo))


def test_pdhg_default_step_converges():
    """step <= 0: 0.9/||A|| from the device's power iteration; on a random LP the 10^4 snapshot is
    optimal to 1e-7 (HiGHS) and the reported violation is ~0."""
    from scipy.optimize import linprog
    inst = _rand_lp(4)
    A, b, c, l, u = lp.normalized_lp(inst)
    ref = linprog(c, A_ub=A.toarray(), b_ub=b, bounds=list(zip(l, u)), method="highs")
    P = chap.Problem.from_instance(inst)
    x, info = chap.lp_pdhg(P, [100, 1000, 10000], 0.0)
    assert abs(info[0, 3] - 0.9 / np.linalg.svd(A.toarray(), compute_uv=False)[0]) <= 1e-3 * info[0, 3]
    assert abs(info[-1, 1] - ref.fun) <= 1e-7 * max(1.0, abs(ref.fun)) and info[-1, 2] <= 1e-7


def test_lp_round_matches_oracle():
    inst = synth.mixed(seed=6, n=4000, m=800, n_long=2, long_lo=200, long_hi=2000, long_kinds=("unb", "cont"))
    P = chap.Problem.from_instance(inst)
    rng = np.random.default_rng(1)
    xin = rng.uniform(-3, 70, inst.n)
    xin[:7] = [0.5, -0.5, 1.5, 2.5, -2.5, 63.5, 1e9]
    g = chap.lp_round(P, torch.from_numpy(xin).cuda()).cpu().numpy()
    assert np.array_equal(g, lp.round_point(inst, xin))


def test_lp_seeded_walkers():
    """LP-seeded start and LP-seeded restart: the rounded 1000-iteration snapshot as x0
    of one walker and as the restart point of another; both trajectories bit-exact vs the oracle."""
    inst = synth.tiny(2)
    P = chap.Problem.from_instance(inst)
    O = oracle.Problem.from_instance(inst)
    xs, _ = chap.lp_pdhg(P, [1000], 0.0)
    x0 = chap.lp_round(P, xs[0].contiguous())
    x0n = x0.cpu().numpy()
    # walker 0 starts from the LP point; walker 1 from x_lower and is restarted from it after 50 steps
    Wk = chap.Walkers(P, torch.stack([x0, torch.from_numpy(synth.x_lower(inst)).cuda()]), chap.default_params())
    log_a = chap.records(Wk.step(50, log=True)).reshape(50, 2)
    Wk.restart(1, x0)
    log_b = chap.records(Wk.step(100, log=True)).reshape(100, 2)
    o0 = oracle.TabuWalker(O, x0n)
    o1 = oracle.TabuWalker(O, synth.x_lower(inst))
    oa0, oa1 = o0.run(50), o1.run(50)
    o1.restart(x0n)
    ob0, ob1 = o0.run(100), o1.run(100)
    for f in ("k", "j", "violated", "obj", "s"):
        assert np.array_equal(log_a[f][:, 0], oa0[f]) and np.array_equal(log_a[f][:, 1], oa1[f]), f
        assert np.array_equal(log_b[f][:, 0], ob0[f]) and np.array_equal(log_b[f][:, 1], ob1[f]), f
