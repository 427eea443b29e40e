"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Bit-exact on every per-variable (x̂_j, s_j), on the chosen move and on whole tabu trajectories,
in the exact domain (integer data and weights) that every synthetic config uses.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
import synth
from tests import exact

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no GPU", allow_module_level=True)

import paper_2605_05086_b200 as chap  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _eval_both(inst, x, w=None, cutoff=math.inf, P=None, O=None):
    P = P or chap.Problem.from_instance(inst)
    O = O or oracle.Problem.from_instance(inst)
    xt = torch.from_numpy(np.ascontiguousarray(x, np.float64)).cuda()
    wt = None if w is None else torch.from_numpy(np.ascontiguousarray(w, np.float32)).cuda()
    xhat, score, best = P.eval_best_shift(xt, wt, cutoff)
    torch.cuda.synchronize()
    oxhat, oscore, obest = O.best_shift(x, w, cutoff)
    return (xhat.cpu().numpy(), score.cpu().numpy(), chap.move_from_bytes(best)), (oxhat, oscore, obest)


def _assert_same(g, o, tag=""):
    gx, gs, gm = g
    ox, os_, ob = o
    bad = np.nonzero((gx != ox) | (gs != os_))[0]
    assert bad.size == 0, f"{tag}: {bad.size} vars differ, first {bad[:5]}: gpu {gx[bad[:5]]} {gs[bad[:5]]} " \
                          f"oracle {ox[bad[:5]]} {os_[bad[:5]]}"
    assert gm["j"] == ob[0], (tag, gm, ob)
    if ob[0] >= 0:
        assert gm["v"] == ob[1] and gm["s"] == ob[2], (tag, gm, ob)


@pytest.mark.parametrize("case", json.load(open(os.path.join(GOLD, "alg1_worked.json")))["cases"],
                         ids=lambda c: c["name"])
def test_worked_cases(case):
    inst = exact.rows_from_json(case)
    g, o = _eval_both(inst, np.array(case["x"], float))
    _assert_same(g, o, case["name"])
    assert list(g[0]) == case["xhat"]


def test_random_tiny_instances():
    n_ok = 0
    for seed in range(400):
        kw = [{}, {"p_inf_bound": 0.3}, {"coef": 6, "bound": 9}, {"p_binary": 0.8}][seed % 4]
        inst = synth.random_tiny(seed, **kw)
        try:
            O = oracle.Problem.from_instance(inst)
        except oracle.OracleError:
            continue
        P = chap.Problem.from_instance(inst)
        lb, ub = exact.bounds(inst)
        x = np.clip(synth.random_point_tiny(inst, seed), lb, ub)
        w = np.random.default_rng(seed).integers(0, 5, P.m_norm).astype(np.float32)
        cut = math.inf if seed % 3 else float(inst.c @ x) - 1.0
        g, o = _eval_both(inst, x, w, cut, P, O)
        _assert_same(g, o, inst.name)
        n_ok += 1
    assert n_ok > 250


@pytest.mark.parametrize("seed", range(10))
def test_config_T(seed):
    inst = synth.tiny(seed)
    x = synth.x_random(inst, seed)
    P = chap.Problem.from_instance(inst)
    w = synth.weights_random(P.m_norm, seed)
    g, o = _eval_both(inst, x, w, P=P)
    _assert_same(g, o, inst.name)


def _mixed_small(seed=5):
    # spans every column class: short binary/general (warp), medium (block), long chunked
    return synth.mixed(seed=seed, n=20_000, m=4_000, n_long=8, long_lo=600, long_hi=12_000)


def test_all_column_classes():
    inst = _mixed_small()
    P = chap.Problem.from_instance(inst)
    assert P.info.n_long_columns >= 2
    for s in range(3):
        x = synth.x_random(inst, s)
        w = synth.weights_random(P.m_norm, s, hi=7)
        cut = math.inf if s == 0 else float(inst.c @ x) - 50.0
        g, o = _eval_both(inst, x, w, cut, P=P)
        _assert_same(g, o, f"mixed s={s}")


def test_config_S_full():
    inst = synth.setcover()
    x = synth.x_bernoulli(inst, (1, 0), 0.05)
    g, o = _eval_both(inst, x)
    _assert_same(g, o, "S")


@pytest.fixture(scope="module")
def config_G():
    """BASELINE configs[2] at full size (10.4 M nonzeros), the instance bench.py times."""
    inst = synth.mixed()
    return inst, chap.Problem.from_instance(inst), oracle.Problem.from_instance(inst)


def test_config_G_full_eval(config_G):
    """Every variable of the 10^7-nonzero instance, bench.py's launch configuration (one walker's
    eval grid), at the start point and at a random point with random weights and an active cutoff."""
    inst, P, O = config_G
    x = synth.x_lower(inst)
    g, o = _eval_both(inst, x, P=P, O=O)
    _assert_same(g, o, "G x_lower")
    x = synth.x_random(inst, 3)
    w = synth.weights_random(P.m_norm, 3, hi=9)
    cut = float(inst.c @ x) - 1000.0
    g, o = _eval_both(inst, x, w, cut, P=P, O=O)
    _assert_same(g, o, "G random")


def test_config_G_full_trajectory(config_G):
    """40 tabu iterations on the full instance with bench.py's parameters (one CUDA graph of 32
    iterations + 8 plain launches): every record, the final point, weights and residuals; then the
    eval at the walker's final state."""
    inst, P, O = config_G
    x0 = synth.x_lower(inst)
    prm = chap.default_params(graph_iters=32)
    Wk = chap.Walkers(P, torch.from_numpy(x0[None, :]).cuda(), prm)
    log = chap.records(Wk.step(40, log=True)).reshape(40, 1)[:, 0]
    st = Wk.get()
    ow = oracle.TabuWalker(O, x0)
    olog = ow.run(40)
    for f in ("k", "j", "violated", "obj", "s"):
        bad = np.nonzero(log[f] != olog[f])[0]
        assert bad.size == 0, (f, bad[:3], log[bad[:3]], olog[bad[:3]])
    assert np.array_equal(st["x"][0], ow.x[: inst.n])
    assert np.array_equal(st["w"][0], ow.w)
    assert np.array_equal(st["r"][0], O.residuals(st["x"][0], ow.cutoff_rhs))
    g, o = _eval_both(inst, st["x"][0], st["w"][0], ow.cutoff_rhs, P=P, O=O)
    _assert_same(g, o, "G after 40 iterations")


def test_config_P_full_eval():
    """BASELINE configs[3]'s packing instance (10^6 nonzeros) at a walker start point."""
    inst = synth.packing()
    P = chap.Problem.from_instance(inst)
    x = synth.x_bernoulli(inst, (3, 7), 0.5)
    w = synth.weights_random(P.m_norm, 5, hi=12)
    g, o = _eval_both(inst, x, w, float(inst.c @ x) - 10.0, P=P)
    _assert_same(g, o, "P")


def test_config_X_largest_eval():
    """The top of BASELINE configs[4]'s scaling sweep: generator X at 5·10^7 requested nonzeros
    (46 M nonzeros, 5 M variables, 10^6 rows), every variable at two points."""
    inst = synth.scaled(50_000_000)
    P = chap.Problem.from_instance(inst)
    O = oracle.Problem.from_instance(inst)
    g, o = _eval_both(inst, synth.x_lower(inst), P=P, O=O)
    _assert_same(g, o, "X50M x_lower")
    x = synth.x_random(inst, 8)
    w = synth.weights_random(P.m_norm, 8, hi=6)
    g, o = _eval_both(inst, x, w, float(inst.c @ x) - 100.0, P=P, O=O)
    _assert_same(g, o, "X50M random")


def test_host_buffer_variant_equals_device():
    inst = _mixed_small(6)
    P = chap.Problem.from_instance(inst)
    x = synth.x_random(inst, 2)
    w = synth.weights_random(P.m_norm, 2)
    xh, sh, mh = P.eval_best_shift_host(x, w)
    xd, sd, md = P.eval_best_shift(torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda())
    torch.cuda.synchronize()
    assert np.array_equal(xh, xd.cpu().numpy()) and np.array_equal(sh, sd.cpu().numpy())
    assert mh.tobytes() == chap.move_from_bytes(md).tobytes()


def _traj_compare(inst, x0s, n_iters, params=None, graph_iters=16, weight_cap=1e6, tenure=10, binary_kernel=0,
                  aspiration=0, lazy=0, perturb=0, rng_seed=0, perturb_radius=16, smooth_prob=0.0, split=None):
    P = chap.Problem.from_instance(inst)
    O = oracle.Problem.from_instance(inst)
    prm = chap.default_params(graph_iters=graph_iters, weight_cap=weight_cap, tenure=tenure,
                              binary_kernel=binary_kernel, aspiration=aspiration, lazy=lazy, perturb=perturb,
                              rng_seed=rng_seed, perturb_radius=perturb_radius, smooth_prob=smooth_prob)
    oprm = oracle.TabuParams(tenure=tenure, weight_cap=weight_cap, aspiration=aspiration, perturb=perturb,
                             rng_seed=rng_seed, perturb_radius=perturb_radius, smooth_prob=smooth_prob)
    X0 = torch.from_numpy(np.ascontiguousarray(np.stack(x0s), np.float64)).cuda()
    Wk = chap.Walkers(P, X0, prm)
    if split is None:   # one chap_tabu_step call
        log = chap.records(Wk.step(n_iters, log=True)).reshape(n_iters, len(x0s))
    else:               # several calls (state such as a pending perturbation crosses them)
        parts = [chap.records(Wk.step(q, log=True)).reshape(q, len(x0s)) for q in split]
        log = np.concatenate(parts)
        assert sum(split) == n_iters
    st = Wk.get()
    for wi, x0 in enumerate(x0s):
        ow = oracle.TabuWalker(O, x0, oprm, walker_id=wi)
        olog = ow.run(n_iters)
        glog = log[:, wi]
        for f in ("k", "j", "flags", "violated", "obj", "s"):
            ne = ~((glog[f] == olog[f]) | (np.isnan(glog[f]) & np.isnan(olog[f]))) if f == "s" else glog[f] != olog[f]
            bad = np.nonzero(ne)[0]
            assert bad.size == 0, (inst.name, wi, f, bad[:3], glog[bad[:3]], olog[bad[:3]])
        mv = glog["j"] >= 0
        assert np.array_equal(glog["v"][mv], olog["v"][mv])
        assert np.array_equal(st["x"][wi], ow.x[: inst.n])
        assert np.array_equal(st["w"][wi], ow.w)
        assert np.array_equal(st["tabu_until"][wi], ow.tabu_until[: inst.n])
        assert st["stats"][wi]["has_incumbent"] == int(ow.has_incumbent)
        if ow.has_incumbent:
            assert st["stats"][wi]["best_obj"] == ow.best_obj
            assert np.array_equal(st["best_x"][wi], ow.best_x[: inst.n])
        # residual invariant: r == A x - b (exact domain)
        r = O.residuals(st["x"][wi], ow.cutoff_rhs)
        assert np.array_equal(st["r"][wi], r)
    return log


@pytest.fixture(params=[0, 2, 1], ids=["binrow_auto", "binrow_forced", "colwise_forced"])
def binrow(request):
    """chap_params.binary_kernel: 0 = the size rule (chap.cu), 2 = the row-wise kernel forced on
    small instances, 1 = the column-wise kernel forced."""
    return request.param


@pytest.mark.parametrize("seed", range(8))
def test_trajectory_config_T(seed, binrow):
    inst = synth.tiny(seed)
    _traj_compare(inst, [synth.x_lower(inst)], 600, graph_iters=16 if seed % 2 else 0, binary_kernel=binrow)


def test_trajectory_multi_walker():
    inst = synth.tiny(3)
    x0s = [synth.x_lower(inst)] + [np.clip(synth.x_random(inst, s), inst.lb, inst.ub) for s in range(5)]
    _traj_compare(inst, x0s, 300)


def test_trajectory_mixed_small(binrow):
    inst = synth.mixed(seed=9, n=4000, m=800, n_long=4, long_lo=300, long_hi=6000)
    _traj_compare(inst, [synth.x_lower(inst), synth.x_random(inst, 1)], 60, binary_kernel=binrow)


def test_trajectory_setcover_small(binrow):
    inst = synth.setcover(seed=4, m=500, n=2500)
    _traj_compare(inst, [synth.x_lower(inst)], 400, binary_kernel=binrow)


@pytest.mark.parametrize("W", [3, 17, 33])
def test_trajectory_walker_groups_packing(W):
    """Walker-minor row-state groups (rg = 4, 32, 32 + a 1-walker group): every walker's
    trajectory equals its own oracle run (k_eval_bin_wm, the group bitset, strided apply)."""
    inst = synth.packing(seed=5, n=3000, m=600)
    x0s = [synth.x_bernoulli(inst, (3, wi), 0.5) for wi in range(W)]
    _traj_compare(inst, x0s, 120)


def test_trajectory_walker_groups_mixed():
    """40 walkers (groups of 32 + 8) on a mixed instance with long binary and long bounded-integer
    columns: binary columns by k_eval_bin_wm, general columns by the strided general kernels."""
    inst = synth.mixed(seed=9, n=4000, m=800, n_long=4, long_lo=300, long_hi=6000)
    x0s = [synth.x_lower(inst)] + [synth.x_random(inst, s) for s in range(39)]
    _traj_compare(inst, x0s, 40)


def test_config_P_64_walkers_trajectory():
    """BASELINE configs[3] in bench.py's launch configuration: 64 walkers on the 10^6-nonzero
    packing instance (two walker-minor groups of 32), 12 iterations of every walker vs the oracle."""
    inst = synth.packing()
    x0s = [synth.x_bernoulli(inst, (3, wi), 0.5) for wi in range(64)]
    _traj_compare(inst, x0s, 12)


@pytest.mark.parametrize("cap", [3.0, 3.5])
def test_trajectory_weight_cap(cap, binrow):
    """Weights reach the cap: an integral cap keeps the row-wise binary kernel (k_eval_binrow), a
    fractional one (weights 3.5, half-integral penalties) takes the column-wise kernel."""
    inst = synth.setcover(seed=6, m=400, n=2000)
    _traj_compare(inst, [synth.x_lower(inst)], 300, weight_cap=cap, tenure=3, binary_kernel=binrow)


def test_trajectory_rowwise_two_rounds():
    """Generator X at 2·10^7 requested nonzeros: ~1.4 M packed binary columns, more than one round
    of k_eval_binrow blocks per cluster (forced on); 6 iterations of one walker vs the oracle."""
    inst = synth.scaled(20_000_000)
    _traj_compare(inst, [synth.x_lower(inst)], 6, binary_kernel=2)


def test_invalid_x0_rejected():
    inst = synth.tiny(0)
    P = chap.Problem.from_instance(inst)
    x0 = synth.x_lower(inst)
    x0[31] = 0.5   # fractional on an integer variable
    with pytest.raises(chap.ChapError) as e:
        chap.Walkers(P, torch.from_numpy(x0[None, :]).cuda())
    assert e.value.status == 1


def test_single_walker_restart_matches_oracle(binrow):
    """One walker (row-wise binary kernel forced or by the size rule): 60 iterations, a restart from
    another point (residuals recomputed, weights kept, tabu cleared; the bitset incumbent rebuilt),
    60 more; the trajectory and final state equal the oracle's same sequence."""
    inst = synth.setcover(seed=8, m=500, n=2500)
    P = chap.Problem.from_instance(inst)
    O = oracle.Problem.from_instance(inst)
    x0 = synth.x_lower(inst)
    x1 = synth.x_bernoulli(inst, (8, 1), 0.3)
    Wk = chap.Walkers(P, torch.from_numpy(x0[None, :]).cuda(),
                      chap.default_params(graph_iters=16, binary_kernel=binrow))
    ow = oracle.TabuWalker(O, x0)
    for step in range(2):
        log = chap.records(Wk.step(60, log=True))
        olog = ow.run(60)
        for f in ("k", "j", "violated", "obj", "s"):
            assert np.array_equal(log[f], olog[f]), (step, f)
        if step == 0:
            Wk.restart(0, torch.from_numpy(x1).cuda())
            ow.restart(x1)
    st = Wk.get()
    assert np.array_equal(st["x"][0], ow.x[: inst.n])
    assert np.array_equal(st["w"][0], ow.w)
    assert np.array_equal(st["r"][0], O.residuals(st["x"][0], ow.cutoff_rhs))


def test_continuous_columns_tolerance_mode():
    """Continuous variables (SURVEY 8(c) tolerance mode, NEXT row f4). The oracle's recomputed
    activities carry an ulp of error exactly at a tight breakpoint, which can flip "satisfied" and
    move its score by a whole weight ("continuous variables are bit-exact-
    incompatible"), so the reference here is Algorithm 1 itself in exact rational arithmetic
    (tests/exact.alg1) on the same double inputs: on random tiny instances with 40 % continuous
    variables at fractional points, every per-variable score is within 1e-9 relative of it and the
    chosen value within 1e-9 relative of its x̂."""
    from fractions import Fraction as Fr
    n_ok = n_cmp = 0
    for seed in range(200):
        inst = synth.random_tiny(seed, p_cont=0.4, p_inf_bound=0.2 if seed % 2 else 0.0)
        try:
            oracle.Problem.from_instance(inst)   # feasible bounds
        except oracle.OracleError:
            continue
        P = chap.Problem.from_instance(inst)
        lb, ub = exact.bounds(inst)
        rng = np.random.default_rng([0xC0, seed])
        x = synth.random_point_tiny(inst, seed).astype(np.float64)
        cont = inst.is_int == 0
        x[cont] = x[cont] + rng.uniform(-0.5, 0.5, int(cont.sum()))
        x = np.clip(x, lb, ub)
        w = rng.integers(0, 5, P.m_norm).astype(np.float32)
        cut = math.inf if seed % 3 else float(inst.c @ x) - 0.75
        rows = exact.normalized_rows(inst)
        if math.isfinite(cut):
            rows.append(({j: Fr(float(inst.c[j])) for j in range(inst.n) if inst.c[j] != 0}, Fr(cut), -1, +1))
        else:
            rows.append(({}, Fr(0), -1, +1))   # the inactive cutoff row (no entries)
        assert len(rows) == P.m_norm
        r = exact.residuals(rows, x)
        xt = torch.from_numpy(x).cuda()
        gx, gs, _ = P.eval_best_shift(xt, torch.from_numpy(w).cuda(), cut)
        torch.cuda.synchronize()
        gx, gs = gx.cpu().numpy(), gs.cpu().numpy()
        for j in range(inst.n):
            if lb[j] == ub[j]:
                continue
            v, sc = exact.alg1(rows, r, x, w, j, lb[j], ub[j], bool(inst.is_int[j]))
            if sc is None:
                assert gs[j] == -math.inf, (inst.name, j)
                continue
            sc = float(sc)
            assert abs(gs[j] - sc) <= 1e-9 * max(1.0, abs(sc)), (inst.name, j, gs[j], sc)
            assert abs(gx[j] - float(v)) <= 1e-9 * max(1.0, abs(float(v))), (inst.name, j, gx[j], float(v))
            n_cmp += 1
        n_ok += 1
    assert n_ok > 100 and n_cmp > 200


def _sorted_mix(seed=7, kinds=("unb", "big", "bkt", "bin"), n_long=16, hi=2000):
    """Long general columns that are neither binary nor a bounded domain of <= 4096 values:
    unbounded integers [0, inf) and large-domain integers [0, 10000] with 100..2000 nonzeros
    (the sorted class), beside long binary and bounded-integer columns."""
    return synth.mixed(seed=seed, n=20_000, m=4_000, n_long=n_long, long_lo=100, long_hi=hi, long_kinds=kinds)


def test_sorted_columns_eval():
    inst = _sorted_mix()
    P = chap.Problem.from_instance(inst)
    assert P.info.n_sorted_columns >= 6, P.info.n_sorted_columns
    for s in range(4):
        x = synth.x_random(inst, 20 + s, spread=40)
        w = synth.weights_random(P.m_norm, s, hi=7)
        cut = math.inf if s == 0 else float(inst.c @ x) - 50.0
        g, o = _eval_both(inst, x, w, cut, P=P)
        _assert_same(g, o, f"sorted s={s}")


def test_sorted_columns_trajectory(binrow):
    inst = _sorted_mix(seed=8)
    assert chap.Problem.from_instance(inst).info.n_sorted_columns >= 6
    _traj_compare(inst, [synth.x_lower(inst), synth.x_random(inst, 3, spread=30)], 80, binary_kernel=binrow)


def test_sorted_continuous_columns_tolerance_mode():
    """Long continuous columns (sorted class) in tolerance mode: each long continuous column and a
    sample of the others against Algorithm 1 in exact rational arithmetic (tests/exact.alg1) on the
    same double inputs, scores and values within 1e-9 relative."""
    inst = _sorted_mix(seed=9, kinds=("cont", "unb"), n_long=8)
    P = chap.Problem.from_instance(inst)
    assert P.info.n_sorted_columns >= 4 and P.info.n_continuous >= 4
    x = synth.x_random(inst, 5, spread=20)
    w = synth.weights_random(P.m_norm, 5, hi=5)
    cut = float(inst.c @ x) - 20.0
    gx, gs, _ = P.eval_best_shift(torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda(), cut)
    torch.cuda.synchronize()
    gx, gs = gx.cpu().numpy(), gs.cpu().numpy()
    from fractions import Fraction as Fr
    rows = exact.normalized_rows(inst)
    rows.append(({j: Fr(float(inst.c[j])) for j in range(inst.n) if inst.c[j] != 0}, Fr(cut), -1, +1))
    assert len(rows) == P.m_norm
    lb, ub = exact.bounds(inst)
    deg = np.bincount(inst.col_idx, minlength=inst.n)
    long_cols = np.nonzero(deg > 62)[0]
    rng = np.random.default_rng(0)
    sample = np.concatenate([long_cols, rng.choice(inst.n, 150, replace=False)])
    cols = {j: [] for j in sample}
    for i, (a, _, _, _) in enumerate(rows):
        for j in a:
            if j in cols:
                cols[j].append(i)
    r = exact.residuals(rows, x)
    n_cols = n_amb = 0
    for j in sample:
        if lb[j] == ub[j]:
            continue
        sub = [rows[i] for i in cols[j]]
        v, sc = exact.alg1(sub, [r[i] for i in cols[j]], x, w[cols[j]], j, lb[j], ub[j], bool(inst.is_int[j]))
        if sc is None:
            assert gs[j] == -math.inf, j
            continue
        n_cols += 1
        # a column whose result hinges on a residual within rounding of 0 (here typically
        # the cutoff row, c.x - cut nearly 0 after the move) is outside the tolerance contract
        if exact.rounding_ambiguous(rows, r, x, j, cols[j], (v, gx[j]), bool(inst.is_int[j]), lb[j], ub[j]):
            n_amb += 1
            continue
        assert abs(gs[j] - float(sc)) <= 1e-9 * max(1.0, abs(float(sc))), (j, gs[j], float(sc))
        assert abs(gx[j] - float(v)) <= 1e-9 * max(1.0, abs(float(v))), (j, gx[j], float(v))
    assert n_cols > 100 and n_amb <= 0.1 * n_cols, (n_cols, n_amb)


def test_eval_rejects_negative_weights_and_bad_x():
    """chap_eval_best_shift returns CHAP_ERR_INVALID_ARG for w < 0 (negative weights
    break Algorithm 1) and for an x out of bounds or fractional on an integer variable; the restart
    entry point rejects such a point and leaves the walker untouched."""
    inst = synth.tiny(2)
    P = chap.Problem.from_instance(inst)
    x = synth.x_lower(inst)
    w = np.ones(P.m_norm, np.float32)
    P.eval_best_shift(torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda())
    w[3] = -1.0
    with pytest.raises(chap.ChapError) as e:
        P.eval_best_shift(torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda())
    assert e.value.status == 1
    with pytest.raises(chap.ChapError) as e:
        P.eval_best_shift_host(x, w)
    assert e.value.status == 1
    for bad in (0.5, -1.0, 99.0):
        xb = x.copy()
        xb[35] = bad   # integer variable in [0, 7]
        with pytest.raises(chap.ChapError) as e:
            P.eval_best_shift(torch.from_numpy(xb).cuda())
        assert e.value.status == 1
    Wk = chap.Walkers(P, torch.from_numpy(x[None, :]).cuda())
    Wk.step(5)
    before = Wk.get()
    xb = x.copy()
    xb[35] = 0.5
    with pytest.raises(chap.ChapError) as e:
        Wk.restart(0, torch.from_numpy(xb).cuda())
    assert e.value.status == 1
    after = Wk.get()
    assert np.array_equal(before["x"], after["x"]) and np.array_equal(before["r"], after["r"])


def _gridsort_mix(seed=13):
    """Long general columns beyond one block's sort (2100..9000 nonzeros, unbounded and large-domain
    integers): the grid-wide sort of DESIGN §2.5, 2..5 chunks each."""
    return synth.mixed(seed=seed, n=20_000, m=12_000, n_long=6, long_lo=2100, long_hi=9000, long_kinds=("unb", "big"))


def test_gridsort_columns_eval():
    """PAPER.md:355 (grid-wide primitives for vectors longer than a block): per-variable results and
    the best move bit-exact against the oracle, with and without the cutoff row."""
    inst = _gridsort_mix()
    P = chap.Problem.from_instance(inst)
    assert P.info.n_gridsort_columns >= 4, P.info.n_gridsort_columns
    O = oracle.Problem.from_instance(inst)
    for s in range(3):
        x = synth.x_random(inst, 40 + s, spread=60)
        w = synth.weights_random(P.m_norm, 10 + s, hi=9)
        cut = math.inf if s == 0 else float(inst.c @ x) - 40.0
        g, o = _eval_both(inst, x, w, cut, P=P, O=O)
        _assert_same(g, o, f"gridsort s={s}")


def test_gridsort_columns_trajectory(binrow):
    inst = _gridsort_mix(seed=14)
    assert chap.Problem.from_instance(inst).info.n_gridsort_columns >= 4
    _traj_compare(inst, [synth.x_lower(inst), synth.x_random(inst, 5, spread=30)], 25, binary_kernel=binrow)


def test_gridsort_1e5_column():
    """An unbounded integer column with 10^5 nonzeros (49+ chunks): its (x̂, s) bit-exact against
    Algorithm 1 run verbatim in exact rationals (tests/exact.alg1; the oracle's brute force would
    take O(deg^2)), every other variable against the oracle."""
    from fractions import Fraction as Fr
    inst = synth.mixed(seed=15, n=200_000, m=110_000, n_long=1, long_lo=1e5, long_hi=1e5, long_kinds=("unb",))
    P = chap.Problem.from_instance(inst)
    assert P.info.n_gridsort_columns == 1
    deg = np.bincount(inst.col_idx, minlength=inst.n)
    jl = int(np.argmax(deg))
    assert deg[jl] == 100_000
    x = synth.x_random(inst, 7, spread=40)
    w = synth.weights_random(P.m_norm, 7, hi=9)
    xt = torch.from_numpy(x).cuda()
    gx, gs, _ = P.eval_best_shift(xt, torch.from_numpy(w).cuda())
    torch.cuda.synchronize()
    gx, gs = gx.cpu().numpy(), gs.cpu().numpy()
    O = oracle.Problem.from_instance(inst)
    ox, os_ = np.zeros(inst.n), np.zeros(inst.n)
    O.best_shift_range(x, 0, jl, w, out=(ox, os_))
    O.best_shift_range(x, jl + 1, inst.n, w, out=(ox, os_))
    others = np.arange(inst.n) != jl
    assert np.array_equal(gx[others], ox[others]) and np.array_equal(gs[others], os_[others])
    rows = exact.normalized_rows(inst)
    rows.append(({}, Fr(0), -1, +1))   # the inactive cutoff row
    assert len(rows) == P.m_norm
    col = [i for i, (a, _, _, _) in enumerate(rows) if jl in a]
    sub = [rows[i] for i in col]
    r = exact.residuals(sub, x)
    lb, ub = exact.bounds(inst)
    v, sc = exact.alg1(sub, r, x, w[col], jl, lb[jl], ub[jl], True)
    assert sc is not None
    assert gs[jl] == float(sc) and gx[jl] == float(v), (gx[jl], gs[jl], float(v), float(sc))


@pytest.mark.parametrize("seed", range(6))
def test_trajectory_aspiration_config_T(seed, binrow):
    """NEXT f1 (R18, incumbent aspiration): 300-iteration trajectories bit-exact against the oracle's
    rule (itself replayed in exact arithmetic by tests/test_oracle_tabu.py), which takes aspiration
    moves on every one of these walks."""
    inst = synth.tiny(seed)
    _traj_compare(inst, [synth.x_lower(inst)], 300, aspiration=1, binary_kernel=binrow)


def test_trajectory_aspiration_mixed_and_groups():
    """Aspiration through every column class (general tiles, long chunks, sorted columns) and with
    walker groups (6 walkers: the walker-minor kernels note tabu columns per lane)."""
    inst = _sorted_mix(seed=21)
    _traj_compare(inst, [synth.x_lower(inst)], 60, aspiration=1, tenure=6)
    inst = synth.mixed(seed=4, n=3000, m=600, n_long=4, long_lo=300, long_hi=5000)
    _traj_compare(inst, [synth.x_random(inst, s) for s in range(6)], 60, aspiration=1, tenure=5)


@pytest.mark.parametrize("seed", range(6))
def test_trajectory_lazy_config_T(seed):
    """NEXT f2 (selective re-evaluation, chap_params.lazy): only the columns whose x̄ or row state
    changed are re-evaluated; the trajectory (moves, stuck bumps, incumbents that move the dense
    cutoff row) is bit-exact against the oracle's from-scratch walk, with and without aspiration."""
    inst = synth.tiny(seed)
    _traj_compare(inst, [synth.x_lower(inst)], 400, lazy=1, graph_iters=16 if seed % 2 else 0)
    _traj_compare(inst, [synth.x_lower(inst)], 200, lazy=1, aspiration=1)


def test_trajectory_lazy_all_classes():
    """Selective re-evaluation through every column class: packed binary and general tiles, long
    binary and bounded-integer chunks (tickets), block-sorted and grid-sorted general columns."""
    _traj_compare(_sorted_mix(seed=22), [synth.x_lower(_sorted_mix(seed=22))], 80, lazy=1)
    inst = _gridsort_mix(seed=23)
    _traj_compare(inst, [synth.x_random(inst, 2, spread=30)], 20, lazy=1)
    inst = synth.setcover(seed=3, m=1500, n=6000)
    _traj_compare(inst, [synth.x_lower(inst)], 300, lazy=1)


def test_lazy_rejects_walker_sets():
    inst = synth.tiny(1)
    P = chap.Problem.from_instance(inst)
    X0 = torch.from_numpy(np.stack([synth.x_lower(inst)] * 2)).cuda()
    with pytest.raises(chap.ChapError):
        chap.Walkers(P, X0, chap.default_params(lazy=1))


@pytest.mark.parametrize("seed", range(6))
def test_trajectory_perturb_config_T(seed, binrow):
    """NEXT f1 (R21, perturbation after a stuck iteration, counter-based draws): trajectories
    bit-exact against the oracle's step-by-step rule (pinned in tests/test_oracle_perturb.py),
    including the drawn row, entry and value of every perturbation."""
    inst = synth.tiny(seed)
    log = _traj_compare(inst, [synth.x_lower(inst)], 500, graph_iters=16 if seed % 2 else 0, binary_kernel=binrow,
                        perturb=1, rng_seed=1000 + seed, tenure=4)
    assert (log["flags"] == 1).any()


def test_trajectory_perturb_classes_groups_lazy():
    """Perturbations through every column class, with walker groups (distinct draws per walker id),
    selective re-evaluation, aspiration, and across chap_tabu_step calls (a pending perturbation
    drawn by the last iteration of one call is applied by the first of the next)."""
    inst = synth.mixed(seed=5, n=600, m=400, n_long=6, long_lo=100, long_hi=600,
                       long_kinds=("unb", "big", "bkt", "bin"))
    assert chap.Problem.from_instance(inst).info.n_sorted_columns >= 1
    log = _traj_compare(inst, [inst.x_star, synth.x_lower(inst)], 300, perturb=1, rng_seed=8, tenure=3)
    assert (log["flags"] == 1).sum() >= 10
    inst = synth.mixed(seed=5, n=3000, m=600, n_long=6, long_lo=100, long_hi=600)
    x0s = [synth.x_lower(inst), inst.x_star] + [synth.x_random(inst, s) for s in range(4)]
    log = _traj_compare(inst, x0s, 300, perturb=1, rng_seed=8, tenure=3)
    assert (log["flags"] == 1).any()
    inst = synth.tiny(2)
    log = _traj_compare(inst, [synth.x_lower(inst)], 300, lazy=1, perturb=1, rng_seed=9, tenure=4)
    assert (log["flags"] == 1).any()
    log = _traj_compare(inst, [synth.x_lower(inst)], 300, aspiration=1, perturb=1, rng_seed=10, tenure=4,
                        split=[7, 1, 13, 29, 250])
    assert (log["flags"] == 1).any()


@pytest.mark.parametrize("seed", range(4))
def test_trajectory_weight_smoothing(seed, binrow):
    """NEXT f1 (R22, weight smoothing): stuck iterations that draw u < smooth_prob lower the weights
    of the satisfied rows instead of bumping the violated ones; trajectories and final weights
    bit-exact against the oracle, alone and with the perturbation, with walker groups."""
    inst = synth.tiny(seed)
    _traj_compare(inst, [synth.x_lower(inst)], 500, binary_kernel=binrow, smooth_prob=0.4, rng_seed=seed, tenure=4)
    _traj_compare(inst, [synth.x_lower(inst)], 400, binary_kernel=binrow, smooth_prob=0.3, perturb=1,
                  rng_seed=50 + seed, tenure=4, graph_iters=0)
    if seed == 0:
        inst = synth.mixed(seed=5, n=3000, m=600, n_long=6, long_lo=100, long_hi=600)
        x0s = [synth.x_lower(inst), inst.x_star] + [synth.x_random(inst, s) for s in range(4)]
        _traj_compare(inst, x0s, 300, perturb=1, smooth_prob=0.5, rng_seed=8, tenure=3)


def test_walker_groups_continuous_columns_match_single_walkers():
    """a10 for continuous columns: in walker groups k_eval_gen_wm evaluates the packed continuous
    columns for the whole group (gen_column_serial per lane, the group's row-state layout). The
    continuous path is checked against exact-rational Algorithm 1 in tolerance mode above
    (test_continuous_columns_tolerance_mode); here every walker of a 12-walker group follows,
    bit for bit, the trajectory the same walker follows alone (one walker: k_eval_gen's per-walker
    path with the same arithmetic)."""
    import dataclasses
    inst = synth.mixed(seed=9, n=4000, m=800, n_long=0)
    rng = np.random.default_rng(31)
    gen = np.nonzero((inst.is_int == 1) & (inst.ub > 1.0) & np.isfinite(inst.ub))[0]
    cont = rng.choice(gen, size=len(gen) // 2, replace=False)
    is_int = inst.is_int.copy()
    is_int[cont] = 0
    inst = dataclasses.replace(inst, is_int=is_int, name=inst.name + "-cont")
    P = chap.Problem.from_instance(inst)
    assert P.info.n_continuous >= 100
    x0s = np.stack([synth.x_lower(inst)] + [synth.x_random(inst, s) for s in range(11)])
    prm = chap.default_params(graph_iters=0)
    G = chap.Walkers(P, torch.from_numpy(x0s).cuda(), prm)
    glog = chap.records(G.step(40, log=True)).reshape(40, len(x0s))
    gst = G.get()
    for wi in range(len(x0s)):
        S1 = chap.Walkers(P, torch.from_numpy(x0s[wi:wi + 1]).cuda(), prm)
        slog = chap.records(S1.step(40, log=True)).reshape(40, 1)[:, 0]
        sst = S1.get()
        for f in ("k", "j", "flags", "violated"):
            assert np.array_equal(glog[f][:, wi], slog[f]), (wi, f)
        mv = slog["j"] >= 0
        assert np.array_equal(glog["v"][mv, wi], slog["v"][mv]), wi
        # c.x of fractional points is a grid-wide sum (k_cut_dot) whose order follows the launch
        # shape: the objective and the cutoff row's residual agree to rounding
        assert np.allclose(glog["obj"][:, wi], slog["obj"], rtol=1e-12, atol=1e-9), wi
        assert np.array_equal(gst["x"][wi], sst["x"][0]), wi
        assert np.array_equal(gst["r"][wi][:-1], sst["r"][0][:-1]), wi
        assert np.allclose(gst["r"][wi][-1:], sst["r"][0][-1:], rtol=1e-12, atol=1e-9), wi
        S1.close()


@pytest.mark.parametrize("kind", ["big_int_weights", "float_weights", "huge_residuals", "huge_and_float"])
def test_eval_edge_domains(kind):
    """The kernels' alternative paths against the oracle, bit for bit, on an instance with packed
    general tiles, long bounded-integer and long binary columns:
      - integral weights above 2^20 (the general kernels' float-word path instead of the int path,
        and the double binary penalties instead of the integer flip sums);
      - non-integral float weights (the same paths; every term and sum still exact in double);
      - unbounded integer variables at ~1e9 and rows far from tight, so residuals reach ~1e11:
        the double division of lines 3-4 instead of the float quotient (|r| >= 2^23), and offsets
        beyond the int path (|d| >= 2^28: the tile re-evaluated in double by gen_column_serial)."""
    inst = synth.mixed(seed=5, n=4000, m=800, n_long=6, long_lo=300, long_hi=3000)
    P = chap.Problem.from_instance(inst)
    O = oracle.Problem.from_instance(inst)
    rng = np.random.default_rng([0xED, len(kind)])
    x = synth.x_random(inst, 7)
    if kind in ("huge_residuals", "huge_and_float"):
        unb = np.nonzero(np.isinf(inst.ub) & (inst.is_int == 1))[0]
        assert unb.size > 10
        x[unb] = rng.integers(10**8, 10**9, unb.size).astype(np.float64)
    if kind == "big_int_weights":
        w = rng.integers(2**20 + 1, 2**22, P.m_norm).astype(np.float32)
    elif kind in ("float_weights", "huge_and_float"):
        w = rng.uniform(0.1, 10.0, P.m_norm).astype(np.float32)
    else:
        w = rng.integers(1, 6, P.m_norm).astype(np.float32)
    for cut in (math.inf, float(inst.c @ x) - 1.0):
        g, o = _eval_both(inst, x, w, cut, P, O)
        _assert_same(g, o, f"{kind} cut={cut}")


def test_trajectory_huge_residuals():
    """A walk started with the unbounded integer variables at ~1e9 (residuals ~1e11: the double
    division and the double re-evaluation of offsets beyond the int path, inside the tabu step with
    its dynamic item hand-out) stays bit-exact with the oracle's walk."""
    inst = synth.mixed(seed=5, n=4000, m=800, n_long=6, long_lo=300, long_hi=3000)
    rng = np.random.default_rng(0xED)
    x = synth.x_random(inst, 7)
    unb = np.nonzero(np.isinf(inst.ub) & (inst.is_int == 1))[0]
    x[unb] = rng.integers(10**8, 10**9, unb.size).astype(np.float64)
    _traj_compare(inst, [x], 40)
