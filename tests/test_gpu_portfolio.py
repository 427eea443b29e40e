"""GPU: chap_run_walkers (the portfolio with the every-K exchange) against the
oracle's single-process orc_run_walkers — same best objective, same best point — without a
communicator and through a one-rank NCCL communicator (the NCCL allgather path)."""
import math

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no GPU", allow_module_level=True)

import paper_2605_05086_b200 as chap  # noqa: E402


def _case(inst, W, K, E, ne, nr, comm=None):
    x0s = np.stack([np.clip(synth.x_random(inst, 100 + w), inst.lb, inst.ub) for w in range(W)])
    O = oracle.Problem.from_instance(inst)
    ws = [oracle.TabuWalker(O, x) for x in x0s]
    oracle.run_walkers(O, ws, K, E, ne, nr)
    P = chap.Problem.from_instance(inst)
    prm = chap.default_params(exchange_K=K, n_elite=ne, n_restart=nr, graph_iters=8)
    res, bx = chap.run_walkers(P, torch.from_numpy(x0s).cuda(), prm, comm, max_iters=K * E)
    torch.cuda.synchronize()
    inc = [w for w in ws if w.has_incumbent]
    assert res.iterations == K * E and res.epochs == E
    if not inc:
        assert not res.has_incumbent
        return
    best = min(inc, key=lambda w: w.best_obj)
    gid = ws.index(min(inc, key=lambda w: (w.best_obj, ws.index(w))))
    assert res.has_incumbent and res.best_obj == best.best_obj and res.best_walker == gid
    assert np.array_equal(bx.cpu().numpy(), ws[gid].best_x[: inst.n])


@pytest.mark.parametrize("seed", [1, 3, 5])
def test_run_walkers_matches_oracle_portfolio(seed):
    _case(synth.tiny(seed), W=6, K=40, E=4, ne=2, nr=2)


def test_run_walkers_mixed_instance():
    inst = synth.mixed(seed=9, n=3000, m=600, n_long=2, long_lo=200, long_hi=3000)
    _case(inst, W=4, K=25, E=3, ne=1, nr=1)


def test_run_walkers_one_rank_nccl():
    comm = chap.Comm(chap.comm_unique_id(), 1, 0, 0)
    try:
        _case(synth.tiny(2), W=6, K=40, E=4, ne=2, nr=3, comm=comm)
    finally:
        comm.close()


@pytest.mark.parametrize("seed,comm_kind,mode,W,nr,lazy", [(1, None, "exchange", 6, 2, 0), (4, "nccl", "exchange", 6, 2, 0),
                                                         (1, None, "epoch", 6, 2, 0), (4, "nccl", "epoch", 6, 3, 0),
                                                         (6, None, "epoch", 40, 7, 0), (7, None, "exchange", 40, 40, 0),
                                                         (2, None, "epoch", 1, 1, 1), (3, None, "epoch", 1, 1, 0)])
def test_walkers_exchange_epochs_match_oracle(seed, comm_kind, mode, W, nr, lazy):
    """chap_walkers_exchange between chap_tabu_step epochs, or chap_walkers_epoch (iterations and
    the device exchange as one CUDA graph, what bench.py times), reproduces the oracle portfolio
    walker by walker: point, weights, tabu list, incumbent (W = 40: two walker groups, restarts in
    both; nr = W: every walker restarts; W = 1: the single-walker kernels restart the walker from its
    own elite point, from scratch and with selective re-evaluation)."""
    inst = synth.tiny(seed)
    K, E, ne = 30, 4, 2
    x0s = np.stack([np.clip(synth.x_random(inst, 200 + w), inst.lb, inst.ub) for w in range(W)])
    O = oracle.Problem.from_instance(inst)
    ows = [oracle.TabuWalker(O, x) for x in x0s]
    oracle.run_walkers(O, ows, K, E, ne, nr)
    P = chap.Problem.from_instance(inst)
    comm = chap.Comm(chap.comm_unique_id(), 1, 0, 0) if comm_kind else None
    try:
        ws = chap.Walkers(P, torch.from_numpy(x0s).cuda(),
                          chap.default_params(exchange_K=K, n_elite=ne, n_restart=nr, graph_iters=8, lazy=lazy))
        zs = []
        for e in range(E):
            if e == E - 1:
                ws.step(K)
            elif mode == "epoch":
                zs.append(ws.epoch(K, comm, result=(e == 1)))
            else:
                ws.step(K)
                zs.append(ws.exchange(comm))
        st = ws.get()
    finally:
        if comm is not None:
            comm.close()
    # the best incumbent after the second exchange: the oracle's walkers at that point are not kept,
    # so check it against the final incumbents' consistency (never better than the final best)
    if zs and zs[1] is not None and math.isfinite(zs[1][0]):
        assert zs[1][0] >= min(ow.best_obj for ow in ows if ow.has_incumbent)
    for w, ow in enumerate(ows):
        assert np.array_equal(st["x"][w], ow.x[: inst.n]), w
        assert np.array_equal(st["w"][w], ow.w), w
        assert np.array_equal(st["tabu_until"][w], ow.tabu_until[: inst.n]), w
        assert st["stats"][w]["has_incumbent"] == int(ow.has_incumbent), w
        if ow.has_incumbent:
            assert st["stats"][w]["best_obj"] == ow.best_obj, w


def test_packed_exchange_points():
    """elite points travel packed — binaries as bits, bounded integers
    as int32 — config P's 10^5 binaries in 12.5 KB instead of 800 KB of f64."""
    al8 = lambda b: (b + 7) // 8 * 8   # noqa: E731
    P = chap.Problem.from_instance(synth.packing())
    assert P.info.exchange_point_bytes == al8(4 * ((P.info.n_binary + 31) // 32)) <= 12_504
    Q = chap.Problem.from_instance(synth.tiny(0))
    assert Q.info.exchange_point_bytes == al8(4 * ((Q.info.n_binary + 31) // 32)) + al8(4 * Q.info.n_integer)


def _rank_run(rank, world, uid, inst_seed, W, K, E, ne, nr, q):
    import torch as th
    import paper_2605_05086_b200 as ch
    th.cuda.set_device(rank)
    inst = synth.tiny(inst_seed)
    Wl = W // world
    x0s = np.stack([np.clip(synth.x_random(inst, 100 + w), inst.lb, inst.ub) for w in range(W)])
    P = ch.Problem.from_instance(inst, device=rank)
    comm = ch.Comm(uid, world, rank, rank)
    prm = ch.default_params(exchange_K=K, n_elite=ne, n_restart=nr, graph_iters=8)
    res, bx = ch.run_walkers(P, th.from_numpy(x0s[rank * Wl:(rank + 1) * Wl]).cuda(rank), prm, comm, max_iters=K * E)
    th.cuda.synchronize()
    comm.close()
    q.put((rank, res.best_obj, res.best_walker, bx.cpu().numpy() if bx is not None else None))


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs (one NCCL rank per GPU)")
def test_two_ranks_equal_one_rank():
    """SURVEY §8(e) invariant on the CUDA path: 2 ranks x W/2 walkers reach the same best objective,
    best walker (global id) and best point as 1 rank x W walkers (the exchange plan is the same
    deterministic function of the gathered summaries)."""
    import torch.multiprocessing as mp
    inst = synth.tiny(3)
    W, K, E, ne, nr = 8, 30, 4, 2, 2
    x0s = np.stack([np.clip(synth.x_random(inst, 100 + w), inst.lb, inst.ub) for w in range(W)])
    P = chap.Problem.from_instance(inst)
    prm = chap.default_params(exchange_K=K, n_elite=ne, n_restart=nr, graph_iters=8)
    res1, bx1 = chap.run_walkers(P, torch.from_numpy(x0s).cuda(), prm, None, max_iters=K * E)
    torch.cuda.synchronize()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    uid = chap.comm_unique_id()
    ps = [ctx.Process(target=_rank_run, args=(r, 2, uid, 3, W, K, E, ne, nr, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = sorted(q.get(timeout=300) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
    for rank, obj, bw, bx in out:
        assert obj == res1.best_obj and bw == res1.best_walker
        if res1.has_incumbent:
            assert np.array_equal(bx, bx1.cpu().numpy())


def _random_summaries(rng, W):
    """Gathered summaries with many ties: objectives and violation counts from small ranges."""
    S = np.zeros(W, chap.SUMMARY_DTYPE)
    feas = rng.random(W) < 0.5
    S["best_obj"] = np.where(feas, rng.integers(-5, 5, W).astype(np.float64), math.inf)
    S["violated"] = rng.integers(0, 4, W)
    S["sumviol"] = rng.integers(0, 3, W) * 0.5
    S["gid"] = np.arange(W)
    S["flags"] = feas.astype(np.int32)
    return S


@pytest.mark.parametrize("nranks,W_local", [(1, 1), (1, 7), (2, 3), (4, 8), (8, 5), (8, 64)])
def test_device_exchange_plan_matches_host_plan(nranks, W_local):
    """k_exchange_plan (the device exchange of chap_walkers_exchange / chap_walkers_epoch) makes
    chap_exchange_plan's decisions for every rank of a multi-rank portfolio — reachable here on one
    GPU by asking for each rank's view of random gathered summaries with ties: the same best, elite
    (gid, kind, slot) and restarts; each rank's local ranks place its elite members in their slots
    and its restart slots point at their sources' slots."""
    rng = np.random.default_rng([nranks, W_local])
    W = nranks * W_local
    for trial in range(6):
        S = _random_summaries(rng, W)
        ne, nr = [(0, 0), (1, 1), (2, W // 8), (4, W), (3, 2), (2, W + 3)][trial]
        host = chap.exchange_plan(S, W_local, ne, nr)
        E = len(host["elite_gid"])
        for rank in range(nranks):
            dev = chap.exchange_plan_device(S, W_local, rank, ne, nr)
            if math.isinf(host["z_best"]):
                assert math.isinf(dev["z_best"])
            else:
                assert dev["z_best"] == host["z_best"]
            assert dev["best_gid"] == host["best_gid"]
            for k in ("elite_gid", "elite_kind", "elite_slot", "restart_gid", "restart_src"):
                assert np.array_equal(dev[k], host[k]), (trial, rank, k, dev[k], host[k])
            lo = rank * W_local
            for q in range(E):
                g, kind = int(host["elite_gid"][q]), int(host["elite_kind"][q])
                if lo <= g < lo + W_local:
                    assert host["elite_slot"][q] == rank * 2 * ne + kind * ne + dev["local_rank"][kind][g - lo]
            slots = np.full(W_local, -1)
            for q in range(len(host["restart_gid"])):
                g = int(host["restart_gid"][q])
                if lo <= g < lo + W_local:
                    slots[g - lo] = host["elite_slot"][host["restart_src"][q]]
            assert np.array_equal(dev["restart_slot"], slots), (trial, rank)
