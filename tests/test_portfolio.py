"""CPU: the exchange rule of the walker portfolio.

- chap_exchange_plan (the product's host rule) on a hand-derived case;
- the portfolio driven by chap_exchange_plan over oracle walkers equals the oracle's own
  single-process orc_run_walkers, walker by walker (one process);
- the same split across two gloo processes (world_size 2) gives the identical result:
  the rule is independent of the rank count.
"""
import json
import math
import os
import socket
import tempfile

import numpy as np
import pytest

import oracle
import paper_2605_05086_b200 as chap
import synth
from tests import portfolio_driver as drv

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_exchange_plan_golden():
    g = json.load(open(os.path.join(GOLD, "exchange_plan.json")))
    S = np.zeros(len(g["summaries"]), chap.SUMMARY_DTYPE)
    for i, s in enumerate(g["summaries"]):
        S[i] = (math.inf if s["best_obj"] is None else s["best_obj"], s["violated"], s["sumviol"], i, s["flags"])
    plan = chap.exchange_plan(S, g["W_local"], g["n_elite"], g["n_restart"])
    exp = g["expected"]
    assert plan["z_best"] == exp["z_best"] and plan["best_gid"] == exp["best_gid"]
    for k in ("elite_gid", "elite_kind", "elite_slot", "restart_gid", "restart_src"):
        assert list(plan[k]) == exp[k], k


def _setup(seed, W):
    inst = synth.tiny(seed)
    P = oracle.Problem.from_instance(inst)
    x0s = [np.clip(synth.x_random(inst, 100 + w), inst.lb, inst.ub) for w in range(W)]
    return inst, P, x0s


def _reference(seed, W, K, E, n_elite, n_restart):
    inst, P, x0s = _setup(seed, W)
    ws = [oracle.TabuWalker(P, x) for x in x0s]
    oracle.run_walkers(P, ws, K, E, n_elite, n_restart)
    return inst, [drv.state(w, inst.n) for w in ws]


def _same(a, b):
    for k in a:
        if isinstance(a[k], np.ndarray):
            assert np.array_equal(a[k], b[k]), k
        else:
            assert a[k] == b[k], (k, a[k], b[k])


@pytest.mark.parametrize("seed", [1, 4])
def test_plan_driven_portfolio_equals_oracle_rule(seed):
    W, K, E, ne, nr = 6, 40, 4, 2, 2
    inst, ref = _reference(seed, W, K, E, ne, nr)
    _, P, x0s = _setup(seed, W)
    ws = [oracle.TabuWalker(P, x) for x in x0s]
    drv.run_portfolio(ws, 0, 1, inst.n, K, E, ne, nr, lambda obj: [obj])
    for a, w in zip(ref, ws):
        _same(a, drv.state(w, inst.n))
    assert sum(1 for a in ref if a["inc"]) >= 1


def _rank_main(rank, world, port, seed, W, K, E, ne, nr, outdir):
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    inst, P, x0s = _setup(seed, W)
    W_local = W // world
    ws = [oracle.TabuWalker(P, x) for x in x0s[rank * W_local:(rank + 1) * W_local]]

    def allgather(obj):
        out = [None] * world
        dist.all_gather_object(out, obj)
        return out

    drv.run_portfolio(ws, rank, world, inst.n, K, E, ne, nr, allgather)
    for w, wk in enumerate(ws):
        np.savez(os.path.join(outdir, f"w{rank * W_local + w}.npz"), **{k: np.asarray(v) for k, v in
                                                                        drv.state(wk, inst.n).items()})
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_gloo_ranks_equal_one_process():
    import torch.multiprocessing as mp
    seed, W, K, E, ne, nr = 3, 6, 40, 4, 2, 3
    inst, ref = _reference(seed, W, K, E, ne, nr)
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_rank_main, args=(2, _free_port(), seed, W, K, E, ne, nr, d), nprocs=2, join=True)
        for g in range(W):
            z = np.load(os.path.join(d, f"w{g}.npz"))
            got = {k: (z[k] if z[k].ndim else z[k].item()) for k in z.files}
            _same(ref[g], got)
