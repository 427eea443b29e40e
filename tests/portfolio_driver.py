"""Test-side driver of the walker portfolio over ORACLE walkers: the
exchange decisions come from the product's host rule chap_exchange_plan (no GPU needed), the
points and summaries travel through an `allgather` callable (identity in one process,
torch.distributed all_gather_object with gloo across processes)."""
import math

import numpy as np

import paper_2605_05086_b200 as chap


def local_summaries(walkers, rank, W_local, stop=False):
    S = np.zeros(len(walkers), chap.SUMMARY_DTYPE)
    for w, wk in enumerate(walkers):
        v, sv = wk.summary()
        S[w]["best_obj"] = wk.best_obj if wk.has_incumbent else math.inf
        S[w]["violated"] = v
        S[w]["sumviol"] = sv
        S[w]["gid"] = rank * W_local + w
        S[w]["flags"] = (1 if wk.has_incumbent else 0) | (2 if stop else 0)
    return S


def local_elite_points(walkers, summaries, n, n_elite):
    """Slots [0, n_elite): the rank's best incumbents by (best_obj, gid); [n_elite, 2 n_elite): its
    current points by (violated, sumviol, gid)."""
    pts = [None] * (2 * n_elite)
    feas = sorted([(s["best_obj"], int(s["gid"]), w) for w, s in enumerate(summaries) if s["flags"] & 1])
    for q, (_, _, w) in enumerate(feas[:n_elite]):
        pts[q] = walkers[w].best_x[:n].copy()
    inf = sorted([(int(s["violated"]), float(s["sumviol"]), int(s["gid"]), w) for w, s in enumerate(summaries)])
    for q, (_, _, _, w) in enumerate(inf[:n_elite]):
        pts[n_elite + q] = walkers[w].x[:n].copy()
    return pts


def run_portfolio(walkers, rank, nranks, n, K, n_epochs, n_elite, n_restart, allgather):
    W_local = len(walkers)
    for ep in range(n_epochs):
        for wk in walkers:
            wk.run(K)
        if ep == n_epochs - 1:
            break
        mine = local_summaries(walkers, rank, W_local)
        allS = np.concatenate(allgather(mine))
        plan = chap.exchange_plan(allS, W_local, n_elite, n_restart)
        recv = allgather(local_elite_points(walkers, mine, n, n_elite))
        if plan["z_best"] < math.inf:
            for wk in walkers:
                wk.set_cutoff(plan["z_best"])
        for q, gid in enumerate(plan["restart_gid"]):
            if gid // W_local != rank:
                continue
            slot = int(plan["elite_slot"][plan["restart_src"][q]])
            point = recv[slot // (2 * n_elite)][slot % (2 * n_elite)]
            walkers[gid % W_local].restart(point)
    return walkers


def state(wk, n):
    return {"x": wk.x[:n].copy(), "w": wk.w.copy(), "tabu": wk.tabu_until[:n].copy(), "k": wk.k,
            "best_obj": wk.best_obj, "best_x": wk.best_x[:n].copy(), "cut": wk.cutoff_rhs,
            "inc": wk.has_incumbent}
