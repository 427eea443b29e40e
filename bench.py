#!/usr/bin/env python
"""bench.py — best-shift tabu core of CHAP (arxiv 2605.05086) on B200.

A "step" is one tabu iteration of every walker on the GPU: the exact best shift of every
variable (Algorithm 1, all column classes), the global select, and the apply / weight bump /
incumbent check — the whole hot path of SURVEY.md §8(a). Default workload: config G
(BASELINE.json configs[2]: 200k rows x 1M vars, ~10.4M nnz, 100 long columns), one walker per
GPU; N>1 GPUs run independent walker replicas (weak scaling, no collective in the timed region).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config G|S|P] [--impl chap|reference]

Prints ONE JSON line (rank 0). --impl reference times the plain fp64 CPU oracle (oracle/) on
the same workload on the host cores (the reference arm of this tier).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "best-shift move evaluations/sec and tabu iterations/sec; % of HBM roofline"
UNIT = "move_evals/s"
# kernels of one epoch's tail (chap_walkers_epoch): the incumbent flush (2) and the device exchange
# (summaries, plan, packing, cutoff, restart batch: 14 with elite points and the bitset kept)
EXCHANGE_KERNELS = 16

CONFIGS = {
    "G": dict(desc="G: synthetic mixed general-integer MIP 200k rows x 1M vars, ~10.4M nnz, 100 long columns "
                   "(BASELINE.json configs[2])", walkers=1),
    "T": dict(desc="T: tiny synthetic MIP, 40 vars x 25 rows (knapsack + cover + general; BASELINE.json "
                   "configs[0], a test configuration)", walkers=1),
    "S": dict(desc="S: synthetic set cover 10k rows x 50k binaries, ~500k nnz (BASELINE.json configs[1])", walkers=1),
    "P": dict(desc="P: packing MIP 20k rows x 100k binaries, ~1M nnz, 64 walkers (BASELINE.json configs[3])",
              walkers=64),
    # BASELINE.json configs[4], the scaling sweep: generator X at a requested nonzero count
    "X1e5": dict(desc="X: scaling sweep, generator G scaled to ~1e5 nnz (BASELINE.json configs[4])", walkers=1),
    "X3e5": dict(desc="X: scaling sweep, generator G scaled to ~3e5 nnz (BASELINE.json configs[4])", walkers=1),
    "X1e6": dict(desc="X: scaling sweep, generator G scaled to ~1e6 nnz (BASELINE.json configs[4])", walkers=1),
    "X3e6": dict(desc="X: scaling sweep, generator G scaled to ~3e6 nnz (BASELINE.json configs[4])", walkers=1),
    "X1e7": dict(desc="X: scaling sweep, generator G scaled to ~1e7 nnz (BASELINE.json configs[4])", walkers=1),
    "X2e7": dict(desc="X: scaling sweep, generator G scaled to ~2e7 nnz (BASELINE.json configs[4])", walkers=1),
    "X5e7": dict(desc="X: scaling sweep, generator G scaled to ~5e7 nnz (BASELINE.json configs[4])", walkers=1),
    # diagnostic variants of G (not BASELINE configs): same structure, one variable class only
    "Gbin": dict(desc="diagnostic: config G structure with every short variable binary", walkers=1),
    "Gint": dict(desc="diagnostic: config G structure with every short variable bounded integer", walkers=1),
    "Gnl": dict(desc="diagnostic: config G without its 100 long columns", walkers=1),
}


def make_instance(cfg: str):
    if cfg == "T":
        return synth.tiny(0)
    if cfg == "G":
        return synth.mixed()
    if cfg == "S":
        return synth.setcover()
    if cfg == "P":
        return synth.packing()
    if cfg == "Gbin":
        return synth.mixed(p_binary=1.0, p_bounded=0.0)
    if cfg == "Gint":
        return synth.mixed(p_binary=0.0, p_bounded=1.0)
    if cfg == "Gnl":
        return synth.mixed(n_long=0)
    if cfg.startswith("X"):
        return synth.scaled(int(float(cfg[1:])))
    raise ValueError(cfg)


def start_points(inst, cfg: str, W: int, rank: int):
    """x0 of the W walkers of a rank. Config P: Bernoulli(0.5) keyed (3, global walker id) (SURVEY
    8(d)). Otherwise walker 0 of rank 0 starts at x_lower (0); every other walker (global id g > 0)
    at x_lower with 1 % of its variables raised by one step (keyed by g), so that weak-scaling
    replicas walk different trajectories over the same amount of work per iteration."""
    if cfg == "P":
        return np.stack([synth.x_bernoulli(inst, (3, rank * W + w), 0.5) for w in range(W)])
    return np.stack([synth.x_lower(inst) if rank * W + w == 0 else synth.x_perturbed(inst, (5, rank * W + w), 0.01)
                     for w in range(W)])


def config_dict(cfg: str, inst, W: int, world: int, z_star):
    """The `config` object of the JSON line: identical for both arms (--impl chap / reference)."""
    a_bytes = 12 * (inst.nnz + int(np.count_nonzero(inst.c))) + 4 * (inst.n + 1)   # SURVEY 8(d) model of A
    l2 = (f"inputs larger than L2: A in CSC alone is {a_bytes / 1e6:.0f} MB vs 126 MB L2; no flush"
          if a_bytes > 126e6 else
          f"working set L2-resident (A in CSC {a_bytes / 1e6:.0f} MB + {W} walkers' state) and kept so on "
          "purpose: consecutive tabu iterations reuse it, no flush; the HBM fraction is not the bound here")
    return {"workload": CONFIGS[cfg]["desc"], "walkers_per_gpu": W, "n": inst.n, "m": inst.m, "nnz": inst.nnz,
            "l2": l2,
            "parallelism": f"walker portfolio x{world}: independent walkers per GPU (weak scaling, distinct start "
                           f"points), exchange every 1000 iterations",
            "cutoff": ("active from the start: c.x <= z* - delta, z* = c.x* of the instance's planted feasible "
                       "point (PAPER.md:373)" if z_star is not None else "none")}


def maybe_spawn(args):
    """--gpus N with no torchrun environment: re-launch this command under torch.distributed.run with
    N ranks (one process per GPU, rendezvous on 127.0.0.1); returns only in the child ranks or at N=1."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    sys.stdout.flush()
    os.execvp(sys.executable, cmd)


def measured_peak_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def planted_objective(inst):
    """The objective of the instance's planted feasible point: the walkers search with the cutoff
    c.x <= z* - delta active from the start, as CHAP's tabu workers do with the pool's best-known
    objective (SURVEY 8(d) 'G, 1 walker, tabu step (cutoff active)')."""
    xs = getattr(inst, "x_star", None)
    return None if xs is None else float(np.asarray(inst.c, np.float64) @ np.asarray(xs, np.float64))


def cpu_model() -> str:
    try:
        for line in subprocess.check_output(["lscpu"], text=True).splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def oracle_baseline(inst, x0, seconds_target: float = 12.0, max_iters: int = 400):
    """The oracle as it stands, on the host cores: tabu iterations of one walker (bounded sample),
    timed with all cores and with one thread."""
    import oracle
    O = oracle.Problem.from_instance(inst)
    z = planted_objective(inst)
    n_eval = int(np.sum(O.vars()[2] != 0))
    cores = os.cpu_count() or 1
    out = {}
    for threads in (cores, 1):
        ow = oracle.TabuWalker(O, x0)
        if z is not None:
            ow.set_cutoff(z)
        t0 = time.perf_counter()
        ow.run(1, threads=threads)
        t1 = time.perf_counter() - t0
        budget = seconds_target if threads == cores else seconds_target / 2
        iters = int(max(1, min(max_iters, budget / max(t1, 1e-6))))
        t0 = time.perf_counter()
        ow.run(iters, threads=threads)
        dt = time.perf_counter() - t0
        out[threads] = (n_eval * iters / dt, iters, dt)
    v, iters, dt = out[cores]
    v1, iters1, dt1 = out[1]
    return {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{iters} tabu iterations of 1 walker (after 1 warm-up iteration), all {n_eval} non-fixed "
                      f"variables evaluated per iteration, OpenMP over variables on {cores} threads",
            "seconds": dt, "iters_per_s": iters / dt, "cpu_model": cpu_model(),
            "one_thread": {"value": v1, "unit": UNIT, "cores": 1, "iters": iters1, "seconds": dt1}}


def run_reference(args):
    """The reference arm: the oracle (oracle/, test infrastructure) on the host cores, on this
    arm's config and metric. A step is one tabu iteration of the walker when (warmup + steps)
    iterations fit the time budget; otherwise a bounded sample of one: the activities from scratch
    and Eq. (1) for a rotating slice of the variables, sized so the whole run ends within the
    budget."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return   # under torchrun (N > 1) rank 0 alone runs the oracle; the other ranks exit 0
    budget_s = float(os.environ.get("CHAP_REF_BUDGET_S", "150"))
    cfg = args.config
    inst = make_instance(cfg)
    x0 = start_points(inst, cfg, 1, 0)[0]
    import oracle
    O = oracle.Problem.from_instance(inst)
    ow = oracle.TabuWalker(O, x0)
    z = planted_objective(inst)
    if z is not None:
        ow.set_cutoff(z)
    n_eval = int(np.sum(O.vars()[2] != 0))
    t0 = time.perf_counter()
    ow.run(1)   # one full iteration sizes the run
    t_iter = time.perf_counter() - t0
    total = args.warmup + args.steps
    if total * t_iter <= budget_s:
        ow.run(max(0, args.warmup - 1))
        t0 = time.perf_counter()
        ow.run(args.steps)
        dt = time.perf_counter() - t0
        evals = n_eval * args.steps
        sample = f"{args.steps} full tabu iterations of 1 walker after {args.warmup} warm-up"
    else:
        frac = max(1e-4, budget_s / (total * t_iter))
        span = max(1, int(inst.n * frac))
        x = ow.x[: inst.n].copy()
        w = ow.w.copy()
        bufs = (np.zeros(inst.n), np.zeros(inst.n))
        j0 = 0
        for _ in range(args.warmup):
            O.best_shift_range(x, j0, min(inst.n, j0 + span), w, ow.cutoff_rhs, out=bufs)
            j0 = (j0 + span) % inst.n
        evals = 0
        t0 = time.perf_counter()
        for _ in range(args.steps):
            j1 = min(inst.n, j0 + span)
            O.best_shift_range(x, j0, j1, w, ow.cutoff_rhs, out=bufs)
            evals += j1 - j0
            j0 = j1 % inst.n
        dt = time.perf_counter() - t0
        sample = (f"bounded sample per step: activities from scratch + Eq. (1) for {span} of {inst.n} "
                  f"variables (rotating slice), {args.steps} steps after {args.warmup} warm-up")
    value = evals / dt
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generator synth/, no dataset)",
            "config": config_dict(cfg, inst, 1, args.gpus, z),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": os.cpu_count(), "kind": "oracle",
                             "sample": sample, "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "launcher": {"world_size": int(os.environ.get("WORLD_SIZE", "1")), "rank": rank}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=4000)
    ap.add_argument("--warmup", type=int, default=50)
    ap.add_argument("--config", default="G", choices=sorted(CONFIGS))
    ap.add_argument("--walkers", type=int, default=0)
    ap.add_argument("--impl", default="chap", choices=["chap", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-iters", type=int, default=200)
    ap.add_argument("--e2e-iters", type=int, default=20)
    ap.add_argument("--no-cutoff", action="store_true",
                    help="A/B runs: leave the cutoff row inactive (no planted objective)")
    ap.add_argument("--param", action="append", default=[],
                    help="chap_params field override NAME=VALUE (A/B runs, e.g. l2_persist=0)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    maybe_spawn(args)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    import paper_2605_05086_b200 as chap

    cfg = args.config
    W = args.walkers or CONFIGS[cfg]["walkers"]
    inst = make_instance(cfg)
    P = chap.Problem.from_instance(inst, device=local)
    info = P.info
    n_eval = info.n - info.n_fixed
    x0 = torch.from_numpy(start_points(inst, cfg, W, rank)).to(dev)
    prm = chap.default_params(graph_iters=32)
    for kv in args.param:
        k, v = kv.split("=", 1)
        setattr(prm, k, type(getattr(prm, k))(float(v)) if isinstance(getattr(prm, k), float) else int(v))
    ws = chap.Walkers(P, x0, prm)
    z_star = None if args.no_cutoff else planted_objective(inst)
    if z_star is not None:
        ws.set_cutoff(z_star)   # the cutoff row is active from the start
    ws.timing(1)   # per-kernel %globaltimer spans inside the graphs (no events), on before the warm-up
    comm = None    # the portfolio exchange every exchange_K iterations: NCCL across ranks
    if world > 1:
        uid = [chap.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = chap.Comm(uid[0], world, rank, local)
    K_x = int(prm.exchange_K)

    def barrier():
        if world > 1:
            dist.barrier()

    ws.step(args.warmup)
    if args.steps > K_x:   # the epoch graph (exchange_K iterations + the exchange) is captured here,
        ws.epoch(K_x, comm)   # untimed, like the iteration graphs
    torch.cuda.synchronize()
    ws.timing(1)   # zero the sums: they cover exactly the timed region
    barrier()
    stream = torch.cuda.current_stream()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        e0.record(stream)
        done = n_exchanges = 0
        while done < args.steps:   # epochs of exchange_K tabu iterations with the exchange between:
            k = min(K_x, args.steps - done)   # each one CUDA graph (iterations + device exchange)
            if done + k < args.steps:
                ws.epoch(k, comm)
                n_exchanges += 1
            else:
                ws.step(k)
            done += k
        e1.record(stream)
        torch.cuda.synchronize()
    barrier()
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    sec = ms_max / 1e3
    value = n_eval * W * args.steps * world / sec
    kt = ws.timing(0).astype(np.float64)   # sums over the timed region, then timing off
    st = ws.get()["stats"]
    names = ["binary (k_eval_binrow / k_eval_bin)", "k_eval_gen", "k_eval", "-", "k_apply"]
    classes = ["packed binary columns", "long binary, general, empty, long bounded-integer columns",
               "sorted general columns + row state"]
    n_kt = max(1.0, kt[5])
    ktm = [kt[0] / n_kt / 1e6, kt[1] / n_kt / 1e6, kt[2] / n_kt / 1e6, 0.0, kt[3] / n_kt / 1e6]

    # CUDA-event timing of the same kernels (event-record nodes between them in a captured graph,
    # same walker state continuing): a conservative cross-check, inflated by the event nodes
    kms = ws.profile(args.profile_iters)
    # batched model: A and the static per-variable data once per pass of the W
    # walkers, the walker state (x̄, tabu expiry, row state) once per walker
    mw_ = [int(info.model_bytes_walker_kernel[i]) for i in range(3)]
    mb = [int(info.model_bytes_kernel[i]) + (W - 1) * mw_[i] for i in range(3)]
    # the eval kernels' device time: first eval kernel start to the apply kernel's start
    eval_ms = float((kt[4] - kt[3]) / n_kt / 1e6)
    eval_ms_events = float(kms[0] + kms[1] + kms[2])
    eval_bytes = mb[0] + mb[1] + mb[2]
    achieved = eval_bytes / (eval_ms * 1e-3) / 1e9
    peak, peak_kind = measured_peak_hbm()
    traffic = None
    winstr = {}
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf):
        try:
            tj = json.load(open(tf))
            if tj.get("config") == cfg:
                traffic = tj.get("dram_bytes_per_launch")
                winstr = tj.get("warp_instructions_per_launch", {}) or {}
        except Exception:
            traffic = None
    step_ms_profiled = float(kt[4] / n_kt / 1e6)
    pass_bytes = int(info.model_bytes_pass) + (W - 1) * sum(mw_)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic,
                "kernel": "the best-shift pass of every variable + select: binary columns (k_eval_binrow "
                          "row-wise, long ones k_eval_bin), k_eval_gen, then k_eval",
                "model": "SURVEY 8(d): 12 B per original nonzero and cutoff entry + 4 B col_ptr per var + static "
                         "per var (1 B binary / 17 B other) + walker state (x̄ 1 bit / 8 B, 4 B tabu per var, "
                         "12 B per normalised row)",
                "peak_kind": peak_kind, "algorithmic_bytes_per_launch": eval_bytes,
                "timing": "per-kernel first-block-start to last-block-end (%globaltimer) inside the timed "
                          "region's CUDA graphs, averaged over its iterations (chap_walkers_timing)",
                "kernel_ms": {names[i]: float(ktm[i]) for i in (0, 1, 2, 4)},
                "model_bytes_by_class": {classes[i]: mb[i] for i in (0, 1, 2)},
                "kernel_share_of_step": eval_ms / step_ms_profiled if step_ms_profiled > 0 else None,
                "events": {"kernel_ms": {names[i]: float(kms[i]) for i in (0, 1, 2, 4)},
                           "achieved": eval_bytes / (eval_ms_events * 1e-3) / 1e9,
                           "frac": eval_bytes / (eval_ms_events * 1e-3) / 1e9 / peak,
                           "how": "CUDA-event pairs around each kernel node of a captured graph "
                                  f"({args.profile_iters} iterations right after the timed region)"},
                # the dominant kernel is issue-bound, not bandwidth-bound: its warp instructions per
                # launch (ncu capture of the same configuration, profiles/traffic.json) over its
                # in-graph time, against the issue peak 148 SMs x 4 schedulers x the SM clock
                "issue": ({"kernel": "k_eval_gen", "bound": "issue",
                           "warp_instructions_per_launch": winstr["k_eval_gen"],
                           "achieved": winstr["k_eval_gen"] / (ktm[1] * 1e-3),
                           "peak": 148 * 4 * 1.965e9, "unit": "warp instructions/s",
                           "frac": winstr["k_eval_gen"] / (ktm[1] * 1e-3) / (148 * 4 * 1.965e9)}
                          if winstr.get("k_eval_gen") and ktm[1] > 0 else None),
                "whole_step": {"model_bytes": pass_bytes, "ms": ms_max / args.steps,
                               "achieved": pass_bytes / (ms_max / args.steps * 1e-3) / 1e9,
                               "frac": pass_bytes / (ms_max / args.steps * 1e-3) / 1e9 / peak}}

    # e2e: the public C-ABI call with HOST buffers (page-locked), copies inside the timed region
    def pinned(nel, dt):
        return torch.empty(nel, dtype=dt, pin_memory=True).numpy()
    xh = pinned(inst.n, torch.float64)
    xh[:] = start_points(inst, cfg, 1, rank)[0]
    wh = pinned(P.m_norm, torch.float32)
    wh[:] = 1.0
    outs = (pinned(inst.n, torch.float64), pinned(inst.n, torch.float64))
    cut_rhs = math.inf
    if z_star is not None:   # the same active cutoff: rhs = z* - delta (R14)
        dlt = float(info.auto_cutoff_delta)
        cut_rhs = z_star - (dlt if math.isfinite(dlt) else 1e-6 * max(1.0, abs(z_star)))
    def e2e_time(full):
        kw = {"out": outs} if full else {"outputs": False}
        P.eval_best_shift_host(xh, wh, cut_rhs, **kw)
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_iters):
            P.eval_best_shift_host(xh, wh, cut_rhs, **kw)
        e2e_s = time.perf_counter() - t0
        et = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        return float(et.item())
    # the step's result is the best move (what a tabu iteration consumes); the per-variable outputs
    # (x̂, s: 16 bytes per variable back over PCIe) are timed alongside
    e2e_s, full_s = e2e_time(False), e2e_time(True)
    e2e = {"value": n_eval * args.e2e_iters * world / e2e_s, "unit": UNIT,
           "h2d_bytes_per_step": 8 * info.n + 4 * P.m_norm, "d2h_bytes_per_step": 24,
           "call": "chap_eval_best_shift_host (x, w in; the best move out; page-locked host buffers; synchronous)",
           "with_per_variable_outputs": {"value": n_eval * args.e2e_iters * world / full_s,
                                         "d2h_bytes_per_step": 16 * info.n + 24}}

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = oracle_baseline(inst, start_points(inst, cfg, 1, 0)[0])

    launches_per_iter = ws.launches_per_iter()   # [k_eval_bin], [k_eval_binrow], [k_eval_gen], k_eval, k_apply
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded generator synth/, no dataset or weights)",
                "config": config_dict(cfg, inst, W, world, z_star),
                "workload_detail": {"m_norm": P.m_norm, "nnz_norm_with_cutoff": int(info.nnz_norm + info.nnz_cut),
                           "non_fixed_vars": n_eval, "exchanges_in_timed_region": n_exchanges},
                "tabu_iters_per_s": W * args.steps * world / sec,
                # nonzeros visited per second (every nonzero incl. cutoff-row entries, per walker)
                "nnz_visits_per_s": float(info.nnz_norm + info.nnz_cut) * W * args.steps * world / sec,
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches_per_iter * args.steps + 4 + EXCHANGE_KERNELS * n_exchanges,
                "clocks": clk.summary(),
                "walker": {"moves": int(st["n_moves"].sum()), "stuck": int(st["n_stuck"].sum()),
                           "has_incumbent": int(st["has_incumbent"].sum()),
                           "best_obj": float(np.min(st["best_obj"])), "violated": int(st["violated"].min())}}
        print(json.dumps(line), flush=True)
    ws.close()
    if comm is not None:
        comm.close()
    P.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
