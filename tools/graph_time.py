"""Experiment: in-graph per-kernel device times (chap_walkers_timing, as bench.py's roofline) and the
step time by CUDA events of alternative builds of libchap, in the bench state (cutoff row active,
graph_iters 32). Libraries alternate for `rounds` rounds.
Usage: python tools/graph_time.py CFG[:walkers] iters rounds lib1.so [lib2.so ...]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_05086_b200 as chap  # noqa: E402

notiming = "--notiming" in sys.argv   # step time by events only, kernel timestamps off
argv = [a for a in sys.argv[1:] if not a.startswith("--param=") and a != "--notiming"]
params = [a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--param=")]   # --param=NAME=VALUE
cfg, _, nw = argv[0].partition(":")
W = int(nw) if nw else 1
iters = int(argv[1])
rounds = int(argv[2])
inst = bench.make_instance(cfg)
x0 = bench.start_points(inst, cfg, W, 0)
z = bench.planted_objective(inst)
orig = chap._lib
libs = []
for path in argv[3:]:
    lib = ctypes.CDLL(os.path.abspath(path))
    for name in chap.EXPORTED:
        f = getattr(lib, name)
        f.restype, f.argtypes = getattr(orig, name).restype, getattr(orig, name).argtypes
    libs.append((path, lib))


def use(lib):
    for name in chap.EXPORTED:
        setattr(chap, name, getattr(lib, name))
    chap._lib = lib


for r in range(rounds):
    for path, lib in libs:
        use(lib)
        P = chap.Problem.from_instance(inst)
        prm = chap.default_params(graph_iters=32)
        for kv in params:
            k, v = kv.split("=", 1)
            setattr(prm, k, type(getattr(prm, k))(float(v)) if isinstance(getattr(prm, k), float) else int(v))
        ws = chap.Walkers(P, torch.from_numpy(x0).cuda(), prm)
        if z is not None:
            ws.set_cutoff(z)
        if not notiming:
            ws.timing(1)
        ws.step(64)
        torch.cuda.synchronize()
        if not notiming:
            ws.timing(1)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        ws.step(iters)
        e1.record()
        torch.cuda.synchronize()
        kt = ws.timing(-1).astype(np.float64) if notiming else ws.timing(0).astype(np.float64)
        n = max(1.0, kt[5])
        print("%-14s step %.4f ms  bin %.4f gen %.4f eval %.4f apply %.4f  eval-span %.4f" % (
            os.path.basename(path), e0.elapsed_time(e1) / iters, kt[0] / n / 1e6, kt[1] / n / 1e6, kt[2] / n / 1e6,
            kt[3] / n / 1e6, (kt[4] - kt[3]) / n / 1e6), flush=True)
        ws.close()
        P.close()
