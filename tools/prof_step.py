"""Profiling driver (ncu target): config G, one walker, plain launches (no graph) so that ncu
sees individual k_eval / k_apply launches. Usage: python tools/prof_step.py [warmup] [iters] [cfg]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_05086_b200 as chap  # noqa: E402
import synth  # noqa: E402

warm = int(sys.argv[1]) if len(sys.argv) > 1 else 20
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 5
cfg = sys.argv[3] if len(sys.argv) > 3 else "G"
inst = {"G": synth.mixed, "S": synth.setcover, "P": synth.packing,
        "Gbin": lambda: synth.mixed(p_binary=1.0, p_bounded=0.0),
        "Gnl": lambda: synth.mixed(n_long=0), "Gint": lambda: synth.mixed(p_binary=0.0, p_bounded=1.0)}[cfg]()
P = chap.Problem.from_instance(inst)
W = int(sys.argv[4]) if len(sys.argv) > 4 else (64 if cfg == "P" else 1)
x0 = np.stack([synth.x_lower(inst)] * W) if cfg != "P" else \
    np.stack([synth.x_bernoulli(inst, (3, w), 0.5) for w in range(W)])
ws = chap.Walkers(P, torch.from_numpy(x0).cuda(), chap.default_params(graph_iters=0))
if getattr(inst, "x_star", None) is not None:   # as bench.py: the cutoff row active from the start
    ws.set_cutoff(float(inst.c @ inst.x_star))
ws.step(warm)
torch.cuda.synchronize()
ws.step(iters)
torch.cuda.synchronize()
print("info", P.info.n_long_columns, list(P.info.nnz_kernel), list(P.info.model_bytes_kernel))
