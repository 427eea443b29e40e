"""Per-kernel device time inside chap_tabu_step's CUDA graphs, from a -DCHAP_KTIMING build
(%globaltimer at the first block start / last block end of every kernel; no events).
Usage: python tools/ktime.py CFG path/to/libchap_ktiming.so [iters]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_05086_b200 as chap  # noqa: E402
import synth  # noqa: E402

cfg, path = sys.argv[1], sys.argv[2]
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 2048
lib = ctypes.CDLL(os.path.abspath(path))
for name in chap.EXPORTED:
    f = getattr(lib, name)
    f.restype, f.argtypes = getattr(chap._lib, name).restype, getattr(chap._lib, name).argtypes
    setattr(chap, name, f)
chap._lib = lib
inst = {"G": synth.mixed, "S": synth.setcover, "Gint": lambda: synth.mixed(p_binary=0.0, p_bounded=1.0),
        "Gbin": lambda: synth.mixed(p_binary=1.0, p_bounded=0.0)}[cfg]()
P = chap.Problem.from_instance(inst)
ws = chap.Walkers(P, torch.from_numpy(synth.x_lower(inst)[None, :]).cuda(), chap.default_params(graph_iters=32))
ws.step(64)
torch.cuda.synchronize()
out = (ctypes.c_ulonglong * 6)()
lib.chap_debug_ktimes(out, 1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
ws.step(iters)
e1.record()
torch.cuda.synchronize()
lib.chap_debug_ktimes(out, 0)
n = max(1, out[5])
names = ["k_eval_bin", "k_eval_gen", "k_eval", "k_apply"]
print(cfg, "iterations", out[5], "event ms/iter %.4f" % (e0.elapsed_time(e1) / iters))
for q in range(4):
    print(f"  {names[q]:12s} {out[q] / n / 1000:8.2f} us")
print(f"  {'span':12s} {out[4] / n / 1000:8.2f} us (first kernel start -> apply end)")
