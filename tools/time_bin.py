"""Debug: per-stage clock64 totals of k_eval_bin (tools/libchap_timing.so, built with -DCHAP_TIMING)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_05086_b200 as chap  # noqa: E402
import synth  # noqa: E402

dbg = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libchap_timing.so"))
# swap the binding's library for the timing build
for name in chap.EXPORTED:
    f = getattr(dbg, name)
    f.restype, f.argtypes = getattr(chap._lib, name).restype, getattr(chap._lib, name).argtypes
    setattr(chap, name, f)
chap._lib = dbg
cfg = sys.argv[1] if len(sys.argv) > 1 else "G"
inst = {"G": synth.mixed, "Gbin": lambda: synth.mixed(p_binary=1.0, p_bounded=0.0)}[cfg]()
P = chap.Problem.from_instance(inst)
ws = chap.Walkers(P, torch.from_numpy(synth.x_lower(inst)[None, :]).cuda(), chap.default_params(graph_iters=0))
ws.step(20)
torch.cuda.synchronize()
out = (ctypes.c_ulonglong * 8)()
dbg.chap_debug_counters(out, 1)
ws.step(50)
torch.cuda.synchronize()
dbg.chap_debug_counters(out, 1)
v = list(out)
tiles = v[6]
names = ["stream issue + desc + cols", "mbar wait (stream i+1)", "gathers issue", "cp.async wait (gathers i)",
         "compute", "-"]
tot = sum(v[:5])
print("tiles", tiles, "per-tile cycles (lane0, summed over warps):")
for i in range(5):
    print(f"  {names[i]:28s} {v[i] / max(tiles, 1):10.1f} cycles/tile  {100 * v[i] / max(tot, 1):5.1f}%")
