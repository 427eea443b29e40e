"""Experiment: per-kernel device times (chap_walkers_profile) of alternative builds of libchap.
Usage: python tools/variant_time.py CFG lib1.so [lib2.so ...]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_05086_b200 as chap  # noqa: E402
import synth  # noqa: E402

cfg, _, nw = sys.argv[1].partition(":")   # CFG[:walkers]
W = int(nw) if nw else 1
inst = {"G": synth.mixed, "S": synth.setcover, "P": synth.packing,
        "Gbin": lambda: synth.mixed(p_binary=1.0, p_bounded=0.0),
        "Gint": lambda: synth.mixed(p_binary=0.0, p_bounded=1.0),
        "Gnl": lambda: synth.mixed(n_long=0)}[cfg]()
X0 = np.stack([synth.x_lower(inst)] + [synth.x_random(inst, s) for s in range(1, W)])
orig = chap._lib
for path in sys.argv[2:]:
    lib = ctypes.CDLL(os.path.abspath(path))
    for name in chap.EXPORTED:
        f = getattr(lib, name)
        f.restype, f.argtypes = getattr(orig, name).restype, getattr(orig, name).argtypes
        setattr(chap, name, f)
    chap._lib = lib
    P = chap.Problem.from_instance(inst)
    ws = chap.Walkers(P, torch.from_numpy(X0).cuda(), chap.default_params(graph_iters=0))
    ws.step(20)
    torch.cuda.synchronize()
    k = ws.profile(200)
    print(os.path.basename(path), "bin %.4f gen %.4f eval %.4f apply %.4f" % (k[0], k[1], k[2], k[4]), flush=True)
    ws.close()
    P.close()
