"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck): the eval API on the
tiny, mixed and sorted-class instances, tabu steps with the row-wise binary kernel forced (one
walker) and with walker groups (W = 6: row-state groups of 8) including the device exchange and
an epoch graph, the column-wise kernel forced.
Usage: compute-sanitizer --tool TOOL python tools/sanitize_run.py [T|S|M]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_05086_b200 as chap  # noqa: E402
import synth  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "M"
if which == "T":
    inst = synth.tiny(0)
elif which == "S":
    inst = synth.setcover(n=5000, m=1000)
else:
    inst = synth.mixed(seed=7, n=6000, m=6000, n_long=6, long_lo=100, long_hi=5000,
                       long_kinds=("unb", "big", "bkt", "bin"))
P = chap.Problem.from_instance(inst)
x = synth.x_random(inst, 1)
w = synth.weights_random(P.m_norm, 1)
xhat, score, best = P.eval_best_shift(torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda())
torch.cuda.synchronize()
for bk in (2, 1):   # row-wise forced, column-wise forced
    Wk = chap.Walkers(P, torch.from_numpy(synth.x_lower(inst)[None, :]).cuda(),
                      chap.default_params(graph_iters=4, binary_kernel=bk))
    Wk.step(10)
    torch.cuda.synchronize()
    Wk.close()
X0 = np.stack([synth.x_random(inst, s) for s in range(6)])
Wk = chap.Walkers(P, torch.from_numpy(X0).cuda(), chap.default_params(graph_iters=4, n_elite=2, n_restart=3))
Wk.step(10)
Wk.exchange()          # the device exchange: plan, packing, cutoff, restarts
Wk.epoch(5)            # iterations + exchange as one captured graph, then replayed
Wk.epoch(5, result=True)
torch.cuda.synchronize()
print("sanitize workload done", which, inst.n, inst.m)
