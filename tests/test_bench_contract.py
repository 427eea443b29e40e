"""CPU-only: bench.py's reference arm (the oracle, per the task's tier framing) prints one JSON line
with the contract's keys; the same keys the driver reads from the CUDA arm's line."""
import json
import os

import numpy as np
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "S",
                          "--steps", "1", "--warmup", "3"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["warmup"] >= 3
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert "workload" in d["config"]


def test_gpus_flag_launches_ranks():
    """`bench.py --gpus 2` without a torchrun environment re-launches itself with 2 ranks
    (torch.distributed.run, 127.0.0.1); rank 0 prints the one line, with WORLD_SIZE = 2 seen."""
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "T",
                          "--gpus", "2", "--steps", "2", "--warmup", "3"], capture_output=True, text=True,
                         timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["launcher"]["world_size"] == 2 and d["launcher"]["rank"] == 0


def test_start_points_distinct_per_rank():
    sys.path.insert(0, ROOT)
    import bench
    import synth
    inst = synth.mixed(seed=9, n=4000, m=800, n_long=4, long_lo=300, long_hi=3000)
    x = [bench.start_points(inst, "G", 1, r)[0] for r in range(4)]
    assert not any(np.array_equal(x[a], x[b]) for a in range(4) for b in range(a + 1, 4))
    assert all(np.all((xi >= inst.lb) & (xi <= inst.ub)) for xi in x)
