"""GPU: bench.py's CUDA arm prints the contract's JSON line (the keys the driver reads), with the
timed region holding epoch graphs (exchange_K iterations + the device exchange) and the last epoch
as iteration graphs; config T with a few walkers so the run takes seconds."""
import json
import math
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no GPU", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cuda_arm_json_line_with_epochs():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "T", "--walkers", "4",
                          "--steps", "2500", "--warmup", "5", "--profile-iters", "20", "--e2e-iters", "3"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["steps"] == 2500 and d["warmup"] >= 3 and d["n_gpus"] == 1
    assert d["value"] > 0 and math.isfinite(d["ms_per_step"]) and d["ms_per_step"] > 0
    rf = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in rf, k
    assert 0 < rf["frac"] <= 1.0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["gpu_launches"] > 2500   # at least one kernel per iteration, plus the exchanges
    assert d["config"]["walkers_per_gpu"] == 4 and "workload" in d["config"]
