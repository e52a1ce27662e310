"""Sharded search end to end: two ranks on one GPU (--same-device), gloo
all-gather once per device search.  Every rank must replay the same control flow, so each
merged search result has to be identical on all ranks (a divergence deadlocks the
all-gather); the plan must equal the single-GPU / reference plan bit for bit."""
import json
import os
import subprocess
import sys

import pytest

from conftest import hexf, load_golden

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("workload,port", [("cfg3", 29561), ("cfg4", 29562)])
def test_two_ranks_same_plan(workload, port):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--workload",
           workload, "--steps", "1", "--warmup", "3", "--dist-backend", "gloo",
           "--same-device", "--no-cpu-baseline"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=240)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([x for x in out.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2
    gold = load_golden("configs.json")[workload]["solve"]
    assert line["best_plan_iteration_time"] == hexf(gold["iteration_time"])
