"""Shared helpers for the cfg5 trajectory pinning tests (tests/golden/make_cfg5_trajectory.py):
the reference records streamed into tests/golden/trajectory_ref.jsonl and the GPU trajectory
tests/golden/trajectory_gpu.json.  TEST INFRASTRUCTURE."""
import json
import os

from conftest import GOLDEN


def load_ref() -> dict:
    """key -> latest record (keys: SHAPE|stage|MASK, SHAPE|feas_last_ok|MASK, ...)."""
    out = {}
    path = os.path.join(GOLDEN, "trajectory_ref.jsonl")
    if os.path.exists(path):
        with open(path) as f:
            for line in f:
                d = json.loads(line)
                out[d["key"]] = d
    return out


def load_gpu() -> dict:
    with open(os.path.join(GOLDEN, "trajectory_gpu.json")) as f:
        return json.load(f)


def done(rec) -> bool:
    return rec is not None and rec.get("rc") == 0 and "out" in rec


def bits(m: int) -> list:
    return [i for i in range(64) if m >> i & 1]
