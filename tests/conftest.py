import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def hexf(s):
    return float.fromhex(s)


def alloc_tuples(alloc):
    """golden alloc list -> [(module, d, units, gpus)]"""
    return [(e["m"], e["d"], e["u"], list(e["gpus"])) for e in alloc]


def result_tuples(res):
    return [(e.module, e.option.dp_degree, e.option.quota_units, list(e.gpus))
            for e in res.allocation.entries]
