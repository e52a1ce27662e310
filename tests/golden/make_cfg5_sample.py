"""The identical-work sample bench.py times on BOTH arms (like-for-like ratio).

Sample: the stage_eval calls of the cfg5 GAHC solve (solver.hpp:157-289) that the reference
finishes in seconds — every EvalCache entry of the GPU trajectory (tests/golden/
trajectory_gpu.json) with k <= 4 modules, in cache (= call) order, cold cache.  For each
mask the instrumented reference (oracle/_ref/ref_driver_instr: the unmodified headers with a
counter on verify_complete, stage_eval.hpp:254) records its complete-allocation count
("plans" in the reference's own sense), its result and its single-core time here.  Both
arms report value = sum(leaves) / their time, so the ratio of the two values is the ratio
of times on identical work.

    make -C oracle ref && python tests/golden/make_cfg5_sample.py
"""
from __future__ import annotations

import json
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
DRIVER = os.path.join(ROOT, "oracle", "_ref", "ref_driver_instr")
MAX_K = 4


def sample_masks() -> list[int]:
    with open(os.path.join(HERE, "trajectory_gpu.json")) as f:
        traj = json.load(f)["cfg5@L32"]
    return [c["mask"] for c in traj["cache"] if c["k"] <= MAX_K]


def main() -> None:
    out = []
    for m in sample_masks():
        p = subprocess.run([DRIVER, "cfg5", "stage", str(m)], capture_output=True, text=True,
                           check=True)
        d = json.loads(p.stdout)
        out.append({"mask": m, "k": bin(m).count("1"), "leaves": d["leaves"], "t": d["t"],
                    "feasibility_calls": d["feasibility_calls"], "cpu_s": d["times"][0]})
        print(out[-1], flush=True)
    with open(os.path.join(HERE, "cfg5_sample.json"), "w") as f:
        json.dump({"spec": "cfg5", "max_k": MAX_K, "masks": out,
                   "leaves": sum(x["leaves"] for x in out),
                   "cpu_s": sum(x["cpu_s"] for x in out)}, f, indent=0)


if __name__ == "__main__":
    main()
