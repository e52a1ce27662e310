"""Generate the golden fixtures under tests/golden/ from the REAL reference.

Runs oracle/_ref/ref_driver (the unmodified reference headers compiled in place by
oracle/Makefile) and records its outputs.  Run here, where /root/reference exists:

    make -C oracle ref && python tests/golden/make_golden.py

The fixtures travel with the repo; nothing at test time reads /root/reference.
"""
from __future__ import annotations

import itertools
import json
import os
import random
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
DRIVER = os.path.join(ROOT, "oracle", "_ref", "ref_driver")


def ref(*args: str, timeout: float = 600) -> dict:
    out = subprocess.run([DRIVER, *args], capture_output=True, text=True, timeout=timeout)
    if out.returncode not in (0, 3):
        raise RuntimeError(f"{args}: {out.stderr}")
    d = json.loads(out.stdout)
    d.pop("times", None)
    d["args"] = list(args)
    return d


def dump(name: str, obj) -> None:
    path = os.path.join(HERE, name)
    with open(path, "w") as f:
        json.dump(obj, f, separators=(",", ":"))
    print(f"wrote {path} ({os.path.getsize(path)} bytes)", flush=True)


def configs() -> None:
    out = {}
    for c in ["cfg1", "cfg2", "cfg3", "cfg4"]:
        out[c] = {"solve": ref(c, "solve"), "options": ref(c, "options")}
        out[c]["solve_noprune_nocache"] = ref(c, "solve", "noprune", "nocache")
    out["cfg1"]["oracle"] = ref("cfg1", "oracle")
    out["cfg2"]["oracle"] = ref("cfg2", "oracle")
    out["cfg5"] = {"options": ref("cfg5", "options")}
    dump("configs.json", out)


def cfg5_stages() -> None:
    """Per-mask stage_eval parity on cfg5 for every mask the CPU finishes quickly."""
    out = []
    enc = list(range(7))
    for k in (1, 2, 3):
        for c in itertools.combinations(enc, k):
            mask = sum(1 << i for i in c)
            out.append(ref("cfg5", "stage", str(mask)))
    out.append(ref("cfg5", "stage", str(1 << 7)))  # backbone alone
    for mask in (15, 0b1010101, 0b1110000):
        out.append(ref("cfg5", "stage", str(mask), timeout=1200))
    feas = []
    for mask in (7, 15):
        for tau in ("0.0851", "0.0852", "0.0896", "0.09", "0.1", "0.2"):
            feas.append(ref("cfg5", "feas", str(mask), tau))
    dump("cfg5_stages.json", {"stage": out, "feas": feas})


def random_sets() -> None:
    # acceptance.cpp:94-120 (C2): stage_eval vs exhaustive at L=2
    c2 = []
    for seed in range(1, 201):
        n = 1 + seed % 3
        g = 2 if n >= 2 else 1
        inst = f"random:{seed}:{n}:{g}"
        mask = str((1 << n) - 1)
        c2.append({"stage": ref(inst, "stage", mask, "levels=2"),
                   "exact": ref(inst, "exact", mask, "levels=2")})
    # test_stage_eval.cpp:113-127: 60 seeds, 3 modules, 2 GPUs, L=4
    se = []
    for seed in range(1, 61):
        inst = f"random:{seed}:3:2"
        se.append({"stage": ref(inst, "stage", "7", "levels=4"),
                   "exact": ref(inst, "exact", "7", "levels=4")})
    # acceptance.cpp:57-90 (C1): solve vs oracle, 4 GPUs, L=4
    c1 = []
    for seed in range(1, 101):
        n = 2 + seed % 3
        inst = f"random:{seed}:{n}:4"
        c1.append({"solve": ref(inst, "solve", "levels=4"),
                   "oracle": ref(inst, "oracle", "levels=4")})
    c1b = []
    for seed in range(1, 21):
        inst = f"random:{seed}:6:4"
        c1b.append({"solve": ref(inst, "solve", "levels=4"),
                    "oracle": ref(inst, "oracle", "levels=4")})
    # larger random stages (G=8..32, L=10) for exact/stage parity
    big = []
    for seed in range(1, 41):
        n = 2 + seed % 3
        g = [8, 16, 32][seed % 3]
        inst = f"random:{seed}:{n}:{g}"
        mask = str((1 << n) - 1)
        big.append({"stage": ref(inst, "stage", mask),
                    "exact": ref(inst, "exact", mask) if n <= 3 and g <= 8 else None})
    dump("random_sets.json", {"c2": c2, "stage_eval_60": se, "c1": c1, "c1_6mod": c1b,
                              "big": big})


def stime_edge() -> None:
    """K1 edge cases against the reference's stage_time: dp degrees off the profiled d grid
    (log2 interpolation), any quota unit, duplicate modules (StageAllocation::find takes the
    first entry), repeated and unsorted GPU ids, negative coefficients."""
    rng = random.Random(777)
    out, all_cases = [], []
    for inst, n, g, L in [("cfg5", 8, 128, 32), ("cfg3", 4, 32, 10), ("random:3:6:24", 6, 24, 10)]:
        cases = []
        for t in range(40):
            k = rng.randint(1, min(n + 2, 10))
            mods = [rng.randrange(n) for _ in range(k)]
            if t % 2 == 0:
                mods = sorted(set(mods))
            ents = []
            for m in mods:
                d = rng.randint(1, g)
                u = rng.randint(1, L)
                gp = rng.sample(range(g), d)
                if t % 3 == 0:
                    gp = sorted(gp)
                if t % 5 == 0 and gp:
                    gp.append(gp[0])  # a repeated GPU id
                ents.append((m, d, u, gp))
            cases.append(ents)
        all_cases += [(inst, c) for c in cases]
    # lazy range errors: an out-of-hull option (a = 1/32 < 0.1) on a duplicate entry is
    # never looked up unless that entry is counted as a resident on a self entry's GPU
    lo = list(range(8))
    cases_cfg5 = [[(0, 8, 16, lo), (0, 4, 1, [100, 101, 102, 103])],
                  [(0, 8, 16, lo), (0, 4, 1, [4, 5, 6, 7])],
                  [(0, 8, 16, lo), (1, 4, 1, [4, 5, 6, 7])],
                  [(0, 8, 16, lo), (1, 4, 8, [4, 5, 6, 7]), (0, 2, 1, [120, 7])]]
    for inst, ents in [("cfg5", c) for c in cases_cfg5] + all_cases:
        spec = ";".join(f"{m}:{d}:{u}:{'.'.join(map(str, gp))}" for m, d, u, gp in ents)
        for extra in ([], ["noself"], ["additive"], ["e=1e-3,-2e-4,5e-4"],
                      ["noself", "e=1e-3,-2e-4,5e-4"]):
            r = ref(inst, "stime", spec, *extra)
            out.append({"inst": inst, "extra": extra, "entries": ents, "t": r.get("t")})
    dump("stime_edge.json", out)


def stime_large_g() -> None:
    """K1 on clusters beyond 128 GPUs (the shared-atomics path of k_evaluate): random
    allocations of random instances at G = 256, 512, 1024, scored by the reference."""
    rng = random.Random(4242)
    out = []
    for inst, n, g in [("random:5:4:256", 4, 256), ("random:6:5:512", 5, 512),
                       ("random:7:3:1024", 3, 1024)]:
        opts = ref(inst, "options")["modules"]
        for t in range(30):
            k = rng.randint(1, n)
            mods = sorted(rng.sample(range(n), k))
            ents = []
            for m in mods:
                rows = opts[m]["rows"]
                d, u = rows[rng.randrange(len(rows))][:2]
                gp = sorted(rng.sample(range(g), d))
                ents.append((m, d, u, gp))
            spec = ";".join(f"{m}:{d}:{u}:{'.'.join(map(str, gp))}" for m, d, u, gp in ents)
            for extra in ([], ["noself"]):
                r = ref(inst, "stime", spec, *extra)
                out.append({"inst": inst, "extra": extra, "entries": ents, "t": r.get("t")})
    dump("stime_large_g.json", out)


def large_clusters() -> None:
    """stage_eval (and solve where the CPU finishes in 120 s) beyond 128 GPUs: random
    instances at G = 256 and 512 (blocks stay <= 128 per level for these stages)."""
    out = []
    for inst, n in [("random:5:4:256", 4), ("random:9:3:512", 3)]:
        for mask in range(1, 1 << n):
            if bin(mask).count("1") > 2:
                continue
            try:
                out.append(ref(inst, "stage", str(mask), timeout=120))
            except subprocess.TimeoutExpired:
                pass
        try:
            out.append(ref(inst, "solve", timeout=120))
        except subprocess.TimeoutExpired:
            pass
    dump("large_clusters.json", out)


def random_solves() -> None:
    """Full GAHC solves of medium random instances (4-6 modules, 16-64 GPUs, L=10): the
    regime where device searches use shared walkers and GAHC rounds are batched.  Instances
    the CPU cannot solve in 60 s are skipped."""
    import concurrent.futures as cf
    jobs = []
    for seed in range(1, 61):
        n = 4 + seed % 3
        g = [16, 32, 64][(seed // 3) % 3]
        jobs.append(f"random:{seed}:{n}:{g}")

    def run(inst):
        try:
            return ref(inst, "solve", timeout=60)
        except subprocess.TimeoutExpired:
            return None
    with cf.ThreadPoolExecutor(2) as ex:
        out = [r for r in ex.map(run, jobs) if r is not None]
    dump("random_solves.json", out)


def exact_negative() -> None:
    """ExactStageSolver with negative interference coefficients: its option cut
    (oracle.hpp:127-139) is not a bound there, so its answer depends on the sequential DFS —
    every module set of small instances, two negative models."""
    out = []
    for inst, n in [("cfg1", 2), ("random:11:4:8", 4), ("cfg2", 3)]:
        for extra in (["e=1e-3,-2e-4,5e-4"], ["e=2e-3,1e-3,-4e-4"], ["e=-1e-4,3e-4,2e-4"]):
            for mask in range(1, 1 << n):
                try:  # the cut is weak for these models: sets the CPU cannot finish are skipped
                    r = ref(inst, "exact", str(mask), "levels=4", *extra, timeout=20)
                except subprocess.TimeoutExpired:
                    continue
                out.append({"inst": inst, "extra": extra, "mask": mask, "r": r})
    dump("exact_negative.json", out)


def presets() -> None:
    # acceptance.cpp:171-198 (C5): all presets at 8 GPUs, with and without prune+cache
    out = []
    for name, count in [("clip", 3), ("qwen3vl", 3), ("unifiedio2", 4), ("imagebind", 7),
                        ("ofasys", 10)]:
        inst = f"preset:{name}:{count}:8"
        out.append({"solve": ref(inst, "solve"),
                    "solve_noprune_nocache": ref(inst, "solve", "noprune", "nocache")})
    # ofasys-8 at G=32, L=32: cfg5 shape at a CPU-finishable size
    out.append({"solve": ref("preset:ofasys:8:32", "solve", "levels=32", timeout=1800)})
    dump("presets.json", out)


def variants() -> None:
    """Model variants the reference tests exercise: include_self=false, additive-only,
    negative coefficients, tight memory, infeasible modules."""
    out = []
    for seed in range(1, 16):
        inst = f"random:{seed}:3:4"
        for extra in (["noself"], ["additive"], ["e=0.4e-3,1.2e-3,0"],
                      ["e=1e-3,-2e-4,5e-4"], ["mem=20e9"], ["mem=6e9"]):
            row = {"extra": extra,
                   "stage": ref(inst, "stage", "7", "levels=4", *extra),
                   "exact": ref(inst, "exact", "7", "levels=4", *extra),
                   "solve": ref(inst, "solve", "levels=4", *extra)}
            out.append(row)
    dump("variants.json", out)


def stime() -> None:
    """K1 evaluator parity: random explicit allocations scored by the reference."""
    rng = random.Random(12345)
    out = []
    for inst, n, g, L in [("cfg4", 6, 64, 10), ("cfg5", 8, 128, 32), ("random:7:5:16", 5, 16, 10),
                          ("random:11:4:8", 4, 8, 10)]:
        opts = ref(inst, "options")["modules"]
        for t in range(60):
            k = rng.randint(1, n)
            mods = sorted(rng.sample(range(n), k))
            ents = []
            for m in mods:
                rows = opts[m]["rows"]
                d, u = rows[rng.randrange(len(rows))][:2]
                gp = sorted(rng.sample(range(g), d))
                ents.append((m, d, u, gp))
            spec = ";".join(f"{m}:{d}:{u}:{'.'.join(map(str, gp))}" for m, d, u, gp in ents)
            for extra in ([], ["noself"], ["additive"]):
                r = ref(inst, "stime", spec, *extra)
                out.append({"inst": inst, "extra": extra, "entries": ents, "t": r["t"]})
    dump("stime.json", out)




def io_files() -> None:
    """Reference JSON v1 files (io.hpp) and the plan solve() writes, for the N3 loaders."""
    out = {}
    for inst, extra in [("cfg3", []), ("cfg4", []), ("random:7:5:16", []),
                        ("preset:ofasys:8:32", ["levels=32"])]:
        d = ref(inst, "json", *extra)
        out[inst] = {"args": [inst, "json", *extra], "files": d["files"]}
    dump("io_files.json", out)


def _plan_spec(stages) -> str:
    return "|".join(";".join(f"{m}:{d}:{u}:{'.'.join(map(str, gp))}" for m, d, u, gp in st)
                    for st in stages)


def _mutate(stages, rng: random.Random, n: int, g: int, L: int):
    st = [[list(e) for e in s] for s in stages]
    kind = rng.choice(["none", "drop", "dup", "swap", "units", "dp", "gpu_oob", "coloc",
                       "empty", "merge", "big", "neg_module", "memstack"])
    flat = [(i, j) for i, s in enumerate(st) for j in range(len(s))]
    i, j = rng.choice(flat)
    e = st[i][j]
    if kind == "drop":
        del st[i][j]
        st = [s for s in st if s] or [[]]
    elif kind == "dup":
        st[rng.randrange(len(st))].append(list(e))
    elif kind == "swap" and len(st) > 1:
        a, b = rng.sample(range(len(st)), 2)
        st[a], st[b] = st[b], st[a]
    elif kind == "units":
        e[2] = min(L, e[2] + rng.randint(1, L))
    elif kind == "dp":
        e[1] = e[1] + 1
    elif kind == "gpu_oob":
        e[3] = e[3][:-1] + [g + rng.randint(0, 3)]
    elif kind == "coloc" and e[1] >= 2:
        e[3] = [e[3][0]] * 2 + e[3][2:]
    elif kind == "empty":
        st.insert(rng.randrange(len(st) + 1), [])
    elif kind == "merge":
        st = [[x for s in st for x in s]]
    elif kind == "big":
        e[2] = L
        st[i] = [x for x in st[i]] + [[m, e[1], L, e[3]] for m in range(n)
                                     if all(y[0] != m for s in st for y in s)]
    elif kind == "memstack":  # every replica on GPU 0 at d=1, u=1: memory, not quota
        st = [[[x[0], 1, 1, [0]] for x in s] for s in st]
    elif kind == "neg_module":
        e[0] = rng.choice([-1, n])
    return kind, st


def _mutate_kind(stages, kind):
    return kind, [[[x[0], 1, 1, [0]] for x in s] for s in stages]


def validate() -> None:
    """H15 validate_plan verdicts of the reference on solved plans and fuzzed mutations."""
    rng = random.Random(2605)
    out = []
    insts = [("cfg1", 2, 8, 10, []), ("cfg2", 4, 8, 10, []), ("cfg3", 4, 16, 10, []),
             ("cfg4", 6, 64, 10, [])]
    for seed in range(1, 13):
        for extra in ([], ["mem=20e9"], ["mem=6e9"], ["mem=3e9"]):
            insts.append((f"random:{seed}:{2 + seed % 4}:4", 2 + seed % 4, 4, 4,
                          ["levels=4", *extra]))
    for inst, n, g, L, extra in insts:
        sol = ref(inst, "solve", *extra)
        if "stages" not in sol:
            continue
        g, L = sol["gpus"], sol["levels"]
        base = [[(a["m"], a["d"], a["u"], a["gpus"]) for a in s["alloc"]] for s in sol["stages"]]
        cases = [("none", base), _mutate_kind(base, "memstack")] + [
            _mutate(base, rng, n, g, L) for _ in range(12)]
        for kind, st in cases:
            spec = _plan_spec(st)
            r = ref(inst, "validate", spec, *extra)
            out.append({"inst": inst, "extra": extra, "kind": kind,
                        "stages": [[list(x) for x in s] for s in st],
                        "code": r.get("code"), "exception": r.get("exception")})
    dump("validate.json", out)


def simulate() -> None:
    """N4: make_baseline_plan (Megatron / DistMM) and simulate() of the reference."""
    out = []
    insts = [("cfg1", []), ("cfg2", []), ("cfg3", []), ("cfg4", []),
             ("preset:imagebind:7:8", []), ("preset:ofasys:10:16", []),
             ("random:3:4:32", ["levels=8"]), ("random:7:5:16", ["mem=6e9"])]
    # 12 modules on 16 GPUs: dependency waves wider than 8 take the greedy branch (no solve:
    # the reference GAHC is too slow there)
    insts += [(f"random:{sd}:12:16", ["nosolve"]) for sd in (1, 2, 3, 4, 5, 6)]
    for inst, extra in insts:
        nosolve = "nosolve" in extra
        extra = [x for x in extra if x != "nosolve"]
        for pol in ("megatron", "distmm"):
            out.append({"inst": inst, "extra": extra, "op": "baseline", "policy": pol,
                        "r": ref(inst, "baseline", pol, *extra)})
        for which, cfg in [("solve", []), ("solve", ["iters=5", "sigma=0.1", "seed=11"]),
                           ("megatron", ["ondemand", "iters=2"]),
                           ("distmm", ["iters=3", "sigma=0.05", "seed=9"]),
                           ("solve", ["iters=7", "sigma=0.3", "seed=123456789", "ondemand"])]:
            if nosolve and which == "solve":
                continue
            out.append({"inst": inst, "extra": extra, "op": "simulate", "policy": which,
                        "cfg": cfg, "r": ref(inst, "simulate", which, *cfg, *extra)})
    dump("simulate.json", out)
    dump("normals.json", [ref("cfg1", "normals", str(sd), "400")
                          for sd in (0, 7, 11, 123456789, 2**64 - 1)])


if __name__ == "__main__":
    which = sys.argv[1:] or ["configs", "cfg5_stages", "random_sets", "presets", "variants",
                             "stime", "io_files", "validate", "simulate"]
    for w in which:
        globals()[w]()
