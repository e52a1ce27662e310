"""ctypes wrapper of oracle/_ref/libmosaic_oracle.so (the plain-C restatement of the
reference planner, oracle/mosaic_oracle.c).  TEST INFRASTRUCTURE ONLY."""
from __future__ import annotations

import ctypes as C
import math
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(_HERE, "_ref", "libmosaic_oracle.so")


class Stage(C.Structure):
    _fields_ = [("status", C.c_int), ("stage_time", C.c_double), ("n_entries", C.c_int),
                ("ent", C.c_int * (64 * 4)), ("gpus", C.c_int * (64 * 1024)),
                ("probes", C.c_longlong)]


class Plan(C.Structure):
    _fields_ = [("status", C.c_int), ("n_stages", C.c_int), ("masks", C.c_uint64 * 64),
                ("times", C.c_double * 64), ("iteration_time", C.c_double),
                ("stage_eval_calls", C.c_longlong), ("feasibility_calls", C.c_longlong),
                ("partitions", C.c_longlong)]


_lib = None


def available() -> bool:
    return os.path.exists(LIB)


def lib():
    global _lib
    if _lib is None:
        if not available():
            import subprocess
            subprocess.check_call(["make", "-s", "-C", _HERE, "restatement"])
        L = C.CDLL(LIB)
        L.mo_synth.restype = C.c_void_p
        L.mo_synth.argtypes = [C.c_char_p, C.c_int]
        L.mo_free.argtypes = [C.c_void_p]
        L.mo_set_model.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_double, C.c_int,
                                   C.c_int, C.c_double]
        L.mo_set_solve_flags.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.mo_num_modules.argtypes = [C.c_void_p]
        L.mo_options.argtypes = [C.c_void_p, C.c_int] + [C.c_void_p] * 5
        L.mo_options.restype = C.c_int
        for f in (L.mo_stage_eval, L.mo_exact):
            f.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(Stage)]
        L.mo_feasible.argtypes = [C.c_void_p, C.c_uint64, C.c_double, C.POINTER(Stage)]
        L.mo_stage_time.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.mo_stage_time.restype = C.c_double
        for f in (L.mo_solve, L.mo_brute_force):
            f.argtypes = [C.c_void_p, C.POINTER(Plan)]
        L.mo_plan_stage.argtypes = [C.c_void_p, C.c_int, C.POINTER(Stage)]
        L.mo_normals.argtypes = [C.c_uint64, C.c_int, C.POINTER(C.c_double)]
        _lib = L
    return _lib


class Problem:
    def __init__(self, spec: str, levels: int = 0, extra=()):
        self.p = lib().mo_synth(spec.encode(), levels)
        if not self.p:
            raise ValueError(spec)
        e = [math.nan] * 3
        self_, add, mem = -1, -1, math.nan
        for x in extra:
            if x == "noself":
                self_ = 0
            elif x == "additive":
                add = 1
            elif x.startswith("e="):
                e = [float(v) for v in x[2:].split(",")]
            elif x.startswith("mem="):
                mem = float(x[4:])
        lib().mo_set_model(self.p, e[0], e[1], e[2], self_, add, mem)

    def __del__(self):
        if getattr(self, "p", None):
            lib().mo_free(self.p)
            self.p = None

    def set_flags(self, prune: bool, cache: bool):
        lib().mo_set_solve_flags(self.p, int(prune), int(cache))

    def options(self, m):
        n = lib().mo_options(self.p, m, None, None, None, None, None)
        d, u = (C.c_int * max(n, 1))(), (C.c_int * max(n, 1))()
        b, bw, fp = [(C.c_double * max(n, 1))() for _ in range(3)]
        lib().mo_options(self.p, m, d, u, b, bw, fp)
        return [(d[i], u[i], b[i], bw[i], fp[i]) for i in range(n)]

    @staticmethod
    def _stage(s: Stage):
        if s.status != 0:
            return {"status": s.status}
        ents, off = [], 0
        for e in range(s.n_entries):
            m, d, u, ng = s.ent[4 * e:4 * e + 4]
            ents.append((m, d, u, list(s.gpus[off:off + ng])))
            off += ng
        return {"status": 0, "stage_time": s.stage_time, "alloc": ents, "probes": s.probes}

    def stage_eval(self, mask):
        s = Stage()
        lib().mo_stage_eval(self.p, mask, C.byref(s))
        return self._stage(s)

    def exact(self, mask):
        s = Stage()
        lib().mo_exact(self.p, mask, C.byref(s))
        return self._stage(s)

    def feasible(self, mask, tau):
        s = Stage()
        lib().mo_feasible(self.p, mask, tau, C.byref(s))
        return self._stage(s)

    def stage_time(self, entries):
        ent, gp = [], []
        for m, d, u, g in entries:
            ent += [m, d, u, len(g)]
            gp += list(g)
        E = (C.c_int * max(1, len(ent)))(*ent)
        G = (C.c_int * max(1, len(gp)))(*gp)
        return lib().mo_stage_time(self.p, len(entries), E, G)

    def _plan(self, pl: Plan):
        if pl.status != 0:
            return {"status": pl.status}
        stages = []
        for i in range(pl.n_stages):
            s = Stage()
            lib().mo_plan_stage(self.p, i, C.byref(s))
            stages.append(self._stage(s))
        return {"status": 0, "iteration_time": pl.iteration_time,
                "masks": list(pl.masks[:pl.n_stages]), "times": list(pl.times[:pl.n_stages]),
                "stages": stages, "stage_eval_calls": pl.stage_eval_calls,
                "feasibility_calls": pl.feasibility_calls, "partitions": pl.partitions}

    def solve(self):
        pl = Plan()
        lib().mo_solve(self.p, C.byref(pl))
        return self._plan(pl)

    def brute_force(self):
        pl = Plan()
        lib().mo_brute_force(self.p, C.byref(pl))
        return self._plan(pl)


def stage_eval(spec: str, levels: int, modules) -> dict | None:
    r = Problem(spec, levels).stage_eval(sum(1 << m for m in modules))
    return r if r["status"] == 0 else None


def normals(seed: int, n: int) -> list[float]:
    """std::normal_distribution<double>(0,1) over std::mt19937_64(seed), restated in C."""
    out = (C.c_double * n)()
    lib().mo_normals(seed, n, out)
    return list(out)
