"""Python mirror of the reference planner API over the C ABI (include/mosaic_gpu.h).

The reference is header-only C++ (namespace mosaic); this module keeps its names,
argument meaning and error behaviour so parity tests read like the reference's own
doctest suites:

    reference (C++)                                  here
    stage_eval(ctx, cluster, modules, cfg)           stage_eval(planner, modules)
    detail::ExactStageSolver(ctx, cluster, L).solve  exact_stage(planner, modules)
    detail::FeasibilitySearch(...).run(tau)          feasibility_run(planner, modules, tau)
    solve(ctx, cluster, cfg)                         solve(planner)
    brute_force_optimum(ctx, cluster, L)             brute_force_optimum(planner)
    stage_time / rectified_latency                   stage_time(planner, allocs)
    candidate_options(ctx, cluster, m, L)            candidate_options(planner, m)
    ScalingSurface::lookup                           planner.lookup(m, d, a)

`Planner` plays the role of PerfContext + ClusterSpec + SolveConfig (one device
context).  Every search runs in the CUDA library; if it is not built, importing
fails loudly — there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MOSAIC_LIB") or os.path.join(_HERE, "libmosaic_gpu.so")  # override: A/B runs

MAX_STAGE_MODULES = 12
MAX_GPUS = 1024
MAX_STAGES = 64
MAX_MODULES = 64

(OK, INFEASIBLE, MODULE_NO_OPTION, RANGE, TOO_LARGE, CUDA, EMPTY, BASELINE_INFEASIBLE,
 INVALID_ARGUMENT) = range(9)


class MosaicError(RuntimeError):
    pass


class StageInfeasibleError(MosaicError):
    """stage_eval.hpp:26 — a module has no feasible deployment option."""


class SurfaceRangeError(MosaicError):
    """perf_model.hpp:46 — query outside the profiled hull / invalid input."""


class OracleTooLargeError(MosaicError):
    """oracle.hpp:24 — more than 8 modules, or a stage beyond kernel limits."""


class EmptyPlanError(MosaicError):
    """solver.hpp:25."""


class InfeasibleBaselineError(MosaicError):
    """simulator.hpp:127-129 InfeasibleBaselineError."""


class InvalidArgumentError(MosaicError, ValueError):
    """std::invalid_argument (e.g. SimConfig checks, simulator.hpp:70-73)."""


class DeviceError(MosaicError):
    pass


# ---------------------------------------------------------------------------
# ctypes mirror of include/mosaic_gpu.h
# ---------------------------------------------------------------------------
class Point(C.Structure):
    _fields_ = [("d", C.c_int32), ("a", C.c_double), ("latency", C.c_double),
                ("bandwidth_util", C.c_double), ("memory", C.c_double), ("sm_active", C.c_double)]


class WorkloadC(C.Structure):
    _fields_ = [("id", C.c_char_p), ("flops_per_iter", C.c_double),
                ("bytes_per_iter", C.c_double), ("gradient_bytes", C.c_double),
                ("sm_efficiency_knee", C.c_double), ("memory_act_base", C.c_double),
                ("memory_per_quota", C.c_double), ("fixed_overhead", C.c_double),
                ("dp_penalty", C.c_double)]


class ClusterC(C.Structure):
    _fields_ = [("gpu_count", C.c_int32), ("memory_capacity", C.c_double),
                ("peak_compute", C.c_double), ("peak_bandwidth", C.c_double),
                ("interconnect_alpha", C.c_double), ("interconnect_beta", C.c_double)]


class SimConfigC(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("stream_mode", C.c_int32),
                ("pooled_overhead", C.c_double), ("on_demand_overhead", C.c_double),
                ("perturbation_sigma", C.c_double)]


class IntervalC(C.Structure):
    _fields_ = [("gpu", C.c_int32), ("module", C.c_int32), ("start", C.c_double),
                ("end", C.c_double), ("quota", C.c_double)]


class ModuleC(C.Structure):
    _fields_ = [("id", C.c_char_p), ("memory_base", C.c_double), ("points", C.POINTER(Point)),
                ("n_points", C.c_int32)]


class ProblemC(C.Structure):
    _fields_ = [("modules", C.POINTER(ModuleC)), ("n_modules", C.c_int32),
                ("edges", C.POINTER(C.c_int32)), ("n_edges", C.c_int32),
                ("gpu_count", C.c_int32), ("memory_capacity", C.c_double),
                ("e1", C.c_double), ("e2", C.c_double), ("e3", C.c_double),
                ("additive_only", C.c_int32), ("include_self", C.c_int32),
                ("quota_levels", C.c_int32), ("bisect_rel_tol", C.c_double),
                ("enable_prune", C.c_int32), ("enable_cache", C.c_int32)]


class EntryC(C.Structure):
    _fields_ = [("module", C.c_int32), ("dp_degree", C.c_int32), ("quota_units", C.c_int32),
                ("n_gpus", C.c_int32), ("gpus", C.c_int32 * MAX_GPUS)]


class StageResultC(C.Structure):
    _fields_ = [("status", C.c_int32), ("stage_time", C.c_double), ("n_entries", C.c_int32),
                ("entries", EntryC * MAX_STAGE_MODULES), ("probes", C.c_int64),
                ("gpu_searches", C.c_int64), ("nodes", C.c_int64), ("leaves", C.c_int64)]


class EvalEntryC(C.Structure):
    _fields_ = [("module", C.c_int32), ("dp_degree", C.c_int32), ("quota_units", C.c_int32),
                ("n_gpus", C.c_int32), ("quota_levels", C.c_int32), ("pad", C.c_int32),
                ("gpu_off", C.c_int64)]


class PlanResultC(C.Structure):
    _fields_ = [("status", C.c_int32), ("n_stages", C.c_int32),
                ("stage_mask", C.c_uint64 * MAX_STAGES), ("stage_time", C.c_double * MAX_STAGES),
                ("iteration_time", C.c_double), ("partitions_examined", C.c_int64),
                ("rounds", C.c_int64), ("stage_eval_calls", C.c_int64),
                ("feasibility_calls", C.c_int64), ("cache_hits", C.c_int64),
                ("prunes", C.c_int64), ("gpu_searches", C.c_int64), ("nodes", C.c_int64),
                ("leaves", C.c_int64), ("elapsed_s", C.c_double)]


ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t)

# every symbol include/mosaic_gpu.h declares (checked by the CPU tests)
EXPORTS = [
    "mosaic_gpu_create", "mosaic_gpu_destroy", "mosaic_gpu_last_error",
    "mosaic_gpu_num_options", "mosaic_gpu_options", "mosaic_gpu_lookup",
    "mosaic_gpu_stage_time", "mosaic_gpu_stage_eval", "mosaic_gpu_exact_stage",
    "mosaic_gpu_feasible", "mosaic_gpu_plan_stage", "mosaic_gpu_solve",
    "mosaic_gpu_brute_force", "mosaic_gpu_trace_rounds", "mosaic_gpu_trace_round",
    "mosaic_gpu_trace_cand", "mosaic_gpu_clear_cache", "mosaic_gpu_set_shard",
    "mosaic_gpu_rank_record_size", "mosaic_gpu_rank_record", "mosaic_gpu_merge_ranks",
    "mosaic_gpu_search", "mosaic_gpu_nccl_id", "mosaic_gpu_set_shard_nccl",
    "mosaic_gpu_launch_count", "mosaic_gpu_search_ms",
    "mosaic_gpu_reset_counters", "mosaic_gpu_synth_problem", "mosaic_gpu_free_problem",
    "mosaic_gpu_own_launches", "mosaic_gpu_ksearch_ms", "mosaic_gpu_ksearch_launches",
    "mosaic_gpu_h2d_bytes", "mosaic_gpu_d2h_bytes", "mosaic_gpu_mark", "mosaic_gpu_marked_ms", "mosaic_gpu_alg_bytes", "mosaic_gpu_stage_min",
    "mosaic_gpu_validate_plan", "mosaic_gpu_generate_surfaces", "mosaic_gpu_synth_workloads",
    "mosaic_gpu_baseline_plan", "mosaic_gpu_simulate",
    "mosaic_gpu_cache_masks", "mosaic_gpu_cache_entry", "mosaic_gpu_set_tuning",
    "mosaic_gpu_device_bytes", "mosaic_gpu_evaluate", "mosaic_gpu_evaluate_stats",
    "mosaic_gpu_evaluate_paths", "mosaic_gpu_peer_links", "mosaic_gpu_smem_peak",
]

_lib = None


def load_library(path: str = LIB_PATH) -> C.CDLL:
    """Load the CUDA library; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(path)
    P = C.POINTER
    vp = C.c_void_p
    sig = {
        "mosaic_gpu_create": (C.c_int, [P(ProblemC), C.c_int, P(vp)]),
        "mosaic_gpu_destroy": (None, [vp]),
        "mosaic_gpu_last_error": (C.c_char_p, []),
        "mosaic_gpu_num_options": (C.c_int, [vp, C.c_int, P(C.c_int32)]),
        "mosaic_gpu_options": (C.c_int, [vp, C.c_int, P(C.c_int32), P(C.c_int32), P(C.c_double),
                                         P(C.c_double), P(C.c_double)]),
        "mosaic_gpu_lookup": (C.c_int, [vp, C.c_int, C.c_int, C.c_double, P(C.c_double)]),
        "mosaic_gpu_stage_time": (C.c_int, [vp, P(EvalEntryC), P(C.c_int32), P(C.c_int64),
                                            C.c_int64, P(C.c_double), P(C.c_double)]),
        "mosaic_gpu_stage_eval": (C.c_int, [vp, C.c_uint64, P(StageResultC)]),
        "mosaic_gpu_exact_stage": (C.c_int, [vp, C.c_uint64, P(StageResultC)]),
        "mosaic_gpu_feasible": (C.c_int, [vp, C.c_uint64, C.c_double, P(StageResultC)]),
        "mosaic_gpu_plan_stage": (C.c_int, [vp, C.c_int, P(StageResultC)]),
        "mosaic_gpu_solve": (C.c_int, [vp, P(PlanResultC)]),
        "mosaic_gpu_brute_force": (C.c_int, [vp, P(PlanResultC)]),
        "mosaic_gpu_trace_rounds": (C.c_int, [vp, P(C.c_int64)]),
        "mosaic_gpu_trace_round": (C.c_int, [vp, C.c_int64, P(C.c_uint64), P(C.c_uint64),
                                             P(C.c_double), P(C.c_int64)]),
        "mosaic_gpu_trace_cand": (C.c_int, [vp, C.c_int64, C.c_int64, P(C.c_uint64),
                                            P(C.c_uint64), P(C.c_int32), P(C.c_int32),
                                            P(C.c_double)]),
        "mosaic_gpu_clear_cache": (None, [vp]),
        "mosaic_gpu_set_shard": (C.c_int, [vp, C.c_int, C.c_int, ALLGATHER_FN, vp]),
        "mosaic_gpu_rank_record_size": (C.c_size_t, []),
        "mosaic_gpu_nccl_id": (C.c_int, [vp, C.c_size_t]),
        "mosaic_gpu_set_shard_nccl": (C.c_int, [vp, C.c_int, C.c_int, vp]),
        "mosaic_gpu_rank_record": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int,
                                             P(C.c_uint16), P(C.c_uint16), P(C.c_uint16),
                                             C.c_double]),
        "mosaic_gpu_merge_ranks": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, P(C.c_int),
                                             P(C.c_int), P(C.c_double), P(C.c_int), P(C.c_int),
                                             P(C.c_double)]),
        "mosaic_gpu_search": (C.c_int, [vp, P(C.c_uint64), C.c_int64, C.c_int,
                                        P(StageResultC), P(C.c_double), P(C.c_int32)]),
        "mosaic_gpu_launch_count": (C.c_int64, [vp]),
        "mosaic_gpu_search_ms": (C.c_double, [vp]),
        "mosaic_gpu_reset_counters": (None, [vp]),
        "mosaic_gpu_synth_problem": (C.c_int, [C.c_char_p, C.c_int, P(P(ProblemC))]),
        "mosaic_gpu_free_problem": (None, [P(ProblemC)]),
        "mosaic_gpu_own_launches": (C.c_int64, [vp]),
        "mosaic_gpu_ksearch_ms": (C.c_double, [vp]),
        "mosaic_gpu_ksearch_launches": (C.c_int64, [vp]),
        "mosaic_gpu_h2d_bytes": (C.c_int64, [vp]),
        "mosaic_gpu_d2h_bytes": (C.c_int64, [vp]),
        "mosaic_gpu_mark": (None, [vp, C.c_int]),
        "mosaic_gpu_marked_ms": (C.c_double, [vp]),
        "mosaic_gpu_alg_bytes": (C.c_int64, [vp]),
        "mosaic_gpu_stage_min": (C.c_int, [vp, C.c_uint64, C.c_double, C.c_int,
                                           P(C.c_double), P(StageResultC)]),
        "mosaic_gpu_generate_surfaces": (C.c_int, [P(WorkloadC), C.c_int32, P(ClusterC),
                                                   P(C.c_int32), C.c_int32, P(C.c_double),
                                                   C.c_int32, C.c_double, C.c_int, P(Point),
                                                   P(C.c_int32), P(C.c_int32)]),
        "mosaic_gpu_synth_workloads": (C.c_int, [C.c_char_p, P(WorkloadC), C.c_int32,
                                                 P(C.c_int32), P(ClusterC)]),
        "mosaic_gpu_baseline_plan": (C.c_int, [vp, C.c_int, P(PlanResultC)]),
        "mosaic_gpu_simulate": (C.c_int, [vp, P(EvalEntryC), P(C.c_int32), P(C.c_int64),
                                          C.c_int64, P(SimConfigC), P(C.c_uint64), C.c_int64,
                                          P(C.c_double), P(C.c_double), P(C.c_double),
                                          P(C.c_double), P(IntervalC), C.c_int64,
                                          P(C.c_int64)]),
        "mosaic_gpu_validate_plan": (C.c_int, [vp, P(EvalEntryC), P(C.c_int32), P(C.c_int64),
                                               C.c_int64, C.c_char_p, C.c_size_t]),
        "mosaic_gpu_set_tuning": (C.c_int, [vp, C.c_char_p, C.c_double]),
        "mosaic_gpu_device_bytes": (C.c_int64, [vp]),
        "mosaic_gpu_evaluate": (C.c_int, [vp, vp, C.c_int64, vp, C.c_int64, vp, C.c_int64,
                                          vp, vp, C.c_uint32]),
        "mosaic_gpu_evaluate_paths": (C.c_int, [vp, P(C.c_double), P(C.c_int64)]),
        "mosaic_gpu_peer_links": (C.c_int, [vp]),
        "mosaic_gpu_smem_peak": (C.c_int, [C.c_int, P(C.c_double)]),
        "mosaic_gpu_evaluate_stats": (C.c_int, [vp, P(C.c_double), P(C.c_int64),
                                                P(C.c_int64)]),
        "mosaic_gpu_cache_masks": (C.c_int, [vp, P(C.c_uint64), C.c_int64, P(C.c_int64)]),
        "mosaic_gpu_cache_entry": (C.c_int, [vp, C.c_uint64, P(StageResultC), P(C.c_double),
                                             P(C.c_int32), C.c_int64, P(C.c_int64)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def _raise(code: int) -> None:
    if code in (OK, INFEASIBLE):
        return
    msg = load_library().mosaic_gpu_last_error().decode()
    exc = {MODULE_NO_OPTION: StageInfeasibleError, RANGE: SurfaceRangeError,
           TOO_LARGE: OracleTooLargeError, EMPTY: EmptyPlanError,
           BASELINE_INFEASIBLE: InfeasibleBaselineError,
           INVALID_ARGUMENT: InvalidArgumentError}.get(code, DeviceError)
    raise exc(msg or f"status {code}")


# ---------------------------------------------------------------------------
# result types (core.hpp:64-104, stage_eval.hpp:30-54, solver.hpp:106-131)
# ---------------------------------------------------------------------------
@dataclass
class DeploymentOption:
    dp_degree: int
    quota_units: int
    quota_levels: int

    def quota(self) -> float:
        return self.quota_units / self.quota_levels


@dataclass
class Entry:
    module: int
    option: DeploymentOption
    gpus: list[int]


@dataclass
class StageAllocation:
    entries: list[Entry] = field(default_factory=list)

    def module_indices(self) -> list[int]:
        return [e.module for e in self.entries]


@dataclass
class SolverStats:
    feasibility_calls: int = 0
    gpu_searches: int = 0
    nodes: int = 0
    leaves: int = 0


@dataclass
class StageEvalResult:
    stage_time: float
    allocation: StageAllocation
    stats: SolverStats


@dataclass
class DeploymentPlan:
    stages: list[StageAllocation] = field(default_factory=list)
    predicted_stage_times: list[float] = field(default_factory=list)
    predicted_iteration_time: float = 0.0


@dataclass
class TraceCandidate:
    mask_x: int
    mask_y: int
    pruned: bool
    cache_hit: bool
    gain: float


@dataclass
class TraceRound:
    candidates: list[TraceCandidate]
    chosen_x: int
    chosen_y: int
    applied_gain: float


@dataclass
class SolveTrace:
    rounds: list[TraceRound]
    stage_eval_calls: int
    feasibility_calls: int
    cache_hits: int
    prunes: int
    gpu_searches: int
    nodes: int
    leaves: int
    elapsed: float


@dataclass
class SolveResult:
    plan: DeploymentPlan
    trace: SolveTrace


@dataclass
class OracleResult:
    plan: DeploymentPlan
    iteration_time: float
    partitions_examined: int


@dataclass
class CandidateOption:
    opt: DeploymentOption
    base_latency: float
    solo_bandwidth: float
    footprint: float


# ---------------------------------------------------------------------------
class Planner:
    """One device context: PerfContext + ClusterSpec + SolveConfig of the reference."""

    def __init__(self, problem: C.POINTER(ProblemC), device: int = 0, _owned=None):
        L = load_library()
        self._owned = None
        self._ctx = C.c_void_p()
        _raise(L.mosaic_gpu_create(problem, device, C.byref(self._ctx)))
        self._owned = _owned  # freed by close() only once the context exists
        p = problem.contents
        self.n_modules = p.n_modules
        self.gpu_count = p.gpu_count
        self.quota_levels = p.quota_levels
        self._keep = None

    @classmethod
    def from_spec(cls, spec: str, quota_levels: int = 0, device: int = 0,
                  enable_prune: bool = True, enable_cache: bool = True) -> "Planner":
        """Synthetic BASELINE inputs: 'cfg1'..'cfg5', 'random:SEED:N:G', 'preset:NAME:K:G'."""
        L = load_library()
        pp = C.POINTER(ProblemC)()
        _raise(L.mosaic_gpu_synth_problem(spec.encode(), quota_levels, C.byref(pp)))
        pp.contents.enable_prune = int(enable_prune)
        pp.contents.enable_cache = int(enable_cache)
        try:
            return cls(pp, device, _owned=pp)
        except Exception:
            L.mosaic_gpu_free_problem(pp)
            raise

    @classmethod
    def from_surfaces(cls, modules: Sequence[dict], edges: Sequence[tuple[int, int]],
                      gpu_count: int, quota_levels: int = 10, memory_capacity: float = 80e9,
                      e: tuple[float, float, float] = (0.4e-3, 1.2e-3, 0.8e-3),
                      additive_only: bool = False, include_self: bool = True,
                      bisect_rel_tol: float = 1e-3, enable_prune: bool = True,
                      enable_cache: bool = True, device: int = 0) -> "Planner":
        """modules: [{'id': str, 'memory_base': float, 'points': [(d,a,lat,bw,mem,sm), ...]}]"""
        keep = []
        mods = (ModuleC * max(1, len(modules)))()
        for i, m in enumerate(modules):
            pts = (Point * len(m["points"]))(*[Point(*p) for p in m["points"]])
            idb = m["id"].encode()
            keep += [pts, idb]
            mods[i] = ModuleC(idb, m.get("memory_base", 0.0), pts, len(m["points"]))
        flat = [x for uv in edges for x in uv]
        ed = (C.c_int32 * max(1, len(flat)))(*flat)
        prob = ProblemC(mods, len(modules), ed, len(edges), gpu_count, memory_capacity,
                        e[0], e[1], e[2], int(additive_only), int(include_self), quota_levels,
                        bisect_rel_tol, int(enable_prune), int(enable_cache))
        keep += [mods, ed, prob]
        pl = cls(C.pointer(prob), device)
        pl._keep = keep
        return pl

    def close(self) -> None:
        if self._ctx:
            load_library().mosaic_gpu_destroy(self._ctx)
            self._ctx = C.c_void_p()
        if self._owned is not None:
            load_library().mosaic_gpu_free_problem(self._owned)
            self._owned = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- helpers --------------------------------------------------------------
    def _stage(self, r: StageResultC) -> StageEvalResult:
        ents = []
        for i in range(r.n_entries):
            e = r.entries[i]
            ents.append(Entry(e.module, DeploymentOption(e.dp_degree, e.quota_units,
                                                         self.quota_levels),
                              list(e.gpus[:e.n_gpus])))
        return StageEvalResult(r.stage_time, StageAllocation(ents),
                               SolverStats(r.probes, r.gpu_searches, r.nodes, r.leaves))

    @staticmethod
    def _mask(modules: Sequence[int]) -> int:
        m = 0
        for x in modules:
            m |= 1 << int(x)
        return m

    # -- API -----------------------------------------------------------------
    def lookup(self, module: int, d: int, a: float) -> tuple[float, float, float, float]:
        out = (C.c_double * 4)()
        _raise(load_library().mosaic_gpu_lookup(self._ctx, module, d, a, out))
        return tuple(out)

    def candidate_options(self, module: int) -> list[CandidateOption]:
        L = load_library()
        n = C.c_int32()
        _raise(L.mosaic_gpu_num_options(self._ctx, module, C.byref(n)))
        k = n.value
        d = (C.c_int32 * max(1, k))()
        u = (C.c_int32 * max(1, k))()
        b = (C.c_double * max(1, k))()
        bw = (C.c_double * max(1, k))()
        fp = (C.c_double * max(1, k))()
        _raise(L.mosaic_gpu_options(self._ctx, module, d, u, b, bw, fp))
        return [CandidateOption(DeploymentOption(d[i], u[i], self.quota_levels), b[i], bw[i], fp[i])
                for i in range(k)]

    def stage_eval(self, modules: Sequence[int]) -> Optional[StageEvalResult]:
        r = StageResultC()
        code = load_library().mosaic_gpu_stage_eval(self._ctx, self._mask(modules), C.byref(r))
        _raise(code)
        if r.status == MODULE_NO_OPTION:
            raise StageInfeasibleError("module has no feasible deployment option")
        return self._stage(r) if r.status == OK else None

    def search(self, module_sets: Sequence[Sequence[int]], exact: bool = False,
               times_only: bool = False):
        """Batched stage_eval (or ExactStageSolver::solve with exact=True) of many module sets
        (mosaic_gpu_search): the computations advance together, one launch per wave.
        times_only: just the stage times (None where infeasible), no allocations."""
        n = len(module_sets)
        masks = (C.c_uint64 * max(1, n))(*[self._mask(m) for m in module_sets])
        if times_only:
            t = (C.c_double * max(1, n))()
            stt = (C.c_int32 * max(1, n))()
            _raise(load_library().mosaic_gpu_search(self._ctx, masks, n, 1 if exact else 0,
                                                    None, t, stt))
            if not exact and any(stt[i] == MODULE_NO_OPTION for i in range(n)):
                raise StageInfeasibleError("module has no feasible deployment option")
            return [t[i] if stt[i] == OK else None for i in range(n)]
        out = (StageResultC * max(1, n))()
        _raise(load_library().mosaic_gpu_search(self._ctx, masks, n, 1 if exact else 0, out,
                                                None, None))
        res = []
        for i in range(n):
            r = out[i]
            if r.status == MODULE_NO_OPTION and not exact:
                raise StageInfeasibleError("module has no feasible deployment option")
            res.append(self._stage(r) if r.status == OK else None)
        return res

    def exact_stage(self, modules: Sequence[int]) -> Optional[StageEvalResult]:
        r = StageResultC()
        _raise(load_library().mosaic_gpu_exact_stage(self._ctx, self._mask(modules), C.byref(r)))
        return self._stage(r) if r.status == OK else None

    def stage_min(self, modules: Sequence[int], ub: float = float("inf"),
                  restart: bool = True) -> float:
        """T* of the module set below ub (one device MIN search when restart=False)."""
        t = C.c_double()
        r = StageResultC()
        _raise(load_library().mosaic_gpu_stage_min(self._ctx, self._mask(modules),
                                                    min(ub, 1e300), int(restart), C.byref(t),
                                                    C.byref(r)))
        return t.value

    def feasibility_run(self, modules: Sequence[int], tau: float) -> Optional[StageEvalResult]:
        r = StageResultC()
        _raise(load_library().mosaic_gpu_feasible(self._ctx, self._mask(modules), tau, C.byref(r)))
        return self._stage(r) if r.status == OK else None

    def _plan(self, pr: PlanResultC) -> DeploymentPlan:
        L = load_library()
        plan = DeploymentPlan()
        for s in range(pr.n_stages):
            r = StageResultC()
            _raise(L.mosaic_gpu_plan_stage(self._ctx, s, C.byref(r)))
            plan.stages.append(self._stage(r).allocation)
            plan.predicted_stage_times.append(pr.stage_time[s])
        plan.predicted_iteration_time = pr.iteration_time
        return plan

    def solve(self) -> SolveResult:
        L = load_library()
        pr = PlanResultC()
        _raise(L.mosaic_gpu_solve(self._ctx, C.byref(pr)))
        plan = self._plan(pr)
        rounds = []
        nr = C.c_int64()
        L.mosaic_gpu_trace_rounds(self._ctx, C.byref(nr))
        for r in range(nr.value):
            cx, cy, g, nc = C.c_uint64(), C.c_uint64(), C.c_double(), C.c_int64()
            _raise(L.mosaic_gpu_trace_round(self._ctx, r, C.byref(cx), C.byref(cy), C.byref(g),
                                            C.byref(nc)))
            cands = []
            for c in range(nc.value):
                mx, my, pru, hit, gain = (C.c_uint64(), C.c_uint64(), C.c_int32(), C.c_int32(),
                                          C.c_double())
                _raise(L.mosaic_gpu_trace_cand(self._ctx, r, c, C.byref(mx), C.byref(my),
                                               C.byref(pru), C.byref(hit), C.byref(gain)))
                cands.append(TraceCandidate(mx.value, my.value, bool(pru.value), bool(hit.value),
                                            gain.value))
            rounds.append(TraceRound(cands, cx.value, cy.value, g.value))
        tr = SolveTrace(rounds, pr.stage_eval_calls, pr.feasibility_calls, pr.cache_hits,
                        pr.prunes, pr.gpu_searches, pr.nodes, pr.leaves, pr.elapsed_s)
        return SolveResult(plan, tr)

    def brute_force_optimum(self) -> Optional[OracleResult]:
        pr = PlanResultC()
        code = load_library().mosaic_gpu_brute_force(self._ctx, C.byref(pr))
        _raise(code)
        if pr.status != OK:
            return None
        return OracleResult(self._plan(pr), pr.iteration_time, pr.partitions_examined)

    def stage_time(self, allocs: Sequence[StageAllocation],
                   with_rectified: bool = False):
        """Batched stage_time (and per-entry rectified_latency) on the device."""
        ents, gpus, off = [], [], [0]
        for a in allocs:
            for e in a.entries:
                ents.append(EvalEntryC(e.module, e.option.dp_degree, e.option.quota_units,
                                       len(e.gpus), e.option.quota_levels, 0, len(gpus)))
                gpus.extend(e.gpus)
            off.append(len(ents))
        n = len(allocs)
        E = (EvalEntryC * max(1, len(ents)))(*ents)
        G = (C.c_int32 * max(1, len(gpus)))(*gpus)
        O = (C.c_int64 * len(off))(*off)
        st = (C.c_double * max(1, n))()
        rect = (C.c_double * max(1, len(ents)))()
        _raise(load_library().mosaic_gpu_stage_time(self._ctx, E, G, O, n, st, rect))
        if with_rectified:
            return list(st[:n]), [list(rect[off[i]:off[i + 1]]) for i in range(n)]
        return list(st[:n])

    def evaluate(self, entries, gpus, alloc_off, stage_time_out, rect_out=None,
                 device: bool = False) -> None:
        """K1 on flat arrays (mosaic_gpu_evaluate): `entries` holds mosaic_gpu_eval_entry
        records as an (n_entries, 8) int32 array (see pack_eval_entries), `gpus` int32,
        `alloc_off` int64 (n_allocs + 1), outputs float64.  numpy arrays (host) or, with
        device=True, CUDA tensors on this planner's device (the caller synchronises the
        stream that wrote them)."""
        def ptr(x):
            if x is None:
                return None
            if hasattr(x, "data_ptr"):
                return x.data_ptr()
            return x.ctypes.data
        n = len(alloc_off) - 1
        _raise(load_library().mosaic_gpu_evaluate(
            self._ctx, ptr(entries), len(entries), ptr(gpus), len(gpus), ptr(alloc_off), n,
            ptr(stage_time_out), ptr(rect_out), 1 if device else 0))

    def evaluate_stats(self) -> dict:
        ms, n, b = C.c_double(), C.c_int64(), C.c_int64()
        _raise(load_library().mosaic_gpu_evaluate_stats(self._ctx, C.byref(ms), C.byref(n),
                                                        C.byref(b)))
        fms, nf = C.c_double(), C.c_int64()
        _raise(load_library().mosaic_gpu_evaluate_paths(self._ctx, C.byref(fms), C.byref(nf)))
        return {"kernel_ms": ms.value, "launches": n.value, "alg_bytes": b.value,
                "fast_kernel_ms": fms.value, "full_path_allocs": nf.value}

    def make_baseline_plan(self, policy: str) -> "DeploymentPlan":
        """make_baseline_plan (simulator.hpp:283-313): 'megatron' or 'distmm', full-quota
        options; raises InfeasibleBaselineError like the reference."""
        pol = {"megatron": 0, "distmm": 1}[policy.lower()]
        pr = PlanResultC()
        _raise(load_library().mosaic_gpu_baseline_plan(self._ctx, pol, C.byref(pr)))
        return self._plan(pr)

    def simulate(self, plan: "DeploymentPlan", config: Optional["SimConfig"] = None,
                 seeds: Optional[Sequence[int]] = None) -> list["SimulationReport"]:
        """simulate (simulator.hpp:68-119) of `plan` on the device, one report per seed
        (default: [config.seed]); the timeline is filled for the first seed only."""
        cfg = config or SimConfig()
        seeds = list(seeds) if seeds is not None else [cfg.seed]
        ents, gpus, off = [], [], [0]
        for st in plan.stages:
            for e in st.entries:
                ents.append(EvalEntryC(e.module, e.option.dp_degree, e.option.quota_units,
                                       len(e.gpus), e.option.quota_levels, 0, len(gpus)))
                gpus.extend(e.gpus)
            off.append(len(ents))
        n, S, G = len(seeds), len(plan.stages), self.gpu_count
        E = (EvalEntryC * max(1, len(ents)))(*ents)
        Gp = (C.c_int32 * max(1, len(gpus)))(*gpus)
        O = (C.c_int64 * len(off))(*off)
        sc = SimConfigC(cfg.iterations, 1 if cfg.stream_mode == "on_demand" else 0,
                        cfg.pooled_overhead, cfg.on_demand_overhead, cfg.perturbation_sigma)
        sd = (C.c_uint64 * max(1, n))(*[s & (2**64 - 1) for s in seeds])
        it = (C.c_double * max(1, n))()
        ps = (C.c_double * max(1, n * S))()
        bz = (C.c_double * max(1, n * G))()
        mb = (C.c_double * max(1, n))()
        tl = (IntervalC * max(1, len(gpus)))()
        ntl = C.c_int64()
        _raise(load_library().mosaic_gpu_simulate(self._ctx, E, Gp, O, S, C.byref(sc), sd, n, it,
                                                  ps, bz, mb, tl, len(gpus), C.byref(ntl)))
        out = []
        for i in range(n):
            rep = SimulationReport(it[i], list(ps[i * S:(i + 1) * S]),
                                   list(bz[i * G:(i + 1) * G]), mb[i], [])
            if i == 0:
                rep.timeline = [TimelineInterval(x.gpu, x.module, x.start, x.end, x.quota)
                                for x in tl[:ntl.value]]
            out.append(rep)
        return out

    def validate_plan(self, plan: "DeploymentPlan") -> tuple[str, str]:
        """validate_plan (core.hpp:281-351) -> (ValidationCode name, message)."""
        ents, gpus, off = [], [], [0]
        for st in plan.stages:
            for e in st.entries:
                ents.append(EvalEntryC(e.module, e.option.dp_degree, e.option.quota_units,
                                       len(e.gpus), e.option.quota_levels, 0, len(gpus)))
                gpus.extend(e.gpus)
            off.append(len(ents))
        E = (EvalEntryC * max(1, len(ents)))(*ents)
        G = (C.c_int32 * max(1, len(gpus)))(*gpus)
        O = (C.c_int64 * len(off))(*off)
        buf = C.create_string_buffer(64)
        L = load_library()
        _raise(L.mosaic_gpu_validate_plan(self._ctx, E, G, O, len(plan.stages), buf, 64))
        return buf.value.decode(), L.mosaic_gpu_last_error().decode()

    def launch_count(self) -> int:
        return load_library().mosaic_gpu_launch_count(self._ctx)

    def device_ms(self) -> float:
        return load_library().mosaic_gpu_search_ms(self._ctx)

    def reset_counters(self) -> None:
        load_library().mosaic_gpu_reset_counters(self._ctx)

    def counters(self) -> dict:
        L = load_library()
        return {"own_launches": L.mosaic_gpu_own_launches(self._ctx),
                "launches": L.mosaic_gpu_launch_count(self._ctx),
                "ksearch_ms": L.mosaic_gpu_ksearch_ms(self._ctx),
                "ksearch_launches": L.mosaic_gpu_ksearch_launches(self._ctx),
                "h2d_bytes": L.mosaic_gpu_h2d_bytes(self._ctx),
                "d2h_bytes": L.mosaic_gpu_d2h_bytes(self._ctx),
                "device_ms": L.mosaic_gpu_search_ms(self._ctx),
                "alg_bytes": L.mosaic_gpu_alg_bytes(self._ctx),
                "peer_links": L.mosaic_gpu_peer_links(self._ctx)}

    def mark(self, which: int) -> None:
        load_library().mosaic_gpu_mark(self._ctx, which)

    def marked_ms(self) -> float:
        return load_library().mosaic_gpu_marked_ms(self._ctx)

    def set_tuning(self, **knobs: float) -> None:
        """Search-engine knobs for experiments (include/mosaic_gpu.h, mosaic_gpu_set_tuning)."""
        for k, v in knobs.items():
            _raise(load_library().mosaic_gpu_set_tuning(self._ctx, k.encode(), float(v)))

    def device_bytes(self) -> int:
        return load_library().mosaic_gpu_device_bytes(self._ctx)

    def clear_cache(self) -> None:
        load_library().mosaic_gpu_clear_cache(self._ctx)

    def eval_cache(self) -> list[tuple[int, StageEvalResult, list[tuple[float, bool]]]]:
        """EvalCache after a solve, in insertion order: (mask, result, probes), where probes
        are the (tau, feasible) of every FeasibilitySearch::run the stage_eval replayed."""
        L = load_library()
        n = C.c_int64()
        _raise(L.mosaic_gpu_cache_masks(self._ctx, None, 0, C.byref(n)))
        masks = (C.c_uint64 * max(1, n.value))()
        _raise(L.mosaic_gpu_cache_masks(self._ctx, masks, n.value, C.byref(n)))
        out = []
        for m in masks[:n.value]:
            r = StageResultC()
            npb = C.c_int64()
            _raise(L.mosaic_gpu_cache_entry(self._ctx, m, C.byref(r), None, None, 0,
                                            C.byref(npb)))
            tau = (C.c_double * max(1, npb.value))()
            ok = (C.c_int32 * max(1, npb.value))()
            _raise(L.mosaic_gpu_cache_entry(self._ctx, m, C.byref(r), tau, ok, npb.value,
                                            C.byref(npb)))
            out.append((int(m), self._stage(r),
                        [(tau[i], bool(ok[i])) for i in range(npb.value)]))
        return out

    def set_shard_nccl(self, rank: int, world: int, nccl_id: bytes) -> None:
        """Shard every device search over `world` ranks with the library's own NCCL
        communicator (mosaic_gpu_set_shard_nccl); nccl_id from nccl_unique_id() on rank 0."""
        buf = C.create_string_buffer(bytes(nccl_id), len(nccl_id))
        _raise(load_library().mosaic_gpu_set_shard_nccl(self._ctx, rank, world, buf))

    def set_shard(self, rank: int, world: int, allgather=None) -> None:
        """allgather(send: bytes) -> list[bytes] over ranks (torch.distributed in bench.py)."""
        if world <= 1:
            _raise(load_library().mosaic_gpu_set_shard(self._ctx, 0, 1, ALLGATHER_FN(), None))
            return

        def _cb(user, send, recv, nbytes):
            try:
                parts = allgather(C.string_at(send, nbytes))
                C.memmove(recv, b"".join(parts), nbytes * world)
                return 0
            except Exception:
                return 1

        self._ag = ALLGATHER_FN(_cb)
        _raise(load_library().mosaic_gpu_set_shard(self._ctx, rank, world, self._ag, None))


# module-level spellings of the reference entry points
def stage_eval(planner: Planner, modules: Sequence[int]) -> Optional[StageEvalResult]:
    return planner.stage_eval(modules)


def exact_stage(planner: Planner, modules: Sequence[int]) -> Optional[StageEvalResult]:
    return planner.exact_stage(modules)


def feasibility_run(planner: Planner, modules: Sequence[int], tau: float):
    return planner.feasibility_run(modules, tau)


def solve(planner: Planner) -> SolveResult:
    return planner.solve()


def brute_force_optimum(planner: Planner) -> Optional[OracleResult]:
    return planner.brute_force_optimum()


def pack_eval_entries(module, dp_degree, quota_units, n_gpus, gpu_off, quota_levels=None):
    """(n, 8) int32 view of mosaic_gpu_eval_entry records from per-entry columns (numpy):
    module, dp_degree, quota_units, n_gpus, quota_levels (0 = the context's), reserved,
    gpu_off (int64, little-endian low/high words)."""
    import numpy as np
    n = len(module)
    out = np.zeros((n, 8), dtype=np.int32)
    out[:, 0] = module
    out[:, 1] = dp_degree
    out[:, 2] = quota_units
    out[:, 3] = n_gpus
    if quota_levels is not None:
        out[:, 4] = quota_levels
    out[:, 6:8] = np.asarray(gpu_off, dtype=np.int64).reshape(n, 1).view(np.int32)
    return out


def stage_time(planner: Planner, allocation: StageAllocation) -> float:
    return planner.stage_time([allocation])[0]


def rectified_latency(planner: Planner, allocation: StageAllocation, module: int) -> float:
    _, rect = planner.stage_time([allocation], with_rectified=True)
    for e, r in zip(allocation.entries, rect[0]):
        if e.module == module:
            return r
    raise ValueError("module not in stage")


def candidate_options(planner: Planner, module: int) -> list[CandidateOption]:
    return planner.candidate_options(module)


MAXB = 128  # GPU blocks per search level (search_core.cuh)


def smem_peak_gbs(device: int = 0) -> float:
    """Measured shared-memory load bandwidth of the device (GB/s): the on-chip roofline
    denominator of SURVEY.md §8(d)."""
    g = C.c_double()
    _raise(load_library().mosaic_gpu_smem_peak(device, C.byref(g)))
    return g.value


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId through the library (128 bytes, to hand to every rank)."""
    buf = C.create_string_buffer(128)
    _raise(load_library().mosaic_gpu_nccl_id(buf, 128))
    return buf.raw


def rank_record(has_hit: bool, inc: float, path=(), aborted: bool = False,
                overflow: bool = False, leaf_value: float = 0.0) -> bytes:
    """One rank's RankRecord of a sharded search (Engine::merge_ranks): path = [(option,
    [block counts...]) per level] of its FIRST hit / argmin leaf."""
    L = load_library()
    buf = C.create_string_buffer(L.mosaic_gpu_rank_record_size())
    k = len(path)
    opt = (C.c_uint16 * max(1, k))(*[o for o, _ in path])
    nb = (C.c_uint16 * max(1, k))(*[len(x) for _, x in path])
    x = (C.c_uint16 * (max(1, k) * MAXB))()
    for l, (_, xs) in enumerate(path):
        for b, v in enumerate(xs):
            x[l * MAXB + b] = v
    _raise(L.mosaic_gpu_rank_record(buf, int(has_hit), int(aborted), int(overflow), inc, k,
                                    opt, nb, x, leaf_value))
    return buf.raw


def merge_ranks(records: bytes, world: int, mode: int, k: int) -> dict:
    """The engine's merge of one sharded search over `world` concatenated RankRecords:
    mode 0 MIN, 1 FIRST (include/mosaic_gpu.h, mosaic_gpu_merge_ranks)."""
    w, f, a, o = C.c_int(), C.c_int(), C.c_int(), C.c_int()
    v, lv = C.c_double(), C.c_double()
    buf = C.create_string_buffer(records, len(records))
    _raise(load_library().mosaic_gpu_merge_ranks(buf, world, mode, k, C.byref(w), C.byref(f),
                                                 C.byref(v), C.byref(a), C.byref(o),
                                                 C.byref(lv)))
    return {"winner": w.value, "found": bool(f.value), "value": v.value,
            "aborted": bool(a.value), "overflow": bool(o.value), "leaf_value": lv.value}


# ---------------------------------------------------------------------------
# N2: input generation on the device (profiler.hpp)
# ---------------------------------------------------------------------------
@dataclass
class SimConfig:
    """SimConfig (simulator.hpp:28-35); stream_mode 'pooled' or 'on_demand'."""
    iterations: int = 1
    stream_mode: str = "pooled"
    pooled_overhead: float = 0.013e-3
    on_demand_overhead: float = 37e-3
    perturbation_sigma: float = 0.0
    seed: int = 0


@dataclass
class TimelineInterval:
    gpu: int
    module: int
    start: float
    end: float
    quota: float


@dataclass
class SimulationReport:
    """SimulationReport (simulator.hpp:45-55)."""
    iteration_time: float
    per_stage_times: list
    per_gpu_busy_fraction: list
    mean_busy_fraction: float
    timeline: list


@dataclass
class ModuleWorkload:
    """ModuleWorkload (profiler.hpp:26-40)."""
    id: str
    flops_per_iter: float
    bytes_per_iter: float
    gradient_bytes: float
    sm_efficiency_knee: float
    memory_act_base: float
    memory_per_quota: float
    fixed_overhead: float
    dp_penalty: float


@dataclass
class ClusterSpec:
    """ClusterSpec (core.hpp:52-59)."""
    gpu_count: int = 1
    memory_capacity: float = 80e9
    peak_compute: float = 500e12
    peak_bandwidth: float = 3.35e12
    interconnect_alpha: float = 5e-6
    interconnect_beta: float = 2.2e-12


def synth_workloads(spec: str) -> tuple[list[ModuleWorkload], ClusterSpec]:
    """Workloads (module order) and cluster behind a synthetic spec ('cfg1'..'cfg5',
    'random:SEED:N:G', 'preset:NAME:K:G'): make_workload / make_preset / random_instance."""
    L = load_library()
    buf = (WorkloadC * MAX_MODULES)()
    n = C.c_int32()
    cl = ClusterC()
    _raise(L.mosaic_gpu_synth_workloads(spec.encode(), buf, MAX_MODULES, C.byref(n), C.byref(cl)))
    pp = C.POINTER(ProblemC)()
    _raise(L.mosaic_gpu_synth_problem(spec.encode(), 0, C.byref(pp)))
    ids = [pp.contents.modules[i].id.decode() for i in range(n.value)]
    L.mosaic_gpu_free_problem(pp)
    ws = [ModuleWorkload(ids[i], *[getattr(buf[i], f) for f, _ in WorkloadC._fields_[1:]])
          for i in range(n.value)]
    return ws, ClusterSpec(*[getattr(cl, f) for f, _ in ClusterC._fields_])


def generate_surfaces(workloads: Sequence[ModuleWorkload], cluster: ClusterSpec,
                      d_set: Optional[Sequence[int]] = None,
                      a_set: Optional[Sequence[float]] = None, demand_scale: float = 1.0,
                      device: int = 0) -> list[list[tuple]]:
    """generate_surfaces (profiler.hpp:65-111) on the device (k_gen_surfaces): per workload,
    the (d, a, latency, bandwidth_util, memory, sm_active) grid, d-major then a — the
    `points` format Planner.from_surfaces takes.  d_set/a_set default to
    default_dp_degrees(gpu_count) / default_quota_grid()."""
    L = load_library()
    W = (WorkloadC * max(1, len(workloads)))(*[
        WorkloadC(None, w.flops_per_iter, w.bytes_per_iter, w.gradient_bytes,
                  w.sm_efficiency_knee, w.memory_act_base, w.memory_per_quota,
                  w.fixed_overhead, w.dp_penalty) for w in workloads])
    cl = ClusterC(*[getattr(cluster, f) for f, _ in ClusterC._fields_])
    D = (C.c_int32 * len(d_set))(*d_set) if d_set is not None else None
    A = (C.c_double * len(a_set))(*a_set) if a_set is not None else None
    nd, na = C.c_int32(), C.c_int32()
    args = (W, len(workloads), C.byref(cl), D, len(d_set or []), A, len(a_set or []),
            demand_scale, device)
    _raise(L.mosaic_gpu_generate_surfaces(*args, None, C.byref(nd), C.byref(na)))
    per = nd.value * na.value
    out = (Point * max(1, per * len(workloads)))()
    _raise(L.mosaic_gpu_generate_surfaces(*args, out, C.byref(nd), C.byref(na)))
    return [[(p.d, p.a, p.latency, p.bandwidth_util, p.memory, p.sm_active)
             for p in out[i * per:(i + 1) * per]] for i in range(len(workloads))]
