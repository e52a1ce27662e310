"""Reference JSON v1 file formats in and out of the C ABI.

Restates io.hpp (version check :38-46, required-field errors :48-58, model :63-96,
cluster :102-124, profile :130-174, interference :210-231, plan :237-285, trace :291-314)
so a user of the reference CLI can hand its `model.json / cluster.json / profile.json /
interference.json` straight to the B200 planner and get a plan JSON with the same schema.
"""
from __future__ import annotations

import json
import math
from typing import Any, Optional

from . import mosaic

FORMAT_VERSION = 1  # kFormatVersion, io.hpp:32


class IoError(RuntimeError):
    """io.hpp:28"""


def _check_version(j: Any, kind: str) -> None:
    if not isinstance(j, dict):
        raise IoError(f"{kind}: expected a JSON object")
    v = j.get("version")
    if not isinstance(v, int) or isinstance(v, bool):
        raise IoError(f"{kind}: missing integer 'version'")
    if v != FORMAT_VERSION:
        raise IoError(f"{kind}: unsupported version {v}")


def _require(j: dict, key: str, kind: str, typ=None):
    if key not in j:
        raise IoError(f"{kind}: missing field '{key}'")
    v = j[key]
    if typ is float and isinstance(v, (int, float)) and not isinstance(v, bool):
        return float(v)
    if typ is not None and not isinstance(v, typ):
        raise IoError(f"{kind}: bad field '{key}'")
    return v


def _load(x):
    if isinstance(x, (str, bytes)) and not str(x).lstrip().startswith("{"):
        with open(x) as f:
            return json.load(f)
    if isinstance(x, (str, bytes)):
        return json.loads(x)
    return x


def model_from_json(j) -> dict:
    j = _load(j)
    _check_version(j, "model")
    mods = []
    for jm in _require(j, "modules", "model", list):
        mods.append({"id": _require(jm, "id", "model.module", str),
                     "name": jm.get("name", jm["id"]),
                     "memory_base": float(jm.get("memory_base", 0.0)),
                     "tags": list(jm.get("tags", []))})
    ids = [m["id"] for m in mods]
    edges = []
    for je in _require(j, "edges", "model", list):
        if not isinstance(je, list) or len(je) != 2:
            raise IoError("model: each edge must be a [from, to] pair")
        edges.append((je[0], je[1]))
    if len(set(ids)) != len(ids):
        raise IoError("model: duplicate module id")
    for u, v in edges:
        if u not in ids or v not in ids:
            raise IoError(f"model: edge references unknown module: {u if u not in ids else v}")
    return {"modules": mods, "edges": edges}


def cluster_from_json(j) -> dict:
    j = _load(j)
    _check_version(j, "cluster")
    c = {"gpu_count": _require(j, "gpu_count", "cluster", int),
         "memory_capacity": float(j.get("memory_capacity", 80e9)),
         "peak_compute": float(j.get("peak_compute", 500e12)),
         "peak_bandwidth": float(j.get("peak_bandwidth", 3.35e12)),
         "interconnect_alpha": float(j.get("interconnect_alpha", 5e-6)),
         "interconnect_beta": float(j.get("interconnect_beta", 2.2e-12))}
    if c["gpu_count"] < 1:
        raise IoError("cluster: gpu_count must be >= 1")
    if c["memory_capacity"] <= 0 or c["peak_compute"] <= 0 or c["peak_bandwidth"] <= 0:
        raise IoError("cluster: capacities must be positive")
    return c


def surfaces_from_json(j) -> dict:
    j = _load(j)
    _check_version(j, "profile")
    out = {}
    for js in _require(j, "surfaces", "profile", list):
        mid = _require(js, "module", "profile.surface", str)
        pts = []
        for jp in _require(js, "points", "profile.surface", list):
            pts.append((_require(jp, "d", "profile.point", int),
                        _require(jp, "a", "profile.point", float),
                        _require(jp, "latency", "profile.point", float),
                        _require(jp, "bandwidth_util", "profile.point", float),
                        _require(jp, "memory", "profile.point", float),
                        float(jp.get("sm_active", 1.0))))
        out[mid] = pts
    return out


def interference_from_json(j) -> dict:
    j = _load(j)
    _check_version(j, "interference")
    return {"e1": _require(j, "e1", "interference", float),
            "e2": _require(j, "e2", "interference", float),
            "e3": _require(j, "e3", "interference", float),
            "r_squared": float(j.get("r_squared", 1.0)),
            "sample_count": int(j.get("sample_count", 0)),
            "additive_only": bool(j.get("additive_only", False))}


def load_scenario(model, cluster, profile, interference, granularity: Optional[float] = None,
                  quota_levels: Optional[int] = None, include_self: bool = True,
                  enable_prune: bool = True, enable_cache: bool = True,
                  device: int = 0) -> "mosaic.Planner":
    """Build a device Planner from the reference's JSON files (cmd_plan, mosaic_main.cpp:146).
    `granularity` maps to quota_levels = lround(1/g) as the CLI does (mosaic_main.cpp:154)."""
    g = model_from_json(model)
    c = cluster_from_json(cluster)
    s = surfaces_from_json(profile)
    im = interference_from_json(interference)
    if quota_levels is None:
        q = 1.0 / (granularity if granularity else 0.1)
        # std::lround: halves away from zero (Python's round() is banker's rounding)
        quota_levels = int(math.floor(q + 0.5)) if q >= 0 else -int(math.floor(-q + 0.5))
    ids = [m["id"] for m in g["modules"]]
    mods = []
    for m in g["modules"]:
        if m["id"] not in s:
            raise IoError(f"profile: no surface for module {m['id']}")
        mods.append({"id": m["id"], "memory_base": m["memory_base"], "points": s[m["id"]]})
    edges = [(ids.index(u), ids.index(v)) for u, v in g["edges"]]
    pl = mosaic.Planner.from_surfaces(
        mods, edges, c["gpu_count"], quota_levels=quota_levels,
        memory_capacity=c["memory_capacity"], e=(im["e1"], im["e2"], im["e3"]),
        additive_only=im["additive_only"], include_self=include_self,
        enable_prune=enable_prune, enable_cache=enable_cache, device=device)
    pl.module_ids = ids
    return pl


def plan_to_json(plan: "mosaic.DeploymentPlan", module_ids) -> dict:
    """to_json(DeploymentPlan, ModelGraph), io.hpp:237-258."""
    stages = []
    for i, st in enumerate(plan.stages):
        js = {}
        if i < len(plan.predicted_stage_times):
            js["predicted_time"] = plan.predicted_stage_times[i]
        js["modules"] = [{"module": module_ids[e.module], "dp_degree": e.option.dp_degree,
                          "quota_units": e.option.quota_units,
                          "quota_levels": e.option.quota_levels, "gpus": list(e.gpus)}
                         for e in st.entries]
        stages.append(js)
    return {"version": FORMAT_VERSION,
            "predicted_iteration_time": plan.predicted_iteration_time, "stages": stages}


def plan_from_json(j, module_ids) -> "mosaic.DeploymentPlan":
    """plan_from_json, io.hpp:260-285."""
    j = _load(j)
    _check_version(j, "plan")
    plan = mosaic.DeploymentPlan()
    for js in _require(j, "stages", "plan", list):
        ents = []
        for jm in _require(js, "modules", "plan.stage", list):
            mid = _require(jm, "module", "plan.entry", str)
            if mid not in module_ids:
                raise IoError(f"plan: unknown module {mid}")
            ents.append(mosaic.Entry(module_ids.index(mid), mosaic.DeploymentOption(
                _require(jm, "dp_degree", "plan.entry", int),
                _require(jm, "quota_units", "plan.entry", int),
                _require(jm, "quota_levels", "plan.entry", int)),
                list(_require(jm, "gpus", "plan.entry", list))))
        ents.sort(key=lambda e: e.module)
        plan.stages.append(mosaic.StageAllocation(ents))
        if "predicted_time" in js:
            plan.predicted_stage_times.append(float(js["predicted_time"]))
    plan.predicted_iteration_time = float(j.get("predicted_iteration_time", 0.0))
    return plan


def trace_to_json(t: "mosaic.SolveTrace") -> dict:
    """to_json(SolveTrace), io.hpp:291-314 (+ device counters)."""
    return {"version": FORMAT_VERSION, "stage_eval_calls": t.stage_eval_calls,
            "feasibility_calls": t.feasibility_calls, "cache_hits": t.cache_hits,
            "prunes": t.prunes, "elapsed": t.elapsed,
            "rounds": [{"chosen_x": r.chosen_x, "chosen_y": r.chosen_y,
                        "applied_gain": r.applied_gain,
                        "candidates": [{"mask_x": c.mask_x, "mask_y": c.mask_y,
                                        "pruned": c.pruned, "cache_hit": c.cache_hit,
                                        "gain": c.gain} for c in r.candidates]}
                       for r in t.rounds],
            "device": {"gpu_searches": t.gpu_searches, "nodes": t.nodes, "leaves": t.leaves}}
