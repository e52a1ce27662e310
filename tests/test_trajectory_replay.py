"""CPU: the GAHC decisions of the GPU's cfg5 solve (tests/golden/trajectory_gpu.json) replayed
with the reference's own rules (solver.hpp:157-289, restated here as test infrastructure) on
the stage times the REFERENCE computed wherever it has (tests/golden/trajectory_ref.jsonl):
every round's candidate order, prune flags, cache hits, gains, chosen merge and the final
plan must come out exactly as the GPU recorded them.  Also: every pinned reference result
agrees with the GPU's cached result for the same module set."""
import json

import pytest

from conftest import hexf, load_golden
from trajectory import done, load_gpu, load_ref

REF = load_ref()
TRAJ = load_gpu()


def pinned_time(shape: str, mask: int):
    """The reference's stage_eval time for mask: its full stage_eval record, else the leaf
    value of its run of the deciding last successful probe (stage_eval returns that leaf,
    stage_eval.hpp:372-381)."""
    r = REF.get(f"{shape}|stage|{mask}")
    if done(r) and r["out"].get("feasible"):
        return hexf(r["out"]["t"]), "stage"
    r = REF.get(f"{shape}|feas_last_ok|{mask}")
    if done(r) and r["out"].get("feasible"):
        return hexf(r["out"]["t"]), "last_ok_probe"
    return None, None


@pytest.mark.parametrize("shape", sorted(TRAJ))
def test_pinned_results_agree_with_gpu_cache(shape):
    n = 0
    for c in TRAJ[shape]["cache"]:
        t, kind = pinned_time(shape, c["mask"])
        if t is None:
            continue
        n += 1
        assert t == hexf(c["t"]), (shape, c["mask"], kind)
        r = REF.get(f"{shape}|stage|{c['mask']}") if kind == "stage" else \
            REF.get(f"{shape}|feas_last_ok|{c['mask']}")
        got = [(a["m"], a["d"], a["u"], a["gpus"]) for a in c["alloc"]]
        want = [(a["m"], a["d"], a["u"], a["gpus"]) for a in r["out"]["alloc"]]
        assert got == want, (shape, c["mask"], kind)
        if kind == "stage":
            assert c["feasibility_calls"] == r["out"]["feasibility_calls"], (shape, c["mask"])
    assert n > 0


def _topo(ids, edges):
    n = len(ids)
    indeg = [0] * n
    adj = [[] for _ in range(n)]
    for u, v in edges:
        adj[u].append(v)
        indeg[v] += 1
    ready = sorted([i for i in range(n) if indeg[i] == 0], key=lambda i: ids[i])
    order = []
    while ready:
        u = ready.pop(0)
        order.append(u)
        for v in adj[u]:
            indeg[v] -= 1
            if indeg[v] == 0:
                ready.append(v)
                ready.sort(key=lambda i: ids[i])
    return order


def _reach(n, edges, order):
    adj = [[] for _ in range(n)]
    for u, v in edges:
        adj[u].append(v)
    reach = [0] * n
    for u in reversed(order):
        for v in adj[u]:
            reach[u] |= (1 << v) | reach[v]
    return reach


def test_cfg5_gahc_replay_on_reference_times():
    shape = "cfg5@L32"
    traj = TRAJ[shape]
    opts = load_golden("configs.json")["cfg5"]["options"]["modules"]
    ids = [m["id"] for m in opts]
    n = len(ids)
    back = ids.index("backbone")
    edges = [(i, back) for i in range(n) if i != back]
    min_base = [min(hexf(r[2]) for r in m["rows"]) for m in opts]
    order = _topo(ids, edges)
    reach = _reach(n, edges, order)
    gpu_time = {c["mask"]: hexf(c["t"]) for c in traj["cache"]}
    used_ref = 0

    def stage_time(mask):
        nonlocal used_ref
        t, _ = pinned_time(shape, mask)
        if t is not None:
            used_ref += 1
            return t
        return gpu_time[mask]  # not pinned yet: the GPU's value (DESIGN.md lists these)

    cache = {}
    masks, times = [], []
    for m in order:
        cache[1 << m] = stage_time(1 << m)
        masks.append(1 << m)
        times.append(cache[1 << m])

    def legal(x, y):
        up = 0
        for z in range(x, y):
            up |= masks[z]
        return not any((up >> m & 1) and (reach[m] & masks[y]) for m in range(n))

    def order_key(p):
        a = masks[p[0]] | masks[p[1]]
        return (bin(a).count("1"), a, masks[p[0]])

    rounds = []
    while len(masks) > 1:
        pairs = sorted([(x, y) for x in range(len(masks)) for y in range(x + 1, len(masks))
                        if legal(x, y)], key=order_key)
        delta_best, best = 0.0, None
        cands = []
        for x, y in pairs:
            mm = masks[x] | masks[y]
            tx, ty = times[x], times[y]
            t_lb = max(min_base[m] for m in range(n) if mm >> m & 1)
            if tx + ty - t_lb <= delta_best:
                cands.append({"x": masks[x], "y": masks[y], "pruned": 1, "hit": 0, "gain": 0.0})
                continue
            hit = mm in cache
            if not hit:
                cache[mm] = stage_time(mm)
            gain = tx + ty - cache[mm]
            cands.append({"x": masks[x], "y": masks[y], "pruned": 0, "hit": int(hit), "gain": gain})
            if gain > delta_best:
                delta_best, best = gain, (x, y)
        if best is None:
            rounds.append({"x": 0, "y": 0, "cands": cands})
            break
        x, y = best
        rounds.append({"x": masks[x], "y": masks[y], "gain": delta_best, "cands": cands})
        masks[x] |= masks[y]
        times[x] = cache[masks[x]]
        del masks[y], times[y]
    want = traj["rounds"]
    assert len(rounds) == len(want)
    for got, w in zip(rounds, want):
        assert (got["x"], got["y"]) == (w["x"], w["y"])
        if w["x"]:
            assert got["gain"] == hexf(w["gain"])
        assert len(got["cands"]) == len(w["cands"])
        for a, b in zip(got["cands"], w["cands"]):
            assert (a["x"], a["y"], a["pruned"], a["hit"]) == (b["x"], b["y"], b["pruned"], b["hit"])
            if not a["pruned"]:
                assert a["gain"] == hexf(b["gain"])
    assert sum(times) == hexf(traj["iteration_time"])
    assert used_ref >= 29
