"""Differential check of the host mirror against the reference itself on
random specs: `build_layout` (units, sizes, replica ranks, nodes), every
plan (`plan_equal` / `plan_adaptive` / `plan_baseline`, all phases,
per-rank workloads, bottleneck), `build_phase_assignment` for random due
sets, the checkpoint-size formulas and the selectors (SURVEY.md §8(a) rows
a3-a9; reference topology.py:212-356, planner.py:150-353, selector.py:21-100).
Validation errors must agree too (same constraint string).

Imports the reference in place from /root/reference (skipped where it is not
mounted, e.g. on the GPU box)."""

import importlib
import random
import sys
from pathlib import Path

import pytest

REF_SRC = Path("/root/reference/pkg/src")
pytestmark = pytest.mark.skipif(not (REF_SRC / "mocsim").exists(), reason="reference not mounted")


@pytest.fixture(scope="module")
def ref():
    sys.path.insert(0, str(REF_SRC))
    try:
        mods = {m: importlib.import_module(f"mocsim.{m}")
                for m in ("topology", "planner", "selector")}
    finally:
        sys.path.remove(str(REF_SRC))
    return mods


def _ours():
    from paper_2408_04307_b200 import planner, selector, topology
    return {"topology": topology, "planner": planner, "selector": selector}


def _spec(rng: random.Random):
    E = rng.choice([1, 2, 3, 4, 6, 8, 16])
    L = rng.randint(1, 4)
    ep = rng.choice([d for d in (1, 2, 4, 8) if d <= 8])
    dp = ep * rng.choice([1, 2, 3])
    gpn = rng.choice([d for d in range(1, dp + 1) if dp % d == 0])
    mods = tuple((f"m{i}", rng.randint(1, 5000)) for i in range(rng.randint(1, 7)))
    if rng.random() < 0.3:  # duplicate sizes exercise the stable NE order
        mods = mods + (("dup", mods[0][1]),)
    return dict(E=E, L=L, dp=dp, ep=ep, gpn=gpn, mods=mods, epp=rng.randint(1, 3000),
                bw=rng.choice([2, 4]), bo=rng.choice([8, 12]), other=rng.choice([0, 0, 7, 4097]),
                k=rng.randint(1, E))


def _build(m, sp):
    T = m["topology"]
    model = T.ModelSpec(num_moe_layers=sp["L"], experts_per_layer=sp["E"], top_k=1,
                        non_expert_params=sum(c for _, c in sp["mods"]),
                        expert_params_per_expert=sp["epp"], bytes_weight=sp["bw"],
                        bytes_optim=sp["bo"], other_states_bytes=sp["other"],
                        non_expert_modules=sp["mods"])
    par = T.ParallelSpec(dp_degree=sp["dp"], ep_degree=sp["ep"])
    cl = T.ClusterSpec(num_nodes=sp["dp"] // sp["gpn"], gpus_per_node=sp["gpn"],
                       snapshot_bandwidth=1e9, persist_bandwidth=1e8, fb_time=0.01,
                       update_time=0.002, restart_time=1.0)
    return model, par, T.build_layout(model, par, cl)


def _units(layout):
    return sorted((u.key, u.kind, u.layer, u.expert, u.size_bytes, tuple(sorted(u.replica_ranks)))
                  for u in layout.units)


def _phase(ph):
    return {r: [tuple(a) for a in ranges] for r, ranges in sorted(ph.items())}


def _plan(plan):
    return (plan.period, [_phase(ph) for ph in plan.assignments],
            [dict(sorted(w.items())) for w in plan.workload_bytes])


def _try(fn, *a, **kw):
    try:
        return ("ok", fn(*a, **kw))
    except Exception as exc:
        return ("err", type(exc).__name__, str(exc))


@pytest.mark.parametrize("seed", range(25))
def test_random_specs_layouts_plans_and_sizes_match_reference(ref, seed):
    ours = _ours()
    rng = random.Random(seed)
    for trial in range(12):
        sp = _spec(rng)
        out = []
        for m in (ref, ours):
            P = m["planner"]
            res = _try(_build, m, sp)
            if res[0] == "err":
                out.append(res)
                continue
            model, par, layout = res[1]
            pec = P.PecConfig(k_pec=sp["k"])
            plans = {}
            for name, fn in (("equal", lambda: P.plan_equal(layout, pec)),
                             ("adaptive", lambda: P.plan_adaptive(layout, pec)),
                             ("baseline", lambda: P.plan_baseline(layout)),
                             ("equal_full", lambda: P.plan_equal(layout))):
                r = _try(fn)
                plans[name] = r if r[0] == "err" else ("ok", _plan(r[1]),
                                                       P.bottleneck_workload(r[1], 0))
            rng_due = random.Random(seed * 1000 + trial)
            dues = [{l: frozenset(rng_due.sample(range(sp["E"]), rng_due.randint(0, sp["E"])))
                     for l in range(sp["L"])} for _ in range(3)]
            phases = [_phase(P.build_phase_assignment(layout, due, s))
                      for due in dues for s in ("equal_pec", "adaptive_pec", "baseline")]
            sizes = (P.full_checkpoint_size(model), P.pec_checkpoint_size(model, sp["k"]),
                     P.pec_imbalance(model, par, sp["k"]))
            out.append(("ok", _units(layout), sorted(layout.nodes), plans, phases, sizes))
        assert out[0] == out[1], (seed, trial, sp)


@pytest.mark.parametrize("seed", range(10))
def test_random_selections_match_reference(ref, seed):
    ours = _ours()
    rng = random.Random(seed)
    for _ in range(40):
        n = rng.randint(1, 40)
        width, stride, c, m = rng.randint(1, n + 2), rng.randint(0, n + 2), rng.randint(0, 99), \
            rng.randint(0, 9)
        assert ref["selector"].select_window(c, m, n, width, stride) == \
            ours["selector"].select_window(c, m, n, width, stride)
        assert ref["selector"].schedule_period(n, max(1, stride), width) == \
            ours["selector"].schedule_period(n, max(1, stride), width)
        L = rng.randint(1, 3)
        counts = {(l, e): rng.choice([0, 1, 5, 5, 9, rng.randint(0, 10 ** 6)])
                  for l in range(L) for e in range(n)}
        k = rng.randint(1, n)
        pool = frozenset(rng.sample(range(n), rng.randint(1, n))) if rng.random() < 0.5 else None
        sels = []
        for mod in (ref, ours):
            lc = mod["selector"].LoadCounters(L, n)
            for (l, e), v in counts.items():
                lc.add(l, e, v)
            sels.append([mod["selector"].select_load_aware(lc, l, k, restrict_to=pool)
                         for l in range(L)])
        assert sels[0] == sels[1]
