"""Host mirror (topology/selector/planner) vs. the reference's own outputs.

tests/golden/plans.json and selection.json were produced by running the
reference (`mocsim`) on the same specs (tests/golden/make_golden.py)."""

import hashlib
import json

import pytest

from conftest import GOLDEN
from paper_2408_04307_b200 import (
    ClusterSpec,
    ModelSpec,
    ParallelSpec,
    PecConfig,
    bottleneck_workload,
    build_layout,
    build_phase_assignment,
    configs,
    full_checkpoint_size,
    ideal_rank_workload,
    pec_checkpoint_size,
    pec_imbalance,
    plan_adaptive,
    plan_baseline,
    plan_equal,
    select_load_aware,
    select_window,
    unit_sizes,
)
from paper_2408_04307_b200.selector import LoadCounters

PLANS = json.loads((GOLDEN / "plans.json").read_text())
SEL = json.loads((GOLDEN / "selection.json").read_text())


def digest(obj):
    return hashlib.sha256(json.dumps(obj, sort_keys=True).encode()).hexdigest()


def layout_doc(layout):
    units = [[u.key, u.kind, u.size_bytes, sorted(u.replica_ranks), u.layer, u.expert,
              u.module, u.rank] for u in layout.units]
    sizes = unit_sizes(layout.model, layout.parallel)
    return {
        "units_digest": digest(units), "n_units": len(units),
        "rank_info": {str(r): list(v) for r, v in sorted(layout.rank_info.items())},
        "hosted_digest": digest({str(r): sorted(map(list, s))
                                 for r, s in sorted(layout.hosted_experts.items())}),
        "unit_sizes": json.loads(json.dumps({k: v for k, v in sizes.items()
                                             if k != "non_expert_weight"})),
    }


def plan_doc(plan, full=False):
    doc = plan.to_json_dict()
    out = {"digest": digest(doc), "period": plan.period,
           "workload": [{str(r): w for r, w in sorted(p.items())} for p in plan.workload_bytes],
           "bottleneck": [list(bottleneck_workload(plan, c)) for c in range(plan.period)]}
    if full:
        out["plan"] = doc
    return out


def _workloads():
    wl = {"toy": configs.toy(), "gpt125m": configs.gpt125m_8e(),
          "mixtral": configs.mixtral_8x7b()}
    for k in (1, 2, 4, 8, 16):
        wl[f"gpt350m_k{k}"] = configs.gpt350m_16e(k_pec=k)
    return wl


@pytest.mark.parametrize("name", sorted(PLANS["workloads"]))
def test_workload_layouts_plans_and_sizes_match_reference(name):
    w = _workloads()[name]
    want = PLANS["workloads"][name]
    layout = w.layout()
    assert layout_doc(layout) == want["layout"]
    assert full_checkpoint_size(w.model) == want["full_size"]
    for k, v in want["pec_size"].items():
        assert pec_checkpoint_size(w.model, int(k)) == v
    assert ideal_rank_workload(w.model, layout.parallel) == want["ideal"]
    assert pec_imbalance(w.model, layout.parallel, w.pec.k_pec) == want["imbalance"]
    seq = PecConfig(k_pec=w.pec.k_pec)
    got = {"equal_pec": plan_doc(plan_equal(layout, seq), full=name == "toy"),
           "adaptive_pec": plan_doc(plan_adaptive(layout, seq)),
           "equal_full": plan_doc(plan_equal(layout)),
           "baseline": plan_doc(plan_baseline(layout))}
    assert got == want["plans"]


def _small_layout(case):
    m = case["model"]
    model = ModelSpec(**{**m, "non_expert_modules": tuple(map(tuple, m["non_expert_modules"]))})
    gpn = case["gpus_per_node"]
    cluster = ClusterSpec(num_nodes=case["dp"] // gpn, gpus_per_node=gpn,
                          snapshot_bandwidth=1e9, persist_bandwidth=1e8, fb_time=0.01,
                          update_time=0.002, restart_time=1.0)
    return build_layout(model, ParallelSpec(case["dp"], case["ep"]), cluster)


@pytest.mark.parametrize("i", range(len(PLANS["small"])))
def test_random_small_layouts_match_reference(i):
    case = PLANS["small"][i]
    layout = _small_layout(case)
    assert layout_doc(layout) == case["layout"]
    pec = PecConfig(k_pec=case["k_snapshot"], k_snapshot=case["k_snapshot"],
                    k_persist=case["k_persist"])
    assert plan_doc(plan_equal(layout, pec), full=True) == case["equal_pec"]
    assert plan_doc(plan_adaptive(layout, pec), full=True) == case["adaptive_pec"]
    assert plan_doc(plan_baseline(layout), full=True) == case["baseline"]
    due = {int(m): frozenset(v) for m, v in case["due"].items()}
    for strat, want in case["phase_by_strategy"].items():
        ph = build_phase_assignment(layout, due, strat)
        got = {str(r): [[a.key, a.start, a.stop, a.part] for a in v] for r, v in sorted(ph.items())}
        assert got == want, strat


def test_sequential_windows_match_reference():
    for c, m, n, width, stride, want in SEL["sequential"]:
        assert sorted(select_window(c, m, n, width, stride)) == want


def test_load_aware_matches_reference():
    for case in SEL["load_aware"]:
        n = len(case["counts"])
        lc = LoadCounters(1, n)
        for e, v in enumerate(case["counts"]):
            lc.add(0, e, v)
        got = sorted(select_load_aware(lc, 0, case["k"], restrict_to=case["pool"]))
        assert got == case["selected"]
