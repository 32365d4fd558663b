"""Differential check of the two-level manager against the reference itself:
the same random operation sequences (checkpoint, snapshot completion,
persist of a random expert subset, node faults, recovery resolution) drive
the reference `mocsim.engine.CheckpointEngine` and this package's
`engine.CheckpointEngine`, and every observable result must agree — buffer
roles, versions, persist entry lists, published versions, recovery decisions
and the exceptions raised (rows a11, a12, a14 of SURVEY.md §8(a);
reference engine.py:71-293).

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
                for m in ("topology", "planner", "engine", "store")}
    finally:
        sys.path.remove(str(REF_SRC))
    assert "tests/compat" not in mods["engine"].__file__
    return mods


def _ours():
    from paper_2408_04307_b200 import engine, planner, store, topology
    return {"topology": topology, "planner": planner, "engine": engine, "store": store}


def _layout(m, n_experts, n_layers, dp, ep, gpn):
    T = m["topology"]
    modules = (("embed", 700), ("attn0", 400), ("ffn_ne", 350), ("attn1", 250), ("lnf", 16))
    model = T.ModelSpec(num_moe_layers=n_layers, experts_per_layer=n_experts, top_k=1,
                        non_expert_params=sum(c for _, c in modules),
                        expert_params_per_expert=300 + 7 * n_experts, bytes_weight=2,
                        bytes_optim=12, other_states_bytes=40, non_expert_modules=modules)
    cluster = T.ClusterSpec(num_nodes=dp // gpn, gpus_per_node=gpn, snapshot_bandwidth=1e9,
                            persist_bandwidth=1e8, fb_time=0.01, update_time=0.002,
                            restart_time=1.0)
    return T.build_layout(model, T.ParallelSpec(dp_degree=dp, ep_degree=ep), cluster)


def _state(eng):
    return [(b.buffer_id, b.status, b.version, b.iteration, b.checkpoint_index,
             tuple(sorted(b.valid_nodes))) for b in eng.buffers.buffers]


def _call(fn, *a, **kw):
    try:
        return ("ok", fn(*a, **kw))
    except Exception as exc:  # the exception TYPE is part of the contract
        return ("err", type(exc).__name__)


def _bid(buf):
    return None if buf is None else buf.buffer_id


CASES = [  # n_experts, n_layers, dp, ep, gpus_per_node, k_pec, strategy
    (4, 2, 4, 2, 2, 1, "equal_pec"), (8, 1, 4, 4, 1, 2, "adaptive_pec"),
    (4, 3, 4, 4, 2, 2, "equal_pec"), (2, 2, 2, 2, 1, 1, "baseline"),
    (8, 2, 8, 4, 2, 3, "adaptive_pec"), (6, 1, 4, 2, 2, 2, "equal_pec"),
]


@pytest.mark.parametrize("case", range(len(CASES)))
@pytest.mark.parametrize("seed", range(6))
def test_random_operation_sequences_match_reference_engine(ref, case, seed):
    ours = _ours()
    E, L, dp, ep, gpn, k, strategy = CASES[case]
    sides = []
    for m in (ref, ours):
        layout = _layout(m, E, L, dp, ep, gpn)
        P = m["planner"]
        if strategy == "baseline":
            plan = P.plan_baseline(layout)
        elif strategy == "adaptive_pec":
            plan = P.plan_adaptive(layout, P.PecConfig(k_pec=k))
        else:
            plan = P.plan_equal(layout, P.PecConfig(k_pec=k))
        eng = m["engine"].CheckpointEngine(layout, m["store"].MemoryStore())
        sides.append((layout, plan, eng))
    nodes = list(sides[0][0].nodes)
    rng = random.Random(1000 * case + seed)
    it, c = 0, 0
    for step in range(80):
        op = rng.choice(["ckpt", "ckpt", "snap", "snap", "persist", "persist", "fault",
                         "recover"])
        failed = set(rng.sample(nodes, rng.randint(1, max(1, len(nodes) - 1))))
        keep = {m_: frozenset(rng.sample(range(E), rng.randint(0, E))) for m_ in range(L)}
        max_it = rng.choice([None, it, max(0, it - 2)])
        outs = []
        for layout, plan, eng in sides:
            if op == "ckpt":
                a = plan.assignments[plan.phase_of(c)]
                r = _call(eng.begin_snapshot, it + 1, c, a)
                out = (r[0], _bid(r[1]) if r[0] == "ok" else r[1])
            elif op == "snap":
                b = eng.buffers.snapshotting
                out = None if b is None else _call(lambda: _bid(eng.complete_snapshot(b)))
            elif op == "persist":
                b = eng.buffers.persisting
                if b is None:
                    out = None
                else:
                    entries = eng.persist_entries(b, keep)
                    rows = [(e.store_key, e.rank, e.unit_key, e.start, e.stop) for e in entries]
                    out = (rows, _call(lambda: _bid(eng.complete_persist(b, entries))))
            elif op == "fault":
                out = _call(eng.on_fault, failed)
            else:
                r = _call(eng.resolve_recovery, failed, max_iteration=max_it)
                if r[0] == "ok":
                    p = r[1]
                    out = ("ok", sorted((u, tuple(d)) for u, d in p.decisions.items()),
                           p.restart_iteration, p.version_skew)
                else:
                    out = r
            outs.append((out, _state(eng), eng.store.complete_versions(), eng.next_version))
        assert outs[0] == outs[1], (step, op)
        if op == "ckpt" and outs[0][0][0] == "ok":
            it, c = it + 1, c + 1
        elif op == "ckpt":
            it += 1
