"""Generate the golden fixtures in tests/golden/ by running the REFERENCE.

Run in the authoring container, where the reference is mounted read-only:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every fixture is an output of `mocsim` (the reference package) on inputs
built from this repo's workload definitions (`paper_2408_04307_b200.configs`
only supplies module lists and sizes, converted into *reference* specs here).
The GPU box never reads /root/reference; tests read only these JSON files.
"""

from __future__ import annotations

import hashlib
import json
import random
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

import mocsim  # noqa: E402  (the reference)
from mocsim import planner as rp  # noqa: E402
from mocsim import selector as rs  # noqa: E402
from mocsim import store as rstore  # noqa: E402
from mocsim.engine import CheckpointEngine as RefEngine  # noqa: E402
from mocsim.scenario import RoutingSpec, Scenario  # noqa: E402

from paper_2408_04307_b200 import configs  # noqa: E402  (module lists only)


def digest(obj) -> str:
    return hashlib.sha256(json.dumps(obj, sort_keys=True).encode()).hexdigest()


def ref_model(m):
    return mocsim.ModelSpec(
        num_moe_layers=m.num_moe_layers, experts_per_layer=m.experts_per_layer,
        top_k=m.top_k, non_expert_params=m.non_expert_params,
        expert_params_per_expert=m.expert_params_per_expert, bytes_weight=m.bytes_weight,
        bytes_optim=m.bytes_optim, other_states_bytes=m.other_states_bytes,
        non_expert_modules=m.non_expert_modules)


def ref_cluster(num_nodes, gpn):
    return mocsim.ClusterSpec(num_nodes=num_nodes, gpus_per_node=gpn, snapshot_bandwidth=1e9,
                              persist_bandwidth=1e8, fb_time=0.01, update_time=0.002,
                              restart_time=1.0)


def make_model(n_experts=4, n_layers=2, top_k=1, p_ne=1000, epp=500, b_w=2, b_o=12,
               other=0, modules=None):
    if modules is None:
        modules = (("attn0", 400), ("ffn0", 350), ("attn1", 250))
    return dict(num_moe_layers=n_layers, experts_per_layer=n_experts, top_k=top_k,
                non_expert_params=p_ne, expert_params_per_expert=epp, bytes_weight=b_w,
                bytes_optim=b_o, other_states_bytes=other,
                non_expert_modules=[list(x) for x in modules])


def layout_doc(layout):
    units = [[u.key, u.kind, u.size_bytes, sorted(u.replica_ranks), u.layer, u.expert,
              u.module, u.rank] for u in layout.units]
    return {
        "units_digest": digest(units),
        "n_units": len(units),
        "rank_info": {str(r): list(v) for r, v in sorted(layout.rank_info.items())},
        "hosted_digest": digest({str(r): sorted(map(list, s))
                                 for r, s in sorted(layout.hosted_experts.items())}),
        "unit_sizes": {k: (v if not isinstance(v, dict) else v)
                       for k, v in mocsim.unit_sizes(layout.model, layout.parallel).items()
                       if k != "non_expert_weight"},
    }


def plan_doc(plan, full=False):
    doc = plan.to_json_dict()
    out = {"digest": digest(doc), "period": plan.period,
           "workload": [{str(r): w for r, w in sorted(p.items())} for p in plan.workload_bytes],
           "bottleneck": [list(rp.bottleneck_workload(plan, c)) for c in range(plan.period)]}
    if full:
        out["plan"] = doc
    return out


# ---------------------------------------------------------------------------

def gen_routing():
    cases = []
    for seed, it, L, E, tokens, top_k, s, cf in [
            (7, 1, 4, 8, 4096, 2, 1.1, 1.25), (7, 10, 6, 8, 16384, 2, 1.1, 1.25),
            (7, 3, 1, 4, 50, 2, 1.0, None), (1234, 5, 12, 16, 2000, 2, 1.2, 1.0),
            (7, 2, 32, 8, 16384, 2, 1.1, 1.25), (99, 7, 3, 64, 10007, 1, 0.7, 2.0)]:
        model = mocsim.ModelSpec(num_moe_layers=L, experts_per_layer=E, top_k=top_k,
                                 non_expert_params=1000, expert_params_per_expert=10,
                                 bytes_weight=2, bytes_optim=12)
        sc = Scenario(model=model, parallel=mocsim.ParallelSpec(1, 1),
                      cluster=ref_cluster(1, 1), strategy="equal_full", i_ckpt=1,
                      i_total=100, rng_seed=seed, tokens_per_iteration=tokens,
                      routing=RoutingSpec(kind="zipf", zipf_s=s), capacity_factor=cf)
        counts = mocsim.route_tokens(it, sc)
        cases.append({"seed": seed, "iteration": it, "layers": L, "experts": E,
                      "tokens": tokens, "top_k": top_k, "total": tokens * top_k, "s": s,
                      "capacity_factor": cf, "counts": counts.tolist()})
    return {"zipf": cases}


def gen_selection():
    seq = []
    for n in (1, 3, 4, 8, 16):
        for width in sorted({1, 2, n, max(1, n - 1)}):
            for stride in sorted({1, 2, width}):
                for c in (0, 1, 7, 33):
                    for m in range(5):
                        seq.append([c, m, n, width, stride,
                                    sorted(rs.select_window(c, m, n, width, stride))])
    rng = random.Random(20240804)
    la = [{"counts": [10, 40, 40, 5], "k": 2, "pool": None, "selected": [1, 2]},
          {"counts": [0, 0, 0, 0], "k": 1, "pool": None, "selected": [0]},
          {"counts": [1, 2, 3, 4], "k": 1, "pool": [0, 1], "selected": [1]}]
    for _ in range(200):
        n = rng.choice([1, 2, 4, 8, 16, 64])
        counts = [rng.choice([0, 1, 2, rng.randint(0, 10**9)]) for _ in range(n)]
        k = rng.randint(1, n)
        pool = None
        if rng.random() < 0.5:
            pool = sorted(rng.sample(range(n), rng.randint(1, n)))
        lc = rs.LoadCounters(1, n)
        for e, v in enumerate(counts):
            lc.add(0, e, v)
        sel = sorted(rs.select_load_aware(lc, 0, k, restrict_to=pool))
        la.append({"counts": counts, "k": k, "pool": pool, "selected": sel})
    return {"sequential": seq, "load_aware": la}


def gen_loadaware_sim():
    """Reference Simulation with load-aware selection: the per-checkpoint
    snapshot/persist sets (drives parity of hist -> select on device)."""
    traces = []
    for L, E, tokens, k_s, k_p, s, cf, seed in [(4, 8, 512, 2, 1, 1.1, 1.25, 7),
                                                (6, 8, 1024, 1, 1, 1.1, 1.25, 7),
                                                (3, 16, 700, 4, 2, 0.9, None, 11)]:
        model = mocsim.ModelSpec(num_moe_layers=L, experts_per_layer=E, top_k=2,
                                 non_expert_params=1000, expert_params_per_expert=100,
                                 bytes_weight=2, bytes_optim=12)
        pec = mocsim.PecConfig(k_pec=k_s, selection="load_aware", k_snapshot=k_s,
                               k_persist=k_p)
        sc = Scenario(model=model, parallel=mocsim.ParallelSpec(1, 1),
                      cluster=ref_cluster(1, 1), strategy="equal_pec", i_ckpt=5,
                      i_total=40, rng_seed=seed, tokens_per_iteration=tokens, pec=pec,
                      routing=RoutingSpec(kind="zipf", zipf_s=s), capacity_factor=cf)
        sim = mocsim.Simulation(sc)
        rec = []
        orig = sim._selections

        def spy(c, tiers, _orig=orig, _rec=rec):
            snap, persist = _orig(c, tiers)
            _rec.append({"c": c, "snap": [sorted(snap[m]) for m in sorted(snap)],
                         "persist": [sorted(persist[m]) for m in sorted(persist)]})
            return snap, persist
        sim._selections = spy
        for _ in range(sc.i_total):
            sim.step()
        traces.append({"layers": L, "experts": E, "tokens": tokens, "top_k": 2,
                       "k_snapshot": k_s, "k_persist": k_p, "zipf_s": s,
                       "capacity_factor": cf, "seed": seed, "i_ckpt": 5, "i_total": 40,
                       "checkpoints": rec})
    return {"traces": traces}


def gen_fault_sim():
    """Reference Simulation with load-aware selection on 2 nodes and scripted
    node faults: per-checkpoint selections (including the checkpoints of
    replayed iterations), and for every fault the recovery decisions, the
    restart point / skew and both counter tiers after the reset
    (simulator.py:473-544) -- drives parity of PecCheckpointer.recover."""
    from mocsim.scenario import FaultSpec
    traces = []
    for L, E, tokens, k_s, k_p, seed, events in [
            (3, 4, 600, 2, 1, 5, ((13, (1,)), (27, (0,)))),
            (2, 8, 800, 2, 2, 9, ((8, (1,)), (21, (1,)), (33, (0,))))]:
        model = mocsim.ModelSpec(num_moe_layers=L, experts_per_layer=E, top_k=2,
                                 non_expert_params=1000, expert_params_per_expert=100,
                                 bytes_weight=2, bytes_optim=12)
        pec = mocsim.PecConfig(k_pec=k_s, selection="load_aware", k_snapshot=k_s,
                               k_persist=k_p)
        sc = Scenario(model=model, parallel=mocsim.ParallelSpec(2, 2),
                      cluster=ref_cluster(2, 1), strategy="equal_pec", i_ckpt=5,
                      i_total=40, rng_seed=seed, tokens_per_iteration=tokens, pec=pec,
                      routing=RoutingSpec(kind="zipf", zipf_s=1.1), capacity_factor=1.25,
                      faults=FaultSpec(kind="scripted", events=events))
        sim = mocsim.Simulation(sc)
        rec, faults = [], []
        orig_sel, orig_fault = sim._selections, sim._handle_fault

        def spy(c, tiers, _orig=orig_sel, _rec=rec):
            snap, persist = _orig(c, tiers)
            _rec.append({"c": c, "snap": [sorted(snap[m]) for m in sorted(snap)],
                         "persist": [sorted(persist[m]) for m in sorted(persist)]})
            return snap, persist

        def fault_spy(iteration, failed, _orig=orig_fault, _sim=sim, _faults=faults):
            plan = None
            if _sim.store.newest_complete() is not None:
                plan = _sim.engine.resolve_recovery(failed, max_iteration=iteration)
            _orig(iteration, failed)
            fr = _sim.fault_records[-1]
            _faults.append({
                "iteration": iteration, "failed": sorted(failed),
                "restart": fr.restart_iteration, "skew": fr.version_skew,
                "decisions": None if plan is None else {
                    k: [d.source, d.node, d.version, d.restored_iteration]
                    for k, d in sorted(plan.decisions.items())},
                "snap_counters": [[_sim.snap_counters.unsaved_tokens[(m, e)] for e in range(E)]
                                  for m in range(L)],
                "persist_counters": [[_sim.persist_counters.unsaved_tokens[(m, e)]
                                      for e in range(E)] for m in range(L)]})
        sim._selections = spy
        sim._handle_fault = fault_spy
        n_steps = 0
        while sim.next_iteration <= sc.i_total and n_steps < 500:
            sim.step()
            n_steps += 1
        traces.append({"layers": L, "experts": E, "tokens": tokens, "top_k": 2,
                       "k_snapshot": k_s, "k_persist": k_p, "zipf_s": 1.1,
                       "capacity_factor": 1.25, "seed": seed, "i_ckpt": 5, "i_total": 40,
                       "events": [[it, list(n)] for it, n in events],
                       "checkpoints": rec, "faults": faults})
    return {"traces": traces}


def gen_plans():
    out = {"workloads": {}, "small": []}
    wl = {"toy": configs.toy(), "gpt125m": configs.gpt125m_8e(),
          "mixtral": configs.mixtral_8x7b()}
    for k in (1, 2, 4, 8, 16):
        wl[f"gpt350m_k{k}"] = configs.gpt350m_16e(k_pec=k)
    for name, w in wl.items():
        model = ref_model(w.model)
        layout = mocsim.build_layout(model, mocsim.ParallelSpec(w.parallel.dp_degree,
                                                                w.parallel.ep_degree),
                                     ref_cluster(w.cluster.num_nodes, w.cluster.gpus_per_node))
        k = w.pec.k_pec
        doc = {"layout": layout_doc(layout),
               "full_size": rp.full_checkpoint_size(model),
               "pec_size": {str(kk): rp.pec_checkpoint_size(model, kk)
                            for kk in sorted({1, k, model.experts_per_layer})},
               "ideal": rp.ideal_rank_workload(model, layout.parallel),
               "imbalance": rp.pec_imbalance(model, layout.parallel, k),
               "plans": {}}
        seq = mocsim.PecConfig(k_pec=k)
        doc["plans"]["equal_pec"] = plan_doc(rp.plan_equal(layout, seq), full=name == "toy")
        doc["plans"]["adaptive_pec"] = plan_doc(rp.plan_adaptive(layout, seq))
        doc["plans"]["equal_full"] = plan_doc(rp.plan_equal(layout))
        doc["plans"]["baseline"] = plan_doc(rp.plan_baseline(layout))
        out["workloads"][name] = doc
    rng = random.Random(4307)
    for i in range(60):
        n = rng.choice([2, 3, 4, 6, 8])
        ep = rng.choice([d for d in (1, 2, 3, 4, 8) if n % d == 0])
        groups = rng.randint(1, 3)
        dp = ep * groups
        n_mod = rng.randint(1, 6)
        mods = [(f"m{j}", rng.randint(1, 900)) for j in range(n_mod)]
        mkw = make_model(n_experts=n, n_layers=rng.randint(1, 4), p_ne=sum(c for _, c in mods),
                         epp=rng.choice([0, 1, 7, 100, 1001]), b_w=rng.choice([1, 2, 4]),
                         b_o=rng.choice([4, 8, 12]), other=rng.choice([0, 0, 5, 97]),
                         modules=mods)
        gpn = rng.choice([d for d in (1, 2, 3, 4) if dp % d == 0])
        model = mocsim.ModelSpec(**{**mkw, "non_expert_modules": tuple(map(tuple, mods))})
        layout = mocsim.build_layout(model, mocsim.ParallelSpec(dp, ep),
                                     ref_cluster(dp // gpn, gpn))
        k_s = rng.randint(1, n)
        k_p = rng.randint(1, k_s)
        pec = mocsim.PecConfig(k_pec=k_s, k_snapshot=k_s, k_persist=k_p)
        due = {m: frozenset(rng.sample(range(n), rng.randint(0, n)))
               for m in range(model.num_moe_layers)}
        case = {"model": mkw, "dp": dp, "ep": ep, "gpus_per_node": gpn,
                "k_snapshot": k_s, "k_persist": k_p,
                "layout": layout_doc(layout),
                "equal_pec": plan_doc(rp.plan_equal(layout, pec), full=True),
                "adaptive_pec": plan_doc(rp.plan_adaptive(layout, pec), full=True),
                "baseline": plan_doc(rp.plan_baseline(layout), full=True),
                "due": {str(m): sorted(v) for m, v in due.items()},
                "phase_by_strategy": {}}
        for strat in ("baseline", "equal_pec", "adaptive_pec"):
            ph = rp.build_phase_assignment(layout, due, strat)
            case["phase_by_strategy"][strat] = {
                str(r): [[a.key, a.start, a.stop, a.part] for a in v]
                for r, v in sorted(ph.items())}
        out["small"].append(case)
    return out


def gen_store():
    entries = [
        rstore.StoreEntry("ew.L0.E0", rank=0, unit_key="ew.L0.E0", start=0, stop=100),
        rstore.StoreEntry("ew.L0.E1.part0", rank=0, unit_key="ew.L0.E1", start=0, stop=50),
        rstore.StoreEntry("ew.L0.E1.part1", rank=1, unit_key="ew.L0.E1", start=50, stop=100),
        rstore.StoreEntry("ew.L10.E1", rank=1, unit_key="ew.L10.E1", start=0, stop=64),
        rstore.StoreEntry("neo.r0", rank=0, unit_key="neo.r0", start=0, stop=64),
        rstore.StoreEntry("neo.r1", rank=1, unit_key="neo.r1", start=0, stop=64),
    ]
    with tempfile.TemporaryDirectory() as d:
        st = rstore.DiskStore(d)
        st.write_version(3, iteration=17, checkpoint_index=2, entries=entries)
        vdir = Path(d) / "v000003"
        files = sorted(str(p.relative_to(vdir)) for p in vdir.rglob("*") if p.is_file())
        doc = {"entries": [list(e) for e in entries],
               "meta_json": (vdir / "meta.json").read_text(),
               "manifest_tsv": (vdir / "manifest.tsv").read_text(),
               "files": files,
               "payload_crc": {e.store_key: rstore.crc32c(rstore.entry_payload(e.store_key, 3, 17))
                               for e in entries}}
    rng = np.random.default_rng(49)
    crc = []
    for n in (0, 1, 3, 8, 9, 15, 16, 17, 100, 4096, 24575, 24577, 100003):
        b = rng.bytes(n)
        crc.append({"seed_len": n, "hex": b.hex() if n <= 64 else None,
                    "sha": hashlib.sha256(b).hexdigest(), "crc": rstore.crc32c(b)})
    doc["crc_vectors"] = crc
    doc["crc_seed"] = 49
    return doc


def gen_recovery():
    """Reference recovery decisions after scripted snapshot/persist cycles."""
    cases = []
    rng = random.Random(1234)
    for trial in range(40):
        n = rng.choice([2, 4])
        ep = n
        dp = rng.choice([n, 2 * n]) if n == 2 else n
        ep = min(ep, dp)
        model_kw = make_model(n_experts=n, n_layers=rng.randint(1, 2), epp=rng.choice([80, 101]))
        model = mocsim.ModelSpec(**{**model_kw,
                                    "non_expert_modules": tuple(map(tuple, model_kw["non_expert_modules"]))})
        gpn = 2
        layout = mocsim.build_layout(model, mocsim.ParallelSpec(dp, ep), ref_cluster(dp // gpn, gpn))
        k_s = rng.choice([1, 2, n])
        k_p = rng.randint(1, k_s)
        pec = mocsim.PecConfig(k_pec=k_s, k_snapshot=k_s, k_persist=k_p)
        plan = rp.plan_equal(layout, pec)
        eng = RefEngine(layout, mocsim.MemoryStore())
        ops = []
        n_ck = rng.randint(1, 6)
        for c in range(n_ck):
            it = (c + 1) * 10
            buf = eng.begin_snapshot(it, c, plan.assignments[plan.phase_of(c)])
            promoted = eng.complete_snapshot(buf)
            sel = {m: rs.select_window(c, m, n, k_p, k_p) for m in range(model.num_moe_layers)}
            do_persist = promoted is not None and rng.random() < 0.8
            if do_persist:
                entries = eng.persist_entries(buf, sel)
                eng.complete_persist(buf, entries)
            ops.append({"c": c, "iteration": it, "persisted": do_persist})
            if not do_persist:
                break
        failed = sorted(rng.sample(layout.nodes, rng.randint(0, len(layout.nodes) - 1)))
        max_it = rng.choice([None, 25, 1000])
        try:
            plan_r = eng.resolve_recovery(set(failed), max_iteration=max_it)
            dec = {k: list(v) for k, v in sorted(plan_r.decisions.items())}
            res = {"decisions": dec, "restart_iteration": plan_r.restart_iteration,
                   "version_skew": plan_r.version_skew}
        except Exception as e:  # noqa: BLE001
            res = {"error": type(e).__name__}
        cases.append({"model": model_kw, "dp": dp, "ep": ep, "gpus_per_node": gpn,
                      "k_snapshot": k_s, "k_persist": k_p, "ops": ops, "failed": failed,
                      "max_iteration": max_it, "result": res})
    return {"cases": cases}


def gen_policy():
    """Reference adaptive_configure / analytic_overhead on a grid."""
    from mocsim import adaptive_configure, analytic_overhead
    from mocsim.planner import PecConfig as RPec
    cases = []
    rng = random.Random(740)
    specs = [("gpt350m", configs.gpt350m_16e(k_pec=2)), ("toy", configs.toy()),
             ("mixtral", configs.mixtral_8x7b())]
    for name, w in specs:
        model = ref_model(w.model)
        for strategy in ("equal_pec", "adaptive_pec"):
            for _ in range(4):
                snap_bw = 10 ** rng.uniform(8.5, 12.5)
                pers_bw = 10 ** rng.uniform(8, 10.5)
                fb = rng.choice([0.05, 0.3, 1.0])
                upd = rng.choice([0.01, 0.05])
                target = rng.choice([None, 1.0, 10.0, 60.0])
                cl = mocsim.ClusterSpec(num_nodes=w.cluster.num_nodes,
                                        gpus_per_node=w.cluster.gpus_per_node,
                                        snapshot_bandwidth=snap_bw, persist_bandwidth=pers_bw,
                                        fb_time=fb, update_time=upd, restart_time=1.0)
                sc = Scenario(model=model, parallel=mocsim.ParallelSpec(w.parallel.dp_degree,
                                                                        w.parallel.ep_degree),
                              cluster=cl, strategy=strategy, i_ckpt=1, i_total=10, rng_seed=7,
                              tokens_per_iteration=100, pec=RPec(k_pec=1))
                cfg = adaptive_configure(sc, persist_target_s=target)
                cases.append({"workload": name, "strategy": strategy, "snapshot_bw": snap_bw,
                              "persist_bw": pers_bw, "fb": fb, "update": upd, "target": target,
                              "k_snapshot": cfg.pec.k_snapshot, "k_persist": cfg.pec.k_persist,
                              "i_ckpt": cfg.i_ckpt, "overlapped": cfg.snapshot_overlapped,
                              "target_met": cfg.persist_target_met})
    ana = []
    for _ in range(50):
        kw = dict(o_save_full_us=rng.uniform(1e3, 1e7), i_ckpt_full=rng.randint(1, 100),
                  o_save_moc_us=rng.uniform(1e2, 1e6), i_ckpt_moc=rng.randint(1, 100),
                  iter_time_us=rng.uniform(1e4, 1e7), failure_rate=rng.uniform(0, 0.01),
                  o_restart_us=rng.uniform(1e5, 1e8), i_total=rng.randint(100, 100000))
        r = analytic_overhead(**kw)
        ana.append({"args": kw, "full": r.o_ckpt_full_us, "moc": r.o_ckpt_moc_us,
                    "wins": r.moc_wins})
    return {"configure": cases, "analytic": ana}


def main():
    HERE.mkdir(exist_ok=True)
    for name, fn in [("routing", gen_routing), ("selection", gen_selection),
                     ("loadaware_sim", gen_loadaware_sim), ("fault_sim", gen_fault_sim),
                     ("plans", gen_plans),
                     ("store", gen_store), ("recovery", gen_recovery),
                     ("policy", gen_policy)]:
        doc = fn()
        doc["_generated_by"] = "tests/golden/make_golden.py (reference mocsim 0.1.0)"
        (HERE / f"{name}.json").write_text(json.dumps(doc, indent=None, sort_keys=True) + "\n")
        print(name, (HERE / f"{name}.json").stat().st_size)


if __name__ == "__main__":
    main()
