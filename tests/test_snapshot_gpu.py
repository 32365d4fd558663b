"""End-to-end PEC snapshot path on the GPU: counting -> selection -> pack ->
drain -> persist -> (fault) -> resolve_recovery -> restore, bit-exact."""

import json

import numpy as np
import pytest

from conftest import GOLDEN, make_layout
from oracle import pec_oracle as O

pytestmark = pytest.mark.gpu


def _expected_entries(host_state, arena, assignment, ranks):
    """Oracle: each planned range's bytes from a host copy of the state."""
    out = {}
    for r in ranks:
        for a in assignment.get(r, ()):
            src = arena.slot(a.key).offset + a.start
            out[a.store_key] = bytes(host_state[src:src + a.stop - a.start])
    return out


def _mutate(arena, step):
    """Stand-in for an optimizer step: perturb every resident unit."""
    import torch
    for key, s in arena.slots.items():
        v = arena.buffer[s.offset:s.offset + s.size]
        v[:: 97].add_(step + 1)


@pytest.mark.parametrize("drain_first,recycle", [(None, False), (100_003, False), (None, True)])
def test_toy_sequential_chain_persists_exact_bytes(dev, tmp_path, drain_first, recycle):
    """drain_first=100_003: the pipelined drain splits every pack at odd
    staging offsets (~8 segments, rows cut mid-copy, unaligned pieces).
    recycle: superseded versions are retired during the chain and later
    versions overwrite their files in place; what remains is exact."""
    import torch
    from paper_2408_04307_b200 import configs
    from paper_2408_04307_b200.arena import StateArena
    from paper_2408_04307_b200.snapshot import PecCheckpointer
    from paper_2408_04307_b200.store import DiskStore
    w = configs.toy()
    layout = w.layout()
    arena = StateArena(layout, [0], dev, w.expert_tensors)
    store = DiskStore(tmp_path, recycle=recycle)
    ck = PecCheckpointer(layout, arena, store, w.pec, w.strategy, i_ckpt=5)
    if drain_first is not None:
        ck.engine.drain_first = drain_first
    ck.prepare()        # staging, pinned buffers and every phase's table up front
    assert len(ck.engine._tables) == ck.plan().period
    segs = [t[0].segments for t in ck.engine._tables.values()]
    assert all((s is None) == (drain_first is None) for s in segs)
    if drain_first is not None:
        assert min(len(s) for s in segs) >= 5
    expected = {}
    for it in range(1, 31):
        _mutate(arena, it)  # "optimizer step" of iteration it
        buf = ck.step(it)
        if buf is not None:
            torch.cuda.synchronize()
            expected[buf.version] = (_expected_entries(arena.buffer.cpu().numpy(), arena,
                                                       buf.content, [0]), buf.iteration)
            ck.wait_pack()  # next update must not race the pack
            if recycle:
                for old in store.complete_versions()[:-1]:
                    store.retire(old)
    ck.finish()
    versions = store.complete_versions()
    if recycle:
        assert versions and set(versions) <= set(expected) and versions[-1] == max(expected)
        assert store.recycled_files > 0
    else:
        assert versions == sorted(expected)
    for v in versions:
        got = store.load_checkpoint(v)
        want, it = expected[v]
        persist = ck.persist_sel[v]
        assert store.meta(v).iteration == it
        for k, data in got.items():
            assert data == want[k], (v, k)
        # persisted = non-expert + K_persist experts of each layer
        ks = {k.split(".")[0] for k in got}
        assert {"neo", "new"} <= ks
    ck.close()


def test_multirank_fault_and_partial_expert_restore(dev, tmp_path):
    """4 ranks on 2 nodes emulated in one process, two EP groups (byte-split
    expert weights), snapshot window 2 / persist 1.  After a fault on node 0
    every unit is restored bit-identically from memory, storage or its
    initial image, as resolve_recovery decides."""
    import torch
    from paper_2408_04307_b200 import PecConfig
    from paper_2408_04307_b200.arena import StateArena
    from paper_2408_04307_b200.restore import restore
    from paper_2408_04307_b200.snapshot import PecCheckpointer
    from paper_2408_04307_b200.store import DiskStore
    layout = make_layout(n_experts=4, dp=4, ep=2, gpus_per_node=2, n_layers=2, epp=30_001,
                         p_ne=3_001, modules=(("a", 1000), ("b", 1001), ("c", 1000)), other=33)
    arena = StateArena(layout, range(4), dev)
    initial = arena.buffer.cpu().numpy().copy()
    store = DiskStore(tmp_path)
    pec = PecConfig(k_pec=2, k_snapshot=2, k_persist=1)
    ck = PecCheckpointer(layout, arena, store, pec, "equal_pec", i_ckpt=10, async_persist=False)
    snaps = {}
    for it in range(1, 41):
        _mutate(arena, it)
        buf = ck.step(it)
        if buf is not None:
            torch.cuda.synchronize()
            snaps[buf.version] = arena.buffer.cpu().numpy().copy()
            ck.wait_pack()
    ck.finish()
    assert store.complete_versions()
    plan = ck.engine.resolve_recovery({0})
    ck.engine.on_fault({0})
    arena.buffer.zero_()
    rep = restore(ck.engine, plan)
    torch.cuda.synchronize()
    now = arena.buffer.cpu().numpy()
    sources = set()
    for key, d in plan.decisions.items():
        if not arena.has(key):
            continue
        s = arena.slot(key)
        got = now[s.offset:s.offset + s.size]
        ref = initial if d.source == "initial" else snaps[d.version]
        assert np.array_equal(got, ref[s.offset:s.offset + s.size]), (key, d)
        sources.add(d.source)
    assert {"memory", "storage"} <= sources
    assert rep.units == len(arena.slots)
    ck.close()


def test_device_load_aware_chain_matches_reference_simulation(dev, tmp_path):
    """Router ids from the reference's Zipf stream, counted and selected on
    device, reproduce the reference Simulation's snapshot/persist sets at
    every checkpoint (golden loadaware_sim.json)."""
    import torch
    from paper_2408_04307_b200 import ModelSpec, ParallelSpec, ClusterSpec, PecConfig, build_layout
    from paper_2408_04307_b200.arena import StateArena
    from paper_2408_04307_b200.counting import DeviceTokenCounters
    from paper_2408_04307_b200.snapshot import PecCheckpointer
    from paper_2408_04307_b200.store import MemoryStore
    g = json.loads((GOLDEN / "loadaware_sim.json").read_text())
    for t in g["traces"]:
        L, E = t["layers"], t["experts"]
        model = ModelSpec(num_moe_layers=L, experts_per_layer=E, top_k=2, non_expert_params=1000,
                          expert_params_per_expert=100, bytes_weight=2, bytes_optim=12)
        layout = build_layout(model, ParallelSpec(1, 1), ClusterSpec(1, 1))
        arena = StateArena(layout, [0], dev)
        total = t["tokens"] * t["top_k"]
        cap = DeviceTokenCounters.capacity_for(t["capacity_factor"], [total] * L, E)
        counters = DeviceTokenCounters(L, E, dev, cap)
        pec = PecConfig(k_pec=t["k_snapshot"], selection="load_aware",
                        k_snapshot=t["k_snapshot"], k_persist=t["k_persist"])
        ck = PecCheckpointer(layout, arena, MemoryStore(), pec, "equal_pec", i_ckpt=t["i_ckpt"],
                             counters=counters)
        got = []
        for i in range(1, t["i_total"] + 1):
            ids = np.stack([O.zipf_router_ids(t["seed"], i, m, E, total, t["zipf_s"])
                            for m in range(L)])
            buf = ck.step(i, torch.from_numpy(ids).to(dev))
            if buf is not None:
                ck.resolve(buf)
                snap = {m: set() for m in range(L)}
                for a in buf.content[0]:
                    u = layout.by_key[a.key]
                    if u.layer is not None:
                        snap[u.layer].add(u.expert)
                got.append({"c": buf.checkpoint_index,
                            "snap": [sorted(snap[m]) for m in range(L)],
                            "persist": [sorted(ck.persist_sel[buf.version][m]) for m in range(L)]})
        ck.close()
        assert got == t["checkpoints"]


def test_recover_matches_reference_fault_simulation(dev, tmp_path):
    """PecCheckpointer.recover reproduces the reference's fault handling
    (Simulation._handle_fault, simulator.py:473-544) on a 2-node load-aware
    run with scripted node faults (golden trace): the recovery decisions,
    restart point and skew of every fault, both counter tiers after the
    reset, and every checkpoint's selections before and after (including
    replayed iterations) -- with the bytes actually restored."""
    import json
    import torch
    from conftest import GOLDEN
    from paper_2408_04307_b200 import (ClusterSpec, ModelSpec, ParallelSpec, PecConfig,
                                       build_layout)
    from paper_2408_04307_b200.arena import StateArena
    from paper_2408_04307_b200.counting import DeviceTokenCounters
    from paper_2408_04307_b200.snapshot import PecCheckpointer
    from paper_2408_04307_b200.store import DiskStore
    g = json.loads((GOLDEN / "fault_sim.json").read_text())
    for ti, t in enumerate(g["traces"]):
        L, E = t["layers"], t["experts"]
        model = ModelSpec(num_moe_layers=L, experts_per_layer=E, top_k=t["top_k"],
                          non_expert_params=1000, expert_params_per_expert=100,
                          bytes_weight=2, bytes_optim=12)
        layout = build_layout(model, ParallelSpec(2, 2), ClusterSpec(2, 1))
        arena = StateArena(layout, [0, 1], dev)
        total = t["tokens"] * t["top_k"]
        counters = DeviceTokenCounters(
            L, E, dev, DeviceTokenCounters.capacity_for(t["capacity_factor"], [total] * L, E))
        pec = PecConfig(k_pec=t["k_snapshot"], selection="load_aware",
                        k_snapshot=t["k_snapshot"], k_persist=t["k_persist"])
        ck = PecCheckpointer(layout, arena, DiskStore(tmp_path / f"t{ti}"), pec, "equal_pec",
                             i_ckpt=t["i_ckpt"], counters=counters)
        events = {it: set(n) for it, n in t["events"]}
        got_ckpts, got_faults = [], []
        it, steps = 1, 0
        while it <= t["i_total"] and steps < 500:
            steps += 1
            ids = np.stack([O.zipf_router_ids(t["seed"], it, m, E, total, t["zipf_s"])
                            for m in range(L)])
            buf = ck.step(it, torch.from_numpy(ids).to(dev))
            if buf is not None:
                ck.resolve(buf)
                snap = {m: set() for m in range(L)}
                for ranges in buf.content.values():
                    for a in ranges:
                        u = layout.by_key[a.key]
                        if u.layer is not None:
                            snap[u.layer].add(u.expert)
                got_ckpts.append({"c": buf.checkpoint_index,
                                  "snap": [sorted(snap[m]) for m in range(L)],
                                  "persist": [sorted(ck.persist_sel[buf.version][m])
                                              for m in range(L)]})
                ck.wait_pack()
            if it in events:
                ck.finish()  # the reference's tiny persists have landed by now
                out = ck.recover(events.pop(it), it)
                torch.cuda.synchronize()
                cnt = counters.counts.cpu().tolist()
                got_faults.append({
                    "restart": out.restart_iteration, "skew": out.version_skew,
                    "decisions": None if out.plan is None else {
                        k: [d.source, d.node, d.version, d.restored_iteration]
                        for k, d in sorted(out.plan.decisions.items())},
                    "snap_counters": cnt[0], "persist_counters": cnt[1]})
                assert out.report is None or out.report.units == len(arena.slots)
                it = out.restart_iteration + 1
            else:
                it += 1
        ck.close()
        want = [{k: f[k] for k in ("restart", "skew", "decisions", "snap_counters",
                                   "persist_counters")} for f in t["faults"]]
        assert got_faults == want, ti
        assert got_ckpts == t["checkpoints"], ti


def test_recover_before_any_complete_version_restarts_from_scratch(dev, tmp_path):
    """No COMPLETE version yet: restart iteration 0, every unit back to its
    initial image, buffers dropped, counters zeroed (simulator.py:476-483)."""
    import torch
    from paper_2408_04307_b200 import PecConfig, configs
    from paper_2408_04307_b200.arena import StateArena
    from paper_2408_04307_b200.counting import DeviceTokenCounters
    from paper_2408_04307_b200.engine import FREE
    from paper_2408_04307_b200.snapshot import PecCheckpointer
    from paper_2408_04307_b200.store import DiskStore
    w = configs.toy()
    layout = w.layout()
    L, E = layout.model.num_moe_layers, layout.model.experts_per_layer
    arena = StateArena(layout, [0], dev, w.expert_tensors)
    initial = arena.buffer.cpu().numpy().copy()
    counters = DeviceTokenCounters(L, E, dev)
    pec = PecConfig(k_pec=1, selection="load_aware")
    ck = PecCheckpointer(layout, arena, DiskStore(tmp_path), pec, "equal_pec", i_ckpt=5,
                         counters=counters)
    for it in range(1, 4):
        _mutate(arena, it)
        ck.step(it, torch.randint(0, E, (L, 128), dtype=torch.int32, device=dev))
    out = ck.recover({0}, 3)
    torch.cuda.synchronize()
    assert out.restart_iteration == 0 and out.plan is None
    assert np.array_equal(arena.buffer.cpu().numpy(), initial)
    assert int(counters.counts.abs().sum()) == 0
    assert all(b.status == FREE for b in ck.engine.buffers.buffers)
    ck.close()


@pytest.mark.parametrize("engine", ["bulk", "crc"])
def test_mixtral_rank_full_size_pack_unpack_bit_exact(dev, engine):
    """The headline configuration at full size (Mixtral-shaped rank 0, 84.5 GB
    resident, every phase of the adaptive K=1 plan, up to 12.9 GB per
    checkpoint): each staged entry equals its source range, the device CRCs
    of the CRC engine equal CRCs of the source ranges taken by a second
    kernel pass, the staged total equals the planner workload, and an
    unpack into the wiped ranges restores them bit-exactly (device-side
    comparisons; sizes where a CPU oracle pass would take minutes)."""
    import torch
    from paper_2408_04307_b200 import configs, plan_adaptive
    from paper_2408_04307_b200 import device as D
    from paper_2408_04307_b200.arena import StateArena
    from paper_2408_04307_b200.staging import DeviceTable, StagingLayout
    w = configs.mixtral_8x7b()
    layout = w.layout()
    plan = plan_adaptive(layout, w.pec)
    arena = StateArena(layout, [0], dev, w.expert_tensors)
    lg = D.DEFAULT_CHUNK_LOG2
    phases = range(plan.period) if engine == "bulk" else [0]
    staging = None
    for ph in phases:
        st = StagingLayout.build(plan.assignments[ph][0], arena, 0)
        assert st.payload_bytes == plan.workload_bytes[ph][0]
        if staging is None or staging.numel() < st.nbytes:
            staging = None
            torch.cuda.empty_cache()
            staging = torch.empty(st.nbytes + 256, dtype=torch.uint8, device=dev)
        table, total = st.descriptors(arena.base_address, staging.data_ptr(), chunk_log2=lg)
        dt = DeviceTable(table, total, dev, lg)
        if engine == "bulk":
            D.pack(dt.tensor, dt.n, dt.total_chunks, lg, D.MODE_BULK)
        else:
            chunk = torch.empty(D.crc_scratch_words(total), dtype=torch.int32, device=dev)
            ecrc = torch.empty(dt.n, dtype=torch.int32, device=dev)
            D.pack_crc(dt.tensor, dt.n, dt.total_chunks, chunk, ecrc, lg)
            # independent check: host SSE4.2 CRC-32C of the smallest, a middle and
            # the largest entry (copied back), against the device CRCs
            order = sorted(range(len(st.entries)), key=lambda i: st.entries[i].nbytes)
            for i in {order[0], order[len(order) // 2], order[-1]}:
                e = st.entries[i]
                host = arena.buffer[e.src_offset:e.src_offset + e.nbytes].cpu().numpy()
                assert D.crc32c(host) == int(ecrc[i].item()) & 0xFFFFFFFF, e.store_key
        torch.cuda.synchronize()
        for e in st.entries:
            assert torch.equal(staging[e.stage_offset:e.stage_offset + e.nbytes],
                               arena.buffer[e.src_offset:e.src_offset + e.nbytes]), (ph, e.store_key)
        # restore direction: wipe the ranges, unpack, compare again
        for e in st.entries:
            arena.buffer[e.src_offset:e.src_offset + e.nbytes].zero_()
        D.unpack(dt.tensor, dt.n, dt.total_chunks, lg, D.MODE_BULK)
        torch.cuda.synchronize()
        for e in st.entries:
            assert torch.equal(staging[e.stage_offset:e.stage_offset + e.nbytes],
                               arena.buffer[e.src_offset:e.src_offset + e.nbytes]), (ph, e.store_key)
    del staging, arena
    torch.cuda.empty_cache()


@pytest.mark.parametrize("strategy", ["baseline", "equal_full"])
def test_full_checkpoints_without_pec_save_and_restore_every_unit(dev, tmp_path, strategy):
    """pec=None: the reference's full-checkpoint strategies (plan_baseline /
    plan_equal without K_pec, planner.py:322-334) -- every unit in every
    version, the planner's per-rank workload staged, and a wiped state
    restored bit-exactly from the newest version."""
    import torch
    from paper_2408_04307_b200.arena import StateArena
    from paper_2408_04307_b200.restore import restore
    from paper_2408_04307_b200.snapshot import PecCheckpointer
    from paper_2408_04307_b200.store import DiskStore
    layout = make_layout(n_experts=4, dp=4, ep=2, gpus_per_node=2, epp=300_001, other=1000)
    ranks = list(range(layout.n_ranks))
    arena = StateArena(layout, ranks, dev)
    store = DiskStore(tmp_path)
    ck = PecCheckpointer(layout, arena, store, None, strategy, i_ckpt=2, ranks=ranks)
    plan = ck.plan()
    assert plan.period == 1
    for it in range(1, 7):
        _mutate(arena, it)
        buf = ck.step(it)
        if buf is not None:
            ck.wait_pack()
    ck.finish()
    torch.cuda.synchronize()
    good = arena.buffer.cpu().numpy().copy()
    vs = store.complete_versions()
    assert len(vs) == 3
    units = {e.unit_key for e in store.meta(vs[-1]).entries.values()}
    assert units == {u.key for u in layout.units if u.size_bytes > 0}
    assert sum(ck.engine.stats["snap_bytes"][-1:]) == sum(plan.workload_bytes[0].values())
    rp = ck.engine.resolve_recovery({1})     # node 1 lost: its units come from storage
    arena.buffer.zero_()
    restore(ck.engine, rp)
    now = arena.buffer.cpu().numpy()
    bad = []
    for key, s in arena.slots.items():
        if not np.array_equal(now[s.offset:s.offset + s.size], good[s.offset:s.offset + s.size]):
            d = rp.decisions[key]
            diff = np.nonzero(now[s.offset:s.offset + s.size] != good[s.offset:s.offset + s.size])[0]
            bad.append((key, d.source, d.node, d.version, int(diff[0]), len(diff), s.size))
    assert not bad, bad
    ck.close()


def test_memory_restore_from_a_peer_engines_node_shared_buffer(dev, tmp_path):
    """Two engines in one process stand in for two rank processes of one
    node (shared_host_prefix: /dev/shm buffers registered with CUDA).  After
    a checkpoint on both, rank 0's wiped state is restored from memory, with
    the ranges that rank 1 snapshotted read out of rank 1's shared buffer
    (`peer_buffer`), bit-identically."""
    import os
    import uuid
    import torch
    from paper_2408_04307_b200 import PecConfig
    from paper_2408_04307_b200.arena import StateArena
    from paper_2408_04307_b200.restore import restore
    from paper_2408_04307_b200.snapshot import PecCheckpointer
    from paper_2408_04307_b200.store import MemoryStore
    layout = make_layout(n_experts=4, dp=2, ep=2, gpus_per_node=2, epp=20_001, other=100)
    prefix = f"pec_gpu_{uuid.uuid4().hex[:8]}"
    arenas = [StateArena(layout, [r], dev) for r in (0, 1)]
    cks = [PecCheckpointer(layout, arenas[r], MemoryStore(), PecConfig(k_pec=2), "equal_pec",
                           i_ckpt=1,
                           ranks=[r], shared_host_prefix=prefix, async_persist=False)
           for r in (0, 1)]
    try:
        _mutate(arenas[0], 1)
        _mutate(arenas[1], 1)
        for ck in cks:
            ck.step(1)
        for ck in cks:
            ck.finish()
        torch.cuda.synchronize()
        good = arenas[0].buffer.cpu().numpy().copy()
        plan = cks[0].engine.resolve_recovery(set())
        mem = [k for k, d in plan.decisions.items() if d.source == "memory" and arenas[0].has(k)]
        assert mem
        # ranges of units resident on rank 0 that only rank 1 snapshotted
        peer_keys = {a.key for a in cks[1].engine.buffers.buffers[0].content.get(1, ())}
        assert peer_keys & set(mem)
        arenas[0].buffer.zero_()
        restore(cks[0].engine, plan, keys=mem)
        now = arenas[0].buffer.cpu().numpy()
        for k in mem:
            s = arenas[0].slot(k)
            assert np.array_equal(now[s.offset:s.offset + s.size],
                                  good[s.offset:s.offset + s.size]), k
    finally:
        for ck in cks:
            ck.close()
    assert not [f for f in os.listdir("/dev/shm") if f.startswith(prefix)]


@pytest.mark.parametrize("pack_mode", [0, 3])
def test_device_plans_for_several_local_ranks(dev, tmp_path, pack_mode):
    """Load-aware device plans with four ranks in one engine (fixed per-rank
    staging regions, one expand + pack per rank, per-region drains), in the
    plain and the CRC-computing engine: persisted versions read back
    CRC-verified and equal to the state at snapshot time."""
    import torch
    from paper_2408_04307_b200 import PecConfig
    from paper_2408_04307_b200.arena import StateArena
    from paper_2408_04307_b200.counting import DeviceTokenCounters
    from paper_2408_04307_b200.snapshot import PecCheckpointer
    from paper_2408_04307_b200.store import DiskStore
    layout = make_layout(n_experts=8, n_layers=2, dp=4, ep=2, gpus_per_node=2, epp=30_001,
                         other=77)
    ranks = list(range(4))
    arena = StateArena(layout, ranks, dev)
    L, E = 2, 8
    counters = DeviceTokenCounters(L, E, dev)
    pec = PecConfig(k_pec=3, selection="load_aware", k_snapshot=3, k_persist=2)
    ck = PecCheckpointer(layout, arena, DiskStore(tmp_path), pec, "equal_pec", i_ckpt=1,
                         ranks=ranks, counters=counters, pack_mode=pack_mode)
    assert ck.device_plans and len(ck.engine.templates) == 4
    ck.prepare()
    shadow = {}
    gen = torch.Generator(device=dev).manual_seed(11)
    for it in range(1, 6):
        _mutate(arena, it)
        ids = torch.randint(0, E, (L, 300), dtype=torch.int64, device=dev, generator=gen)
        buf = ck.step(it, ids)
        torch.cuda.synchronize()
        shadow[buf.version] = arena.buffer.cpu().numpy().copy()
        ck.wait_pack()
    ck.finish()
    vs = ck.engine.store.complete_versions()
    assert vs == sorted(shadow)
    for v in vs:
        data = ck.engine.store.load_checkpoint(v)      # CRC-verified read
        meta = ck.engine.store.meta(v)
        assert {e.rank for e in meta.entries.values()} == set(ranks)
        for sk, b in data.items():
            e = meta.entries[sk]
            off = arena.slot(e.unit_key).offset + e.start
            assert b == shadow[v][off:off + e.stop - e.start].tobytes(), (v, sk)
    ck.close()


@pytest.mark.parametrize("k", [1, 2, 4, 8, 16])
def test_gpt350m_k_sweep_pack_bit_exact_on_device(dev, k):
    """K_pec sweep on GPT-MoE 350M-16E (dp=8 x ep=8, ranks 0..7 emulated):
    every staged entry equals its source range (device-side comparison at
    full size) and the staged payload equals the reference planner's
    per-rank workload."""
    import torch
    from paper_2408_04307_b200 import configs, plan_adaptive
    from paper_2408_04307_b200.arena import StateArena
    from paper_2408_04307_b200 import device as D
    from paper_2408_04307_b200.staging import DeviceTable, StagingLayout
    w = configs.gpt350m_16e(k_pec=k)
    layout = w.layout()
    arena = StateArena(layout, range(8), dev, w.expert_tensors)
    plan = plan_adaptive(layout, w.pec)
    for phase_idx in sorted({0, plan.period - 1}):
        phase = plan.assignments[phase_idx]
        for r in range(8):
            st = StagingLayout.build(phase[r], arena, r)
            staging = torch.empty(st.nbytes, dtype=torch.uint8, device=dev)
            table, total = st.descriptors(arena.base_address, staging.data_ptr())
            dt = DeviceTable(table, total, dev)
            D.pack(dt.tensor, dt.n, dt.total_chunks, mode=D.MODE_BULK if r % 2 else D.MODE_VEC)
            for e in st.entries:
                assert torch.equal(staging[e.stage_offset:e.stage_offset + e.nbytes],
                                   arena.buffer[e.src_offset:e.src_offset + e.nbytes]), e
            assert st.payload_bytes == plan.workload_bytes[phase_idx][r]
    del arena
    torch.cuda.empty_cache()


def test_fault_mid_snapshot_and_mid_persist_leaves_consistent_state(dev, tmp_path):
    """A fault while a snapshot drains discards it (its buffer is only freed
    after the copy engine finished), a fault while persisting publishes no
    version; later checkpoints and recovery are unaffected."""
    import torch
    from paper_2408_04307_b200 import configs
    from paper_2408_04307_b200.arena import StateArena
    from paper_2408_04307_b200.engine import FREE, SNAPSHOTTED
    from paper_2408_04307_b200.restore import restore
    from paper_2408_04307_b200.snapshot import PecCheckpointer
    from paper_2408_04307_b200.store import DiskStore
    w = configs.toy()
    layout = w.layout()
    arena = StateArena(layout, [0], dev, w.expert_tensors)
    store = DiskStore(tmp_path)
    ck = PecCheckpointer(layout, arena, store, w.pec, w.strategy, i_ckpt=1)
    b1 = ck.step(1)                    # snapshotting
    ck.engine.on_fault(set())          # fault before the drain is observed
    assert b1.status == FREE
    ck.hold_persist(True)
    b2 = ck.step(2)
    ck.wait_snapshot(b2)               # SNAPSHOTTED -> PERSISTING, held (not started)
    ck.hold_persist(False)             # persist starts in the background ...
    ck.engine.on_fault(set())          # ... and is aborted before publishing (or won)
    assert store.complete_versions() in ([], [b2.version])
    assert b2.status == (SNAPSHOTTED if not store.complete_versions() else "recovery")
    ck.on_fault(set())                 # resumes the interrupted persist, if any
    torch.cuda.synchronize()
    good = arena.buffer.cpu().numpy().copy()
    b3 = ck.step(3)
    ck.finish()
    assert b3.version in store.complete_versions()
    plan = ck.engine.resolve_recovery(set())
    arena.buffer.zero_()
    restore(ck.engine, plan)
    assert np.array_equal(arena.buffer.cpu().numpy(), good)
    ck.close()


def test_load_aware_pending_drain_survives_faults_and_poll_order(dev, tmp_path):
    """Device-planned (load-aware) snapshots return before the host knows
    their size: a fault while the drain is still pending discards the
    snapshot cleanly; poll() later enqueues pending drains without blocking;
    the persisted bytes and a restore stay exact."""
    import torch
    from paper_2408_04307_b200 import PecConfig, configs
    from paper_2408_04307_b200.arena import StateArena
    from paper_2408_04307_b200.counting import DeviceTokenCounters
    from paper_2408_04307_b200.engine import FREE
    from paper_2408_04307_b200.restore import restore
    from paper_2408_04307_b200.snapshot import PecCheckpointer
    from paper_2408_04307_b200.store import DiskStore
    w = configs.toy()
    layout = w.layout()
    L, E = layout.model.num_moe_layers, layout.model.experts_per_layer
    arena = StateArena(layout, [0], dev, w.expert_tensors)
    store = DiskStore(tmp_path)
    counters = DeviceTokenCounters(L, E, dev)
    pec = PecConfig(k_pec=2, selection="load_aware", k_snapshot=2, k_persist=1)
    ck = PecCheckpointer(layout, arena, store, pec, "equal_pec", i_ckpt=1, counters=counters)
    ck.engine.reserve(ck.max_snapshot_bytes())
    gen = torch.Generator(device=dev).manual_seed(5)

    def ids():
        return torch.randint(0, E, (L, 256), dtype=torch.int32, device=dev, generator=gen)

    b1 = ck.step(1, ids())
    assert b1.content is None                 # plan still on the GPU
    ck.engine.on_fault(set())                 # drain never enqueued: discarded
    assert b1.status == FREE and ck.engine._pending_bid is None
    expected = {}
    for it in range(2, 7):
        _mutate(arena, it)
        buf = ck.step(it, ids())
        torch.cuda.synchronize()
        ck.poll()                             # the size copy has landed: drain enqueued
        assert buf.content is not None
        expected[buf.version] = _expected_entries(arena.buffer.cpu().numpy(), arena,
                                                  buf.content, [0])
        ck.wait_pack()
    ck.finish()
    assert store.complete_versions() == sorted(expected)
    for v in store.complete_versions():
        got = store.load_checkpoint(v)
        for sk, data in got.items():
            assert data == expected[v][sk], (v, sk)
    torch.cuda.synchronize()
    good = arena.buffer.cpu().numpy().copy()
    plan = ck.engine.resolve_recovery(set())
    arena.buffer.zero_()
    restore(ck.engine, plan)
    got_state = arena.buffer.cpu().numpy()
    for key, d in plan.decisions.items():
        if d.source != "initial" and d.restored_iteration == 6:
            sl = arena.slots[key]
            assert np.array_equal(got_state[sl.offset:sl.offset + sl.size],
                                  good[sl.offset:sl.offset + sl.size]), key
    ck.close()


@pytest.mark.parametrize("selection", ["sequential", "load_aware"])
def test_device_crc_mode_persists_verifiable_versions(dev, tmp_path, selection):
    """MODE_CRC: the pack computes every entry's CRC-32C; the persist writes
    them into the manifest without touching the payload on the host, and
    load_checkpoint's host-side CRC verification accepts every entry."""
    import torch
    from paper_2408_04307_b200 import PecConfig, configs
    from paper_2408_04307_b200 import device as D
    from paper_2408_04307_b200.arena import StateArena
    from paper_2408_04307_b200.counting import DeviceTokenCounters
    from paper_2408_04307_b200.snapshot import PecCheckpointer
    from paper_2408_04307_b200.store import DiskStore, crc32c
    w = configs.toy()
    layout = w.layout()
    L, E = layout.model.num_moe_layers, layout.model.experts_per_layer
    arena = StateArena(layout, [0], dev, w.expert_tensors)
    store = DiskStore(tmp_path)
    counters = None
    pec = w.pec
    if selection == "load_aware":
        counters = DeviceTokenCounters(L, E, dev)
        pec = PecConfig(k_pec=2, selection="load_aware", k_snapshot=2, k_persist=1)
    ck = PecCheckpointer(layout, arena, store, pec, w.strategy, i_ckpt=2, counters=counters,
                         pack_mode=D.MODE_CRC)
    expected = {}
    for it in range(1, 9):
        _mutate(arena, it)
        ids = torch.randint(0, E, (L, 512), dtype=torch.int32, device=dev)
        buf = ck.step(it, ids if counters is not None else None)
        if buf is not None:
            ck.resolve(buf)  # device-planned: content is filled when the drain is enqueued
            torch.cuda.synchronize()
            expected[buf.version] = _expected_entries(arena.buffer.cpu().numpy(), arena,
                                                      buf.content, [0])
            ck.wait_pack()
    ck.finish()
    assert store.complete_versions() == sorted(expected)
    for v in store.complete_versions():
        data = store.load_checkpoint(v)   # verifies every manifest CRC on the host
        for k, b in data.items():
            assert b == expected[v][k]
            assert store.manifest(v).entries[k][2] == crc32c(b)
    ck.close()


def test_empty_shards_and_ragged_ranges_round_trip(dev, tmp_path):
    """Edge shapes the reference admits: an other-states blob smaller than
    dp (last shard is empty: ceil split 3 over 4 -> 1,1,1,0), an expert weight
    of odd size split across 2 EP groups, and a 1-parameter module."""
    import torch
    from paper_2408_04307_b200 import PecConfig
    from paper_2408_04307_b200.arena import StateArena
    from paper_2408_04307_b200.restore import restore
    from paper_2408_04307_b200.snapshot import PecCheckpointer
    from paper_2408_04307_b200.store import DiskStore
    layout = make_layout(n_experts=2, dp=4, ep=2, gpus_per_node=2, n_layers=1, epp=7,
                         b_w=1, b_o=4, p_ne=1001, other=3,
                         modules=(("a", 1000), ("b", 1)))
    assert layout.by_key["other.r3"].size_bytes == 0
    arena = StateArena(layout, range(4), dev)
    store = DiskStore(tmp_path)
    ck = PecCheckpointer(layout, arena, store, PecConfig(k_pec=1), "equal_pec", i_ckpt=1,
                         async_persist=False)
    snaps = {}
    for it in (1, 2):
        _mutate(arena, it)
        buf = ck.step(it)
        torch.cuda.synchronize()
        snaps[buf.version] = arena.buffer.cpu().numpy().copy()
        ck.wait_pack()
    ck.finish()
    for v in store.complete_versions():
        data = store.load_checkpoint(v)
        assert data["other.r3"] == b""
        parts = sorted(k for k in data if k.startswith("ew."))
        assert len(parts) == 2 and [len(data[k]) for k in parts] == [3, 4]  # floor split of 7
    plan = ck.engine.resolve_recovery({0})
    ck.engine.on_fault({0})
    arena.buffer.zero_()
    restore(ck.engine, plan)
    now = arena.buffer.cpu().numpy()
    for key, d in plan.decisions.items():
        if arena.has(key) and d.source != "initial":
            s = arena.slot(key)
            assert np.array_equal(now[s.offset:s.offset + s.size],
                                  snaps[d.version][s.offset:s.offset + s.size]), key
    ck.close()


@pytest.mark.parametrize("verify", ["device", "host"])
def test_restore_detects_a_flipped_byte(dev, tmp_path, verify):
    """Storage restores verify every entry's CRC-32C against the manifest
    (DiskStore.load_checkpoint semantics, store.py:267-282), on the GPU
    (pec_pack_crc scatter) or on the host; a corrupted file raises with its
    key, a clean one restores bit-exactly."""
    import torch
    from paper_2408_04307_b200 import configs
    from paper_2408_04307_b200.arena import StateArena
    from paper_2408_04307_b200.restore import restore
    from paper_2408_04307_b200.snapshot import PecCheckpointer
    from paper_2408_04307_b200.store import ChecksumMismatchError, DiskStore
    w = configs.toy()
    layout = w.layout()
    arena = StateArena(layout, [0], dev, w.expert_tensors)
    store = DiskStore(tmp_path)
    ck = PecCheckpointer(layout, arena, store, w.pec, w.strategy, i_ckpt=1, async_persist=False)
    ck.step(1)
    ck.finish()
    torch.cuda.synchronize()
    good = arena.buffer.cpu().numpy().copy()
    plan = ck.engine.resolve_recovery({0})      # the only node failed: storage / initial
    ck.engine.on_fault({0})
    arena.buffer.zero_()
    rep = restore(ck.engine, plan, verify=verify, slot_bytes=8 << 20)  # several batches
    assert rep.storage_bytes > 0 and rep.batches > 1
    now = arena.buffer.cpu().numpy()
    for key, d in plan.decisions.items():
        if d.source == "storage" and arena.has(key):
            s = arena.slot(key)
            assert np.array_equal(now[s.offset:s.offset + s.size], good[s.offset:s.offset + s.size])
    victim = tmp_path / "v000001" / "rank0000" / "neo.r0.bin"
    orig = victim.read_bytes()
    data = bytearray(orig)
    data[len(data) // 2] ^= 0x40
    victim.write_bytes(bytes(data))
    arena.buffer.fill_(0xA5)                    # sentinel: what "untouched" looks like
    with pytest.raises(ChecksumMismatchError) as exc:
        restore(ck.engine, plan, verify=verify, slot_bytes=8 << 20)
    assert exc.value.key == "neo.r0"
    # verify-before-commit (store.py:267-282): the corrupted entry (split over
    # several slots here) never reached the arena; units reported as committed
    # hold verified bytes, every other unit is untouched
    assert arena.unit_bytes("neo.r0").numel() > (8 << 20)   # the split-entry path
    now = arena.buffer.cpu().numpy()
    committed = set(exc.value.committed_units)
    assert "neo.r0" not in committed
    for key in plan.decisions:
        if not arena.has(key):
            continue
        sl = arena.slot(key)
        got = now[sl.offset:sl.offset + sl.size]
        if key in committed:
            assert np.array_equal(got, good[sl.offset:sl.offset + sl.size]), key
        elif plan.decisions[key].source == "storage":
            assert (got == 0xA5).all(), key
    # the failed restore left nothing in flight on the reused slots: a retry
    # once the file is repaired restores every storage unit bit-exactly
    victim.write_bytes(orig)
    restore(ck.engine, plan, verify=verify, slot_bytes=8 << 20)
    now = arena.buffer.cpu().numpy()
    for key, d in plan.decisions.items():
        if d.source == "storage" and arena.has(key):
            sl = arena.slot(key)
            assert np.array_equal(now[sl.offset:sl.offset + sl.size],
                                  good[sl.offset:sl.offset + sl.size]), key
    ck.close()
