"""Full-shape GPU parity of BASELINE configs 2 and 3 on the load-aware,
device-planned path (counting -> two-tier selection -> `pec_expand_plan` ->
pack), against the oracle on the same router ids.

Config 2: GPT-MoE 125M-8E (6 MoE layers x 8 experts, top-2), bf16 weights +
fp32 master/Adam, dp=1, K_pec=1 load-aware: the whole chain through
`PecCheckpointer` with the persist tier; selections equal the oracle's
two-tier selection (reference selector.py:91-100, simulator.py:339-354) on
bincount+cap of the reference's Zipf stream, and every persisted file equals
the state's bytes at the checkpoint (oracle pack content).

Config 3: GPT-MoE 350M-16E, EP=8 x ZeRO-2 DP=8, K_pec=2 load-aware, all
eight ranks' state on one GPU (26.1 GB).  Each rank counts its own router
ids into its own counters (its own per-iteration capacity cap); at a
checkpoint the counters are summed exactly as the NCCL all-reduce would
(`distributed.global_two_tier_select`), selected once, and the selected
entries zeroed in every rank's local counters.  Selections equal the oracle
on the summed counts; every rank's device-expanded plan equals the host
planner (reference planner.py:263-295, topology.py:286-356), its staged
bytes equal the oracle pack, and the ranks' payloads add up to the
reference's pec_checkpoint_size(K) (planner.py:158-167).
"""

import numpy as np
import pytest

from oracle import pec_oracle as O

pytestmark = pytest.mark.gpu


def _perturb(arena, it):
    """Optimizer-step stand-in: every 4-byte word of every unit changes."""
    import torch
    arena.buffer.view(torch.int32).add_(it)


def test_config2_gpt125m_load_aware_chain_full_shape(dev, tmp_path):
    import torch
    from paper_2408_04307_b200 import configs
    from paper_2408_04307_b200.arena import StateArena
    from paper_2408_04307_b200.counting import DeviceTokenCounters
    from paper_2408_04307_b200.snapshot import PecCheckpointer
    from paper_2408_04307_b200.store import DiskStore
    w = configs.gpt125m_8e()
    layout = w.layout()
    L, E = layout.model.num_moe_layers, layout.model.experts_per_layer
    total = w.tokens_per_rank * layout.model.top_k
    arena = StateArena(layout, [0], dev, w.expert_tensors)
    assert arena.resident_bytes() > 4.5e9
    cap = DeviceTokenCounters.capacity_for(w.capacity_factor, [total] * L, E)
    counters = DeviceTokenCounters(L, E, dev, cap)
    ck = PecCheckpointer(layout, arena, DiskStore(tmp_path), w.pec, w.strategy, i_ckpt=2,
                         counters=counters)
    assert ck.device_plans
    snap_c = np.zeros((L, E), np.int64)
    pers_c = np.zeros((L, E), np.int64)
    expected = {}
    for it in range(1, 7):
        _perturb(arena, it)
        ids = np.stack([O.zipf_router_ids(7, it, m, E, total, 1.1) for m in range(L)])
        counts = O.route_counts(ids, E, O.capacity(w.capacity_factor, total, E))
        snap_c += counts
        pers_c += counts
        buf = ck.step(it, torch.from_numpy(ids).to(dev))
        if buf is None:
            continue
        ss, ps, snap_c, pers_c = O.two_tier_load_aware(snap_c, pers_c, 1, 1)
        torch.cuda.synchronize()
        host = arena.buffer.cpu().numpy()
        ck.resolve(buf)
        due = {m: set() for m in range(L)}
        want = {}
        for a in buf.content[0]:
            u = layout.by_key[a.key]
            if u.layer is not None:
                due[u.layer].add(u.expert)
            src = arena.slot(a.key).offset + a.start
            want[a.store_key] = host[src:src + a.stop - a.start].copy()
        assert [sorted(due[m]) for m in range(L)] == ss, it
        assert [sorted(ck.persist_sel[buf.version][m]) for m in range(L)] == ps, it
        expected[buf.version] = want
        ck.wait_pack()
    ck.finish()
    assert sorted(expected) == ck.engine.store.complete_versions()
    for v, want in expected.items():
        got = ck.engine.store.load_checkpoint(v)        # CRC-verified (device CRCs)
        assert got and set(got) <= set(want)
        for k, data in got.items():
            assert np.array_equal(np.frombuffer(data, np.uint8), want[k]), (v, k)
    ck.close()


def test_config3_gpt350m_dp8_load_aware_summed_counts_full_shape(dev):
    import torch
    from paper_2408_04307_b200 import build_phase_assignment, configs, pec_checkpoint_size
    from paper_2408_04307_b200 import device as D
    from paper_2408_04307_b200.arena import StateArena
    from paper_2408_04307_b200.counting import DeviceTokenCounters
    from paper_2408_04307_b200.staging import PlanTemplate, StagingLayout
    w = configs.gpt350m_16e_load_aware(k_pec=2)
    layout = w.layout()
    L, E = layout.model.num_moe_layers, layout.model.experts_per_layer
    K = w.pec.k_snapshot
    R = layout.n_ranks
    assert R == 8 and layout.parallel.ep_degree == 8
    total = w.tokens_per_rank * layout.model.top_k
    arena = StateArena(layout, range(R), dev, w.expert_tensors)
    cap = DeviceTokenCounters.capacity_for(w.capacity_factor, [total] * L, E)
    counters = [DeviceTokenCounters(L, E, dev, cap) for _ in range(R)]
    tmpls = [PlanTemplate(layout, arena, r, w.strategy, dev) for r in range(R)]
    staging = torch.empty(max(t.max_bytes for t in tmpls) + 512, dtype=torch.uint8, device=dev)
    table = torch.empty(max(t.n for t in tmpls) * 4, dtype=torch.int64, device=dev)
    totals = torch.zeros(2, dtype=torch.int64, device=dev)

    def select_fn(counts2d, k, pool):
        out = torch.empty((L, k), dtype=torch.int32, device=dev)
        D.select_load_aware(counts2d, k, out, pool=pool)
        return out

    snap_c = np.zeros((L, E), np.int64)
    pers_c = np.zeros((L, E), np.int64)
    for it in range(1, 7):
        _perturb(arena, it)
        for r in range(R):
            ids = np.stack([O.zipf_router_ids(7 + r, it, m, E, total, 1.1) for m in range(L)])
            counts = O.route_counts(ids, E, O.capacity(w.capacity_factor, total, E))
            snap_c += counts
            pers_c += counts
            counters[r].add_iteration(torch.from_numpy(ids).to(dev))
        if it % 2:
            continue
        ss, ps, snap_c, pers_c = O.two_tier_load_aware(snap_c, pers_c, K, K)
        # global = sum of locals (what dist.all_reduce(SUM) computes in
        # global_two_tier_select), one selection, selected entries zeroed in
        # every local tier
        glob = torch.stack([c.counts for c in counters]).sum(0)
        snap = select_fn(glob[0], K, None)
        pers = select_fn(glob[1], K, snap)
        for c in counters:
            c.counts[0].scatter_(1, snap.long().clamp_min(0), 0)
            c.counts[1].scatter_(1, pers.long().clamp_min(0), 0)
        assert snap.cpu().tolist() == ss and pers.cpu().tolist() == ps, it
        # the invariant the multi-GPU protocol relies on: sum(local) == oracle
        glob_after = torch.stack([c.counts for c in counters]).sum(0).cpu().numpy()
        assert np.array_equal(glob_after[0], snap_c) and np.array_equal(glob_after[1], pers_c)
        host = None
        host = arena.buffer.cpu().numpy()
        due = {m: frozenset(ss[m]) for m in range(L)}
        assignment = build_phase_assignment(layout, due, w.strategy)
        payload = 0
        for r in range(R):
            staging.zero_()
            D.expand_plan(tmpls[r].tensor, tmpls[r].n, snap, arena.base_address,
                          staging.data_ptr(), table, totals)
            D.pack_indirect(table, tmpls[r].n, tmpls[r].max_chunks(), totals)
            st = StagingLayout.build(assignment.get(r, ()), arena, r)
            got = staging[:st.nbytes + 1].cpu().numpy()
            assert int(totals[1]) == st.nbytes and int(totals[0]) == st.descriptors(0, 0)[1]
            copies = [(e.src_offset, e.stage_offset, e.nbytes) for e in st.entries]
            assert np.array_equal(got, O.pack(host, copies, st.nbytes + 1)), (it, r)
            payload += st.payload_bytes
        assert payload == pec_checkpoint_size(layout.model, K)
    del arena, staging
    torch.cuda.empty_cache()
