"""Snapshot consistency under real overlap (no host synchronisation).

The reference's rule: a snapshot photographs the state between two weight
updates — it must start after the update that precedes it and complete
before the next one (simulator.py:425-438, stall law :551-556).  The B200
path enforces it with two stream dependencies only: the pack stream waits
for the compute stream at the checkpoint (`ps.wait_stream(compute)`), and
the next update waits for the pack (`wait_pack`).

Here a training loop runs with NO host sync between a checkpoint and the
next update: an F&B proxy (bf16 GEMMs, several ms) overlaps every pack and
drain, the update (an in-place pass over the whole state arena) is issued
right after it, and the persist thread writes versions concurrently.  The
expected image of each checkpoint is a stream-ordered fingerprint: the
CRC-32C of every planned entry's source range, computed on the compute
stream at the checkpoint point (`pec_crc_device`, no copy).  Every persisted
file and the host snapshot buffer must equal it — for host-planned
(pipelined drain segments) and device-planned (load-aware) snapshots, with
the plain and the CRC-computing pack.

Negative controls prove the check has teeth: with the pack stream held back
(a spin kernel), dropping `wait_pack` lets the next update land before the
pack reads the state; with the compute stream held back, dropping the pack
stream's wait makes the pack read the state before the update that precedes
the checkpoint.  Both must be detected.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SPIN = 20_000_000   # ~10 ms spin kernel (torch.cuda._sleep cycles)


def _crc_table(entries, arena, dev):
    """DeviceTable of (arena src range) rows for pec_crc_device."""
    from paper_2408_04307_b200 import device as D
    from paper_2408_04307_b200.staging import DeviceTable
    table = np.zeros(len(entries), dtype=D.DESC_DTYPE)
    for i, (_, src, n) in enumerate(entries):
        table[i] = (arena.base_address + src, 0, n, 0)
    total = D.plan_chunks(table, 15)
    return DeviceTable(table, total, dev, 15)


def _run(dev, tmp_path, selection, pack_mode, lag=None, drop=None, iters=12, i_ckpt=2):
    """Training loop with checkpoints; returns (mismatches, checked entries).
    ``lag``: "pack" / "compute" holds that stream back with a spin kernel at
    every checkpoint; ``drop``: "wait_pack" / "stream_wait" removes that
    dependency (negative controls)."""
    import torch
    from paper_2408_04307_b200 import PecConfig, configs
    from paper_2408_04307_b200 import device as D
    from paper_2408_04307_b200.arena import StateArena
    from paper_2408_04307_b200.counting import DeviceTokenCounters
    from paper_2408_04307_b200.snapshot import PecCheckpointer
    from paper_2408_04307_b200.store import DiskStore

    w = configs.toy()
    layout = w.layout()
    L, E = layout.model.num_moe_layers, layout.model.experts_per_layer
    arena = StateArena(layout, [0], dev, w.expert_tensors)
    store = DiskStore(tmp_path)
    counters = None
    if selection == "load_aware":
        pec = PecConfig(k_pec=2, selection="load_aware", k_snapshot=2, k_persist=1)
        counters = DeviceTokenCounters(L, E, dev)
        strategy = "equal_pec"
    else:
        pec, strategy = w.pec, w.strategy
    ck = PecCheckpointer(layout, arena, store, pec, strategy, i_ckpt=i_ckpt,
                         counters=counters, pack_mode=pack_mode)
    eng = ck.engine
    eng.drain_first = 1 << 20            # host plans: ~6 pipelined drain segments
    ck.prepare()
    if drop == "stream_wait":
        eng._consistency_wait = False

    # fingerprint tables, built before the loop (building one copies H2D)
    if ck.device_plans:
        t = eng.templates[0]
        ents = [(a.store_key, int(t.table[i]["src_offset"]), int(t.table[i]["nbytes"]))
                for i, a in enumerate(t.ranges)]
        fp_tables = {None: (ents, _crc_table(ents, arena, dev))}
    else:
        plan = ck.plan()
        fp_tables = {}
        for p in range(plan.period):
            st = eng.layouts_for(plan.assignments[p], ("phase", p))[0]
            ents = [(e.store_key, e.src_offset, e.nbytes) for e in st.entries]
            fp_tables[p] = (ents, _crc_table(ents, arena, dev))
    n_ckpt = iters // i_ckpt
    outs = [torch.empty(max(len(v[0]) for v in fp_tables.values()), dtype=torch.int32,
                        device=dev) for _ in range(n_ckpt)]
    scratch = torch.empty(max(D.crc_scratch_words(v[1].total_chunks)
                              for v in fp_tables.values()), dtype=torch.int32, device=dev)
    ids = [torch.randint(0, E, (L, 2048), dtype=torch.int32, device=dev,
                         generator=torch.Generator(device=dev).manual_seed(100 + it))
           for it in range(iters + 1)]
    a = torch.randn(4096, 4096, device=dev, dtype=torch.bfloat16)
    b = torch.randn(4096, 4096, device=dev, dtype=torch.bfloat16)
    c = torch.empty_like(a)
    words = arena.buffer.view(torch.int32)
    compute = torch.cuda.current_stream(dev)
    torch.cuda.synchronize()

    fps = []     # (version, fingerprint keys, device crcs)
    for it in range(1, iters + 1):
        for _ in range(12):                       # F&B proxy, ~3 ms of GEMMs
            torch.matmul(a, b, out=c)
        if counters is not None:
            counters.add_iteration(ids[it])
        ck.poll()
        if lag == "compute" and it % i_ckpt == 0:
            torch.cuda._sleep(SPIN)               # the compute stream lags the host
        if drop != "wait_pack":
            ck.wait_pack(stream=compute)          # the update may not race the pack
        words.add_(it)                            # optimizer step: every byte changes
        if it % i_ckpt == 0:
            c_idx = it // i_ckpt - 1
            key = None if ck.device_plans else ck.plan().phase_of(c_idx)
            ents, tab = fp_tables[key]
            out = outs[len(fps)]
            D.crc_device(tab.tensor, tab.n, tab.total_chunks, scratch, out, 15, stream=compute)
            if lag == "pack":
                with torch.cuda.stream(eng.pack_stream):
                    torch.cuda._sleep(SPIN)       # the pack starts late
            buf = ck.checkpoint(it)
            fps.append((buf.version, [k for k, _, _ in ents], out))
    ck.finish()
    torch.cuda.synchronize()

    mismatches, checked = [], 0
    for version, keys, out in fps:
        want = dict(zip(keys, (int(x) for x in out[:len(keys)].cpu().numpy().view(np.uint32))))
        got = store.load_checkpoint(version)      # also verifies the manifest CRCs
        assert got, version
        for k, data in got.items():
            checked += 1
            if D.crc32c(data) != want[k]:
                mismatches.append((version, k))
    # the newest snapshot's host buffer is still resident: check it too
    last = fps[-1][0]
    buf = next(b for b in eng.buffers.buffers if b.version == last)
    ck.resolve(buf)
    want = dict(zip(fps[-1][1], (int(x) for x in fps[-1][2][:len(fps[-1][1])].cpu().numpy()
                                 .view(np.uint32))))
    for e in eng.snapshot_layout(buf, 0).entries:
        checked += 1
        if D.crc32c(eng.entry_view(buf, 0, e.store_key)) != want[e.store_key]:
            mismatches.append(("host", e.store_key))
    ck.close()
    return mismatches, checked


@pytest.mark.parametrize("selection", ["sequential", "load_aware"])
@pytest.mark.parametrize("pack_mode", [2, 3], ids=["bulk", "crc"])
def test_snapshots_equal_the_stream_ordered_state_under_overlap(dev, tmp_path, selection,
                                                                pack_mode):
    mismatches, checked = _run(dev, tmp_path, selection, pack_mode)
    assert checked > 50
    assert mismatches == []


@pytest.mark.parametrize("lag", ["pack", "compute"])
@pytest.mark.parametrize("selection", ["sequential", "load_aware"])
def test_snapshots_stay_exact_when_a_stream_lags(dev, tmp_path, selection, lag):
    """The negative controls' spin kernels with both dependencies in place:
    still exact (the late pack holds the next update back; the early pack
    waits for the late update)."""
    mismatches, checked = _run(dev, tmp_path, selection, 3, lag=lag)
    assert checked > 50
    assert mismatches == []


@pytest.mark.parametrize("lag,drop", [("pack", "wait_pack"), ("compute", "stream_wait")])
@pytest.mark.parametrize("selection", ["sequential", "load_aware"])
def test_negative_controls_detect_a_torn_snapshot(dev, tmp_path, selection, lag, drop):
    """Either the bytes differ from the fingerprint, or — device-planned
    snapshots whose expansion raced the selection it depends on — the
    engine's check of every expanded row against the host plan refuses the
    snapshot (snapshot.finalize_pending)."""
    try:
        mismatches, checked = _run(dev, tmp_path, selection, 3, lag=lag, drop=drop)
    except RuntimeError as exc:
        assert selection == "load_aware" and "disagrees with the host plan" in str(exc), exc
        return
    assert checked > 50
    assert mismatches, f"dropping {drop} was not detected"
