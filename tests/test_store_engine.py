"""Store format, CRC-32C and recovery decisions vs. the reference (CPU)."""

import hashlib
import json

import numpy as np
import pytest

from conftest import GOLDEN, make_layout
from paper_2408_04307_b200 import ClusterSpec, ModelSpec, ParallelSpec, PecConfig, build_layout, plan_equal
from paper_2408_04307_b200.engine import (
    FREE,
    PERSISTING,
    RECOVERY,
    SNAPSHOTTED,
    SNAPSHOTTING,
    CheckpointEngine,
    NoFreeBufferError,
    TripleBufferSet,
    UnrecoverableStateError,
)
from paper_2408_04307_b200.selector import select_window
from paper_2408_04307_b200.store import (
    ChecksumMismatchError,
    CrashPoint,
    DiskStore,
    IncompleteVersionError,
    MemoryStore,
    StoreEntry,
    StoreError,
    TruncatingInjector,
    crc32c,
    entry_payload,
)

STORE = json.loads((GOLDEN / "store.json").read_text())
RECOVERY_G = json.loads((GOLDEN / "recovery.json").read_text())


def _entries():
    return [StoreEntry(*e) for e in STORE["entries"]]


# -- CRC ----------------------------------------------------------------------

def test_crc32c_known_vectors():
    assert crc32c(b"123456789") == 0xE3069283
    assert crc32c(b"") == 0


def test_crc32c_golden_vectors_and_chaining():
    rng = np.random.default_rng(STORE["crc_seed"])
    for v in STORE["crc_vectors"]:
        b = rng.bytes(v["seed_len"])
        assert hashlib.sha256(b).hexdigest() == v["sha"]
        assert crc32c(b) == v["crc"]
        k = len(b) // 3
        assert crc32c(b[k:], crc32c(b[:k])) == v["crc"]


def test_crc32c_many_and_combine_large():
    from paper_2408_04307_b200 import device as D
    rng = np.random.default_rng(3)
    buf = rng.integers(0, 256, size=(200 << 20) + 12345, dtype=np.uint8)
    offs = [0, 7, 1 << 20, (64 << 20) - 3, 5]
    lens = [len(buf), (130 << 20) + 1, 0, 70 << 20, 1]
    got = D.crc32c_many(buf, offs, lens, threads=4)
    for o, n, c in zip(offs, lens, got):
        assert int(c) == crc32c(buf[o:o + n])
    a, b = buf[:1000].tobytes(), buf[1000:300000].tobytes()
    assert D.crc32c_combine(crc32c(a), crc32c(b), len(b)) == crc32c(a + b)


def test_oracle_crc_agrees_with_product_crc():
    from oracle import pec_oracle as O
    rng = np.random.default_rng(11)
    for n in (0, 1, 15, 16, 17, 4095, 100001):
        b = rng.bytes(n)
        assert O.crc32c(b) == crc32c(b)
        if n <= 2000:
            assert O.crc32c_py(b) == crc32c(b)


# -- store format ---------------------------------------------------------------

def test_disk_layout_meta_and_manifest_are_byte_identical(tmp_path):
    st = DiskStore(tmp_path)
    st.write_version(3, iteration=17, checkpoint_index=2, entries=_entries())
    vdir = tmp_path / "v000003"
    assert (vdir / "meta.json").read_text() == STORE["meta_json"]
    assert (vdir / "manifest.tsv").read_text() == STORE["manifest_tsv"]
    files = sorted(str(p.relative_to(vdir)) for p in vdir.rglob("*") if p.is_file())
    assert files == STORE["files"]
    assert (vdir / "COMPLETE").stat().st_size == 0


def test_real_payload_round_trip_and_flip_detection(tmp_path):
    st = DiskStore(tmp_path, io_threads=4)
    rng = np.random.default_rng(5)
    ents = _entries()
    pay = {e.store_key: rng.bytes(e.stop - e.start) for e in ents}
    man = st.write_version(1, iteration=7, checkpoint_index=0, entries=ents, payloads=pay)
    assert man.complete_marker
    assert st.load_checkpoint(1) == pay
    for k, (path, size, c) in st.manifest(1).entries.items():
        assert size == len(pay[k]) and c == crc32c(pay[k])
    # read_into places the bytes into a host buffer
    buf = bytearray(1000)
    st.read_into(1, {"neo.r1": (buf, 100)})
    assert bytes(buf[100:164]) == pay["neo.r1"]
    victim = tmp_path / "v000001" / "rank0000" / "neo.r0.bin"
    data = bytearray(victim.read_bytes())
    data[5] ^= 0xFF
    victim.write_bytes(bytes(data))
    with pytest.raises(ChecksumMismatchError) as exc:
        st.load_checkpoint(1)
    assert exc.value.key == "neo.r0"


def test_split_write_then_publish_equals_single_writer(tmp_path):
    a, b = DiskStore(tmp_path / "a"), DiskStore(tmp_path / "b")
    ents = _entries()
    a.write_version(4, 9, 1, ents)
    rows = []
    for rank in (0, 1):
        rows += b.write_entries(4, 9, [e for e in ents if e.rank == rank])
    b.publish(4, 9, 1, ents, rows)
    for name in ("meta.json", "manifest.tsv"):
        assert (tmp_path / "a/v000004" / name).read_bytes() == \
            (tmp_path / "b/v000004" / name).read_bytes()


def test_incomplete_version_ignored_and_crash_budget(tmp_path):
    st = DiskStore(tmp_path)
    st.write_version(1, 5, 0, _entries())
    total = st.serialized_size(2, 9, 1, _entries())
    with pytest.raises(CrashPoint):
        st.write_version(2, 9, 1, _entries(), injector=TruncatingInjector(total // 2))
    assert st.complete_versions() == [1]
    with pytest.raises(IncompleteVersionError):
        st.load_checkpoint(2)
    st2 = DiskStore(tmp_path / "x")
    total = st2.serialized_size(1, 5, 0, _entries())
    st2.write_version(1, 5, 0, _entries(), injector=TruncatingInjector(total + 1))
    assert st2.newest_complete() == 1
    with pytest.raises(StoreError):
        st2.write_version(1, 6, 1, _entries())


def test_memory_store_parity(tmp_path):
    disk, mem = DiskStore(tmp_path), MemoryStore()
    for s in (disk, mem):
        s.write_version(1, iteration=7, checkpoint_index=0, entries=_entries())
    assert disk.load_checkpoint(1) == mem.load_checkpoint(1)
    assert disk.manifest(1).entries == mem.manifest(1).entries
    assert disk.meta(1).entries == mem.meta(1).entries
    for k, v in mem.load_checkpoint(1).items():
        assert v == entry_payload(k, 1, 7)


# -- state machine ---------------------------------------------------------------

def test_triple_buffer_transitions():
    bufs = TripleBufferSet()
    b1 = bufs.begin_snapshot(1, 10, 0, None, nodes=[0])
    assert b1.status == SNAPSHOTTING
    with pytest.raises(RuntimeError):
        bufs.begin_snapshot(9, 99, 9, None, nodes=[0])
    assert bufs.complete_snapshot(b1) is b1 and b1.status == PERSISTING
    b2 = bufs.begin_snapshot(2, 20, 1, None, nodes=[0])
    assert bufs.complete_snapshot(b2) is None and b2.status == SNAPSHOTTED
    b3 = bufs.begin_snapshot(3, 30, 2, None, nodes=[0])
    bufs.complete_snapshot(b3)
    with pytest.raises(NoFreeBufferError):
        bufs.begin_snapshot(4, 40, 3, None, nodes=[0])
    assert bufs.complete_persist(b1) is b2 and b1.status == RECOVERY
    with pytest.raises(NoFreeBufferError):
        bufs.begin_snapshot(4, 40, 3, None, nodes=[0])
    assert bufs.complete_persist(b2) is b3
    assert b1.status == FREE and b1.content is None
    assert bufs.begin_snapshot(4, 40, 3, None, nodes=[0]) is b1


# -- recovery decisions vs reference -----------------------------------------------

def _layout_from(case):
    m = case["model"]
    model = ModelSpec(**{**m, "non_expert_modules": tuple(map(tuple, m["non_expert_modules"]))})
    gpn = case["gpus_per_node"]
    cluster = ClusterSpec(num_nodes=case["dp"] // gpn, gpus_per_node=gpn, snapshot_bandwidth=1e9,
                          persist_bandwidth=1e8, fb_time=0.01, update_time=0.002,
                          restart_time=1.0)
    return build_layout(model, ParallelSpec(case["dp"], case["ep"]), cluster)


@pytest.mark.parametrize("i", range(len(RECOVERY_G["cases"])))
def test_recovery_decisions_match_reference(i):
    case = RECOVERY_G["cases"][i]
    layout = _layout_from(case)
    n = layout.model.experts_per_layer
    pec = PecConfig(k_pec=case["k_snapshot"], k_snapshot=case["k_snapshot"],
                    k_persist=case["k_persist"])
    plan = plan_equal(layout, pec)
    eng = CheckpointEngine(layout, MemoryStore())
    kp = case["k_persist"]
    for op in case["ops"]:
        c = op["c"]
        buf = eng.begin_snapshot(op["iteration"], c, plan.assignments[plan.phase_of(c)])
        eng.complete_snapshot(buf)
        if op["persisted"]:
            sel = {m: select_window(c, m, n, kp, kp) for m in range(layout.model.num_moe_layers)}
            eng.complete_persist(buf, eng.persist_entries(buf, sel))
    want = case["result"]
    if "error" in want:
        with pytest.raises(Exception) as exc:
            eng.resolve_recovery(set(case["failed"]), max_iteration=case["max_iteration"])
        assert type(exc.value).__name__ == want["error"]
        return
    got = eng.resolve_recovery(set(case["failed"]), max_iteration=case["max_iteration"])
    assert {k: list(v) for k, v in sorted(got.decisions.items())} == want["decisions"]
    assert got.restart_iteration == want["restart_iteration"]
    assert got.version_skew == want["version_skew"]


def test_fig7_two_level_recovery():
    layout = make_layout(n_experts=4, dp=4, ep=4, gpus_per_node=2, n_layers=1, epp=100)
    pec = PecConfig(k_pec=2, k_snapshot=2, k_persist=1)
    plan = plan_equal(layout, pec)
    eng = CheckpointEngine(layout, MemoryStore())
    for c, it in enumerate((10, 20, 30)):
        buf = eng.begin_snapshot(it, c, plan.assignments[plan.phase_of(c)])
        eng.complete_snapshot(buf)
        sel = {0: select_window(c, 0, 4, 1, 1)}
        eng.complete_persist(buf, eng.persist_entries(buf, sel))
    d = eng.resolve_recovery({0}).decisions
    assert d["ew.L0.E0"][:1] == ("storage",) and d["ew.L0.E0"].restored_iteration == 10
    assert d["ew.L0.E2"].source == "memory" and d["ew.L0.E2"].node == 1
    assert d["ew.L0.E3"].source == "memory" and d["ew.L0.E3"].restored_iteration == 30
    d1 = eng.resolve_recovery({1}).decisions
    assert d1["ew.L0.E3"].source == "initial"
    with pytest.raises(UnrecoverableStateError):
        CheckpointEngine(layout, MemoryStore()).resolve_recovery(set())


def test_shared_host_buffer_visible_to_a_peer_mapping():
    import uuid
    from paper_2408_04307_b200.hostmem import SharedHostBuffer, buffer_name
    assert buffer_name("pfx", 3, 1) == "pfx.r0003.b1"   # peers derive each other's names
    name = f"pec_test_{uuid.uuid4().hex}"
    owner = SharedHostBuffer(name, 1 << 16, create=True, register=False)
    owner.array[100:110] = np.arange(10, dtype=np.uint8)
    peer = SharedHostBuffer(name, create=False, register=False)
    assert peer.nbytes == 1 << 16
    assert bytes(peer.array[100:110]) == bytes(range(10))
    peer.close()
    owner.close()
    import os
    assert not os.path.exists(owner.path)


def test_arena_slots_are_recomputable_for_peers():
    from paper_2408_04307_b200.arena import PeerSlots, arena_slots
    layout = make_layout(n_experts=4, dp=4, ep=2, epp=1001, other=13)
    for r in range(4):
        a = arena_slots(layout, [r])
        assert PeerSlots(layout, r).slots == a
        offs = sorted(s.offset for s in a.values())
        assert all(o % 256 == 0 for o in offs)
        ends = sorted((s.offset, s.offset + s.size) for s in a.values())
        assert all(e0[1] <= e1[0] for e0, e1 in zip(ends, ends[1:]))


def test_durable_store_fsyncs_and_still_reads_back(tmp_path):
    """DiskStore(fsync=True, direct_io=True): entry files fsynced by the
    native writer (O_DIRECT where the filesystem allows), metadata and
    directories fsynced before the COMPLETE rename; same bytes and format."""
    from paper_2408_04307_b200.store import DiskStore, StoreEntry, crc32c
    rng = np.random.default_rng(3)
    entries = [StoreEntry("ew.L0.E1", 0, "ew.L0.E1", 0, 5000),
               StoreEntry("neo.r1", 1, "neo.r1", 0, (1 << 20) + 7)]
    pay = {e.store_key: rng.integers(0, 256, e.stop - e.start, dtype=np.uint8) for e in entries}
    durable = DiskStore(tmp_path / "d", fsync=True, direct_io=True)
    plain = DiskStore(tmp_path / "p")
    for st in (durable, plain):
        st.write_version(1, 9, 0, entries, payloads=pay)
    got = durable.load_checkpoint(1)
    assert {k: bytes(v) for k, v in got.items()} == {k: v.tobytes() for k, v in pay.items()}
    for f in ("meta.json", "manifest.tsv"):
        assert (tmp_path / "d" / "v000001" / f).read_bytes() == \
            (tmp_path / "p" / "v000001" / f).read_bytes()
    assert durable.manifest(1).entries["neo.r1"][2] == crc32c(pay["neo.r1"])


@pytest.mark.parametrize("recycle", [False, True])
def test_retire_recycles_files_without_changing_what_readers_see(tmp_path, recycle):
    """DiskStore.retire (bench retention): a retired version disappears for
    readers at once (COMPLETE first); with ``recycle`` its entry files become
    spares that the next version of the same sizes overwrites in place
    (same inodes: no page reclaim), and every version still reads back
    CRC-verified and byte-identical to a fresh store's tree."""
    import os
    st = DiskStore(tmp_path / "s", io_threads=3, recycle=recycle)
    ref = DiskStore(tmp_path / "r", io_threads=3)
    rng = np.random.default_rng(9)
    ents = _entries()
    for v in (1, 2, 3):
        pay = {e.store_key: rng.bytes(e.stop - e.start) for e in ents}
        if v == 3:
            inodes = {p.stat().st_ino for p in (tmp_path / "s").rglob("*.bin")
                      if ".spare" in str(p)}
        st.write_version(v, iteration=10 * v, checkpoint_index=v, entries=ents, payloads=pay)
        ref.write_version(v, iteration=10 * v, checkpoint_index=v, entries=ents, payloads=pay)
        assert st.load_checkpoint(v) == pay
        if v == 2:
            assert st.retire(1) is True
            assert st.complete_versions() == [2]
            assert not (tmp_path / "s" / "v000001").exists()
    got = {p.stat().st_ino for p in (tmp_path / "s" / "v000003").rglob("*.bin")}
    assert bool(got & inodes) == recycle         # v3 overwrote v1's files in place
    for v in (2, 3):
        for name in ("meta.json", "manifest.tsv"):
            assert (tmp_path / "s" / f"v{v:06d}" / name).read_bytes() == \
                (tmp_path / "r" / f"v{v:06d}" / name).read_bytes()
    st.trim_spares([0, 1], keep_bytes=0)
    assert not any(p.is_file() for p in (tmp_path / "s").rglob("*.bin") if ".spare" in str(p))
    assert os.listdir(tmp_path / "s")  # the store itself remains


class _SequentialInjector(TruncatingInjector):
    """Same budget semantics, but (not being a TruncatingInjector itself)
    routes the store through its sequential Python write loop."""


@pytest.mark.parametrize("direct", [False, True])
def test_native_writer_crash_budget_matches_the_sequential_writer(tmp_path, direct):
    """Crash injection on the native parallel writer (pec_write_files_budget):
    at budgets before, inside and after every file boundary, real multi-MiB
    payloads of several ranks leave the byte-identical partial tree, the same
    CrashPoint and the same unspent budget as the sequential writer loop
    (TruncatingInjector semantics, reference store.py:124-146)."""
    rng = np.random.default_rng(11)
    sizes = [0, 3 << 20, 1, (5 << 20) + 7, 4096, 700_001, 2 << 20]
    ents = [StoreEntry(f"ew.L{i}.E{i % 3}", i % 3, f"ew.L{i}.E{i % 3}", 0, n)
            for i, n in enumerate(sizes)]
    pay = {e.store_key: rng.bytes(e.stop - e.start) for e in ents}
    order = [e.stop - e.start for e in sorted(ents)]
    edges = np.cumsum(order)
    total = DiskStore(tmp_path / "probe").serialized_size(1, 5, 0, ents, payloads=pay)
    budgets = sorted({0, 1, total - 1, total, total + 5} |
                     {int(x) + d for x in edges for d in (-1, 0, 1) if x + d >= 0})
    for b in budgets:
        outs, trees = [], []
        for name, inj_cls, threads in (("native", TruncatingInjector, 4),
                                       ("seq", _SequentialInjector, 1)):
            root = tmp_path / f"{name}{b}"
            st = DiskStore(root, io_threads=threads, direct_io=direct)
            inj = inj_cls(b)
            try:
                st.write_version(1, 5, 0, ents, injector=inj, payloads=pay)
                res = "ok"
            except CrashPoint:
                res = "crash"
            outs.append((res, inj.remaining, st.complete_versions()))
            trees.append({str(p.relative_to(root)): p.read_bytes()
                          for p in sorted(root.rglob("*")) if p.is_file()})
        assert outs[0] == outs[1], b
        assert trees[0] == trees[1], b
    ok = DiskStore(tmp_path / "full", io_threads=4, direct_io=direct)
    ok.write_version(1, 5, 0, ents, injector=TruncatingInjector(total + 1), payloads=pay)
    assert ok.load_checkpoint(1) == pay


@pytest.mark.parametrize("payload_kind", ["synthetic", "real"])
def test_crashtest_newest_complete_survives_random_crashes(tmp_path, payload_kind):
    """The reference's `mocsim crashtest` loop (cli.py:233-269) on this store
    and its native writer: version 1 complete, version 2 crashed at a random
    byte budget; the newest complete version is 1 exactly when the write
    crashed, and it loads CRC-verified with the bytes that were written."""
    import random
    import shutil
    rng = random.Random(7)
    prng = np.random.default_rng(7)
    ents = [StoreEntry(f"ew.L0.E{i}" if i < 4 else f"neo.r{i - 4}", i % 2,
                       f"ew.L0.E{i}" if i < 4 else f"neo.r{i - 4}", 0, 64 if i % 3 else 70_001)
            for i in range(6)]

    def pay(v):
        if payload_kind == "synthetic":
            return None
        return {e.store_key: prng.bytes(e.stop - e.start) for e in ents}

    for trial in range(60):
        root = tmp_path / f"t{trial}"
        st = DiskStore(root, io_threads=3)
        p1, p2 = pay(1), pay(2)
        st.write_version(1, 10, 0, ents, payloads=p1)
        total = st.serialized_size(2, 20, 1, ents, payloads=p2)
        budget = rng.randint(0, total + 1)
        try:
            st.write_version(2, 20, 1, ents, injector=TruncatingInjector(budget), payloads=p2)
            crashed = False
        except CrashPoint:
            crashed = True
        newest = st.newest_complete()
        assert newest == (1 if crashed else 2), (trial, budget)
        got = st.load_checkpoint(newest)
        want = (p1 if newest == 1 else p2) or {
            e.store_key: bytes(entry_payload(e.store_key, newest, 10 if newest == 1 else 20))
            for e in ents}
        assert got == {k: bytes(v) for k, v in want.items()}
        shutil.rmtree(root)
