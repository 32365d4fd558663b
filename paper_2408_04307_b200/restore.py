"""Partial-expert restore: the byte side of `resolve_recovery`.

The reference decides, per unit, where its newest full copy lives
(`CheckpointEngine.resolve_recovery`, engine.py:231-284) but never moves
bytes.  Here the decisions are executed:

  memory   the unit's ranges are copied H2D straight out of the pinned host
           snapshot buffer of the decided version on the decided (surviving)
           node (the two-level engine's in-memory copy; engine.py:214-229),
  storage  the unit's entry files of the decided version are read into a
           pinned bounce slot, CRC-32C verified against the manifest
           (DiskStore.load_checkpoint semantics, store.py:267-282), and
           copied H2D,
  initial  experts never saved anywhere are regenerated from their seed
           (arena.fill_unit).

Streaming: pieces are grouped into batches of at most ``slot_bytes``; two
pinned host slots and two device slots alternate, so file reads of batch
i+1 (a host thread pool) overlap the H2D copy and the `pec_unpack` scatter
of batch i into the state arena (one launch per batch).  A host slot is
refilled as soon as its own H2D has run (an event), not after its batch's
verification and scatter, so reads and H2D copies never take turns (they
did: 19-20 GB/s; now 36.6 GB/s for 26.1 GB, the reads at ~42 GB/s being the
bound).  Entries larger
than a slot are split; their CRC is chained across the pieces.
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass
from typing import Dict, Iterable, List, Optional, Tuple

import numpy as np

from . import device as D
from .engine import RecoveryPlan
from .staging import STAGE_ALIGN, DeviceTable
from .store import ChecksumMismatchError, crc32c


@dataclass
class RestoreReport:
    units: int
    memory_bytes: int
    storage_bytes: int
    initial_units: int
    unpack_ms: float      # sum of the per-batch unpack kernel times
    batches: int = 0
    wall_s: float = 0.0
    phases: Optional[Dict[str, float]] = None   # host seconds per restore phase


@dataclass
class _Piece:
    unit: str
    start: int            # byte range of the unit image
    stop: int
    kind: str             # "file" | "host" | "bytes"
    path: Optional[str] = None       # file pieces
    file_off: int = 0
    entry: Optional[str] = None
    entry_crc: int = 0
    entry_size: int = 0
    last: bool = False
    host: object = None              # host pieces: pinned tensor + offset
    host_off: int = 0

    @property
    def nbytes(self) -> int:
        return self.stop - self.start


def _place(pos: int, src_offset: int, align: int = STAGE_ALIGN) -> int:
    return pos + ((src_offset - pos) % align)


class _Ring:
    """Two pinned host slots + two device slots, allocated once per engine."""

    def __init__(self, device, slot_bytes: int):
        import torch
        self.slot_bytes = slot_bytes
        self.host = [torch.empty(slot_bytes, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
        self.dev = [torch.empty(slot_bytes, dtype=torch.uint8, device=device) for _ in range(2)]
        # event: the host slot's H2D finished (the host slot may be refilled).
        # A device slot is reused in stream order: batch i+2's H2D is enqueued
        # after batch i's unpack on the same stream.
        self.free = [None, None]


def _ring(engine, slot_bytes: int) -> _Ring:
    r = getattr(engine, "_restore_ring", None)
    if r is None or r.slot_bytes < slot_bytes:
        r = _Ring(engine.device, slot_bytes)
        engine._restore_ring = r
    return r


def _pieces(engine, plan: RecoveryPlan, wanted, slot_bytes: int):
    """Expand decisions into ordered pieces (entries split at slot size)."""
    arena, store, layout = engine.arena, engine.store, engine.layout
    step = slot_bytes - STAGE_ALIGN
    pieces: List[_Piece] = []
    initial: List[str] = []
    metas: Dict[int, object] = {}
    manifests: Dict[int, object] = {}
    peers: Dict[Tuple[int, int], object] = {}
    for key in wanted:
        d = plan.decisions[key]
        if d.source == "initial":
            initial.append(key)
            continue
        if d.source == "memory":
            buf = next((b for b in engine.buffers.buffers
                        if b.version == d.version and b.snapshot_completed), None)
            if buf is None or not engine.has_bytes(buf):
                raise RuntimeError(f"memory source v{d.version} for {key} is not in this process")
            found = False
            for r in layout.ranks_of_node(d.node):  # only the decided (surviving) node
                if r in engine.ranks:                # this process's pinned buffer: H2D
                    st, base0, kind = (engine.snapshot_layout(buf, r),
                                       engine.snapshot_region(buf, r), "host")
                    src = engine.host[buf.buffer_id]
                else:                                # a peer process's node-shared buffer
                    peer = peers.get((r, d.version))
                    if peer is None and (r, d.version) not in peers:
                        peer = engine.peer_buffer(r, d.version) if hasattr(engine, "peer_buffer") \
                            else None
                        peers[(r, d.version)] = peer
                    if peer is None:
                        continue
                    src, st = peer[0].array, peer[1]
                    base0, kind = peer[2], "bytes"
                for e in st.entries:
                    if e.unit_key != key:
                        continue
                    found = True
                    base = base0 + e.stage_offset
                    for lo in range(e.start, e.stop, step):
                        hi = min(e.stop, lo + step)
                        pieces.append(_Piece(key, lo, hi, kind, host=src,
                                             host_off=base + (lo - e.start)))
            if not found:
                raise RuntimeError(f"unit {key} not held in this process's buffer v{d.version}")
            continue
        v = d.version
        if v not in metas:
            metas[v] = store.meta(v)
            manifests[v] = store.manifest(v)
        if not hasattr(store, "version_dir"):  # MemoryStore: verified bytes in RAM
            for sk, e in sorted(metas[v].entries.items()):
                if e.unit_key == key:
                    data = store.load_checkpoint(v, [sk])[sk]
                    for lo in range(e.start, e.stop, step):
                        hi = min(e.stop, lo + step)
                        pieces.append(_Piece(key, lo, hi, "bytes", host=data,
                                             host_off=lo - e.start))
            continue
        vdir = store.version_dir(v)
        for sk, e in sorted(metas[v].entries.items()):
            if e.unit_key != key:
                continue
            rel, size, crc = manifests[v].entries[sk]
            path = str(vdir / rel)
            if not os.path.exists(path):
                raise ChecksumMismatchError(sk, "entry file missing")
            if os.path.getsize(path) != size or size != e.stop - e.start:
                raise ChecksumMismatchError(sk, f"size {os.path.getsize(path)} != manifest {size}")
            for lo in range(e.start, e.stop, step):
                hi = min(e.stop, lo + step)
                pieces.append(_Piece(key, lo, hi, "file", path=path, file_off=lo - e.start,
                                     entry=sk, entry_crc=crc, entry_size=e.stop - e.start,
                                     last=hi == e.stop))
    return pieces, initial, peers


_READ_STEP = 4 << 20   # CRC each 4 MiB right after reading it, while cache-hot
_SUB_READ = 8 << 20    # file pieces are read as independent sub-ranges of this size


def _sub_jobs(files):
    """Split file pieces [(piece, slot_off, host)] into <= 8 MiB sub-reads so
    the pool's threads share one large entry instead of one thread per
    entry."""
    jobs = []
    for k, (p, off, host) in enumerate(files):
        for lo in range(0, p.nbytes, _SUB_READ):
            jobs.append((k, p.path, p.file_off + lo, host, off + lo, min(_SUB_READ, p.nbytes - lo),
                         p.entry))
    return jobs


def _read_sub(job, want_crc: bool):
    """pread one sub-range into the pinned slot; its CRC-32C if asked (4 MiB
    steps, cache-hot)."""
    _, path, file_off, host, slot_off, n, entry = job
    view = memoryview(host.numpy()).cast("B")[slot_off:slot_off + n]
    crc = 0
    fd = os.open(path, os.O_RDONLY)
    try:
        got = 0
        while got < n:
            want = min(_READ_STEP, n - got)
            k = os.preadv(fd, [view[got:got + want]], file_off + got)
            if not k:
                raise ChecksumMismatchError(entry, "short read")
            if want_crc:
                crc = crc32c(view[got:got + k], crc)
            got += k
    finally:
        os.close(fd)
    return crc


def _read_files(pool, files, want_crc: bool):
    """Read every file piece of a batch with all pool threads; per-piece
    CRC-32Cs (sub-range CRCs combined in order) when ``want_crc``."""
    jobs = _sub_jobs(files)
    crcs = list(pool.map(lambda j: _read_sub(j, want_crc), jobs))
    if not want_crc:
        return None
    out = [None] * len(files)
    for j, c in zip(jobs, crcs):
        k, n = j[0], j[5]
        out[k] = c if out[k] is None else D.crc32c_combine(out[k], c, n)
    return [0 if c is None else c for c in out]


def _chain(running: Dict[str, int], p: "_Piece", crc: int) -> None:
    """Fold a piece's CRC into its entry's running CRC; verify at the end."""
    prev = running.get(p.entry)
    running[p.entry] = crc if prev is None else D.crc32c_combine(prev, crc, p.nbytes)
    if p.last and running.pop(p.entry) != p.entry_crc:
        raise ChecksumMismatchError(p.entry, "crc32c mismatch")


def restore(engine, plan: RecoveryPlan, keys: Optional[Iterable[str]] = None,
            chunk_log2: int = D.DEFAULT_CHUNK_LOG2, stream=None,
            slot_bytes: int = 256 << 20, io_threads: Optional[int] = None,
            verify: str = "device") -> RestoreReport:
    """Execute ``plan`` for the units resident in ``engine.arena`` (or the
    given subset ``keys``).  ``engine`` is a DeviceCheckpointEngine whose
    ``store`` (a DiskStore) holds the storage versions.

    Every storage entry is verified BEFORE any of its bytes reach the state
    arena (the reference's load_checkpoint verifies every entry before it
    returns bytes, store.py:267-282): the bytes land in a device slot (or,
    for an entry larger than a slot, a device buffer of the entry's size),
    ``verify="device"`` checksums them there with `pec_crc_device` and
    ``"host"`` while reading the files, and only entries whose CRC-32C
    matches the manifest are scattered (`pec_unpack`).  A batch is committed
    after the next batch's files are read, so verification never stalls the
    file reads.  A mismatch raises ChecksumMismatchError before the entry's
    unit is touched; ``err.committed_units`` lists the units already
    restored (from verified bytes) when it was raised."""
    if verify not in ("device", "host"):
        raise ValueError("verify must be 'device' or 'host'")
    if io_threads is None:          # one reader per usable core
        io_threads = max(4, len(os.sched_getaffinity(0)))
    import time
    import torch
    t_start = time.perf_counter()
    arena = engine.arena
    dev = arena.device
    wanted = [k for k in (keys if keys is not None else plan.decisions) if arena.has(k)]
    slot_bytes = max(1 << 20, slot_bytes)
    pieces, initial, peers = _pieces(engine, plan, wanted, slot_bytes)
    for key in initial:
        arena.fill_unit(key)
    rep = RestoreReport(len(wanted), 0, 0, len(initial), 0.0)
    ph = dict.fromkeys(("plan", "slot_wait", "read", "h2d_enqueue", "verify_enqueue",
                        "commit", "drain"), 0.0)
    ph["plan"] = time.perf_counter() - t_start
    rep.phases = ph
    if not pieces:
        torch.cuda.synchronize(dev)
        rep.wall_s = time.perf_counter() - t_start
        return rep
    split = {p.entry for p in pieces if p.kind == "file" and not (p.last and p.file_off == 0)}

    # batches of pieces, each laid out like a staging buffer (congruent mod 256)
    batches: List[List[Tuple[_Piece, int]]] = []
    cur: List[Tuple[_Piece, int]] = []
    pos = 0
    for p in pieces:
        off = _place(pos, arena.slot(p.unit).offset + p.start)
        if cur and off + p.nbytes > slot_bytes:
            batches.append(cur)
            cur = []
            off = _place(0, arena.slot(p.unit).offset + p.start)
        cur.append((p, off))
        pos = off + p.nbytes
    if cur:
        batches.append(cur)

    ring = _ring(engine, slot_bytes)
    s = stream or torch.cuda.Stream(device=dev)
    s.wait_stream(torch.cuda.current_stream(dev))  # e.g. initial fills / prior wipes
    running: Dict[str, int] = {}   # entry -> chained CRC of the pieces verified so far
    landing: Dict[str, Tuple[object, int]] = {}   # split entry -> (device buffer, src offset)
    committed: List[str] = []
    timers = []
    crc_host = torch.empty(len(pieces) if verify == "device" else 1, dtype=torch.int32,
                           pin_memory=True)
    crc_pos = 0
    crc_scratch: Dict[int, Tuple[object, object]] = {}

    def dev_src(p: _Piece, dslot, off: int) -> int:
        if p.entry in split:
            buf, base = landing[p.entry]
            return buf.data_ptr() + base + p.file_off
        return dslot.data_ptr() + off

    def commit(rec) -> None:
        """Verify a batch's storage pieces, then scatter what verified."""
        batch, slot, dslot, hcrc, ready, crcs, _table = rec
        if ready is not None:
            ready.synchronize()
            crcs = [int(v) for v in hcrc.numpy().view(np.uint32)]
        rows = []
        units = []
        keep = []              # landing buffers stay referenced until their scatter is enqueued
        try:
            fi = 0
            for p, off in batch:
                if p.kind == "file":
                    _chain(running, p, crcs[fi])
                    fi += 1
                    if p.entry in split:
                        if p.last:       # the whole entry verified: scatter it at once
                            buf, base = landing.pop(p.entry)
                            keep.append(buf)
                            e0 = p.start - p.file_off
                            rows.append((buf.data_ptr() + base,
                                         arena.base_address + arena.slot(p.unit).offset + e0,
                                         p.stop - e0))
                            units.append(p.unit)
                        continue
                rows.append((dslot.data_ptr() + off,
                             arena.base_address + arena.slot(p.unit).offset + p.start, p.nbytes))
                units.append(p.unit)
        except ChecksumMismatchError as err:
            err.committed_units = sorted(set(committed))
            raise
        table = np.zeros(len(rows), dtype=D.DESC_DTYPE)
        for i, (a, b, n) in enumerate(rows):
            table[i] = (a, b, n, 0)
        nchunks = D.plan_chunks(table, chunk_log2)
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(s)
        if rows:
            dt = DeviceTable(table, nchunks, dev, chunk_log2)
            D.unpack(dt.tensor, dt.n, dt.total_chunks, chunk_log2, D.MODE_AUTO, stream=s)
            timers.append((t0, t1, dt))
        t1.record(s)
        committed.extend(units)

    pending = None
    try:
        with ThreadPoolExecutor(max_workers=io_threads) as pool:
            for bi, batch in enumerate(batches):
                slot = bi % 2
                tp = time.perf_counter()
                if ring.free[slot] is not None:
                    ring.free[slot].synchronize()   # the slot's previous H2D has run
                hslot, dslot = ring.host[slot], ring.dev[slot]
                files = [(p, off, hslot) for p, off in batch if p.kind == "file"]
                tq = time.perf_counter()
                ph["slot_wait"] += tq - tp
                crcs = _read_files(pool, files, want_crc=verify == "host")
                for p, off in batch:
                    if p.kind == "bytes":
                        hslot.numpy()[off:off + p.nbytes] = np.frombuffer(
                            p.host, dtype=np.uint8)[p.host_off:p.host_off + p.nbytes]
                        if p.entry is None and plan.decisions[p.unit].source == "memory":
                            rep.memory_bytes += p.nbytes
                        else:
                            rep.storage_bytes += p.nbytes
                    elif p.kind == "file":
                        rep.storage_bytes += p.nbytes
                tp = time.perf_counter()
                ph["read"] += tp - tq
                with torch.cuda.stream(s):
                    for p, off in batch:
                        if p.kind == "file" and p.entry in split and p.entry not in landing:
                            # a device buffer for the whole entry, allocated on s (reused in
                            # stream order once its scatter has run)
                            lo = arena.slot(p.unit).offset + p.start - p.file_off
                            buf = torch.empty(p.entry_size + STAGE_ALIGN, dtype=torch.uint8,
                                              device=dev)
                            landing[p.entry] = (buf, (lo - buf.data_ptr()) % STAGE_ALIGN)
                    for p, off in batch:
                        if p.kind == "host":
                            dslot[off:off + p.nbytes].copy_(p.host[p.host_off:p.host_off + p.nbytes],
                                                            non_blocking=True)
                            rep.memory_bytes += p.nbytes
                        elif p.kind == "file" and p.entry in split:
                            buf, base = landing[p.entry]
                            o = base + p.file_off
                            buf[o:o + p.nbytes].copy_(hslot[off:off + p.nbytes], non_blocking=True)
                        else:
                            dslot[off:off + p.nbytes].copy_(hslot[off:off + p.nbytes],
                                                            non_blocking=True)
                h2d_done = torch.cuda.Event()
                h2d_done.record(s)
                ring.free[slot] = h2d_done
                tq = time.perf_counter()
                ph["h2d_enqueue"] += tq - tp
                hcrc, ready = None, None
                if verify == "device" and files:
                    table = np.zeros(len(files), dtype=D.DESC_DTYPE)
                    for i, (p, off, _) in enumerate(files):
                        table[i] = (dev_src(p, dslot, off), 0, p.nbytes, 0)
                    nchunks = D.plan_chunks(table, chunk_log2)
                    dt = DeviceTable(table, nchunks, dev, chunk_log2)
                    need = D.crc_scratch_words(nchunks)
                    sc = crc_scratch.get(slot)
                    if sc is None or sc[0].numel() < need or sc[1].numel() < len(files):
                        sc = (torch.empty(need, dtype=torch.int32, device=dev),
                              torch.empty(max(len(files), 1), dtype=torch.int32, device=dev))
                        crc_scratch[slot] = sc
                    D.crc_device(dt.tensor, dt.n, dt.total_chunks, sc[0], sc[1], chunk_log2, stream=s)
                    hcrc = crc_host[crc_pos:crc_pos + dt.n]
                    crc_pos += dt.n
                    with torch.cuda.stream(s):
                        hcrc.copy_(sc[1][:dt.n], non_blocking=True)
                    ready = torch.cuda.Event()
                    ready.record(s)
                    rec_table = dt     # alive until the batch commits (after `ready`)
                else:
                    rec_table = None
                rec = (batch, slot, dslot, hcrc, ready, crcs, rec_table)
                tp = time.perf_counter()
                ph["verify_enqueue"] += tp - tq
                # the previous batch commits now: its verification ran while this
                # batch's files were read
                if pending is not None:
                    commit(pending)
                pending = rec
                ph["commit"] += time.perf_counter() - tp
            tp = time.perf_counter()
            if pending is not None:
                commit(pending)
    except BaseException:
        # a failed restore (e.g. ChecksumMismatchError) must not leave H2D copies or
        # scatters in flight on the ring's slots: the next restore reuses them
        s.synchronize()
        for peer in peers.values():
            if peer is not None:
                peer[0].close()
        raise
    torch.cuda.current_stream(dev).wait_stream(s)
    s.synchronize()
    ph["drain"] = time.perf_counter() - tp
    for peer in peers.values():
        if peer is not None:
            peer[0].close()
    rep.unpack_ms = sum(a.elapsed_time(b) for a, b, _ in timers)
    rep.batches = len(batches)
    rep.wall_s = time.perf_counter() - t_start
    return rep
