"""Partial-expert restore: the byte side of `resolve_recovery`.

The reference decides, per unit, where its newest full copy lives
(`CheckpointEngine.resolve_recovery`, engine.py:231-284) but never moves
bytes.  Here the decisions are executed:

  memory   the unit's ranges are copied H2D straight out of the pinned host
           snapshot buffer of the decided version (the two-level engine's
           in-memory copy; engine.py:214-229),
  storage  the unit's entry files of the decided version are read (CRC
           verified, DiskStore.load_checkpoint semantics, store.py:267-282)
           into a pinned restore buffer, then copied H2D,
  initial  experts never saved anywhere are regenerated from their seed
           (arena.fill_unit).

All restored ranges then go through ONE `pec_unpack` launch that scatters
them from the device restore staging into the state arena.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, Iterable, List, Optional, Tuple

import numpy as np

from . import device as D
from .engine import RecoveryPlan
from .staging import STAGE_ALIGN, DeviceTable


@dataclass
class RestoreReport:
    units: int
    memory_bytes: int
    storage_bytes: int
    initial_units: int
    unpack_ms: float


def _place(pos: int, src_offset: int, align: int = STAGE_ALIGN) -> int:
    return pos + ((src_offset - pos) % align)


def restore(engine, plan: RecoveryPlan, keys: Optional[Iterable[str]] = None,
            chunk_log2: int = D.DEFAULT_CHUNK_LOG2, stream=None) -> RestoreReport:
    """Execute ``plan`` for the units resident in ``engine.arena`` (or the
    given subset ``keys``).  ``engine`` is a DeviceCheckpointEngine."""
    import torch
    arena = engine.arena
    store = engine.store
    dev = arena.device
    wanted = [k for k in (keys if keys is not None else plan.decisions) if arena.has(k)]

    # (unit, start, stop, host source) pieces; host source = (array, offset)
    mem_pieces: List[Tuple[str, int, int, object, int]] = []
    by_version: Dict[int, List[Tuple[str, object]]] = {}
    initial = []
    for key in wanted:
        d = plan.decisions[key]
        if d.source == "initial":
            initial.append(key)
        elif d.source == "memory":
            buf = next((b for b in engine.buffers.buffers
                        if b.version == d.version and b.snapshot_completed), None)
            if buf is None or not engine.has_bytes(buf):
                raise RuntimeError(f"memory source v{d.version} for {key} is not in this process")
            rec = engine._inflight[buf.buffer_id]
            host = engine.host[buf.buffer_id]  # pinned: H2D slices stay async
            found = False
            for r, st in rec.layouts.items():
                if engine.layout.node_of_rank(r) != d.node:
                    continue  # only the decided (surviving) node's copy
                for e in st.entries:
                    if e.unit_key == key:
                        mem_pieces.append((key, e.start, e.stop, host, rec.region[r] + e.stage_offset))
                        found = True
            if not found:
                raise RuntimeError(f"unit {key} not held in this process's buffer v{d.version}")
        else:
            by_version.setdefault(d.version, []).append(key)

    # storage pieces: entry files of each version, read into one pinned buffer
    sto_pieces: List[Tuple[str, int, int, int]] = []  # unit, start, stop, restore-host offset
    placements: Dict[int, Dict[str, Tuple[object, int]]] = {}
    pos = 0
    for version, units in sorted(by_version.items()):
        meta = store.meta(version)
        uset = set(units)
        for sk, e in sorted(meta.entries.items()):
            if e.unit_key in uset:
                src = arena.slot(e.unit_key).offset + e.start
                off = _place(pos, src)
                placements.setdefault(version, {})[sk] = off
                sto_pieces.append((e.unit_key, e.start, e.stop, off))
                pos = off + (e.stop - e.start)
    # memory pieces follow in the same device staging
    mem_off = []
    for key, start, stop, host, hoff in mem_pieces:
        src = arena.slot(key).offset + start
        off = _place(pos, src)
        mem_off.append(off)
        pos = off + (stop - start)
    total = pos

    for key in initial:
        arena.fill_unit(key)
    if total == 0:
        torch.cuda.synchronize(dev)
        return RestoreReport(len(wanted), 0, 0, len(initial), 0.0)

    stage = torch.empty(total, dtype=torch.uint8, device=dev)
    s = stream or torch.cuda.current_stream(dev)
    sto_bytes = 0
    if placements:
        rhost = torch.empty(total, dtype=torch.uint8, pin_memory=True)
        harr = rhost.numpy()
        for version, pl in placements.items():
            store.read_into(version, {k: (harr, off) for k, off in pl.items()})
        sto_end = max(off + (stop - start) for _, start, stop, off in sto_pieces)
        with torch.cuda.stream(s):
            stage[:sto_end].copy_(rhost[:sto_end], non_blocking=True)
        sto_bytes = sum(stop - start for _, start, stop, _ in sto_pieces)
    mem_bytes = 0
    with torch.cuda.stream(s):
        for (key, start, stop, host, hoff), off in zip(mem_pieces, mem_off):
            n = stop - start
            stage[off:off + n].copy_(host[hoff:hoff + n], non_blocking=True)
            mem_bytes += n

    # one unpack over every restored range
    pieces = [(k, a, b, off) for k, a, b, off in sto_pieces] + \
        [(k, a, b, off) for (k, a, b, _, _), off in zip(mem_pieces, mem_off)]
    table = np.zeros(len(pieces), dtype=D.DESC_DTYPE)
    for i, (k, a, b, off) in enumerate(pieces):
        table[i]["src"] = stage.data_ptr() + off
        table[i]["dst"] = arena.base_address + arena.slot(k).offset + a
        table[i]["nbytes"] = b - a
    nchunks = D.plan_chunks(table, chunk_log2)
    dt = DeviceTable(table, nchunks, dev, chunk_log2)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(s)
    D.unpack(dt.tensor, dt.n, dt.total_chunks, chunk_log2, engine.pack_mode, stream=s)
    t1.record(s)
    t1.synchronize()
    if placements:
        del rhost
    return RestoreReport(len(wanted), mem_bytes, sto_bytes, len(initial), t0.elapsed_time(t1))
