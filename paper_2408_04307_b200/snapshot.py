"""The B200 two-level snapshot path: pack -> HBM staging -> D2H -> pinned
host buffer -> persist thread, driven by the reference's buffer state machine.

`DeviceCheckpointEngine` is the reference `CheckpointEngine` (engine.py)
with the byte movement the reference only models
(`transfer_us(snap_bytes, snapshot_bandwidth)`, simulator.py:57-61, 434-438)
made real:

  begin_snapshot   pack stream waits for the compute stream (the state is
                   consistent there), one `pec_pack` launch gathers every
                   local rank's planned ranges into the HBM staging buffer,
                   then the copy stream drains staging into the pinned host
                   buffer whose id the state machine handed out.
  wait_pack        the compute stream waits for the pack before the next
                   optimizer step may modify the state (the only
                   consistency-critical part; the drain overlaps training).
  complete_snapshot  after the drain's event: SNAPSHOTTED = bytes in host RAM.
  start_persist    a background thread writes the persisted subset straight
                   out of the host buffer (CRC-32C via libpec), multi-rank
                   commits through a gloo group (rank files, then rank 0
                   publishes meta/manifest/COMPLETE).
  complete_persist publishes and rotates the buffer roles.

`PecCheckpointer` is the training-loop driver, the counterpart of
`Simulation._trigger_checkpoint` / `step` (simulator.py:396-457, 546-576):
token counting every iteration, selection + plan + snapshot every
``i_ckpt`` iterations, asynchronous completion via `poll`.
"""

from __future__ import annotations

import threading
import time
from concurrent.futures import Future, ThreadPoolExecutor
from dataclasses import dataclass
from typing import Dict, Iterable, List, Optional, Sequence, Tuple

import numpy as np

from . import device as D
from .arena import StateArena
from .engine import Buffer, CheckpointEngine, NoFreeBufferError
from .planner import (
    ADAPTIVE_PEC,
    BASELINE,
    EQUAL_PEC,
    LOAD_AWARE,
    PecConfig,
    PhaseAssignment,
    ShardPlan,
    build_phase_assignment,
    plan_adaptive,
    plan_baseline,
    plan_equal,
)
from .selector import select_window
from .staging import DeviceTable, PlanTemplate, StagingLayout, drain_cuts, split_table
from .store import StoreEntry
from .topology import RankLayout


def _own_control_group():
    """With several processes, the persist thread's commit (all_gather_object
    + barrier, distributed.commit_version) must not share a communicator with
    the training thread's NCCL collectives (the counters' all-reduce): the
    two threads could order them differently on different ranks.  A
    dedicated gloo group — created collectively, every rank builds its
    checkpointer at the same point — carries only the persist protocol.
    Single process: None."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return None
    return dist.new_group(backend="gloo")


class PersistAborted(RuntimeError):
    """A fault interrupted a persist before its version was published."""


@dataclass
class RecoveryOutcome:
    """What `PecCheckpointer.recover` did (the byte-moving counterpart of the
    reference's `_handle_fault` bookkeeping, simulator.py:473-544)."""
    restart_iteration: int        # resume training at restart_iteration + 1
    version_skew: int
    plan: object                  # RecoveryPlan, or None for a restart from scratch
    report: object                # RestoreReport, or None
    expert_restore: Dict[Tuple[int, int], int]   # (layer, expert) -> restored iteration


@dataclass
class _Inflight:
    """Device-side record of one buffer's snapshot."""
    layouts: Dict[int, StagingLayout]     # local rank -> layout (offsets within its region)
    region: Dict[int, int]                # local rank -> byte offset of its region
    nbytes: int
    pack_done: object = None
    drain_done: object = None
    t_begin: float = 0.0
    entry_crc: object = None              # pinned int32 [n] (MODE_CRC)
    crc_keys: object = None
    crc_segments: object = None           # pipelined MODE_CRC: [(pinned crcs, rows, nbytes)]
    pending: object = None                # device plan: (meta, ready) until the drain is enqueued
    persist_due: object = None            # device plan: persist sets per layer
    early: object = None                  # device plan: rank -> fixed-prefix bytes drained early
    drain_start: object = None            # event: the copy stream starts the first drain piece


class DeviceCheckpointEngine(CheckpointEngine):
    """Reference CheckpointEngine + real snapshot/persist bytes on B200."""

    def __init__(self, layout: RankLayout, store, arena: StateArena,
                 ranks: Optional[Sequence[int]] = None, n_buffers: int = 3,
                 pack_mode: int = D.MODE_AUTO, chunk_log2: int = D.DEFAULT_CHUNK_LOG2,
                 control_group=None, persist_threads: int = 1,
                 shared_host_prefix: Optional[str] = None):
        import torch
        super().__init__(layout, store, n_buffers)
        self.shared_prefix = shared_host_prefix
        self._shared: Dict[int, object] = {}
        self.arena = arena
        self.device = arena.device
        self.ranks = tuple(ranks) if ranks is not None else arena.ranks
        if pack_mode == D.MODE_AUTO:
            # with a persist tier, the pack computes every entry's CRC-32C in
            # the same pass (1.0x the plain pack's HBM rate); the persist
            # thread then writes files without reading them for checksums
            pack_mode = D.MODE_CRC if store is not None else D.MODE_BULK
        self.pack_mode = pack_mode
        # split host-planned packs so the drain starts after the first
        # drain_first bytes (cuts grow 4x: 64 MiB, 256 MiB, 1 GiB, ...)
        self.pipelined_drain = True
        self.drain_first = 64 << 20
        self.chunk_log2 = chunk_log2
        if control_group is None and store is not None:
            control_group = _own_control_group()
        # negative-control hook for tests ONLY: False drops the pack stream's
        # wait on the compute stream (the snapshot then races the update it
        # must follow; tests/test_overlap_gpu.py proves the test detects it)
        self._consistency_wait = True
        self.group = control_group
        # high priority: when the pack and training kernels both have CTAs
        # waiting, the pack (the only training-blocking part) goes first
        self.pack_stream = torch.cuda.Stream(device=self.device, priority=-1)
        self.copy_stream = torch.cuda.Stream(device=self.device)
        self.staging = None
        self.host: List[Optional[object]] = [None] * n_buffers
        self._inflight: Dict[int, _Inflight] = {}       # buffer_id -> record
        self._tables: Dict[Tuple, Tuple[DeviceTable, Dict[int, StagingLayout], Dict[int, int], int]] = {}
        self._staging_free = None
        self._persist_pool = ThreadPoolExecutor(max_workers=persist_threads,
                                                thread_name_prefix="pec-persist")
        self._persist: Dict[int, Tuple[Future, List[StoreEntry]]] = {}
        self._abort_persist = threading.Event()
        self._pending_bid: Optional[int] = None  # device-planned snapshot awaiting its drain
        self._pinned_cache: Dict[tuple, object] = {}
        self.stats = {"pack_ms": [], "drain_ms": [], "persist_s": [], "snap_bytes": []}

    # -- buffers -----------------------------------------------------------------
    def _ensure_staging(self, nbytes: int):
        import torch
        if self.staging is None or self.staging.numel() < nbytes:
            if self.staging is not None:
                torch.cuda.current_stream(self.device).synchronize()
                self.pack_stream.synchronize()
                self.copy_stream.synchronize()
            self.staging = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=self.device)
            self._tables.clear()  # addresses changed

    def _ensure_host(self, buffer_id: int, nbytes: int):
        import torch
        h = self.host[buffer_id]
        if h is None or h.numel() < nbytes:
            if self.shared_prefix is None:
                # cudaHostAlloc through torch's pinned allocator (pinning
                # lifetime tied to the tensor).  An anonymous THP mapping +
                # cudaHostRegister sets up 3x faster but was withdrawn, see
                # DESIGN.md section 3.
                self.host[buffer_id] = torch.empty(max(nbytes, 256), dtype=torch.uint8,
                                                   pin_memory=True)
            else:
                from .hostmem import SharedHostBuffer, buffer_name
                # one node-shared file per buffer, named by the engine's first
                # rank; every hosted rank's region is published with its
                # offset (_publish_meta), so peers map the right bytes
                old = self._shared.pop(buffer_id, None)
                self.host[buffer_id] = None
                if old is not None:
                    old.close()
                shb = SharedHostBuffer(buffer_name(self.shared_prefix, self.ranks[0], buffer_id),
                                       max(nbytes, 256))
                self._shared[buffer_id] = shb
                self.host[buffer_id] = shb.tensor
        return self.host[buffer_id]

    def _pinned(self, tag, buffer_id: int, n: int, dtype):
        """A pinned host array of >= n elements owned by (tag, buffer_id),
        allocated once and reused by every later snapshot into that buffer:
        pinning inside a checkpoint would stall the host between the launches
        it enqueues.  Safe to reuse: a buffer's small host-side records (CRCs,
        sizes, selections) are read before the buffer can be snapshotted
        into again (the state machine frees it only after its persist)."""
        import torch
        key = (tag, buffer_id)
        t = self._pinned_cache.get(key)
        if t is None or t.numel() < n or t.dtype != dtype:
            t = torch.empty(max(1, n), dtype=dtype, pin_memory=True)
            self._pinned_cache[key] = t
        return t[:n]

    # -- node-shared snapshot metadata (cross-process memory restore) ---------------
    def _meta_path(self, rank: int, buffer_id: int) -> str:
        from .hostmem import SHM_DIR, buffer_name
        import os
        return os.path.join(SHM_DIR, buffer_name(self.shared_prefix, rank, buffer_id) + ".json")

    def _publish_meta(self, buf: Buffer, rec) -> None:
        import json
        import os
        if self.shared_prefix is None:
            return
        from .hostmem import buffer_name
        for r in rec.layouts:
            path = self._meta_path(r, buf.buffer_id)
            tmp = path + ".tmp"
            with open(tmp, "w") as f:
                json.dump({"version": buf.version, "iteration": buf.iteration,
                           "nbytes": rec.layouts[r].nbytes,
                           "file": buffer_name(self.shared_prefix, self.ranks[0], buf.buffer_id),
                           "offset": rec.region[r]}, f)
            os.replace(tmp, path)

    def _retract_meta(self, buffer_id: int) -> None:
        import os
        if self.shared_prefix is None:
            return
        for r in self.ranks:
            try:
                os.unlink(self._meta_path(r, buffer_id))
            except FileNotFoundError:
                pass

    def peer_buffer(self, rank: int, version: int):
        """(mapped SharedHostBuffer, StagingLayout, region offset) of peer
        ``rank``'s in-memory copy of ``version`` on this node, or None."""
        import json
        from .arena import PeerSlots
        from .hostmem import SharedHostBuffer
        if self.shared_prefix is None:
            return None
        buf = next((b for b in self.buffers.buffers if b.version == version), None)
        if buf is None or buf.content is None:
            return None
        for bid in range(len(self.buffers.buffers)):
            try:
                with open(self._meta_path(rank, bid)) as f:
                    meta = json.load(f)
            except (FileNotFoundError, ValueError):
                continue
            if meta.get("version") != version:
                continue
            st = StagingLayout.build(buf.content.get(rank, ()), PeerSlots(self.layout, rank), rank)
            if meta["nbytes"] != st.nbytes:
                raise RuntimeError(f"peer rank {rank} v{version}: layout size mismatch "
                                   f"({st.nbytes} B vs {meta['nbytes']} B published)")
            shb = SharedHostBuffer(meta["file"], create=False, register=False)
            return shb, st, int(meta["offset"])
        return None

    def reserve(self, nbytes: int, host_buffers: Optional[int] = None) -> None:
        """Pre-allocate the staging buffer and (the first ``host_buffers``
        of) the pinned host buffers (pinning is slow: do it once, before
        training)."""
        self._ensure_staging(nbytes)
        n = len(self.host) if host_buffers is None else min(host_buffers, len(self.host))
        for i in range(n):
            self._ensure_host(i, nbytes)

    def layouts_for(self, assignment: PhaseAssignment, plan_key=None) -> Dict[int, StagingLayout]:
        """Staging layout of every local rank for an assignment (cached per
        plan key)."""
        return self._table_for(assignment, plan_key)[1]

    def snapshot_layout(self, buf: Buffer, rank: int) -> StagingLayout:
        """Staging / host-buffer layout of ``rank``'s entries in ``buf``."""
        return self._inflight[buf.buffer_id].layouts[rank]

    def snapshot_region(self, buf: Buffer, rank: int) -> int:
        """Byte offset of ``rank``'s region in ``buf``'s host buffer."""
        return self._inflight[buf.buffer_id].region[rank]

    def snapshot_nbytes(self, buf: Buffer) -> int:
        return self._inflight[buf.buffer_id].nbytes

    # -- plan -> device table ------------------------------------------------------
    def _table_for(self, assignment: PhaseAssignment, key=None):
        if key is not None and key in self._tables:
            return self._tables[key]
        layouts, region, pos = {}, {}, 0
        for r in self.ranks:
            st = StagingLayout.build(assignment.get(r, ()), self.arena, r)
            layouts[r], region[r] = st, pos
            pos += (st.nbytes + 255) // 256 * 256
        self._ensure_staging(pos)
        tables = [layouts[r].descriptors(self.arena.base_address,
                                         self.staging.data_ptr() + region[r],
                                         chunk_log2=self.chunk_log2)[0] for r in self.ranks]
        table = np.concatenate(tables) if tables else np.zeros(0, dtype=D.DESC_DTYPE)
        total = D.plan_chunks(table, self.chunk_log2)
        dt = DeviceTable(table, total, self.device, self.chunk_log2)
        dt.segments = None
        if self.pipelined_drain and drain_cuts(pos, self.drain_first):
            # the pack in staging-ordered segments, each drained as soon as it
            # is packed (begin_snapshot): the drain starts ~20 us into the pack.
            # CRC mode: per-segment entry CRCs, rows split by a cut are joined
            # on the host (crc32c_combine)
            dt.segments = []
            for sub, n, lo, hi, rows in split_table(
                    table, self.staging.data_ptr(), drain_cuts(pos, self.drain_first),
                    self.chunk_log2, with_rows=True):
                sdt = DeviceTable(sub, n, self.device, self.chunk_log2)
                sdt.rows = rows
                sdt.row_bytes = sub["nbytes"].astype(np.int64)
                if self.pack_mode == D.MODE_CRC:
                    self._crc_scratch(sdt)   # with the table: no allocation at pack time
                dt.segments.append((sdt, lo, pos if hi is None else hi))
        elif self.pack_mode == D.MODE_CRC:
            self._crc_scratch(dt)
        entry = (dt, layouts, region, pos)
        if key is not None:
            self._tables[key] = entry
        return entry

    def _crc_scratch(self, table: DeviceTable) -> None:
        import torch
        if getattr(table, "entry_crc", None) is None:
            table.chunk_crc = torch.empty(D.crc_scratch_words(table.total_chunks),
                                          dtype=torch.int32, device=self.device)
            table.entry_crc = torch.empty(max(1, table.n), dtype=torch.int32, device=self.device)

    DRAIN_PIECE = 256 << 20

    def _drain_range(self, host, start: int, stop: int) -> None:
        for o in range(start, stop, self.DRAIN_PIECE):
            e = min(stop, o + self.DRAIN_PIECE)
            host[o:e].copy_(self.staging[o:e], non_blocking=True)

    def _drain(self, host, nbytes: int) -> None:
        """Staging -> pinned host copy of the snapshot, enqueued on the current
        (copy) stream as 256 MiB pieces: on some B200 boxes one 12.6 GB copy
        runs at 52.5 GB/s where 256 MiB pieces reach 56.1 (a 1 GiB copy: 57.1;
        `profiles/r1/drain_probe.json`); elsewhere both hit the same peak."""
        for o in range(0, nbytes, self.DRAIN_PIECE):
            e = min(nbytes, o + self.DRAIN_PIECE)
            host[o:e].copy_(self.staging[o:e], non_blocking=True)

    def _launch_pack(self, table: DeviceTable, stream) -> None:
        """pec_pack, or pec_pack_crc in MODE_CRC (per-entry CRCs land in
        table.entry_crc on device)."""
        if self.pack_mode != D.MODE_CRC:
            D.pack(table.tensor, table.n, table.total_chunks, table.chunk_log2, self.pack_mode,
                   stream=stream)
            return
        self._crc_scratch(table)
        D.pack_crc(table.tensor, table.n, table.total_chunks, table.chunk_crc, table.entry_crc,
                   table.chunk_log2, stream=stream)

    # -- snapshot --------------------------------------------------------------------
    def pack_only(self, assignment: PhaseAssignment, plan_key=None, stream=None):
        """Pack the local ranks' ranges into HBM staging without draining
        (the consistency-critical device step alone).  Returns
        (start_event, end_event, payload_bytes)."""
        import torch
        table, layouts, region, nbytes = self._table_for(assignment, plan_key)
        s = stream or self.pack_stream
        self.finalize_pending()
        if self._staging_free is not None:
            s.wait_event(self._staging_free)
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(s)
        self._launch_pack(table, s)
        t1.record(s)
        return t0, t1, sum(l.payload_bytes for l in layouts.values())

    def begin_snapshot(self, iteration: int, checkpoint_index: int,
                       assignment: PhaseAssignment, plan_key=None, compute_stream=None) -> Buffer:
        import torch
        self.finalize_pending()
        buf = super().begin_snapshot(iteration, checkpoint_index, assignment)
        self._retract_meta(buf.buffer_id)
        try:
            table, layouts, region, nbytes = self._table_for(assignment, plan_key)
            host = self._ensure_host(buf.buffer_id, nbytes)
        except Exception:
            buf.clear()
            self.next_version -= 1
            raise
        compute = compute_stream or torch.cuda.current_stream(self.device)
        rec = _Inflight(layouts, region, nbytes, t_begin=time.perf_counter())
        ps, cs = self.pack_stream, self.copy_stream
        if self._consistency_wait:
            ps.wait_stream(compute)                   # state is consistent here
        if self._staging_free is not None:
            ps.wait_event(self._staging_free)         # previous drain read staging
        start = torch.cuda.Event(enable_timing=True)
        rec.pack_done = torch.cuda.Event(enable_timing=True)
        start.record(ps)
        rec.drain_done = torch.cuda.Event(enable_timing=True)
        if table.segments is not None:
            crc_mode = self.pack_mode == D.MODE_CRC
            if crc_mode:
                rec.crc_segments = []
                rec.crc_keys = [e.store_key for r in self.ranks for e in layouts[r].entries]
            # every segment's pack first, back to back on the pack stream (the
            # host enqueues the drains while the GPU packs), then each
            # segment's drain behind its own event on the copy stream
            seg_done = []
            for sub, _, _ in table.segments:
                self._launch_pack(sub, ps)
                seg_done.append(torch.cuda.Event())
                seg_done[-1].record(ps)
            for si, (sub, lo, hi) in enumerate(table.segments):
                cs.wait_event(seg_done[si])
                if rec.drain_start is None:
                    rec.drain_start = torch.cuda.Event(enable_timing=True)
                    rec.drain_start.record(cs)
                with torch.cuda.stream(cs):
                    self._drain_range(host, lo, min(hi, nbytes))
                    if crc_mode and sub.n:
                        pinned = self._pinned(("seg_crc", id(table), si), buf.buffer_id, sub.n,
                                              torch.int32)
                        pinned.copy_(sub.entry_crc[:sub.n], non_blocking=True)
                        rec.crc_segments.append((pinned, sub.rows, sub.row_bytes))
            rec.pack_done.record(ps)
        else:
            self._launch_pack(table, ps)
            rec.pack_done.record(ps)
        rec.pack_start = start
        cs.wait_event(rec.pack_done)
        if rec.drain_start is None:
            rec.drain_start = torch.cuda.Event(enable_timing=True)
            rec.drain_start.record(cs)
        with torch.cuda.stream(cs):
            if table.segments is None:
                self._drain(host, nbytes)
            if self.pack_mode == D.MODE_CRC and table.n and table.segments is None:
                rec.entry_crc = self._pinned("entry_crc", buf.buffer_id, table.n, torch.int32)
                rec.entry_crc.copy_(table.entry_crc[:table.n], non_blocking=True)
                rec.crc_keys = [e.store_key for r in self.ranks for e in layouts[r].entries]
        rec.drain_done.record(cs)
        self._staging_free = rec.drain_done
        self._inflight[buf.buffer_id] = rec
        self.stats["snap_bytes"].append(sum(l.payload_bytes for l in layouts.values()))
        return buf

    # -- device-planned snapshots (load-aware: no host round trip before the pack)
    def enable_device_plans(self, strategy: str) -> None:
        """Build each local rank's all-experts template once; afterwards
        `begin_snapshot_device` expands the plans on the GPU from a device
        selection (equal_pec / baseline).  Each local rank owns a fixed
        staging region sized for its largest possible plan, so the regions
        never move whatever the selection."""
        import torch
        self.strategy = strategy
        self.templates = {r: PlanTemplate(self.layout, self.arena, r, strategy, self.device)
                          for r in self.ranks}
        self.template = self.templates[self.ranks[0]]       # the single-rank case
        self._dev_region, pos = {}, 0
        for r in self.ranks:
            self._dev_region[r] = pos
            pos += (self.templates[r].max_bytes + 255) // 256 * 256
        self._dev_region_bytes = pos
        self._ensure_staging(pos)
        self._dev_tables = {r: torch.empty(max(1, t.n) * 4, dtype=torch.int64, device=self.device)
                            for r, t in self.templates.items()}
        self._dev_totals_r = {r: torch.zeros(2, dtype=torch.int64, device=self.device)
                              for r in self.ranks}
        self._dev_table = self._dev_tables[self.ranks[0]]   # single-rank names (bench, tools)
        self._dev_totals = self._dev_totals_r[self.ranks[0]]
        self._meta_stream = torch.cuda.Stream(device=self.device)

    def _expand_and_pack(self, snap_sel_dev, stream):
        import torch
        lg = self.chunk_log2
        for r in self.ranks:
            t = self.templates[r]
            D.expand_plan(t.tensor, t.n, snap_sel_dev, self.arena.base_address,
                          self.staging.data_ptr() + self._dev_region[r], self._dev_tables[r],
                          self._dev_totals_r[r], lg, stream=stream)
        expanded = torch.cuda.Event()
        expanded.record(stream)
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        if self.pack_mode == D.MODE_CRC and getattr(self, "_dev_entry_crc_r", None) is None:
            self._dev_chunk_crc_r = {
                r: torch.empty(D.crc_scratch_words(t.max_chunks(lg)),
                               dtype=torch.int32, device=self.device)
                for r, t in self.templates.items()}
            self._dev_entry_crc_r = {r: torch.empty(max(1, t.n), dtype=torch.int32,
                                                    device=self.device)
                                     for r, t in self.templates.items()}
            self._dev_entry_crc = self._dev_entry_crc_r[self.ranks[0]]
        for r in self.ranks:
            t = self.templates[r]
            if self.pack_mode == D.MODE_CRC:
                D.pack_crc(self._dev_tables[r], t.n, t.max_chunks(lg), self._dev_chunk_crc_r[r],
                           self._dev_entry_crc_r[r], lg, stream=stream,
                           totals_dev=self._dev_totals_r[r])
            else:
                D.pack_indirect(self._dev_tables[r], t.n, t.max_chunks(lg), self._dev_totals_r[r],
                                lg, self.pack_mode, stream=stream)
        t1.record(stream)
        return expanded, t0, t1

    def pack_only_device(self, snap_sel_dev, stream=None):
        """Device-only step of a load-aware snapshot: expand + pack, no drain,
        no host synchronisation.  Returns (start_event, end_event)."""
        s = stream or self.pack_stream
        self.finalize_pending()
        if self._staging_free is not None:
            s.wait_event(self._staging_free)
        _, t0, t1 = self._expand_and_pack(snap_sel_dev, s)
        return t0, t1

    def begin_snapshot_device(self, iteration: int, checkpoint_index: int, snap_sel_dev,
                              persist_sel_dev, compute_stream=None) -> Buffer:
        """Load-aware snapshot from device selections [L, k_s] / [L, k_p]:
        expand + pack are enqueued at once, plus a tiny D2H of the staged
        size and both selections; the call returns without waiting for the
        GPU.  The drain (whose size the host must know) is enqueued by
        `finalize_pending` — from `poll`/`snapshot_ready` once that tiny copy
        has landed, or at the latest by `complete_snapshot` / the next
        snapshot — which also fills the buffer's reference-format content
        and its persist sets (`persist_due`)."""
        import torch
        self.finalize_pending()
        buf = CheckpointEngine.begin_snapshot(self, iteration, checkpoint_index, None)
        self._retract_meta(buf.buffer_id)
        compute = compute_stream or torch.cuda.current_stream(self.device)
        ps, ms = self.pack_stream, self._meta_stream
        if self._consistency_wait:
            ps.wait_stream(compute)
        if self._staging_free is not None:
            ps.wait_event(self._staging_free)
        expanded, t0, t1 = self._expand_and_pack(snap_sel_dev, ps)
        # small D2H of {chunks, bytes} and both selections on a side stream
        ms.wait_event(expanded)
        R = len(self.ranks)
        head = 2 * R
        meta = self._pinned("meta", buf.buffer_id,
                            head + snap_sel_dev.numel() + persist_sel_dev.numel(), torch.int64)
        with torch.cuda.stream(ms):
            for i, r in enumerate(self.ranks):
                meta[2 * i:2 * i + 2].copy_(self._dev_totals_r[r], non_blocking=True)
            meta[head:head + snap_sel_dev.numel()].copy_(snap_sel_dev.reshape(-1),
                                                         non_blocking=True)
            meta[head + snap_sel_dev.numel():].copy_(persist_sel_dev.reshape(-1),
                                                     non_blocking=True)
            # the expanded tables themselves: finalize_pending checks every
            # kept row's staging offset and length against the host plan
            tabs = self._pinned("tabs", buf.buffer_id,
                                sum(4 * self.templates[r].n for r in self.ranks), torch.int64)
            o = 0
            for r in self.ranks:
                n4 = 4 * self.templates[r].n
                tabs[o:o + n4].copy_(self._dev_tables[r][:n4], non_blocking=True)
                o += n4
        ready = torch.cuda.Event()
        ready.record(ms)
        rec = _Inflight({}, dict(self._dev_region), 0, t_begin=time.perf_counter())
        rec.pack_start, rec.pack_done = t0, t1
        rec.pending = (meta, ready, snap_sel_dev.shape[0], snap_sel_dev.numel(), tabs)
        # the fixed-prefix drain (each rank's leading non-expert entries) needs
        # no size from the GPU: enqueue it now, so the host link is busy while
        # the size copy lands and the host enqueues the rest
        rec.early = {r: self.templates[r].fixed_prefix if self.pipelined_drain else 0
                     for r in self.ranks}
        if any(rec.early.values()):
            host = self._ensure_host(buf.buffer_id, self._dev_region_bytes)
            cs = self.copy_stream
            cs.wait_event(t1)
            rec.drain_start = torch.cuda.Event(enable_timing=True)
            rec.drain_start.record(cs)
            with torch.cuda.stream(cs):
                for r in self.ranks:
                    o = self._dev_region[r]
                    self._drain_range(host, o, o + rec.early[r])
        self._inflight[buf.buffer_id] = rec
        self._pending_bid = buf.buffer_id
        return buf

    def finalize_pending(self, block: bool = True) -> bool:
        """Enqueue the drain of the pending device-planned snapshot (if any)
        once its size/selection copy has landed (``block=False``: only if it
        already has).  Returns True when nothing is left pending."""
        import torch
        from .planner import build_phase_assignment
        bid = self._pending_bid
        if bid is None:
            return True
        rec = self._inflight[bid]
        meta, ready, L, n_snap, tabs = rec.pending
        if not block and not ready.query():
            return False
        ready.synchronize()
        buf = self.buffers.buffers[bid]
        # the rest of each region's used bytes first (the fixed prefix is on
        # its way since begin_snapshot_device), the host-side plan after
        used = {r: int(meta[2 * i + 1]) for i, r in enumerate(self.ranks)}
        host = self._ensure_host(bid, self._dev_region_bytes)
        cs = self.copy_stream
        cs.wait_event(rec.pack_done)
        rec.drain_done = torch.cuda.Event(enable_timing=True)
        if rec.drain_start is None:
            rec.drain_start = torch.cuda.Event(enable_timing=True)
            rec.drain_start.record(cs)
        with torch.cuda.stream(cs):
            for r in self.ranks:
                o = self._dev_region[r]
                self._drain_range(host, o + min(rec.early[r], used[r]), o + used[r])
        head = 2 * len(self.ranks)
        snap_h = meta[head:head + n_snap].view(L, -1).tolist()
        pers_h = meta[head + n_snap:].view(L, -1).tolist()
        due = {m: frozenset(e for e in snap_h[m] if e >= 0) for m in range(L)}
        rec.persist_due = {m: frozenset(e for e in pers_h[m] if e >= 0) for m in range(L)}
        assignment = build_phase_assignment(self.layout, due, self.strategy)
        buf.content = assignment
        layouts = {}
        o = 0
        stage0 = self.staging.data_ptr()
        for r in self.ranks:
            st = StagingLayout.build(assignment.get(r, ()), self.arena, r)
            n = self.templates[r].n
            rows = tabs[o:o + 4 * n].numpy().reshape(n, 4).view(np.uint64)
            o += 4 * n
            kept = rows[rows[:, 2] > 0]
            dev_rows = list(zip((kept[:, 1] - np.uint64(stage0 + self._dev_region[r])).tolist(),
                                kept[:, 2].tolist()))
            host_rows = [(e.stage_offset, e.nbytes) for e in st.entries]
            if st.nbytes != used[r] or dev_rows != host_rows:
                raise RuntimeError(f"device plan of rank {r} ({used[r]} B, {len(dev_rows)} "
                                   f"rows) disagrees with the host plan ({st.nbytes} B, "
                                   f"{len(host_rows)} rows)")
            layouts[r] = st
        last = self.ranks[-1]
        nbytes = self._dev_region[last] + used[last]
        rec.layouts, rec.nbytes = layouts, nbytes
        with torch.cuda.stream(cs):
            if self.pack_mode == D.MODE_CRC:
                # template order per rank; dropped entries carry nbytes 0 (crc 0)
                total_n = sum(t.n for t in self.templates.values())
                if total_n:
                    rec.entry_crc = self._pinned("entry_crc", bid, total_n, torch.int32)
                    o, keys = 0, []
                    for r in self.ranks:
                        t = self.templates[r]
                        rec.entry_crc[o:o + t.n].copy_(self._dev_entry_crc_r[r][:t.n],
                                                       non_blocking=True)
                        keys += [a.store_key for a in t.ranges]
                        o += t.n
                    rec.crc_keys = keys
        rec.drain_done.record(cs)
        self._staging_free = rec.drain_done
        self.stats["snap_bytes"].append(sum(st.payload_bytes for st in layouts.values()))
        rec.pending = None
        self._pending_bid = None
        return True

    def persist_due(self, buf: Buffer):
        """Persist sets of a device-planned snapshot (None for host plans)."""
        rec = self._inflight.get(buf.buffer_id)
        if rec is None:
            return None
        if rec.pending is not None:
            self.finalize_pending()
        return rec.persist_due

    def wait_pack(self, buf: Optional[Buffer] = None, stream=None) -> None:
        """Make ``stream`` (default: current) wait for the pack of ``buf`` (or
        the latest snapshot) before it modifies the state."""
        import torch
        rec = self._inflight.get(buf.buffer_id) if buf is not None else \
            (self._inflight[self.buffers.snapshotting.buffer_id]
             if self.buffers.snapshotting is not None else None)
        if rec is not None:
            (stream or torch.cuda.current_stream(self.device)).wait_event(rec.pack_done)

    def snapshot_ready(self, buf: Buffer) -> bool:
        rec = self._inflight.get(buf.buffer_id)
        if rec is None:
            return True
        if rec.pending is not None and not self.finalize_pending(block=False):
            return False
        return rec.drain_done.query()

    def complete_snapshot(self, buf: Buffer) -> Optional[Buffer]:
        rec = self._inflight.get(buf.buffer_id)
        if rec is not None:
            if rec.pending is not None:
                self.finalize_pending()
            rec.drain_done.synchronize()
            self.stats["pack_ms"].append(rec.pack_start.elapsed_time(rec.pack_done))
            # from the first drain piece (pipelined drains start during the pack)
            self.stats["drain_ms"].append(rec.drain_start.elapsed_time(rec.drain_done))
            self._publish_meta(buf, rec)
        return super().complete_snapshot(buf)

    # -- host bytes ---------------------------------------------------------------------
    def entry_view(self, buf: Buffer, rank: int, store_key: str) -> memoryview:
        rec = self._inflight[buf.buffer_id]
        st = rec.layouts[rank]
        e = st.entry(store_key)
        off = rec.region[rank] + e.stage_offset
        host = self.host[buf.buffer_id].numpy()
        return memoryview(host[off:off + e.nbytes])

    def payloads(self, buf: Buffer, entries: Iterable[StoreEntry]) -> Dict[str, memoryview]:
        return {e.store_key: (self.entry_view(buf, e.rank, e.store_key) if e.stop > e.start
                              else memoryview(b"")) for e in entries if e.rank in self.ranks}

    def device_crcs(self, buf: Buffer):
        """store_key -> CRC-32C computed by the pack (MODE_CRC), else None."""
        rec = self._inflight.get(buf.buffer_id)
        if rec is None:
            return None
        if rec.crc_segments is not None:
            # join the pieces of rows split at drain cuts, in staging order
            crcs = [None] * len(rec.crc_keys)
            for pinned, rows, nbytes in rec.crc_segments:
                vals = pinned.numpy().view(np.uint32)
                for v, r, n in zip(vals, rows, nbytes):
                    crcs[r] = int(v) if crcs[r] is None else D.crc32c_combine(crcs[r], int(v),
                                                                               int(n))
            return {k: (0 if c is None else c) for k, c in zip(rec.crc_keys, crcs)}
        if rec.entry_crc is None:
            return None
        vals = rec.entry_crc.numpy().view(np.uint32)
        return {k: int(v) for k, v in zip(rec.crc_keys, vals)}

    def has_bytes(self, buf: Buffer) -> bool:
        return buf.buffer_id in self._inflight

    # -- persist --------------------------------------------------------------------------
    def _write(self, buf: Buffer, entries: List[StoreEntry]) -> float:
        """Write this process's entry files and publish the version
        (multi-process: `distributed.commit_version`)."""
        from .distributed import commit_version
        t0 = time.perf_counter()
        local = [e for e in entries if e.rank in self.ranks]

        def abort_check():
            if self._abort_persist.is_set():
                raise PersistAborted(f"persist of v{buf.version} aborted by a fault")

        commit_version(self.store, buf.version, buf.iteration, buf.checkpoint_index, entries,
                       self.ranks, self.payloads(buf, local), group=self.group,
                       before_publish=abort_check, crcs=self.device_crcs(buf))
        return time.perf_counter() - t0

    def start_persist(self, buf: Buffer, entries: List[StoreEntry]) -> Future:
        fut = self._persist_pool.submit(self._write, buf, list(entries))
        self._persist[buf.buffer_id] = (fut, list(entries))
        return fut

    def persist_ready(self, buf: Buffer) -> bool:
        job = self._persist.get(buf.buffer_id)
        return job is None or job[0].done()

    def finish_persist(self, buf: Buffer) -> Optional[Buffer]:
        fut, _ = self._persist.pop(buf.buffer_id)
        self.stats["persist_s"].append(fut.result())
        return self.buffers.complete_persist(buf)

    def complete_persist(self, buf: Buffer, entries: List[StoreEntry]) -> Optional[Buffer]:
        """Synchronous persist (reference signature, engine.py:195-198)."""
        if buf.buffer_id in self._persist:
            return self.finish_persist(buf)
        if not self.has_bytes(buf):
            return super().complete_persist(buf, entries)  # metadata-only buffer
        self.stats["persist_s"].append(self._write(buf, entries))
        return self.buffers.complete_persist(buf)

    def on_fault(self, failed_nodes: Iterable[int]) -> None:
        """Reference semantics (engine.py:200-212) with real work in flight:
        the in-flight pack/drain is allowed to land (its buffer is then
        cleared, so nothing can reuse it while the copy engine still writes
        it), and an in-flight persist is aborted before it publishes — a
        torn version has no COMPLETE marker and is ignored by readers."""
        self.pack_stream.synchronize()
        self.copy_stream.synchronize()
        if self._pending_bid is not None:
            # a device-planned snapshot whose drain never started: it is
            # discarded with its SNAPSHOTTING buffer below
            self._inflight.pop(self._pending_bid, None)
            self._pending_bid = None
        self._abort_persist.set()
        published = []
        for bid, (fut, _) in self._persist.items():
            try:
                self.stats["persist_s"].append(fut.result())
                published.append(bid)   # it won the race: the version is COMPLETE
            except PersistAborted:
                pass
        self._persist.clear()
        self._abort_persist.clear()
        for bid in published:
            self.buffers.complete_persist(self.buffers.buffers[bid])
        super().on_fault(failed_nodes)

    def close(self) -> None:
        self._persist_pool.shutdown(wait=True)
        for bid, shb in list(self._shared.items()):
            self._retract_meta(bid)
            self.host[bid] = None
            shb.close()
        self._shared.clear()


class _PersistSelections(dict):
    """version -> persist sets per layer.  Host-planned checkpoints store
    theirs at checkpoint time; device-planned (load-aware) ones resolve from
    the engine on first access."""

    def __init__(self, owner: "PecCheckpointer"):
        super().__init__()
        self._owner = owner

    def __missing__(self, version: int):
        eng = self._owner.engine
        buf = next((b for b in eng.buffers.buffers if b.version == version), None)
        due = eng.persist_due(buf) if buf is not None else None
        if due is None:
            raise KeyError(version)
        self[version] = due
        return due


class PecCheckpointer:
    """Training-loop driver of the PEC snapshot path (one per rank process).

    Mirrors the checkpoint parts of `Simulation` (simulator.py:309-457,
    546-576) with real bytes: ``step(iteration, router_ids)`` counts tokens and,
    every ``i_ckpt`` iterations, selects experts (on device), plans, and
    starts the snapshot; ``poll()`` moves completed drains/persists through
    the state machine.
    """

    def __init__(self, layout: RankLayout, arena: StateArena, store, pec: Optional[PecConfig],
                 strategy: str = EQUAL_PEC, i_ckpt: int = 10, ranks: Optional[Sequence[int]] = None,
                 counters=None, group=None, control_group=None, n_buffers: int = 3,
                 pack_mode: int = D.MODE_AUTO, chunk_log2: int = D.DEFAULT_CHUNK_LOG2,
                 async_persist: bool = True, shared_host_prefix: Optional[str] = None):
        self.layout = layout
        self.arena = arena
        self.pec = pec
        self.strategy = strategy
        self.i_ckpt = i_ckpt
        self.group = group
        self.engine = DeviceCheckpointEngine(layout, store, arena, ranks, n_buffers, pack_mode,
                                             chunk_log2, control_group,
                                             shared_host_prefix=shared_host_prefix)
        self.counters = counters
        self.async_persist = async_persist
        self.persist_sel: Dict[int, Dict[int, frozenset]] = _PersistSelections(self)
        self._plan: Optional[ShardPlan] = None
        # host time spent waiting at checkpoints: for the previous snapshot's
        # drain ("snap") and for a persist to free a buffer ("buffer": the
        # reference charges NoFreeBufferError as a stall, simulator.py:413-422)
        self.stall_s = 0.0
        self.waits = {"snap": [0, 0.0], "buffer": [0, 0.0]}
        self._persist_off = False
        # cumulative delivered tokens of the current timeline at every
        # checkpoint iteration (for the counter reset after a recovery)
        self._cum_at: Dict[int, object] = {}
        self._replay_offset = None
        self.device_plans = False
        if pec is not None and pec.selection == LOAD_AWARE:
            if strategy == ADAPTIVE_PEC:
                from .topology import SpecValidationError
                raise SpecValidationError("adaptive_pec requires sequential selection",
                                          "load-aware selection is not periodic")
            if counters is None:
                raise ValueError("load-aware selection needs DeviceTokenCounters")
            self.engine.enable_device_plans(strategy)
            self.device_plans = True

    # -- plans --------------------------------------------------------------------
    def plan(self) -> Optional[ShardPlan]:
        if self._plan is None and (self.pec is None or self.pec.selection != LOAD_AWARE):
            if self.pec is None:
                self._plan = plan_baseline(self.layout) if self.strategy == BASELINE \
                    else plan_equal(self.layout)
            else:
                seq = PecConfig(k_pec=self.pec.k_snapshot, k_snapshot=self.pec.k_snapshot,
                                k_persist=self.pec.k_persist)
                self._plan = plan_adaptive(self.layout, seq) if self.strategy == ADAPTIVE_PEC \
                    else plan_equal(self.layout, seq)
        return self._plan

    def prepare(self, host_buffers: Optional[int] = None) -> None:
        """Do the start-up work once, before training: allocate the HBM
        staging buffer and pin the host snapshot buffers (pinning runs at a
        few GB/s), and build every phase's device descriptor table of a
        periodic (sequential) plan, so no checkpoint plans or allocates."""
        self.engine.reserve(self.max_snapshot_bytes(), host_buffers=host_buffers)
        plan = self.plan()
        if plan is not None:
            for p in range(plan.period):
                self.engine.layouts_for(plan.assignments[p], ("phase", p))

    def max_snapshot_bytes(self) -> int:
        """Upper bound of this process's staging bytes over all phases."""
        plan = self.plan()
        ranks = self.engine.ranks
        if plan is not None:
            return max(sum((StagingLayout.build(ph.get(r, ()), self.arena, r).nbytes + 255)
                           // 256 * 256 for r in ranks) for ph in plan.assignments)
        # load-aware: the heaviest due set is every expert a rank holds
        full = {m: frozenset(range(self.layout.model.experts_per_layer))
                for m in range(self.layout.model.num_moe_layers)}
        ph = build_phase_assignment(self.layout, full, self.strategy)
        return sum((StagingLayout.build(ph.get(r, ()), self.arena, r).nbytes + 255) // 256 * 256
                   for r in ranks)

    def selections(self, c: int):
        """(snapshot sets, persist sets) per layer for checkpoint c
        (simulator.py:339-354)."""
        L, n = self.layout.model.num_moe_layers, self.layout.model.experts_per_layer
        if self.pec is None:
            full = frozenset(range(n))
            return {m: full for m in range(L)}, {m: full for m in range(L)}
        k_s, k_p = self.pec.k_snapshot, self.pec.k_persist
        if self.pec.selection == LOAD_AWARE:
            snap_d, pers_d = self.counters.select(k_s, k_p, group=self.group)
            snap_h, pers_h = snap_d.cpu().tolist(), pers_d.cpu().tolist()
            return ({m: frozenset(e for e in snap_h[m] if e >= 0) for m in range(L)},
                    {m: frozenset(e for e in pers_h[m] if e >= 0) for m in range(L)})
        return ({m: select_window(c, m, n, k_s, k_p) for m in range(L)},
                {m: select_window(c, m, n, k_p, k_p) for m in range(L)})

    # -- the loop ----------------------------------------------------------------
    def step(self, iteration: int, router_ids=None) -> Optional[Buffer]:
        if router_ids is not None and self.counters is not None:
            self.counters.add_iteration(router_ids)
        self.poll()
        if iteration % self.i_ckpt == 0:
            return self.checkpoint(iteration)
        return None

    def _timeline_delivered(self):
        import torch
        d = self.counters.delivered
        if self._replay_offset is None:
            self._replay_offset = torch.zeros_like(d)
        return d - self._replay_offset

    def checkpoint(self, iteration: int) -> Buffer:
        c = iteration // self.i_ckpt - 1
        if self.counters is not None:
            if len(self._cum_at) > 2 * len(self.engine.buffers.buffers) + 8:
                self._prune_history()
            self._cum_at[iteration] = self._timeline_delivered()
        if self.device_plans:
            return self._checkpoint_device(iteration, c)
        snap_sel, persist_sel = self.selections(c)
        plan = self.plan()
        if plan is not None:
            phase = plan.phase_of(c)
            assignment, key = plan.assignments[phase], ("phase", phase)
        else:
            assignment, key = build_phase_assignment(self.layout, snap_sel, self.strategy), None
        while True:
            try:
                # one snapshot at a time: wait for the previous drain
                snapping = self.engine.buffers.snapshotting
                if snapping is not None:
                    t0 = time.perf_counter()
                    self._complete(snapping)
                    self._waited("snap", time.perf_counter() - t0)
                buf = self.engine.begin_snapshot(iteration, c, assignment, plan_key=key)
                break
            except NoFreeBufferError:
                t0 = time.perf_counter()
                if not self._wait_one_persist():
                    raise
                self._waited("buffer", time.perf_counter() - t0)
        self.persist_sel[buf.version] = persist_sel
        return buf

    def _checkpoint_device(self, iteration: int, c: int) -> Buffer:
        """Load-aware checkpoint with selection and plan on the GPU."""
        while True:
            snapping = self.engine.buffers.snapshotting
            if snapping is not None:
                t0 = time.perf_counter()
                self._complete(snapping)
                self._waited("snap", time.perf_counter() - t0)
            if any(b.status == "free" for b in self.engine.buffers.buffers):
                break
            t0 = time.perf_counter()
            if not self._wait_one_persist():
                raise NoFreeBufferError("no free buffer and no persist in flight")
            self._waited("buffer", time.perf_counter() - t0)
        snap_d, pers_d = self.counters.select(self.pec.k_snapshot, self.pec.k_persist,
                                              group=self.group)
        return self.engine.begin_snapshot_device(iteration, c, snap_d, pers_d)

    def resolve(self, buf: Buffer) -> Buffer:
        """Make a device-planned snapshot's host-side view current (its
        `content` and persist sets; enqueues its drain if still pending).
        Host-planned buffers are always current."""
        self.engine.persist_due(buf)
        return buf

    def on_fault(self, failed_nodes) -> None:
        """Engine fault handling, then resume an interrupted persist
        (simulator.py:511-525)."""
        self.engine.on_fault(failed_nodes)
        if self.engine.buffers.persisting is None:
            nxt = self.engine.buffers.promote_if_idle()
            if nxt is not None:
                self._start_persist(nxt)

    def recover(self, failed_nodes, iteration: int, verify: str = "device") -> RecoveryOutcome:
        """Full fault handling with real bytes, in the reference's order
        (`Simulation._handle_fault`, simulator.py:473-544): resolve the
        newest source of every unit (capped at ``iteration``), unwind
        in-flight work (`on_fault`, resuming an interrupted persist from
        surviving memory), move the bytes back into the state arena
        (`restore`: memory / storage / initial), and reset both load-aware
        counter tiers to the tokens each expert received between its restored
        iteration and the restart point (simulator.py:527-532).  With no
        COMPLETE version the run restarts from scratch: every unit is
        re-initialised and the buffers are dropped (simulator.py:476-483).
        The caller resumes training at ``restart_iteration + 1``."""
        from .restore import restore
        failed = frozenset(failed_nodes)
        L, E = self.layout.model.num_moe_layers, self.layout.model.experts_per_layer
        store = self.engine.store
        # unwind in-flight work first: a persist that already published is
        # honoured, one that had not is discarded (no COMPLETE).  The
        # decisions below equal the reference's taken before on_fault: the
        # cleared SNAPSHOTTING buffer was no source, PERSISTING ->
        # SNAPSHOTTED stays one, failed nodes are excluded either way.
        self.engine.on_fault(failed)
        if store is None or store.newest_complete() is None:
            for b in self.engine.buffers.buffers:
                b.clear()
            for key in list(self.arena.slots):
                self.arena.fill_unit(key)
            plan = report = None
            restart, skew = 0, 0
            expert_restore = {(m, e): 0 for m in range(L) for e in range(E)}
        else:
            plan = self.engine.resolve_recovery(failed, max_iteration=iteration)
            if self.engine.buffers.persisting is None:   # resume a cut-off persist
                nxt = self.engine.buffers.promote_if_idle()
                if nxt is not None:
                    self._start_persist(nxt)
            report = restore(self.engine, plan, verify=verify)
            restart, skew = plan.restart_iteration, plan.version_skew
            expert_restore = {}
            for m in range(L):
                for e in range(E):
                    wd = plan.decisions.get(f"ew.L{m}.E{e}")
                    od = plan.decisions.get(f"eo.L{m}.E{e}")
                    expert_restore[(m, e)] = restart if wd is None or od is None else \
                        min(wd.restored_iteration, od.restored_iteration)
        if self.counters is not None:
            self._reset_counters(expert_restore, restart)
        return RecoveryOutcome(restart, skew, plan, report, expert_restore)

    def _prune_history(self) -> None:
        """Bound the per-checkpoint history: a counter reset after a fault
        needs the cumulative delivered tokens only at iterations some expert
        can be restored to — a buffer still holding a snapshot, or the newest
        stored version that holds the expert (resolve_recovery's choice,
        engine.py:231-284) — plus the latest.  Persist sets are needed only
        for buffers that have not been persisted yet."""
        bufs = [b for b in self.engine.buffers.buffers if b.version is not None]
        keep = {b.iteration for b in bufs}
        if self._cum_at:
            keep.add(max(self._cum_at))
        store = self.engine.store
        if store is not None:
            want = {f"{t}.L{m}.E{e}" for t in ("ew", "eo")
                    for m in range(self.layout.model.num_moe_layers)
                    for e in range(self.layout.model.experts_per_layer)}
            metas = self.__dict__.setdefault("_meta_cache", {})
            for v in sorted(store.complete_versions(), reverse=True):
                if not want:
                    break
                if v not in metas:
                    try:
                        meta = store.meta(v)
                    except (OSError, ValueError, KeyError):
                        continue        # removed by an external retention policy meanwhile
                    metas[v] = (meta.iteration, {e.unit_key for e in meta.entries.values()})
                it, units = metas[v]
                hit = want & units
                if hit:
                    keep.add(it)
                    want -= hit
        self._cum_at = {k: v for k, v in self._cum_at.items() if k in keep}
        live = {b.version for b in bufs}
        for v in [v for v in self.persist_sel if v not in live]:
            del self.persist_sel[v]

    def _reset_counters(self, expert_restore: Dict[Tuple[int, int], int], restart: int) -> None:
        """unsaved(m, e) = tokens delivered in (restored(m, e), restart], from
        the cumulative-delivered snapshots taken at checkpoints; the
        timeline then rewinds to the restart point (replayed iterations are
        counted again)."""
        import torch
        timeline = self._timeline_delivered()
        zero = torch.zeros_like(timeline)
        base = self._cum_at.get(restart, zero) if restart else zero
        unsaved = torch.zeros_like(timeline)
        restored = torch.tensor([[expert_restore[(m, e)] for e in range(timeline.shape[1])]
                                 for m in range(timeline.shape[0])], device=timeline.device)
        for r in sorted(set(expert_restore.values())):
            if r >= restart:
                continue
            at_r = self._cum_at.get(r, zero) if r else zero
            mask = restored == r
            unsaved[mask] = (base - at_r)[mask]
        # a checkpoint taken before the counters were attached has no
        # snapshot: never let a missing one turn into negative counts
        unsaved.clamp_(min=0)
        self.counters.reset_to(unsaved, unsaved)
        self._replay_offset = self.counters.delivered - base
        self._cum_at = {k: v for k, v in self._cum_at.items() if k <= restart}

    def _waited(self, kind: str, seconds: float) -> None:
        self.stall_s += seconds
        self.waits[kind][0] += 1
        self.waits[kind][1] += seconds

    def set_persist(self, enabled: bool) -> None:
        """Switch the persist tier off (snapshot tier only: completed
        snapshots become the in-memory recovery copy and buffers recycle
        without writes) or back on (later snapshots persist again)."""
        self._persist_off = not enabled

    def wait_pack(self, stream=None) -> None:
        self.engine.wait_pack(stream=stream)

    def wait_snapshot(self, buf: Buffer) -> None:
        """Block until ``buf``'s drain landed (SNAPSHOTTED) and start its
        persist when it is next in line."""
        self._complete(buf)

    def _complete(self, buf: Buffer) -> None:
        promoted = self.engine.complete_snapshot(buf)
        if promoted is not None:
            self._start_persist(promoted)

    def hold_persist(self, hold: bool = True) -> None:
        """Pause (hold=True) or resume the persist tier.  While held,
        snapshots still complete (SNAPSHOTTED) and queue for persist; on
        resume the oldest queued one starts."""
        self._persist_held = hold
        if not hold:
            p = self.engine.buffers.persisting
            if p is not None and p.buffer_id not in self.engine._persist:
                self._start_persist(p)

    def _start_persist(self, buf: Buffer) -> None:
        if getattr(self, "_persist_held", False) and self.engine.store is not None:
            return  # stays PERSISTING (queued) until hold_persist(False)
        if self.engine.store is None or self._persist_off:
            # snapshot tier only (no persist tier configured, or switched
            # off): the buffer is published to the in-memory recovery role
            # without any writes
            nxt = self.engine.buffers.complete_persist(buf)
            if nxt is not None:
                self._start_persist(nxt)
            return
        entries = self.engine.persist_entries(buf, self.persist_sel[buf.version])
        if self.async_persist:
            self.engine.start_persist(buf, entries)
        else:
            nxt = self.engine.complete_persist(buf, entries)
            if nxt is not None:
                self._start_persist(nxt)

    def _wait_one_persist(self) -> bool:
        p = self.engine.buffers.persisting
        if p is None:
            return False
        if p.buffer_id not in self.engine._persist:
            # queued behind hold_persist: the caller needs the buffer now
            self._persist_held = False
            self._start_persist(p)
            return True
        nxt = self.engine.finish_persist(p)
        if nxt is not None:
            self._start_persist(nxt)
        return True

    def poll(self) -> None:
        self.engine.finalize_pending(block=False)
        snapping = self.engine.buffers.snapshotting
        if snapping is not None and self.engine.snapshot_ready(snapping):
            self._complete(snapping)
        p = self.engine.buffers.persisting
        while p is not None and self.engine.persist_ready(p) and p.buffer_id in self.engine._persist:
            nxt = self.engine.finish_persist(p)
            if nxt is not None:
                self._start_persist(nxt)
            p = self.engine.buffers.persisting

    def finish(self) -> None:
        """Drain all in-flight snapshot and persist work."""
        if getattr(self, "_persist_held", False):
            self.hold_persist(False)
        snapping = self.engine.buffers.snapshotting
        if snapping is not None:
            self._complete(snapping)
        while self.engine.buffers.persisting is not None:
            if not self._wait_one_persist():
                break

    def close(self) -> None:
        self.finish()
        self.engine.close()
