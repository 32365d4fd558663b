"""Staging layout: where each planned byte range lands in the snapshot buffer.

A rank's snapshot is its ordered `RangeAssignment` list for the phase
(reference `planner.py:263-295`).  The pack kernel gathers those ranges, in
that order, into one contiguous device staging buffer, which the copy engine
then drains into a pinned host buffer with the *same* layout; the persist
thread writes each entry file straight out of the host buffer.

Entry i starts at the first offset >= the end of entry i-1 that is congruent
to its source address modulo 256 (``STAGE_ALIGN``).  Unit images are
256-byte aligned in the arena (`arena.py`), so source and destination of
every copy share their alignment: the kernel streams aligned 16-byte vectors
(or TMA bulk copies) from the first full granule to the last, with only
sub-16-byte heads/tails at byte-granular range boundaries (the floor-split
expert weight parts, planner.py:188-195).  Padding is at most 255 B per
entry; entry files carry exact bytes.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Iterable, List, Optional, Sequence, Tuple

import numpy as np

from .device import DEFAULT_CHUNK_LOG2, DESC_DTYPE, TEMPLATE_DTYPE, plan_chunks
from .planner import RangeAssignment

STAGE_ALIGN = 256


@dataclass(frozen=True)
class StagedEntry:
    store_key: str
    unit_key: str
    start: int          # byte range [start, stop) of the unit image
    stop: int
    part: Optional[int]
    rank: int
    src_offset: int     # arena offset of byte `start`
    stage_offset: int   # staging offset of byte `start`

    @property
    def nbytes(self) -> int:
        return self.stop - self.start


class StagingLayout:
    """Placement of one rank's ranges in the staging / host snapshot buffer."""

    def __init__(self, entries: Sequence[StagedEntry], nbytes: int):
        self.entries: Tuple[StagedEntry, ...] = tuple(entries)
        self.nbytes = nbytes
        self.payload_bytes = sum(e.nbytes for e in self.entries)
        self._by_store_key = {e.store_key: e for e in self.entries}

    @classmethod
    def build(cls, ranges: Iterable[RangeAssignment], arena, rank: int = 0,
              align: int = STAGE_ALIGN) -> "StagingLayout":
        out: List[StagedEntry] = []
        pos = 0
        for a in ranges:
            if a.stop <= a.start:
                continue
            src = arena.slot(a.key).offset + a.start
            off = pos + ((src - pos) % align)
            out.append(StagedEntry(a.store_key, a.key, a.start, a.stop, a.part, rank, src, off))
            pos = off + (a.stop - a.start)
        return cls(out, pos)

    def entry(self, store_key: str) -> StagedEntry:
        return self._by_store_key[store_key]

    def __len__(self) -> int:
        return len(self.entries)

    # -- descriptor tables ------------------------------------------------------
    def descriptors(self, state_base: int, stage_base: int, reverse: bool = False,
                    chunk_log2: int = DEFAULT_CHUNK_LOG2,
                    select: Optional[Iterable[str]] = None) -> Tuple[np.ndarray, int]:
        """Host `pec_copy_desc` table (pack: state -> stage; reverse:
        stage -> state) and its total chunk count.  ``select`` limits the
        table to the given store keys (partial restores)."""
        keys = None if select is None else set(select)
        ents = [e for e in self.entries if keys is None or e.store_key in keys]
        table = np.zeros(len(ents), dtype=DESC_DTYPE)
        for i, e in enumerate(ents):
            s = state_base + e.src_offset
            t = stage_base + e.stage_offset
            table[i]["src"], table[i]["dst"] = (t, s) if reverse else (s, t)
            table[i]["nbytes"] = e.nbytes
        total = plan_chunks(table, chunk_log2)
        return table, total


def drain_cuts(nbytes: int, first: int = 64 << 20, growth: int = 4) -> List[int]:
    """Staging offsets at which a snapshot's pack is split so its drain can
    start early: 64 MiB, 256 MiB, 1 GiB, 4 GiB, ... below ``nbytes``.  The
    first drain piece starts after ~20 us of pack instead of the whole pack;
    every later piece is packed long before the host link reaches it."""
    cuts, c = [], first
    while c < nbytes:
        cuts.append(c)
        c *= growth
    return cuts


def split_table(table: np.ndarray, staging_base: int, cuts: Sequence[int],
                chunk_log2: int = DEFAULT_CHUNK_LOG2, with_rows: bool = False
                ) -> List[Tuple[np.ndarray, int, int, Optional[int]]]:
    """Split a pack descriptor table at staging byte offsets ``cuts``:
    returns [(sub_table, total_chunks, lo, hi)] where sub_table copies exactly the bytes the
    original copies into staging [lo, hi) (rows crossing a cut are split into
    two copies; first_chunk re-planned per sub-table).  The segments' ranges
    tile [0, last cut or end) with the final one open-ended (hi = None).
    ``with_rows`` appends, per segment, the original row index of every
    sub-row (a split row's pieces are consecutive bytes of it, in segment
    order: per-piece CRCs combine into the row's CRC)."""
    r0 = table["dst"].astype(np.int64) - staging_base
    r1 = r0 + table["nbytes"].astype(np.int64)
    bounds = [0, *cuts, None]
    out = []
    for lo, hi in zip(bounds[:-1], bounds[1:]):
        a = np.maximum(r0, lo)
        b = r1 if hi is None else np.minimum(r1, hi)
        keep = b > a
        sub = np.zeros(int(keep.sum()), dtype=DESC_DTYPE)
        shift = (a - r0)[keep].astype(np.uint64)
        sub["src"] = table["src"][keep] + shift
        sub["dst"] = table["dst"][keep] + shift
        sub["nbytes"] = (b - a)[keep].astype(np.uint64)
        seg = (sub, plan_chunks(sub, chunk_log2), lo, hi)
        out.append(seg + (np.flatnonzero(keep),) if with_rows else seg)
    return out


class DeviceTable:
    """A descriptor table resident in device memory, ready for pec_pack."""

    def __init__(self, table: np.ndarray, total_chunks: int, device,
                 chunk_log2: int = DEFAULT_CHUNK_LOG2):
        import torch
        self.n = len(table)
        self.total_chunks = total_chunks
        self.chunk_log2 = chunk_log2
        raw = torch.from_numpy(table.view(np.uint8).copy()) if self.n else \
            torch.zeros(DESC_DTYPE.itemsize, dtype=torch.uint8)
        self.tensor = raw.view(torch.int64).to(device)
        self.nbytes_moved = int(table["nbytes"].sum()) if self.n else 0


class PlanTemplate:
    """A rank's entry list with every expert due, in planner order, for the
    device-side plan expansion (`pec_expand_plan`).

    For strategies whose non-expert placement does not depend on the due set
    (equal_*, baseline), the rank's entries for ANY due set are exactly the
    template entries whose (layer, expert) is due, in template order
    (`_expert_entries` iterates due layers/experts in sorted order,
    planner.py:213-240), plus every owned / non-expert entry."""

    def __init__(self, layout, arena, rank: int, strategy: str, device):
        import torch
        from .planner import ADAPTIVE_PEC, build_phase_assignment, full_due_map
        if strategy == ADAPTIVE_PEC:
            raise ValueError("adaptive placement depends on the due set; no device template")
        self.rank = rank
        self.strategy = strategy
        self.layout = layout
        self.ranges = tuple(a for a in build_phase_assignment(layout, full_due_map(layout),
                                                              strategy).get(rank, ())
                            if a.stop > a.start)  # empty ranges carry no bytes
        table = np.zeros(len(self.ranges), dtype=TEMPLATE_DTYPE)
        for i, a in enumerate(self.ranges):
            u = layout.by_key[a.key]
            table[i]["src_offset"] = arena.slot(a.key).offset + a.start
            table[i]["nbytes"] = a.stop - a.start
            table[i]["layer"] = -1 if u.layer is None else u.layer
            table[i]["expert"] = -1 if u.expert is None else u.expert
        self.table = table
        self.n = len(table)
        self.max_bytes = StagingLayout.build(self.ranges, arena, rank).nbytes
        # the leading non-expert rows are kept for every due set, so their
        # staged bytes [0, fixed_prefix) are known before the device plan is
        # (the drain can start on them at once)
        lead = 0
        while lead < self.n and table[lead]["layer"] < 0:
            lead += 1
        self.fixed_prefix = StagingLayout.build(self.ranges[:lead], arena, rank).nbytes \
            if lead else 0
        self.tensor = torch.from_numpy(table.view(np.uint8).copy()).view(torch.int64).to(device) \
            if self.n else torch.zeros(4, dtype=torch.int64, device=device)

    def max_chunks(self, chunk_log2: int = DEFAULT_CHUNK_LOG2) -> int:
        span = 1 << chunk_log2
        return int(sum((int(n) + span - 1) // span for n in self.table["nbytes"]))

    def select(self, due) -> tuple:
        """The rank's RangeAssignments for a due map (host mirror of the
        device filter)."""
        return tuple(a for a, t in zip(self.ranges, self.table)  # noqa: E501
                     if t["layer"] < 0 or int(t["expert"]) in due.get(int(t["layer"]), ()))
