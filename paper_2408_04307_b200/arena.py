"""HBM layout of a rank's checkpointable state: the unit -> byte-image map.

The reference leaves unit contents abstract ("No tensor contents",
`SPEC.md:89`); a unit is only a key and a size (`topology.py:173-189`).  On
B200 the bytes are real, so this module fixes the `UnitMap` of SURVEY.md §7:

* ``ew.L<l>.E<e>``  the expert's weight tensors flattened in declaration
  order (GPT: w1, b1, w2, b2; Mixtral: w1, w2, w3), ``epp * B_w`` bytes;
* ``eo.L<l>.E<e>``  fp32 optimizer planes ``[master | exp_avg | exp_avg_sq]``
  (B_o = 12; B_o = 8 drops the master copy), ``epp * B_o`` bytes;
* ``new.<module>``   the module's weights, ``count * B_w`` bytes;
* ``neo.r<r>``       rank r's ZeRO-2 flat optimizer partition,
  ``unit_sizes()[NON_EXPERT_OPTIM][r]`` bytes;
* ``other.r<r>``     an opaque per-rank blob.

Every unit resident on a rank lives contiguously, 256-byte aligned, inside one
device allocation (the arena).  A training step sees typed views into it (the
optimizer's master/m/v planes are views of the eo image), so the pack kernel
reads each range with one contiguous, aligned stream and the arena can hold
~85 GB of Mixtral-shaped per-rank state in one HBM block.

Initial contents are seeded per unit — ``torch.Generator`` seed
``base_seed ^ crc32c(key)`` — so the "initial" recovery
source of `engine.resolve_recovery` can be regenerated bit-identically.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, Iterable, Optional, Sequence, Tuple

from .topology import EXPERT_OPTIM, EXPERT_WEIGHT, NON_EXPERT_WEIGHT, RankLayout

ARENA_ALIGN = 256
BASE_SEED = 7  # default make_scenario seed (reference tests/test_simulator.py:26)


def _align(x: int, a: int = ARENA_ALIGN) -> int:
    return (x + a - 1) // a * a


@dataclass(frozen=True)
class UnitSlot:
    key: str
    kind: str
    offset: int   # byte offset of the unit image inside the arena
    size: int


def _crc(key: str) -> int:
    from .device import crc32c
    return crc32c(key.encode())


def arena_slots(layout: RankLayout, ranks: Sequence[int]) -> Dict[str, UnitSlot]:
    """Deterministic arena placement of the units resident on ``ranks``
    (unit order of the layout, 256-byte aligned, empty units skipped).  Any
    process can recompute a peer rank's offsets from the layout alone."""
    rs = set(int(r) for r in ranks)
    slots: Dict[str, UnitSlot] = {}
    off = 0
    for u in layout.units:
        if u.size_bytes <= 0 or not (u.replica_ranks & rs):
            continue
        slots[u.key] = UnitSlot(u.key, u.kind, off, u.size_bytes)
        off = _align(off + u.size_bytes)
    return slots


class PeerSlots:
    """`slot()` lookup of a peer rank's arena (no allocation)."""

    def __init__(self, layout: RankLayout, rank: int):
        self.slots = arena_slots(layout, [rank])

    def slot(self, key: str) -> UnitSlot:
        return self.slots[key]


class StateArena:
    """Device-resident images of the units a set of ranks holds.

    ``ranks`` is normally one rank (one process per GPU); tests pass several
    to emulate a multi-rank deployment on one device.
    """

    def __init__(self, layout: RankLayout, ranks: Sequence[int], device=None,
                 expert_tensors: Sequence[Tuple[str, int]] = (), fill: bool = True,
                 base_seed: int = BASE_SEED):
        import torch
        self.layout = layout
        self.ranks = tuple(sorted(set(int(r) for r in ranks)))
        self.device = torch.device(device) if device is not None else torch.device("cuda")
        self.base_seed = base_seed
        epp = layout.model.expert_params_per_expert
        self.expert_tensors: Tuple[Tuple[str, int], ...] = tuple(expert_tensors) or (("w", epp),)
        if epp and sum(c for _, c in self.expert_tensors) != epp:
            raise ValueError("expert_tensors must sum to expert_params_per_expert")
        self.slots: Dict[str, UnitSlot] = arena_slots(layout, self.ranks)
        end = max((s.offset + s.size for s in self.slots.values()), default=0)
        self.nbytes = max(_align(end), ARENA_ALIGN)
        self.buffer = torch.empty(self.nbytes, dtype=torch.uint8, device=self.device)
        if fill:
            self.fill_all()

    # -- addressing -----------------------------------------------------------
    @property
    def base_address(self) -> int:
        return self.buffer.data_ptr()

    def has(self, key: str) -> bool:
        return key in self.slots

    def slot(self, key: str) -> UnitSlot:
        try:
            return self.slots[key]
        except KeyError:
            raise KeyError(f"unit {key!r} is not resident on ranks {self.ranks}") from None

    def unit_bytes(self, key: str):
        s = self.slot(key)
        return self.buffer[s.offset:s.offset + s.size]

    def resident_bytes(self) -> int:
        return sum(s.size for s in self.slots.values())

    # -- typed views (what a training step would bind its tensors to) ---------
    def _float_dtype(self, nbytes: int):
        import torch
        return {4: torch.float32, 2: torch.bfloat16, 1: torch.uint8}.get(nbytes)

    def views(self, key: str) -> Dict[str, "object"]:
        """Named typed views into a unit image."""
        import torch
        s = self.slot(key)
        raw = self.buffer[s.offset:s.offset + s.size]
        model = self.layout.model
        if s.kind == EXPERT_WEIGHT:
            dt = self._float_dtype(model.bytes_weight)
            out, pos = {}, 0
            for name, count in self.expert_tensors:
                nb = count * model.bytes_weight
                out[name] = raw[pos:pos + nb].view(dt) if dt is not None else raw[pos:pos + nb]
                pos += nb
            return out
        if s.kind == EXPERT_OPTIM:
            planes = model.bytes_optim // 4 if model.bytes_optim % 4 == 0 else 0
            names = ("master", "exp_avg", "exp_avg_sq")[-planes:] if 0 < planes <= 3 else ()
            if not names:
                return {"raw": raw}
            epp = model.expert_params_per_expert
            return {n: raw[i * epp * 4:(i + 1) * epp * 4].view(torch.float32)
                    for i, n in enumerate(names)}
        if s.kind == NON_EXPERT_WEIGHT:
            dt = self._float_dtype(model.bytes_weight)
            return {"weight": raw.view(dt) if dt is not None else raw}
        return {"raw": raw}

    # -- seeded contents ------------------------------------------------------
    def unit_seed(self, key: str) -> int:
        return (self.base_seed ^ _crc(key)) & 0x7FFFFFFFFFFFFFFF

    def fill_unit(self, key: str) -> None:
        """(Re)generate the unit's initial image on device, deterministically."""
        import torch
        g = torch.Generator(device=self.device)
        g.manual_seed(self.unit_seed(key))
        s = self.slot(key)
        raw = self.buffer[s.offset:s.offset + s.size]
        for name, view in self.views(key).items():
            if view.dtype == torch.uint8:
                # opaque bytes (ZeRO flat partitions, blobs): fp32-like values
                # over the 4-byte-aligned body, random bytes in the tail
                body = view.numel() // 4 * 4
                if body:
                    view[:body].view(torch.float32).normal_(0.0, 1e-2, generator=g)
                if view.numel() > body:
                    tail = torch.randint(0, 256, (view.numel() - body,), generator=g,
                                         device=self.device, dtype=torch.int32)
                    view[body:].copy_(tail.to(torch.uint8))
            elif name == "exp_avg":
                view.normal_(0.0, 1e-3, generator=g)
            elif name == "exp_avg_sq":
                view.normal_(0.0, 1e-6, generator=g).abs_()
            else:
                view.normal_(0.0, 0.02, generator=g)
        del raw

    def fill_all(self, keys: Optional[Iterable[str]] = None) -> None:
        for key in (list(keys) if keys is not None else list(self.slots)):
            self.fill_unit(key)
