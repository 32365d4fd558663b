"""Device-resident per-expert token counters (both checkpoint tiers).

Device twin of the reference's two `LoadCounters` tiers and the ledger's
`delivered_total` (selector.py:69-88, simulator.py:99-125), fed by
`pec_token_hist` once per iteration (simulator.py:560-567) and consumed by
`pec_select_load_aware` at checkpoint time (simulator.py:339-354, 425-432).

Multi-GPU: every rank histograms its own tokens into local counters.  Counts
are linear, so at a checkpoint one NCCL all-reduce (sum, int64) of the
``[2, L, E]`` counters gives the global unsaved-token counts; every rank then
selects the same experts, and zeroing the selected entries in each rank's
*local* counters zeroes them in the global sum, so the invariant
"global = sum of locals" holds across checkpoints without a second
collective.
"""

from __future__ import annotations

import math
from typing import Optional, Sequence, Tuple

from . import device as D
from .selector import LoadCounters

SNAPSHOT_TIER, PERSIST_TIER = 0, 1


class DeviceTokenCounters:
    def __init__(self, n_layers: int, n_experts: int, device,
                 capacity: Optional[Sequence[int]] = None):
        import torch
        self.n_layers, self.n_experts = n_layers, n_experts
        self.device = torch.device(device)
        self.counts = torch.zeros((2, n_layers, n_experts), dtype=torch.int64, device=self.device)
        self.delivered = torch.zeros((n_layers, n_experts), dtype=torch.int64, device=self.device)
        self._scratch = torch.zeros(n_layers * n_experts + 1, dtype=torch.int32, device=self.device)
        self.cap = None
        if capacity is not None:
            self.cap = torch.tensor(list(capacity), dtype=torch.int64, device=self.device)

    @staticmethod
    def capacity_for(capacity_factor: Optional[float], routed_per_layer: Sequence[int],
                     n_experts: int):
        """ceil(cf * total / N) per layer (simulator.py:92-94)."""
        if capacity_factor is None:
            return None
        return [math.ceil(capacity_factor * t / n_experts) for t in routed_per_layer]

    def add_iteration(self, router_ids, stream=None) -> None:
        """Count one iteration's router top-k ids [L, tokens*top_k] (int32,
        on device) into both tiers and the delivered totals."""
        D.token_hist(router_ids, self.counts, self._scratch, cap=self.cap,
                     delivered=self.delivered, stream=stream)

    def all_reduced(self, group=None):
        """Global counters: a sum all-reduce of a copy of the local ones."""
        import torch.distributed as dist
        g = self.counts.clone()
        if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
            dist.all_reduce(g, op=dist.ReduceOp.SUM, group=group)
        return g

    def select(self, k_snapshot: int, k_persist: int, group=None, stream=None
               ) -> Tuple["object", "object"]:
        """Two-tier load-aware selection on device: snapshot set from the
        snapshot tier, persist set restricted to it from the persist tier,
        both tiers' selected counters reset.  With a process group the
        selection runs on the all-reduced global counts
        (`distributed.global_two_tier_select`).  Returns device int32
        [L, k_s] / [L, k_p] (ids ascending per layer)."""
        import torch
        from .distributed import _world, global_two_tier_select
        L = self.n_layers

        def kernel(counts2d, k, pool, zero=False):
            out = torch.empty((L, k), dtype=torch.int32, device=self.device)
            D.select_load_aware(counts2d, k, out, pool=pool, zero_selected=zero, stream=stream)
            return out

        if _world(group) > 1:
            return global_two_tier_select(self.counts, k_snapshot, k_persist, kernel, group)
        snap = kernel(self.counts[SNAPSHOT_TIER], k_snapshot, None, zero=True)
        pers = kernel(self.counts[PERSIST_TIER], k_persist, snap, zero=True)
        return snap, pers

    def reset_to(self, snapshot_tier, persist_tier) -> None:
        """Overwrite the counters (after a fault the reference resets them to
        the tokens delivered since each expert's restore, simulator.py:529-532)."""
        import torch
        self.counts[SNAPSHOT_TIER].copy_(torch.as_tensor(snapshot_tier, dtype=torch.int64))
        self.counts[PERSIST_TIER].copy_(torch.as_tensor(persist_tier, dtype=torch.int64))

    def as_load_counters(self, tier: int = SNAPSHOT_TIER) -> LoadCounters:
        """Host `LoadCounters` view (reference API) of one tier."""
        rows = self.counts[tier].cpu().tolist()
        lc = LoadCounters(self.n_layers, self.n_experts)
        for m, row in enumerate(rows):
            for e, v in enumerate(row):
                lc.unsaved_tokens[(m, e)] = int(v)
        return lc
