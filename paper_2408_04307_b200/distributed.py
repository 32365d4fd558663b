"""Cross-rank protocol of the PEC path (one process per GPU).

The payload never crosses GPUs; only two small exchanges exist
(SURVEY.md §8(e)):

* `global_two_tier_select` — load-aware selection on the *global* unsaved
  token counts.  One sum all-reduce of a copy of the local ``[2, L, E]``
  int64 counters (NCCL over NVLink on GPU tensors), the same selection on
  every rank, then the selected entries are zeroed in each rank's *local*
  counters, which zeroes them in the global sum (counts are linear), so the
  invariant global == sum(local) holds without a second collective.
* `commit_version` — the multi-writer form of `DiskStore.write_version`
  (store.py:202-228): each rank writes its own entry files, the manifest
  rows are gathered, rank 0 publishes meta.json / manifest.tsv / COMPLETE
  (byte-identical to a single writer), and a barrier makes the version
  visible to all ranks before anyone proceeds.
"""

from __future__ import annotations

from typing import Callable, Iterable, List, Mapping, Optional, Sequence

from .store import StoreEntry


def _world(group) -> int:
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return 1
    return dist.get_world_size(group)


def global_two_tier_select(local_counts, k_snapshot: int, k_persist: int,
                           select_fn: Callable, group=None):
    """local_counts: [2, L, E] int64 tensor (tier 0 = snapshot, 1 = persist).
    select_fn(counts_2d, k, pool) -> [L, k] int32 ids (ascending per row)
    selecting top-k by (count desc, id asc).  Returns (snap, persist) and
    resets the selected entries of ``local_counts`` in place."""
    import torch.distributed as dist
    glob = local_counts.clone()
    if _world(group) > 1:
        dist.all_reduce(glob, op=dist.ReduceOp.SUM, group=group)
    snap = select_fn(glob[0], k_snapshot, None)
    pers = select_fn(glob[1], k_persist, snap)
    local_counts[0].scatter_(1, snap.long().clamp_min(0), 0)
    local_counts[1].scatter_(1, pers.long().clamp_min(0), 0)
    return snap, pers


def commit_version(store, version: int, iteration: int, checkpoint_index: int,
                   entries: Sequence[StoreEntry], local_ranks: Iterable[int],
                   payloads: Optional[Mapping[str, object]], group=None,
                   before_publish: Optional[Callable[[], None]] = None,
                   crcs: Optional[Mapping[str, int]] = None) -> None:
    """Write this process's entries, then publish the version once.
    ``before_publish`` may raise to abandon the version (no COMPLETE);
    ``crcs`` are precomputed entry CRCs (e.g. from pec_pack_crc)."""
    import torch.distributed as dist
    local = set(local_ranks)
    mine = [e for e in entries if e.rank in local]
    world = _world(group)
    if world == 1:
        store.check_version(version)
        rows = store.write_entries(version, iteration, mine, payloads=payloads, crcs=crcs)
        if before_publish is not None:
            before_publish()
        store.publish(version, iteration, checkpoint_index, entries, rows)
        return
    rows = store.write_entries(version, iteration, mine, payloads=payloads, crcs=crcs)
    gathered: List[Optional[list]] = [None] * world
    dist.all_gather_object(gathered, rows, group=group)
    err = None
    if dist.get_rank(group) == 0:
        try:
            if before_publish is not None:
                before_publish()
            store.publish(version, iteration, checkpoint_index, entries,
                          [r for part in gathered for r in part])
        except Exception as e:  # noqa: BLE001 - re-raised after the barrier
            err = e
    dist.barrier(group=group)  # every rank leaves, published or not
    if err is not None:
        raise err
