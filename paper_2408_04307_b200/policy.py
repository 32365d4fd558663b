"""Checkpoint-policy configuration fed by *measured* B200 bandwidths.

SURVEY.md §8(f) row 4: the reference picks K_snapshot / K_persist / I_ckpt
from modelled bandwidths (`adaptive_configure`, simulator.py:672-740) and
compares full vs. partial checkpointing with a closed form
(`analytic_overhead`, simulator.py:635-661).  Both are restated here on a
layout + cluster (no Scenario object, which is out of scope), so the same
decisions can be taken from what the engine actually measured:

* `measured_cluster` turns `DeviceCheckpointEngine.stats` into a
  `ClusterSpec` whose ``snapshot_bandwidth`` is the *pack* rate (on B200 the
  only training-blocking part of a snapshot is the HBM pack; the drain to
  host runs behind) and whose ``persist_bandwidth`` is the measured persist
  rate;
* `b200_configure` adds the one constraint staging introduces: a drain must
  finish before the next snapshot reuses the staging buffer, so I_ckpt also
  covers drain time / iteration time.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, replace
from typing import Optional

from .planner import (
    ADAPTIVE_PEC,
    EQUAL_PEC,
    PecConfig,
    ShardPlan,
    bottleneck_workload,
    pec_imbalance,
    plan_adaptive,
    plan_equal,
)
from .topology import ClusterSpec, RankLayout, SpecValidationError

US = 1_000_000


def _us(seconds: float) -> int:
    return math.ceil(seconds * US)


def transfer_us(nbytes: int, bandwidth: float) -> int:
    """simulator.py:57-61: bytes at bandwidth, rounded up to a microsecond."""
    return 0 if nbytes <= 0 else math.ceil(nbytes * US / bandwidth)


@dataclass(frozen=True)
class AnalyticOverhead:
    o_ckpt_full_us: float
    o_ckpt_moc_us: float
    moc_wins: bool


def analytic_overhead(*, o_save_full_us: float, i_ckpt_full: int, o_save_moc_us: float,
                      i_ckpt_moc: int, iter_time_us: float, failure_rate: float,
                      o_restart_us: float, i_total: int) -> AnalyticOverhead:
    """Expected fault-tolerance overhead of full vs. reduced checkpointing
    (paper Eq. 12-15; reference simulator.py:635-661)."""
    for name, val in (("i_ckpt_full", i_ckpt_full), ("i_ckpt_moc", i_ckpt_moc),
                      ("i_total", i_total), ("iter_time_us", iter_time_us)):
        if val <= 0:
            raise SpecValidationError(f"analytic.{name} > 0", f"got {val}")
    faults = failure_rate * i_total

    def overall(o_save, i_ckpt):
        return o_save * (i_total / i_ckpt) + faults * (o_restart_us + i_ckpt * iter_time_us / 2)

    per_moc = o_save_moc_us / i_ckpt_moc + failure_rate * i_ckpt_moc * iter_time_us / 2
    per_full = o_save_full_us / i_ckpt_full + failure_rate * i_ckpt_full * iter_time_us / 2
    return AnalyticOverhead(overall(o_save_full_us, i_ckpt_full),
                            overall(o_save_moc_us, i_ckpt_moc), per_moc < per_full)


@dataclass(frozen=True)
class AdaptiveConfig:
    pec: PecConfig
    i_ckpt: int
    snapshot_overlapped: bool
    persist_target_met: bool


def adaptive_configure_layout(layout: RankLayout, strategy: str, cluster: ClusterSpec,
                              persist_target_s: Optional[float] = None) -> AdaptiveConfig:
    """The reference's configurator (simulator.py:672-740) on a layout:
    the largest K_snapshot whose bottleneck snapshot hides under F&B (raised
    to the largest K with the same bottleneck when ranks would idle), the
    persist K inside ``persist_target_s`` (1 without a target), and the
    I_ckpt floor set by the persist duration."""
    fb_us = _us(cluster.fb_time)
    iter_us = fb_us + _us(cluster.update_time)
    n = layout.model.experts_per_layer
    strat = EQUAL_PEC if strategy == EQUAL_PEC else ADAPTIVE_PEC
    cache = {}

    def worst(k: int) -> int:
        if k not in cache:
            pec = PecConfig(k_pec=k, selection="sequential", k_snapshot=k, k_persist=k)
            plan: ShardPlan = plan_equal(layout, pec) if strat == EQUAL_PEC \
                else plan_adaptive(layout, pec)
            cache[k] = max(bottleneck_workload(plan, p)[1] for p in range(plan.period))
        return cache[k]

    k_snap, overlapped = 1, False
    for k in range(n, 0, -1):
        if transfer_us(worst(k), cluster.snapshot_bandwidth) <= fb_us:
            k_snap, overlapped = k, True
            break
    if overlapped and pec_imbalance(layout.model, layout.parallel, k_snap):
        same = worst(k_snap)
        k_snap = next((k for k in range(n, k_snap, -1) if worst(k) == same), k_snap)

    def persist_us(k: int) -> int:
        return transfer_us(worst(k), cluster.persist_bandwidth)

    met = True
    k_persist = 1
    if persist_target_s is not None:
        target = _us(persist_target_s)
        fits = [k for k in range(1, k_snap + 1) if persist_us(k) <= target]
        if fits:
            k_persist = max(fits)
        else:
            met = False
    i_ckpt = max(1, math.ceil(persist_us(k_persist) / iter_us))
    pec = PecConfig(k_pec=k_snap, selection="sequential", k_snapshot=k_snap,
                    k_persist=min(k_persist, k_snap))
    return AdaptiveConfig(pec, i_ckpt, overlapped, met)


def measured_cluster(cluster: ClusterSpec, stats: dict) -> ClusterSpec:
    """``cluster`` with the bandwidths a DeviceCheckpointEngine measured:
    snapshot = staged payload / pack time (HBM), persist = persisted payload
    / persist wall time.  Missing measurements keep the given values."""
    snap_bytes, pack_ms = stats.get("snap_bytes", []), stats.get("pack_ms", [])
    persist_s = stats.get("persist_s", [])
    upd = {}
    n = min(len(snap_bytes), len(pack_ms))
    if n and sum(pack_ms[-n:]) > 0:
        upd["snapshot_bandwidth"] = sum(snap_bytes[-n:]) / (sum(pack_ms[-n:]) / 1e3)
    m = min(len(snap_bytes), len(persist_s))
    if m and sum(persist_s[-m:]) > 0:
        upd["persist_bandwidth"] = sum(snap_bytes[-m:]) / sum(persist_s[-m:])
    return replace(cluster, **upd)


def drain_bandwidth(stats: dict) -> Optional[float]:
    n = min(len(stats.get("snap_bytes", [])), len(stats.get("drain_ms", [])))
    if not n or sum(stats["drain_ms"][-n:]) <= 0:
        return None
    return sum(stats["snap_bytes"][-n:]) / (sum(stats["drain_ms"][-n:]) / 1e3)


def b200_configure(layout: RankLayout, strategy: str, cluster: ClusterSpec,
                   drain_bw: float, persist_target_s: Optional[float] = None) -> AdaptiveConfig:
    """`adaptive_configure_layout` on measured numbers, plus the staging
    constraint: the next snapshot may only start once the previous drain
    (bottleneck bytes / host-link bandwidth) has emptied the staging buffer."""
    cfg = adaptive_configure_layout(layout, strategy, cluster, persist_target_s)
    strat = EQUAL_PEC if strategy == EQUAL_PEC else ADAPTIVE_PEC
    pec = PecConfig(k_pec=cfg.pec.k_snapshot, k_snapshot=cfg.pec.k_snapshot,
                    k_persist=cfg.pec.k_snapshot)
    plan = plan_equal(layout, pec) if strat == EQUAL_PEC else plan_adaptive(layout, pec)
    worst = max(bottleneck_workload(plan, p)[1] for p in range(plan.period))
    iter_us = _us(cluster.fb_time) + _us(cluster.update_time)
    drain_floor = max(1, math.ceil(transfer_us(worst, drain_bw) / iter_us))
    return replace(cfg, i_ckpt=max(cfg.i_ckpt, drain_floor))


@dataclass(frozen=True)
class Cadence:
    """The checkpoint cadence a fixed PEC configuration can sustain."""
    i_ckpt_min: int          # smallest interval at which nothing queues up
    persist_floor: int       # ceil(bottleneck persist time / iteration)
    drain_floor: int         # ceil(bottleneck drain time / iteration)
    snapshot_floor: int      # ceil(bottleneck pack time / F&B time) (the reference's overlap rule)
    persist_s: float
    drain_s: float
    pack_s: float


def b200_cadence(layout: RankLayout, strategy: str, pec: PecConfig, cluster: ClusterSpec,
                 drain_bw: float) -> Cadence:
    """For a FIXED K_snapshot / K_persist (a workload's PEC config), the
    smallest I_ckpt whose steady state never waits: the reference's persist
    floor (one persist at a time, oldest first: the persist of a version
    must end before the next one is due, simulator.py:735, engine.py:122-129),
    the staging floor (the drain must empty staging before the next pack),
    and the snapshot-overlap rule (simulator.py:434-438).  Bandwidths are the
    measured ones of `measured_cluster` / `drain_bandwidth`."""
    strat = EQUAL_PEC if strategy == EQUAL_PEC else ADAPTIVE_PEC
    snap = PecConfig(k_pec=pec.k_snapshot, k_snapshot=pec.k_snapshot, k_persist=pec.k_snapshot)
    pers = PecConfig(k_pec=pec.k_persist, k_snapshot=pec.k_persist, k_persist=pec.k_persist)

    def worst(cfg: PecConfig) -> int:
        plan = plan_equal(layout, cfg) if strat == EQUAL_PEC else plan_adaptive(layout, cfg)
        return max(bottleneck_workload(plan, p)[1] for p in range(plan.period))

    w_snap, w_pers = worst(snap), worst(pers)
    iter_us = _us(cluster.fb_time) + _us(cluster.update_time)
    persist_us = transfer_us(w_pers, cluster.persist_bandwidth)
    drain_us = transfer_us(w_snap, drain_bw)
    pack_us = transfer_us(w_snap, cluster.snapshot_bandwidth)
    pf = max(1, math.ceil(persist_us / iter_us))
    df = max(1, math.ceil(drain_us / iter_us))
    sf = max(1, math.ceil(pack_us / max(1, _us(cluster.fb_time))))
    return Cadence(max(pf, df, sf), pf, df, sf, persist_us / US, drain_us / US, pack_us / US)
