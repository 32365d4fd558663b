"""Configurator / analytic model vs. the reference, and the measured-bandwidth
feedback."""

import json

import pytest

from conftest import GOLDEN
from paper_2408_04307_b200 import ClusterSpec, configs
from paper_2408_04307_b200.policy import (
    adaptive_configure_layout,
    analytic_overhead,
    b200_configure,
    drain_bandwidth,
    measured_cluster,
)

POL = json.loads((GOLDEN / "policy.json").read_text())
WL = {"gpt350m": configs.gpt350m_16e(k_pec=2), "toy": configs.toy(),
      "mixtral": configs.mixtral_8x7b()}


@pytest.mark.parametrize("i", range(len(POL["configure"])))
def test_adaptive_configure_matches_reference(i):
    c = POL["configure"][i]
    w = WL[c["workload"]]
    cl = ClusterSpec(w.cluster.num_nodes, w.cluster.gpus_per_node, c["snapshot_bw"],
                     c["persist_bw"], c["fb"], c["update"], 1.0)
    got = adaptive_configure_layout(w.layout(), c["strategy"], cl, c["target"])
    assert (got.pec.k_snapshot, got.pec.k_persist, got.i_ckpt, got.snapshot_overlapped,
            got.persist_target_met) == (c["k_snapshot"], c["k_persist"], c["i_ckpt"],
                                        c["overlapped"], c["target_met"])


def test_analytic_overhead_matches_reference():
    for c in POL["analytic"]:
        r = analytic_overhead(**c["args"])
        assert r.o_ckpt_full_us == pytest.approx(c["full"], rel=1e-12)
        assert r.o_ckpt_moc_us == pytest.approx(c["moc"], rel=1e-12)
        assert r.moc_wins == c["wins"]


def test_measured_bandwidths_feed_the_configurator():
    """With the B200 numbers measured in round 1 (pack 3.1 TB/s payload,
    drain 57 GB/s, persist 11 GB/s to tmpfs) the HBM pack hides any K under a
    100 ms F&B, so the snapshot tier saves every expert; the drain and the
    persist set the checkpoint interval."""
    w = WL["mixtral"]
    layout = w.layout()
    stats = {"snap_bytes": [12_620_806_144] * 2, "pack_ms": [4.05, 4.05],
             "drain_ms": [220.9, 220.9], "persist_s": [1.1, 1.1]}
    base = ClusterSpec(1, 8, 1e9, 1e9, fb_time=0.1, update_time=0.04, restart_time=1.0)
    cl = measured_cluster(base, stats)
    assert cl.snapshot_bandwidth == pytest.approx(12_620_806_144 / 4.05e-3)
    assert cl.persist_bandwidth == pytest.approx(12_620_806_144 / 1.1)
    cfg = b200_configure(layout, "adaptive_pec", cl, drain_bandwidth(stats))
    assert cfg.pec.k_snapshot == layout.model.experts_per_layer and cfg.snapshot_overlapped
    # the reference model with the paper's simulated 1 GB/s snapshot link
    ref = adaptive_configure_layout(layout, "adaptive_pec", base)
    assert ref.pec.k_snapshot < cfg.pec.k_snapshot
    assert cfg.i_ckpt >= 1


def test_b200_cadence_floors_follow_the_measured_rates():
    """policy.b200_cadence (the cadence bench.py's stall leg runs at): each
    floor is ceil(bottleneck time / iteration) for its tier, the minimum
    interval is their maximum, and a slower persist tier never lowers it."""
    import math
    from dataclasses import replace
    from paper_2408_04307_b200 import bottleneck_workload, plan_adaptive
    from paper_2408_04307_b200.policy import b200_cadence
    w = configs.mixtral_8x7b()
    layout = w.layout()
    worst = max(bottleneck_workload(plan_adaptive(layout, w.pec), p)[1] for p in range(8))
    base = replace(layout.cluster, snapshot_bandwidth=3.3e12, fb_time=0.1, update_time=0.025)
    prev = 0
    for persist_gbs in (40, 15, 8, 4):
        cl = replace(base, persist_bandwidth=persist_gbs * 1e9)
        cad = b200_cadence(layout, w.strategy, w.pec, cl, drain_bw=56e9)
        iter_s = 0.125
        assert cad.persist_floor == max(1, math.ceil(worst / (persist_gbs * 1e9) / iter_s - 1e-9))
        assert cad.drain_floor == max(1, math.ceil(worst / 56e9 / iter_s - 1e-9))
        assert cad.snapshot_floor == 1          # a 3.8 ms pack hides under a 100 ms F&B
        assert cad.i_ckpt_min == max(cad.persist_floor, cad.drain_floor, cad.snapshot_floor)
        assert cad.i_ckpt_min >= prev
        prev = cad.i_ckpt_min
    assert prev > 10                            # 4 GB/s persist: I_ckpt = 10 is infeasible
