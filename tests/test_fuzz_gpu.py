"""Randomised end-to-end runs of the B200 path (GPU): random layouts (1-2 EP
groups, 2 nodes), strategies, K, selection policies, checkpoint cadences and
node faults.  A host shadow keeps the arena bytes of every snapshot; after
each fault `PecCheckpointer.recover` must bring every resident unit back
bit-identical to the version its decision names (memory / storage) or to its
seeded initial image, and every persisted version must read back (CRC
verified) equal to the shadow."""

import random

import numpy as np
import pytest

from conftest import make_layout

pytestmark = pytest.mark.gpu


def _mutate(arena, it):
    for key, s in arena.slots.items():
        arena.buffer[s.offset:s.offset + s.size][it % 13:: 89].add_(it + 1)


@pytest.mark.parametrize("seed", range(10))
def test_random_runs_with_faults_restore_exact_bytes(dev, tmp_path, seed):
    import torch
    from paper_2408_04307_b200 import PecConfig
    from paper_2408_04307_b200.arena import StateArena
    from paper_2408_04307_b200.counting import DeviceTokenCounters
    from paper_2408_04307_b200.snapshot import PecCheckpointer
    from paper_2408_04307_b200.store import DiskStore
    rng = random.Random(seed)
    E = rng.choice([2, 4, 8])
    ep = rng.choice([d for d in (1, 2, 4) if E % d == 0 and 4 % d == 0])
    L = rng.randint(1, 3)
    layout = make_layout(n_experts=E, n_layers=L, dp=4, ep=ep, gpus_per_node=2,
                         epp=rng.randint(1000, 90_000), other=rng.choice([0, 333]))
    ranks = list(range(4))
    arena = StateArena(layout, ranks, dev)
    initial = arena.buffer.cpu().numpy().copy()
    selection = rng.choice(["sequential", "load_aware"])
    strategy = "equal_pec" if selection == "load_aware" else rng.choice(["equal_pec",
                                                                         "adaptive_pec"])
    k = rng.randint(1, E)
    pec = PecConfig(k_pec=k, selection=selection, k_snapshot=k, k_persist=rng.randint(1, k))
    counters = DeviceTokenCounters(L, E, dev) if selection == "load_aware" else None
    i_ckpt = rng.choice([1, 2, 3])
    ck = PecCheckpointer(layout, arena, DiskStore(tmp_path), pec, strategy, i_ckpt=i_ckpt,
                         ranks=ranks, counters=counters, async_persist=rng.random() < 0.5)
    shadow = {}
    forced = rng.randint(4, 10)           # every run sees at least one fault
    it, steps, faults = 1, 0, 0
    while it <= 14 and steps < 60:
        steps += 1
        _mutate(arena, it)
        ids = torch.randint(0, E, (L, 64), dtype=torch.int32, device=dev) if counters else None
        buf = ck.step(it, ids)
        if buf is not None:
            torch.cuda.synchronize()
            shadow[buf.version] = arena.buffer.cpu().numpy().copy()
            ck.wait_pack()
        if faults < 2 and it > 2 and (rng.random() < 0.2 or (faults == 0 and it == forced)):
            faults += 1
            ck.finish()
            arena.buffer.zero_()
            out = ck.recover({rng.choice([0, 1])}, it)
            torch.cuda.synchronize()
            now = arena.buffer.cpu().numpy()
            for key, d in (out.plan.decisions.items() if out.plan else []):
                if not arena.has(key):
                    continue
                s = arena.slot(key)
                want = initial if d.source == "initial" else shadow[d.version]
                assert np.array_equal(now[s.offset:s.offset + s.size],
                                      want[s.offset:s.offset + s.size]), (seed, key, d)
            if out.plan is None:
                assert np.array_equal(now, initial)
            it = out.restart_iteration + 1
            continue
        it += 1
    assert faults >= 1
    ck.finish()
    for v in ck.engine.store.complete_versions():
        data = ck.engine.store.load_checkpoint(v)
        meta = ck.engine.store.meta(v)
        for sk, b in data.items():
            e = meta.entries[sk]
            off = arena.slot(e.unit_key).offset + e.start
            assert b == shadow[v][off:off + e.stop - e.start].tobytes(), (seed, v, sk)
    ck.close()
