"""A real toy-MoE training loop whose parameters/Adam states are views of the
state arena, checkpointed by the load-aware PEC path, then restored."""

import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "examples"))


def test_moe_training_loop_checkpoints_and_restores(dev, tmp_path):
    import torch
    import moe_training as ex
    from paper_2408_04307_b200.restore import restore
    snaps = {}

    def grab(buf):
        torch.cuda.synchronize()
        snaps[buf.version] = arena_ref[0].buffer.cpu().numpy().copy()

    arena_ref = []
    orig_build = ex.build

    def build_and_keep(dev_, seed=0):
        out = orig_build(dev_, seed)
        arena_ref.append(out[2])
        return out

    ex.build = build_and_keep
    try:
        ck, arena, losses, params = ex.train(iters=12, i_ckpt=4, store_root=str(tmp_path),
                                             tokens=256, on_checkpoint=grab)
    finally:
        ex.build = orig_build
    assert all(np.isfinite(losses)) and losses[-1] < losses[0]
    versions = ck.engine.store.complete_versions()
    assert versions == sorted(snaps)
    # every persisted entry is the snapshotted state of its version
    for v in versions:
        data = ck.engine.store.load_checkpoint(v)
        for k, b in data.items():
            e = ck.engine.store.meta(v).entries[k]
            off = arena.slot(e.unit_key).offset + e.start
            assert b == snaps[v][off:off + e.stop - e.start].tobytes(), (v, k)
    # lose the GPU state; partial-expert restore from memory/storage/initial
    plan = ck.engine.resolve_recovery(set())
    ck.engine.on_fault(set())
    arena.buffer.zero_()
    restore(ck.engine, plan)
    now = arena.buffer.cpu().numpy()
    for key, d in plan.decisions.items():
        if d.source in ("memory", "storage") and arena.has(key):
            s = arena.slot(key)
            assert np.array_equal(now[s.offset:s.offset + s.size],
                                  snaps[d.version][s.offset:s.offset + s.size]), key
    # training resumes on the restored state
    tok = torch.randint(0, 1024, (256,), device=dev)
    loss, _ = ex.forward(params, dict(d=256, ffn=1024, L=4, E=8, V=1024, top_k=2), tok,
                         torch.roll(tok, -1))
    assert torch.isfinite(loss)
    ck.close()


def test_moe_training_loop_survives_a_node_fault(dev, tmp_path):
    """The same loop with the GPU state wiped at iteration 10 (node 0 lost,
    so only storage and initial images remain): PecCheckpointer.recover
    restores it, training replays from the restart iteration and keeps
    learning; the persisted versions stay loadable."""
    import moe_training as ex
    ck, arena, losses, params = ex.train(iters=16, i_ckpt=4, store_root=str(tmp_path),
                                         tokens=256, fault_at=10)
    assert all(np.isfinite(losses))
    assert len(losses) == 16 + (10 - 8)      # iterations 9..10 replayed after restart 8
    assert losses[-1] < losses[0]
    versions = ck.engine.store.complete_versions()
    assert len(versions) >= 4
    for v in versions:
        ck.engine.store.load_checkpoint(v)   # CRC-verified
    ck.close()
