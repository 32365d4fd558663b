"""Config 5: partial-expert restore from a chain of PEC checkpoints + a K_pec
sweep 1..E on GPT-MoE 350M-16E (dp=ep=8, all 8 ranks emulated on one GPU,
2 nodes x 4 GPUs).

Chain: sequential K_pec (default 1; adaptive
plan), one full selection period (16 checkpoints at K=1), every checkpoint packed, drained and persisted to a
DiskStore on /dev/shm; a stand-in optimizer step perturbs every unit between
checkpoints so versions differ.  Then node 1 fails: `resolve_recovery`
decides per unit (memory on node 0 / storage / initial), the state is wiped
and `restore()` brings it back; every restored unit is compared byte for
byte with the bytes of the version it was restored from (entry files, or
the surviving host snapshot buffer) and its CRC-32C with the arena
fingerprint taken at that checkpoint.

Sweep: for K = 1, 2, 4, 8, 16 (equal plan) one snapshot of all ranks: staged
payload == planner workload, device-side equality of every entry, pack
GB/s.  Prints one JSON document.
"""

import json
import shutil
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import argparse
    import torch
    from paper_2408_04307_b200 import ClusterSpec, PecConfig, build_layout, configs
    from paper_2408_04307_b200 import device as D
    from paper_2408_04307_b200.arena import StateArena
    from paper_2408_04307_b200.restore import restore
    from paper_2408_04307_b200.snapshot import PecCheckpointer
    from paper_2408_04307_b200.store import DiskStore

    ap = argparse.ArgumentParser()
    ap.add_argument("--k", type=int, default=1)
    ap.add_argument("--verify", default="device", choices=["device", "host"])
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    out = {"k_pec": args.k, "verify": args.verify}
    w = configs.gpt350m_16e(k_pec=args.k, strategy="adaptive_pec")
    layout = build_layout(w.model, w.parallel, ClusterSpec(num_nodes=2, gpus_per_node=4))
    arena = StateArena(layout, range(8), dev, w.expert_tensors)
    keys = list(arena.slots)
    offs = [arena.slots[k].offset for k in keys]
    sizes = [arena.slots[k].size for k in keys]

    def fingerprint():
        host = arena.buffer.cpu().numpy()
        return dict(zip(keys, (int(c) for c in D.crc32c_many(host, offs, sizes))))

    initial = fingerprint()
    root = "/dev/shm/pec_chain"
    shutil.rmtree(root, ignore_errors=True)
    store = DiskStore(root, io_threads=16)
    ck = PecCheckpointer(layout, arena, store, PecConfig(k_pec=args.k), "adaptive_pec",
                        i_ckpt=1)
    ck.engine.reserve(ck.max_snapshot_bytes())
    fps = {}
    t0 = time.time()
    period = ck.plan().period  # E / gcd(E, K) checkpoints cover every expert once
    for it in range(1, period + 1):
        buf = ck.step(it)
        torch.cuda.synchronize()
        fps[buf.version] = fingerprint()
        ck.wait_pack()
        for k in keys:  # stand-in optimizer step
            sl = arena.slots[k]
            arena.buffer[sl.offset:sl.offset + sl.size][:: 8191].add_(it)
    ck.finish()
    out["chain"] = {"checkpoints": period, "versions": store.complete_versions(),
                    "seconds": round(time.time() - t0, 1),
                    "pack_ms_avg": round(float(np.mean(ck.engine.stats["pack_ms"])), 3),
                    "drain_ms_avg": round(float(np.mean(ck.engine.stats["drain_ms"])), 2),
                    "persist_s_avg": round(float(np.mean(ck.engine.stats["persist_s"])), 3),
                    "bytes_per_checkpoint": int(np.mean(ck.engine.stats["snap_bytes"]))}

    # ---- fault on node 1, recover -------------------------------------------
    plan = ck.engine.resolve_recovery({1})
    sources = {}
    for k, d in plan.decisions.items():
        sources[d.source] = sources.get(d.source, 0) + 1
    ck.engine.on_fault({1})
    arena.buffer.zero_()
    torch.cuda.synchronize()
    tr = time.time()
    rep = restore(ck.engine, plan, verify=args.verify)
    restore_s = time.time() - tr
    now = arena.buffer.cpu().numpy()
    crc_now = dict(zip(keys, (int(c) for c in D.crc32c_many(now, offs, sizes))))
    crc_ok = exact_ok = True
    bad = []
    for k in keys:
        d = plan.decisions[k]
        want = initial[k] if d.source == "initial" else fps[d.version][k]
        if crc_now[k] != want:
            crc_ok = False
            bad.append(k)
        if d.source == "storage":
            meta = store.meta(d.version)
            parts = sorted((e.start, e.stop, sk) for sk, e in meta.entries.items() if e.unit_key == k)
            data = store.load_checkpoint(d.version, [p[2] for p in parts])
            sl = arena.slots[k]
            for start, stop, sk in parts:
                exact_ok &= data[sk] == bytes(now[sl.offset + start:sl.offset + stop])
    out["restore"] = {"failed_nodes": [1], "sources": sources,
                      "restart_iteration": plan.restart_iteration,
                      "version_skew": plan.version_skew, "units": rep.units,
                      "memory_bytes": rep.memory_bytes, "storage_bytes": rep.storage_bytes,
                      "initial_units": rep.initial_units, "unpack_ms": round(rep.unpack_ms, 3),
                      "unpack_GBps_hbm": round(2 * (rep.memory_bytes + rep.storage_bytes)
                                               / (rep.unpack_ms / 1e3) / 1e9, 1)
                      if rep.unpack_ms else None,
                      "wall_s": round(restore_s, 2),
                      "crc_bit_identical": crc_ok, "storage_bytes_exact": bool(exact_ok),
                      "mismatched_units": bad[:10]}
    ck.close()
    shutil.rmtree(root, ignore_errors=True)

    # ---- K sweep -------------------------------------------------------------
    from paper_2408_04307_b200 import plan_equal
    from paper_2408_04307_b200.snapshot import DeviceCheckpointEngine
    from paper_2408_04307_b200.store import MemoryStore
    sweep = []
    for k in (1, 2, 4, 8, 16):
        plan_k = plan_equal(layout, PecConfig(k_pec=k))
        eng = DeviceCheckpointEngine(layout, MemoryStore(), arena)
        ph = plan_k.assignments[0]
        for _ in range(2):
            a, b, n = eng.pack_only(ph, plan_key=("k", k))
        torch.cuda.synchronize()
        times = []
        for _ in range(5):
            a, b, n = eng.pack_only(ph, plan_key=("k", k))
            b.synchronize()
            times.append(a.elapsed_time(b))
        ok = True
        layouts = eng.layouts_for(ph, ("k", k))
        base = 0
        for r, st in layouts.items():
            for e in st.entries:
                ok &= bool(torch.equal(eng.staging[base + e.stage_offset:base + e.stage_offset + e.nbytes],
                                       arena.buffer[e.src_offset:e.src_offset + e.nbytes]))
            base += (st.nbytes + 255) // 256 * 256
        total = sum(st.payload_bytes for st in layouts.values())
        sweep.append({"k": k, "period": plan_k.period, "bytes_all_ranks": total,
                      "planner_total": sum(plan_k.workload_bytes[0].values()),
                      "pack_ms": round(float(np.median(times)), 3),
                      "pack_GBps_hbm": round(2 * total / (np.median(times) / 1e3) / 1e9, 1),
                      "bit_exact": ok})
        eng.close()
        del eng
        torch.cuda.empty_cache()
    out["k_sweep"] = sweep
    print(json.dumps(out, indent=1))
    good = crc_ok and exact_ok and all(s["bit_exact"] and s["bytes_all_ranks"] == s["planner_total"]
                                       for s in sweep)
    return 0 if good else 1


if __name__ == "__main__":
    sys.exit(main())
