"""Restore throughput: every unit of GPT-MoE 350M-16E (all 8 ranks of dp=ep=8
on one GPU, 2 nodes x 4 GPUs) brought back from storage after both nodes fail.

One PEC checkpoint at K_pec = 16 (every expert, so one version holds the whole
26.1 GB state) is packed, drained and persisted to a DiskStore on /dev/shm.
Then, ``--reps`` times: the arena is wiped, `resolve_recovery` over nodes
{0, 1} decides storage for every unit, and `restore` reads, verifies (CRC-32C
against the manifest, on the device or on the host) and scatters the bytes;
the arena is compared on the device with a clone taken at the checkpoint.

Prints one JSON document: GB/s = storage bytes / restore wall time, the
per-phase host seconds of `RestoreReport.phases`, and the host-side tmpfs
read ceiling measured with the same reader (`restore._read_files`) alone.
"""

import json
import os
import shutil
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def read_ceiling(store, version, threads, slot_bytes):
    """The restore's own reader, alone: every entry file of ``version`` read
    into one pinned slot by ``threads`` threads (no H2D, no CRC)."""
    import torch
    from concurrent.futures import ThreadPoolExecutor
    from paper_2408_04307_b200 import restore as R
    vdir = store.version_dir(version)
    files = sorted(vdir.rglob("*.bin"))
    slot = torch.empty(slot_bytes, dtype=torch.uint8, pin_memory=True)

    class P:
        pass
    total = 0
    t0 = time.perf_counter()
    with ThreadPoolExecutor(threads) as pool:
        for f in files:
            size = f.stat().st_size
            for lo in range(0, size, slot_bytes):
                p = P()
                p.nbytes, p.path, p.file_off, p.entry = min(slot_bytes, size - lo), str(f), lo, f.name
                R._read_files(pool, [(p, 0, slot)], want_crc=False)
                total += p.nbytes
    dt = time.perf_counter() - t0
    return round(total / dt / 1e9, 2)


def main():
    import argparse
    import torch
    from paper_2408_04307_b200 import ClusterSpec, PecConfig, build_layout, configs
    from paper_2408_04307_b200.arena import StateArena
    from paper_2408_04307_b200.restore import restore
    from paper_2408_04307_b200.snapshot import PecCheckpointer
    from paper_2408_04307_b200.store import DiskStore

    ap = argparse.ArgumentParser()
    ap.add_argument("--verify", default="device", choices=["device", "host"])
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--io-threads", type=int, default=None, help="default: one per core")
    ap.add_argument("--slot-mb", type=int, default=256)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    w = configs.gpt350m_16e(k_pec=16, strategy="equal_pec")
    layout = build_layout(w.model, w.parallel, ClusterSpec(num_nodes=2, gpus_per_node=4))
    arena = StateArena(layout, range(8), dev, w.expert_tensors)
    root = "/dev/shm/pec_restore_bench"
    shutil.rmtree(root, ignore_errors=True)
    store = DiskStore(root, io_threads=16)
    ck = PecCheckpointer(layout, arena, store, PecConfig(k_pec=16), "equal_pec", i_ckpt=1)
    ck.engine.reserve(ck.max_snapshot_bytes())
    ck.step(1)
    ck.finish()
    ref = arena.buffer.clone()
    version = store.newest_complete()
    out = {"workload": w.name, "arena_gb": round(arena.buffer.numel() / 1e9, 2),
           "verify": args.verify, "io_threads": args.io_threads, "slot_mb": args.slot_mb,
           "runs": []}
    ck.engine.on_fault({0, 1})
    for _ in range(args.reps):
        plan = ck.engine.resolve_recovery({0, 1})
        arena.buffer.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep = restore(ck.engine, plan, verify=args.verify, io_threads=args.io_threads,
                      slot_bytes=args.slot_mb << 20)
        wall = time.perf_counter() - t0
        ok = bool(torch.equal(arena.buffer, ref))
        out["runs"].append({"wall_s": round(wall, 3), "storage_bytes": rep.storage_bytes,
                            "memory_bytes": rep.memory_bytes, "batches": rep.batches,
                            "GBps": round(rep.storage_bytes / wall / 1e9, 2),
                            "unpack_ms": round(rep.unpack_ms, 2),
                            "phases_s": {k: round(v, 3) for k, v in (rep.phases or {}).items()},
                            "bit_identical": ok})
    threads = args.io_threads or max(4, len(os.sched_getaffinity(0)))
    out["read_ceiling_GBps"] = read_ceiling(store, version, threads, args.slot_mb << 20)
    ck.close()
    shutil.rmtree(root, ignore_errors=True)
    print(json.dumps(out))
    return 0 if all(r["bit_identical"] for r in out["runs"]) else 1


if __name__ == "__main__":
    sys.exit(main())
