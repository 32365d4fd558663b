"""Multi-GPU check of the PEC path (run under torchrun).

GPT-MoE 350M-16E, K_pec=2 load-aware (equal_pec).  Default: dp=ep=N
deployment (N = world size), one rank per process, one process per GPU.
``--config3``: BASELINE config 3 itself — the dp=8 x ep=8 layout on two
4-GPU nodes — as 8 processes (``--ranks-per-proc 1``; more processes than
GPUs share devices round-robin, which NCCL refuses, so run it with
``--backend gloo``) or as fewer processes each hosting several of the eight
ranks in one engine (``--ranks-per-proc 2`` on 4 GPUs over NCCL).
Per checkpoint:
  * every rank counts its own router ids (different seeds) on device,
  * NCCL all-reduce of the [2, L, E] counters -> identical global selection
    on every rank == the oracle's selection on the summed counts,
  * pack + drain + multi-writer persist (gloo control group) to a shared store,
  * every rank verifies its persisted entries against its arena bytes,
then node N-1 fails: `PecCheckpointer.recover` on every rank (identical
decisions; memory / storage / initial bytes back into the wiped arena, checked
bit-exact per unit; the all-reduced counters after the reset equal the global
tokens delivered between each expert's restored iteration and the restart
point).  Prints one JSON line per rank; exits non-zero on any mismatch.
"""

import json
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def fingerprint(arena, buf, ranks):
    """CRC-32C of every resident unit and of these ranks' planned entries,
    taken from a host copy of the arena at snapshot time."""
    from paper_2408_04307_b200 import device as D
    host = arena.buffer.cpu().numpy()
    keys = list(arena.slots)
    units = D.crc32c_many(host, [arena.slots[k].offset for k in keys],
                          [arena.slots[k].size for k in keys])
    ents = [a for r in ranks for a in buf.content.get(r, ())]
    ecrc = D.crc32c_many(host, [arena.slot(a.key).offset + a.start for a in ents],
                         [a.stop - a.start for a in ents])
    return {"units": {k: int(c) for k, c in zip(keys, units)},
            "entries": {a.store_key: int(c) for a, c in zip(ents, ecrc)}}


def main():
    import torch
    import torch.distributed as dist
    from oracle import pec_oracle as O
    from paper_2408_04307_b200 import PecConfig, configs
    from paper_2408_04307_b200.arena import StateArena
    from paper_2408_04307_b200.counting import DeviceTokenCounters
    from paper_2408_04307_b200.snapshot import PecCheckpointer
    from paper_2408_04307_b200.store import DiskStore, crc32c

    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--config3", action="store_true")
    ap.add_argument("--ranks-per-proc", type=int, default=1)
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"])
    args = ap.parse_args()
    rank, local, world = (int(os.environ[k]) for k in ("RANK", "LOCAL_RANK", "WORLD_SIZE"))
    local_dev = local % torch.cuda.device_count()   # >1 process per GPU: gloo only
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    if args.backend == "nccl":
        dist.init_process_group("nccl", device_id=dev)
    else:
        dist.init_process_group("gloo")
    control = dist.new_group(backend="gloo")
    root = os.environ.get("PEC_STORE", "/dev/shm/pec_multirank")
    if rank == 0:
        import shutil
        shutil.rmtree(root, ignore_errors=True)
    dist.barrier()

    R = args.ranks_per_proc
    my_ranks = [rank * R + j for j in range(R)]
    n_ranks = world * R
    from paper_2408_04307_b200 import ClusterSpec, build_layout
    if args.config3:
        if n_ranks != 8:
            raise SystemExit("--config3 needs world * ranks-per-proc == 8")
        w = configs.gpt350m_16e_load_aware(k_pec=2)        # dp=8 x ep=8
        # two nodes of four: a node fault leaves four surviving ranks
        cluster = ClusterSpec(num_nodes=2, gpus_per_node=4)
    else:
        w = configs.gpt350m_16e(k_pec=2, strategy="equal_pec", dp=n_ranks, ep=n_ranks)
        # one rank per "node" so a node fault leaves peers whose host snapshot
        # buffers (node-shared /dev/shm) serve memory-sourced restores
        cluster = ClusterSpec(num_nodes=n_ranks, gpus_per_node=1)
    layout = build_layout(w.model, w.parallel, cluster)
    L, E = layout.model.num_moe_layers, layout.model.experts_per_layer
    arena = StateArena(layout, my_ranks, dev, w.expert_tensors)
    routed = 4096 * 2
    cap = DeviceTokenCounters.capacity_for(1.25, [routed] * L, E)
    counters = DeviceTokenCounters(L, E, dev, cap)
    pec = PecConfig(k_pec=2, selection="load_aware", k_snapshot=2, k_persist=1)
    store = DiskStore(root)
    ck = PecCheckpointer(layout, arena, store, pec, "equal_pec", i_ckpt=3, ranks=my_ranks,
                         counters=counters, group=None, control_group=control,
                         async_persist=False,
                         shared_host_prefix="pec_mr")
    ck.group = dist.group.WORLD  # the counter all-reduce (NCCL, or gloo when GPUs are shared)
    failed_node = layout.cluster.num_nodes - 1

    glob = np.zeros((2, L, E), dtype=np.int64)
    ok = True
    persisted_bytes = {}
    t0 = time.time()
    delivered = {}  # iteration -> global delivered counts [L, E]
    for it in range(1, 10):
        ids = {r: np.stack([O.zipf_router_ids(100 + r, it, m, E, routed, 1.1) for m in range(L)])
               for r in range(n_ranks)}
        delivered[it] = np.zeros((L, E), dtype=np.int64)
        for r in range(n_ranks):
            c = O.route_counts(ids[r], E, cap)
            glob[0] += c
            glob[1] += c
            delivered[it] += c
        for r in my_ranks[1:]:          # every hosted rank counts its own tokens (own cap)
            counters.add_iteration(torch.from_numpy(ids[r]).to(dev))
        buf = ck.step(it, torch.from_numpy(ids[my_ranks[0]]).to(dev))
        if buf is not None:
            ck.resolve(buf)
            ss, ps, glob[0], glob[1] = O.two_tier_load_aware(glob[0], glob[1], 2, 1)
            got_p = [sorted(ck.persist_sel[buf.version][m]) for m in range(L)]
            ok &= got_p == ps
            # snapshot set: experts appearing in the phase assignment (any rank)
            snap = {m: set() for m in range(L)}
            for rr, ranges in buf.content.items():
                for a in ranges:
                    u = layout.by_key[a.key]
                    if u.layer is not None:
                        snap[u.layer].add(u.expert)
            ok &= [sorted(snap[m]) for m in range(L)] == ss
            torch.cuda.synchronize()
            persisted_bytes[buf.version] = fingerprint(arena, buf, my_ranks)
            ck.wait_pack()
        # stand-in optimizer step: versions must differ
        for key, sl in arena.slots.items():
            arena.buffer[sl.offset:sl.offset + sl.size][:: 4099].add_(it)
    ck.finish()
    sel_ok = ok
    # verify persisted entries of this rank against the arena at snapshot time
    versions = store.complete_versions()
    files_ok = bool(versions)
    for v in versions:
        meta = store.meta(v)
        mine = [k for k, e in meta.entries.items() if e.rank in my_ranks]
        data = store.load_checkpoint(v, mine)   # CRC-verified read
        for k in mine:
            files_ok &= crc32c(data[k]) == persisted_bytes[v]["entries"][k]
    dist.barrier()
    # node `world-1` fails: every rank restores all of its resident units from
    # memory (own or a surviving peer's node-shared buffer), storage or initial
    failed = {failed_node}
    arena.buffer.zero_()
    out = ck.recover(failed, 9)       # decisions -> unwind -> restore -> counter reset
    plan, rep = out.plan, out.report
    keys = [k for k in plan.decisions if arena.has(k)]
    after = arena.buffer.cpu().numpy()
    # global unsaved tokens after the reset: delivered in (restored, restart]
    want_unsaved = np.zeros((L, E), dtype=np.int64)
    for (m, e), r in out.expert_restore.items():
        if r < out.restart_iteration:
            want_unsaved[m, e] = sum(delivered[i][m, e]
                                     for i in range(r + 1, out.restart_iteration + 1))
    got = counters.all_reduced(dist.group.WORLD).cpu().numpy()
    counters_ok = bool(np.array_equal(got[0], want_unsaved) and np.array_equal(got[1], want_unsaved))
    restore_ok = bool(keys)
    sources = {}
    for k in keys:
        d = plan.decisions[k]
        sources[d.source] = sources.get(d.source, 0) + 1
        sl = arena.slot(k)
        want = persisted_bytes[d.version]["units"][k] if d.source != "initial" else None
        if want is not None:
            restore_ok &= crc32c(after[sl.offset:sl.offset + sl.size]) == want
    dist.barrier()  # peers may still be reading this rank's shared buffers
    ck.close()
    writers = {e.rank for v in versions for e in store.meta(v).entries.values()}
    res = {"rank": rank, "world": world, "ranks": my_ranks, "layout_ranks": n_ranks,
           "backend": args.backend, "device": local_dev, "writers": len(writers),
           "selection_ok": bool(sel_ok), "files_ok": bool(files_ok),
           "restore_ok": bool(restore_ok), "counters_ok": counters_ok,
           "restart": out.restart_iteration, "versions": versions, "restored_units": len(keys),
           "sources": sources, "memory_bytes": rep.memory_bytes,
           "storage_bytes": rep.storage_bytes, "restore_wall_s": round(rep.wall_s, 2),
           "seconds": round(time.time() - t0, 1)}
    print(json.dumps(res), flush=True)
    dist.barrier()
    if rank == 0:
        import shutil
        shutil.rmtree(root, ignore_errors=True)
    dist.destroy_process_group()
    return 0 if (sel_ok and files_ok and restore_ok and counters_ok) else 1


if __name__ == "__main__":
    sys.exit(main())
