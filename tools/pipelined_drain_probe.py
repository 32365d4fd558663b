"""Pipelined vs. whole-pack-then-drain snapshots, A/B on one box (measurement
tool, one GPU, not product).

Mixtral-shaped rank 0, snapshot tier only: each measured snapshot is
PecCheckpointer.checkpoint() + wait_snapshot() (pack into HBM staging + D2H
drain into a pinned host buffer), wall-clock, alternating the engine's
``pipelined_drain`` off / on so drifts hit both arms.  Prints one JSON
document with the per-arm snapshot times and GB/s."""
import argparse
import json
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="mixtral")
    ap.add_argument("--rounds", type=int, default=6)
    args = ap.parse_args()
    import torch
    import bench
    from paper_2408_04307_b200.arena import StateArena
    from paper_2408_04307_b200.snapshot import PecCheckpointer

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    w, layout, plan = bench.build_workload(argparse.Namespace(workload=args.workload), 0)
    arena = StateArena(layout, ranks=[0], device=dev, expert_tensors=w.expert_tensors)
    arms = {}
    for pipelined in (False, True):
        ck = PecCheckpointer(layout, arena, None, w.pec, w.strategy, i_ckpt=1, ranks=[0])
        ck.engine.pipelined_drain = pipelined
        ck.engine.reserve(ck.max_snapshot_bytes(), host_buffers=2)
        ck.prepare()
        arms[pipelined] = ck
    res = {False: [], True: []}
    it = 0
    for _ in range(args.rounds + 1):
        for pipelined, ck in arms.items():
            it += 1
            torch.cuda.synchronize()
            t = time.perf_counter()
            buf = ck.checkpoint(it)
            ck.wait_snapshot(buf)
            dt = time.perf_counter() - t
            res[pipelined].append((dt, ck.engine.snapshot_nbytes(buf)))
    out = {"workload": w.name, "rounds": args.rounds}
    for pipelined, rows in res.items():
        rows = rows[1:]   # first round warms each arm
        ms = [r[0] * 1e3 for r in rows]
        gbps = [r[1] / r[0] / 1e9 for r in rows]
        out["pipelined" if pipelined else "whole"] = {
            "ms": [round(x, 2) for x in ms], "median_ms": round(statistics.median(ms), 2),
            "GBps": [round(x, 2) for x in gbps], "median_GBps": round(statistics.median(gbps), 2),
            "segments": None if not pipelined else
            len(next(iter(arms[True].engine._tables.values()))[0].segments or [])}
    for ck in arms.values():
        ck.close()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
