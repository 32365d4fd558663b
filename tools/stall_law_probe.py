"""Validate the reference's stall law against measured stalls (SURVEY.md
§8(f) row 4; measurement tool, one GPU, not product).

The reference models an asynchronous snapshot as a duration
snap = bytes / snapshot_bandwidth starting after the checkpoint iteration's
update; the next iteration stalls by max(0, snap_end - fb_end)
(simulator.py:434-438, :551-556).  On B200 the only part of a snapshot that
the next update must wait for is the HBM pack (the drain to pinned host runs
behind on the copy engine and only has to finish before the staging is
reused), so the law predicts, per checkpoint,

    stall = max(0, pack_ms - fb_ms)            (snapshot_bandwidth = pack rate)
          + max(0, drain_ms - (I_ckpt - 1) * iter_ms - fb_ms)   (staging reuse)

This probe measures pack and drain alone, then runs bench.py's synthetic
loop (bf16 GEMM F&B proxy + full-arena update proxy, checkpoint every
I_ckpt-th iteration through PecCheckpointer) for a sweep of F&B durations,
A/B-alternated, and prints the predicted and the measured exposed ms per
checkpoint for each.  Also printed: what the law predicts if the whole
device->host copy were the blocking snapshot (the reference's modelling of a
snapshot), to show what staging buys."""
import argparse
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="mixtral")
    ap.add_argument("--fb-ms", default="1,2,4,8,16,100")
    ap.add_argument("--iters", type=int, default=40)
    ap.add_argument("--i-ckpt", type=int, default=10)
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--modes", default="0",
                    help="comma list of pec_pack modes to compare (0 auto/bulk, 17-20 the "
                         "bulk engine on 1/2..1/8 of the SMs, 3 the CRC engine)")
    args = ap.parse_args()
    import torch
    import bench
    from paper_2408_04307_b200.arena import StateArena
    from paper_2408_04307_b200.counting import DeviceTokenCounters
    from paper_2408_04307_b200.snapshot import PecCheckpointer

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    w, layout, _ = bench.build_workload(argparse.Namespace(workload=args.workload), 0)
    arena = StateArena(layout, ranks=[0], device=dev, expert_tensors=w.expert_tensors)
    L, E = layout.model.num_moe_layers, layout.model.experts_per_layer
    counters = DeviceTokenCounters(L, E, dev)
    modes = [int(m) for m in args.modes.split(",")]
    out = {"workload": w.name, "i_ckpt": args.i_ckpt, "iters": args.iters,
           "rounds": args.rounds, "modes": {}}
    for mode in modes:
        out["modes"][str(mode)] = sweep(args, bench, torch, dev, w, layout, arena, counters,
                                        PecCheckpointer, mode)
    print(json.dumps(out if len(modes) > 1 else {**out, **out["modes"][str(modes[0])]},
                     indent=1))


def sweep(args, bench, torch, dev, w, layout, arena, counters, PecCheckpointer, mode):
    ck = PecCheckpointer(layout, arena, None, w.pec, w.strategy, i_ckpt=1, ranks=[0],
                         counters=counters, pack_mode=mode)
    eng = ck.engine
    eng.reserve(ck.max_snapshot_bytes(), host_buffers=2)

    # pack and drain alone (no training work on the GPU)
    for it in range(1, 6):
        ck.checkpoint(it)
        ck.wait_pack()
        torch.cuda.synchronize()
        ck.finish()
    pack_alone = statistics.median(eng.stats["pack_ms"][-3:])
    drain_alone = statistics.median(eng.stats["drain_ms"][-3:])
    snap_bytes = eng.stats["snap_bytes"][-1]

    rows = []
    for fb in (float(x) for x in args.fb_ms.split(",")):
        s = bench.measure_stall(ck, arena, dev, args.iters, args.i_ckpt, fb, rounds=args.rounds)
        fb_ms, upd = s["fb_ms"], s["update_ms"]
        iter_ms = s["iter_ms_without"]
        pred_pack = max(0.0, pack_alone - fb_ms)
        pred_reuse = max(0.0, drain_alone - (args.i_ckpt - 1) * iter_ms - fb_ms)
        pred_d2h_blocking = max(0.0, pack_alone + drain_alone - fb_ms)
        rows.append({
            "fb_ms": fb_ms, "update_ms": upd, "iter_ms_without": iter_ms,
            "pack_ms_in_loop": s["pack_ms_in_loop"],
            "predicted_ms_per_ckpt": round(pred_pack + pred_reuse, 2),
            "predicted_pack_term": round(pred_pack, 2),
            "predicted_reuse_term": round(pred_reuse, 2),
            "measured_ms_per_ckpt": round(s["exposed_ms_per_iter"] * args.i_ckpt, 2),
            "noise_ms_per_ckpt": round(s["noise_ms_per_iter"] * args.i_ckpt, 2),
            "if_d2h_blocked_ms_per_ckpt": round(pred_d2h_blocking, 2),
            "runs_ms_without": s["runs_ms_without"], "runs_ms_with": s["runs_ms_with"],
        })
        print(json.dumps(rows[-1]), file=sys.stderr, flush=True)
    ck.close()
    return {"snap_bytes": snap_bytes, "pack_ms_alone": round(pack_alone, 3),
            "drain_ms_alone": round(drain_alone, 2), "sweep": rows}


if __name__ == "__main__":
    main()
