"""How much training time does each pack engine cost when it overlaps a
compute-bound training loop?  (measurement tool, one GPU)

Synthetic loop per iteration, as in bench.py's stall leg: an F&B proxy
(bf16 8192^3 GEMMs, ~100 ms) then an update proxy (an in-place HBM pass over
the Mixtral-shaped rank-0 state arena, ~40 ms).  Every 10th iteration the
rank's phase-0 ranges (12.62 GB) are packed into HBM staging on a side
stream after the update and drained to pinned host memory on the copy
stream; the next update waits for the pack.  Engines:

  bulk       pec_pack mode 2 (TMA bulk, one CTA on every SM; the default)
  vec        pec_pack mode 1 (LDG/STG.128)
  narrowN    pec_pack modes 17-20 (the bulk engine on 1/2 .. 1/8 of the SMs)
  memcpy     one cudaMemcpyAsync per entry (torch copy_), the library path

Runs alternate none / engine so drifts hit both; prints one JSON document
with the exposed ms per iteration of each engine and its pack time alone
and in the loop."""
import argparse
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

ENGINES = {"bulk": 2, "vec": 1, "narrow2": 17, "narrow4": 18, "narrow4x6": 19,
           "narrow8x6": 20, "memcpy": None}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--engines", default="bulk,narrow2,narrow4,narrow4x6,narrow8x6,memcpy,vec")
    ap.add_argument("--iters", type=int, default=30)
    ap.add_argument("--rounds", type=int, default=2)
    ap.add_argument("--i-ckpt", type=int, default=10)
    ap.add_argument("--no-drain", action="store_true")
    ap.add_argument("--priorities", default="-1",
                    help="comma list of pack-stream priorities to compare (-1 high, 0 normal)")
    args = ap.parse_args()
    import torch
    from paper_2408_04307_b200 import configs, plan_adaptive
    from paper_2408_04307_b200 import device as D
    from paper_2408_04307_b200.arena import StateArena
    from paper_2408_04307_b200.staging import DeviceTable, StagingLayout
    dev = torch.device("cuda", 0)
    w = configs.mixtral_8x7b()
    layout = w.layout()
    plan = plan_adaptive(layout, w.pec)
    arena = StateArena(layout, [0], dev, w.expert_tensors)
    st = StagingLayout.build(plan.assignments[0][0], arena, 0)
    staging = torch.empty(st.nbytes, dtype=torch.uint8, device=dev)
    lg = D.DEFAULT_CHUNK_LOG2
    table, total = st.descriptors(arena.base_address, staging.data_ptr(), chunk_log2=lg)
    dt = DeviceTable(table, total, dev, lg)
    host = None if args.no_drain else torch.empty(st.nbytes, dtype=torch.uint8, pin_memory=True)
    if host is not None:
        host.copy_(staging)  # first touch of the pinned pages
    compute = torch.cuda.current_stream(dev)
    prio_streams = {int(p): torch.cuda.Stream(device=dev, priority=int(p))
                    for p in args.priorities.split(",")}
    pack_s = prio_streams[int(args.priorities.split(",")[0])]
    copy_s = torch.cuda.Stream(device=dev)
    entries = st.entries

    def pack(engine, stream):
        if ENGINES[engine] is None:
            with torch.cuda.stream(stream):
                for e in entries:
                    staging[e.stage_offset:e.stage_offset + e.nbytes].copy_(
                        arena.buffer[e.src_offset:e.src_offset + e.nbytes], non_blocking=True)
        else:
            D.pack(dt.tensor, dt.n, dt.total_chunks, lg, ENGINES[engine], stream=stream)

    # pack alone
    alone = {}
    for eng in args.engines.split(","):
        ts = []
        for i in range(8):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(pack_s)
            pack(eng, pack_s)
            b.record(pack_s)
            b.synchronize()
            if i >= 3:
                ts.append(a.elapsed_time(b))
        alone[eng] = round(statistics.median(ts), 3)

    a_ = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
    b_ = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
    c_ = torch.empty(8192, 8192, device=dev, dtype=torch.bfloat16)
    words = arena.buffer.view(torch.int32)
    for _ in range(3):
        torch.matmul(a_, b_, out=c_)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        torch.matmul(a_, b_, out=c_)
    e1.record()
    e1.synchronize()
    n_gemm = max(1, round(100.0 / (e0.elapsed_time(e1) / 10)))

    def run(engine, pack_s=pack_s):
        torch.cuda.synchronize()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        pend, drained, packs = None, None, []
        t0.record(compute)
        for it in range(1, args.iters + 1):
            for _ in range(n_gemm):
                torch.matmul(a_, b_, out=c_)
            if pend is not None:
                compute.wait_event(pend[1])
            words.add_(1)
            if engine != "none" and it % args.i_ckpt == 0:
                pack_s.wait_stream(compute)
                if drained is not None:
                    pack_s.wait_event(drained)
                ps, pe = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                ps.record(pack_s)
                pack(engine, pack_s)
                pe.record(pack_s)
                pend = (ps, pe)
                packs.append(pend)
                if host is not None:
                    copy_s.wait_event(pe)
                    with torch.cuda.stream(copy_s):
                        host.copy_(staging, non_blocking=True)
                    drained = torch.cuda.Event()
                    drained.record(copy_s)
        t1.record(compute)
        t1.synchronize()
        torch.cuda.synchronize()
        return t0.elapsed_time(t1) / args.iters, [a.elapsed_time(b) for a, b in packs]

    run("none")  # warm
    variants = [(e, p) for p in prio_streams for e in args.engines.split(",")]
    name = (lambda e, p: e if len(prio_streams) == 1 else f"{e}@prio{p}")  # noqa: E731
    engines = [name(e, p) for e, p in variants]
    base, per = [], {n: [] for n in engines}
    loop_pack = {n: [] for n in engines}
    alone = {name(e, p): alone[e] for e, p in variants}
    for _ in range(args.rounds):
        for e, p in variants:
            base.append(run("none")[0])
            ms, pk = run(e, prio_streams[p])
            per[name(e, p)].append(ms)
            loop_pack[name(e, p)] += pk
    none_ms = statistics.mean(base)
    out = {"workload": w.name, "payload_bytes": st.payload_bytes, "iters": args.iters,
           "rounds": args.rounds, "i_ckpt": args.i_ckpt, "drain": host is not None,
           "fb_gemms": n_gemm, "iter_ms_none": round(none_ms, 3),
           "iter_ms_none_runs": [round(x, 3) for x in base], "engines": {}}
    for e in engines:
        m = statistics.mean(per[e])
        out["engines"][e] = {"pack_ms_alone": alone[e],
                             "pack_GBps_alone": round(2 * st.payload_bytes / alone[e] / 1e6, 1),
                             "pack_ms_in_loop": round(statistics.mean(loop_pack[e]), 3),
                             "iter_ms": round(m, 3), "runs": [round(x, 3) for x in per[e]],
                             "exposed_ms_per_iter": round(m - none_ms, 3),
                             "exposed_ms_per_checkpoint": round((m - none_ms) * args.i_ckpt, 2)}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
