"""Time the copy engines on the Mixtral-shaped rank-0 phase-0 table
(measurement tool; GB/s of 2*S per launch, CUDA events, median of 20).

    python tools/pack_variants.py                 # pack: every engine variant + library baseline
    python tools/pack_variants.py --unpack-only   # restore direction only (for an ncu capture)

Pack variants are `pec_pack` modes (1 = LDG/STG vector engine, 2 = the
default TMA-bulk engine, 10-16 = ring-depth / piece-size / L2-hint variants);
unpack is `pec_unpack` mode 2 (staging -> state arena, the restore scatter),
checked bit-exact against the arena afterwards."""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def _median_ms(fn, reps=20, warm=3):
    import torch
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--modes", default="1,2,10,12,13,16")
    ap.add_argument("--unpack-only", action="store_true")
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
    gbps = lambda ms: round(2 * st.payload_bytes / (ms / 1e3) / 1e9, 1)  # noqa: E731
    out = {"payload_bytes": st.payload_bytes, "entries": len(st.entries)}
    modes = [] if args.unpack_only else [int(m) for m in args.modes.split(",")]
    for mode in modes:
        ms = _median_ms(lambda: D.pack(dt.tensor, dt.n, dt.total_chunks, lg, mode))
        e = st.entries[0]
        ok = torch.equal(staging[e.stage_offset:e.stage_offset + 4096],
                         arena.buffer[e.src_offset:e.src_offset + 4096])
        out[f"pack_mode{mode}"] = {"ms": round(ms, 4), "GBps": gbps(ms), "spot_ok": bool(ok)}

    # restore direction: staging -> arena.  Pack, wipe the ranges, unpack once
    # and compare; the timed unpacks then rewrite the same bytes.
    D.pack(dt.tensor, dt.n, dt.total_chunks, lg, D.MODE_BULK)
    for e in st.entries:
        arena.buffer[e.src_offset:e.src_offset + e.nbytes].zero_()
    D.unpack(dt.tensor, dt.n, dt.total_chunks, lg, D.MODE_BULK)
    ok = all(torch.equal(staging[e.stage_offset:e.stage_offset + e.nbytes],
                         arena.buffer[e.src_offset:e.src_offset + e.nbytes]) for e in st.entries)
    ms = _median_ms(lambda: D.unpack(dt.tensor, dt.n, dt.total_chunks, lg, D.MODE_BULK))
    out["unpack_mode2"] = {"ms": round(ms, 4), "GBps": gbps(ms), "bit_exact": bool(ok)}

    if not args.unpack_only:
        # library baseline: one cudaMemcpyAsync (torch copy_) per staged entry
        def memcpy_pack():
            for e in st.entries:
                staging[e.stage_offset:e.stage_offset + e.nbytes].copy_(
                    arena.buffer[e.src_offset:e.src_offset + e.nbytes])
        ms = _median_ms(memcpy_pack)
        out["cudaMemcpyAsync_per_entry"] = {"ms": round(ms, 4), "GBps": gbps(ms)}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
