"""Time pack-engine variants on the Mixtral-shaped rank-0 phase-0 table
(measurement tool; prints GB/s of 2*S per launch, CUDA events, 10 launches)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
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
    out = {}
    for lg in (15,):
        table, total = st.descriptors(arena.base_address, staging.data_ptr(), chunk_log2=lg)
        dt = DeviceTable(table, total, dev, lg)
        for mode in (1, 2, 10, 12, 13, 16):
            for _ in range(3):
                D.pack(dt.tensor, dt.n, dt.total_chunks, lg, mode)
            ts = []
            for _ in range(20):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                D.pack(dt.tensor, dt.n, dt.total_chunks, lg, mode)
                b.record()
                b.synchronize()
                ts.append(a.elapsed_time(b))
            ms = sorted(ts)[len(ts) // 2]
            out[f"lg{lg}_mode{mode}"] = {"ms": round(ms, 4),
                                         "GBps": round(2 * st.payload_bytes / (ms / 1e3) / 1e9, 1)}
            ok = torch.equal(staging[st.entries[0].stage_offset:st.entries[0].stage_offset + 4096],
                             arena.buffer[st.entries[0].src_offset:st.entries[0].src_offset + 4096])
            out[f"lg{lg}_mode{mode}"]["spot_ok"] = bool(ok)
    # library baseline: one cudaMemcpyAsync (torch copy_) per staged entry
    def memcpy_pack():
        for e in st.entries:
            staging[e.stage_offset:e.stage_offset + e.nbytes].copy_(
                arena.buffer[e.src_offset:e.src_offset + e.nbytes])
    for _ in range(3):
        memcpy_pack()
    ts = []
    for _ in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        memcpy_pack()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ms = sorted(ts)[len(ts) // 2]
    out["cudaMemcpyAsync_per_entry"] = {"ms": round(ms, 4), "entries": len(st.entries),
                                        "GBps": round(2 * st.payload_bytes / (ms / 1e3) / 1e9, 1)}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
