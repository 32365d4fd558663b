"""Drive every libpec kernel once on small inputs, for compute-sanitizer.

    compute-sanitizer --tool {memcheck,racecheck,synccheck,initcheck} \
        python tools/sanitize_kernels.py

Covers token_hist (int32 + int64 ids, dropped ids, cap), both selections
(pool, reset), the vector and TMA bulk pack/unpack engines (aligned,
byte-granular and incongruent ranges), device plan expansion +
pack_indirect, the CRC-computing pack and pec_crc_device (full, partial and
unaligned chunks, empty entries), and checks every result against the
oracle, so a clean sanitizer report is also a correct run.  Prints one line
per kernel family and "sanitize-drive ok" at the end.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def main() -> int:
    import torch
    from conftest import make_layout
    from oracle import pec_oracle as O
    from paper_2408_04307_b200 import build_phase_assignment
    from paper_2408_04307_b200 import device as D
    from paper_2408_04307_b200.arena import StateArena
    from paper_2408_04307_b200.staging import PlanTemplate, StagingLayout

    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(3)

    # -- token histogram ----------------------------------------------------------
    L, E, n = 3, 16, 5000
    for dtype in (torch.int32, torch.int64):
        ids = torch.from_numpy(rng.integers(-2, E + 3, (L, n))).to(dev, dtype)
        counts = torch.zeros((2, L, E), dtype=torch.int64, device=dev)
        delivered = torch.zeros((L, E), dtype=torch.int64, device=dev)
        scratch = torch.zeros(L * E + 1, dtype=torch.int32, device=dev)
        cap = torch.full((L,), 400, dtype=torch.int64, device=dev)
        D.token_hist(ids, counts, scratch, cap=cap, delivered=delivered)
        want = O.route_counts(ids.cpu().numpy(), E, [400] * L)
        assert np.array_equal(counts[0].cpu().numpy(), want)
        assert np.array_equal(delivered.cpu().numpy(), want)
    print("token_hist ok")

    # -- selection ------------------------------------------------------------------
    out = torch.empty((L, 4), dtype=torch.int32, device=dev)
    D.select_sequential(5, L, E, 4, 4, out)
    assert out.cpu().tolist() == [O.select_window(5, m, E, 4, 4) for m in range(L)]
    c = torch.from_numpy(rng.integers(0, 50, (L, E))).to(dev)
    host_c = c.cpu().numpy()
    D.select_load_aware(c, 4, out, zero_selected=True)
    snap = out.clone()
    assert out.cpu().tolist() == [O.select_load_aware(host_c[m], 4) for m in range(L)]
    out2 = torch.empty((L, 2), dtype=torch.int32, device=dev)
    D.select_load_aware(c, 2, out2, pool=snap)
    print("selection ok")

    # -- pack / unpack engines -------------------------------------------------------
    size = 6 << 20
    state = torch.randint(0, 256, (size,), dtype=torch.uint8, device=dev)
    host = state.cpu().numpy()
    for congruent in (True, False):
        copies, pos = [], 0
        for ln in [0, 1, 15, 17, 4095, 32768, 32769, 100_003, 1 << 20]:
            src = int(rng.integers(0, size - ln))
            dst = pos + ((src - pos) % 256) if congruent else pos + int(rng.integers(0, 64))
            copies.append((src, dst, ln))
            pos = dst + ln
        staging = torch.zeros(pos + 64, dtype=torch.uint8, device=dev)
        table = np.zeros(len(copies), dtype=D.DESC_DTYPE)
        for i, (s, t, m) in enumerate(copies):
            table[i] = (state.data_ptr() + s, staging.data_ptr() + t, m, 0)
        total = D.plan_chunks(table, 15)
        dt = torch.from_numpy(table.view(np.uint8).copy()).view(torch.int64).to(dev)
        want = O.pack(host, copies, pos + 64)
        for mode in (D.MODE_VEC, D.MODE_BULK):
            staging.zero_()
            D.pack(dt, len(copies), total, 15, mode)
            assert np.array_equal(staging.cpu().numpy(), want), (congruent, mode)
        chunk = torch.empty(D.crc_scratch_words(total), dtype=torch.int32, device=dev)
        entry = torch.empty(len(copies), dtype=torch.int32, device=dev)
        staging.zero_()
        D.pack_crc(dt, len(copies), total, chunk, entry)
        assert np.array_equal(staging.cpu().numpy(), want)
        got = entry.cpu().numpy().view(np.uint32)
        for (s, _, m), cval in zip(copies, got):
            assert int(cval) == O.crc32c(host[s:s + m])
        D.crc_device(dt, len(copies), total, chunk, entry)
        assert np.array_equal(entry.cpu().numpy().view(np.uint32), got)
        # unpack: staging -> a wiped copy of the state
        back = torch.zeros_like(state)
        rt = np.zeros(len(copies), dtype=D.DESC_DTYPE)
        for i, (s, t, m) in enumerate(copies):
            rt[i] = (staging.data_ptr() + t, back.data_ptr() + s, m, 0)
        D.plan_chunks(rt, 15)
        rdt = torch.from_numpy(rt.view(np.uint8).copy()).view(torch.int64).to(dev)
        D.unpack(rdt, len(copies), total, 15, D.MODE_BULK)
        bh = back.cpu().numpy()
        for s, _, m in copies:
            assert np.array_equal(bh[s:s + m], host[s:s + m])
    print("pack/unpack/pack_crc/crc_device ok")

    # -- device plan expansion + indirect pack ---------------------------------------
    layout = make_layout(n_experts=8, dp=4, ep=2, n_layers=3, epp=20_001, p_ne=3_001, other=9,
                         modules=(("a", 1000), ("b", 1001), ("c", 1000)))
    arena = StateArena(layout, [1], dev)
    hs = arena.buffer.cpu().numpy()
    tmpl = PlanTemplate(layout, arena, 1, "equal_pec", dev)
    staging = torch.zeros(tmpl.max_bytes + 512, dtype=torch.uint8, device=dev)
    table = torch.empty(max(1, tmpl.n) * 4, dtype=torch.int64, device=dev)
    totals = torch.zeros(2, dtype=torch.int64, device=dev)
    sel = np.stack([np.sort(rng.choice(8, size=3, replace=False)) for _ in range(3)])
    sel_d = torch.from_numpy(sel.astype(np.int32)).to(dev)
    D.expand_plan(tmpl.tensor, tmpl.n, sel_d, arena.base_address, staging.data_ptr(), table,
                  totals)
    D.pack_indirect(table, tmpl.n, tmpl.max_chunks(), totals)
    due = {m: frozenset(int(x) for x in sel[m]) for m in range(3)}
    st = StagingLayout.build(build_phase_assignment(layout, due, "equal_pec").get(1, ()), arena, 1)
    copies = [(e.src_offset, e.stage_offset, e.nbytes) for e in st.entries]
    assert np.array_equal(staging.cpu().numpy(), O.pack(hs, copies, tmpl.max_bytes + 512))
    chunk = torch.empty(D.crc_scratch_words(tmpl.max_chunks()), dtype=torch.int32, device=dev)
    entry = torch.empty(tmpl.n, dtype=torch.int32, device=dev)
    D.pack_crc(table, tmpl.n, tmpl.max_chunks(), chunk, entry, totals_dev=totals)
    torch.cuda.synchronize()
    print("expand_plan/pack_indirect ok")
    print("sanitize-drive ok")
    return 0


if __name__ == "__main__":
    sys.exit(main())
