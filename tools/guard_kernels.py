"""Bounds evidence for every libpec kernel without compute-sanitizer.

compute-sanitizer is closed on the B200 pool (runs under it left GPUs
needing a reset), so out-of-bounds behaviour is checked two ways instead:

* every buffer a kernel writes is allocated with 64 KiB guard bands on both
  sides filled with a pattern, and the bands are verified after each launch
  (an overrun or underrun of any output shows up as a changed guard byte);
* run with PEC_LIB=debug, the library is the build with device-side
  invariant checks compiled in (PEC_DCHECK: descriptor index in range,
  chunk inside its descriptor, pipeline counters, selection output slots,
  TMA piece sizes), which trap on a violation.

    PEC_LIB=debug python tools/guard_kernels.py

Covers token_hist (int32 + int64 ids, dropped ids, cap), both selections
(pool, reset), the vector and TMA bulk pack/unpack engines (aligned,
byte-granular and incongruent ranges, ranges ending flush with their
allocation), device plan expansion + pack_indirect, the CRC-computing pack
and pec_crc_device (full, partial and unaligned chunks, empty entries), and
checks every result against the oracle.  Prints one line per kernel family
and "guard-drive ok" at the end.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


GUARD = 64 << 10
PATTERN = 0xA5


def guarded(n, dtype, dev, fill=None):
    """(full, view): ``view`` has n elements, surrounded by GUARD bytes of
    PATTERN on both sides inside ``full``."""
    import torch
    esize = torch.empty(0, dtype=dtype).element_size()
    g = GUARD // esize
    full = torch.empty(n + 2 * g, dtype=dtype, device=dev)
    full.view(torch.uint8).fill_(PATTERN)
    view = full[g:g + n]
    if fill is not None:
        view.fill_(fill)
    return full, view


def check_guards(full, what: str) -> None:
    import torch
    torch.cuda.synchronize()
    b = full.view(torch.uint8)
    head, tail = b[:GUARD], b[b.numel() - GUARD:]
    bad = int((head != PATTERN).sum()) + int((tail != PATTERN).sum())
    assert bad == 0, f"{what}: {bad} guard bytes overwritten"


def main() -> int:
    import os
    import torch
    from paper_2408_04307_b200 import _build
    if os.environ.get("PEC_LIB") == "debug":
        _build.build_debug()          # (re)built in place when missing or stale
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
        cf, counts = guarded(2 * L * E, torch.int64, dev, 0)
        counts = counts.view(2, L, E)
        df, delivered = guarded(L * E, torch.int64, dev, 0)
        delivered = delivered.view(L, E)
        sf, scratch = guarded(L * E + 1, torch.int32, dev, 0)
        cap = torch.full((L,), 400, dtype=torch.int64, device=dev)
        D.token_hist(ids, counts, scratch, cap=cap, delivered=delivered)
        want = O.route_counts(ids.cpu().numpy(), E, [400] * L)
        assert np.array_equal(counts[0].cpu().numpy(), want)
        assert np.array_equal(delivered.cpu().numpy(), want)
        for f, w in ((cf, "counters"), (df, "delivered"), (sf, "hist scratch")):
            check_guards(f, w)
    print("token_hist ok")

    # -- selection ------------------------------------------------------------------
    of, out = guarded(L * 4, torch.int32, dev)
    out = out.view(L, 4)
    D.select_sequential(5, L, E, 4, 4, out)
    assert out.cpu().tolist() == [O.select_window(5, m, E, 4, 4) for m in range(L)]
    c = torch.from_numpy(rng.integers(0, 50, (L, E))).to(dev)
    host_c = c.cpu().numpy()
    D.select_load_aware(c, 4, out, zero_selected=True)
    snap = out.clone()
    assert out.cpu().tolist() == [O.select_load_aware(host_c[m], 4) for m in range(L)]
    of2, out2 = guarded(L * 2, torch.int32, dev)
    out2 = out2.view(L, 2)
    D.select_load_aware(c, 2, out2, pool=snap)
    check_guards(of, "selection")
    check_guards(of2, "pooled selection")
    print("selection ok")

    # -- pack / unpack engines -------------------------------------------------------
    size = 6 << 20
    stf, state = guarded(size, torch.uint8, dev)
    state.copy_(torch.randint(0, 256, (size,), dtype=torch.uint8, device=dev))
    host = state.cpu().numpy()
    for congruent in (True, False):
        copies, pos = [], 0
        for j, ln in enumerate([0, 1, 15, 17, 4095, 32768, 32769, 100_003, 1 << 20, 77_777]):
            # the last range ends flush with the end of the state view
            src = size - ln if j == 9 else int(rng.integers(0, size - ln))
            dst = pos + ((src - pos) % 256) if congruent else pos + int(rng.integers(0, 64))
            copies.append((src, dst, ln))
            pos = dst + ln
        sgf, staging = guarded(pos + 64, torch.uint8, dev, 0)
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
            check_guards(sgf, f"staging (mode {mode})")
        cgf, chunk = guarded(D.crc_scratch_words(total), torch.int32, dev)
        egf, entry = guarded(len(copies), torch.int32, dev)
        staging.zero_()
        D.pack_crc(dt, len(copies), total, chunk, entry)
        assert np.array_equal(staging.cpu().numpy(), want)
        for f, w in ((sgf, "staging (crc)"), (cgf, "chunk crc"), (egf, "entry crc")):
            check_guards(f, w)
        got = entry.cpu().numpy().view(np.uint32)
        for (s, _, m), cval in zip(copies, got):
            assert int(cval) == O.crc32c(host[s:s + m])
        D.crc_device(dt, len(copies), total, chunk, entry)
        assert np.array_equal(entry.cpu().numpy().view(np.uint32), got)
        check_guards(stf, "state (crc_device must not write)")
        # unpack: staging -> a wiped copy of the state
        bgf, back = guarded(size, torch.uint8, dev, 0)
        rt = np.zeros(len(copies), dtype=D.DESC_DTYPE)
        for i, (s, t, m) in enumerate(copies):
            rt[i] = (staging.data_ptr() + t, back.data_ptr() + s, m, 0)
        D.plan_chunks(rt, 15)
        rdt = torch.from_numpy(rt.view(np.uint8).copy()).view(torch.int64).to(dev)
        D.unpack(rdt, len(copies), total, 15, D.MODE_BULK)
        bh = back.cpu().numpy()
        for s, _, m in copies:
            assert np.array_equal(bh[s:s + m], host[s:s + m])
        check_guards(bgf, "unpack target")
    print("pack/unpack/pack_crc/crc_device ok")

    # -- device plan expansion + indirect pack ---------------------------------------
    layout = make_layout(n_experts=8, dp=4, ep=2, n_layers=3, epp=20_001, p_ne=3_001, other=9,
                         modules=(("a", 1000), ("b", 1001), ("c", 1000)))
    arena = StateArena(layout, [1], dev)
    hs = arena.buffer.cpu().numpy()
    tmpl = PlanTemplate(layout, arena, 1, "equal_pec", dev)
    sgf, staging = guarded(tmpl.max_bytes + 512, torch.uint8, dev, 0)
    tgf, table = guarded(max(1, tmpl.n) * 4, torch.int64, dev)
    ogf, totals = guarded(2, torch.int64, dev, 0)
    sel = np.stack([np.sort(rng.choice(8, size=3, replace=False)) for _ in range(3)])
    sel_d = torch.from_numpy(sel.astype(np.int32)).to(dev)
    D.expand_plan(tmpl.tensor, tmpl.n, sel_d, arena.base_address, staging.data_ptr(), table,
                  totals)
    D.pack_indirect(table, tmpl.n, tmpl.max_chunks(), totals)
    due = {m: frozenset(int(x) for x in sel[m]) for m in range(3)}
    st = StagingLayout.build(build_phase_assignment(layout, due, "equal_pec").get(1, ()), arena, 1)
    copies = [(e.src_offset, e.stage_offset, e.nbytes) for e in st.entries]
    assert np.array_equal(staging.cpu().numpy(), O.pack(hs, copies, tmpl.max_bytes + 512))
    cgf, chunk = guarded(D.crc_scratch_words(tmpl.max_chunks()), torch.int32, dev)
    egf, entry = guarded(tmpl.n, torch.int32, dev)
    D.pack_crc(table, tmpl.n, tmpl.max_chunks(), chunk, entry, totals_dev=totals)
    for f, w in ((sgf, "plan staging"), (tgf, "expanded table"), (ogf, "totals"),
                 (cgf, "chunk crc (indirect)"), (egf, "entry crc (indirect)")):
        check_guards(f, w)
    print("expand_plan/pack_indirect ok")
    print(f"guard-drive ok (library: {D.LIB_PATH.name})")
    return 0


if __name__ == "__main__":
    sys.exit(main())
