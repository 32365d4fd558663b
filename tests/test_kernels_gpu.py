"""Parity of the sm_100a kernels (through the C ABI) against the CPU oracle."""

import numpy as np
import pytest

from conftest import make_layout
from oracle import pec_oracle as O

pytestmark = pytest.mark.gpu


# ---------------------------------------------------------------------------
# (a) token histogram
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("L,n,E", [(1, 1, 1), (4, 4096 * 2, 8), (6, 16384 * 2, 8),
                                   (12, 3000, 16), (32, 32768, 8), (3, 100003, 64),
                                   (2, 77, 4096), (2, 0, 8)])
def test_token_hist_matches_bincount_with_cap(dev, L, n, E):
    import torch
    from paper_2408_04307_b200 import device as D
    rng = np.random.default_rng(L * 1000 + E)
    counters = torch.zeros((2, L, E), dtype=torch.int64, device=dev)
    delivered = torch.zeros((L, E), dtype=torch.int64, device=dev)
    scratch = torch.zeros(L * E + 1, dtype=torch.int32, device=dev)
    want = np.zeros((L, E), dtype=np.int64)
    for it in range(3):
        # skewed ids with some out-of-range (dropped) entries
        ids = np.minimum(rng.zipf(1.3, size=(L, n)) - 1, E + 2).astype(np.int32)
        ids[rng.random((L, n)) < 0.01] = -1
        cap = np.array([O.capacity(1.25, n, E) for _ in range(L)], dtype=np.int64)
        cap[0] = max(1, cap[0] // 3)
        D.token_hist(torch.from_numpy(ids).to(dev), counters, scratch,
                     cap=torch.from_numpy(cap).to(dev), delivered=delivered)
        want += O.route_counts(ids, E, cap)
    torch.cuda.synchronize()
    assert np.array_equal(counters[0].cpu().numpy(), want)
    assert np.array_equal(counters[1].cpu().numpy(), want)
    assert np.array_equal(delivered.cpu().numpy(), want)
    assert int(scratch.abs().sum()) == 0  # left zeroed for the next call


def test_token_hist_accepts_int64_ids(dev):
    """torch.topk returns int64 indices: pec_token_hist_i64 counts them
    directly -- equal to the int32 path, and ids outside [0, E) in any width
    (negative, >= E, >= 2^31) are dropped, never aliased into range."""
    import torch
    from paper_2408_04307_b200 import device as D
    rng = np.random.default_rng(64)
    L, n, E = 3, 50_000, 16
    ids = rng.integers(0, E, size=(L, n)).astype(np.int64)
    ids[0, :7] = [-1, E, 2 ** 31 + 3, 2 ** 32 + 5, -(2 ** 40), 2 ** 33, E - 1]
    cap = np.array([O.capacity(1.25, n, E)] * L, dtype=np.int64)
    out = []
    for dt in (torch.int64, torch.int32):
        t = torch.from_numpy(ids).to(dev)
        if dt == torch.int32:
            t = torch.where((t >= 0) & (t < E), t, torch.full_like(t, -1)).to(torch.int32)
        counters = torch.zeros((1, L, E), dtype=torch.int64, device=dev)
        scratch = torch.zeros(L * E + 1, dtype=torch.int32, device=dev)
        D.token_hist(t, counters, scratch, cap=torch.from_numpy(cap).to(dev))
        out.append(counters[0].cpu().numpy())
    assert np.array_equal(out[0], out[1])
    clean = np.where((ids >= 0) & (ids < E), ids, -1)
    assert np.array_equal(out[0], O.route_counts(clean, E, cap))
    # [L, tokens, top_k] (stacked topk indices) is accepted as is
    counters = torch.zeros((1, L, E), dtype=torch.int64, device=dev)
    scratch = torch.zeros(L * E + 1, dtype=torch.int32, device=dev)
    D.token_hist(torch.from_numpy(ids).to(dev).view(L, n // 2, 2), counters, scratch,
                 cap=torch.from_numpy(cap).to(dev))
    assert np.array_equal(counters[0].cpu().numpy(), out[0])


def test_token_hist_reproduces_reference_zipf_routing(dev):
    """Explicit ids drawn from the reference's PCG64 Zipf stream, counted on
    device, equal the reference route_tokens counts (golden)."""
    import json
    import torch
    from conftest import GOLDEN
    from paper_2408_04307_b200 import device as D
    g = json.loads((GOLDEN / "routing.json").read_text())
    for case in g["zipf"]:
        L, E, total = case["layers"], case["experts"], case["total"]
        ids = np.stack([O.zipf_router_ids(case["seed"], case["iteration"], m, E, total,
                                          case["s"]) for m in range(L)])
        cap = O.capacity(case["capacity_factor"], total, E)
        counters = torch.zeros((1, L, E), dtype=torch.int64, device=dev)
        scratch = torch.zeros(L * E + 1, dtype=torch.int32, device=dev)
        capt = None if cap is None else torch.full((L,), cap, dtype=torch.int64, device=dev)
        D.token_hist(torch.from_numpy(ids).to(dev), counters, scratch, cap=capt)
        assert counters[0].cpu().tolist() == case["counts"], case


# ---------------------------------------------------------------------------
# (b) selection
# ---------------------------------------------------------------------------

def test_select_sequential_matches_window(dev):
    import torch
    from paper_2408_04307_b200 import device as D
    for E in (1, 3, 4, 8, 16, 64):
        for width in sorted({1, 2, 3, E // 2 or 1, E, E + 1}):
            for stride in sorted({0, 1, 2, 3, E}):
                for c in (0, 1, 5, 17, 1000003):
                    L = 7
                    w = min(width, E)
                    out = torch.full((L, w), -7, dtype=torch.int32, device=dev)
                    D.select_sequential(c, L, E, width, stride, out)
                    got = out.cpu().tolist()
                    want = [O.select_window(c, m, E, width, stride) for m in range(L)]
                    assert got == want, (E, width, stride, c)


@pytest.mark.parametrize("E", [1, 4, 8, 16, 33, 256, 4096])
def test_select_load_aware_ties_pools_and_reset(dev, E):
    import torch
    from paper_2408_04307_b200 import device as D
    rng = np.random.default_rng(E)
    L = 9 if E <= 256 else 3
    for trial in range(20 if E <= 256 else 4):
        hi = 3 if trial % 2 else 10**12  # many ties vs. wide range
        snap = rng.integers(0, hi, size=(L, E)).astype(np.int64)
        pers = rng.integers(0, hi, size=(L, E)).astype(np.int64)
        k_s = int(rng.integers(1, E + 1))
        k_p = int(rng.integers(1, k_s + 1))
        ss, ps, snap_after, pers_after = O.two_tier_load_aware(snap, pers, k_s, k_p)
        ds, dp = torch.from_numpy(snap).to(dev), torch.from_numpy(pers).to(dev)
        out_s = torch.empty((L, k_s), dtype=torch.int32, device=dev)
        out_p = torch.empty((L, k_p), dtype=torch.int32, device=dev)
        D.select_load_aware(ds, k_s, out_s, zero_selected=True)
        D.select_load_aware(dp, k_p, out_p, pool=out_s, zero_selected=True)
        assert out_s.cpu().tolist() == ss
        assert out_p.cpu().tolist() == ps
        assert np.array_equal(ds.cpu().numpy(), snap_after)
        assert np.array_equal(dp.cpu().numpy(), pers_after)


@pytest.mark.parametrize("E", [8, 300, 4096])
def test_select_load_aware_pools_with_duplicates_and_invalid_ids(dev, E):
    """Pool entries may repeat or fall outside [0, E) (padding -1 of a
    shorter selection): the candidates are the distinct valid ids, exactly
    as the reference's pool semantics (selector.py:91-100, oracle)."""
    import torch
    from paper_2408_04307_b200 import device as D
    rng = np.random.default_rng(E + 7)
    L, P = 4, 24
    counts = rng.integers(0, 5, size=(L, E)).astype(np.int64)
    pool = rng.integers(-3, E + 3, size=(L, P)).astype(np.int32)
    pool[:, 1] = pool[:, 0]                       # a duplicate in every row
    for k in (1, 3, P):
        out = torch.empty((L, k), dtype=torch.int32, device=dev)
        dc = torch.from_numpy(counts).to(dev)
        D.select_load_aware(dc, k, out, pool=torch.from_numpy(pool).to(dev), zero_selected=True)
        got = out.cpu().tolist()
        after = counts.copy()
        for m in range(L):
            want = O.select_load_aware(counts[m], k, pool=pool[m].tolist())
            assert [e for e in got[m] if e >= 0] == want, (m, k)
            assert got[m][len(want):] == [-1] * (k - len(want))
            after[m, want] = 0
        assert np.array_equal(dc.cpu().numpy(), after)


def test_select_load_aware_golden(dev):
    import json
    import torch
    from conftest import GOLDEN
    from paper_2408_04307_b200 import device as D
    g = json.loads((GOLDEN / "selection.json").read_text())
    for case in g["load_aware"]:
        counts = torch.tensor([case["counts"]], dtype=torch.int64, device=dev)
        k = case["k"]
        out = torch.empty((1, k), dtype=torch.int32, device=dev)
        pool = None
        if case["pool"] is not None:
            pool = torch.tensor([case["pool"]], dtype=torch.int32, device=dev)
        D.select_load_aware(counts, k, out, pool=pool)
        got = [e for e in out.cpu().tolist()[0] if e >= 0]
        assert got == case["selected"], case


# ---------------------------------------------------------------------------
# (c)/(d) pack and unpack
# ---------------------------------------------------------------------------

def _random_copies(rng, state_size, n, max_len, congruent):
    copies, pos = [], 0
    for _ in range(n):
        ln = int(rng.integers(0, max_len))
        src = int(rng.integers(0, state_size - ln))
        if congruent:
            dst = pos + ((src - pos) % 256)
        else:
            dst = pos + int(rng.integers(0, 64))
        copies.append((src, dst, ln))
        pos = dst + ln
    return copies, pos


@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("chunk_log2", [12, 15, 18])
@pytest.mark.parametrize("congruent", [True, False])
def test_pack_unpack_random_ranges(dev, mode, chunk_log2, congruent):
    import torch
    from paper_2408_04307_b200 import device as D
    rng = np.random.default_rng(chunk_log2 * 10 + mode + (100 if congruent else 0))
    size = 8 << 20
    state = torch.randint(0, 256, (size,), dtype=torch.uint8, device=dev)
    copies, stage_size = _random_copies(rng, size, 300, 200_000, congruent)
    copies += [(5, stage_size + 3, 0), (size - 17, stage_size + 7, 17)]
    stage_size += 7 + 17
    staging = torch.zeros(stage_size + 64, dtype=torch.uint8, device=dev)
    table = np.zeros(len(copies), dtype=D.DESC_DTYPE)
    for i, (s, t, n) in enumerate(copies):
        table[i] = (state.data_ptr() + s, staging.data_ptr() + t, n, 0)
    total = D.plan_chunks(table, chunk_log2)
    dt = torch.from_numpy(table.view(np.uint8).copy()).view(torch.int64).to(dev)
    D.pack(dt, len(table), total, chunk_log2, mode)
    torch.cuda.synchronize()
    host_state = state.cpu().numpy()
    want = O.pack(host_state, copies, stage_size + 64)
    assert np.array_equal(staging.cpu().numpy(), want)

    # unpack into a zeroed state image: exactly the copied ranges come back
    back = torch.zeros_like(state)
    rtable = table.copy()
    for i, (s, t, n) in enumerate(copies):
        rtable[i]["src"], rtable[i]["dst"] = staging.data_ptr() + t, back.data_ptr() + s
    total = D.plan_chunks(rtable, chunk_log2)
    rt = torch.from_numpy(rtable.view(np.uint8).copy()).view(torch.int64).to(dev)
    D.unpack(rt, len(rtable), total, chunk_log2, mode)
    torch.cuda.synchronize()
    want_back = O.unpack(want, copies, np.zeros(size, dtype=np.uint8))
    assert np.array_equal(back.cpu().numpy(), want_back)


@pytest.mark.parametrize("mode", [1, 2])
def test_pack_plan_phases_bit_exact(dev, mode):
    """Every phase of an adaptive K=1 plan on a 2-EP-group layout with an odd
    expert size (byte-granular weight parts) packs bit-exactly."""
    import torch
    from paper_2408_04307_b200 import PecConfig, plan_adaptive, plan_equal
    from paper_2408_04307_b200.arena import StateArena
    from paper_2408_04307_b200.staging import DeviceTable, StagingLayout
    from paper_2408_04307_b200 import device as D
    layout = make_layout(n_experts=4, dp=4, ep=2, epp=100_001, p_ne=30_001, other=37,
                         modules=(("a", 10_000), ("b", 10_001), ("c", 10_000)))
    arena = StateArena(layout, ranks=range(4), device=dev)
    host_state = arena.buffer.cpu().numpy()
    for plan in (plan_adaptive(layout, PecConfig(k_pec=1)),
                 plan_equal(layout, PecConfig(k_pec=2, k_snapshot=2, k_persist=1))):
        for phase in plan.assignments:
            for rank, ranges in phase.items():
                st = StagingLayout.build(ranges, arena, rank)
                staging = torch.zeros(st.nbytes + 1, dtype=torch.uint8, device=dev)
                table, total = st.descriptors(arena.base_address, staging.data_ptr())
                dtab = DeviceTable(table, total, dev)
                D.pack(dtab.tensor, dtab.n, dtab.total_chunks, mode=mode)
                torch.cuda.synchronize()
                got = staging.cpu().numpy()
                copies = [(e.src_offset, e.stage_offset, e.nbytes) for e in st.entries]
                assert np.array_equal(got, O.pack(host_state, copies, st.nbytes + 1))
                assert st.payload_bytes == plan.workload_bytes[plan.assignments.index(phase)][rank]


@pytest.mark.parametrize("strategy,shape", [("equal_pec", "split"), ("baseline", "split"),
                                            ("equal_pec", "many")])
def test_device_plan_expansion_matches_host_plan(dev, strategy, shape):
    """pec_expand_plan + pec_pack_indirect == host build_phase_assignment +
    StagingLayout + oracle pack, for random selections on a 2-EP-group layout
    (byte-split expert weights, every rank) and on a 64-expert layout whose
    template spans several scan tiles."""
    import torch
    from paper_2408_04307_b200 import build_phase_assignment
    from paper_2408_04307_b200 import device as D
    from paper_2408_04307_b200.arena import StateArena
    from paper_2408_04307_b200.staging import PlanTemplate, StagingLayout
    if shape == "split":
        layout = make_layout(n_experts=8, dp=4, ep=2, n_layers=3, epp=20_001, p_ne=3_001,
                             other=9, modules=(("a", 1000), ("b", 1001), ("c", 1000)))
        L, E, ranks = 3, 8, range(4)
    else:
        layout = make_layout(n_experts=64, dp=1, ep=1, gpus_per_node=1, n_layers=12, epp=333,
                             p_ne=3_001, modules=(("a", 1000), ("b", 1001), ("c", 1000)))
        L, E, ranks = 12, 64, range(1)
    rng = np.random.default_rng(7)
    for rank in ranks:
        arena = StateArena(layout, [rank], dev)
        host_state = arena.buffer.cpu().numpy()
        tmpl = PlanTemplate(layout, arena, rank, strategy, dev)
        staging = torch.zeros(tmpl.max_bytes + 512, dtype=torch.uint8, device=dev)
        table = torch.empty(max(1, tmpl.n) * 4, dtype=torch.int64, device=dev)
        totals = torch.zeros(2, dtype=torch.int64, device=dev)
        for trial in range(6):
            k = int(rng.integers(1, E + 1))
            sel = np.stack([np.sort(rng.choice(E, size=k, replace=False)) for _ in range(L)])
            sel_d = torch.from_numpy(sel.astype(np.int32)).to(dev)
            staging.zero_()
            D.expand_plan(tmpl.tensor, tmpl.n, sel_d, arena.base_address, staging.data_ptr(),
                          table, totals)
            D.pack_indirect(table, tmpl.n, tmpl.max_chunks(), totals)
            torch.cuda.synchronize()
            due = {m: frozenset(int(x) for x in sel[m]) for m in range(L)}
            ranges = build_phase_assignment(layout, due, strategy).get(rank, ())
            st = StagingLayout.build(ranges, arena, rank)
            assert tuple(a for a in ranges if a.stop > a.start) == tmpl.select(due)
            assert int(totals[1]) == st.nbytes
            _, nch = st.descriptors(0, 0)
            assert int(totals[0]) == nch
            copies = [(e.src_offset, e.stage_offset, e.nbytes) for e in st.entries]
            want = O.pack(host_state, copies, tmpl.max_bytes + 512)
            assert np.array_equal(staging.cpu().numpy(), want), (rank, trial)
        del arena


@pytest.mark.parametrize("congruent", [True, False])
def test_pack_crc_copies_and_checksums_every_entry(dev, congruent):
    """pec_pack_crc: staging bit-exact vs the oracle pack, and each entry's
    CRC-32C equals the oracle's (C restatement of store.crc32c) over the
    entry's source bytes — aligned multi-chunk entries, byte-granular and
    incongruent ranges, partial chunks and empty entries."""
    import torch
    from paper_2408_04307_b200 import device as D
    rng = np.random.default_rng(99 + congruent)
    size = 24 << 20
    state = torch.randint(0, 256, (size,), dtype=torch.uint8, device=dev)
    copies, pos = [], 0
    lens = [0, 1, 15, 16, 17, 4095, 32768, 32769, 65536, 3 * 32768 + 5, 5 << 20, 100_003]
    for ln in lens + [int(x) for x in rng.integers(0, 300_000, 20)]:
        src = int(rng.integers(0, size - ln)) if ln < size else 0
        if rng.random() < 0.5:
            src &= ~255  # whole-unit style, 256-aligned
        dst = pos + ((src - pos) % 256) if congruent else pos + int(rng.integers(0, 64))
        copies.append((src, dst, ln))
        pos = dst + ln
    staging = torch.zeros(pos + 64, dtype=torch.uint8, device=dev)
    table = np.zeros(len(copies), dtype=D.DESC_DTYPE)
    for i, (s, t, n) in enumerate(copies):
        table[i] = (state.data_ptr() + s, staging.data_ptr() + t, n, 0)
    total = D.plan_chunks(table, 15)
    dt = torch.from_numpy(table.view(np.uint8).copy()).view(torch.int64).to(dev)
    chunk = torch.empty(D.crc_scratch_words(total), dtype=torch.int32, device=dev)
    entry = torch.empty(len(copies), dtype=torch.int32, device=dev)
    D.pack_crc(dt, len(copies), total, chunk, entry)
    torch.cuda.synchronize()
    host = state.cpu().numpy()
    assert np.array_equal(staging.cpu().numpy(), O.pack(host, copies, pos + 64))
    got = entry.cpu().numpy().view(np.uint32)
    for (s, _, n), c in zip(copies, got):
        assert int(c) == O.crc32c(host[s:s + n]), (s, n)


def test_crc_device_checksums_without_writing(dev):
    """pec_crc_device: per-entry CRC-32C of device ranges (aligned multi-chunk,
    byte-granular, partial chunks, empty) equal to the oracle's, and nothing
    is written anywhere (dst is ignored)."""
    import torch
    from paper_2408_04307_b200 import device as D
    rng = np.random.default_rng(5)
    size = 16 << 20
    state = torch.randint(0, 256, (size,), dtype=torch.uint8, device=dev)
    before = state.clone()
    ranges = [(0, 0), (3, 1), (256, 32768), (4096, 3 * 32768 + 7), (17, 100_003)]
    ranges += [(int(rng.integers(0, size // 2)), int(rng.integers(0, 2 << 20))) for _ in range(12)]
    table = np.zeros(len(ranges), dtype=D.DESC_DTYPE)
    for i, (s_, n) in enumerate(ranges):
        table[i] = (state.data_ptr() + s_, 0, n, 0)
    total = D.plan_chunks(table, 15)
    dt = torch.from_numpy(table.view(np.uint8).copy()).view(torch.int64).to(dev)
    chunk = torch.empty(D.crc_scratch_words(total), dtype=torch.int32, device=dev)
    entry = torch.empty(len(ranges), dtype=torch.int32, device=dev)
    D.crc_device(dt, len(ranges), total, chunk, entry)
    torch.cuda.synchronize()
    assert torch.equal(state, before)
    host = state.cpu().numpy()
    got = entry.cpu().numpy().view(np.uint32)
    for (s_, n), c in zip(ranges, got):
        assert int(c) == O.crc32c(host[s_:s_ + n]), (s_, n)


def test_pack_crc_very_long_entries_use_every_power_table(dev):
    """Entries long enough that the chunk shifts need all three power tables
    (> 65536 whole 32 KiB chunks after a chunk: a 2 GiB+ entry), plus entries
    of exactly k x 32 KiB, k x 32 KiB + 1 and 257 chunks: device CRCs equal the
    host SSE4.2 CRC-32C of the same bytes and the copies are exact."""
    import torch
    from paper_2408_04307_b200 import device as D
    lens = [(1 << 31) + 12345, 32768 * 3, 32768 * 3 + 1, 32768 * 257 - 7, 1]
    size = sum(lens) + 256 * len(lens)
    state = torch.empty(size, dtype=torch.uint8, device=dev)
    state.view(torch.int32)[: size // 4].random_()
    staging = torch.empty(size + 256, dtype=torch.uint8, device=dev)
    table = np.zeros(len(lens), dtype=D.DESC_DTYPE)
    pos = 0
    for i, n in enumerate(lens):
        table[i] = (state.data_ptr() + pos, staging.data_ptr() + pos + 128, n, 0)
        pos += n + 256
    total = D.plan_chunks(table, 15)
    dt = torch.from_numpy(table.view(np.uint8).copy()).view(torch.int64).to(dev)
    chunk = torch.empty(D.crc_scratch_words(total), dtype=torch.int32, device=dev)
    entry = torch.empty(len(lens), dtype=torch.int32, device=dev)
    D.pack_crc(dt, len(lens), total, chunk, entry, 15)
    torch.cuda.synchronize()
    got = entry.cpu().numpy().view(np.uint32)
    pos = 0
    for i, n in enumerate(lens):
        src = state[pos:pos + n]
        assert torch.equal(staging[pos + 128:pos + 128 + n], src), n
        assert int(got[i]) == D.crc32c(src.cpu().numpy()), n
        pos += n + 256
    del state, staging, chunk
    torch.cuda.empty_cache()


def test_c_abi_device_entry_points_from_plain_c(dev, tmp_path):
    """pack / unpack / sequential selection / histogram called from a plain C
    program through include/pec.h (tests/c/abi_check.c, CUDA runtime)."""
    import subprocess
    from conftest import build_abi_check
    exe = build_abi_check(tmp_path, gpu=True)
    res = subprocess.run([str(exe), "gpu"], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "0 failure(s)" in res.stdout
