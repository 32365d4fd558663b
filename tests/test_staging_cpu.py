"""Host-side staging layout and device-plan template properties (CPU)."""

import json
import random

import pytest

from conftest import GOLDEN
from paper_2408_04307_b200 import ClusterSpec, ModelSpec, ParallelSpec, build_layout
from paper_2408_04307_b200 import build_phase_assignment
from paper_2408_04307_b200.arena import PeerSlots, arena_slots
from paper_2408_04307_b200.staging import STAGE_ALIGN, PlanTemplate, StagingLayout

SMALL = json.loads((GOLDEN / "plans.json").read_text())["small"]


def _layout(case):
    m = case["model"]
    model = ModelSpec(**{**m, "non_expert_modules": tuple(map(tuple, m["non_expert_modules"]))})
    gpn = case["gpus_per_node"]
    return build_layout(model, ParallelSpec(case["dp"], case["ep"]),
                        ClusterSpec(num_nodes=case["dp"] // gpn, gpus_per_node=gpn))


@pytest.mark.parametrize("i", range(0, len(SMALL), 3))
def test_staging_layout_invariants(i):
    layout = _layout(SMALL[i])
    due = {int(m): frozenset(v) for m, v in SMALL[i]["due"].items()}
    for strat in ("baseline", "equal_pec", "adaptive_pec"):
        phase = build_phase_assignment(layout, due, strat)
        for r, ranges in phase.items():
            slots = PeerSlots(layout, r)
            st = StagingLayout.build(ranges, slots, r)
            prev_end = 0
            for e in st.entries:
                assert e.stage_offset >= prev_end                          # ordered, no overlap
                assert e.stage_offset - prev_end < STAGE_ALIGN             # bounded padding
                assert (e.stage_offset - e.src_offset) % STAGE_ALIGN == 0  # congruent source
                prev_end = e.stage_offset + e.nbytes
            assert st.nbytes == prev_end
            # (the reference admits negative "other" shards when other_states_bytes
            # is tiny vs dp: ceil split 5 over 4 -> 2,2,2,-1; they carry no bytes)
            assert st.payload_bytes == sum(max(0, a.stop - a.start) for a in ranges)
            table, total = st.descriptors(1 << 40, 1 << 41, chunk_log2=12)
            assert int(table["nbytes"].sum()) == st.payload_bytes
            assert total == sum(-(-int(n) // 4096) for n in table["nbytes"])


@pytest.mark.parametrize("i", range(len(SMALL)))
def test_plan_template_selects_exactly_the_planner_ranges(i):
    """The device-plan template filtered by any due set equals the reference
    planner's ranges for that rank (equal/baseline placement)."""
    layout = _layout(SMALL[i])
    rng = random.Random(i)
    n = layout.model.experts_per_layer
    for strat in ("equal_pec", "baseline"):
        for r in range(layout.n_ranks):
            tmpl = PlanTemplate(layout, PeerSlots(layout, r), r, strat, "cpu")
            for _ in range(4):
                due = {m: frozenset(rng.sample(range(n), rng.randint(0, n)))
                       for m in range(layout.model.num_moe_layers)}
                want = tuple(a for a in build_phase_assignment(layout, due, strat).get(r, ())
                             if a.stop > a.start)
                assert tmpl.select(due) == want


def test_arena_slots_cover_exactly_the_resident_units():
    layout = _layout(SMALL[5])
    for r in range(layout.n_ranks):
        got = set(arena_slots(layout, [r]))
        want = {u.key for u in layout.units if r in u.replica_ranks and u.size_bytes}
        assert got == want


@pytest.mark.parametrize("seed", range(6))
def test_split_table_covers_each_copy_exactly_once(seed):
    """The pipelined-drain split (staging.split_table): the segments' copies
    are the original copies cut at the staging offsets, each inside its
    segment's [lo, hi), tiling every original byte exactly once."""
    import numpy as np
    from paper_2408_04307_b200.device import DESC_DTYPE, plan_chunks
    from paper_2408_04307_b200.staging import drain_cuts, split_table
    rng = random.Random(seed)
    base, pos, rows = 1 << 40, 0, []
    for _ in range(rng.randint(1, 40)):
        n = rng.choice([1, 7, 4096, 65536, rng.randint(1, 3 << 20)])
        rows.append((rng.randrange(1 << 30) * 16, base + pos, n))
        pos += (n + 255) // 256 * 256
    table = np.zeros(len(rows), dtype=DESC_DTYPE)
    for i, (s, d, n) in enumerate(rows):
        table[i] = (s, d, n, 0)
    plan_chunks(table, 15)
    cuts = drain_cuts(pos, first=rng.choice([4096, 65536, 1 << 20]), growth=rng.choice([2, 4]))
    assert all(0 < c < pos for c in cuts) and cuts == sorted(cuts)
    segs = split_table(table, base, cuts, 15)
    assert [lo for _, _, lo, _ in segs] == [0, *cuts]
    assert [hi for _, _, _, hi in segs] == [*cuts, None]
    pieces = []
    for sub, total, lo, hi in segs:
        chk = sub.copy()
        assert plan_chunks(chk, 15) == total
        assert (chk["first_chunk"] == sub["first_chunk"]).all()
        for s, d, n, _ in sub.tolist():
            assert n > 0 and d - base >= lo and (hi is None or d - base + n <= hi)
            pieces.append((s, d, n))
    # re-join: per original row, its pieces are contiguous, in order, and complete
    k = 0
    for s, d, n in rows:
        off = 0
        while off < n:
            ps, pd, pn = pieces[k]
            assert (ps, pd) == (s + off, d + off)
            off += pn
            k += 1
        assert off == n
    assert k == len(pieces)


@pytest.mark.parametrize("seed", range(20))
def test_spans_cover_agrees_with_a_byte_mask(seed):
    """engine.spans_cover (the memory-source coverage of resolve_recovery,
    reference engine.py:257-258) == painting the spans into a byte mask."""
    import random
    from paper_2408_04307_b200.engine import spans_cover
    rng = random.Random(seed)
    size = rng.randint(1, 64)
    for _ in range(50):
        spans = [(lo, lo + rng.randint(0, 20)) for lo in
                 (rng.randint(0, size) for _ in range(rng.randint(1, 6)))]
        mask = [False] * size
        for lo, hi in spans:
            for b in range(lo, min(hi, size)):
                mask[b] = True
        # the reference's rule: sorted by start, no gap before `size`
        reach, ok = 0, True
        for lo, hi in sorted(spans):
            if lo > reach:
                ok = False
                break
            reach = max(reach, hi)
        assert spans_cover(spans, size) == (ok and reach >= size)
        if spans_cover(spans, size):
            assert all(mask)


@pytest.mark.parametrize("n", [1, 3, 8, 16])
def test_window_table_rows_are_the_per_layer_windows(n):
    from paper_2408_04307_b200.selector import select_window, window_table
    for width in range(1, n + 2):
        for stride in range(0, n + 1):
            for c in range(0, 2 * n + 1):
                tab = window_table(c, 5, n, width, stride)
                for m in range(5):
                    assert tab[m].tolist() == sorted(select_window(c, m, n, width, stride))
