"""Property tests (hypothesis, as the reference's suite uses,
pyproject.toml:12-13) for the host pieces the device path leans on:
CRC-32C chaining and combination (the pack's per-chunk CRCs are joined with
crc32c_combine), the oracle's CRC restatement, staging placement, window
tables and the store's spare recycling.  CPU only."""

import numpy as np
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_2408_04307_b200 import device as D
from paper_2408_04307_b200.selector import select_window, window_table
from paper_2408_04307_b200.staging import STAGE_ALIGN
from paper_2408_04307_b200.store import crc32c
from oracle import pec_oracle as O


@settings(max_examples=200, deadline=None)
@given(st.binary(max_size=3000), st.binary(max_size=3000))
def test_crc_combine_equals_crc_of_concatenation(a, b):
    """crc32c(A||B) == combine(crc32c(A), crc32c(B), len(B)) (store.py:49-70
    semantics; the fold kernel's chunk joins rely on it)."""
    assert D.crc32c_combine(crc32c(a), crc32c(b), len(b)) == crc32c(a + b)
    assert crc32c(b, crc32c(a)) == crc32c(a + b)


@settings(max_examples=100, deadline=None)
@given(st.binary(max_size=5000))
def test_native_crc_equals_the_oracle_restatement(data):
    assert crc32c(data) == O.crc32c(np.frombuffer(data, dtype=np.uint8))


@settings(max_examples=200, deadline=None)
@given(st.integers(0, 50), st.integers(1, 12), st.integers(1, 64), st.integers(1, 64),
       st.integers(1, 64))
def test_window_table_rows_are_the_reference_windows(c, L, N, width, stride):
    """Every row of the [L, W] table is select_window(c, m) (selector.py:21-27),
    ascending, W = min(width, N)."""
    t = window_table(c, L, N, width, stride)
    assert t.shape == (L, min(width, N))
    for m in range(L):
        assert list(t[m]) == sorted(select_window(c, m, N, width, stride))


@settings(max_examples=300, deadline=None)
@given(st.integers(0, 1 << 40), st.integers(0, 1 << 40))
def test_staging_placement_is_congruent_and_minimal(pos, src):
    """An entry goes to the first offset >= pos congruent to its source
    address mod 256, so source and staging share alignment."""
    from paper_2408_04307_b200.restore import _place
    off = _place(pos, src)
    assert off >= pos and off - pos < STAGE_ALIGN
    assert (off - src) % STAGE_ALIGN == 0


@settings(max_examples=25, deadline=None)
@given(st.lists(st.lists(st.integers(0, 3), min_size=1, max_size=5), min_size=2, max_size=6),
       st.integers(0, 2 ** 31))
def test_recycled_store_always_reads_back_the_newest_version(size_codes, seed):
    """Versions with entry sizes drawn from a small set (so spares fit some
    later entries and not others), the previous version retired after each
    publish with recycling on: the newest version always loads CRC-verified
    with exactly its own bytes, and no retired version stays readable."""
    import shutil
    import tempfile
    from paper_2408_04307_b200.store import DiskStore, StoreEntry
    sizes = [0, 1, 4096, 70_001]
    rng = np.random.default_rng(seed)
    root = tempfile.mkdtemp(prefix="pec_prop_")
    try:
        st_ = DiskStore(root, io_threads=2, recycle=True)
        for v, codes in enumerate(size_codes, start=1):
            ents = [StoreEntry(f"ew.L{i}.E0", i % 2, f"ew.L{i}.E0", 0, sizes[c])
                    for i, c in enumerate(codes)]
            pay = {e.store_key: rng.bytes(e.stop - e.start) for e in ents}
            st_.write_version(v, 10 * v, v, ents, payloads=pay)
            if v > 1:
                assert st_.retire(v - 1)
            assert st_.complete_versions() == [v]
            assert st_.load_checkpoint(v) == pay
    finally:
        shutil.rmtree(root, ignore_errors=True)
