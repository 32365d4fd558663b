"""C-ABI library loads and exports include/pec.h; oracle pinned to golden (CPU)."""

import ctypes
import json
import re

import numpy as np
import pytest

from conftest import GOLDEN, ROOT
from oracle import pec_oracle as O


def header_functions():
    text = (ROOT / "include" / "pec.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\*?\s+\*?(pec_[a-z0-9_]+)\(",
                                 text, re.M)))


def test_library_exports_every_header_symbol():
    from paper_2408_04307_b200 import _build, device as D
    _build.build()
    lib = ctypes.CDLL(str(D.LIB_PATH))
    names = header_functions()
    assert len(names) >= 11
    for name in names:
        assert hasattr(lib, name), name
    assert sorted(D.exported_symbols()) == names
    assert D.lib().pec_abi_version() == D.ABI_VERSION


def test_host_side_validation_rejects_bad_arguments_without_a_gpu():
    from paper_2408_04307_b200 import device as D
    L = D.lib()
    assert L.pec_token_hist(None, 0, 10, 8, None, None, 1, None, None, None) == D.PEC_E_INVAL
    assert L.pec_token_hist(None, 1, 10, 5000, None, None, 1, None, None, None) == D.PEC_E_RANGE
    assert L.pec_select_sequential(0, 0, 8, 1, 1, None, None) == D.PEC_E_INVAL
    assert L.pec_select_load_aware(None, 1, 8, 1, None, 0, None, 0, None) == D.PEC_E_INVAL
    assert L.pec_pack(None, 1, 1, 15, 1, None) == D.PEC_E_INVAL
    assert L.pec_pack(None, 1, 1, 30, 1, None) == D.PEC_E_INVAL
    assert L.pec_unpack(None, 0, 0, 15, 1, None) == D.PEC_OK  # empty table: no-op
    assert L.pec_strerror(D.PEC_E_CUDA).decode().startswith("CUDA")


def test_plan_chunks_prefix():
    from paper_2408_04307_b200 import device as D
    t = np.zeros(5, dtype=D.DESC_DTYPE)
    t["nbytes"] = [0, 1, 32768, 32769, 0]
    assert D.plan_chunks(t, 15) == 0 + 1 + 1 + 2 + 0
    assert t["first_chunk"].tolist() == [0, 0, 1, 2, 4]


def test_oracle_zipf_counts_match_reference_route_tokens():
    g = json.loads((GOLDEN / "routing.json").read_text())
    for case in g["zipf"]:
        L, E, total = case["layers"], case["experts"], case["total"]
        ids = np.stack([O.zipf_router_ids(case["seed"], case["iteration"], m, E, total,
                                          case["s"]) for m in range(L)])
        cap = O.capacity(case["capacity_factor"], total, E)
        assert O.route_counts(ids, E, cap).tolist() == case["counts"]


def test_oracle_selection_matches_reference():
    g = json.loads((GOLDEN / "selection.json").read_text())
    for c, m, n, width, stride, want in g["sequential"]:
        assert O.select_window(c, m, n, width, stride) == want
    for case in g["load_aware"]:
        assert O.select_load_aware(case["counts"], case["k"], case["pool"]) == case["selected"]


def test_oracle_load_aware_simulation_trace():
    """Replaying the reference Simulation's token stream through the oracle's
    count + two-tier selection reproduces every checkpoint's sets."""
    g = json.loads((GOLDEN / "loadaware_sim.json").read_text())
    for t in g["traces"]:
        L, E = t["layers"], t["experts"]
        total = t["tokens"] * t["top_k"]
        cap = O.capacity(t["capacity_factor"], total, E)
        snap = np.zeros((L, E), dtype=np.int64)
        pers = np.zeros((L, E), dtype=np.int64)
        got = []
        for i in range(1, t["i_total"] + 1):
            ids = np.stack([O.zipf_router_ids(t["seed"], i, m, E, total, t["zipf_s"])
                            for m in range(L)])
            counts = O.route_counts(ids, E, cap)
            snap += counts
            pers += counts
            if i % t["i_ckpt"] == 0:
                ss, ps, snap, pers = O.two_tier_load_aware(snap, pers, t["k_snapshot"],
                                                           t["k_persist"])
                got.append({"c": i // t["i_ckpt"] - 1, "snap": ss, "persist": ps})
        assert got == t["checkpoints"]


def test_oracle_pack_unpack_roundtrip():
    rng = np.random.default_rng(0)
    state = rng.integers(0, 256, 10000, dtype=np.uint8)
    copies = [(10, 0, 100), (5000, 300, 17), (9000, 400, 1000)]
    st = O.pack(state, copies, 1500)
    assert bytes(st[300:317]) == bytes(state[5000:5017])
    back = O.unpack(st, copies, np.zeros_like(state))
    for s, _, n in copies:
        assert np.array_equal(back[s:s + n], state[s:s + n])


@pytest.mark.parametrize("direct,fsync", [(False, False), (True, False), (True, True)])
def test_native_writer_writes_exact_bytes_and_crcs(tmp_path, direct, fsync):
    """Buffered and O_DIRECT (bounce buffer, padded last block, truncate
    back) writes produce the exact bytes and their CRC-32Cs; sizes cover
    empty, sub-block, block+1 and multi-piece files."""
    from paper_2408_04307_b200 import device as D
    from paper_2408_04307_b200.store import crc32c
    rng = np.random.default_rng(8)
    bufs = [rng.integers(0, 256, size=n, dtype=np.uint8)
            for n in (0, 1, 4096, 4097, (4 << 20) + 5, (8 << 20))]
    bufs.append(bufs[3][3:])  # unaligned source address
    # O_DIRECT splits files above 64 MiB into ranges written by different
    # threads at their offsets (CRCs of the ranges combined in order)
    bufs.append(rng.integers(0, 256, size=(150 << 20) + 12_345, dtype=np.uint8))
    bufs.append(bufs[-1][1:(128 << 20) + 1])   # exactly two ranges, unaligned source
    paths = [tmp_path / f"e{i}.bin" for i in range(len(bufs))]
    crcs = D.write_files(paths, bufs, threads=3, direct=direct, fsync=fsync,
                         background=direct)
    for p, b, c in zip(paths, bufs, crcs):
        assert p.read_bytes() == b.tobytes()
        assert int(c) == crc32c(b)
    with pytest.raises(OSError):
        D.write_files([tmp_path / "missing" / "x.bin"], [bufs[2]])


def test_c_abi_host_entry_points_from_plain_c(tmp_path):
    """include/pec.h compiles as C11 and the host entry points behave as
    documented when called from C (tests/c/abi_check.c)."""
    import subprocess
    from conftest import build_abi_check
    exe = build_abi_check(tmp_path, gpu=False)
    res = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "0 failure(s)" in res.stdout
