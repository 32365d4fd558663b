"""The bench contract pieces that run without a GPU: the reference arm
(`bench.py --impl reference`, the oracle pack on host cores) prints one JSON
line with the driver's keys, and the host-buffer budget helper."""

import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def test_reference_arm_prints_one_contract_line():
    cmd = [sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "2",
           "--warmup", "1", "--cpu-sample-gb", "0.05"]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "impl", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0 and d["steps"] == 2
    assert d["config"]["workload"].startswith("mixtral")
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == d["value"]
    assert cb["components"]["py_crc32c_MBps_1core"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_host_buffer_budget_never_exceeds_available_memory(monkeypatch):
    sys.path.insert(0, str(ROOT))
    import bench
    avail = 0
    with open("/proc/meminfo") as f:
        for ln in f:
            if ln.startswith("MemAvailable"):
                avail = int(ln.split()[1]) * 1024
    monkeypatch.setenv("LOCAL_WORLD_SIZE", "1")
    assert bench.host_buffers_that_fit(1 << 20, 3) == 3
    assert bench.host_buffers_that_fit(avail, 3) == 0
    monkeypatch.setenv("LOCAL_WORLD_SIZE", "4")
    n = bench.host_buffers_that_fit(avail // 20, 3)
    assert n * 4 * (avail // 20) <= 0.7 * avail + 1


_RETENTION_WORKER = r'''
import os, sys, numpy as np, torch.distributed as dist
sys.path.insert(0, sys.argv[3])
import bench
from paper_2408_04307_b200.store import DiskStore, StoreEntry
from paper_2408_04307_b200.distributed import commit_version
dist.init_process_group("gloo")
r, w = dist.get_rank(), dist.get_world_size()
st = DiskStore(sys.argv[1], io_threads=2, recycle=sys.argv[2] == "1")
one = 8 * (1 << 20)
bench.store_bytes_per_version[id(st)] = 8 * one
ret = bench.Retention(st, [r], r == 0, keep=1, max_old=1)
bufs = [np.full(one, i, np.uint8) for i in range(8)]
worst = 0
for v in range(1, 25):
    ents = [StoreEntry(f"k{v % 3}_{i}_r{q}", q, f"u{i}", 0, one) for q in range(w) for i in range(8)]
    commit_version(st, v, v, v, ents, [r], {e.store_key: bufs[i % 8] for i, e in enumerate(ents) if e.rank == r})
    ret.submit()
    if r == 0:
        worst = max(worst, len(st.version_numbers()))
ret.close()
dist.barrier()
if r == 0:
    tot = sum(p.stat().st_size for p in __import__("pathlib").Path(sys.argv[1]).rglob("*.bin"))
    print("RESULT", worst, tot, st.complete_versions(), flush=True)
'''


def test_multirank_retention_bounds_the_store(tmp_path):
    """bench.Retention with 4 gloo ranks sharing one store: every rank retires
    its own files of superseded versions even after the coordinator has
    unlinked their COMPLETE markers (a rank that only saw the kept versions as
    complete once skipped retention and the /dev/shm tier grew without bound
    at N=4), so the store holds at most ~3 versions (+1 spare with recycling)
    and the newest complete version survives."""
    script = tmp_path / "worker.py"
    script.write_text(_RETENTION_WORKER)
    one_version = 4 * 8 * 8 * (1 << 20)
    for recycle in ("0", "1"):
        root = tmp_path / f"store{recycle}"
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nproc-per-node", "4",
               "--master-addr", "127.0.0.1", "--master-port", str(29480 + int(recycle)),
               str(script), str(root), recycle, str(ROOT)]
        res = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
        assert res.returncode == 0, res.stderr[-3000:]
        line = [ln for ln in res.stdout.splitlines() if ln.startswith("RESULT")][0]
        worst, tot, complete = line.split(" ", 3)[1:]
        assert int(worst) <= 4
        assert int(tot) <= (4 + int(recycle)) * one_version
        assert complete.strip() == "[24]"


def test_tmpfs_room_flags_a_filesystem_too_small_for_the_versions(tmp_path):
    """The persist tier is dropped (and the line says so) when the store's
    filesystem cannot hold the versions in flight for every local rank."""
    sys.path.insert(0, str(ROOT))
    import bench
    free, short = bench.tmpfs_room(tmp_path, 1)
    assert free > 0 and short is False
    free, short = bench.tmpfs_room(tmp_path, free * 2)
    assert short is True
    assert bench.tmpfs_room(tmp_path / "missing" / "dir", 1) == (None, False)
