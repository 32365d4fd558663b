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
