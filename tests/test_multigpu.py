"""Multi-process (one process per GPU) check over NCCL, when the box has >= 2
GPUs: tools/multirank_gpu.py under torchrun -- global load-aware selection on
all-reduced counters == the oracle, multi-writer persist, node fault handled
by PecCheckpointer.recover on every rank (bit-identical restore, counters
reset).  Skipped on a single-GPU box (the driver's round-end run); the
recorded N=2/4 runs are in DESIGN.md / profiles."""

import json
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_multirank_selection_persist_and_recover(dev):
    import torch
    n = min(torch.cuda.device_count(), 4)
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           str(ROOT / "tools" / "multirank_gpu.py")]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    lines = [json.loads(ln) for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-2000:]
    assert len(lines) == n
    for r in lines:
        assert r["selection_ok"] and r["files_ok"] and r["restore_ok"] and r["counters_ok"], r
