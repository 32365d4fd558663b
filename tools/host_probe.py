"""Host-side ceilings of the persist tier on this box (no GPU work).

Prints one JSON object:
* topology: sockets / NUMA nodes / cores (lscpu), `nvidia-smi topo -m` when present;
* memcpy: aggregate numpy copy bandwidth with 1..T threads (each thread copies
  its own buffer; GIL released inside the copy);
* tmpfs: `pec_write_files` into /dev/shm with W writer groups at once (one per
  simulated rank, `threads` each), fresh files vs recycled files (overwrite
  in place), GB/s aggregate.

Used to tell whether a persist rate measured by bench.py at N>1 is at the
box's host-memory ceiling.  Example:
    python tools/host_probe.py --gb 4 --ranks 4 --threads 4
"""

from __future__ import annotations

import argparse
import json
import os
import shutil
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def sh(cmd):
    try:
        return subprocess.run(cmd, capture_output=True, text=True, timeout=30).stdout
    except (OSError, subprocess.TimeoutExpired):
        return ""


def topology():
    out = {}
    for ln in sh(["lscpu"]).splitlines():
        k, _, v = ln.partition(":")
        if k.strip() in ("Socket(s)", "NUMA node(s)", "CPU(s)", "Model name",
                         "Thread(s) per core") or k.strip().startswith("NUMA node"):
            out[k.strip()] = v.strip()
    topo = sh(["nvidia-smi", "topo", "-m"])
    if topo:
        out["nvidia_topo"] = topo.splitlines()[:12]
    return out


def memcpy_bw(gb_per_thread: float, threads: int, reps: int = 3) -> float:
    n = int(gb_per_thread * (1 << 30))
    src = [np.ones(n, np.uint8) for _ in range(threads)]
    dst = [np.empty(n, np.uint8) for _ in range(threads)]
    for d, s in zip(dst, src):
        np.copyto(d, s)                            # first touch
    best = 0.0
    for _ in range(reps):
        ts = [threading.Thread(target=np.copyto, args=(d, s)) for d, s in zip(dst, src)]
        t0 = time.perf_counter()
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        best = max(best, threads * n / (time.perf_counter() - t0) / 1e9)
    return round(best, 2)


def tmpfs_bw(gb_per_rank: float, ranks: int, threads: int, file_mb: int = 256,
             rounds: int = 3):
    from paper_2408_04307_b200 import device as D
    n_files = max(1, int(gb_per_rank * 1024 // file_mb))
    bufs = [np.full(file_mb << 20, r + 1, np.uint8) for r in range(ranks)]
    root = Path(tempfile.mkdtemp(prefix="pec_hostprobe_", dir="/dev/shm"))
    res = {"fresh": [], "overwrite": []}
    try:
        for rnd in range(rounds):
            for mode in ("fresh", "overwrite"):
                if mode == "fresh":
                    shutil.rmtree(root, ignore_errors=True)
                    root.mkdir(parents=True)

                def one(r):
                    paths = [root / f"r{r}_{i}.bin" for i in range(n_files)]
                    D.write_files(paths, [bufs[r]] * n_files, threads=threads, want_crc=False,
                                  overwrite=mode == "overwrite")
                ts = [threading.Thread(target=one, args=(r,)) for r in range(ranks)]
                t0 = time.perf_counter()
                for t in ts:
                    t.start()
                for t in ts:
                    t.join()
                dt = time.perf_counter() - t0
                res[mode].append(round(ranks * n_files * (file_mb << 20) / dt / 1e9, 2))
    finally:
        shutil.rmtree(root, ignore_errors=True)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gb", type=float, default=2.0, help="GB per simulated rank / thread")
    ap.add_argument("--ranks", type=int, default=4)
    ap.add_argument("--threads", type=int, default=4, help="writer threads per rank")
    ap.add_argument("--max-threads", type=int, default=0)
    args = ap.parse_args()
    ncpu = len(os.sched_getaffinity(0))
    out = {"topology": topology(), "cores": ncpu}
    tmax = args.max_threads or ncpu
    ts, t = [], 1
    while t <= tmax:
        ts.append(t)
        t *= 2
    out["memcpy_GBps"] = {str(t): memcpy_bw(min(args.gb, 1.0), t) for t in ts}
    out["tmpfs_write_GBps"] = {f"{args.ranks}x{args.threads}": tmpfs_bw(args.gb, args.ranks,
                                                                       args.threads),
                               f"1x{args.threads}": tmpfs_bw(args.gb, 1, args.threads)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
