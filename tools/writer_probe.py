"""Native persist writer on the box's tmpfs (measurement tool): Mixtral-rank-0
shaped entry sizes (2.1 GB optimizer entries, expert and module weights),
GB/s including CRCs with all host threads.  (A variant that filled large
files through a shared mapping as 16 MiB ranges from all threads measured
8.5-8.9 GB/s against 17.5-17.9 GB/s for whole-file write() jobs on the B200
box -- parallel page faults on one shmem file serialise -- and was dropped.)
Prints one JSON document."""
import json
import os
import shutil
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    from paper_2408_04307_b200 import device as D
    sizes = [2_113_929_216] * 4 + [352_321_536] * 4 + [201_326_592] * 8 + [50_000_000] * 20
    total = sum(sizes)
    src = np.empty(total, dtype=np.uint8)
    src[::4096] = 7
    bufs, off = [], 0
    for n in sizes:
        bufs.append(src[off:off + n])
        off += n
    threads = len(os.sched_getaffinity(0))
    out = {"bytes": total, "threads": threads, "files": len(sizes), "runs": {}}
    for rep in range(3):
        for nt in (8, threads):
            d = Path(tempfile.mkdtemp(dir="/dev/shm", prefix="pec_wp_"))
            paths = [d / f"f{i}.bin" for i in range(len(bufs))]
            t = time.perf_counter()
            D.write_files(paths, bufs, threads=nt)
            dt = time.perf_counter() - t
            out["runs"].setdefault(f"threads_{nt}", []).append(round(total / dt / 1e9, 2))
            shutil.rmtree(d)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
