"""Zero-copy restore probe: can the H2D read tmpfs file pages directly?

For a file of ``--gb`` GB on /dev/shm: (a) pread into a pinned bounce buffer
with T threads, then H2D (what `restore` does today); (b) mmap the file,
`cudaHostRegister` the mapping (read-only), H2D straight from the page cache,
unregister.  Prints the seconds of every step and the end-to-end GB/s of both.
"""

import json
import mmap
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import argparse
    import torch
    ap = argparse.ArgumentParser()
    ap.add_argument("--gb", type=float, default=4.0)
    ap.add_argument("--threads", type=int, default=16)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--flags", type=int, default=0, help="cudaHostRegister flags (8 = ReadOnly)")
    args = ap.parse_args()
    n = int(args.gb * (1 << 30)) // (1 << 21) * (1 << 21)
    path = "/dev/shm/pec_register_probe.bin"
    src = np.random.default_rng(1).integers(0, 255, size=1 << 26, dtype=np.uint8)
    with open(path, "wb") as f:
        for lo in range(0, n, src.size):
            f.write(src[:min(src.size, n - lo)].tobytes())
    dev = torch.empty(n, dtype=torch.uint8, device="cuda")
    bounce = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    bounce.numpy()[:] = 0
    cudart = torch.cuda.cudart()
    out = {"bytes": n, "threads": args.threads, "bounce": [], "register": []}

    def pread_all(view):
        step = 8 << 20

        def one(lo):
            fd = os.open(path, os.O_RDONLY)
            try:
                os.preadv(fd, [view[lo:lo + min(step, n - lo)]], lo)
            finally:
                os.close(fd)
        with ThreadPoolExecutor(args.threads) as pool:
            list(pool.map(one, range(0, n, step)))

    for _ in range(args.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pread_all(memoryview(bounce.numpy()).cast("B"))
        t1 = time.perf_counter()
        dev.copy_(bounce, non_blocking=True)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        out["bounce"].append({"read_s": round(t1 - t0, 3), "h2d_s": round(t2 - t1, 3),
                              "GBps": round(n / (t2 - t0) / 1e9, 2)})

    for _ in range(args.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fd = os.open(path, os.O_RDWR)
        mm = mmap.mmap(fd, n, mmap.MAP_SHARED, mmap.PROT_READ | mmap.PROT_WRITE)
        os.close(fd)
        arr = np.frombuffer(mm, dtype=np.uint8)
        addr = arr.ctypes.data
        t1 = time.perf_counter()
        rc = int(cudart.cudaHostRegister(addr, n, args.flags))
        t2 = time.perf_counter()
        if rc != 0:
            out["register"].append({"error": f"cudaHostRegister rc={rc}"})
            del arr
            mm.close()
            break
        host = torch.from_numpy(arr)
        dev.copy_(host, non_blocking=True)
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        cudart.cudaHostUnregister(addr)
        del host, arr
        mm.close()
        t4 = time.perf_counter()
        out["register"].append({"mmap_s": round(t1 - t0, 3), "register_s": round(t2 - t1, 3),
                                "h2d_s": round(t3 - t2, 3), "unregister_s": round(t4 - t3, 3),
                                "GBps": round(n / (t4 - t0) / 1e9, 2)})
    ok = bool(torch.equal(dev[:src.size].cpu(), torch.from_numpy(src[:min(src.size, n)])))
    out["last_copy_correct"] = ok
    os.unlink(path)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
