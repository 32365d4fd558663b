"""Host-link probe: pinned D2H/H2D GB/s vs copy size, chunking and streams,
alone and while the pack kernel runs (measurement tool; not product)."""

import json
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def timed(fn, reps=3):
    best = 1e30
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    return best


def main():
    dev = torch.device("cuda", 0)
    out = {}
    big = 12 << 30
    src = torch.empty(big, dtype=torch.uint8, device=dev)
    src.fill_(3)
    t = time.perf_counter()
    host = torch.empty(big, dtype=torch.uint8, pin_memory=True)
    out["pin_alloc_12GiB_s"] = round(time.perf_counter() - t, 2)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for size_gb in (0.25, 1, 4, 12):
        n = int(size_gb * (1 << 30))

        def one():
            with torch.cuda.stream(s1):
                host[:n].copy_(src[:n], non_blocking=True)
        out[f"d2h_single_{size_gb}GiB"] = round(n / timed(one) / 1e9, 2)

        def h2d():
            with torch.cuda.stream(s1):
                src[:n].copy_(host[:n], non_blocking=True)
        out[f"h2d_single_{size_gb}GiB"] = round(n / timed(h2d) / 1e9, 2)
    n = big
    for chunk_mb in (16, 64, 256, 1024):
        c = chunk_mb << 20

        def chunked():
            with torch.cuda.stream(s1):
                for o in range(0, n, c):
                    host[o:o + c].copy_(src[o:o + c], non_blocking=True)
        out[f"d2h_chunked_{chunk_mb}MiB"] = round(n / timed(chunked) / 1e9, 2)

    def two_streams():
        h = n // 2
        with torch.cuda.stream(s1):
            host[:h].copy_(src[:h], non_blocking=True)
        with torch.cuda.stream(s2):
            host[h:].copy_(src[h:], non_blocking=True)
    out["d2h_two_streams_12GiB"] = round(n / timed(two_streams) / 1e9, 2)
    # write-combined / portable variants via cudart
    print(json.dumps(out, indent=1), flush=True)


if __name__ == "__main__":
    main()
