"""Drain probe (measurement tool): staging -> pinned host copy GB/s for the
bench's 12.62 GB Mixtral snapshot size vs a 1 GiB copy into pinned
(cudaHostAlloc) memory, single copy vs 1 GiB / 256 MiB chunks on one stream
vs two streams.  Best of 3 each.  Prints one JSON document."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch
    dev = torch.device("cuda", 0)
    n = 12_620_806_144
    staging = torch.empty(n, dtype=torch.uint8, device=dev)
    staging.view(torch.int32)[: n // 4].random_()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    cha = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    out = {}

    def best(fn, nbytes):
        b = 1e30
        for _ in range(3):
            torch.cuda.synchronize()
            t = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            b = min(b, time.perf_counter() - t)
        return round(nbytes / b / 1e9, 2)

    for name, host in (("cudaHostAlloc", cha),):
        host[:n].copy_(staging)  # first touch
        res = {}
        res["1GiB"] = best(lambda: host[: 1 << 30].copy_(staging[: 1 << 30], non_blocking=True),
                           1 << 30)
        res["single"] = best(lambda: host.copy_(staging, non_blocking=True), n)
        for c in (1 << 30, 256 << 20):
            def chunked(c=c):
                with torch.cuda.stream(s1):
                    for o in range(0, n, c):
                        host[o:o + c].copy_(staging[o:o + c], non_blocking=True)
            res[f"chunks_{c >> 20}MiB"] = best(chunked, n)

        def two():
            h = n // 2 // 4096 * 4096
            with torch.cuda.stream(s1):
                host[:h].copy_(staging[:h], non_blocking=True)
            with torch.cuda.stream(s2):
                host[h:].copy_(staging[h:], non_blocking=True)
        res["two_streams"] = best(two, n)
        out[name] = res
    print(json.dumps(out, indent=1), flush=True)


if __name__ == "__main__":
    main()
