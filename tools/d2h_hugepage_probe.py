"""Host-buffer flavours for the snapshot drain (measurement tool; not product):
pin time and pinned D2H GB/s of a 12 GiB buffer allocated as
  pinned       torch pin_memory (cudaHostAlloc)
  thp          anonymous mmap + madvise(MADV_HUGEPAGE), touched, cudaHostRegister
  4k           anonymous mmap (no advice), touched, cudaHostRegister
Prints one JSON document."""

import json
import mmap
import time

import numpy as np
import torch


def main():
    dev = torch.device("cuda", 0)
    big = 12 << 30
    src = torch.empty(big, dtype=torch.uint8, device=dev)
    src.fill_(5)
    s = torch.cuda.Stream()
    out = {"thp_enabled": open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip()}

    def bench(host, label):
        res = {}
        for n in (1 << 30, big):
            best = 1e30
            for _ in range(3):
                torch.cuda.synchronize()
                t = time.perf_counter()
                with torch.cuda.stream(s):
                    host[:n].copy_(src[:n], non_blocking=True)
                s.synchronize()
                best = min(best, time.perf_counter() - t)
            res[f"d2h_{n >> 30}GiB_GBps"] = round(n / best / 1e9, 2)
        assert int(host[big - 1]) == 5
        out[label].update(res)

    t = time.perf_counter()
    h = torch.empty(big, dtype=torch.uint8, pin_memory=True)
    out["pinned"] = {"alloc_pin_s": round(time.perf_counter() - t, 2)}
    bench(h, "pinned")
    del h

    for label, advise in (("thp", True), ("4k", False)):
        t = time.perf_counter()
        mm = mmap.mmap(-1, big, mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
        if advise:
            mm.madvise(mmap.MADV_HUGEPAGE)
        arr = np.frombuffer(mm, dtype=np.uint8)
        arr[::4096] = 0   # touch every page
        t_touch = time.perf_counter() - t
        t = time.perf_counter()
        rc = torch.cuda.cudart().cudaHostRegister(arr.ctypes.data, big, 0)
        out[label] = {"touch_s": round(t_touch, 2), "register_s": round(time.perf_counter() - t, 2),
                      "rc": int(rc)}
        if int(rc) == 0:
            bench(torch.from_numpy(arr), label)
            torch.cuda.cudart().cudaHostUnregister(arr.ctypes.data)
        try:
            ahp = open("/proc/meminfo").read().split("AnonHugePages:")[1].split("\n")[0].strip()
            out[label]["AnonHugePages_after"] = ahp
        except (OSError, IndexError):
            pass
        del arr
        mm.close()
    print(json.dumps(out, indent=1), flush=True)


if __name__ == "__main__":
    main()
