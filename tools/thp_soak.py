"""Soak test for THP-advised anonymous host memory pinned with
cudaHostRegister (the host-buffer flavour DESIGN.md §10 withdrew after one
unexplained mismatch).  Each round: map + advise + touch + register a
buffer, D2H a random device image into it (256 MiB pieces), compare on the
host, H2D it back into a second device buffer and compare on the device;
between rounds a subprocess is sometimes forked; with --leak buffers are
sometimes dropped without unregistering (left to the GC: the next
registration at a reused address then fails -- a mapping must never be freed
while registered).  Prints one JSON line with the mismatch count."""
import gc
import json
import mmap
import subprocess
import sys

import numpy as np
import torch


class ThpBuf:
    def __init__(self, n):
        self.mm = mmap.mmap(-1, n, mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
        self.mm.madvise(mmap.MADV_HUGEPAGE)
        self.a = np.frombuffer(self.mm, dtype=np.uint8)
        self.a[::4096] = 0
        rc = torch.cuda.cudart().cudaHostRegister(self.a.ctypes.data, n, 0)
        assert int(rc) == 0, rc
        self.t = torch.from_numpy(self.a)
        self.reg = True

    def close(self):
        if self.reg:
            torch.cuda.cudart().cudaHostUnregister(self.a.ctypes.data)
            self.reg = False
        self.t = None
        self.a = None
        try:
            self.mm.close()
        except BufferError:
            pass


def main():
    rounds = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 40
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(0)
    bad, leaked = 0, []
    s = torch.cuda.Stream()
    for r in range(rounds):
        n = int(rng.integers(64, 1200)) << 20
        src = torch.empty(n, dtype=torch.uint8, device=dev)
        src.view(torch.int32)[: n // 4].random_()
        b = ThpBuf(n)
        with torch.cuda.stream(s):
            for o in range(0, n, 256 << 20):
                b.t[o:o + (256 << 20)].copy_(src[o:o + (256 << 20)], non_blocking=True)
        s.synchronize()
        ok_host = np.array_equal(b.a, src.cpu().numpy())
        back = torch.empty_like(src)
        with torch.cuda.stream(s):
            back.copy_(b.t, non_blocking=True)
        s.synchronize()
        ok_dev = bool(torch.equal(back, src))
        bad += (not ok_host) + (not ok_dev)
        action = r % 3
        if action == 0:
            b.close()
        elif action == 1 and "--leak" in sys.argv:
            leaked.append(b)          # dropped later without unregistering
            if len(leaked) > 2:
                leaked.pop(0)
                gc.collect()
        elif action == 1:
            gc.collect()
            b.close()
        else:
            subprocess.run(["true"], check=True)  # fork + exec while registered
            b.close()
    print(json.dumps({"rounds": rounds, "mismatches": bad}))


if __name__ == "__main__":
    main()
