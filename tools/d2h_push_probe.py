"""Copy-engine D2H vs SM-driven push into mapped pinned memory (probe)."""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch
    from paper_2408_04307_b200 import device as D
    dev = torch.device("cuda", 0)
    n = 2 << 30
    src = torch.randint(0, 256, (n,), dtype=torch.uint8, device=dev)
    host = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    host.copy_(src)  # first touch
    out = {}

    def timeit(fn, reps=5):
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b))
        return min(ts)

    out["ce_d2h_GBps"] = round(n / (timeit(lambda: host.copy_(src, non_blocking=True)) / 1e3) / 1e9, 2)
    for mode in (1, 2):
        t = np.zeros(1, dtype=D.DESC_DTYPE)
        t[0] = (src.data_ptr(), host.data_ptr(), n, 0)
        total = D.plan_chunks(t, 15)
        dt = torch.from_numpy(t.view(np.uint8).copy()).view(torch.int64).to(dev)
        try:
            ms = timeit(lambda: D.pack(dt, 1, total, 15, mode))
            ok = bool(torch.equal(host[:1 << 20].to(dev), src[:1 << 20]))
            out[f"sm_push_mode{mode}_GBps"] = round(n / (ms / 1e3) / 1e9, 2)
            out[f"sm_push_mode{mode}_ok"] = ok
        except Exception as e:  # noqa: BLE001
            out[f"sm_push_mode{mode}"] = repr(e)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
