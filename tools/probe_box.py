"""Probe the GPU box: host RAM, cores, NUMA, disk, pinned D2H/H2D bandwidth."""
import os, subprocess, time, json
import torch

def sh(c):
    try:
        return subprocess.run(c, shell=True, capture_output=True, text=True, timeout=60).stdout
    except Exception as e:
        return str(e)

out = {}
out["cores_affinity"] = len(os.sched_getaffinity(0))
out["lscpu"] = sh("lscpu | egrep 'Model name|Socket|NUMA|^CPU\\(s\\)'")
out["meminfo"] = sh("head -3 /proc/meminfo")
out["df"] = sh("df -h /root /tmp . /dev/shm 2>/dev/null")
out["nvidia_smi_topo"] = sh("nvidia-smi topo -m")
out["nvidia_smi"] = sh("nvidia-smi --query-gpu=index,name,pcie.link.gen.current,pcie.link.width.current,memory.total --format=csv")
d = torch.device("cuda:0")
n = 1 << 30
dev = torch.empty(n, dtype=torch.uint8, device=d)
t0 = time.time()
host = torch.empty(n, dtype=torch.uint8, pin_memory=True)
out["pin_alloc_1GiB_s"] = time.time() - t0
s = torch.cuda.Stream()
def bw(fn):
    best = 1e9
    for _ in range(10):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s); fn(); e1.record(s)
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return n / best / 1e6
out["d2h_GBps"] = bw(lambda: host.copy_(dev, non_blocking=True))
out["h2d_GBps"] = bw(lambda: dev.copy_(host, non_blocking=True))
# disk write speed
p = "/tmp/probe_write.bin"
buf = host.numpy()
t0 = time.time()
with open(p, "wb") as f:
    f.write(memoryview(buf)[: 1 << 30]); f.flush(); os.fsync(f.fileno())
out["disk_write_GBps_tmp"] = (1 << 30) / (time.time() - t0) / 1e9
os.remove(p)
print(json.dumps(out, indent=1))
