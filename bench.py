#!/usr/bin/env python
"""PEC snapshot benchmark (the driver's bench contract).

One *step* = one PEC checkpoint snapshot of this rank's shard: on-device K_pec
selection for checkpoint c, then the pack of the rank's planned byte ranges
(experts' bf16 weights + fp32 master/m/v, its ZeRO-2 non-expert optimizer
shard, its share of the non-expert weights) from the HBM state arena into the
HBM staging buffer.  `value` is that with the state already resident in HBM;
`e2e` adds the copy-engine drain of the staging buffer into a pinned host
snapshot buffer (the reference's SNAPSHOTTED state: bytes in CPU memory) and
the host read of the step result, through the package's public API.

Workload (default): Mixtral-8x7B-shaped state, K_pec=1, adaptive_pec plan of
the dp=ep=8 deployment; with N GPUs, ranks 0..N-1 of that plan (weak scaling:
each GPU holds the same-size ~85 GB rank shard at every N).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "PEC snapshot GB/s per GPU (vs HBM/PCIe roofline); exposed ckpt stall ms/iter"
UNIT = "GB/s"
FALLBACK_HBM = 6650.0
# nominal HBM3e bandwidth of an HGX B200 (B200_PROFILING.md hardware table)
HBM_NOMINAL_GBS = 7700.0


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return FALLBACK_HBM, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for name, val in zip(names, f[5:9]):
                if val.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_init(n_gpus):
    rank, local, world = env_rank()
    if world > 1:
        import torch.distributed as dist
        import torch
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, local, world


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, world, device):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x, world, device):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def host_buffers_that_fit(nbytes: int, want: int, frac: float = 0.7) -> int:
    """How many pinned host snapshot buffers of ``nbytes`` each local rank
    can take (LOCAL_WORLD_SIZE ranks pin at once) within ``frac`` of the
    node's MemAvailable."""
    try:
        with open("/proc/meminfo") as f:
            info = {ln.split(":")[0]: int(ln.split()[1]) * 1024 for ln in f if ":" in ln}
        avail = info.get("MemAvailable", info.get("MemFree", 0))
    except OSError:
        return want
    local = max(1, int(os.environ.get("LOCAL_WORLD_SIZE", "1")))
    return max(0, min(want, int(frac * avail // (local * max(1, nbytes)))))


# ---------------------------------------------------------------------------
# CPU baseline: the oracle's pack restatement on host cores
# ---------------------------------------------------------------------------

def cpu_pack_sample(entries, sample_bytes: int, threads: int, min_seconds: float):
    """Pack a bounded sample of this rank's planned ranges from a
    host-resident state image with the oracle's threaded numpy restatement:
    every entry of the plan, each cut to the same fraction of its length
    (sample_bytes / total; at least 256 B), so the sample keeps the
    workload's mix of entry sizes and alignments.  Repeat until
    `min_seconds` of CPU work.  Returns (GB/s of payload, description)."""
    from oracle import pec_oracle as O
    entries = [e for e in entries if e.nbytes > 0]
    total = sum(e.nbytes for e in entries)
    frac = min(1.0, sample_bytes / max(1, total))
    copies, src_pos, dst_pos = [], 0, 0
    for e in entries:
        n = min(e.nbytes, max(256, int(e.nbytes * frac)))
        src = src_pos + (e.src_offset % 256)
        dst = dst_pos + ((src - dst_pos) % 256)
        copies.append((src, dst, n))
        src_pos = src + n + 256
        dst_pos = dst + n
    state = np.random.default_rng(0).integers(0, 256, size=src_pos + 256, dtype=np.uint8)
    out = np.empty(dst_pos + 256, dtype=np.uint8)
    payload = sum(c[2] for c in copies)
    O.pack_threaded(state, copies, out, threads)  # warm
    t0 = time.perf_counter()
    reps = 0
    while True:
        O.pack_threaded(state, copies, out, threads)
        reps += 1
        if time.perf_counter() - t0 >= min_seconds:
            break
    dt = time.perf_counter() - t0
    desc = (f"oracle numpy pack of {payload / 1e9:.2f} GB: every one of the rank's "
            f"{len(copies)} planned entries cut to {100 * frac:.1f} % of its length, "
            f"x{reps} passes, {threads} threads")
    return payload * reps / dt / 1e9, desc


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_components(layout, strategy: str, k_pec: int, crc_sample: int = 1 << 20):
    """The reference's other per-checkpoint CPU costs:
    two-tier load-aware selection (oracle restatement of the reference's
    Python sort, selector.py:91-100 / simulator.py:339-354), one checkpoint's
    range plan (build_phase_assignment, planner.py:263-295) and the
    reference's byte-at-a-time pure-Python CRC-32C (store.py:49-70,
    restated in the oracle) on a 1 MiB sample, 1 core."""
    from oracle import pec_oracle as O
    from paper_2408_04307_b200 import build_phase_assignment
    m = layout.model
    L, E = m.num_moe_layers, m.experts_per_layer
    rng = np.random.default_rng(1)
    snap = rng.integers(0, 1 << 20, (L, E))
    pers = snap.copy()
    t0 = time.perf_counter()
    reps = 0
    while time.perf_counter() - t0 < 0.5:
        O.two_tier_load_aware(snap.copy(), pers.copy(), k_pec, k_pec)
        reps += 1
    sel_us = (time.perf_counter() - t0) / reps * 1e6
    due = {l: frozenset(range(k_pec)) for l in range(L)}
    t0 = time.perf_counter()
    reps = 0
    while time.perf_counter() - t0 < 0.5:
        build_phase_assignment(layout, due, strategy)
        reps += 1
    plan_ms = (time.perf_counter() - t0) / reps * 1e3
    data = rng.integers(0, 256, crc_sample, dtype=np.uint8).tobytes()
    t0 = time.perf_counter()
    O.crc32c_py(data)
    crc_mbs = crc_sample / (time.perf_counter() - t0) / 1e6
    return {"select_two_tier_us": round(sel_us, 1), "plan_ms": round(plan_ms, 3),
            "py_crc32c_MBps_1core": round(crc_mbs, 2),
            "what": "oracle two-tier load-aware selection [L,E]; host planner "
                    "build_phase_assignment for one due set; reference-style pure-Python "
                    "CRC-32C on 1 MiB"}


# ---------------------------------------------------------------------------
# exposed checkpoint stall: synthetic training loop with and without PEC
# ---------------------------------------------------------------------------

def prune_store(store, keep: int = 1) -> None:
    """Bench-only retention: drop all but the newest ``keep`` complete
    versions (each is a full rank shard; /dev/shm is host RAM)."""
    if store is None or not hasattr(store, "version_dir"):
        return
    import shutil
    for v in store.complete_versions()[:-keep]:
        shutil.rmtree(store.version_dir(v), ignore_errors=True)


def measure_stall(ck, arena, dev, iters: int, i_ckpt: int, fb_ms: float, rounds: int = 3):
    """Synthetic per-rank training loop on the compute stream: an F&B proxy
    (bf16 8192^3 GEMMs, calibrated to ~fb_ms) then an update proxy (one
    in-place pass over the whole state arena: HBM-bound like a fused Adam
    step over the rank's ~85 GB shard).  With checkpointing, every i_ckpt-th
    iteration calls PecCheckpointer.checkpoint after its update (the pack
    photographs the updated state on the side stream, overlapping the next
    F&B) and every update first waits for the pending pack.  Returns the
    device time per iteration with/without and the difference."""
    import torch
    a = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
    b = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
    c = torch.empty(8192, 8192, device=dev, dtype=torch.bfloat16)
    words = arena.buffer.view(torch.int32)
    compute = torch.cuda.current_stream(dev)
    for _ in range(3):
        torch.matmul(a, b, out=c)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        torch.matmul(a, b, out=c)
    e1.record()
    e1.synchronize()
    gemm_ms = e0.elapsed_time(e1) / 10
    n_gemm = max(1, int(round(fb_ms / gemm_ms)))
    e0.record()
    words.add_(1)
    e1.record()
    e1.synchronize()
    update_ms = e0.elapsed_time(e1)

    def run(with_ckpt: bool, base_it: int) -> float:
        torch.cuda.synchronize()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(compute)
        for k in range(1, iters + 1):
            it = base_it + k
            for _ in range(n_gemm):                 # forward + backward
                torch.matmul(a, b, out=c)
            if with_ckpt:
                ck.poll()
                ck.wait_pack(stream=compute)        # the update may not race the pack
            words.add_(1)                           # optimizer step
            if with_ckpt and it % i_ckpt == 0:
                ck.checkpoint(it)                   # select + plan + pack + drain
        t1.record(compute)
        t1.synchronize()
        return t0.elapsed_time(t1) / iters

    run(False, 0)  # warm
    n_before = len(ck.engine.stats["pack_ms"])
    # alternate without / with (A B A B) so slow drifts (clocks, other
    # tenants of the host) hit both arms alike; each arm = mean of its runs
    runs_without, runs_with = [], []
    for r in range(rounds):
        runs_without.append(run(False, 0))
        runs_with.append(run(True, 10 ** 6 * (r + 1)))
        ck.finish()
        prune_store(ck.engine.store)
    without, with_ = statistics.mean(runs_without), statistics.mean(runs_with)
    packs = ck.engine.stats["pack_ms"][n_before:]
    return {"i_ckpt": i_ckpt, "iters": iters, "rounds": rounds,
            "checkpoints": rounds * (iters // i_ckpt),
            "fb_ms": round(n_gemm * gemm_ms, 1), "fb_gemms": n_gemm,
            "update_ms": round(update_ms, 2),
            "iter_ms_without": round(without, 3), "iter_ms_with": round(with_, 3),
            "runs_ms_without": [round(x, 3) for x in runs_without],
            "runs_ms_with": [round(x, 3) for x in runs_with],
            "exposed_ms_per_iter": round(with_ - without, 3),
            # spread of the baseline runs: differences below it are noise
            "noise_ms_per_iter": round((max(runs_without) - min(runs_without)) / 2, 3),
            "pack_ms_in_loop": round(statistics.mean(packs), 3) if packs else None,
            "overhead_frac": round((with_ - without) / without, 5)}


# ---------------------------------------------------------------------------

def build_workload(args, rank):
    from paper_2408_04307_b200 import configs
    from paper_2408_04307_b200.planner import plan_adaptive, plan_equal
    w = configs.WORKLOADS[args.workload]()
    layout = w.layout()
    if w.pec.selection == "load_aware":
        plan = None  # assignments are built per checkpoint (on device)
    elif w.strategy == "adaptive_pec":
        plan = plan_adaptive(layout, w.pec)
    else:
        plan = plan_equal(layout, w.pec)
    if rank >= layout.n_ranks:
        raise SystemExit(f"rank {rank} >= dp degree {layout.n_ranks} of {w.name}")
    return w, layout, plan


def run_reference(args):
    rank, local, world = env_rank()
    if rank != 0:
        return 0
    threads = len(os.sched_getaffinity(0))
    from paper_2408_04307_b200.staging import StagingLayout
    w, layout, plan = build_workload(args, 0)

    class _Slots:  # arena-less offsets (host-only reference arm)
        def __init__(self):
            off, self.o = 0, {}
            for u in layout.units:
                if 0 in u.replica_ranks and u.size_bytes:
                    self.o[u.key] = off
                    off = (off + u.size_bytes + 255) // 256 * 256

        def slot(self, key):
            class S:
                pass
            s = S()
            s.offset = self.o[key]
            return s

    if plan is not None:
        ranges0 = plan.assignments[0][0]
    else:  # load-aware: a representative due set of the same size (window c=0)
        from paper_2408_04307_b200.planner import build_phase_assignment
        from paper_2408_04307_b200.selector import select_window
        n = layout.model.experts_per_layer
        due = {m: select_window(0, m, n, w.pec.k_snapshot, w.pec.k_persist)
               for m in range(layout.model.num_moe_layers)}
        ranges0 = build_phase_assignment(layout, due, w.strategy)[0]
    st = StagingLayout.build(ranges0, _Slots(), 0)
    sample = min(args.cpu_sample_gb, st.payload_bytes / 1e9)
    per_step = []
    for i in range(args.warmup + args.steps):
        gbs, desc = cpu_pack_sample(st.entries, int(sample * 1e9), threads, 0.0)
        if i >= args.warmup:
            per_step.append(gbs)
    value = statistics.mean(per_step)
    try:
        components = cpu_components(layout, w.strategy, w.pec.k_pec)
    except Exception as exc:  # reported, never fatal to the line
        components = {"error": f"{type(exc).__name__}: {exc}"[:200]}
    line = {"metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(sample * 1e9 / (value * 1e9) * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": w.name, "plan": w.strategy, "selection": w.pec.selection,
                       "k_pec": w.pec.k_pec, "ranks": f"0 of dp={layout.n_ranks} (host cores)",
                       "parallelism": f"dp{layout.n_ranks}-ep{layout.parallel.ep_degree}",
                       "sample_gb": round(sample, 3)},
            "cpu_baseline": {"value": round(value, 3), "unit": UNIT, "cores": threads,
                             "kind": "port", "sample": desc, "cpu_model": cpu_model(),
                             "components": components},
            "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    emit(line)
    return 0


def run_b200(args):
    import shutil
    import tempfile
    import torch
    rank, local, world = dist_init(args.gpus)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_2408_04307_b200 import device as D
    from paper_2408_04307_b200.arena import StateArena
    from paper_2408_04307_b200.counting import DeviceTokenCounters
    from paper_2408_04307_b200.snapshot import PecCheckpointer
    from paper_2408_04307_b200.staging import StagingLayout
    from paper_2408_04307_b200.store import DiskStore

    w, layout, plan = build_workload(args, rank)
    t_fill = time.time()
    arena = StateArena(layout, ranks=[rank], device=dev, expert_tensors=w.expert_tensors)
    torch.cuda.synchronize()
    t_fill = time.time() - t_fill
    L, E, top_k = layout.model.num_moe_layers, layout.model.experts_per_layer, layout.model.top_k
    routed = w.tokens_per_rank * top_k
    counters = DeviceTokenCounters(L, E, dev, DeviceTokenCounters.capacity_for(
        w.capacity_factor, [routed] * L, E))
    persist = args.persist if args.persist != "auto" else ("shm" if world == 1 else "none")
    store_root = None
    store = None
    if persist != "none":
        base = "/dev/shm" if persist == "shm" else tempfile.gettempdir()
        store_root = tempfile.mkdtemp(prefix="pec_bench_", dir=base)
        store = DiskStore(store_root, io_threads=len(os.sched_getaffinity(0)),
                          direct_io=args.direct_io)
    control = None
    if world > 1 and store is not None:
        import torch.distributed as dist
        control = dist.new_group(backend="gloo")
    mode = {"vec": D.MODE_VEC, "bulk": D.MODE_BULK, "crc": D.MODE_CRC}[args.engine]
    ck = PecCheckpointer(layout, arena, store, w.pec, w.strategy, i_ckpt=1, ranks=[rank],
                         counters=counters, control_group=control, pack_mode=mode,
                         chunk_log2=args.chunk_log2)
    eng = ck.engine
    eng.pipelined_drain = not args.no_pipelined_drain
    eng.reserve(ck.max_snapshot_bytes(), host_buffers=0)
    k_s = w.pec.k_snapshot
    sel = torch.empty((L, min(k_s, E)), dtype=torch.int32, device=dev)
    stream = eng.pack_stream

    ids_step = torch.randint(0, E, (L, routed), dtype=torch.int32, device=dev,
                             generator=torch.Generator(device=dev).manual_seed(1234 + rank))
    pt = getattr(eng, "template", None)
    la_bytes = None
    if plan is None:
        # payload of the load-aware steps: measured from the host mirror of
        # each step's selection after the timed region
        la_bytes = []

    def step(c):
        """One checkpoint's device work; returns (t0, t1, bytes or None).
        sequential: select kernel + pack of the plan phase; load-aware: one
        iteration's token histogram + two-tier selection + device plan
        expansion + pack (no host synchronisation)."""
        if plan is not None:
            p = plan.phase_of(c)
            D.select_sequential(c, L, E, k_s, w.pec.k_persist, sel, stream=stream)
            return eng.pack_only(plan.assignments[p], plan_key=("phase", p), stream=stream)
        with torch.cuda.stream(stream):
            counters.add_iteration(ids_step, stream=stream)
            snap_d, pers_d = counters.select(k_s, w.pec.k_persist, stream=stream)
        a, b = eng.pack_only_device(snap_d, stream=stream)
        la_bytes.append(snap_d)
        return a, b, None

    if plan is not None:
        # every phase's device table (and CRC scratch) is built before timing
        for p in range(plan.period):
            eng.layouts_for(plan.assignments[p], ("phase", p))
    for c in range(args.warmup):
        step(c)
    stream.synchronize()
    barrier(world)
    torch.cuda.synchronize()

    # ---- timed device region: inputs resident in HBM ------------------------
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    evs = []
    moved = 0
    # L2 (126 MB) must not serve a step's bytes from the previous step: the
    # default workloads move >= 0.85 GB per step; smaller ones get a 512 MiB
    # write between steps, inside the timed region (and say so in config)
    step_bytes = (max(plan.workload_bytes[p][rank] for p in range(plan.period))
                  if plan is not None else pt.max_bytes)
    flush = None
    if 2 * step_bytes < (1 << 30):
        flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    with ClockSampler(local) as clk:
        t0.record(stream)
        for k in range(args.steps):
            if flush is not None:
                with torch.cuda.stream(stream):
                    flush.fill_(k & 0xFF)
            a, b, n = step(args.warmup + k)
            evs.append((a, b))
            moved += n or 0
        t1.record(stream)
        stream.synchronize()
    torch.cuda.synchronize()
    barrier(world)
    elapsed_ms = t0.elapsed_time(t1)
    pack_ms = [a.elapsed_time(b) for a, b in evs]
    if plan is None:
        # bytes of each load-aware step from the host mirror of its selection
        sels = la_bytes[-args.steps:]
        moved = 0
        for sd in sels:
            h = sd.cpu().tolist()
            due = {m: frozenset(x for x in h[m] if x >= 0) for m in range(L)}
            moved += sum(a.stop - a.start for a in pt.select(due))
    max_ms = max_over_ranks(elapsed_ms, world, dev)
    total_moved = sum_over_ranks(moved, world, dev)
    value = total_moved / (max_ms / 1e3) / 1e9

    hbm_peak, peak_kind = measured_peaks()
    avg_pack_ms = statistics.mean(pack_ms)
    achieved = 2 * (moved / args.steps) / (avg_pack_ms / 1e3) / 1e9
    traffic = None
    tp = ROOT / "profiles" / "pack_traffic.json"
    if tp.exists():
        try:
            traffic = json.loads(tp.read_text()).get(w.name)
        except Exception:
            traffic = None

    # ---- e2e through the public API: router ids H2D -> count -> select ->
    #      pack -> drain into pinned host memory (SNAPSHOTTED) -> host read;
    #      the persist of each version runs behind on the persist thread
    e2e = None
    persist_info = None
    pin_s = 0.0
    if not (args.no_e2e and args.no_stall):
        # pin the host snapshot buffers once, before any timing (pinning runs
        # at ~4-5 GB/s; a training job does this at start-up): 3 with a
        # persist tier, 2 without (buffers then recycle through RECOVERY)
        tpin = time.perf_counter()
        pin_error = None
        want = 3 if store is not None else 2
        # never pin more than ~70 % of the node's available RAM (all local
        # ranks pin at once); every rank uses the node-wide minimum
        fit = host_buffers_that_fit(eng.staging.numel(), want)
        n_host = int(-max_over_ranks(-float(fit), world, dev))
        if n_host < want:
            print(f"bench: host RAM fits {n_host} of {want} pinned snapshot buffers per rank",
                  file=sys.stderr)
        # pinned buffers each leg cycles through (an unpinned one would be
        # allocated inside a timed region): the stall loop needs RECOVERY +
        # PERSISTING + SNAPSHOTTING with a persist tier (2 without); the e2e
        # leg holds the persist tier, so its warm step plus every timed step
        # need their own buffer with one (buffers recycle without)
        if n_host < (3 if store is not None else 2):
            args.no_stall = True
        warm_e2e = n_host >= 2
        if store is not None:
            e2e_cap = n_host - 1 if warm_e2e else 1
        else:
            e2e_cap = 2 if warm_e2e else 1
        args.e2e_steps = max(1, min(args.e2e_steps, e2e_cap))
        if n_host < 1:
            pin_error = "host RAM too small for one pinned snapshot buffer per local rank"
        else:
            try:
                eng.reserve(eng.staging.numel(), host_buffers=n_host)
            except (RuntimeError, MemoryError, OSError) as exc:  # e.g. pinning refused
                pin_error = f"{type(exc).__name__}: {exc}"[:200]
        pin_s = time.perf_counter() - tpin
        if max_over_ranks(1.0 if pin_error else 0.0, world, dev) > 0:
            # every rank skips the host-buffer legs together (no stranded collectives)
            print(f"bench: pinned host buffers unavailable ({pin_error}); "
                  "skipping e2e and stall legs", file=sys.stderr)
            args.no_e2e = args.no_stall = True
    link_alone = link_conc = None
    if not args.no_e2e:
        # host-link roofline measured in this run (1 GiB pinned D2H, best of 3,
        # after the buffers' first touch): each rank alone in turn, then all
        # N ranks at once (max over ranks)
        n_ = min(1 << 30, eng.staging.numel(), eng.host[0].numel())
        eng.host[0][:n_].copy_(eng.staging[:n_])  # first touch of the pinned pages

        def d2h_ms():
            a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a_.record(eng.copy_stream)
            with torch.cuda.stream(eng.copy_stream):
                eng.host[0][:n_].copy_(eng.staging[:n_], non_blocking=True)
            b_.record(eng.copy_stream)
            b_.synchronize()
            return a_.elapsed_time(b_)

        alone = 1e30
        for r_ in range(world):
            barrier(world)
            if r_ == rank:
                alone = min(d2h_ms() for _ in range(3))
        barrier(world)
        conc = 1e30
        for _ in range(3):
            barrier(world)
            torch.cuda.synchronize()
            conc = min(conc, max_over_ranks(d2h_ms(), world, dev))
        link_alone = n_ / (alone / 1e3) / 1e9
        link_conc = n_ / (conc / 1e3) / 1e9
    if not args.no_e2e:
        e2e_steps = max(1, min(args.e2e_steps, 2))  # <= 2 so no buffer waits on persist
        rng = np.random.default_rng(1234 + rank)
        ids_host = [torch.from_numpy(rng.integers(0, E, size=(L, routed), dtype=np.int32)).pin_memory()
                    for _ in range(e2e_steps + 1)]
        ids_dev = torch.empty((L, routed), dtype=torch.int32, device=dev)
        # first D2H into a freshly pinned buffer runs slow (IOMMU/page-table
        # warm-up): touch every host buffer once before timing
        for hb in eng.host:
            if hb is not None:
                n_ = min(hb.numel(), eng.staging.numel())
                hb[:n_].copy_(eng.staging[:n_])
        h2d = d2h = 0
        base_it = args.warmup + args.steps + 10

        def e2e_step(k, it):
            nonlocal h2d, d2h
            ids_dev.copy_(ids_host[k], non_blocking=True)
            h2d += ids_host[k].numel() * 4
            counters.add_iteration(ids_dev)
            buf = ck.checkpoint(it)               # select + plan + pack + drain
            ck.wait_snapshot(buf)                 # wait for SNAPSHOTTED
            first = eng.snapshot_layout(buf, rank).entries[0]
            _ = int(eng.entry_view(buf, rank, first.store_key)[0])  # host read
            d2h += eng.snapshot_nbytes(buf)

        # one untimed step through the same calls (first-call host costs), then
        # its persist drains before the timed steps
        if warm_e2e:
            e2e_step(e2e_steps, base_it - args.i_ckpt)
            ck.finish()
        h2d = d2h = 0
        n_persist0 = len(eng.stats["persist_s"])
        barrier(world)
        torch.cuda.synchronize()
        ck.hold_persist(True)   # measure the snapshot tier alone; persist after
        tw = time.perf_counter()
        for k in range(e2e_steps):
            e2e_step(k, base_it + k)
        e2e_s = time.perf_counter() - tw
        e2e_s = max_over_ranks(e2e_s, world, dev)
        e2e_moved = sum_over_ranks(sum(eng.stats["snap_bytes"][-e2e_steps:]), world, dev)
        e2e = {"value": round(e2e_moved / e2e_s / 1e9, 3), "unit": UNIT,
               "h2d_bytes_per_step": h2d // e2e_steps, "d2h_bytes_per_step": d2h // e2e_steps,
               "steps": e2e_steps, "ms_per_step": round(e2e_s / e2e_steps * 1e3, 2),
               "drain_ms": [round(x, 2) for x in eng.stats["drain_ms"][-e2e_steps:]],
               "what": "router-id H2D + count + select + pack + D2H drain to pinned host",
               "host_pin_s": round(pin_s, 1)}
        tp0 = time.perf_counter()
        ck.finish()
        timed_persist = eng.stats["persist_s"][n_persist0:]
        if store is not None and timed_persist:
            persisted = sum(eng.stats["snap_bytes"][-e2e_steps:])
            persist_info = {"target": persist, "direct_io": bool(args.direct_io),
                            "versions": len(timed_persist),
                            "seconds": [round(x, 2) for x in timed_persist],
                            "GBps": round(persisted / max(sum(timed_persist), 1e-9) / 1e9, 2)}
    stall = None
    if not args.no_stall:
        prune_store(store)
        stall = measure_stall(ck, arena, dev, args.stall_iters, args.i_ckpt, args.fb_ms)
        stall["exposed_ms_per_iter"] = round(max_over_ranks(stall["exposed_ms_per_iter"],
                                                            world, dev), 3)
    ck.close()
    if store_root:
        shutil.rmtree(store_root, ignore_errors=True)

    # ---- CPU baseline (rank 0, N == 1 only) ----------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = len(os.sched_getaffinity(0))
        if plan is not None:
            first_layout = eng.layouts_for(plan.assignments[0], ("phase", 0))[rank]
        else:
            first_layout = StagingLayout.build(pt.select({m: frozenset({m % E})
                                                          for m in range(L)}), arena, rank)
        gbs, desc = cpu_pack_sample(first_layout.entries, int(args.cpu_sample_gb * 1e9), threads,
                                    args.cpu_seconds)
        cpu = {"value": round(gbs, 3), "unit": UNIT, "cores": threads, "kind": "port",
               "sample": desc, "cpu_model": cpu_model()}
        try:
            cpu["components"] = cpu_components(layout, w.strategy, w.pec.k_pec)
        except Exception as exc:  # reported, never fatal to the bench line
            cpu["components"] = {"error": f"{type(exc).__name__}: {exc}"[:200]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(max_ms / args.steps, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": w.name, "plan": w.strategy, "selection": w.pec.selection,
                       "k_pec": w.pec.k_pec,
                       "ranks": f"0..{world - 1} of dp={layout.n_ranks}",
                       "bytes_per_step_rank0": moved // args.steps,
                       "state_resident_gb": round(arena.resident_bytes() / 1e9, 2),
                       "engine": args.engine, "chunk_log2": args.chunk_log2,
                       "l2": (f"no flush needed: each step reads "
                              f"{(moved // args.steps) / 1e9:.2f} GB (> 126 MB L2)"
                              if flush is None else
                              "512 MiB L2 flush written between steps, inside the timed "
                              "region (steps move less than 4x the 126 MB L2)"),
                       "parallelism": f"dp{layout.n_ranks}-ep{layout.parallel.ep_degree}"},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_peak,
                         "unit": "GB/s", "frac": round(achieved / hbm_peak, 4),
                         "traffic": traffic, "peak_kind": peak_kind,
                         # frac > 1 is possible: `peak` is torch's copy_ kernel, and the
                         # TMA bulk ring moves bytes faster than it; the nominal HBM3e
                         # figure (7.7 TB/s, B200_PROFILING.md) bounds both
                         "nominal": HBM_NOMINAL_GBS,
                         "frac_of_nominal": round(achieved / HBM_NOMINAL_GBS, 4),
                         "kernel": f"pec_pack ({args.engine})",
                         "avg_launch_ms": round(avg_pack_ms, 4)},
            "e2e": e2e,
            "host_link": ({"achieved": round(statistics.mean(
                              [e2e["d2h_bytes_per_step"] / (m / 1e3) / 1e9 for m in e2e["drain_ms"]]), 2),
                           "peak": round(link_alone, 2), "unit": "GB/s",
                           "peak_kind": "measured in this run: 1 GiB pinned D2H, this GPU alone, "
                                        "best of 3",
                           "peak_all_gpus_concurrent": round(link_conc, 2)}
                          if e2e else None),
            "persist": persist_info,
            "stall": stall,
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
            # our kernels per timed step: selection (1 sequential; hist + 2
            # selects + plan expansion load-aware) + the pack (1 launch; the
            # CRC engine adds its chunk fold and final kernels)
            "gpu_launches": ((1 if plan is not None else 4) +
                             (3 if args.engine == "crc" else 1)) * args.steps,
            "fill_s": round(t_fill, 2),
        }
        if line["host_link"]:
            hl = line["host_link"]
            hl["frac"] = round(hl["achieved"] / link_alone, 4)
            hl["frac_of_concurrent"] = round(hl["achieved"] / link_conc, 4)
            # e2e is bounded by the host link every GPU drains through at once
            e2e["per_gpu"] = round(e2e["value"] / world, 3)
            e2e["frac_of_host_link"] = round(e2e["per_gpu"] / link_conc, 4)
        emit(line)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


_RESULT = None  # the real stdout: the JSON line only


def _claim_stdout() -> None:
    """Route fd 1 to stderr for the whole run and keep the original stdout
    for the one JSON line: libraries that print from C (NCCL's version
    banner on rank 0 under torchrun) cannot corrupt the contract line."""
    global _RESULT
    sys.stdout.flush()
    _RESULT = os.fdopen(os.dup(1), "w", buffering=1)
    os.dup2(2, 1)


def emit(line: dict) -> None:
    print(json.dumps(line), file=_RESULT or sys.stdout, flush=True)


def main():
    _claim_stdout()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="mixtral",
                    choices=["toy", "gpt125m", "gpt350m", "gpt350m_la", "mixtral"])
    ap.add_argument("--engine", default="crc", choices=["vec", "bulk", "crc"],
                    help="pack engine: TMA bulk ring with fused per-entry CRC-32C (default; "
                         "the persist tier then never reads payloads for checksums), plain "
                         "TMA bulk, or LDG/STG vector")
    ap.add_argument("--chunk-log2", type=int, default=15)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--persist", default="auto", choices=["auto", "none", "shm", "disk"])
    ap.add_argument("--direct-io", action="store_true",
                    help="persist with O_DIRECT (meaningful with --persist disk)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-stall", action="store_true")
    ap.add_argument("--no-pipelined-drain", action="store_true",
                    help="drain each snapshot only after its whole pack (A/B of the default)")
    ap.add_argument("--stall-iters", type=int, default=40)
    ap.add_argument("--i-ckpt", type=int, default=10)
    ap.add_argument("--fb-ms", type=float, default=100.0)
    ap.add_argument("--cpu-sample-gb", type=float, default=2.0)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "b200":
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
