#!/usr/bin/env python
"""PEC snapshot benchmark (the driver's bench contract).

One *step* = one PEC checkpoint snapshot of this rank's shard: on-device K_pec
selection for checkpoint c, then the pack of the rank's planned byte ranges
(experts' bf16 weights + fp32 master/m/v, its ZeRO-2 non-expert optimizer
shard, its share of the non-expert weights) from the HBM state arena into the
HBM staging buffer, with every entry's CRC-32C computed in the same pass (the
default engine).  `value` is that with the state already resident in HBM: the
training-blocking part of a snapshot.  `e2e` is the reference's SNAPSHOTTED
state (bytes in CPU memory, simulator.py:434-438) through the package's public
API: router-id H2D + count + select + pack + copy-engine drain into a pinned
host snapshot buffer + host read, every step.

Workload (default): Mixtral-8x7B-shaped state, K_pec=1, adaptive_pec plan of
the dp=ep=8 deployment; with N GPUs, ranks 0..N-1 of that plan (weak scaling:
each GPU holds the same-size ~85 GB rank shard at every N).

Legs (all in one run): device steps (`value`, `roofline`), host-link peaks,
e2e (>= 5 steps, snapshot tier only), one persist probe, the checkpoint
cadence the policy derives from this run's measured pack / drain / persist
rates, then the steady-state training-stall A/B with the persist tier on
(>= 12 checkpoints per arm, every drain and persist inside the timed window),
and on rank 0 at N=1 the CPU baseline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
"""

from __future__ import annotations

import argparse
import importlib
import json
import math
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
    """SM clocks + throttle reasons sampled during the timed region: NVML
    polled every 10 ms on a thread (the value leg lasts ~80 ms, too short for
    nvidia-smi's 100 ms floor), nvidia-smi -lms 100 when NVML is missing."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, gpu_index: int, period_s: float = 0.01):
        self.gpu = gpu_index
        self.period = period_s
        self.proc = None
        self.lines = []
        self.samples = []            # (sm_mhz, max_mhz, set of reasons)
        self._stop = threading.Event()
        self._t = None
        self.source = "none"

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            bits = {"hw_slowdown": pynvml.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": pynvml.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": pynvml.nvmlClocksEventReasonSwPowerCap}
            mx = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))

            def poll():
                while not self._stop.is_set():
                    sm = float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                    r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.samples.append((sm, mx, {k for k, b in bits.items() if r & b}))
                    self._stop.wait(self.period)
            self._t = threading.Thread(target=poll, daemon=True)
            self._t.start()
            self.source = "nvml, 10 ms"
            return self
        except Exception:  # noqa: BLE001 - fall back to nvidia-smi
            pass
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
            self.source = "nvidia-smi, 100 ms"
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
        elif self._t is not None:
            self._stop.set()
            self._t.join(timeout=5)

    def summary(self):
        samples = list(self.samples)
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                samples.append((float(f[1]), float(f[2]),
                                {n for n, v in zip(self.NAMES, f[5:9]) if v.lower() == "active"}))
            except ValueError:
                continue
        sm = [x[0] for x in samples]
        reasons = set().union(*[x[2] for x in samples]) if samples else set()
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": samples[-1][1] if samples else None,
                "reasons": sorted(reasons), "samples": len(sm), "source": self.source}


def dist_backend() -> str:
    """NCCL (the contract).  PEC_DIST_BACKEND=gloo exists only to exercise
    the N-rank code path with more ranks than GPUs (ranks then share devices
    round-robin, which NCCL refuses); it is reported in the line."""
    return os.environ.get("PEC_DIST_BACKEND", "nccl")


def dist_init(n_gpus):
    import torch
    rank, local, world = env_rank()
    local = local % max(1, torch.cuda.device_count())
    if world > 1:
        import torch.distributed as dist
        if dist_backend() == "gloo":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, local, world


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def _reduce(x, world, device, op):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64,
                     device="cpu" if dist_backend() == "gloo" else device)
    dist.all_reduce(t, op=op)
    return float(t.item())


def max_over_ranks(x, world, device):
    import torch.distributed as dist
    return _reduce(x, world, device, dist.ReduceOp.MAX if world > 1 else None)


def min_over_ranks(x, world, device):
    return -max_over_ranks(-x, world, device)


def sum_over_ranks(x, world, device):
    import torch.distributed as dist
    return _reduce(x, world, device, dist.ReduceOp.SUM if world > 1 else None)


def mem_available() -> int:
    try:
        with open("/proc/meminfo") as f:
            info = {ln.split(":")[0]: int(ln.split()[1]) * 1024 for ln in f if ":" in ln}
        return info.get("MemAvailable", info.get("MemFree", 0))
    except OSError:
        return 0


def host_buffers_that_fit(nbytes: int, want: int, frac: float = 0.7, reserve: int = 0) -> int:
    """How many pinned host snapshot buffers of ``nbytes`` each local rank
    can take (LOCAL_WORLD_SIZE ranks pin at once) within ``frac`` of the
    node's MemAvailable, after ``reserve`` bytes per rank for other uses
    (the persist tier's /dev/shm versions)."""
    avail = mem_available()
    if not avail:
        return want
    local = max(1, int(os.environ.get("LOCAL_WORLD_SIZE", "1")))
    per_rank = frac * avail / local - reserve
    return max(0, min(want, int(per_rank // max(1, nbytes))))


# versions of every rank's shard the /dev/shm persist tier holds at once in
# steady state: the newest complete one (retention keeps 1), one being written,
# one complete but not yet pruned (retention runs on a background thread)
SHM_VERSIONS_IN_FLIGHT = 3

# versions the persist probe writes before taking its rate (the policy's
# persist bandwidth): the first ones pay tmpfs page allocation, the last one
# is the steady-state cost
PERSIST_PROBE_VERSIONS = 3
# then versions checkpointed back to back (drain and persist overlapping as in
# training); their rates, times CADENCE_MARGIN, set the policy's I_ckpt floor
SUSTAINED_PROBE_VERSIONS = 4
CADENCE_MARGIN = 1.1
# the stall leg's runtime check of that cadence: up to CADENCE_TRIALS short
# checkpointed runs of TRIAL_CHECKPOINTS checkpoints; any host wait -> I_ckpt x4/3
CADENCE_TRIALS = 3
TRIAL_CHECKPOINTS = 4


def tmpfs_room(root, need_bytes: int, margin: float = 1.05):
    """(free bytes, too small?) of the filesystem holding ``root`` for
    ``need_bytes`` (+5 %) of persist versions; (None, False) when unknown."""
    try:
        st = os.statvfs(str(root))
    except OSError:
        return None, False
    free = st.f_bavail * st.f_frsize
    return free, free < margin * need_bytes


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ---------------------------------------------------------------------------
# The reference's CPU path: its own planner on host cores
# ---------------------------------------------------------------------------

def load_reference():
    """The UNMODIFIED reference package `mocsim`: installed into
    baseline/_ref (pip --target, travels to the GPU box), else imported in
    place from /root/reference (this container).  (module, where) or
    (None, why)."""
    for path, where in ((ROOT / "baseline" / "_ref", "baseline/_ref"),
                        (Path("/root/reference/pkg/src"), "/root/reference")):
        if (path / "mocsim" / "__init__.py").exists():
            sys.path.insert(0, str(path))
            try:
                return importlib.import_module("mocsim"), where
            finally:
                sys.path.remove(str(path))
    return None, "mocsim not installed (baseline/_ref missing)"


def reference_layout(ref, w):
    """The workload's layout built by the reference's own topology code from
    the same spec numbers (reference topology.py:286-356)."""
    import dataclasses
    m = ref.ModelSpec(**{f.name: getattr(w.model, f.name) for f in dataclasses.fields(w.model)})
    p = ref.ParallelSpec(**{f.name: getattr(w.parallel, f.name)
                           for f in dataclasses.fields(w.parallel)})
    c = ref.ClusterSpec(**{f.name: getattr(w.cluster, f.name)
                          for f in dataclasses.fields(w.cluster)})
    return ref.build_layout(m, p, c)


def reference_ranges(ref, w, layout, rank: int):
    """Rank ``rank``'s ranges of checkpoint 0 from the reference planner:
    the periodic plan (planner.py:298-353) for sequential selection, the
    per-checkpoint build_phase_assignment (planner.py:263-295) for a
    load-aware due set of the same size."""
    pec = ref.PecConfig(k_pec=w.pec.k_pec, selection=w.pec.selection,
                        k_snapshot=w.pec.k_snapshot, k_persist=w.pec.k_persist)
    if w.pec.selection == "load_aware":
        n = layout.model.experts_per_layer
        due = {m: ref.select_window(0, m, n, pec.k_snapshot, pec.k_snapshot)
               for m in range(layout.model.num_moe_layers)}
        return ref.planner.build_phase_assignment(layout, due, w.strategy).get(rank, ())
    plan = ref.plan_adaptive(layout, pec) if w.strategy == "adaptive_pec" \
        else ref.plan_equal(layout, pec)
    return plan.assignments[0].get(rank, ())


def host_copies(layout, ranges, rank: int, cap_bytes: int = 0):
    """(src, dst, n) copies of a rank's ranges over a host image of the
    units they read (layout order, 256-byte aligned), packed back to back;
    ``cap_bytes`` > 0 cuts every range to the same fraction (tests)."""
    used = {a.key for a in ranges if a.stop > a.start}
    off, pos = {}, 0
    for u in layout.units:
        if u.key in used:
            off[u.key] = pos
            pos = (pos + u.size_bytes + 255) // 256 * 256
    total = sum(a.stop - a.start for a in ranges)
    frac = 1.0 if not cap_bytes or cap_bytes >= total else cap_bytes / total
    copies, dst = [], 0
    for a in ranges:
        n = a.stop - a.start
        if n <= 0:
            continue
        n = n if frac == 1.0 else max(256, int(n * frac))
        copies.append((off[a.key] + a.start, dst, n))
        dst += n
    return copies, pos, dst


def fill_sources(state, copies, threads: int) -> None:
    """First touch of every source range (a byte pattern), multi-threaded."""
    from concurrent.futures import ThreadPoolExecutor
    piece = 64 << 20
    jobs = [(s + o, min(piece, n - o)) for s, _, n in copies for o in range(0, n, piece)]

    def run(job):
        s, n = job
        state[s:s + n] = (s >> 20) & 0xFF

    with ThreadPoolExecutor(max_workers=threads) as ex:
        list(ex.map(run, jobs))


def reference_components(ref, layout, w):
    """The reference's other per-checkpoint CPU costs, its own code as-is:
    two-tier load-aware selection (select_load_aware per layer and tier,
    selector.py:91-100 as called by simulator.py:339-354), one
    build_phase_assignment (planner.py:263-295), one plan_adaptive
    (planner.py:335-342) and its pure-Python CRC-32C (store.py:49-70) on
    1 MiB, one core."""
    m = layout.model
    L, E, k = m.num_moe_layers, m.experts_per_layer, w.pec.k_pec
    rng = np.random.default_rng(1)
    counts = rng.integers(0, 1 << 20, (2, L, E))
    tiers = []
    for t in range(2):
        lc = ref.LoadCounters(L, E)
        for li in range(L):
            for e in range(E):
                lc.unsaved_tokens[(li, e)] = int(counts[t, li, e])
        tiers.append(lc)

    def timed(fn, budget=0.5):
        t0, reps = time.perf_counter(), 0
        while True:
            fn()
            reps += 1
            if time.perf_counter() - t0 >= budget:
                return (time.perf_counter() - t0) / reps

    def two_tier():
        for li in range(L):
            s = ref.select_load_aware(tiers[0], li, k)
            ref.select_load_aware(tiers[1], li, k, restrict_to=s)

    pec = ref.PecConfig(k_pec=k)
    due = {li: frozenset(range(k)) for li in range(L)}
    data = rng.integers(0, 256, 1 << 20, dtype=np.uint8).tobytes()
    return {"select_two_tier_us": round(timed(two_tier) * 1e6, 1),
            "build_phase_assignment_ms": round(timed(
                lambda: ref.planner.build_phase_assignment(layout, due, w.strategy)) * 1e3, 3),
            "plan_adaptive_ms": round(timed(lambda: ref.plan_adaptive(layout, pec), 1.0) * 1e3, 2),
            "py_crc32c_MBps_1core": round(len(data) / timed(lambda: ref.crc32c(data), 0.2) / 1e6,
                                          2),
            "what": "the reference's own select_load_aware x L layers x 2 tiers, "
                    "build_phase_assignment, plan_adaptive, crc32c (mocsim, unmodified)"}


def cpu_pack_shards(w, n_ranks: int, steps: int, warmup: int, threads: int,
                    cap_bytes: int = 0, min_seconds: float = 0.0):
    """Pack ranks 0..n_ranks-1's checkpoint-0 shards — ranges from the
    reference's own planner — on the host cores, one after another in every
    step, with the oracle's threaded numpy pack (the reference moves no bytes:
    it models the snapshot as bytes / bandwidth, simulator.py:57-61).
    Returns (per-step seconds, payload bytes per step, description, ref,
    layout)."""
    from oracle import pec_oracle as O
    ref, where = load_reference()
    if ref is not None:
        layout = reference_layout(ref, w)
        get = lambda r: reference_ranges(ref, w, layout, r)  # noqa: E731
        src_of = f"mocsim planner ({where})"
    else:
        from paper_2408_04307_b200 import build_phase_assignment, plan_adaptive
        from paper_2408_04307_b200.selector import select_window
        layout = w.layout()
        plan = None if w.pec.selection == "load_aware" else plan_adaptive(layout, w.pec)

        def get(r):
            if plan is not None:
                return plan.assignments[0].get(r, ())
            n = layout.model.experts_per_layer
            due = {m: select_window(0, m, n, w.pec.k_snapshot, w.pec.k_snapshot)
                   for m in range(layout.model.num_moe_layers)}
            return build_phase_assignment(layout, due, w.strategy).get(r, ())
        src_of = f"this package's planner ({where})"
    shards = [host_copies(layout, get(r), r, cap_bytes) for r in range(n_ranks)]
    state = np.empty(max(s[1] for s in shards) + 256, dtype=np.uint8)
    out = np.empty(max(s[2] for s in shards) + 256, dtype=np.uint8)
    for copies, _, _ in shards:
        fill_sources(state, copies, threads)
    payload = sum(s[2] for s in shards)
    times = []
    t_start = time.perf_counter()
    k = 0
    while True:
        t0 = time.perf_counter()
        for copies, _, _ in shards:
            O.pack_threaded(state, copies, out, threads)
        dt = time.perf_counter() - t0
        if k >= warmup:
            times.append(dt)
        k += 1
        if k >= warmup + steps and time.perf_counter() - t_start >= min_seconds:
            break
    n_entries = sum(len(s[0]) for s in shards)
    who = f"ranks 0..{n_ranks - 1}" if n_ranks > 1 else "rank 0"
    desc = (f"oracle threaded numpy pack of {who}'s full checkpoint-0 shard(s) "
            f"({payload / 1e9:.2f} GB, {n_entries} entries, ranges from {src_of}) "
            f"from host-resident state, x{len(times)} timed passes, {threads} threads")
    if cap_bytes:
        desc += f" [capped to {cap_bytes / 1e9:.2f} GB per rank]"
    return times, payload, desc, ref, layout


def run_reference(args):
    rank, local, world = env_rank()
    if rank != 0:
        return 0
    n_ranks = max(1, args.gpus)
    threads = len(os.sched_getaffinity(0))
    w, _, _ = build_workload(args, 0)
    cap = int(args.cpu_sample_gb * 1e9) if args.cpu_sample_gb else 0
    times, payload, desc, ref, layout = cpu_pack_shards(w, n_ranks, args.steps, args.warmup,
                                                        threads, cap)
    value = payload / statistics.mean(times) / 1e9
    try:
        comps = reference_components(ref, layout, w) if ref is not None else \
            {"error": "reference not importable"}
    except Exception as exc:  # reported, never fatal to the line
        comps = {"error": f"{type(exc).__name__}: {exc}"[:200]}
    line = {"metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(statistics.mean(times) * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": w.name, "plan": w.strategy, "selection": w.pec.selection,
                       "k_pec": w.pec.k_pec,
                       "ranks": f"0..{n_ranks - 1} of dp={layout.parallel.dp_degree} "
                                "(host cores, one after another)",
                       "parallelism": f"dp{layout.parallel.dp_degree}-"
                                      f"ep{layout.parallel.ep_degree}",
                       "bytes_per_step": payload, "same_config": not cap},
            "cpu_baseline": {"value": round(value, 3), "unit": UNIT, "cores": threads,
                             "kind": "port", "sample": desc, "cpu_model": cpu_model(),
                             "components": comps},
            "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    emit(line)
    return 0


# ---------------------------------------------------------------------------
# B200 arm
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


def prune_store(store, keep: int = 1, ranks=None, coordinator: bool = True) -> int:
    """Bench-only retention of a /dev/shm persist tier (host RAM): every
    version older than the newest ``keep`` complete ones is retired — each
    rank process retires its own rank directories (freeing or recycling
    tmpfs pages runs at ~10-20 GB/s per thread, so one deleter cannot keep
    up with N ranks' versions) and the coordinator removes the version
    itself once no rank directory is left (`DiskStore.retire`; with
    ``recycle`` the entry files become spares later versions overwrite in
    place).  Returns the number of old versions still present."""
    if store is None or not hasattr(store, "version_dir"):
        return 0
    complete = store.complete_versions()
    if not complete or len(complete) < keep:
        return 0
    # not `<= keep`: the coordinator unlinks COMPLETE first, so the other
    # ranks may see only the kept versions while older ones still hold files
    cutoff = complete[-keep] if keep else complete[-1] + 1
    left = 0
    for v in store.version_numbers():
        if v >= cutoff:
            break
        if not store.retire(v, ranks=ranks, coordinator=coordinator):
            left += 1
    if ranks is not None and getattr(store, "recycle", False):
        # spares beyond one version's worth of this rank's files are dropped
        store.trim_spares(ranks, keep_bytes=store_bytes_per_version.get(id(store), 1 << 62))
    return left


# bench-side record of one version's bytes per rank (the spare-pool cap)
store_bytes_per_version = {}


class Retention:
    """`prune_store` on a background thread of every rank: freeing a
    version's tmpfs pages takes ~0.5 s per 12.6 GB, which must not block the
    training thread (a blocked launch thread starves the GPU).  Memory is
    bounded all the same: when more than ``max_old`` superseded versions are
    still present, `submit` waits for the deleter (never observed at the
    policy's cadence; a guard against running the node out of RAM)."""

    def __init__(self, store, ranks, coordinator: bool, keep: int = 1, max_old: int = 1):
        import queue
        self.store, self.keep, self.ranks = store, keep, list(ranks)
        self.coordinator, self.max_old = coordinator, max_old
        self.q = queue.Queue()
        self.left = 0
        self.waited_s = 0.0
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    def _run(self):
        while True:
            item = self.q.get()
            if item is None:
                self.q.task_done()
                return
            self.left = prune_store(self.store, self.keep, self.ranks, self.coordinator)
            self.q.task_done()

    def submit(self):
        if len(self.store.version_numbers()) - self.keep - 1 > self.max_old:
            t0 = time.perf_counter()
            self.q.join()                       # back-pressure: let the deleter catch up
            self.waited_s += time.perf_counter() - t0
        if self.q.empty():
            self.q.put(1)

    def close(self):
        self.q.put(None)
        self.t.join()


def sweep_stale_stores(base: str = "/dev/shm") -> None:
    """Remove persist stores of earlier bench runs whose process is gone (a
    killed run leaves its versions in host RAM)."""
    import glob
    import shutil
    for d in glob.glob(os.path.join(base, "pec_bench_*")):
        owner = os.path.basename(d).split("_")[2] if d.count("_") >= 3 else ""
        if owner.isdigit() and not os.path.exists(f"/proc/{owner}"):
            shutil.rmtree(d, ignore_errors=True)


def measure_host_link(eng, world, dev):
    """Host-link roofline measured in this run, on the drain's own path (the
    copy stream, 256 MiB pieces): 4 GiB pinned D2H (or the whole staging
    buffer if smaller), best of 5, each rank alone in turn, then all ranks
    started together (per-trial max over ranks).  With one GPU the two are
    the same measurement."""
    import torch
    n = min(4 << 30, eng.staging.numel(), eng.host[0].numel())
    eng.host[0][:n].copy_(eng.staging[:n])  # first touch of the pinned pages
    rank = int(os.environ.get("RANK", 0))

    def d2h_ms():
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(eng.copy_stream)
        with torch.cuda.stream(eng.copy_stream):
            eng._drain_range(eng.host[0], 0, n)
        b.record(eng.copy_stream)
        b.synchronize()
        return a.elapsed_time(b)

    alone = 1e30
    for r in range(world):
        barrier(world)
        if r == rank:
            alone = min(d2h_ms() for _ in range(5))
    link_alone = n / (alone / 1e3) / 1e9
    if world == 1:
        return link_alone, link_alone
    conc = 1e30
    for _ in range(5):
        barrier(world)
        torch.cuda.synchronize()
        conc = min(conc, max_over_ranks(d2h_ms(), world, dev))
    return link_alone, n / (conc / 1e3) / 1e9


def measure_stall(ck, arena, dev, i_ckpt: int, n_ckpt: int, fb_ms: float, rounds: int,
                  world: int, rank: int):
    """Steady-state training-stall A/B on a synthetic per-rank loop: an F&B
    proxy (bf16 8192^3 GEMMs, ~fb_ms) then an update proxy (one in-place
    pass over the whole state arena: HBM-bound like a fused Adam step over the
    rank's ~85 GB shard).  The checkpointed arm takes ``n_ckpt`` checkpoints,
    one every ``i_ckpt`` iterations after the update, with the persist tier
    ON (retention keeps the newest complete version), then runs one more interval
    without a checkpoint, then waits for every drain and persist — all inside
    the timed window, so a persist tier that cannot keep up shows as stall.
    The next update always waits for the pending pack.  Arms alternate
    (A B A B) so drifts hit both; device time per iteration, max over ranks."""
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
    iters = (n_ckpt + 1) * i_ckpt
    store = ck.engine.store
    stats = ck.engine.stats
    retention = Retention(store, ranks=[rank], coordinator=rank == 0) \
        if store is not None else None

    def run(with_ckpt: bool, base_it: int, i_ckpt: int = i_ckpt, n_ckpt: int = n_ckpt):
        iters = (n_ckpt + 1) * i_ckpt
        barrier(world)
        torch.cuda.synchronize()
        w0 = {k: list(v) for k, v in ck.waits.items()}
        p0 = len(stats["persist_s"])
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        marks = [torch.cuda.Event(enable_timing=True) for _ in range(iters + 1)]
        host = {"checkpoint_s": 0.0, "finish_s": 0.0}
        t0.record(compute)
        marks[0].record(compute)
        for k in range(1, iters + 1):
            it = base_it + k
            for _ in range(n_gemm):                 # forward + backward
                torch.matmul(a, b, out=c)
            if with_ckpt:
                ck.poll()
                ck.wait_pack(stream=compute)        # the update may not race the pack
            words.add_(1)                           # optimizer step
            if with_ckpt and k % i_ckpt == 0 and k <= n_ckpt * i_ckpt:
                h0 = time.perf_counter()
                ck.checkpoint(it)                   # select + plan + pack + drain
                host["checkpoint_s"] += time.perf_counter() - h0
                if retention is not None:
                    retention.submit()              # bench-only: old versions off /dev/shm
            marks[k].record(compute)
        if with_ckpt:
            h0 = time.perf_counter()
            ck.finish()                             # every drain and persist, in the window
            host["finish_s"] = time.perf_counter() - h0
        t1.record(compute)
        t1.synchronize()
        waits = {k: [ck.waits[k][0] - w0[k][0], ck.waits[k][1] - w0[k][1]] for k in w0}
        per_it = [marks[k - 1].elapsed_time(marks[k]) for k in range(1, iters + 1)]
        top = sorted(range(iters), key=lambda j: -per_it[j])[:6]
        host["slowest_iters"] = [(j + 1, round(per_it[j], 2)) for j in top]
        host["median_iter_ms"] = round(statistics.median(per_it), 3)
        host["tail_ms"] = round(marks[iters].elapsed_time(t1), 2)
        return t0.elapsed_time(t1) / iters, waits, stats["persist_s"][p0:], host

    # checkpoint c = iteration // i_ckpt - 1 walks the plan's phases in order
    ck.i_ckpt = i_ckpt
    run(False, 0)  # warm
    # runtime check of the policy's cadence: a short checkpointed trial; if
    # any rank waited on a drain or for a persist-freed buffer, I_ckpt grows
    # by a third and the trial repeats (the policy's rates come from probes
    # without the training loop, which also contends for the GPU and host)
    trials = []
    if store is not None:
        for t in range(CADENCE_TRIALS):
            # iterations stay increasing: e2e/probe legs ~1e6, trials here, rounds >= 1e7
            _, tw, _, _ = run(True, i_ckpt * 10 ** 5 * (t + 2), i_ckpt=i_ckpt,
                              n_ckpt=TRIAL_CHECKPOINTS)
            n_wait = int(max_over_ranks(float(tw["snap"][0] + tw["buffer"][0]), world, dev))
            trials.append({"i_ckpt": i_ckpt, "host_waits": n_wait})
            if n_wait == 0:
                break
            i_ckpt = int(math.ceil(i_ckpt * 4 / 3))
            ck.i_ckpt = i_ckpt
            if rank == 0:
                print(f"bench: {n_wait} host waits in the cadence trial; I_ckpt -> {i_ckpt}",
                      file=sys.stderr)
    iters = (n_ckpt + 1) * i_ckpt
    runs_without, runs_with, waits_all, persists, hosts = [], [], [], [], []
    gpu = torch.cuda.current_device()
    clk_arms = {"without": [], "with": []}
    for r in range(rounds):
        with ClockSampler(gpu, period_s=0.05) as cw:
            runs_without.append(run(False, 0, i_ckpt=i_ckpt)[0])
        with ClockSampler(gpu, period_s=0.05) as cc:
            ms, waits, pers, host = run(True, i_ckpt * 10 ** 6 * (r + 1), i_ckpt=i_ckpt)
        clk_arms["without"].append(cw.summary()["sm_mhz"])
        clk_arms["with"].append(cc.summary()["sm_mhz"])
        runs_with.append(ms)
        waits_all.append(waits)
        persists += pers
        hosts.append({k: (round(v, 3) if isinstance(v, float) else v) for k, v in host.items()})
    retention_wait_s = 0.0
    if retention is not None:
        retention.close()
        retention_wait_s = retention.waited_s
    without = max_over_ranks(statistics.mean(runs_without), world, dev)
    with_ = max_over_ranks(statistics.mean(runs_with), world, dev)
    packs = stats["pack_ms"][-rounds * n_ckpt:]
    wait_sum = {k: [sum(w[k][0] for w in waits_all), sum(w[k][1] for w in waits_all)]
                for k in waits_all[0]}
    shard = statistics.mean(stats["snap_bytes"][-rounds * n_ckpt:])
    return {"i_ckpt": i_ckpt, "checkpoints_per_arm": n_ckpt, "iters_per_arm": iters,
            "rounds": rounds, "fb_ms": round(n_gemm * gemm_ms, 1), "fb_gemms": n_gemm,
            "update_ms": round(update_ms, 2),
            "iter_ms_without": round(without, 3), "iter_ms_with": round(with_, 3),
            "runs_ms_without": [round(x, 3) for x in runs_without],
            "runs_ms_with": [round(x, 3) for x in runs_with],
            "exposed_ms_per_iter": round(with_ - without, 3),
            "noise_ms_per_iter": round((max(runs_without) - min(runs_without)) / 2, 3),
            "pack_ms_in_loop": round(statistics.mean(packs), 3) if packs else None,
            "overhead_frac": round((with_ - without) / without, 5),
            "host_waits": {"snapshot_drain": {"count": wait_sum["snap"][0],
                                              "s": round(wait_sum["snap"][1], 3)},
                           "buffer_for_persist": {"count": wait_sum["buffer"][0],
                                                  "s": round(wait_sum["buffer"][1], 3)},
                           "what": "host time at checkpoints waiting for the previous drain / "
                                   "for a persist to free a buffer (NoFreeBufferError, "
                                   "simulator.py:413-422), summed over the checkpointed arms"},
            "persist_in_window": {"versions": len(persists),
                                  "s_mean": round(statistics.mean(persists), 3) if persists
                                  else None,
                                  "GBps": round(shard / statistics.mean(persists) / 1e9, 2)
                                  if persists else None},
            "window": "every drain and persist of the arm completes inside the timed window",
            "cadence_trials": trials,
            "sm_mhz_median_per_arm": clk_arms,
            "retention_backpressure_s": round(retention_wait_s, 3),
            "diag_with_arms": hosts}


def run_b200(args):
    import shutil
    import tempfile
    from dataclasses import replace
    import torch
    rank, local, world = dist_init(args.gpus)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_2408_04307_b200 import device as D
    from paper_2408_04307_b200.arena import StateArena
    from paper_2408_04307_b200.counting import DeviceTokenCounters
    from paper_2408_04307_b200.policy import b200_cadence, b200_configure
    from paper_2408_04307_b200.snapshot import PecCheckpointer
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
    persist = args.persist if args.persist != "auto" else "shm"
    persist_dropped = None
    store = None
    store_root = None
    if persist != "none":
        # one store root for all ranks (multi-writer commit, distributed.py)
        base = "/dev/shm" if persist == "shm" else tempfile.gettempdir()
        if rank == 0:
            sweep_stale_stores(base)
        root = [tempfile.mkdtemp(prefix=f"pec_bench_{os.getpid()}_", dir=base)
                if rank == 0 else None]
        if world > 1:
            import torch.distributed as dist
            dist.broadcast_object_list(root, src=0)
        store_root = root[0]
        store = DiskStore(store_root, io_threads=args.persist_threads or
                          len(os.sched_getaffinity(0)), direct_io=args.direct_io,
                          recycle=persist == "shm" and not args.no_recycle)
    mode = {"vec": D.MODE_VEC, "bulk": D.MODE_BULK, "crc": D.MODE_CRC}[args.engine]
    if args.pack_mode is not None:          # experiments: a pec_pack engine variant
        mode = args.pack_mode
    # the persist protocol gets its own gloo group (created collectively inside)
    ck = PecCheckpointer(layout, arena, store, w.pec, w.strategy, i_ckpt=1, ranks=[rank],
                         counters=counters, pack_mode=mode, chunk_log2=args.chunk_log2)
    eng = ck.engine
    eng.pipelined_drain = not args.no_pipelined_drain
    eng.reserve(ck.max_snapshot_bytes(), host_buffers=0)
    if store is not None:
        store_bytes_per_version[id(store)] = ck.max_snapshot_bytes() + (64 << 20)
    k_s = w.pec.k_snapshot
    sel = torch.empty((L, min(k_s, E)), dtype=torch.int32, device=dev)
    stream = eng.pack_stream

    ids_step = torch.randint(0, E, (L, routed), dtype=torch.int32, device=dev,
                             generator=torch.Generator(device=dev).manual_seed(1234 + rank))
    pt = getattr(eng, "template", None)
    la_sel = [] if plan is None else None

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
            snap_d, _ = counters.select(k_s, w.pec.k_persist, stream=stream)
        a, b = eng.pack_only_device(snap_d, stream=stream)
        la_sel.append(snap_d)
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
        moved = 0
        for sd in la_sel[-args.steps:]:
            h = sd.cpu().tolist()
            due = {m: frozenset(x for x in h[m] if x >= 0) for m in range(L)}
            moved += sum(a.stop - a.start for a in pt.select(due))
    max_ms = max_over_ranks(elapsed_ms, world, dev)
    total_moved = sum_over_ranks(moved, world, dev)
    value = total_moved / (max_ms / 1e3) / 1e9
    hbm_peak, peak_kind = measured_peaks()
    avg_pack_ms = statistics.mean(pack_ms)
    pack_bw = (moved / args.steps) / (avg_pack_ms / 1e3)          # payload B/s
    achieved = 2 * pack_bw / 1e9
    traffic = None
    tp = ROOT / "profiles" / "pack_traffic.json"
    if tp.exists():
        try:
            t = json.loads(tp.read_text()).get(w.name)
            traffic = t.get(args.engine) if isinstance(t, dict) else t
        except Exception:
            traffic = None

    # ---- host buffers: pinned once, before any host-side timing -------------
    tpin = time.perf_counter()
    # a /dev/shm persist tier holds SHM_VERSIONS_IN_FLIGHT shards per rank in
    # host RAM next to the pinned buffers; when both do not fit, the persist
    # tier is dropped (the line says so) rather than the node running out
    shard = step_bytes
    # (+1 version of spare files when retired versions are recycled)
    shm_versions = SHM_VERSIONS_IN_FLIGHT + (1 if getattr(store, "recycle", False) else 0)
    shm_reserve = shm_versions * shard if (store is not None and persist == "shm") else 0
    fit = host_buffers_that_fit(eng.staging.numel(), 3, reserve=shm_reserve)
    if store is not None and persist == "shm" and \
            min_over_ranks(float(fit), world, dev) < 3:
        fit_np = host_buffers_that_fit(eng.staging.numel(), 3)
        if min_over_ranks(float(fit_np), world, dev) >= 2:
            print(f"bench: host RAM ({mem_available() / 1e9:.0f} GB available) cannot hold 3 "
                  f"pinned buffers + {shm_versions} /dev/shm versions per rank; "
                  "persist tier off", file=sys.stderr)
            persist_dropped = f"host RAM: {mem_available() / 1e9:.0f} GB available for " \
                              f"{os.environ.get('LOCAL_WORLD_SIZE', '1')} ranks"
            store = None
            ck.engine.store = None
            fit = fit_np
    if store is not None and persist == "shm":
        # the tmpfs itself may be smaller than RAM (container /dev/shm limits)
        local_n = max(1, int(os.environ.get("LOCAL_WORLD_SIZE", "1")))
        shm_free, short = tmpfs_room(store.root, shm_versions * shard * local_n)
        if max_over_ranks(1.0 if short else 0.0, world, dev) > 0:
            shm_free = shm_free or 0
            print(f"bench: /dev/shm has {shm_free / 1e9:.0f} GB free, the persist tier needs "
                  f"{shm_versions} versions x {local_n} ranks x {shard / 1e9:.1f} GB; "
                  "persist tier off", file=sys.stderr)
            persist_dropped = f"/dev/shm: {shm_free / 1e9:.0f} GB free for {local_n} ranks"
            store = None
            ck.engine.store = None
            fit = host_buffers_that_fit(eng.staging.numel(), 3)
    n_host = int(min_over_ranks(float(fit), world, dev))    # node-wide minimum
    pin_error = None
    if n_host < 2:
        pin_error = f"host RAM fits {n_host} pinned snapshot buffers per rank (need >= 2)"
    else:
        try:
            eng.reserve(eng.staging.numel(), host_buffers=n_host)
            for hb in eng.host:                    # first D2H into fresh pages runs slow
                if hb is not None:
                    m_ = min(hb.numel(), eng.staging.numel())
                    hb[:m_].copy_(eng.staging[:m_])
        except (RuntimeError, MemoryError, OSError) as exc:  # e.g. pinning refused
            pin_error = f"{type(exc).__name__}: {exc}"[:200]
    pin_s = time.perf_counter() - tpin
    if max_over_ranks(1.0 if pin_error else 0.0, world, dev) > 0:
        print(f"bench: pinned host buffers unavailable ({pin_error}); skipping the host legs",
              file=sys.stderr)
        args.no_e2e = args.no_stall = True
    if n_host < (3 if store is not None else 2):
        # the steady state needs RECOVERY + PERSISTING + SNAPSHOTTING (2 without a persist tier)
        args.no_stall = True

    link_alone = link_conc = None
    e2e = host_link = persist_info = cadence = stall = None
    if not args.no_e2e:
        link_alone, link_conc = measure_host_link(eng, world, dev)

        # ---- e2e through the public API (snapshot tier only) ------------------
        ck.set_persist(False)
        n_e2e = max(5, args.e2e_steps)
        rng = np.random.default_rng(1234 + rank)
        ids_host = [torch.from_numpy(rng.integers(0, E, size=(L, routed), dtype=np.int32))
                    .pin_memory() for _ in range(n_e2e + 1)]
        ids_dev = torch.empty((L, routed), dtype=torch.int32, device=dev)
        base_it = 10 ** 6

        def e2e_step(k, it):
            ids_dev.copy_(ids_host[k], non_blocking=True)          # H2D of the step's input
            counters.add_iteration(ids_dev)
            buf = ck.checkpoint(it)                                 # select + plan + pack + drain
            ck.wait_snapshot(buf)                                   # SNAPSHOTTED: bytes in RAM
            first = eng.snapshot_layout(buf, rank).entries[0]
            _ = int(eng.entry_view(buf, rank, first.store_key)[0])  # host read of the result
            return ids_host[k].numel() * 4, eng.snapshot_nbytes(buf)

        e2e_step(n_e2e, base_it)                  # untimed: first-call host costs
        barrier(world)
        torch.cuda.synchronize()
        h2d = d2h = 0
        tw = time.perf_counter()
        for k in range(n_e2e):
            hb, db = e2e_step(k, base_it + 1 + k)
            h2d += hb
            d2h += db
        e2e_s = max_over_ranks(time.perf_counter() - tw, world, dev)
        e2e_moved = sum_over_ranks(sum(eng.stats["snap_bytes"][-n_e2e:]), world, dev)
        drains = eng.stats["drain_ms"][-n_e2e:]
        e2e = {"value": round(e2e_moved / e2e_s / 1e9, 3), "unit": UNIT,
               "h2d_bytes_per_step": h2d // n_e2e, "d2h_bytes_per_step": d2h // n_e2e,
               "steps": n_e2e, "ms_per_step": round(e2e_s / n_e2e * 1e3, 2),
               "drain_ms": [round(x, 2) for x in drains],
               "what": "router-id H2D + count + select + pack(+CRC) + D2H drain to pinned host "
                       "+ host read, through PecCheckpointer (snapshot tier)",
               "host_pin_s": round(pin_s, 1)}
        drain_gbs = statistics.mean([(d2h // n_e2e) / (m / 1e3) / 1e9 for m in drains])
        e2e["per_gpu"] = round(e2e["value"] / world, 3)
        link_ref = link_conc if world > 1 else link_alone
        e2e["frac_of_host_link"] = round(e2e["per_gpu"] / link_ref, 4)
        host_link = {"achieved": round(drain_gbs, 2), "peak": round(link_alone, 2),
                     "unit": "GB/s",
                     "peak_kind": "measured in this run: 4 GiB pinned D2H in the drain's "
                                  "256 MiB pieces on its copy stream, best of 5, this GPU alone",
                     "peak_all_gpus_concurrent": round(link_conc, 2),
                     # this rank's drain vs the link alone; the whole-job rate against
                     # the all-ranks-at-once peak is e2e.frac_of_host_link
                     "frac": round(drain_gbs / link_alone, 4)}

        # ---- persist probe: this run's steady persist rate --------------------
        # three versions with retention between them: the first two create
        # their files (cold tmpfs pages), the third is what every later
        # version costs (with recycling it overwrites the first one's files)
        if store is not None:
            ck.set_persist(True)
            probe_s = []
            for j in range(PERSIST_PROBE_VERSIONS):
                ck.checkpoint(base_it + n_e2e + 1 + j)
                ck.finish()
                probe_s.append(eng.stats["persist_s"][-1])
                barrier(world)
                prune_store(store, ranks=[rank], coordinator=rank == 0)
                barrier(world)
                prune_store(store, ranks=[rank], coordinator=rank == 0)
            p_s = probe_s[-1]
            persist_info = {"target": persist, "direct_io": bool(args.direct_io),
                            "crc": "device (pack)" if mode == D.MODE_CRC else "host",
                            "recycle": bool(getattr(store, "recycle", False)),
                            "seconds": round(p_s, 3),
                            "GBps": round(eng.stats["snap_bytes"][-1] / p_s / 1e9, 2),
                            "seconds_per_probe_version": [round(x, 3) for x in probe_s],
                            "what": f"{PERSIST_PROBE_VERSIONS} versions, retention between "
                                    "them; seconds/GBps = the last (steady) one"}
            # sustained: checkpoints issued back to back, so every persist
            # overlaps the next drain(s) as in the training loop (they share
            # the host memory); the policy's floors come from these rates
            ret = Retention(store, ranks=[rank], coordinator=rank == 0)
            np0, nd0 = len(eng.stats["persist_s"]), len(eng.stats["drain_ms"])
            barrier(world)
            ts = time.perf_counter()
            for j in range(SUSTAINED_PROBE_VERSIONS):
                ck.checkpoint(base_it + n_e2e + 1 + PERSIST_PROBE_VERSIONS + j)
                ret.submit()
            ck.finish()
            cycle_s = (time.perf_counter() - ts) / SUSTAINED_PROBE_VERSIONS
            ret.close()
            barrier(world)
            prune_store(store, ranks=[rank], coordinator=rank == 0)
            sus_p = eng.stats["persist_s"][np0:]
            sus_d = [m / 1e3 for m in eng.stats["drain_ms"][nd0:]]
            persist_info["sustained"] = {
                "versions": SUSTAINED_PROBE_VERSIONS,
                "persist_s": [round(x, 3) for x in sus_p],
                "drain_s": [round(x, 3) for x in sus_d],
                "cycle_s": round(cycle_s, 3),
                "what": "back-to-back checkpoints: persist and drain rates under each other's "
                        "host-memory contention, and the seconds per checkpoint the pipeline "
                        "sustains; the cadence floors use these x CADENCE_MARGIN"}

        # ---- the cadence the policy derives from this run's measurements ------
        if store is not None and not args.no_stall:
            sus = persist_info["sustained"]
            nbytes = eng.stats["snap_bytes"][-1]
            # slowest rank, under contention, with a margin: a floor computed
            # with zero slack waits on every variance (simulator.py:413-422)
            p_eff = CADENCE_MARGIN * max(statistics.mean(sus["persist_s"][1:] or
                                                         sus["persist_s"]), 1e-9)
            d_eff = CADENCE_MARGIN * max(statistics.mean(sus["drain_s"][1:] or
                                                         sus["drain_s"]), 1e-9)
            cl = replace(layout.cluster,
                         snapshot_bandwidth=min_over_ranks(pack_bw, world, dev),
                         persist_bandwidth=min_over_ranks(nbytes / p_eff, world, dev),
                         fb_time=args.fb_ms / 1e3, update_time=args.update_ms / 1e3)
            dbw = min_over_ranks(nbytes / d_eff, world, dev)
            cad = b200_cadence(layout, w.strategy, w.pec, cl, dbw)
            cadence = {"i_ckpt_requested": args.i_ckpt, "i_ckpt_min": cad.i_ckpt_min,
                       "feasible": cad.i_ckpt_min <= args.i_ckpt,
                       "floors": {"persist": cad.persist_floor, "drain": cad.drain_floor,
                                  "snapshot_overlap": cad.snapshot_floor},
                       "persist_s": round(cad.persist_s, 3), "drain_s": round(cad.drain_s, 3),
                       "pack_ms": round(cad.pack_s * 1e3, 3),
                       "floor_GBps": {"pack": round(cl.snapshot_bandwidth / 1e9, 1),
                                         "drain": round(dbw / 1e9, 2),
                                         "persist": round(cl.persist_bandwidth / 1e9, 2)},
                       "margin": CADENCE_MARGIN,
                       "what": "policy.b200_cadence on this run's slowest-rank pack rate and "
                               "sustained drain / persist rates (back-to-back checkpoints, "
                               "x margin), F&B + update proxy times"}
            try:
                free = b200_configure(layout, w.strategy, cl, dbw)
                cadence["policy_free_choice"] = {"k_snapshot": free.pec.k_snapshot,
                                                 "k_persist": free.pec.k_persist,
                                                 "i_ckpt": free.i_ckpt}
            except Exception as exc:  # informational only
                cadence["policy_free_choice"] = {"error": str(exc)[:120]}

    if not args.no_stall:
        i_ckpt = max(args.i_ckpt, cadence["i_ckpt_min"]) if cadence else args.i_ckpt
        if cadence and not cadence["feasible"]:
            print(f"bench: I_ckpt={args.i_ckpt} is infeasible on this box (persist/drain "
                  f"floor {cadence['i_ckpt_min']}); the stall leg runs at I_ckpt={i_ckpt}",
                  file=sys.stderr)
        if args.stall_no_persist:
            ck.set_persist(False)
        with ClockSampler(local, period_s=0.1) as stall_clk:
            stall = measure_stall(ck, arena, dev, i_ckpt, args.stall_checkpoints, args.fb_ms,
                                  args.stall_rounds, world, rank)
        stall["clocks"] = stall_clk.summary()
        if store is not None and getattr(store, "recycle", False):
            stall["persist_recycled_files"] = store.recycled_files
        stall["persist_tier"] = "off (diagnostic)" if args.stall_no_persist else \
            (f"off ({persist_dropped})" if persist_dropped else
             ("on" if store is not None else "none configured"))
        if cadence:
            stall["cadence"] = cadence
    ck.close()
    barrier(world)
    if store_root and rank == 0:
        shutil.rmtree(store_root, ignore_errors=True)

    # ---- CPU baseline (rank 0, N == 1 only): the reference arm's pack --------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = len(os.sched_getaffinity(0))
        try:
            times, payload, desc, ref, rlayout = cpu_pack_shards(
                w, 1, 1, 1, threads, int(args.cpu_sample_gb * 1e9) if args.cpu_sample_gb
                else 0, min_seconds=args.cpu_seconds)
            cpu = {"value": round(payload / statistics.mean(times) / 1e9, 3), "unit": UNIT,
                   "cores": threads, "kind": "port", "sample": desc, "cpu_model": cpu_model()}
            cpu["components"] = reference_components(ref, rlayout, w) if ref is not None \
                else {"error": "reference not importable"}
        except Exception as exc:  # reported, never fatal to the bench line
            cpu = {"error": f"{type(exc).__name__}: {exc}"[:200]}

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
                       **({"pack_mode": args.pack_mode} if args.pack_mode is not None else {}),
                       "value_is": "HBM-staged snapshot: selection + pack (+ per-entry CRC-32C) "
                                   "into HBM staging, the training-blocking step; e2e = bytes "
                                   "in pinned host memory (the reference's SNAPSHOTTED)",
                       "l2": (f"no flush needed: each step reads "
                              f"{(moved // args.steps) / 1e9:.2f} GB (> 126 MB L2)"
                              if flush is None else
                              "512 MiB L2 flush written between steps, inside the timed "
                              "region (steps move less than 4x the 126 MB L2)"),
                       "parallelism": f"dp{layout.n_ranks}-ep{layout.parallel.ep_degree}",
                       "dist_backend": dist_backend() if world > 1 else None},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_peak,
                         "unit": "GB/s", "frac": round(achieved / hbm_peak, 4),
                         "traffic": traffic, "peak_kind": peak_kind,
                         # frac > 1 is possible: `peak` is torch's copy_ kernel, and the
                         # TMA bulk ring moves bytes faster than it; the nominal HBM3e
                         # figure (7.7 TB/s, B200_PROFILING.md) bounds both
                         "nominal": HBM_NOMINAL_GBS,
                         "frac_of_nominal": round(achieved / HBM_NOMINAL_GBS, 4),
                         "kernel": f"pec_pack{'_crc' if args.engine == 'crc' else ''} "
                                   f"({args.engine})",
                         "avg_launch_ms": round(avg_pack_ms, 4)},
            "e2e": e2e,
            "host_link": host_link,
            "persist": persist_info if persist_info else
            ({"off": persist_dropped} if persist_dropped else None),
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
    ap.add_argument("--pack-mode", type=int, default=None,
                    help="experiments only: a pec_pack mode (engine variant, csrc/pec_kernels.cu "
                         "launch_copy); CRCs then come from the host writer")
    ap.add_argument("--e2e-steps", type=int, default=6)
    ap.add_argument("--persist", default="auto", choices=["auto", "none", "shm", "disk"])
    ap.add_argument("--direct-io", action="store_true",
                    help="persist with O_DIRECT (meaningful with --persist disk)")
    ap.add_argument("--persist-threads", type=int, default=0,
                    help="writer threads per rank (0 = all host cores; background priority)")
    ap.add_argument("--no-recycle", action="store_true",
                    help="retire superseded /dev/shm versions by deleting their files instead "
                         "of recycling them as spares (A/B)")
    ap.add_argument("--stall-no-persist", action="store_true",
                    help="diagnostic: run the stall leg with the persist tier off")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-stall", action="store_true")
    ap.add_argument("--no-pipelined-drain", action="store_true",
                    help="drain each snapshot only after its whole pack (A/B of the default)")
    ap.add_argument("--i-ckpt", type=int, default=10)
    ap.add_argument("--stall-checkpoints", type=int, default=12,
                    help="checkpoints per checkpointed arm (>= 4 triple-buffer cycles)")
    ap.add_argument("--stall-rounds", type=int, default=2)
    ap.add_argument("--fb-ms", type=float, default=100.0)
    ap.add_argument("--update-ms", type=float, default=25.0,
                    help="update time the policy assumes (the proxy's pass over the arena)")
    ap.add_argument("--cpu-sample-gb", type=float, default=0.0,
                    help="cap per rank for the CPU pack (0 = the full shard, same config)")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "b200":
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
