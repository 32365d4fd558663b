"""World-size-2 gloo tests (CPU) of the cross-rank protocol: global
load-aware selection over all-reduced counts and the multi-writer commit."""

import json
import os
import socket
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _init(rank, world, port):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _oracle_select_fn(counts2d, k, pool):
    import torch
    sys.path.insert(0, str(ROOT))
    from oracle import pec_oracle as O
    rows = counts2d.tolist()
    pl = None if pool is None else pool.tolist()
    out = [O.select_load_aware(rows[m], k, None if pl is None else pl[m]) for m in range(len(rows))]
    return torch.tensor(out, dtype=torch.int32)


def _select_worker(rank, world, port, outdir):
    import torch
    import torch.distributed as dist
    sys.path.insert(0, str(ROOT))
    from oracle import pec_oracle as O
    from paper_2408_04307_b200.distributed import global_two_tier_select
    _init(rank, world, port)
    L, E = 5, 8
    local = torch.zeros((2, L, E), dtype=torch.int64)
    glob_snap = np.zeros((L, E), dtype=np.int64)
    glob_pers = np.zeros((L, E), dtype=np.int64)
    log = []
    for ck in range(6):
        for it in range(4):
            adds = [np.random.default_rng(1000 * r + 10 * ck + it).integers(0, 50, size=(L, E))
                    for r in range(world)]
            local[0] += torch.from_numpy(adds[rank])
            local[1] += torch.from_numpy(adds[rank])
            glob_snap += sum(adds)
            glob_pers += sum(adds)
        snap, pers = global_two_tier_select(local, 3, 2, _oracle_select_fn)
        ss, ps, glob_snap, glob_pers = O.two_tier_load_aware(glob_snap, glob_pers, 3, 2)
        assert snap.tolist() == ss and pers.tolist() == ps
        # invariant: sum of locals == oracle global
        g = local.clone()
        dist.all_reduce(g)
        assert np.array_equal(g[0].numpy(), glob_snap)
        assert np.array_equal(g[1].numpy(), glob_pers)
        log.append(snap.tolist())
    Path(outdir, f"sel{rank}.json").write_text(json.dumps(log))
    dist.destroy_process_group()


def _commit_worker(rank, world, port, root):
    sys.path.insert(0, str(ROOT))
    import torch.distributed as dist
    from paper_2408_04307_b200.distributed import commit_version
    from paper_2408_04307_b200.store import DiskStore, StoreEntry
    _init(rank, world, port)
    entries = _entries()
    store = DiskStore(root)
    pay = {e.store_key: _payload(e) for e in entries if e.rank == rank}
    for v in (1, 2):
        commit_version(store, v, 10 * v, v - 1, entries, [rank], pay)
    dist.destroy_process_group()


def _entries():
    from paper_2408_04307_b200.store import StoreEntry
    return [StoreEntry("ew.L0.E0.part0", 0, "ew.L0.E0", 0, 501),
            StoreEntry("ew.L0.E0.part1", 1, "ew.L0.E0", 501, 1003),
            StoreEntry("eo.L0.E0", 0, "eo.L0.E0", 0, 6018),
            StoreEntry("neo.r0", 0, "neo.r0", 0, 777),
            StoreEntry("neo.r1", 1, "neo.r1", 0, 775),
            StoreEntry("new.a", 1, "new.a", 0, 64)]


def _payload(e):
    import zlib
    return np.random.default_rng(zlib.crc32(e.store_key.encode())).integers(
        0, 256, e.stop - e.start, dtype=np.uint8).tobytes()


def test_global_selection_over_gloo_matches_oracle_on_summed_counts(tmp_path):
    import torch.multiprocessing as mp
    mp.spawn(_select_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    a = json.loads((tmp_path / "sel0.json").read_text())
    b = json.loads((tmp_path / "sel1.json").read_text())
    assert a == b


def test_multi_writer_commit_equals_single_writer(tmp_path):
    import torch.multiprocessing as mp
    sys.path.insert(0, str(ROOT))
    from paper_2408_04307_b200.store import DiskStore
    multi = tmp_path / "multi"
    mp.spawn(_commit_worker, args=(2, _free_port(), str(multi)), nprocs=2, join=True)
    single = DiskStore(tmp_path / "single")
    ents = _entries()
    pay = {e.store_key: _payload(e) for e in ents}
    m = DiskStore(multi)
    assert m.complete_versions() == [1, 2]
    for v in (1, 2):
        single.write_version(v, 10 * v, v - 1, ents, payloads=pay)
        for name in ("meta.json", "manifest.tsv", "COMPLETE"):
            assert (multi / f"v{v:06d}" / name).read_bytes() == \
                (tmp_path / "single" / f"v{v:06d}" / name).read_bytes()
        assert m.load_checkpoint(v) == single.load_checkpoint(v)
