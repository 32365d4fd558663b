"""Versioned, CRC-32C-checked, completion-marked checkpoint store.

The on-disk format is the reference's (`pkg/src/mocsim/store.py`), byte for
byte (store.py:1-8, 149-228), so either implementation reads the other's
versions:

    v%06d/rank%04d/<store_key>.bin   entry payloads
    v%06d/meta.json                  json.dumps(sort_keys=True, indent=0) + "\\n"
    v%06d/manifest.tsv               key<TAB>path<TAB>size<TAB>%08x crc, sorted by key
    v%06d/COMPLETE                   empty, via .COMPLETE.tmp + os.replace

What changes on B200 is the payload: the reference writes a synthetic
blake2b stand-in per entry (store.py:118-121); here `write_version` takes
the real snapshot bytes (``payloads``: store_key -> bytes-like, normally
views into a pinned host snapshot buffer) with their CRC-32Cs computed by the
pack on the GPU (``crcs``; libpec's multithreaded SSE4.2 CRC-32C otherwise)
and writes the entry files with the native writer (`pec_write_files`).
Without ``payloads`` it falls back to the reference's synthetic payloads,
so metadata-only callers (the reference's own engine tests) behave exactly as
before.  Manifest ``size`` is the payload length in both cases.

The write is split so several rank processes can publish one version:
`write_entries` (each rank, its own files) then `publish` (one writer:
meta.json, manifest.tsv, COMPLETE), exactly the files a single
`write_version` would produce.
"""

from __future__ import annotations

import hashlib
import json
import os
import threading
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field
from pathlib import Path
from typing import Dict, Iterable, List, Mapping, NamedTuple, Optional, Tuple


from . import device as _dev


class StoreError(Exception):
    pass


class IncompleteVersionError(StoreError):
    """The version has no COMPLETE marker."""


class ChecksumMismatchError(StoreError):
    """An entry's bytes disagree with the manifest; ``key`` names it."""

    def __init__(self, key: str, detail: str):
        self.key = key
        super().__init__(f"entry {key!r}: {detail}")


class CrashPoint(RuntimeError):
    """Raised by a fault injector when its write budget runs out."""


def crc32c(data, crc: int = 0) -> int:
    """CRC-32C (Castagnoli), identical to reference store.crc32c
    (store.py:49-70); SSE4.2 implementation in libpec."""
    return _dev.crc32c(data, crc)


class StoreEntry(NamedTuple):
    """Which rank wrote which byte range of which unit (store.py:73-80)."""

    store_key: str
    rank: int
    unit_key: str
    start: int
    stop: int


@dataclass(frozen=True)
class VersionMeta:
    version: int
    iteration: int
    checkpoint_index: int
    entries: Dict[str, StoreEntry]

    def units_covered(self, unit_sizes: Mapping[str, int]) -> set:
        """Units whose whole byte span is present (store.py:91-106)."""
        spans: Dict[str, List[Tuple[int, int]]] = {}
        for e in self.entries.values():
            spans.setdefault(e.unit_key, []).append((e.start, e.stop))
        done = set()
        for unit, rs in spans.items():
            reach = 0
            for lo, hi in sorted(rs):
                if lo > reach:
                    break
                reach = max(reach, hi)
            if reach >= unit_sizes[unit]:
                done.add(unit)
        return done


@dataclass(frozen=True)
class StoreManifest:
    version: int
    iteration: int
    entries: Dict[str, Tuple[str, int, int]]  # key -> (path, size, crc)
    complete_marker: bool


def entry_payload(store_key: str, version: int, iteration: int) -> bytes:
    """The reference's synthetic payload (store.py:118-121), used only when a
    caller supplies no real bytes."""
    head = f"mocsim\t{store_key}\tv{version}\ti{iteration}\n".encode()
    return head + hashlib.blake2b(head, digest_size=32).digest()


class TruncatingInjector:
    """Crash a persist after a byte budget (store.py:124-146): payload bytes
    consume budget, the COMPLETE rename consumes one unit."""

    def __init__(self, crash_after_bytes: int):
        self.remaining = crash_after_bytes

    def write(self, fileobj, data) -> None:
        n = len(data)
        if n <= self.remaining:
            fileobj.write(data)
            self.remaining -= n
            return
        fileobj.write(memoryview(data)[:self.remaining])
        self.remaining = 0
        raise CrashPoint("write budget exhausted")

    def charge_op(self) -> None:
        if self.remaining <= 0:
            raise CrashPoint("no budget left for rename")
        self.remaining -= 1


def _meta_bytes(meta: VersionMeta) -> bytes:
    body = {"version": meta.version, "iteration": meta.iteration,
            "checkpoint_index": meta.checkpoint_index,
            "entries": {k: {"rank": e.rank, "unit": e.unit_key, "start": e.start, "stop": e.stop}
                        for k, e in sorted(meta.entries.items())}}
    return (json.dumps(body, sort_keys=True, indent=0) + "\n").encode()


def _manifest_bytes(rows: Iterable[Tuple[str, str, int, int]]) -> bytes:
    lines = [f"{k}\t{p}\t{s}\t{c:08x}" for k, p, s, c in rows]
    return ("\n".join(lines) + "\n").encode()


def _entry_path(rank: int, store_key: str) -> str:
    return f"rank{rank:04d}/{store_key}.bin"


def _nbytes(buf) -> int:
    return memoryview(buf).nbytes


def _crcs(payloads: List, threads: int) -> List[int]:
    """CRC-32C of many payloads; large ones in parallel through libpec."""
    out = []
    big = []
    for i, p in enumerate(payloads):
        if _nbytes(p) >= (8 << 20):
            big.append(i)
            out.append(None)
        else:
            out.append(crc32c(p))
    if big:
        if threads > 1:
            with ThreadPoolExecutor(max_workers=min(threads, len(big))) as ex:
                vals = list(ex.map(lambda i: crc32c(payloads[i]), big))
        else:
            vals = [crc32c(payloads[i]) for i in big]
        for i, v in zip(big, vals):
            out[i] = v
    return out


PayloadSource = Optional[Mapping[str, object]]


def _fsync_path(path) -> None:
    fd = os.open(str(path), os.O_RDONLY)
    try:
        os.fsync(fd)
    finally:
        os.close(fd)


class DiskStore:
    """One directory per version under ``root`` (store.py:171-282)."""

    def __init__(self, root, io_threads: int = 8, direct_io: bool = False, fsync: bool = False,
                 background: bool = True, recycle: bool = False):
        """B200 additions: ``io_threads`` for the native writer/reader,
        ``direct_io`` writes real payloads with O_DIRECT (page-cache bypass
        on real storage, large files range-parallel; buffered where the
        filesystem refuses it), ``fsync`` makes every entry file durable
        before the version is published, ``background`` runs the writer
        threads at nice +10 (a persist yields host cores to the training
        loop's launch thread), ``recycle`` lets `retire` keep a superseded
        version's entry files as spares that later versions overwrite in
        place (on tmpfs / page-cache targets rewriting a file keeps its
        pages: 1.7-2.6x faster than truncating and rewriting it)."""
        self.root = Path(root)
        self.root.mkdir(parents=True, exist_ok=True)
        self.io_threads = max(1, io_threads)
        self.direct_io = direct_io
        self.fsync = fsync
        self.background = background
        self.recycle = recycle
        self._spares: Dict[int, Dict[int, List[Path]]] = {}   # rank -> size -> files
        self._spare_lock = threading.Lock()
        self.recycled_files = 0      # entry files written over a retired version's file

    def version_dir(self, version: int) -> Path:
        return self.root / f"v{version:06d}"

    # -- writing ------------------------------------------------------------
    def _put(self, path: Path, data, injector) -> None:
        path.parent.mkdir(parents=True, exist_ok=True)
        with open(path, "wb", buffering=0) as f:
            if injector is None:
                mv = memoryview(data).cast("B")
                while mv.nbytes:
                    n = f.write(mv)
                    mv = mv[n:]
            else:
                injector.write(f, data)

    def _payloads(self, entries, version, iteration, payloads: PayloadSource):
        if payloads is None:
            return [entry_payload(e.store_key, version, iteration) for e in entries]
        return [payloads[e.store_key] for e in entries]

    def serialized_size(self, version: int, iteration: int, checkpoint_index: int,
                        entries: Iterable[StoreEntry], payloads: PayloadSource = None) -> int:
        """Bytes write_version would stream, rename excluded (store.py:185-200)."""
        entries = sorted(entries)
        data = self._payloads(entries, version, iteration, payloads)
        rows = [(e.store_key, _entry_path(e.rank, e.store_key), _nbytes(p), 0)
                for e, p in zip(entries, data)]
        meta = VersionMeta(version, iteration, checkpoint_index, {e.store_key: e for e in entries})
        return sum(r[2] for r in rows) + len(_meta_bytes(meta)) + len(_manifest_bytes(rows))

    def write_entries(self, version: int, iteration: int, entries: Iterable[StoreEntry],
                      payloads: PayloadSource = None, injector: Optional[TruncatingInjector] = None,
                      crcs: Optional[Mapping[str, int]] = None) -> List[Tuple[str, str, int, int]]:
        """Entry files of (a subset of) a version; returns manifest rows.
        ``crcs`` supplies precomputed CRC-32Cs (device-computed by the pack);
        missing ones are computed here."""
        entries = sorted(entries)
        data = self._payloads(entries, version, iteration, payloads)
        vdir = self.version_dir(version)
        for r in {e.rank for e in entries}:
            (vdir / f"rank{r:04d}").mkdir(parents=True, exist_ok=True)
        given = crcs is not None and payloads is not None and \
            all(e.store_key in crcs for e in entries)
        if entries and (injector is None or type(injector) is TruncatingInjector):
            # native writer: threads take whole files (largest first) and CRC
            # each 4 MiB piece right after writing it.  A TruncatingInjector's
            # byte budget is spent natively in entry order, exactly as the
            # sequential loop below spends it (pec_write_files_budget)
            paths = [vdir / _entry_path(e.rank, e.store_key) for e in entries]
            reused = self._adopt_spares(entries, data, paths) if self.recycle else 0
            kw = dict(threads=self.io_threads, want_crc=not given, fsync=self.fsync,
                      direct=self.direct_io, background=self.background, overwrite=reused > 0)
            if injector is None:
                got = _dev.write_files(paths, data, **kw)
            else:
                got, injector.remaining, crashed = _dev.write_files(
                    paths, data, budget=injector.remaining, **kw)
                if crashed:
                    raise CrashPoint("write budget exhausted")
            crc_list = [crcs[e.store_key] for e in entries] if given else [int(c) for c in got]
            return [(e.store_key, _entry_path(e.rank, e.store_key), _nbytes(p), c)
                    for e, p, c in zip(entries, data, crc_list)]
        crc_list = [crcs[e.store_key] for e in entries] if given else \
            _crcs(data, self.io_threads if injector is None else 1)
        rows = [(e.store_key, _entry_path(e.rank, e.store_key), _nbytes(p), c)
                for e, p, c in zip(entries, data, crc_list)]
        if injector is not None or self.io_threads == 1 or len(entries) < 2:
            for (_, rel, _, _), p in zip(rows, data):
                self._put(vdir / rel, p, injector)
        else:
            with ThreadPoolExecutor(max_workers=min(self.io_threads, len(entries))) as ex:
                list(ex.map(lambda rp: self._put(vdir / rp[0][1], rp[1], None), zip(rows, data)))
        return rows

    # -- recycling (B200 addition; never changes what a reader sees) -----------
    def _spare_dir(self, rank: int) -> Path:
        return self.root / ".spare" / f"rank{rank:04d}"

    def _adopt_spares(self, entries, data, paths) -> int:
        """Rename a spare file of exactly the payload's size onto each entry
        path (same filesystem: O(1)); the writer then overwrites it in place.
        Returns how many entries got one."""
        n = 0
        with self._spare_lock:
            for e, p, path in zip(entries, data, paths):
                pool = self._spares.get(e.rank, {}).get(_nbytes(p))
                if pool:
                    os.replace(pool.pop(), path)
                    n += 1
            self.recycled_files += n
        return n

    def retire(self, version: int, ranks: Optional[Iterable[int]] = None,
               coordinator: bool = True) -> bool:
        """Drop a superseded version (retention), keeping its entry files of
        ``ranks`` (all ranks by default) as spares when ``recycle`` is set.
        The COMPLETE marker goes first, so a half-retired version is never
        readable; the coordinator removes the directory once no rank
        directory is left.  Returns True when the version is gone."""
        import shutil
        import uuid
        vdir = self.version_dir(version)
        if not vdir.exists():
            return True
        if coordinator:
            try:
                os.unlink(vdir / "COMPLETE")
            except FileNotFoundError:
                pass
        rank_dirs = sorted(vdir.glob("rank*")) if ranks is None else \
            [vdir / f"rank{r:04d}" for r in ranks]
        for rd in rank_dirs:
            if not rd.exists():
                continue
            r = int(rd.name[4:])
            if self.recycle:
                spare = self._spare_dir(r)
                spare.mkdir(parents=True, exist_ok=True)
                for f in rd.glob("*.bin"):
                    size = f.stat().st_size
                    dst = spare / f"{size}.{uuid.uuid4().hex}.bin"
                    os.replace(f, dst)
                    with self._spare_lock:
                        self._spares.setdefault(r, {}).setdefault(size, []).append(dst)
            shutil.rmtree(rd, ignore_errors=True)
        if coordinator and not any(vdir.glob("rank*")):
            shutil.rmtree(vdir, ignore_errors=True)
            return True
        return False

    def trim_spares(self, ranks: Iterable[int], keep_bytes: int) -> None:
        """Delete spare files beyond ``keep_bytes`` per rank (sizes no
        version asked for again stay bounded)."""
        for r in ranks:
            with self._spare_lock:
                pool = self._spares.get(r, {})
                files = [(size, p) for size, ps in pool.items() for p in ps]
                total = sum(size for size, _ in files)
                drop = []
                for size, p in sorted(files, reverse=True):
                    if total <= keep_bytes:
                        break
                    pool[size].remove(p)
                    drop.append(p)
                    total -= size
            for p in drop:
                try:
                    os.unlink(p)
                except FileNotFoundError:
                    pass

    def publish(self, version: int, iteration: int, checkpoint_index: int,
                entries: Iterable[StoreEntry], rows: Iterable[Tuple[str, str, int, int]],
                injector: Optional[TruncatingInjector] = None) -> StoreManifest:
        """meta.json, manifest.tsv, then the atomic COMPLETE (store.py:217-228)."""
        entries = sorted(entries)
        rows = sorted(rows)
        vdir = self.version_dir(version)
        vdir.mkdir(parents=True, exist_ok=True)
        meta = VersionMeta(version, iteration, checkpoint_index, {e.store_key: e for e in entries})
        self._put(vdir / "meta.json", _meta_bytes(meta), injector)
        self._put(vdir / "manifest.tsv", _manifest_bytes(rows), injector)
        tmp = vdir / ".COMPLETE.tmp"
        self._put(tmp, b"", injector)
        if injector is not None:
            injector.charge_op()
        if self.fsync:
            # durable before visible: metadata files and every directory
            # entry reach storage before the COMPLETE rename, the rename after
            for f in (vdir / "meta.json", vdir / "manifest.tsv", tmp):
                _fsync_path(f)
            for d in sorted({(vdir / r).parent for _, r, _, _ in rows} | {vdir}):
                _fsync_path(d)
        os.replace(tmp, vdir / "COMPLETE")
        if self.fsync:
            _fsync_path(vdir)
            _fsync_path(self.root)
        return StoreManifest(version, iteration, {k: (p, s, c) for k, p, s, c in rows}, True)

    def check_version(self, version: int) -> None:
        newest = self.newest_complete()
        if newest is not None and version <= newest:
            raise StoreError(f"version {version} not above newest complete {newest}")

    def write_version(self, version: int, iteration: int, checkpoint_index: int,
                      entries: Iterable[StoreEntry], injector: Optional[TruncatingInjector] = None,
                      payloads: PayloadSource = None) -> StoreManifest:
        """Entry files, meta, manifest, COMPLETE (store.py:202-228)."""
        entries = sorted(entries)
        self.check_version(version)
        rows = self.write_entries(version, iteration, entries, payloads, injector)
        return self.publish(version, iteration, checkpoint_index, entries, rows, injector)

    # -- reading ------------------------------------------------------------
    def version_numbers(self) -> List[int]:
        """Every version directory present, complete or not (retention)."""
        found = []
        for child in self.root.iterdir():
            if child.name.startswith("v") and child.name[1:].isdigit():
                found.append(int(child.name[1:]))
        return sorted(found)

    def complete_versions(self) -> List[int]:
        found = []
        for child in self.root.iterdir():
            if child.name.startswith("v") and (child / "COMPLETE").exists():
                try:
                    found.append(int(child.name[1:]))
                except ValueError:
                    pass
        return sorted(found)

    def newest_complete(self) -> Optional[int]:
        v = self.complete_versions()
        return v[-1] if v else None

    def meta(self, version: int) -> VersionMeta:
        doc = json.loads((self.version_dir(version) / "meta.json").read_text())
        ents = {k: StoreEntry(k, v["rank"], v["unit"], v["start"], v["stop"])
                for k, v in doc["entries"].items()}
        return VersionMeta(doc["version"], doc["iteration"], doc["checkpoint_index"], ents)

    def manifest(self, version: int) -> StoreManifest:
        vdir = self.version_dir(version)
        if not (vdir / "COMPLETE").exists():
            raise IncompleteVersionError(f"version {version} has no COMPLETE marker")
        meta = self.meta(version)
        ents = {}
        for line in (vdir / "manifest.tsv").read_text().splitlines():
            if not line:
                # an entry-less version's manifest is "\n"; the reference's
                # reader fails on it (store.py:251-252), this one reads {}
                continue
            k, p, s, c = line.split("\t")
            ents[k] = (p, int(s), int(c, 16))
        return StoreManifest(version, meta.iteration, ents, True)

    def load_checkpoint(self, version: int, keys: Optional[Iterable[str]] = None) -> Dict[str, bytes]:
        """Entries of a COMPLETE version with verified checksums
        (store.py:267-282); ``keys`` limits the read."""
        man = self.manifest(version)
        want = sorted(man.entries) if keys is None else sorted(keys)
        vdir = self.version_dir(version)
        out = {}
        for k in want:
            rel, size, crc = man.entries[k]
            path = vdir / rel
            if not path.exists():
                raise ChecksumMismatchError(k, "entry file missing")
            data = path.read_bytes()
            if len(data) != size:
                raise ChecksumMismatchError(k, f"size {len(data)} != manifest {size}")
            if crc32c(data) != crc:
                raise ChecksumMismatchError(k, "crc32c mismatch")
            out[k] = data
        return out

    def read_into(self, version: int, placements: Mapping[str, Tuple[object, int]],
                  verify: bool = True) -> None:
        """Read entries straight into host buffers: placements maps
        store_key -> (writable buffer, offset).  CRC-verified, parallel."""
        man = self.manifest(version)
        vdir = self.version_dir(version)

        def one(item):
            k, (buf, off) = item
            rel, size, crc = man.entries[k]
            path = vdir / rel
            if not path.exists():
                raise ChecksumMismatchError(k, "entry file missing")
            if path.stat().st_size != size:
                raise ChecksumMismatchError(k, f"size {path.stat().st_size} != manifest {size}")
            view = memoryview(buf).cast("B")[off:off + size]
            with open(path, "rb", buffering=0) as f:
                got = 0
                while got < size:
                    n = f.readinto(view[got:])
                    if not n:
                        raise ChecksumMismatchError(k, "short read")
                    got += n
            if verify and crc32c(view) != crc:
                raise ChecksumMismatchError(k, "crc32c mismatch")

        items = sorted(placements.items())
        with ThreadPoolExecutor(max_workers=max(1, min(self.io_threads, len(items) or 1))) as ex:
            list(ex.map(one, items))


@dataclass
class MemoryStore:
    """Disk-free store with the same interface (store.py:285-335)."""

    _versions: Dict[int, Tuple[VersionMeta, Dict[str, bytes]]] = field(default_factory=dict)
    _pending: Dict[int, Dict[str, bytes]] = field(default_factory=dict)

    def write_entries(self, version: int, iteration: int, entries: Iterable[StoreEntry],
                      payloads: PayloadSource = None, injector=None, crcs=None):
        if injector is not None:
            raise StoreError("crash injection requires the disk store")
        entries = sorted(entries)
        if payloads is None:
            data = {e.store_key: entry_payload(e.store_key, version, iteration) for e in entries}
        else:
            data = {e.store_key: bytes(memoryview(payloads[e.store_key]).cast("B"))
                    for e in entries}
        self._pending.setdefault(version, {}).update(data)
        return [(e.store_key, _entry_path(e.rank, e.store_key), len(data[e.store_key]),
                 crc32c(data[e.store_key])) for e in entries]

    def publish(self, version: int, iteration: int, checkpoint_index: int,
                entries: Iterable[StoreEntry], rows, injector=None) -> StoreManifest:
        entries = sorted(entries)
        data = self._pending.pop(version, {})
        meta = VersionMeta(version, iteration, checkpoint_index, {e.store_key: e for e in entries})
        self._versions[version] = (meta, data)
        return self.manifest(version)

    def check_version(self, version: int) -> None:
        newest = self.newest_complete()
        if newest is not None and version <= newest:
            raise StoreError(f"version {version} not above newest complete {newest}")

    def write_version(self, version: int, iteration: int, checkpoint_index: int,
                      entries: Iterable[StoreEntry], injector=None,
                      payloads: PayloadSource = None) -> StoreManifest:
        if injector is not None:
            raise StoreError("crash injection requires the disk store")
        self.check_version(version)
        entries = sorted(entries)
        if payloads is None:
            data = {e.store_key: entry_payload(e.store_key, version, iteration) for e in entries}
        else:
            data = {e.store_key: bytes(memoryview(payloads[e.store_key]).cast("B"))
                    for e in entries}
        meta = VersionMeta(version, iteration, checkpoint_index, {e.store_key: e for e in entries})
        self._versions[version] = (meta, data)
        return self.manifest(version)

    def complete_versions(self) -> List[int]:
        return sorted(self._versions)

    def newest_complete(self) -> Optional[int]:
        return max(self._versions) if self._versions else None

    def meta(self, version: int) -> VersionMeta:
        return self._versions[version][0]

    def manifest(self, version: int) -> StoreManifest:
        if version not in self._versions:
            raise IncompleteVersionError(f"version {version} is not complete")
        meta, data = self._versions[version]
        return StoreManifest(version, meta.iteration,
                             {k: (_entry_path(meta.entries[k].rank, k), len(v), crc32c(v))
                              for k, v in data.items()}, True)

    def load_checkpoint(self, version: int, keys: Optional[Iterable[str]] = None) -> Dict[str, bytes]:
        if version not in self._versions:
            raise IncompleteVersionError(f"version {version} is not complete")
        data = self._versions[version][1]
        return dict(data) if keys is None else {k: data[k] for k in keys}

    def read_into(self, version: int, placements, verify: bool = True) -> None:
        data = self.load_checkpoint(version, list(placements))
        for k, (buf, off) in placements.items():
            v = data[k]
            memoryview(buf).cast("B")[off:off + len(v)] = v
