"""Node-shared pinned host snapshot buffers.

The two-level design keeps each completed snapshot in CPU memory so that the
surviving nodes' copies can serve recovery (engine.py:214-229; paper §4.2).
With one process per GPU, a node's snapshot buffers belong to several
processes; for a rank restored on that node to read a peer rank's in-memory
copy, the buffers live in POSIX shared memory (/dev/shm) and are registered
with CUDA (`cudaHostRegister`) by their owner, so the owner's drain is an
ordinary pinned async D2H and any process on the node can map them.
"""

from __future__ import annotations

import mmap
import os
import weakref
from typing import Optional

import numpy as np

SHM_DIR = "/dev/shm"


def _unregister(addr: int) -> None:
    import torch
    torch.cuda.cudart().cudaHostUnregister(addr)


def buffer_name(prefix: str, rank: int, buffer_id: int) -> str:
    return f"{prefix}.r{rank:04d}.b{buffer_id}"


class SharedHostBuffer:
    """A /dev/shm-backed host buffer; the owner creates and pins it, peers
    map it read-only."""

    def __init__(self, name: str, nbytes: Optional[int] = None, create: bool = True,
                 register: bool = True):
        import torch
        self.name = name
        self.path = os.path.join(SHM_DIR, name)
        self.owner = create
        if create:
            fd = os.open(self.path, os.O_CREAT | os.O_RDWR | os.O_TRUNC, 0o600)
            try:
                os.ftruncate(fd, nbytes)
                self.mm = mmap.mmap(fd, nbytes, mmap.MAP_SHARED,
                                    mmap.PROT_READ | mmap.PROT_WRITE)
            finally:
                os.close(fd)
            self.nbytes = nbytes
        else:
            fd = os.open(self.path, os.O_RDONLY)
            try:
                self.nbytes = os.fstat(fd).st_size
                self.mm = mmap.mmap(fd, self.nbytes, mmap.MAP_SHARED, mmap.PROT_READ)
            finally:
                os.close(fd)
        self.array = np.frombuffer(self.mm, dtype=np.uint8)
        self.tensor = torch.from_numpy(self.array) if create else None
        self._unregister = None
        if create and register:
            rc = torch.cuda.cudart().cudaHostRegister(self.array.ctypes.data, self.nbytes, 0)
            if int(rc) != 0:
                raise RuntimeError(f"cudaHostRegister({self.path}) failed: {rc}")
            # unregister even if the owner is dropped without close(): a
            # mapping freed while registered leaves a stale registration and
            # the next registration at that address fails (tools/thp_soak.py)
            self._unregister = weakref.finalize(self, _unregister, self.array.ctypes.data)

    @property
    def registered(self) -> bool:
        return self._unregister is not None and self._unregister.alive

    def close(self) -> None:
        if self._unregister is not None:
            self._unregister()
        self.tensor = None
        self.array = None
        try:
            self.mm.close()
        except BufferError:
            pass  # a view still exists; the mapping goes with the process
        if self.owner:
            try:
                os.unlink(self.path)
            except FileNotFoundError:
                pass
