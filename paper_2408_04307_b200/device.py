"""ctypes binding of libpec.so (include/pec.h) — the only way into the kernels.

There is no fallback: if the shared object is missing or fails to load, every
entry point raises.  Build it with `python -m paper_2408_04307_b200._build`
or `__graft_entry__.build()`.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path
from typing import Optional

import numpy as np

from .topology import SpecValidationError

# PEC_LIB=debug loads the build with device-side invariant checks (test
# tooling, tools/guard_kernels.py); there is no other variant and no fallback
LIB_PATH = Path(__file__).resolve().parent / "_lib" / (
    "libpec_debug.so" if os.environ.get("PEC_LIB") == "debug" else "libpec.so")
ABI_VERSION = 1

PEC_OK = 0
PEC_E_INVAL = -1
PEC_E_CUDA = -2
PEC_E_RANGE = -3
PEC_E_IO = -4
PEC_E_CRASH = -5

# numpy mirror of `pec_copy_desc`
DESC_DTYPE = np.dtype([("src", "<u8"), ("dst", "<u8"), ("nbytes", "<u8"),
                       ("first_chunk", "<u8")])
# numpy mirror of `pec_plan_template`
TEMPLATE_DTYPE = np.dtype([("src_offset", "<u8"), ("nbytes", "<u8"), ("layer", "<i4"),
                           ("expert", "<i4"), ("reserved", "<u8")])
DEFAULT_CHUNK_LOG2 = 15  # 32 KiB work chunks

MODE_AUTO, MODE_VEC, MODE_BULK = 0, 1, 2


def crc_scratch_words(total_chunks: int) -> int:
    """pec_pack_crc / pec_crc_device scratch: one uint32 per 32 KiB chunk plus
    the kernel's work counter."""
    return int(total_chunks) + 1


MODE_CRC = 3  # engine-level: pack with fused per-entry CRC-32C (pec_pack_crc); default with a store

_lib = None


class PecKernelError(RuntimeError):
    """A libpec call failed on the device side."""


def _load():
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: the PEC CUDA extension is not built "
            "(run `python -m paper_2408_04307_b200._build`); there is no CPU fallback")
    lib = ctypes.CDLL(str(LIB_PATH))
    c_int, c_i64, c_u64, c_u32, vp = (ctypes.c_int, ctypes.c_int64, ctypes.c_uint64,
                                      ctypes.c_uint32, ctypes.c_void_p)
    sig = {
        "pec_abi_version": (c_int, []),
        "pec_strerror": (ctypes.c_char_p, [c_int]),
        "pec_token_hist": (c_int, [vp, c_int, c_i64, c_int, vp, vp, c_int, vp, vp, vp]),
        "pec_token_hist_i64": (c_int, [vp, c_int, c_i64, c_int, vp, vp, c_int, vp, vp, vp]),
        "pec_select_sequential": (c_int, [c_i64, c_int, c_int, c_int, c_int, vp, vp]),
        "pec_select_load_aware": (c_int, [vp, c_int, c_int, c_int, vp, c_int, vp, c_int, vp]),
        "pec_pack": (c_int, [vp, c_int, c_u64, c_int, c_int, vp]),
        "pec_unpack": (c_int, [vp, c_int, c_u64, c_int, c_int, vp]),
        "pec_plan_chunks": (c_i64, [vp, c_int, c_int]),
        "pec_expand_plan": (c_int, [vp, c_int, vp, c_int, c_int, c_u64, c_u64, c_int, c_int,
                                    vp, vp, vp]),
        "pec_pack_indirect": (c_int, [vp, c_int, c_u64, vp, c_int, c_int, vp]),
        "pec_pack_crc": (c_int, [vp, c_int, c_u64, vp, c_int, vp, vp, vp]),
        "pec_crc_device": (c_int, [vp, c_int, c_u64, vp, c_int, vp, vp, vp]),
        "pec_crc32c": (c_u32, [vp, ctypes.c_size_t, c_u32]),
        "pec_crc32c_combine": (c_u32, [c_u32, c_u32, c_u64]),
        "pec_crc32c_many": (c_int, [vp, vp, vp, c_int, vp, c_int]),
        "pec_write_files": (c_int, [vp, vp, vp, c_int, vp, c_int, c_int]),
        "pec_write_files_budget": (c_int, [vp, vp, vp, c_int, vp, c_int, c_int, vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    got = lib.pec_abi_version()
    if got != ABI_VERSION:
        raise ImportError(f"libpec ABI {got} != expected {ABI_VERSION}; rebuild")
    _lib = lib
    return lib


def lib():
    return _load()


def exported_symbols():
    """Names declared in include/pec.h (for the ABI tests)."""
    return ["pec_abi_version", "pec_strerror", "pec_token_hist", "pec_token_hist_i64",
            "pec_select_sequential",
            "pec_select_load_aware", "pec_pack", "pec_unpack", "pec_plan_chunks",
            "pec_expand_plan", "pec_pack_indirect", "pec_pack_crc", "pec_crc_device",
            "pec_crc32c", "pec_crc32c_combine", "pec_crc32c_many", "pec_write_files",
            "pec_write_files_budget"]


def _check(rc: int, what: str) -> None:
    if rc == PEC_OK:
        return
    text = lib().pec_strerror(rc).decode()
    if rc in (PEC_E_INVAL, PEC_E_RANGE):
        raise SpecValidationError(f"{what} arguments", text)
    if rc == PEC_E_IO:
        raise OSError(f"{what}: {text}")
    raise PecKernelError(f"{what}: {text} (code {rc})")


# ---------------------------------------------------------------------------
# torch helpers (imported lazily so host-only users need no torch)
# ---------------------------------------------------------------------------

def _stream_handle(stream=None, device=None) -> int:
    import torch
    if stream is None:
        stream = torch.cuda.current_stream(device)
    return int(stream.cuda_stream)


def _dev_ptr(t, dtype, what: str, ndim: Optional[int] = None) -> int:
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise SpecValidationError(f"{what} is a CUDA tensor", f"got {type(t).__name__}")
    if t.dtype != dtype:
        raise SpecValidationError(f"{what}.dtype == {dtype}", f"got {t.dtype}")
    if not t.is_contiguous():
        raise SpecValidationError(f"{what} contiguous", "non-contiguous tensor")
    if ndim is not None and t.dim() != ndim:
        raise SpecValidationError(f"{what}.dim() == {ndim}", f"got {t.dim()}")
    return t.data_ptr()


# ---------------------------------------------------------------------------
# device entry points
# ---------------------------------------------------------------------------

def token_hist(idx, counters, scratch, cap=None, delivered=None, stream=None) -> None:
    """counters[t] += min(bincount(idx[l]), cap[l]) for every tier t
    (pec_token_hist / pec_token_hist_i64).  idx [L, n] int32 or int64 (as
    torch.topk returns it), counters [tiers, L, E] int64, scratch [L*E+1]
    int32 zeros (reused), cap [L] int64, delivered [L, E]."""
    import torch
    if idx.dim() == 3 and idx.is_contiguous():   # [L, tokens, top_k] as stacked topk output
        idx = idx.view(idx.shape[0], -1)
    L, n = idx.shape
    tiers, L2, E = counters.shape
    if L2 != L:
        raise SpecValidationError("counters.shape[1] == idx.shape[0]", f"{L2} != {L}")
    if scratch.numel() < L * E + 1:
        raise SpecValidationError("scratch.numel() >= L*E+1", f"got {scratch.numel()}")
    cap_p = _dev_ptr(cap, torch.int64, "cap", 1) if cap is not None else None
    del_p = _dev_ptr(delivered, torch.int64, "delivered", 2) if delivered is not None else None
    wide = idx.dtype == torch.int64
    fn = lib().pec_token_hist_i64 if wide else lib().pec_token_hist
    rc = fn(_dev_ptr(idx, torch.int64 if wide else torch.int32, "idx", 2), L, n, E, cap_p,
            _dev_ptr(counters, torch.int64, "counters", 3), tiers, del_p,
            _dev_ptr(scratch, torch.int32, "scratch"), _stream_handle(stream, idx.device))
    _check(rc, "pec_token_hist")


def select_sequential(c: int, n_layers: int, n_experts: int, width: int, stride: int,
                      out, stream=None) -> None:
    import torch
    w = min(width, n_experts)
    if out.numel() != n_layers * w:
        raise SpecValidationError("out.numel() == L*min(width,E)", f"got {out.numel()}")
    rc = lib().pec_select_sequential(int(c), n_layers, n_experts, width, stride,
                                     _dev_ptr(out, torch.int32, "out"),
                                     _stream_handle(stream, out.device))
    _check(rc, "pec_select_sequential")


def select_load_aware(counters, k: int, out, pool=None, zero_selected: bool = False,
                      stream=None) -> None:
    """counters [L, E] int64 (modified when zero_selected), out [L, k] int32,
    pool [L, P] int32 or None."""
    import torch
    L, E = counters.shape
    if tuple(out.shape) != (L, k):
        raise SpecValidationError("out.shape == (L, k)", f"got {tuple(out.shape)}")
    pool_p, P = None, 0
    if pool is not None:
        pool_p = _dev_ptr(pool, torch.int32, "pool", 2)
        P = pool.shape[1]
    rc = lib().pec_select_load_aware(_dev_ptr(counters, torch.int64, "counters", 2), L, E, k,
                                     pool_p, P, _dev_ptr(out, torch.int32, "out", 2),
                                     1 if zero_selected else 0,
                                     _stream_handle(stream, counters.device))
    _check(rc, "pec_select_load_aware")


def plan_chunks(table: np.ndarray, chunk_log2: int = DEFAULT_CHUNK_LOG2) -> int:
    """Fill table['first_chunk'] in place (pec_plan_chunks); returns total."""
    if table.dtype != DESC_DTYPE or not table.flags["C_CONTIGUOUS"]:
        raise SpecValidationError("table is a contiguous DESC_DTYPE array", str(table.dtype))
    total = lib().pec_plan_chunks(table.ctypes.data if len(table) else None, len(table),
                                  chunk_log2)
    if total < 0:
        _check(int(total), "pec_plan_chunks")
    return int(total)


def _copy(fn_name: str, desc_dev, n: int, total_chunks: int, chunk_log2: int, mode: int,
          stream=None) -> None:
    import torch
    if n == 0 or total_chunks == 0:
        return
    if desc_dev.numel() * desc_dev.element_size() < n * DESC_DTYPE.itemsize:
        raise SpecValidationError("descriptor table holds n entries",
                                  f"{desc_dev.numel()} elements for n={n}")
    ptr = _dev_ptr(desc_dev, desc_dev.dtype, "descriptor table")
    if ptr % 8:
        raise SpecValidationError("descriptor table 8-byte aligned", hex(ptr))
    fn = getattr(lib(), fn_name)
    _check(fn(ptr, n, total_chunks, chunk_log2, mode, _stream_handle(stream, desc_dev.device)),
           fn_name)


def pack(desc_dev, n, total_chunks, chunk_log2=DEFAULT_CHUNK_LOG2, mode=MODE_AUTO, stream=None):
    _copy("pec_pack", desc_dev, n, total_chunks, chunk_log2, mode, stream)


def unpack(desc_dev, n, total_chunks, chunk_log2=DEFAULT_CHUNK_LOG2, mode=MODE_AUTO, stream=None):
    _copy("pec_unpack", desc_dev, n, total_chunks, chunk_log2, mode, stream)


def expand_plan(tmpl_dev, n: int, sel, state_base: int, stage_base: int, out_dev, totals_dev,
                chunk_log2: int = DEFAULT_CHUNK_LOG2, stage_align: int = 256, stream=None) -> None:
    """Device-side plan expansion (pec_expand_plan): filter the rank's
    all-experts template by sel [L, K] into a ready descriptor table."""
    import torch
    if stage_align & (stage_align - 1):
        raise SpecValidationError("stage_align is a power of two", str(stage_align))
    L, K = sel.shape
    rc = lib().pec_expand_plan(_dev_ptr(tmpl_dev, tmpl_dev.dtype, "template"), n,
                               _dev_ptr(sel, torch.int32, "sel", 2), L, K, state_base, stage_base,
                               chunk_log2, stage_align,
                               _dev_ptr(out_dev, out_dev.dtype, "descriptor table"),
                               _dev_ptr(totals_dev, torch.int64, "totals"),
                               _stream_handle(stream, sel.device))
    _check(rc, "pec_expand_plan")


def _crc_call(fn_name: str, desc_dev, n: int, total_chunks: int, chunk_crc_dev, entry_crc_dev,
              chunk_log2: int, stream, totals_dev) -> None:
    import torch
    if n == 0:
        return
    if chunk_crc_dev.numel() < crc_scratch_words(total_chunks) \
            or entry_crc_dev.numel() < n:
        raise SpecValidationError("crc buffers large enough", "chunk/entry crc buffers too small")
    tdev = _dev_ptr(totals_dev, torch.int64, "totals") if totals_dev is not None else None
    rc = getattr(lib(), fn_name)(_dev_ptr(desc_dev, desc_dev.dtype, "descriptor table"), n,
                                 total_chunks, tdev, chunk_log2,
                                 _dev_ptr(chunk_crc_dev, torch.int32, "chunk crc"),
                                 _dev_ptr(entry_crc_dev, torch.int32, "entry crc"),
                                 _stream_handle(stream, desc_dev.device))
    _check(rc, fn_name)


def pack_crc(desc_dev, n: int, total_chunks: int, chunk_crc_dev, entry_crc_dev,
             chunk_log2: int = DEFAULT_CHUNK_LOG2, stream=None, totals_dev=None) -> None:
    """pec_pack with the CRC-32C of every entry computed in the same pass
    (entry_crc_dev [n] int32 device; chunk_crc_dev [total] scratch)."""
    _crc_call("pec_pack_crc", desc_dev, n, total_chunks, chunk_crc_dev, entry_crc_dev,
              chunk_log2, stream, totals_dev)


def crc_device(desc_dev, n: int, total_chunks: int, chunk_crc_dev, entry_crc_dev,
               chunk_log2: int = DEFAULT_CHUNK_LOG2, stream=None, totals_dev=None) -> None:
    """pec_crc_device: CRC-32C of each descriptor's device source range, no copy."""
    _crc_call("pec_crc_device", desc_dev, n, total_chunks, chunk_crc_dev, entry_crc_dev,
              chunk_log2, stream, totals_dev)


def pack_indirect(desc_dev, n: int, max_chunks: int, totals_dev,
                  chunk_log2: int = DEFAULT_CHUNK_LOG2, mode: int = MODE_AUTO, stream=None) -> None:
    """pec_pack over a device-built table; chunk count read from totals_dev[0]."""
    import torch
    if n == 0 or max_chunks == 0:
        return
    rc = lib().pec_pack_indirect(_dev_ptr(desc_dev, desc_dev.dtype, "descriptor table"), n,
                                 max_chunks, _dev_ptr(totals_dev, torch.int64, "totals"),
                                 chunk_log2, mode, _stream_handle(stream, desc_dev.device))
    _check(rc, "pec_pack_indirect")


# ---------------------------------------------------------------------------
# host CRC-32C
# ---------------------------------------------------------------------------

def _host_buffer(data):
    """(address, nbytes, keepalive) of a bytes-like object, ndarray or CPU tensor."""
    if isinstance(data, (bytes, bytearray, memoryview)):
        arr = np.frombuffer(data, dtype=np.uint8)
        return (arr.ctypes.data if arr.nbytes else 0), arr.nbytes, (arr, data)
    if isinstance(data, np.ndarray):
        if not data.flags["C_CONTIGUOUS"]:
            data = np.ascontiguousarray(data)
        return data.ctypes.data, data.nbytes, data
    import torch
    if isinstance(data, torch.Tensor):
        if data.is_cuda:
            raise SpecValidationError("crc32c input on host", "got a CUDA tensor")
        t = data.contiguous()
        return t.data_ptr(), t.numel() * t.element_size(), t
    raise TypeError(f"unsupported buffer type {type(data).__name__}")


def crc32c(data, crc: int = 0) -> int:
    """CRC-32C, identical to the reference store.crc32c (store.py:49-70)."""
    addr, n, keep = _host_buffer(data)
    if n == 0:
        return crc & 0xFFFFFFFF
    out = lib().pec_crc32c(addr, n, crc & 0xFFFFFFFF)
    del keep
    return int(out)


def crc32c_combine(crc_a: int, crc_b: int, len_b: int) -> int:
    return int(lib().pec_crc32c_combine(crc_a & 0xFFFFFFFF, crc_b & 0xFFFFFFFF, len_b))


def crc32c_many(base, offsets, lengths, threads: Optional[int] = None) -> np.ndarray:
    """CRC-32C of many regions of one host buffer, multithreaded."""
    addr, nbytes, keep = _host_buffer(base)
    offs = np.ascontiguousarray(offsets, dtype=np.uint64)
    lens = np.ascontiguousarray(lengths, dtype=np.uint64)
    if offs.shape != lens.shape:
        raise SpecValidationError("len(offsets) == len(lengths)", f"{offs.shape} {lens.shape}")
    if len(offs) and int((offs + lens).max()) > nbytes:
        raise SpecValidationError("regions inside buffer", "region exceeds buffer")
    out = np.zeros(len(offs), dtype=np.uint32)
    if threads is None:
        threads = max(1, len(os.sched_getaffinity(0)))
    rc = lib().pec_crc32c_many(addr, offs.ctypes.data, lens.ctypes.data, len(offs),
                               out.ctypes.data, int(threads))
    _check(rc, "pec_crc32c_many")
    del keep
    return out


def write_files(paths, buffers, threads: Optional[int] = None, want_crc: bool = True,
                fsync: bool = False, direct: bool = False, background: bool = False,
                overwrite: bool = False, budget: Optional[int] = None):
    """Native multi-threaded writer (pec_write_files): file i <- buffers[i]
    (bytes-like / ndarray / CPU tensor).  Returns the CRC-32C of each file
    (uint32 ndarray) when ``want_crc``.  ``direct`` opens files O_DIRECT
    (page-cache bypass; buffered where the filesystem refuses it; large files
    range-parallel); ``background`` runs the writer threads at nice +10;
    ``overwrite`` rewrites existing files in place (recycled files).

    ``budget`` (crash injection, pec_write_files_budget): at most that many
    bytes are written, spent in file order like the sequential writer; then
    the return value is ``(crcs or None, bytes_left, crashed)``."""
    n = len(paths)
    keep = [_host_buffer(b) for b in buffers]
    c_paths = (ctypes.c_char_p * n)(*[os.fsencode(str(p)) for p in paths])
    c_bufs = (ctypes.c_void_p * n)(*[k[0] for k in keep])
    lens = np.array([k[1] for k in keep], dtype=np.uint64)
    out = np.zeros(n, dtype=np.uint32) if want_crc else None
    if threads is None:
        threads = max(1, len(os.sched_getaffinity(0)))
    flags = (1 if fsync else 0) | (2 if direct else 0) | (4 if background else 0) | \
        (8 if overwrite else 0)
    args = (ctypes.cast(c_paths, ctypes.c_void_p), ctypes.cast(c_bufs, ctypes.c_void_p),
            lens.ctypes.data if n else None, n, out.ctypes.data if want_crc and n else None,
            int(threads), flags)
    if budget is None:
        rc = lib().pec_write_files(*args)
        _check(rc, "pec_write_files")
        del keep
        return out
    left = np.array([max(0, int(budget))], dtype=np.uint64)
    rc = lib().pec_write_files_budget(*args, left.ctypes.data)
    if rc != PEC_E_CRASH:
        _check(rc, "pec_write_files_budget")
    del keep
    return (out if rc == PEC_OK else None), int(left[0]), rc == PEC_E_CRASH
