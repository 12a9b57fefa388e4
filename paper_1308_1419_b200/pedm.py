"""PEDM binary dump of a packed EDM (reference format, edm.cpp:65-96):
16-byte header "PEDM", u32 LE version = 1, u32 N, u32 d, then the packed
binary32 values in lambda order.  Byte-compatible with the reference's
save_packed_edm / load_packed_edm.

The GPU writer streams the device buffer (8.6 GB at N=65536) through two
pinned staging buffers, overlapping the D2H copy of chunk k+1 with the file
write of chunk k.
"""
from __future__ import annotations

import struct

import numpy as np

MAGIC = b"PEDM"
VERSION = 1
_CHUNK = 64 << 20  # elements per staging chunk (256 MB)


def _header(n: int, d: int) -> bytes:
    return MAGIC + struct.pack("<III", VERSION, n, d)


def _stream_device(values, write) -> None:
    """D2H of a CUDA tensor through two pinned staging buffers: the copy of
    chunk k+1 overlaps write(bytes) of chunk k."""
    import torch
    total = values.numel()
    chunk = min(_CHUNK, total)
    if chunk == 0:
        return
    stage = [torch.empty(chunk, dtype=torch.float32).pin_memory() for _ in range(2)]
    done = [torch.cuda.Event(), torch.cuda.Event()]
    stream = torch.cuda.Stream(values.device)
    stream.wait_stream(torch.cuda.current_stream(values.device))
    pending = None
    for k, off in enumerate(range(0, total, chunk)):
        m = min(chunk, total - off)
        buf = stage[k % 2]
        with torch.cuda.stream(stream):
            buf[:m].copy_(values[off:off + m], non_blocking=True)
            done[k % 2].record(stream)
        if pending is not None:  # write the previous chunk while this one copies
            pb, pm, pe = pending
            pe.synchronize()
            write(memoryview(pb[:pm].numpy()).cast("B"))
        pending = (buf, m, done[k % 2])
    pb, pm, pe = pending
    pe.synchronize()
    write(memoryview(pb[:pm].numpy()).cast("B"))


def _check_values(values, count: int, what: str) -> None:
    if isinstance(values, np.ndarray):
        if values.dtype != np.float32 or values.size != count:
            raise ValueError(f"{what}: values must be float32[{count}]")
        return
    import torch
    if values.numel() != count or values.dtype != torch.float32:
        raise ValueError(f"{what}: values must be float32[{count}]")


def save_packed_edm(values, n: int, features: int, path: str) -> None:
    """save_packed_edm (edm.cpp:65-77).  values: packed float32 of T(n)
    elements -- a numpy array or a CUDA tensor."""
    total = n * (n + 1) // 2
    _check_values(values, total, "save_packed_edm")
    try:
        f = open(path, "wb")
    except OSError:
        raise RuntimeError(f"cannot open for writing: {path}") from None
    with f:
        f.write(_header(n, features))
        if isinstance(values, np.ndarray):
            f.write(np.ascontiguousarray(values).tobytes())
        else:
            _stream_device(values.reshape(-1), f.write)


def save_packed_edm_shard(values, n: int, features: int, path: str, elem_begin: int) -> None:
    """One lambda-range shard of a packed EDM into ONE shared PEDM file: the
    shard's elements [elem_begin, elem_begin + len(values)) (global packed
    order, trigrid.shard_elems) land at byte 16 + 4 elem_begin of a file
    preallocated to the full 16 + 4 T(n) bytes.  Every rank of a sharded job
    calls it with its own slice (in any order, concurrently); each writes the
    same header, so the result is byte-identical to save_packed_edm of the
    whole matrix (edm.cpp:65-77) once all shards are written."""
    import os
    total = n * (n + 1) // 2
    count = values.size if isinstance(values, np.ndarray) else values.numel()
    if elem_begin < 0 or elem_begin + count > total:
        raise ValueError("save_packed_edm_shard: shard range outside [0, T(N))")
    _check_values(values, count, "save_packed_edm_shard")
    try:
        fd = os.open(path, os.O_RDWR | os.O_CREAT, 0o644)
    except OSError:
        raise RuntimeError(f"cannot open for writing: {path}") from None
    try:
        size = 16 + 4 * total
        if os.fstat(fd).st_size < size:
            os.ftruncate(fd, size)  # sparse preallocation; shards fill it
        os.pwrite(fd, _header(n, features), 0)
        pos = [16 + 4 * elem_begin]

        def write(b):
            mv = memoryview(b).cast("B")
            while len(mv):
                k = os.pwrite(fd, mv, pos[0])
                pos[0] += k
                mv = mv[k:]

        if isinstance(values, np.ndarray):
            write(np.ascontiguousarray(values))
        else:
            _stream_device(values.reshape(-1), write)
    except OSError as exc:
        raise RuntimeError(f"write failed: {path}: {exc}") from None
    finally:
        os.close(fd)


def load_packed_edm(path: str):
    """Returns (values float32[T(N)], N, d); RuntimeError like the reference."""
    try:
        f = open(path, "rb")
    except OSError:
        raise RuntimeError(f"cannot open for reading: {path}") from None
    with f:
        head = f.read(16)
        if len(head) < 4 or head[:4] != MAGIC:
            raise RuntimeError(f"not a PEDM file: {path}")
        if len(head) < 16:
            raise RuntimeError(f"truncated PEDM file: {path}")
        version, n, d = struct.unpack("<III", head[4:16])
        if version != VERSION:
            raise RuntimeError("unsupported PEDM version")
        total = n * (n + 1) // 2
        data = np.fromfile(f, dtype=np.float32, count=total)
        if data.size != total:
            raise RuntimeError(f"truncated PEDM file: {path}")
    return data, n, d
