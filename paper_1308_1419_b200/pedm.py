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


def save_packed_edm(values, n: int, features: int, path: str) -> None:
    """values: packed float32 of T(n) elements -- a numpy array or a CUDA tensor."""
    total = n * (n + 1) // 2
    try:
        f = open(path, "wb")
    except OSError:
        raise RuntimeError(f"cannot open for writing: {path}") from None
    with f:
        f.write(_header(n, features))
        if isinstance(values, np.ndarray):
            if values.dtype != np.float32 or values.size != total:
                raise ValueError("save_packed_edm: values must be float32[T(N)]")
            f.write(np.ascontiguousarray(values).tobytes())
            return
        import torch
        if values.numel() != total or values.dtype != torch.float32:
            raise ValueError("save_packed_edm: values must be float32[T(N)]")
        chunk = min(_CHUNK, total)
        stage = [torch.empty(chunk, dtype=torch.float32).pin_memory() for _ in range(2)]
        done = [torch.cuda.Event(), torch.cuda.Event()]
        stream = torch.cuda.Stream(values.device)
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
                f.write(pb[:pm].numpy().tobytes())
            pending = (buf, m, done[k % 2])
        if pending is not None:
            pb, pm, pe = pending
            pe.synchronize()
            f.write(pb[:pm].numpy().tobytes())


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
