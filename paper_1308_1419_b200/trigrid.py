"""Drop-in mirror of the reference's Python module ``trigrid`` / ``_trigrid``
(/root/reference/proj/python/trigrid/__init__.py:5-51,
 /root/reference/proj/bindings/module.cpp:55-183), running on a B200.

Same 21 names, argument names, defaults, return shapes and exception classes
as the reference.  The hot calls (``edm_strategy``, ``coverage_ok``,
``gen_points``) run the sm_100a kernels of libtrigrid_b200.so through its
C-ABI; the scalar mapping helpers (``ltm_map``, ``utm_map``, ...) run the same
``__host__ __device__`` mapping code on the host with the reference's binary32
arithmetic and repair policy.  ``edm_reference`` is the reference API's
sequential oracle (edm.cpp:53-63) and stays sequential host code by contract --
it is what device results are checked against, never a fallback for them.
Differences from the reference, all documented in DESIGN.md: ``workers`` is
accepted and ignored; ``DispatchStats.wall_time_ns`` is device time;
``rec_decompose(n, 0)`` returns None where the reference divides by zero.

Extensions beyond the reference surface (same module): ``edm`` (any d, device
tensors, shards), ``launch``, ``collide``, ``coverage``, ``grid_spec``,
``lambda_sweep``, ``sqrt_selftest``, ``shard_rows``, ``shard_elems``,
``dispatch_stats``.
"""
from __future__ import annotations

import ctypes as C
import operator

import numpy as np

from . import _lib

__version__ = "0.1.0"

_ENGINE_NAMES = {"native": 0, "ltm-x": 0, "newton": 1, "ltm-n": 1, "reciprocal": 2, "ltm-r": 2, "exact": 3}
_REF_STRATEGIES = ("bb", "ltm-x", "ltm-n", "ltm-r", "utm", "rb", "rec")


def _L():
    return _lib.load()


def _u64(x, name: str) -> int:
    """pybind11's uint64 caster: integral (incl. __index__) and >= 0, else TypeError."""
    if isinstance(x, float):
        raise TypeError(f"incompatible function arguments: {name} must be an integer")
    try:
        v = operator.index(x)
    except TypeError:
        raise TypeError(f"incompatible function arguments: {name} must be an integer") from None
    if v < 0 or v >= 1 << 64:
        raise TypeError(f"incompatible function arguments: {name} out of uint64 range")
    return v


def _engine(name: str) -> int:
    if name not in _ENGINE_NAMES:
        raise ValueError(f"unknown engine '{name}'")
    return _ENGINE_NAMES[name]


def _strategy(name: str, allow_extended: bool = False) -> int:
    if name in _lib.STRATEGIES and (allow_extended or name in _REF_STRATEGIES):
        return _lib.STRATEGIES[name]
    raise ValueError(f"unknown strategy '{name}'")


def _points(points) -> np.ndarray:
    """py::array_t<float, c_style> without forcecast (module.cpp:29-36): safe
    casts and sequences convert, float64/int32 arrays raise TypeError."""
    if isinstance(points, np.ndarray):
        if points.dtype != np.float32 and not np.can_cast(points.dtype, np.float32, "safe"):
            raise TypeError("edm_strategy(): incompatible function arguments: points must be "
                            "a float32-compatible array")
        arr = np.ascontiguousarray(points, dtype=np.float32)
    else:
        try:
            arr = np.ascontiguousarray(np.asarray(points, dtype=np.float32))
        except (TypeError, ValueError):
            raise TypeError("incompatible function arguments: points") from None
    if arr.ndim != 2:
        raise ValueError("points must be a 2-D float32 array")
    return arr


# ------------------------------------------------------------ L0 core

def tri_count(n, with_diag: bool = True) -> int:
    """Lower-triangular cell count over an n x n grid (tri.hpp:39-41)."""
    return int(_L().tg_tri_count(_u64(n, "n"), int(bool(with_diag))))


def tri_linear_index(i, j) -> int:
    """Packed row-major index i(i+1)/2 + j (tri.cpp:17-21)."""
    out = C.c_uint64()
    _lib.check(_L().tg_tri_linear_index(_u64(i, "i"), _u64(j, "j"), C.byref(out)))
    return out.value


def grid_side_balanced(n) -> int:
    """Balanced grid side ceil(sqrt(n(n+1)/2)) (tri.cpp:23-26)."""
    out = C.c_uint64()
    _lib.check(_L().tg_grid_side_balanced(_u64(n, "n"), C.byref(out)))
    return out.value


def enumerate_lower(n, with_diag: bool = True):
    """All (i, j) of the lower triangle in ascending lambda order (module.cpp:66-76)."""
    n = _u64(n, "n")
    if tri_count(n, with_diag) > (1 << 24):
        raise ValueError("enumeration too large to materialize")
    return [(i, j) for i in range(0 if with_diag else 1, n) for j in range(i + 1 if with_diag else i)]


def isqrt(v) -> int:
    """Exact floor square root (fastmath.cpp:8-16)."""
    return int(_L().tg_isqrt(_u64(v, "v")))


def fast_inv_sqrt(x: float, iterations: int = 3) -> float:
    """Carmack 0x5f3759df inverse square root, binary32 (fastmath.hpp:22-34)."""
    return float(_L().tg_fast_inv_sqrt(float(x), int(iterations)))


def rsqrt_single(x: float) -> float:
    """Binary32 reciprocal square root (fastmath.hpp:39)."""
    return float(_L().tg_rsqrt_single(float(x)))


def sqrt_via(engine: str, x: float) -> float:
    """sqrt(x) through an engine: native, newton, reciprocal or exact (fastmath.cpp:33-59)."""
    out = C.c_double()
    _lib.check(_L().tg_sqrt_via(_engine(engine), float(x), C.byref(out)))
    return out.value


# ------------------------------------------------------------ L1 mappers

_REPAIR = {"auto": 0, "off": 1, "on": 2}


def ltm_map(lam, engine: str = "reciprocal", with_diag: bool = True, repair: str = "auto"):
    """g(lambda): packed block index to (i, j) (strategies.cpp:60-83) with the
    reference's RepairPolicy (fastmath.hpp:84-103; module.cpp:90-96 uses Auto)."""
    i, j = C.c_uint64(), C.c_uint64()
    if repair not in _REPAIR:
        raise ValueError(f"unknown repair policy '{repair}'")
    _lib.check(_L().tg_ltm_map_policy(_u64(lam, "lam"), _engine(engine), int(bool(with_diag)), _REPAIR[repair],
                                      C.byref(i), C.byref(j)))
    return i.value, j.value


def bb_map(x, y):
    """Bounding-box block map; None when the block is discarded (strategies.hpp:94-97)."""
    i, j = C.c_uint64(), C.c_uint64()
    if not _L().tg_bb_map(_u64(x, "x"), _u64(y, "y"), C.byref(i), C.byref(j)):
        return None
    return i.value, j.value


def utm_map(k, n, engine: str = "newton"):
    """Upper-triangular pair (a, b), 0-based, a < b (strategies.cpp:85-91)."""
    a, b = C.c_uint64(), C.c_uint64()
    _lib.check(_L().tg_utm_map(_u64(k, "k"), _u64(n, "n"), _engine(engine), C.byref(a), C.byref(b)))
    return a.value, b.value


def rb_rect(n):
    """Rectangular-box thread rectangle (width, height) (strategies.cpp:93-97)."""
    w, h = C.c_uint64(), C.c_uint64()
    _lib.check(_L().tg_rb_rect(_u64(n, "n"), C.byref(w), C.byref(h)))
    return w.value, h.value


def rb_map(tx, ty, n):
    """Rectangular-box thread map; None outside the rectangle (strategies.hpp:182-193)."""
    i, j = C.c_uint64(), C.c_uint64()
    if not _L().tg_rb_map(_u64(tx, "tx"), _u64(ty, "ty"), _u64(n, "n"), C.byref(i), C.byref(j)):
        return None
    return i.value, j.value


def rec_decompose(n, rho=16):
    """Largest-k decomposition N = m*2^k, or None (strategies.cpp:142-151)."""
    m, k = C.c_uint64(), C.c_uint32()
    if not _L().tg_rec_decompose(_u64(n, "n"), _u64(rho, "rho"), C.byref(m), C.byref(k)):
        return None
    return m.value, k.value


def count_wasted(strategy: str, n) -> int:
    """Closed-form wasted blocks, bb and ltm flavors only (engine.cpp:205-217)."""
    out = C.c_uint64()
    _lib.check(_L().tg_count_wasted(_strategy(strategy), _u64(n, "n"), C.byref(out)))
    return out.value


def ltm_diag_waste_blocks(n) -> float:
    """engine.cpp:219-221: n / 2 (no pybind binding in the reference; C++ surface)."""
    return float(_L().tg_ltm_diag_waste_blocks(_u64(n, "n")))


def improvement_model(beta: float, tau: float, n: float) -> float:
    """Modeled improvement factor 2*beta*n^2/(tau*n^2 + tau*n) (bench.cpp:138-144)."""
    out = C.c_double()
    _lib.check(_L().tg_improvement_model(float(beta), float(tau), float(n), C.byref(out)))
    return out.value


# ----------------------------------------------------- GPU hot path

def gen_points(n, d, seed=42) -> np.ndarray:
    """Deterministic uniform [0,1) points, shape (n, d) float32 (edm.cpp:38-51),
    generated on device."""
    n, d, seed = _u64(n, "n"), _u64(d, "d"), _u64(seed, "seed")
    if n == 0:
        raise ValueError("gen_points: N must be >= 1")
    if n > (1 << 20):
        raise ValueError("gen_points: N exceeds the 2^20 cap")
    if d < 1 or d > 4:
        raise ValueError("gen_points: d must be in [1, 4]")
    out = np.empty((n, d), dtype=np.float32)
    _lib.check(_L().tg_gen_points_host(n, d, seed, out.ctypes.data, -1))
    return out


def _stats_dict(st: _lib.tg_dispatch_stats) -> dict:
    return st.as_dict()


def edm_strategy(strategy: str, points, rho=16, workers=0, *, out: np.ndarray | None = None,
                 device: int = -1, mode: str = "auto", shard: tuple[int, int] | None = None,
                 devices: list[int] | None = None, rec: tuple[int, int] | None = None):
    """Packed distance matrix through a mapping strategy, plus dispatch stats
    (module.cpp:149-161).  Runs the sm_100a td-kernel; host in, host out.

    Extensions: ``out`` -- a preallocated host float32 buffer of T(N) (or the
    shard's) elements, ideally pinned, written in place and returned;
    ``shard=(g, G)`` -- compute lambda-range shard g of G only;
    ``devices=[d0, d1, ...]`` -- split the lambda range over several GPUs of
    this process, each copying its slice out over its own PCIe link;
    ``rec=(m, k)`` -- an explicit rec_schedule (strategies.cpp:116-140)."""
    s = _strategy(strategy, allow_extended=True)
    pts = _points(points)
    rho = _u64(rho, "rho")
    _u64(workers, "workers")
    n, d = pts.shape
    if n == 0:
        raise ValueError("ProblemSize: N must be >= 1")
    if shard is not None and shard[1] > 1:
        b, e = shard_elems(n, rho, shard[0], shard[1])
        size = e - b
    else:
        size = tri_count(n)
    if out is None:
        out = np.empty(size, dtype=np.float32)
    elif out.dtype != np.float32 or out.size < size or not out.flags.c_contiguous:
        raise ValueError("edm_strategy: out must be a C-contiguous float32 array of the packed size")
    st = _lib.tg_dispatch_stats()
    dv = (C.c_int32 * len(devices))(*devices) if devices else None
    o = _lib.opts(device=device, mode=mode, shard=shard, devices=dv, rec=rec)
    _lib.check(_L().tg_edm_strategy_host(s, pts.ctypes.data, n, d, rho, out.ctypes.data,
                                         C.byref(o), C.byref(st)))
    return out[:size] if out.size != size else out, _stats_dict(st)


def edm_reference(points) -> np.ndarray:
    """The reference's sequential oracle (edm.cpp:53-63): every pair j <= i in
    row-major order with edm_pair's binary32 arithmetic, any d.  Sequential
    host code by contract (it is what launch results are verified against)."""
    pts = _points(points)
    n, d = pts.shape
    if n == 0:
        raise ValueError("ProblemSize: N must be >= 1")
    out = np.empty(n * (n + 1) // 2, dtype=np.float32)
    _lib.check(_L().tg_edm_reference_host(pts.ctypes.data, n, d, out.ctypes.data))
    return out


def coverage_ok(strategy: str, n, rho=16, workers=0) -> bool:
    """True when the strategy touches every domain cell exactly once
    (module.cpp:163-172); the COUNT kernel runs on device in the execution
    shape the EDM / write launches use (span where eligible)."""
    s = _strategy(strategy)
    ok = C.c_int()
    _u64(workers, "workers")
    _lib.check(_L().tg_coverage_ok(s, _u64(n, "n"), _u64(rho, "rho"), -1, C.byref(ok)))
    return bool(ok.value)


def coverage(strategy: str, n: int, rho: int = 16, mode: str = "auto", rec: tuple[int, int] | None = None,
             engine: str | None = None, device: int = -1) -> dict:
    """Exactly-once check with its details: {"ok", "bad", "first_bad"}; mode
    "span" checks the owned-chunk rule of the span kernels, "grid" the
    paper-faithful one-thread-per-cell kernel."""
    ok, bad, first = C.c_int(), C.c_uint64(), C.c_uint64()
    o = _lib.opts(device=device, mode=mode, rec=rec, engine=None if engine is None else _engine(engine))
    _lib.check(_L().tg_coverage_ok_opts(_strategy(strategy, True), n, rho, C.byref(o), C.byref(ok), C.byref(bad),
                                        C.byref(first)))
    return {"ok": bool(ok.value), "bad": bad.value,
            "first_bad": None if first.value == (1 << 64) - 1 else first.value}


def grid_spec(strategy: str, n: int, rho: int = 16, rec: tuple[int, int] | None = None) -> list[dict]:
    """grid_of(make_strategy(...)).passes (strategies.hpp:393-400)."""
    o = _lib.opts(rec=rec)
    cnt = C.c_uint32()
    _lib.check(_L().tg_grid_spec(_strategy(strategy, True), n, rho, C.byref(o), None, 0, C.byref(cnt)))
    arr = (_lib.tg_pass * cnt.value)()
    _lib.check(_L().tg_grid_spec(_strategy(strategy, True), n, rho, C.byref(o), arr, cnt.value, C.byref(cnt)))
    return [p.as_dict() for p in arr]


# ------------------------------------------------------------ extensions

def dispatch_stats(strategy: str, n: int, rho: int = 16, shard: tuple[int, int] | None = None,
                   rec: tuple[int, int] | None = None, per_pass: bool = False) -> dict:
    """Closed-form DispatchStats (what run_strategy tallies, engine.cpp:70-136);
    per_pass=True adds the per-pass list (LaunchOptions::per_pass)."""
    st = _lib.tg_dispatch_stats()
    npass = len(grid_spec(strategy, n, rho, rec)) if per_pass else 0
    pp = (_lib.tg_dispatch_stats * npass)() if per_pass else None
    o = _lib.opts(shard=shard, rec=rec, per_pass=pp)
    _lib.check(_L().tg_dispatch_stats_opts(_strategy(strategy, True), n, rho, C.byref(o), C.byref(st)))
    d = _stats_dict(st)
    if per_pass:
        d["per_pass"] = [x.as_dict() for x in pp]
    return d


def shard_rows(n: int, rho: int, shard_count: int) -> list[int]:
    rows = (C.c_uint64 * (shard_count + 1))()
    _lib.check(_L().tg_shard_rows(n, rho, shard_count, rows))
    return [int(r) for r in rows]


def shard_elems(n: int, rho: int, shard_index: int, shard_count: int, with_diag: bool = True):
    b, e = C.c_uint64(), C.c_uint64()
    _lib.check(_L().tg_shard_elems(n, rho, shard_index, shard_count, int(with_diag), C.byref(b), C.byref(e)))
    return b.value, e.value


def _device_of(*tensors) -> int:
    """The CUDA ordinal the launch runs on: that of its tensors (they must
    agree), else torch's current device."""
    import torch
    devs = {t.device.index for t in tensors if t is not None and hasattr(t, "device") and t.device.type == "cuda"}
    if len(devs) > 1:
        raise ValueError(f"tensors on different CUDA devices: {sorted(devs)}")
    return devs.pop() if devs else torch.cuda.current_device()


def _stream_ptr(stream, device: int):
    if stream is None:
        import torch
        return torch.cuda.current_stream(device).cuda_stream
    return int(getattr(stream, "cuda_stream", stream))


def launch(kernel: str, strategy: str, n: int, *, points=None, out=None, d: int = 0, rho: int = 16,
           mode: str = "auto", shard: tuple[int, int] | None = None, persistent: bool = False,
           stream=None, sync: bool = True, sentinel: int | None = None, sink=None,
           rec: tuple[int, int] | None = None, engine: str | None = None, per_pass: bool = False) -> dict:
    """tg_launch on device tensors (torch CUDA tensors or raw pointers), on the
    tensors' device and that device's current stream unless `stream` is given.
    kernel in {dummy, write, edm, count}; returns DispatchStats (+ "per_pass"
    when per_pass=True: one entry per grid pass, each device-timed)."""
    dev = _device_of(points, out, sink)
    pp = points.data_ptr() if hasattr(points, "data_ptr") else (points or 0)
    op = out.data_ptr() if hasattr(out, "data_ptr") else (out or 0)
    sp = sink.data_ptr() if hasattr(sink, "data_ptr") else sink
    if points is not None and hasattr(points, "shape") and not d:
        d = points.shape[1]
    npass = len(grid_spec(strategy, n, rho, rec)) if per_pass else 0
    ppa = (_lib.tg_dispatch_stats * npass)() if per_pass else None
    o = _lib.opts(device=dev, mode=mode, stream=_stream_ptr(stream, dev), async_=not sync,
                  persistent=persistent, shard=shard, sentinel=sentinel, sink=sp, rec=rec,
                  engine=None if engine is None else _engine(engine), per_pass=ppa)
    st = _lib.tg_dispatch_stats()
    _lib.check(_L().tg_launch(_lib.KERNELS[kernel], _strategy(strategy, True), n, d, rho, pp, op,
                              C.byref(o), C.byref(st)))
    res = _stats_dict(st)
    if per_pass:
        res["per_pass"] = [x.as_dict() for x in ppa]
    return res


def edm(points, strategy: str = "ltm-r", rho: int = 16, out=None, shard=None, mode: str = "auto",
        persistent: bool = False, stream=None, sync: bool = True):
    """Packed EDM of a CUDA float32 tensor [N, d] (any d >= 1); returns the
    packed tensor (the shard's slice when ``shard=(g, G)``)."""
    import torch
    assert points.is_cuda and points.dtype == torch.float32 and points.dim() == 2
    pts = points.contiguous()
    n, d = pts.shape
    if shard:
        b, e = shard_elems(n, rho, shard[0], shard[1])
        size = e - b
    else:
        size = tri_count(n)
    if out is None:
        out = torch.empty(size, dtype=torch.float32, device=pts.device)
    launch("edm", strategy, n, points=pts, out=out, d=d, rho=rho, mode=mode, shard=shard,
           persistent=persistent, stream=stream, sync=sync)
    return out


def collide(spheres, r_max: float, strategy: str = "ltm-r", rho: int = 16, shard=None,
            mode: str = "auto", persistent: bool = False, stream=None, sync: bool = True):
    """Collision table of CUDA float32 spheres [N, 4] (x, y, z, u; radius u*r_max).
    Returns (bits uint32 tensor, hits uint64 tensor[1]) for the shard."""
    import torch
    assert spheres.is_cuda and spheres.dtype == torch.float32 and spheres.shape[1] == 4
    sph = spheres.contiguous()
    n = sph.shape[0]
    g, G = shard if shard else (0, 1)
    b, e = shard_elems(n, rho, g, G, with_diag=False)
    words = max(1, (e - b + 31) // 32)
    bits = torch.empty(words, dtype=torch.int32, device=sph.device)
    hits = torch.zeros(1, dtype=torch.int64, device=sph.device)
    o = _lib.opts(device=sph.device.index, mode=mode, stream=_stream_ptr(stream, sph.device.index),
                  async_=not sync, persistent=persistent, shard=shard)
    st = _lib.tg_dispatch_stats()
    _lib.check(_L().tg_collide(_strategy(strategy, True), n, rho, sph.data_ptr(), float(r_max),
                               bits.data_ptr(), hits.data_ptr(), C.byref(o), C.byref(st)))
    return bits, hits


def lambda_sweep(engine: str, begin: int, end: int, with_diag: bool = True, fixup: bool = True,
                 device: int = -1):
    """Exhaustive on-device g(lambda) row check vs isqrt(8L+1) (checks.cpp:81-95)."""
    m, f = C.c_uint64(), C.c_uint64()
    _lib.check(_L().tg_lambda_sweep(_engine(engine), int(with_diag), int(fixup), begin, end, device,
                                    C.byref(m), C.byref(f)))
    return m.value, (None if f.value == (1 << 64) - 1 else f.value)


def sqrt_selftest(lo_bits: int, hi_bits: int, device: int = -1) -> int:
    m = C.c_uint64()
    _lib.check(_L().tg_sqrt_selftest(lo_bits, hi_bits, device, C.byref(m)))
    return m.value


def gen_values(count: int, seed: int = 42, device=None):
    """First `count` values of the gen_points stream as a CUDA tensor."""
    import torch
    dev = torch.device("cuda") if device is None else torch.device(device)
    out = torch.empty(count, dtype=torch.float32, device=dev)
    o = _lib.opts(device=out.device.index if out.device.index is not None else -1,
                  stream=torch.cuda.current_stream(out.device).cuda_stream)
    _lib.check(_L().tg_gen_values(count, seed, out.data_ptr(), C.byref(o)))
    return out


__all__ = [
    "__version__", "bb_map", "count_wasted", "coverage_ok", "edm_reference", "edm_strategy",
    "enumerate_lower", "fast_inv_sqrt", "gen_points", "grid_side_balanced", "improvement_model",
    "isqrt", "ltm_map", "rb_map", "rb_rect", "rec_decompose", "rsqrt_single", "sqrt_via",
    "tri_count", "tri_linear_index", "utm_map",
]
