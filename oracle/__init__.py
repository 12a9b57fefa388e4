"""CPU oracle for the triangular-domain hot path -- TEST INFRASTRUCTURE ONLY.

Two checkers live here, both loaded through ctypes:

* ``lib()``  -- this repo's plain-C restatement (``oracle/trigrid_oracle.c``,
  built to ``oracle/_build/liboracle.so``).  Every function cites the
  reference file:line it restates.
* ``ref()``  -- the unmodified reference compiled from its own sources under
  /root/reference (``oracle/_ref/libtrigrid_ref.so``, see ``oracle/Makefile``).
  Present only where the reference was built; tests that need it skip
  otherwise.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (the
``cpu_baseline`` leg and ``--impl reference``) may import this package, and
only as the checker / baseline.  The product (``paper_1308_1419_b200``)
never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libtrigrid_ref.so")
REF_DIR = os.path.join(HERE, "_ref")

ENGINES = {"native": 0, "newton": 1, "reciprocal": 2, "exact": 3}
REPAIR = {"auto": 0, "off": 1, "on": 2}
# the product's tg_strategy order
STRATEGIES = {"bb": 0, "ltm-x": 1, "ltm-n": 2, "ltm-r": 3, "ltm-exact": 4, "utm": 5, "rb": 6, "rec": 7}

_u64 = C.c_uint64
_u32 = C.c_uint32
_pu64 = C.POINTER(C.c_uint64)
_pf = C.POINTER(C.c_float)

_lib = None
_ref = None


def build(quiet: bool = True) -> None:
    """Compile the C restatement (and the reference when its sources exist)."""
    targets = ["oracle"]
    if os.path.isdir("/root/reference/proj"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


def _ptr(a: np.ndarray, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        L.or_tri_count.restype = _u64
        L.or_tri_count.argtypes = [_u64, C.c_int]
        L.or_isqrt.restype = _u64
        L.or_isqrt.argtypes = [_u64]
        L.or_ceil_sqrt.restype = _u64
        L.or_ceil_sqrt.argtypes = [_u64]
        L.or_grid_side_balanced.restype = _u64
        L.or_grid_side_balanced.argtypes = [_u64]
        L.or_fast_inv_sqrt.restype = C.c_float
        L.or_fast_inv_sqrt.argtypes = [C.c_float, C.c_int]
        L.or_rsqrt_single.restype = C.c_float
        L.or_rsqrt_single.argtypes = [C.c_float]
        L.or_sqrt_via.restype = C.c_double
        L.or_sqrt_via.argtypes = [C.c_int, C.c_double, C.POINTER(C.c_int)]
        L.or_repair_lower_row.restype = _u64
        L.or_repair_lower_row.argtypes = [_u64, _u64, C.c_int]
        L.or_ltm_map.restype = None
        L.or_ltm_map.argtypes = [_u64, C.c_int, C.c_int, C.c_int, _pu64, _pu64]
        L.or_ltm_map_range.restype = None
        L.or_ltm_map_range.argtypes = [_u64, _u64, C.c_int, C.c_int, C.c_int, _pu64, _pu64]
        L.or_ltm_exactness_sweep.restype = None
        L.or_ltm_exactness_sweep.argtypes = [_u64, C.c_int, C.c_int, _pu64, _pu64, _pu64]
        L.or_utm_pair.restype = None
        L.or_utm_pair.argtypes = [_u64, _u64, C.c_int, _pu64, _pu64]
        L.or_rb_rect.restype = C.c_int
        L.or_rb_rect.argtypes = [_u64, _pu64, _pu64]
        L.or_rb_map.restype = C.c_int
        L.or_rb_map.argtypes = [_u64, _u64, _u64, _pu64, _pu64]
        L.or_rec_decompose.restype = C.c_int
        L.or_rec_decompose.argtypes = [_u64, _u32, _pu64, C.POINTER(C.c_uint32)]
        L.or_gen_points.restype = None
        L.or_gen_points.argtypes = [_u64, _u32, _u64, _pf]
        L.or_edm_pair.restype = C.c_float
        L.or_edm_pair.argtypes = [_pf, _pf, _u32]
        L.or_edm_reference.restype = None
        L.or_edm_reference.argtypes = [_pf, _u64, _u32, _pf]
        L.or_edm_rows.restype = None
        L.or_edm_rows.argtypes = [_pf, _u64, _u32, _u64, _u64, _pf]
        L.or_edm_cells.restype = None
        L.or_edm_cells.argtypes = [_pf, _u32, _pu64, _pu64, _u64, _pf]
        L.or_collide_reference.restype = _u64
        L.or_collide_reference.argtypes = [_pf, _u64, C.c_float, C.POINTER(C.c_uint8)]
        L.or_collide_rows_u8.restype = _u64
        L.or_collide_rows_u8.argtypes = [_pf, C.c_float, _u64, _u64, C.POINTER(C.c_uint8)]
        L.or_run_strategy.restype = C.c_int
        L.or_run_strategy.argtypes = [C.c_int, _u64, _u32, C.c_int, C.POINTER(C.c_uint32), _pu64]
        L.or_count_wasted.restype = _u64
        L.or_count_wasted.argtypes = [C.c_int, _u64]
        L.or_improvement_model.restype = C.c_double
        L.or_improvement_model.argtypes = [C.c_double, C.c_double, C.c_double]
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_PATH)


def ref():
    """The reference library (oracle/_ref); raises if it was not built."""
    global _ref
    if _ref is None:
        if not ref_available():
            raise FileNotFoundError(f"{REF_PATH} not built (needs /root/reference)")
        R = C.CDLL(REF_PATH)
        R.ref_last_error.restype = C.c_char_p
        R.ref_ltm_map_range.restype = None
        R.ref_ltm_map_range.argtypes = [_u64, _u64, C.c_int, C.c_int, C.c_int, _pu64, _pu64]
        R.ref_utm_map_range.restype = C.c_int
        R.ref_utm_map_range.argtypes = [_u64, _u64, _u64, C.c_int, _pu64, _pu64]
        R.ref_rb_map.restype = C.c_int
        R.ref_rb_map.argtypes = [_u64, _u64, _u64, _pu64, _pu64]
        R.ref_rec_decompose.restype = C.c_int
        R.ref_rec_decompose.argtypes = [_u64, _u32, _pu64, C.POINTER(C.c_uint32)]
        R.ref_grid_side_balanced.restype = _u64
        R.ref_grid_side_balanced.argtypes = [_u64]
        R.ref_isqrt.restype = _u64
        R.ref_isqrt.argtypes = [_u64]
        R.ref_fast_inv_sqrt.restype = C.c_float
        R.ref_fast_inv_sqrt.argtypes = [C.c_float, C.c_int]
        R.ref_rsqrt_single.restype = C.c_float
        R.ref_rsqrt_single.argtypes = [C.c_float]
        R.ref_sqrt_via.restype = C.c_int
        R.ref_sqrt_via.argtypes = [C.c_int, C.c_double, C.POINTER(C.c_double)]
        R.ref_count_wasted.restype = C.c_int
        R.ref_count_wasted.argtypes = [C.c_char_p, _u64, _pu64]
        R.ref_gen_points.restype = None
        R.ref_gen_points.argtypes = [_u64, _u32, _u64, _pf]
        R.ref_edm_reference.restype = None
        R.ref_edm_reference.argtypes = [_pf, _u64, _u32, _pf]
        R.ref_ltm_exactness_sweep.restype = None
        R.ref_ltm_exactness_sweep.argtypes = [_u64, C.c_int, C.c_int, _pu64]
        R.ref_launch_count.restype = C.c_int
        R.ref_launch_count.argtypes = [C.c_char_p, _u64, _u32, C.c_uint, C.POINTER(C.c_uint32), _pu64]
        R.ref_launch_dummy.restype = C.c_int
        R.ref_launch_dummy.argtypes = [C.c_char_p, _u64, _u32, C.c_uint, _pu64]
        R.ref_verify_strategies.restype = C.c_int
        R.ref_verify_strategies.argtypes = [C.c_char_p, _u64, _u32]
        R.ref_edm_session_create.restype = C.c_void_p
        R.ref_edm_session_create.argtypes = [C.c_char_p, _pf, _u64, _u32, _u32]
        R.ref_edm_session_run.restype = C.c_int
        R.ref_edm_session_run.argtypes = [C.c_void_p, C.c_uint, _pu64]
        R.ref_edm_session_data.restype = C.c_void_p
        R.ref_edm_session_data.argtypes = [C.c_void_p]
        R.ref_edm_session_destroy.restype = None
        R.ref_edm_session_destroy.argtypes = [C.c_void_p]
        R.ref_hardware_concurrency.restype = C.c_uint
        _ref = R
    return _ref


# ---------------------------------------------------------------- numpy API

def tri_count(n: int, with_diag: bool = True) -> int:
    return int(lib().or_tri_count(n, int(with_diag)))


def gen_points(n: int, d: int, seed: int = 42) -> np.ndarray:
    """edm.cpp:38-51 (no d cap; d=64 equals gen_points(16N,4).reshape(N,64))."""
    out = np.empty((n, d), dtype=np.float32)
    lib().or_gen_points(n, d, seed, _ptr(out, C.c_float))
    return out


def edm_reference(pts: np.ndarray) -> np.ndarray:
    pts = np.ascontiguousarray(pts, dtype=np.float32)
    n, d = pts.shape
    out = np.empty(tri_count(n), dtype=np.float32)
    lib().or_edm_reference(_ptr(pts, C.c_float), n, d, _ptr(out, C.c_float))
    return out


def edm_rows(pts: np.ndarray, r0: int, r1: int) -> np.ndarray:
    """Packed rows [r0, r1): elements [T(r0), T(r1))."""
    pts = np.ascontiguousarray(pts, dtype=np.float32)
    n, d = pts.shape
    out = np.empty(tri_count(r1) - tri_count(r0), dtype=np.float32)
    lib().or_edm_rows(_ptr(pts, C.c_float), n, d, r0, r1, _ptr(out, C.c_float))
    return out


def edm_cells(pts: np.ndarray, ci: np.ndarray, cj: np.ndarray) -> np.ndarray:
    pts = np.ascontiguousarray(pts, dtype=np.float32)
    ci = np.ascontiguousarray(ci, dtype=np.uint64)
    cj = np.ascontiguousarray(cj, dtype=np.uint64)
    out = np.empty(ci.size, dtype=np.float32)
    lib().or_edm_cells(_ptr(pts, C.c_float), pts.shape[1], _ptr(ci, C.c_uint64),
                       _ptr(cj, C.c_uint64), ci.size, _ptr(out, C.c_float))
    return out


def ltm_map_range(lam0: int, count: int, engine: str = "reciprocal", with_diag: bool = True,
                  repair: str = "auto"):
    oi = np.empty(count, dtype=np.uint64)
    oj = np.empty(count, dtype=np.uint64)
    lib().or_ltm_map_range(lam0, count, ENGINES[engine], int(with_diag), REPAIR[repair],
                           _ptr(oi, C.c_uint64), _ptr(oj, C.c_uint64))
    return oi, oj


def ltm_map(lam: int, engine: str = "reciprocal", with_diag: bool = True, repair: str = "auto"):
    i, j = ltm_map_range(lam, 1, engine, with_diag, repair)
    return int(i[0]), int(j[0])


def utm_map(k: int, n: int, engine: str = "newton"):
    a, b = _u64(), _u64()
    lib().or_utm_pair(k, n, ENGINES[engine], C.byref(a), C.byref(b))
    return a.value, b.value


def rb_map(tx: int, ty: int, n: int):
    i, j = _u64(), _u64()
    if not lib().or_rb_map(tx, ty, n, C.byref(i), C.byref(j)):
        return None
    return i.value, j.value


def rec_decompose(n: int, rho: int = 16):
    m, k = _u64(), C.c_uint32()
    if not lib().or_rec_decompose(n, rho, C.byref(m), C.byref(k)):
        return None
    return m.value, k.value


def run_strategy(strategy: str, n: int, rho: int = 16, mode: str = "count"):
    """Serial restatement of run_strategy/process_block.  Returns (buf, stats)
    with buf the u32 count (mode 'count') or i+j write table (mode 'write'),
    or None for mode 'none'.  stats = (launched, discarded, threads_discarded)."""
    m = {"count": 0, "write": 1, "none": 2}[mode]
    buf = np.zeros(tri_count(n), dtype=np.uint32) if m < 2 else np.zeros(1, dtype=np.uint32)
    st = np.zeros(4, dtype=np.uint64)
    ok = lib().or_run_strategy(STRATEGIES[strategy], n, rho, m, _ptr(buf, C.c_uint32),
                               _ptr(st, C.c_uint64))
    if not ok:
        raise ValueError(f"strategy {strategy} cannot be built for N={n}, rho={rho}")
    return (buf if m < 2 else None), tuple(int(x) for x in st[:3])


def write_reference(n: int) -> np.ndarray:
    """out[T(i)+j] = i+j in enumerate_lower order (tri.hpp:53-105)."""
    i = np.repeat(np.arange(n, dtype=np.uint64), np.arange(1, n + 1))
    starts = np.repeat((np.arange(n, dtype=np.uint64) * (np.arange(n, dtype=np.uint64) + 1)) // 2,
                       np.arange(1, n + 1))
    j = np.arange(i.size, dtype=np.uint64) - starts
    return (i + j).astype(np.uint32)


def collide_reference(sph: np.ndarray, r_max: float):
    """Packed no-diagonal collision bit table + hit count (semantics in
    trigrid_oracle.c; parity unpinned w.r.t. the reference)."""
    sph = np.ascontiguousarray(sph, dtype=np.float32)
    n = sph.shape[0]
    nbytes = (tri_count(n, False) + 7) // 8
    bits = np.zeros(max(nbytes, 1), dtype=np.uint8)
    hits = lib().or_collide_reference(_ptr(sph, C.c_float), n, r_max, _ptr(bits, C.c_uint8))
    return bits[:nbytes], int(hits)


def collide_rows_u8(sph: np.ndarray, r_max: float, r0: int, r1: int):
    sph = np.ascontiguousarray(sph, dtype=np.float32)
    out = np.zeros(tri_count(r1, False) - tri_count(r0, False), dtype=np.uint8)
    hits = lib().or_collide_rows_u8(_ptr(sph, C.c_float), r_max, r0, r1, _ptr(out, C.c_uint8))
    return out, int(hits)
