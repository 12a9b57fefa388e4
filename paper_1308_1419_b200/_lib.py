"""ctypes binding of include/trigrid_b200.h (libtrigrid_b200.so).

The product has exactly one implementation: the sm_100a CUDA library.  If the
shared library is missing this module raises ImportError -- there is no CPU
fallback.  Device entry points raise RuntimeError when no CUDA device exists.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# TG_LIB_PATH: an alternative in-tree build of the same library (A/B tuning only)
LIB_PATH = os.environ.get("TG_LIB_PATH") or os.path.join(HERE, "libtrigrid_b200.so")

TG_OK, TG_EINVAL, TG_ERANGE, TG_ERUNTIME, TG_ECUDA, TG_ENOMEM = range(6)
STRATEGIES = {"bb": 0, "ltm-x": 1, "ltm-n": 2, "ltm-r": 3, "ltm-exact": 4, "utm": 5, "rb": 6, "rec": 7}
STRATEGY_NAMES = {v: k for k, v in STRATEGIES.items()}
KERNELS = {"dummy": 0, "write": 1, "edm": 2, "count": 3}
MODES = {"auto": 0, "grid": 1, "span": 2, "gram": 3}


class tg_dispatch_stats(C.Structure):
    _fields_ = [("blocks_launched", C.c_uint64), ("blocks_discarded", C.c_uint64),
                ("threads_discarded", C.c_uint64), ("wall_time_ns", C.c_uint64)]

    def as_dict(self) -> dict:
        return {k: int(getattr(self, k)) for k, _ in self._fields_}


class tg_launch_opts(C.Structure):
    _fields_ = [("device", C.c_int32), ("mode", C.c_uint32), ("stream", C.c_void_p),
                ("async_", C.c_uint32), ("persistent", C.c_uint32), ("shard_index", C.c_uint32),
                ("shard_count", C.c_uint32), ("sentinel", C.c_uint64), ("sink", C.c_void_p),
                # API version 2
                ("rec_m", C.c_uint64), ("rec_k", C.c_uint32), ("engine", C.c_int32),
                ("per_pass", C.POINTER(tg_dispatch_stats)), ("per_pass_cap", C.c_uint32),
                ("n_devices", C.c_uint32), ("devices", C.POINTER(C.c_int32))]


class tg_pass(C.Structure):
    _fields_ = [("blocks_x", C.c_uint64), ("blocks_y", C.c_uint64), ("has_level", C.c_uint32),
                ("level", C.c_uint32), ("side", C.c_uint64), ("squares", C.c_uint64)]

    def as_dict(self) -> dict:
        d = {"blocks_x": int(self.blocks_x), "blocks_y": int(self.blocks_y)}
        if self.has_level:
            d["level"] = {"level": int(self.level), "side": int(self.side), "squares": int(self.squares)}
        return d


_u64, _u32, _i32 = C.c_uint64, C.c_uint32, C.c_int
_pu64 = C.POINTER(C.c_uint64)
_st = C.c_int  # tg_status
_popts = C.POINTER(tg_launch_opts)
_pstats = C.POINTER(tg_dispatch_stats)

_SIGS = {
    "tg_launch_opts_init": (None, [_popts]),
    "tg_last_error": (C.c_char_p, []),
    "tg_api_version": (C.c_int, []),
    "tg_last_launch_count": (_u64, []),
    "tg_tri_count": (_u64, [_u64, C.c_int]),
    "tg_tri_linear_index": (_st, [_u64, _u64, _pu64]),
    "tg_grid_side_balanced": (_st, [_u64, _pu64]),
    "tg_isqrt": (_u64, [_u64]),
    "tg_fast_inv_sqrt": (C.c_float, [C.c_float, C.c_int]),
    "tg_rsqrt_single": (C.c_float, [C.c_float]),
    "tg_sqrt_via": (_st, [C.c_int, C.c_double, C.POINTER(C.c_double)]),
    "tg_ltm_map": (_st, [_u64, C.c_int, C.c_int, _pu64, _pu64]),
    "tg_bb_map": (C.c_int, [_u64, _u64, _pu64, _pu64]),
    "tg_utm_map": (_st, [_u64, _u64, C.c_int, _pu64, _pu64]),
    "tg_rb_rect": (_st, [_u64, _pu64, _pu64]),
    "tg_rb_map": (C.c_int, [_u64, _u64, _u64, _pu64, _pu64]),
    "tg_rec_decompose": (C.c_int, [_u64, _u32, _pu64, C.POINTER(C.c_uint32)]),
    "tg_count_wasted": (_st, [C.c_int, _u64, _pu64]),
    "tg_ltm_diag_waste_blocks": (C.c_double, [_u64]),
    "tg_improvement_model": (_st, [C.c_double, C.c_double, C.c_double, C.POINTER(C.c_double)]),
    "tg_parse_strategy": (_st, [C.c_char_p, C.POINTER(C.c_int)]),
    "tg_dispatch_stats_for": (_st, [C.c_int, _u64, _u32, _u32, _u32, _pstats]),
    "tg_shard_rows": (_st, [_u64, _u32, _u32, _pu64]),
    "tg_shard_elems": (_st, [_u64, _u32, _u32, _u32, C.c_int, _pu64, _pu64]),
    "tg_launch": (_st, [C.c_int, C.c_int, _u64, _u32, _u32, C.c_void_p, C.c_void_p, _popts, _pstats]),
    "tg_collide": (_st, [C.c_int, _u64, _u32, C.c_void_p, C.c_float, C.c_void_p, C.c_void_p, _popts, _pstats]),
    "tg_edm_strategy_host": (_st, [C.c_int, C.c_void_p, _u64, _u32, _u32, C.c_void_p, _popts, _pstats]),
    "tg_coverage_ok": (_st, [C.c_int, _u64, _u32, C.c_int, C.POINTER(C.c_int)]),
    "tg_lambda_sweep": (_st, [C.c_int, C.c_int, C.c_int, _u64, _u64, C.c_int, _pu64, _pu64]),
    "tg_sqrt_selftest": (_st, [_u32, _u32, C.c_int, _pu64]),
    "tg_gen_values": (_st, [_u64, _u64, C.c_void_p, _popts]),
    "tg_gen_points_host": (_st, [_u64, _u32, _u64, C.c_void_p, C.c_int]),
    # API version 2
    "tg_grid_spec": (_st, [C.c_int, _u64, _u32, _popts, C.POINTER(tg_pass), _u32, C.POINTER(C.c_uint32)]),
    "tg_ltm_map_policy": (_st, [_u64, C.c_int, C.c_int, C.c_int, _pu64, _pu64]),
    "tg_dispatch_stats_opts": (_st, [C.c_int, _u64, _u32, _popts, _pstats]),
    "tg_coverage_ok_opts": (_st, [C.c_int, _u64, _u32, _popts, C.POINTER(C.c_int), _pu64, _pu64]),
    "tg_count_host": (_st, [C.c_int, _u64, _u32, C.c_void_p, _popts, _pstats]),
    "tg_dummy_host": (_st, [C.c_int, _u64, _u32, _popts, _pstats, _pu64]),
    "tg_edm_reference_host": (_st, [C.c_void_p, _u64, _u32, C.c_void_p]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def load():
    """Load libtrigrid_b200.so (raises ImportError when it is not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is not built; run `python -m paper_1308_1419_b200.build` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


class TrigridError(RuntimeError):
    pass


def check(status: int) -> None:
    """Map a tg_status to the exception pybind raises for the reference's C++
    exception class (std::invalid_argument -> ValueError, out_of_range ->
    IndexError, runtime_error -> RuntimeError)."""
    if status == TG_OK:
        return
    msg = load().tg_last_error().decode(errors="replace")
    if status == TG_EINVAL:
        raise ValueError(msg)
    if status == TG_ERANGE:
        raise IndexError(msg)
    if status == TG_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)


def opts(device: int = -1, mode: str = "auto", stream: int | None = None, async_: bool = False,
         persistent: bool = False, shard: tuple[int, int] | None = None, sentinel: int | None = None,
         sink: int | None = None, rec: tuple[int, int] | None = None, engine: int | None = None,
         per_pass=None, devices=None) -> tg_launch_opts:
    """Build a tg_launch_opts.  per_pass: a ctypes array of tg_dispatch_stats;
    devices: a ctypes c_int32 array (kept alive by the caller)."""
    o = tg_launch_opts()
    load().tg_launch_opts_init(C.byref(o))
    if rec is not None:
        o.rec_m, o.rec_k = int(rec[0]), int(rec[1])
    if engine is not None:
        o.engine = int(engine)
    if per_pass is not None:
        o.per_pass = C.cast(per_pass, C.POINTER(tg_dispatch_stats))
        o.per_pass_cap = len(per_pass)
    if devices is not None:
        o.devices = C.cast(devices, C.POINTER(C.c_int32))
        o.n_devices = len(devices)
    o.device = device
    o.mode = MODES[mode]
    o.stream = stream or None
    o.async_ = int(async_)
    o.persistent = int(persistent)
    if shard is not None:
        o.shard_index, o.shard_count = int(shard[0]), int(shard[1])
    if sentinel is not None:
        o.sentinel = sentinel
    o.sink = sink or None
    return o
