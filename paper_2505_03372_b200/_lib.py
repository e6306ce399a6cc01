"""ctypes binding of libwt_b200.so (the C-ABI declared in include/wt_b200.h).

There is no CPU fallback: if the shared library is missing or cannot be
loaded, importing the package raises.  Build it with
``python -c "import __graft_entry__ as g; g.build()"`` (or ``make`` in
``paper_2505_03372_b200/csrc``).
"""

from __future__ import annotations

import ctypes as C
import os
import threading
import weakref

import numpy as np

from .errors import BuildError, DeviceError, SymbolError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("WT_B200_LIB", os.path.join(_HERE, "libwt_b200.so"))

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"libwt_b200.so not found at {LIB_PATH}: the CUDA library is required "
        "(no CPU fallback). Build it with `make -C paper_2505_03372_b200/csrc`.")

lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)

WT_OK, WT_ERR_CUDA, WT_ERR_ARG, WT_ERR_OOM, WT_ERR_SYMBOL, WT_ERR_NCCL, WT_ERR_BUILD = range(7)
Q_ACCESS, Q_RANK, Q_SELECT = 0, 1, 2
B_RANK1, B_RANK0, B_SELECT1, B_SELECT0, B_BIT = range(5)
F_DEVICE_PTRS, F_SYMBOLS, F_ACCESS_IDS, F_SORT, F_PHASES = 1, 2, 4, 8, 16
(A_SYMBOLS, A_CODE_VALUES, A_CODE_LENS, A_CUM_HIST, A_LEVEL_SIZES, A_REGION_OFFS, A_WORDS,
 A_L1, A_L2, A_ONES, A_ZEROS, A_NODE_STARTS, A_NODE_RANK0, A_QLINES, A_QSEL1, A_QSEL0) = range(16)


class Meta(C.Structure):
    _fields_ = [("n", C.c_uint64), ("sigma", C.c_uint32), ("levels", C.c_uint32),
                ("symbol_width", C.c_uint32), ("l2_bits", C.c_uint32),
                ("sample_rate", C.c_uint64), ("first_coded", C.c_uint32),
                ("device", C.c_uint32), ("n_words", C.c_uint64), ("device_bytes", C.c_uint64)]


class LevelMeta(C.Structure):
    _fields_ = [(k, C.c_uint64) for k in
                ("n_bits", "total_ones", "n_l1", "n_l2", "n_ones", "n_zeros", "n_nodes")]


class QueryStats(C.Structure):
    """wt_query_stats (include/wt_b200.h): the host pipeline's accounting."""
    _fields_ = [("chunks", C.c_uint64), ("slots", C.c_uint64), ("chunk_records", C.c_uint64),
                ("peak_records", C.c_uint64), ("h2d_ms", C.c_float), ("kernel_ms", C.c_float),
                ("d2h_ms", C.c_float), ("total_ms", C.c_float), ("h2d_bytes", C.c_uint64),
                ("narrow_chunks", C.c_uint64)]


_vp, _u64, _u32, _i32, _f32p = C.c_void_p, C.c_uint64, C.c_uint32, C.c_int, C.POINTER(C.c_float)

_SIGS = {
    "wt_last_error": ([], C.c_char_p),
    "wt_last_error_index": ([], C.c_int64),
    "wt_abi_version": ([], C.c_int),
    "wt_device_count": ([C.POINTER(C.c_int)], C.c_int),
    "wt_construct": ([_vp, _u64, _i32, _i32, _vp, _u32, _i32, _u32, _u64, _i32, _vp,
                      C.POINTER(_vp), _f32p], C.c_int),
    "wt_tree_from_arrays": ([C.POINTER(Meta), _vp, _vp, _vp, C.POINTER(LevelMeta), _vp, _vp,
                             _vp, _vp, _i32, C.POINTER(_vp)], C.c_int),
    "wt_tree_meta": ([_vp, C.POINTER(Meta)], C.c_int),
    "wt_tree_level_meta": ([_vp, _u32, C.POINTER(LevelMeta)], C.c_int),
    "wt_tree_get": ([_vp, _i32, _u32, _vp, _u64], C.c_int),
    "wt_tree_build_profile": ([_vp, _f32p, _u32], C.c_int),
    "wt_tree_destroy": ([_vp], C.c_int),
    "wt_tree_query": ([_vp, _i32, _vp, _vp, _vp, _u64, _u64, _i32, _vp, C.POINTER(C.c_int64), _f32p], C.c_int),
    "wt_tree_query_ex": ([_vp, _i32, _vp, _vp, _vp, _u64, _u64, _i32, _vp, C.POINTER(C.c_int64),
                          _f32p, C.POINTER(QueryStats)], C.c_int),
    "wt_tree_level_query": ([_vp, _u32, _i32, _vp, _vp, _u64], C.c_int),
    "wt_host_alloc": ([_u64, C.POINTER(_vp)], C.c_int),
    "wt_host_free": ([_vp], C.c_int),
    "wt_host_register": ([_vp, _u64], C.c_int),
    "wt_host_unregister": ([_vp], C.c_int),
    "wt_nccl_unique_id": ([_vp], C.c_int),
    "wt_tree_replicate": ([_vp, _vp, _i32, _i32, _i32, C.POINTER(_vp), _f32p], C.c_int),
    "wt_bits_build": ([_vp, _u64, _i32, _u32, _u64, _i32, C.POINTER(_vp)], C.c_int),
    "wt_bits_level_meta": ([_vp, C.POINTER(LevelMeta)], C.c_int),
    "wt_bits_get": ([_vp, _i32, _vp, _u64], C.c_int),
    "wt_bits_query": ([_vp, _i32, _vp, _vp, _u64, _i32], C.c_int),
    "wt_bits_destroy": ([_vp], C.c_int),
    "wt_bits_from_arrays": ([_vp, _u64, _u32, _u64, _u64, _vp, _u64, _vp, _u64, _vp, _u64, _vp,
                             _u64, _i32, C.POINTER(_vp)], C.c_int),
    "wt_minimal_alphabet": ([_vp, _u64, _i32, _i32, _vp, _vp, C.POINTER(_u32)], C.c_int),
    "wt_map_text": ([_vp, _u64, _i32, _vp, _u32, _i32, _vp], C.c_int),
    "wt_encode_histogram": ([_vp, _u64, _vp, _u32, _i32, _vp, _vp], C.c_int),
    "wt_sort_by_prefix": ([_vp, _u64, _u32, _i32, _vp], C.c_int),
    "wt_fill_level": ([_vp, _u64, _u32, _i32, _vp], C.c_int),
}
EXPORTS = tuple(_SIGS)

for _name, (_args, _res) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.argtypes = _args
    _f.restype = _res


def check(rc: int, what: str = "") -> None:
    """Map a nonzero status to the reference's exception classes."""
    if rc == WT_OK:
        return
    msg = lib.wt_last_error().decode(errors="replace")
    if rc == WT_ERR_SYMBOL:
        raise SymbolError(msg)
    if rc == WT_ERR_BUILD:
        raise BuildError(msg)
    if rc == WT_ERR_OOM:
        raise MemoryError(f"{what}: {msg}")
    raise DeviceError(f"{what}: {msg} (status {rc})")


def ptr(a: np.ndarray | None):
    """c_void_p to a's data that keeps `a` alive (ctypes ``_objects``): a
    temporary array passed as ``ptr(np.concatenate(...))`` must outlive the
    call it is an argument of."""
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def current_device() -> int:
    return int(os.environ.get("WT_DEVICE", "0"))


# ---------------------------------------------------------------------------
# pinned result arrays: device -> host copies into page-locked memory are
# asynchronous (the query pipeline overlaps them with the next chunk's
# kernel).  Blocks come in power-of-two size classes and return to a free
# list when the last numpy view of them is dropped; the free lists hold at
# most PINNED_CACHE_BYTES (the excess is released with wt_host_free), so a
# process answering batches of many sizes does not accumulate page-locked
# memory.
# ---------------------------------------------------------------------------
PINNED_MIN_BYTES = 1 << 20
PINNED_CACHE_BYTES = int(os.environ.get("WT_PINNED_CACHE_BYTES", 8 << 30))
_pin_lock = threading.Lock()
_pin_free: dict[int, list[int]] = {}
_pin_cached = 0   # bytes on the free lists


def _pin_class(nbytes: int) -> int:
    return 1 << (int(nbytes) - 1).bit_length()


def _pin_release(cls: int, addr: int) -> None:
    global _pin_cached
    with _pin_lock:
        if _pin_cached + cls <= PINNED_CACHE_BYTES:
            _pin_free.setdefault(cls, []).append(addr)
            _pin_cached += cls
            return
    lib.wt_host_free(C.c_void_p(addr))


def pinned_cached_bytes() -> int:
    return _pin_cached


def pinned_empty(count: int, dtype) -> np.ndarray:
    """An uninitialised array in pinned host memory (plain np.empty below
    PINNED_MIN_BYTES, or when page-locked memory cannot be had)."""
    global _pin_cached
    dtype = np.dtype(dtype)
    nbytes = int(count) * dtype.itemsize
    if nbytes < PINNED_MIN_BYTES:
        return np.empty(count, dtype)
    cls = _pin_class(nbytes)
    with _pin_lock:
        free = _pin_free.get(cls)
        addr = free.pop() if free else None
        if addr is not None:
            _pin_cached -= cls
    if addr is None:
        p = C.c_void_p()
        if lib.wt_host_alloc(cls, C.byref(p)) != WT_OK or not p.value:
            return np.empty(count, dtype)
        addr = p.value
    holder = (C.c_uint8 * cls).from_address(addr)
    weakref.finalize(holder, _pin_release, cls, addr)
    return np.frombuffer(holder, dtype, count)
