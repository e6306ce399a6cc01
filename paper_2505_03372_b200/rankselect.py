"""Rank/select directories (reference rankselect.py) backed by the GPU.

``build_index`` runs the fused directory kernel (csrc/wt_bits.cu) over one
region; every rank/select -- scalar or bulk -- is answered by the device
kernels of csrc/wt_rs.cuh.  The host object mirrors the reference's
``RankSelectIndex`` attributes (l1_counts, l2_counts, samples, ...) lazily.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass
from typing import BinaryIO

import numpy as np

from . import _lib
from ._lib import check, lib, ptr
from .bitvec import WORD_BITS, BitArray
from .errors import CorruptIndexError, OrdinalError, PositionError, TruncatedError

L1_BITS = 65536
DEFAULT_L2_BITS = 512
DEFAULT_SAMPLE_RATE = 16384
TREE_SAMPLE_RATE = 4096
_WORD_MASK = (1 << WORD_BITS) - 1


@dataclass(frozen=True)
class RankSelectParams:
    """Directory parameters (rankselect.py:42-56)."""
    l1_bits: int = L1_BITS
    l2_bits: int = DEFAULT_L2_BITS
    sample_rate: int = DEFAULT_SAMPLE_RATE

    def __post_init__(self):
        if self.l1_bits != L1_BITS:
            raise ValueError(f"l1_bits is fixed at {L1_BITS}")
        if self.l2_bits < WORD_BITS or self.l2_bits % WORD_BITS:
            raise ValueError("l2_bits must be a multiple of the word size")
        if self.l1_bits % self.l2_bits:
            raise ValueError("l2_bits must divide l1_bits")
        if self.sample_rate < 1:
            raise ValueError("sample_rate must be positive")


def select_in_word(word: int, k: int) -> int:
    """0-based position of the k-th set bit of word (rankselect.py:59-80)."""
    w = int(word) & _WORD_MASK
    assert 1 <= k <= w.bit_count(), "select_in_word ordinal out of range"
    for _ in range(k - 1):
        w &= w - 1            # drop the lowest set bit k-1 times
    return (w & -w).bit_length() - 1


class RankSelectIndex:
    """Rank/select over one bit region; queries run on the device.

    ``backend`` is a callable (kind, int64 args) -> int64 results bound to a
    ``wt_bits`` handle or to one level of a device tree; ``fetch(what)``
    returns the directory arrays (lazy D2H).
    """

    def __init__(self, params: RankSelectParams, meta, backend, fetch, words_fn, owner=None):
        self.params = params
        self.n_bits = int(meta.n_bits)
        self.total_ones = int(meta.total_ones)
        self._n_l1, self._n_l2 = int(meta.n_l1), int(meta.n_l2)
        self._n_ones, self._n_zeros = int(meta.n_ones), int(meta.n_zeros)
        self._backend = backend
        self._fetch = fetch
        self._words_fn = words_fn
        self._owner = owner        # keeps the device handle alive
        self._cache = {}

    # -- lazily mirrored arrays --------------------------------------------
    def _arr(self, what):
        if what not in self._cache:
            self._cache[what] = self._fetch(what)
        return self._cache[what]

    @property
    def l1_counts(self) -> np.ndarray:
        return self._arr(_lib.A_L1)

    @property
    def l2_counts(self) -> np.ndarray:
        return self._arr(_lib.A_L2)

    @property
    def one_samples(self) -> np.ndarray:
        return self._arr(_lib.A_ONES)

    @property
    def zero_samples(self) -> np.ndarray:
        return self._arr(_lib.A_ZEROS)

    @property
    def _words(self) -> np.ndarray:
        return self._words_fn()

    @property
    def total_zeros(self) -> int:
        return self.n_bits - self.total_ones

    @property
    def rank_support_bytes(self) -> int:
        return self._n_l1 * 8 + self._n_l2 * 2

    @property
    def select_support_bytes(self) -> int:
        return (self._n_ones + self._n_zeros) * 8

    # -- device queries --------------------------------------------------------
    def _q(self, kind: int, args) -> np.ndarray:
        a = np.ascontiguousarray(np.asarray(args, np.int64).reshape(-1))
        return self._backend(kind, a)

    def get_bit(self, i: int) -> int:
        if not 0 <= i < self.n_bits:
            raise PositionError(f"bit index {i} outside [0, {self.n_bits})")
        return int(self._q(_lib.B_BIT, [i])[0])

    def get_bits_bulk(self, pos) -> np.ndarray:
        return self._q(_lib.B_BIT, pos)

    def rank1(self, i: int) -> int:
        if not 0 <= i <= self.n_bits:
            raise PositionError(f"rank position {i} outside [0, {self.n_bits}]")
        return int(self._q(_lib.B_RANK1, [i])[0])

    def rank0(self, i: int) -> int:
        return i - self.rank1(i)

    def rank0_with_bit(self, i: int):
        if not 0 <= i < self.n_bits:
            raise PositionError(f"position {i} outside [0, {self.n_bits})")
        r = self._q(_lib.B_RANK0, [i])[0]
        return int(r), int(self._q(_lib.B_BIT, [i])[0])

    def rank1_bulk(self, pos) -> np.ndarray:
        pos = np.asarray(pos, np.int64)
        if self.n_bits == 0 or len(pos) == 0:
            return np.zeros(len(pos), np.int64)
        return self._q(_lib.B_RANK1, pos)

    def rank0_bulk(self, pos) -> np.ndarray:
        pos = np.asarray(pos, np.int64)
        return pos - self.rank1_bulk(pos)

    def _select(self, k: int, ones: bool) -> int:
        total = self.total_ones if ones else self.total_zeros
        if not 1 <= k <= total:
            kind = "one" if ones else "zero"
            raise OrdinalError(f"select ordinal {k} outside [1, {total}] ({kind}s)")
        return int(self._q(_lib.B_SELECT1 if ones else _lib.B_SELECT0, [k])[0])

    def select1(self, k: int) -> int:
        return self._select(k, True)

    def select0(self, k: int) -> int:
        return self._select(k, False)

    def select1_bulk(self, ks) -> np.ndarray:
        ks = np.asarray(ks, np.int64)
        return self._q(_lib.B_SELECT1, ks) if len(ks) else np.zeros(0, np.int64)

    def select0_bulk(self, ks) -> np.ndarray:
        ks = np.asarray(ks, np.int64)
        return self._q(_lib.B_SELECT0, ks) if len(ks) else np.zeros(0, np.int64)

    def rebind(self, words: np.ndarray) -> None:
        """Point the index at another copy of its region's words
        (rankselect.py:135-136): the directory arrays are kept and the words
        uploaded to a fresh device index over them."""
        words = np.ascontiguousarray(words, np.uint64)
        handle = _bits_from_arrays(words, self.n_bits, self.params, self.total_ones,
                                   self.l1_counts, self.l2_counts, self.one_samples,
                                   self.zero_samples)
        self._backend = _bits_backend(handle)
        self._words_fn = lambda: words
        self._owner = handle

    # -- serialization (rankselect.py:387-394) ---------------------------------
    @classmethod
    def read(cls, src: BinaryIO, words: np.ndarray) -> "RankSelectIndex":
        """Deserialize one directory written by ``write`` over ``words``
        (rankselect.py:396-411), with the reference's validation
        (``_validate``, :413-430); the arrays are uploaded as stored."""
        l1_bits, l2_bits, rate, n_bits, total_ones = _read_struct(src, "<IIIQQ")
        try:
            params = RankSelectParams(l1_bits, l2_bits, rate)
        except ValueError as e:
            raise CorruptIndexError(str(e)) from e
        l1 = _read_array(src, "<u8").astype(np.int64)
        l2 = _read_array(src, "<u2")
        ones = _read_array(src, "<u8").astype(np.int64)
        zeros = _read_array(src, "<u8").astype(np.int64)
        words = np.ascontiguousarray(words, np.uint64)
        n = n_bits
        if n and len(words) != (n + WORD_BITS - 1) >> 6:
            raise CorruptIndexError("word count does not match region length")
        if len(l1) != -(-n // L1_BITS):
            raise CorruptIndexError("L1 directory length mismatch")
        if len(l2) != -(-n // params.l2_bits):
            raise CorruptIndexError("L2 directory length mismatch")
        if not 0 <= total_ones <= n:
            raise CorruptIndexError("total ones outside [0, n]")
        if len(l1) and (int(l1[0]) != 0 or np.any(np.diff(l1) < 0)):
            raise CorruptIndexError("L1 counts not a non-decreasing prefix sum")
        if len(ones) != total_ones // params.sample_rate:
            raise CorruptIndexError("one-sample count mismatch")
        if len(zeros) != (n - total_ones) // params.sample_rate:
            raise CorruptIndexError("zero-sample count mismatch")
        handle = _bits_from_arrays(words, n, params, total_ones, l1, l2, ones, zeros)
        meta = _lib.LevelMeta()
        check(lib.wt_bits_level_meta(handle.h, _lib.C.byref(meta)), "wt_bits_level_meta")
        idx = cls(params, meta, _bits_backend(handle), _bits_fetch(handle, meta),
                  lambda: words, owner=handle)
        idx._cache.update({_lib.A_L1: l1, _lib.A_L2: l2, _lib.A_ONES: ones, _lib.A_ZEROS: zeros})
        return idx

    def write(self, out: BinaryIO) -> None:
        p = self.params
        out.write(struct.pack("<IIIQQ", p.l1_bits, p.l2_bits, p.sample_rate,
                              self.n_bits, self.total_ones))
        for arr, code in ((self.l1_counts, "<u8"), (self.l2_counts, "<u2"),
                          (self.one_samples, "<u8"), (self.zero_samples, "<u8")):
            out.write(struct.pack("<Q", len(arr)))
            out.write(arr.astype(code, copy=False).tobytes())


class _BitsHandle:
    """Owns one ``wt_bits`` device handle."""

    def __init__(self, h):
        self.h = h

    def __del__(self):
        if self.h:
            lib.wt_bits_destroy(self.h)
            self.h = None


def _bits_fetch(handle: _BitsHandle, meta):
    sizes = {_lib.A_L1: (meta.n_l1, np.int64), _lib.A_L2: (meta.n_l2, np.uint16),
             _lib.A_ONES: (meta.n_ones, np.int64), _lib.A_ZEROS: (meta.n_zeros, np.int64)}

    def fetch(what):
        n, dt = sizes[what]
        out = np.empty(int(n), dt)
        check(lib.wt_bits_get(handle.h, what, ptr(out), out.nbytes), "wt_bits_get")
        return out
    return fetch


def _read_struct(src, fmt: str):
    n = struct.calcsize(fmt)
    data = src.read(n)
    if len(data) != n:
        raise TruncatedError(f"expected {n} bytes, got {len(data)}")
    return struct.unpack(fmt, data)


def _read_array(src, dtype: str):
    (count,) = _read_struct(src, "<Q")
    if count > 1 << 40:
        raise CorruptIndexError(f"array length {count} is implausible")
    nbytes = count * np.dtype(dtype).itemsize
    data = src.read(nbytes)
    if len(data) != nbytes:
        raise TruncatedError(f"expected {nbytes} bytes, got {len(data)}")
    return np.frombuffer(data, dtype=dtype).copy()


def _bits_backend(handle: "_BitsHandle"):
    def backend(kind, args):
        out = np.empty(len(args), np.int64)
        check(lib.wt_bits_query(handle.h, kind, ptr(args), ptr(out), len(args), 0),
              "wt_bits_query")
        return out
    return backend


def _bits_from_arrays(words, n_bits, params, total_ones, l1, l2, ones, zeros) -> "_BitsHandle":
    arrs = [np.ascontiguousarray(a, dt) for a, dt in ((l1, np.int64), (l2, np.uint16),
                                                      (ones, np.int64), (zeros, np.int64))]
    h = _lib.C.c_void_p()
    check(lib.wt_bits_from_arrays(ptr(words) if len(words) else None, n_bits, params.l2_bits,
                                  params.sample_rate, total_ones,
                                  ptr(arrs[0]), len(arrs[0]), ptr(arrs[1]), len(arrs[1]),
                                  ptr(arrs[2]), len(arrs[2]), ptr(arrs[3]), len(arrs[3]),
                                  _lib.current_device(), _lib.C.byref(h)), "wt_bits_from_arrays")
    return _BitsHandle(h)


def build_index(ba: BitArray, region: int, params: RankSelectParams | None = None,
                workers: int = 1) -> RankSelectIndex:
    """Rank/select directory of one region (rankselect.py:442-536), built on
    the GPU.  ``workers`` is accepted for API compatibility (results are
    worker-invariant by contract)."""
    if params is None:
        params = RankSelectParams()
    words = np.ascontiguousarray(ba.region_words(region), dtype=np.uint64)
    n = int(ba.region_nbits[region])
    h = _lib.C.c_void_p()
    check(lib.wt_bits_build(ptr(words) if len(words) else None, n, 0, params.l2_bits,
                            params.sample_rate, _lib.current_device(), _lib.C.byref(h)),
          "wt_bits_build")
    handle = _BitsHandle(h)
    meta = _lib.LevelMeta()
    check(lib.wt_bits_level_meta(h, _lib.C.byref(meta)), "wt_bits_level_meta")

    return RankSelectIndex(params, meta, _bits_backend(handle), _bits_fetch(handle, meta),
                           lambda: words, owner=handle)
