"""Alphabet maps and reduced-tree codes.

The O(n) work of the reference's alphabet module runs on the GPU: fused into
``wt_construct`` for a build, and as stand-alone device ops behind the
reference's own names -- ``minimal_alphabet`` (alphabet.py:94-111),
``AlphabetMap.map_text`` (:76-84) and ``encode_and_histogram`` (:210-242)
call ``wt_minimal_alphabet`` / ``wt_map_text`` / ``wt_encode_histogram``
(csrc/wt_ops.cu).  The O(sigma) surface stays on the host: ``AlphabetMap``
(alphabet.py:51-91), ``CodeTable`` (:123-157) and the small helpers.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import BuildError, SymbolError

MAX_SIGMA = 1 << 16  # alphabet.py:20
# alphabet.py:23: the reference's thread fan-out threshold.  Kept as a module
# attribute for callers that tune it; the device ops do not split by workers.
PARALLEL_MIN_ELEMENTS = 1 << 22


def prev_pow_two(x: int) -> int:
    """Largest power of two strictly below x (1 for x <= 2), alphabet.py:28-32."""
    x = int(x)
    return 1 if x <= 2 else 1 << ((x - 1).bit_length() - 1)


_PREV_POW = None


def prev_pow_two_table() -> np.ndarray:
    """prev_pow_two(w) for every width w in [0, MAX_SIGMA] (alphabet.py:35-43)."""
    global _PREV_POW
    if _PREV_POW is None:
        w = np.arange(MAX_SIGMA + 1, dtype=np.int64)
        t = np.ones(MAX_SIGMA + 1, np.int64)
        _, e = np.frexp((w[3:] - 1).astype(np.float64))  # e = bit_length(w - 1)
        t[3:] = np.int64(1) << (e.astype(np.int64) - 1)
        _PREV_POW = t
    return _PREV_POW


def ceil_log2(sigma: int) -> int:
    """Tree levels for an alphabet of ``sigma`` symbols, alphabet.py:46-48."""
    return int(sigma - 1).bit_length()


class AlphabetMap:
    """Order-preserving bijection between original symbols and [0, sigma)."""

    __slots__ = ("sorted_symbols", "_ids")

    def __init__(self, sorted_symbols: np.ndarray):
        self.sorted_symbols = sorted_symbols
        self._ids = None

    def _table(self):
        if self._ids is None:
            self._ids = {int(s): i for i, s in enumerate(self.sorted_symbols.tolist())}
        return self._ids

    @property
    def size(self) -> int:
        return len(self.sorted_symbols)

    def __contains__(self, symbol) -> bool:
        return int(symbol) in self._table()

    def id_for(self, symbol) -> int:
        try:
            return self._table()[int(symbol)]
        except KeyError:
            raise SymbolError(f"symbol {symbol!r} is not in the alphabet") from None

    def symbol_for(self, sym_id: int) -> int:
        return int(self.sorted_symbols[sym_id])

    def map_text(self, text: np.ndarray) -> np.ndarray:
        """Map original symbols to minimal ids (uint16) on the device,
        rejecting unknown symbols with the first offending position
        (alphabet.py:76-84)."""
        text = np.asarray(text)
        if len(text) == 0:
            return np.zeros(0, np.uint16)
        syms = np.ascontiguousarray(self.sorted_symbols)
        if text.dtype not in (np.uint8, np.uint16):
            if not np.issubdtype(text.dtype, np.integer):
                raise SymbolError(f"cannot map text of dtype {text.dtype}")
            # values outside u16 can never be alphabet symbols
            out_of_range = np.flatnonzero((text < 0) | (text >= MAX_SIGMA))
            first_oor = int(out_of_range[0]) if len(out_of_range) else len(text)
            # an unknown symbol before first_oor raises from the device map first
            ids = self.map_text(text[:first_oor].astype(np.uint16))
            if first_oor < len(text):
                raise SymbolError(f"symbol {int(text[first_oor])} at position {first_oor} "
                                  "is not in the alphabet")
            return ids
        text = np.ascontiguousarray(text)
        sym16 = np.ascontiguousarray(syms.astype(np.int64))
        keep = sym16 < (256 if text.dtype == np.uint8 else MAX_SIGMA)
        ids_of = np.flatnonzero(keep)
        if len(ids_of) and ids_of[-1] != len(ids_of) - 1:  # pragma: no cover (sorted symbols)
            raise SymbolError("alphabet symbols are not sorted")
        table = np.ascontiguousarray(sym16[keep].astype(np.uint16))
        out = np.empty(len(text), np.uint16)
        _lib.check(_lib.lib.wt_map_text(_lib.ptr(text), len(text), text.dtype.itemsize,
                                        _lib.ptr(table), len(table), _lib.current_device(),
                                        _lib.ptr(out)), "wt_map_text")
        return out

    def ids_bulk(self, symbols: np.ndarray):
        """Minimal ids plus a validity mask, without raising (alphabet.py:86-91)."""
        symbols = np.asarray(symbols)
        ids = np.searchsorted(self.sorted_symbols, symbols)
        clipped = np.minimum(ids, self.size - 1)
        ok = self.sorted_symbols[clipped] == symbols
        return clipped.astype(np.int64), ok


@dataclass(frozen=True)
class Code:
    value: int
    length: int


class CodeTable:
    """Per-symbol left-aligned path words (alphabet.py:123-157)."""

    __slots__ = ("sigma", "total_bits", "first_coded", "values", "lens")

    def __init__(self, sigma, total_bits, first_coded, values, lens):
        self.sigma = sigma
        self.total_bits = total_bits
        self.first_coded = first_coded
        self.values = values
        self.lens = lens

    @property
    def is_trivial(self) -> bool:
        return self.first_coded == self.sigma

    @property
    def num_explicit(self) -> int:
        return self.sigma - self.first_coded

    def code(self, sym_id: int) -> Code:
        return Code(int(self.values[sym_id]), int(self.lens[sym_id]))

    def length(self, sym_id: int) -> int:
        return int(self.lens[sym_id])

    def explicit_items(self):
        return [(s, self.code(s)) for s in range(self.first_coded, self.sigma)]


def create_codes(sigma: int) -> CodeTable:
    """Codes of the reduced tree shape (alphabet.py:160-207): the root-to-leaf
    path of every symbol when node [a, b) splits at a + prev_pow_two(b - a),
    left-aligned in a ceil_log2(sigma)-bit field.  (The device build uses the
    same construction in C++, wt_capi.cu plan_codes.)"""
    if sigma < 1:
        raise BuildError(f"alphabet size must be positive, got {sigma}")
    L = ceil_log2(sigma)
    values = np.arange(sigma, dtype=np.uint16)
    lens = np.full(sigma, L, np.uint8)
    if sigma & (sigma - 1) == 0:
        return CodeTable(sigma, L, sigma, values, lens)
    first = prev_pow_two(sigma)
    todo = [(first, sigma, 1, 1)]
    while todo:
        a, b, depth, path = todo.pop()
        w = b - a
        if w & (w - 1) == 0:
            k = w.bit_length() - 1
            values[a:b] = (((path << k) + np.arange(w, dtype=np.int64)) << (L - depth - k))
            lens[a:b] = depth + k
            continue
        p = prev_pow_two(w)
        todo.append((a, a + p, depth + 1, path << 1))
        todo.append((a + p, b, depth + 1, (path << 1) | 1))
    return CodeTable(sigma, L, first, values, lens)


def minimal_alphabet(text: np.ndarray):
    """Remap ``text`` onto its minimal alphabet (alphabet.py:94-111): returns
    (uint16 ids, AlphabetMap).  The histogram and the map run on the device
    (csrc/wt_ops.cu)."""
    text = np.asarray(text)
    if len(text) == 0:
        raise BuildError("text must be non-empty")
    dtype = text.dtype
    if dtype not in (np.uint8, np.uint16):
        if not np.issubdtype(dtype, np.integer) or int(text.min()) < 0 \
                or int(text.max()) >= MAX_SIGMA:
            raise BuildError(f"symbol values must lie in [0, {MAX_SIGMA})")
        text = text.astype(np.uint16)
    text = np.ascontiguousarray(text)
    ids = np.empty(len(text), np.uint16)
    syms = np.empty(256 if text.dtype == np.uint8 else MAX_SIGMA, np.uint16)
    sigma = _lib.C.c_uint32(0)
    _lib.check(_lib.lib.wt_minimal_alphabet(_lib.ptr(text), len(text), text.dtype.itemsize,
                                            _lib.current_device(), _lib.ptr(ids), _lib.ptr(syms),
                                            _lib.C.byref(sigma)), "wt_minimal_alphabet")
    return ids, AlphabetMap(syms[:sigma.value].astype(dtype))


def encode_and_histogram(text_ids: np.ndarray, codes: CodeTable, workers: int = 1):
    """(encoded uint16 path words, int64 histogram of the minimal ids)
    (alphabet.py:210-242), on the device.  ``workers`` is accepted for API
    compatibility; the result does not depend on it."""
    sigma = codes.sigma
    ids = np.asarray(text_ids)
    if ids.dtype != np.uint16:
        if len(ids) and (int(ids.min()) < 0 or int(ids.max()) >= MAX_SIGMA):
            bad = int(np.flatnonzero((ids < 0) | (ids >= sigma))[0])
            raise SymbolError(f"symbol id {int(ids[bad])} outside [0, {sigma})")
        ids = ids.astype(np.uint16)
    ids = np.ascontiguousarray(ids)
    encoded = np.empty(len(ids), np.uint16)
    hist = np.zeros(sigma, np.int64)
    values = np.ascontiguousarray(codes.values, np.uint16)
    _lib.check(_lib.lib.wt_encode_histogram(_lib.ptr(ids), len(ids), _lib.ptr(values), sigma,
                                            _lib.current_device(), _lib.ptr(encoded),
                                            _lib.ptr(hist)), "wt_encode_histogram")
    return encoded, hist


def cumulative_histogram(hist: np.ndarray) -> np.ndarray:
    """Exclusive prefix sum with a trailing total (alphabet.py:245-249)."""
    out = np.zeros(len(hist) + 1, np.int64)
    np.cumsum(hist, out=out[1:])
    return out


def level_sizes(codes: CodeTable, hist: np.ndarray) -> np.ndarray:
    """Bits per tree level (alphabet.py:252-261)."""
    L = ceil_log2(codes.sigma)
    lens = codes.lens.astype(np.int64)
    return np.array([int(np.asarray(hist)[lens > l].sum()) for l in range(L)], np.int64)
