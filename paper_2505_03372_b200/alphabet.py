"""Alphabet maps and reduced-tree codes -- host-side O(sigma) mirror.

The O(n) work of the reference's alphabet module (the bincount / unique of
``minimal_alphabet`` and ``encode_and_histogram``, alphabet.py:94-111,
:210-242) runs on the GPU inside ``wt_construct``.  What lives here is the
O(sigma) surface the reference exposes on a tree: ``AlphabetMap``
(alphabet.py:51-91), ``CodeTable`` (alphabet.py:123-157) and the small helpers.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import BuildError, SymbolError

MAX_SIGMA = 1 << 16  # alphabet.py:20


def prev_pow_two(x: int) -> int:
    """Largest power of two strictly below x (1 for x <= 2), alphabet.py:28-32."""
    x = int(x)
    return 1 if x <= 2 else 1 << ((x - 1).bit_length() - 1)


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
