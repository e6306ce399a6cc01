"""Order-preserving batched queries (reference batch.py) on the device.

``BatchRunner.run`` keeps the reference's contract (batch.py:1-13, :152-239):
kind-homogeneous batches, the whole batch rejected with ``BatchError(index,
cause)`` for its first invalid query, results in query order, at most two
chunks staged.  The mapping of original symbols to minimal ids and the range
checks run inside the query kernels (flag WT_F_SYMBOLS); queries stream
through two device chunk buffers on two CUDA streams so the copy of chunk
j+1 overlaps the kernel of chunk j.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import BatchError, OrdinalError, PositionError, SymbolError
from .wtree import WaveletTree

DEFAULT_CHUNK_SIZE = 65536
KINDS = ("access", "rank", "select")
_KIND_ID = {"access": _lib.Q_ACCESS, "rank": _lib.Q_RANK, "select": _lib.Q_SELECT}


@dataclass
class QueryBatch:
    """positions for access, (symbol, position) for rank, (symbol, ordinal)
    for select (batch.py:31-58)."""

    kind: str
    args: np.ndarray
    symbols: np.ndarray | None = None
    chunk_size: int = DEFAULT_CHUNK_SIZE

    def __post_init__(self):
        if self.kind not in KINDS:
            raise ValueError(f"unknown batch kind {self.kind!r}")
        self.args = np.asarray(self.args, np.int64)
        if self.kind == "access":
            if self.symbols is not None:
                raise ValueError("access batches carry no symbols")
        else:
            if self.symbols is None:
                raise ValueError(f"{self.kind} batches need a symbol array")
            self.symbols = np.asarray(self.symbols, np.int64)
            if len(self.symbols) != len(self.args):
                raise ValueError("symbol and argument arrays differ in length")
        if self.chunk_size < 1:
            raise ValueError("chunk_size must be positive")

    def __len__(self) -> int:
        return len(self.args)


def sort_queries_by_symbol(batch: QueryBatch):
    """Stable sort of a rank/select batch by symbol + inverse permutation
    (batch.py:61-75)."""
    if batch.kind == "access":
        raise ValueError("access queries carry no symbol to sort by")
    order = np.argsort(batch.symbols, kind="stable")
    inverse = np.empty(len(order), np.int64)
    inverse[order] = np.arange(len(order), dtype=np.int64)
    return QueryBatch(batch.kind, batch.args[order], batch.symbols[order],
                      batch.chunk_size), inverse


class BatchRunner:
    """Runs batches against one device tree; one in-flight batch per runner."""

    def __init__(self, tree: WaveletTree, chunk_size: int = DEFAULT_CHUNK_SIZE,
                 workers: int = 1, *, sort: bool = False):
        """``sort=True`` (extension): each chunk is sorted on the device into
        buckets of (coarse text position, symbol) before the walk -- the
        device counterpart of `sort_queries_by_symbol` (the paper's query
        sorting); results stay in query order and errors
        report the first bad index of the unsorted batch."""
        if chunk_size < 1:
            raise ValueError("chunk_size must be positive")
        self.tree = tree
        self.sort = bool(sort)
        self.chunk_size = chunk_size
        self.workers = max(1, int(workers))
        self.staging_allocated_records = 0
        self.staging_peak_records = 0
        self.stage_seconds = 0.0     # host->device copies of the chunks (device time)
        self.h2d_bytes = 0           # bytes copied host->device by the last run
        self.narrow_chunks = 0       # its chunks that crossed on the narrow wire
        self.process_seconds = 0.0   # query kernels (device time)
        self.unstage_seconds = 0.0   # kernel end -> results copied back
        self.wall_seconds = 0.0
        self.chunks = 0

    def _cause(self, batch: QueryBatch, i: int) -> Exception:
        """The reference's cause for query i (batch.py:130-148)."""
        tree = self.tree
        arg = int(batch.args[i])
        if batch.kind == "access":
            return PositionError(f"position {arg} outside [0, {tree.n})")
        sym = int(batch.symbols[i])
        if sym not in tree.alphabet:
            return SymbolError(f"symbol {sym} is not in the alphabet")
        if batch.kind == "rank":
            return PositionError(f"position {arg} outside [0, {tree.n}]")
        occ = tree.occurrences(sym)
        return OrdinalError(f"ordinal {arg} outside [1, {occ}]")

    def run(self, batch: QueryBatch) -> np.ndarray:
        nq = len(batch)
        tree = self.tree
        self.h2d_bytes = 0
        self.narrow_chunks = 0
        self.stage_seconds = 0.0
        self.process_seconds = 0.0
        if nq == 0:
            self.staging_peak_records = 0
            if batch.kind == "access":
                return tree.alphabet.sorted_symbols[np.zeros(0, np.int64)]
            return np.zeros(0, np.int64)
        chunk = min(self.chunk_size, nq)
        syms = None if batch.kind == "access" else batch.symbols
        st = _lib.QueryStats()
        t0 = time.perf_counter()
        out, bad = tree.query(_KIND_ID[batch.kind], syms, batch.args, symbols=True,
                              chunk=chunk, sort=self.sort, stats=st)
        self.wall_seconds = time.perf_counter() - t0
        # measured by the C pipeline (CUDA events on its copy-in / kernel /
        # copy-out streams, wt_query_stats): staging = the host->device copies
        # of the chunks, processing = the kernels; the peak is the most
        # queries that were resident in the device slots at once
        self.stage_seconds = st.h2d_ms / 1e3
        self.process_seconds = st.kernel_ms / 1e3
        self.unstage_seconds = st.d2h_ms / 1e3
        self.staging_allocated_records = int(st.slots * st.chunk_records)
        self.staging_peak_records = int(st.peak_records)
        self.chunks = int(st.chunks)
        self.h2d_bytes = int(st.h2d_bytes)          # as copied (narrow wire: 6 / 4 B per query)
        self.narrow_chunks = int(st.narrow_chunks)
        if bad >= 0:
            raise BatchError(bad, self._cause(batch, bad))
        return out


def run_batch(tree: WaveletTree, batch: QueryBatch, workers: int = 1, *,
              sort: bool = False) -> np.ndarray:
    return BatchRunner(tree, batch.chunk_size, workers, sort=sort).run(batch)


def access_batch(tree: WaveletTree, positions, workers: int = 1,
                 chunk_size: int = DEFAULT_CHUNK_SIZE, *, sort: bool = False) -> np.ndarray:
    """Batched access; original symbols in query order (batch.py:251-254)."""
    return run_batch(tree, QueryBatch("access", positions, None, chunk_size), workers, sort=sort)


def rank_batch(tree: WaveletTree, symbols, positions, workers: int = 1,
               chunk_size: int = DEFAULT_CHUNK_SIZE, *, sort: bool = False) -> np.ndarray:
    """Batched rank over (symbol, position) pairs (batch.py:257-260)."""
    return run_batch(tree, QueryBatch("rank", positions, symbols, chunk_size), workers, sort=sort)


def select_batch(tree: WaveletTree, symbols, ordinals, workers: int = 1,
                 chunk_size: int = DEFAULT_CHUNK_SIZE, *, sort: bool = False) -> np.ndarray:
    """Batched select over (symbol, ordinal) pairs (batch.py:263-266)."""
    return run_batch(tree, QueryBatch("select", ordinals, symbols, chunk_size), workers, sort=sort)
