"""Device-resident wavelet tree with the reference's ``WaveletTree`` surface.

``construct`` / ``construct_with_alphabet`` (reference wtree.py:438-466) hand
the coerced text to ``wt_construct`` (csrc/wt_capi.cu): histogram kernel,
O(sigma) plan, one fused K2 launch per level.  All queries -- scalar and
bulk -- run on the device (csrc/wt_query.cu, csrc/wt_rs.cuh).  The host keeps
the O(sigma) tables and materialises the big arrays (``bits.words``,
``rs[l].l1_counts`` ...) lazily, on first access, from device memory.
"""

from __future__ import annotations

import io
import struct
from pathlib import Path
from typing import BinaryIO

import numpy as np

from . import _lib
from ._lib import C, check, lib, ptr
from .alphabet import MAX_SIGMA, AlphabetMap, CodeTable, ceil_log2, create_codes
from .bitvec import BitArray, region_layout
from .errors import (BadMagicError, BadVersionError, BuildError, CorruptIndexError,
                     OrdinalError, PositionError, SymbolError, TruncatedError)
from .rankselect import RankSelectIndex, RankSelectParams, TREE_SAMPLE_RATE

MAGIC = b"WTIDX001"
VERSION = 1
_FLAG_WIDE_SYMBOLS = 1


# ---------------------------------------------------------------------------
# input coercion (wtree.py:59-89)
# ---------------------------------------------------------------------------
def _coerce_text(text) -> tuple[np.ndarray, int]:
    if isinstance(text, (bytes, bytearray, memoryview)):
        return np.frombuffer(bytes(text), dtype=np.uint8), 1
    arr = np.asarray(text)
    if arr.dtype == np.uint8:
        return arr, 1
    if arr.dtype == np.uint16:
        return arr, 2
    if arr.size == 0:
        return arr.astype(np.uint8), 1
    if not np.issubdtype(arr.dtype, np.integer):
        raise BuildError(f"unsupported text dtype {arr.dtype}")
    lo, hi = int(arr.min()), int(arr.max())
    if lo < 0 or hi >= MAX_SIGMA:
        raise BuildError(f"symbol values must lie in [0, {MAX_SIGMA})")
    if hi < 256:
        return arr.astype(np.uint8), 1
    return arr.astype(np.uint16), 2


def _symbol_value(c) -> int:
    if isinstance(c, str):
        if len(c) != 1:
            raise SymbolError(f"symbol string must be one character, got {c!r}")
        return ord(c)
    if isinstance(c, (bytes, bytearray)):
        if len(c) != 1:
            raise SymbolError(f"symbol bytes must be one byte, got {c!r}")
        return c[0]
    return int(c)


def _device_text(text):
    """(data_ptr, n, sym_bytes) for a CUDA torch tensor of uint8/uint16, else None."""
    if not hasattr(text, "data_ptr") or not getattr(text, "is_cuda", False):
        return None
    import torch
    if text.dtype == torch.uint8:
        sb = 1
    elif text.dtype in (torch.uint16, torch.int16):
        sb = 2
    else:
        raise BuildError(f"unsupported device text dtype {text.dtype}")
    if not text.is_contiguous():
        raise BuildError("device text must be contiguous")
    # the build runs on its own (non-blocking) stream: kernels still producing
    # the text on the caller's stream must finish first
    torch.cuda.current_stream(text.device).synchronize()
    return text.data_ptr(), int(text.numel()), sb


class _TreeHandle:
    """Owns one ``wt_tree`` device handle.  Closures of the lazy host
    mirrors capture this object, never the WaveletTree, so dropping the tree
    frees device memory immediately (no reference cycle waiting for the GC)."""

    def __init__(self, h):
        self.h = h

    def get(self, what: int, level: int, count: int, dtype) -> np.ndarray:
        out = np.empty(int(count), dtype)
        check(lib.wt_tree_get(self.h, what, level, ptr(out), out.nbytes), "wt_tree_get")
        return out

    def __del__(self):
        if self.h:
            lib.wt_tree_destroy(self.h)
            self.h = None


# ---------------------------------------------------------------------------
# the per-level building blocks of _build (wtree.py:92-107), as device ops;
# wt_construct fuses both into one kernel per level
# ---------------------------------------------------------------------------
def stable_sort_by_prefix(encoded: np.ndarray, l: int, num_levels: int) -> np.ndarray:
    """Stably sort code words by their top ``l`` bits, i.e. by
    ``encoded >> (num_levels - l)`` (wtree.py:92-100), on the device
    (``wt_sort_by_prefix``: one stable popcount split per key bit)."""
    enc = np.asarray(encoded)
    dtype = enc.dtype
    shift = int(num_levels) - int(l)
    if len(enc) == 0:
        return enc.copy()
    if dtype != np.uint16:
        if not np.issubdtype(dtype, np.integer) or int(enc.min()) < 0 \
                or int(enc.max()) >= MAX_SIGMA:
            raise BuildError("code words must lie in [0, 65536)")
    if shift >= 16:
        return enc.copy()
    if shift < 0:
        raise BuildError(f"prefix length {l} exceeds {num_levels} levels")
    codes = np.ascontiguousarray(enc, np.uint16)
    out = np.empty(len(codes), np.uint16)
    check(lib.wt_sort_by_prefix(ptr(codes), len(codes), shift, _lib.current_device(), ptr(out)),
          "wt_sort_by_prefix")
    return out if dtype == np.uint16 else out.astype(dtype)


def fill_level(ba: BitArray, l: int, encoded: np.ndarray, count: int,
               num_levels: int, workers: int = 1) -> None:
    """Write region ``l``: bit j = bit ``num_levels-1-l`` of code word j
    (wtree.py:103-107, packed as BitArray.fill_region does, bitvec.py:119-151),
    packed on the device (``wt_fill_level``)."""
    n = int(ba.region_nbits[l])
    count = int(count)
    if count != n:
        raise BuildError(f"region {l} holds {n} bits, got {count}")
    if n == 0:
        return
    enc = np.asarray(encoded)[:count]
    if enc.dtype != np.uint16:
        if int(enc.min()) < 0 or int(enc.max()) >= MAX_SIGMA:
            raise BuildError("code words must lie in [0, 65536)")
    codes = np.ascontiguousarray(enc, np.uint16)
    words = np.empty((n + 63) // 64, np.uint64)
    check(lib.wt_fill_level(ptr(codes), n, num_levels - 1 - l, _lib.current_device(),
                            ptr(words)), "wt_fill_level")
    w0 = ba.region_word_offset(l)
    ba.words[w0:w0 + len(words)] = words


# ---------------------------------------------------------------------------
# the tree
# ---------------------------------------------------------------------------
class WaveletTree:
    """Immutable wavelet tree over a byte or 16-bit symbol text, held in HBM.

    Attributes mirror the reference (wtree.py:113-133): n, symbol_width,
    alphabet, codes, cum_hist, level_sizes, bits, rs, node_starts, node_rank0,
    sigma, num_levels.  Safe for concurrent reads.
    """

    def __init__(self, handle: _TreeHandle, symbol_width: int, sym_dtype, build_ms: float = 0.0):
        self._h = handle
        h = handle.h
        meta = _lib.Meta()
        check(lib.wt_tree_meta(h, C.byref(meta)), "wt_tree_meta")
        self._meta = meta
        self.build_ms = build_ms
        self.n = int(meta.n)
        self.symbol_width = symbol_width
        self.sigma = int(meta.sigma)
        self.num_levels = int(meta.levels)
        self.params = RankSelectParams(l2_bits=int(meta.l2_bits),
                                       sample_rate=int(meta.sample_rate))
        L = self.num_levels
        syms = self._get(_lib.A_SYMBOLS, 0, self.sigma, np.uint16)
        self.alphabet = AlphabetMap(syms.astype(sym_dtype))
        values = self._get(_lib.A_CODE_VALUES, 0, self.sigma, np.uint16)
        lens = self._get(_lib.A_CODE_LENS, 0, self.sigma, np.uint8)
        self.codes = CodeTable(self.sigma, L, int(meta.first_coded), values, lens)
        self.cum_hist = self._get(_lib.A_CUM_HIST, 0, self.sigma + 1, np.int64)
        self.level_sizes = self._get(_lib.A_LEVEL_SIZES, 0, L, np.int64)
        offsets = self._get(_lib.A_REGION_OFFS, 0, L, np.int64)
        n_words = int(meta.n_words)
        hd = self._h
        self.bits = BitArray(None, offsets, self.level_sizes.copy(),
                             fetch=lambda: hd.get(_lib.A_WORDS, 0, n_words, np.uint64))
        self._lmeta = []
        self.rs = []
        self.node_starts, self.node_rank0 = [], []
        for l in range(L):
            lm = _lib.LevelMeta()
            check(lib.wt_tree_level_meta(h, l, C.byref(lm)), "wt_tree_level_meta")
            self._lmeta.append(lm)
            self.rs.append(self._make_rs(l, lm))
            self.node_starts.append(self._get(_lib.A_NODE_STARTS, l, lm.n_nodes, np.int64))
            self.node_rank0.append(self._get(_lib.A_NODE_RANK0, l, lm.n_nodes, np.int64))
        self._spine_starts = self._compute_spine_starts()

    # -- device plumbing ---------------------------------------------------
    @property
    def handle(self):
        return self._h.h

    def _get(self, what: int, level: int, count: int, dtype) -> np.ndarray:
        return self._h.get(what, level, count, dtype)

    def _make_rs(self, l: int, lm) -> RankSelectIndex:
        handle = self._h
        bits = self.bits
        sizes = {_lib.A_L1: (lm.n_l1, np.int64), _lib.A_L2: (lm.n_l2, np.uint16),
                 _lib.A_ONES: (lm.n_ones, np.int64), _lib.A_ZEROS: (lm.n_zeros, np.int64)}

        def fetch(what):
            n, dt = sizes[what]
            return handle.get(what, l, n, dt)

        def backend(kind, args):
            out = np.empty(len(args), np.int64)
            check(lib.wt_tree_level_query(handle.h, l, kind, ptr(args), ptr(out), len(args)),
                  "wt_tree_level_query")
            return out

        return RankSelectIndex(self.params, lm, backend, fetch,
                               lambda: bits.region_words(l), owner=handle)

    def query(self, kind: int, ids, args, *, symbols: bool = False, access_ids: bool = False,
              chunk: int = 0, sort: bool = False, out: np.ndarray | None = None,
              stats: "_lib.QueryStats | None" = None):
        """Run one batch on the device; returns (out, first_bad_index).
        ``out`` (optional): a contiguous array of the result dtype and length
        the answers are copied into (e.g. one rank's slice of a shared,
        page-locked result array, parallel.SharedResult)."""
        args = np.ascontiguousarray(np.asarray(args, np.int64).reshape(-1))
        m = len(args)
        if kind == _lib.Q_ACCESS:
            dt = np.dtype(np.int64 if access_ids else self.alphabet.sorted_symbols.dtype)
            ids_a = None
        else:
            dt = np.dtype(np.int64)
            ids_a = np.ascontiguousarray(np.asarray(ids, np.int64).reshape(-1))
        if out is None:
            out = _lib.pinned_empty(m, dt)
        elif (out.dtype != dt or len(out) != m or not out.flags.c_contiguous
              or not out.flags.writeable):
            raise ValueError(f"out must be a writeable contiguous {dt} array of length {m}")
        if m == 0:
            return out, -1
        flags = ((_lib.F_SYMBOLS if symbols else 0) | (_lib.F_ACCESS_IDS if access_ids else 0)
                 | (_lib.F_SORT if sort else 0))
        bad = C.c_int64(-1)
        check(lib.wt_tree_query_ex(self._h.h, kind, ptr(ids_a), ptr(args), ptr(out), m, chunk,
                                   flags, None, C.byref(bad), None,
                                   None if stats is None else C.byref(stats)), "wt_tree_query_ex")
        return out, int(bad.value)

    # -- shape helpers (wtree.py:137-190) -------------------------------------
    def _compute_spine_starts(self) -> np.ndarray:
        from .alphabet import prev_pow_two
        spine = np.zeros(self.num_levels + 1, np.int64)
        ns = 0
        for l in range(1, self.num_levels + 1):
            if self.sigma - ns >= 2:
                ns += prev_pow_two(self.sigma - ns)
            spine[l] = ns
        return spine

    def occurrences(self, c) -> int:
        cid = self.alphabet.id_for(_symbol_value(c))
        return int(self.cum_hist[cid + 1] - self.cum_hist[cid])

    def node_start(self, c_id: int, l: int) -> int:
        """Smallest symbol of the level-l node containing id c_id (Alg. 8,
        wtree.py:150-170); O(1) host arithmetic on the code table."""
        if c_id < 0 or c_id >= self.sigma:
            raise SymbolError(f"symbol id {c_id} outside [0, {self.sigma})")
        if l <= 0:
            return 0
        if self.sigma & (self.sigma - 1) == 0:
            width = 1 << (self.num_levels - l)
            return c_id & ~(width - 1)
        code = self.codes.code(c_id)
        if (code.value >> (self.num_levels - l)).bit_count() == l:
            return int(self._spine_starts[l])
        drop = max(code.length - l, 0)
        return c_id & ~((1 << drop) - 1)

    # -- scalar queries (wtree.py:194-279), answered by the device kernels ----
    def access(self, i: int):
        if not 0 <= i < self.n:
            raise PositionError(f"position {i} outside [0, {self.n})")
        out, _ = self.query(_lib.Q_ACCESS, None, [i])
        return int(out[0])

    def _access_id(self, i: int) -> int:
        return int(self.access_ids_bulk(np.array([i]))[0])

    def rank(self, c, i: int) -> int:
        cid = self.alphabet.id_for(_symbol_value(c))
        if not 0 <= i <= self.n:
            raise PositionError(f"position {i} outside [0, {self.n}]")
        return self._rank_id(cid, i)

    def _rank_id(self, cid: int, i: int) -> int:
        return int(self.rank_ids_bulk(np.array([cid]), np.array([i]))[0])

    def select(self, c, k: int) -> int:
        cid = self.alphabet.id_for(_symbol_value(c))
        occ = int(self.cum_hist[cid + 1] - self.cum_hist[cid])
        if not 1 <= k <= occ:
            raise OrdinalError(f"ordinal {k} outside [1, {occ}] for symbol {c!r}")
        return self._select_id(cid, k)

    def _select_id(self, cid: int, k: int) -> int:
        return int(self.select_ids_bulk(np.array([cid]), np.array([k]))[0])

    # -- bulk, minimal-id domain (wtree.py:283-375) ----------------------------
    def access_ids_bulk(self, pos: np.ndarray) -> np.ndarray:
        return self.query(_lib.Q_ACCESS, None, pos, access_ids=True)[0]

    def rank_ids_bulk(self, ids: np.ndarray, pos: np.ndarray) -> np.ndarray:
        return self.query(_lib.Q_RANK, ids, pos)[0]

    def select_ids_bulk(self, ids: np.ndarray, ks: np.ndarray) -> np.ndarray:
        return self.query(_lib.Q_SELECT, ids, ks)[0]

    # -- serialization -----------------------------------------------------------
    def save(self, sink) -> None:
        save(self, sink)

    def index_bytes(self) -> int:
        buf = io.BytesIO()
        save(self, buf)
        return buf.tell()

    @property
    def device_bytes(self) -> int:
        return int(self._meta.device_bytes)


# ---------------------------------------------------------------------------
# construction
# ---------------------------------------------------------------------------
def _build(text, alphabet_syms, sym_dtype, symbol_width, params, device_text=None):
    if params is None:
        params = RankSelectParams(sample_rate=TREE_SAMPLE_RATE)
    h = C.c_void_p()
    ms = C.c_float(0.0)
    if device_text is not None:
        dptr, n, sb = device_text
        text_ptr, on_dev, keep = C.c_void_p(dptr), 1, None
    else:
        keep = np.ascontiguousarray(text)
        n, sb = len(keep), keep.dtype.itemsize
        text_ptr, on_dev = ptr(keep), 0
    alpha = None if alphabet_syms is None else np.ascontiguousarray(alphabet_syms, np.uint16)
    rc = lib.wt_construct(text_ptr, n, sb, on_dev, ptr(alpha),
                          0 if alpha is None else len(alpha), np.dtype(sym_dtype).itemsize,
                          params.l2_bits, params.sample_rate, _lib.current_device(), None,
                          C.byref(h), C.byref(ms))
    check(rc, "wt_construct")
    del keep
    return WaveletTree(_TreeHandle(h), symbol_width, sym_dtype, float(ms.value))


def construct(text, workers: int = 1, params: RankSelectParams | None = None) -> WaveletTree:
    """Build a wavelet tree, inferring the alphabet (wtree.py:438-445).

    ``text``: bytes / numpy integer array (as the reference) or a contiguous
    CUDA ``torch`` uint8/uint16 tensor already resident in HBM.
    """
    dev = _device_text(text)
    if dev is not None:
        if dev[1] == 0:
            raise BuildError("cannot build an index over an empty text")
        dt = np.uint8 if dev[2] == 1 else np.uint16
        return _build(None, None, dt, dev[2], params, device_text=dev)
    arr, width = _coerce_text(text)
    if len(arr) == 0:
        raise BuildError("cannot build an index over an empty text")
    return _build(arr, None, arr.dtype, width, params)


def construct_with_alphabet(text, alphabet, workers: int = 1,
                            params: RankSelectParams | None = None) -> WaveletTree:
    """Build with a caller-declared (possibly superset) alphabet (wtree.py:448-466)."""
    dev = _device_text(text)
    if dev is not None:
        if dev[1] == 0:
            raise BuildError("cannot build an index over an empty text")
        width = dev[2]
        arr = None
    else:
        arr, width = _coerce_text(text)
        if len(arr) == 0:
            raise BuildError("cannot build an index over an empty text")
    alpha, awidth = _coerce_text(alphabet)
    if len(alpha) == 0:
        raise BuildError("declared alphabet is empty")
    symbols = np.unique(alpha)
    if len(symbols) > MAX_SIGMA:
        raise BuildError(f"alphabet size {len(symbols)} exceeds {MAX_SIGMA}")
    return _build(arr, symbols, symbols.dtype, max(width, awidth), params, device_text=dev)


# ---------------------------------------------------------------------------
# index file (wtree.py:472-577, rankselect.py:387-430, serial.py)
# ---------------------------------------------------------------------------
def _write_array(out, arr, dtype, length_prefix=True):
    if length_prefix:
        out.write(struct.pack("<Q", len(arr)))
    out.write(np.asarray(arr).astype(dtype, copy=False).tobytes())


def save(tree: WaveletTree, sink) -> None:
    """Serialize to the reference's WTIDX001 format, byte for byte."""
    if isinstance(sink, (str, Path)):
        with open(sink, "wb") as f:
            save(tree, f)
        return
    out: BinaryIO = sink
    flags = _FLAG_WIDE_SYMBOLS if tree.symbol_width == 2 else 0
    out.write(MAGIC)
    out.write(struct.pack("<IIQQI", VERSION, flags, tree.n, tree.sigma, tree.num_levels))
    _write_array(out, tree.alphabet.sorted_symbols, "<u2" if tree.symbol_width == 2 else "<u1",
                 length_prefix=False)
    out.write(struct.pack("<Q", tree.codes.num_explicit))
    for s in range(tree.codes.first_coded, tree.sigma):
        out.write(struct.pack("<IB", int(tree.codes.values[s]), int(tree.codes.lens[s])))
    _write_array(out, tree.level_sizes, "<u8", length_prefix=False)
    _write_array(out, tree.cum_hist, "<u8", length_prefix=False)
    _write_array(out, tree.bits.words, "<u8")
    for rs in tree.rs:
        rs.write(out)
    for starts, vals in zip(tree.node_starts, tree.node_rank0):
        out.write(struct.pack("<Q", len(starts)))
        _write_array(out, starts, "<u8", length_prefix=False)
        _write_array(out, vals, "<u8", length_prefix=False)


def _read_exact(src, count: int) -> bytes:
    data = src.read(count)
    if len(data) != count:
        raise TruncatedError(f"expected {count} bytes, got {len(data)}")
    return data


def _read_struct(src, fmt: str):
    return struct.unpack(fmt, _read_exact(src, struct.calcsize(fmt)))


def _read_array(src, dtype: str, count=None, max_count=1 << 40):
    if count is None:
        (count,) = _read_struct(src, "<Q")
    if count > max_count:
        raise CorruptIndexError(f"array length {count} is implausible")
    item = np.dtype(dtype).itemsize
    return np.frombuffer(_read_exact(src, count * item), dtype=dtype).copy()


def load(source) -> WaveletTree:
    """Deserialize and validate an index (wtree.py:500-577), then upload it."""
    if isinstance(source, (str, Path)):
        with open(source, "rb") as f:
            return load(f)
    src: BinaryIO = source
    magic = _read_exact(src, len(MAGIC))
    if magic != MAGIC:
        raise BadMagicError(f"bad magic {magic!r}")
    version, flags, n, sigma, num_levels = _read_struct(src, "<IIQQI")
    if version != VERSION:
        raise BadVersionError(f"unsupported index version {version}")
    if flags & ~_FLAG_WIDE_SYMBOLS:
        raise CorruptIndexError(f"unknown flag bits {flags:#x}")
    width = 2 if flags & _FLAG_WIDE_SYMBOLS else 1
    if not 1 <= sigma <= MAX_SIGMA or n < 1:
        raise CorruptIndexError("implausible n or sigma")
    if num_levels != ceil_log2(sigma):
        raise CorruptIndexError("level count does not match alphabet size")
    symbols = _read_array(src, "<u2" if width == 2 else "<u1", count=sigma)
    if np.any(np.diff(symbols.astype(np.int64)) <= 0):
        raise CorruptIndexError("alphabet symbols not strictly increasing")
    codes = create_codes(sigma)
    (num_explicit,) = _read_struct(src, "<Q")
    if num_explicit != codes.num_explicit:
        raise CorruptIndexError("explicit code count mismatch")
    for s in range(codes.first_coded, sigma):
        value, length = _read_struct(src, "<IB")
        if value != int(codes.values[s]) or length != int(codes.lens[s]):
            raise CorruptIndexError(f"stored code for symbol {s} is inconsistent")
    sizes = _read_array(src, "<u8", count=num_levels).astype(np.int64)
    cum = _read_array(src, "<u8", count=sigma + 1).astype(np.int64)
    if cum[0] != 0 or int(cum[-1]) != n or np.any(np.diff(cum) < 0):
        raise CorruptIndexError("cumulative histogram is not a valid prefix sum")
    lens = codes.lens.astype(np.int64)
    hist = np.diff(cum)
    expected = np.array([int(hist[lens > l].sum()) for l in range(num_levels)], np.int64)
    if not np.array_equal(sizes, expected):
        raise CorruptIndexError("level sizes inconsistent with histogram")
    offsets, n_words = region_layout(sizes)
    words = _read_array(src, "<u8").astype(np.uint64)
    if len(words) != n_words:
        raise CorruptIndexError("bit array word count mismatch")
    lms, l1s, l2s, ones, zeros = [], [], [], [], []
    for l in range(num_levels):
        l1_bits, l2_bits, rate, n_bits, total_ones = _read_struct(src, "<IIIQQ")
        try:
            params = RankSelectParams(l1_bits, l2_bits, rate)
        except ValueError as e:
            raise CorruptIndexError(str(e)) from e
        a1 = _read_array(src, "<u8").astype(np.int64)
        a2 = _read_array(src, "<u2")
        a3 = _read_array(src, "<u8").astype(np.int64)
        a4 = _read_array(src, "<u8").astype(np.int64)
        # RankSelectIndex._validate (rankselect.py:413-430)
        if len(a1) != -(-n_bits // 65536):
            raise CorruptIndexError("L1 directory length mismatch")
        if len(a2) != -(-n_bits // params.l2_bits):
            raise CorruptIndexError("L2 directory length mismatch")
        if not 0 <= total_ones <= n_bits:
            raise CorruptIndexError("total ones outside [0, n]")
        if len(a1) and (int(a1[0]) != 0 or np.any(np.diff(a1) < 0)):
            raise CorruptIndexError("L1 counts not a non-decreasing prefix sum")
        if len(a3) != total_ones // params.sample_rate:
            raise CorruptIndexError("one-sample count mismatch")
        if len(a4) != (n_bits - total_ones) // params.sample_rate:
            raise CorruptIndexError("zero-sample count mismatch")
        if n_bits != int(sizes[l]):
            raise CorruptIndexError(f"rank structure length mismatch at level {l}")
        if l and (params.l2_bits, params.sample_rate) != (lms[0][0].l2_bits,
                                                          lms[0][0].sample_rate):
            raise CorruptIndexError("per-level parameters differ")
        lm = _lib.LevelMeta(n_bits, total_ones, len(a1), len(a2), len(a3), len(a4), 0)
        lms.append((params, lm))
        l1s.append(a1)
        l2s.append(a2)
        ones.append(a3)
        zeros.append(a4)
    params = lms[0][0] if lms else RankSelectParams(sample_rate=TREE_SAMPLE_RATE)
    node_tables = []
    for l in range(num_levels):
        (count,) = _read_struct(src, "<Q")
        starts = _read_array(src, "<u8", count=count).astype(np.int64)
        vals = _read_array(src, "<u8", count=count).astype(np.int64)
        node_tables.append((starts, vals))
    if src.read(1):
        raise CorruptIndexError("trailing bytes after index payload")
    meta = _lib.Meta(n, sigma, num_levels, symbols.dtype.itemsize, params.l2_bits,
                     params.sample_rate, 0, 0, n_words, 0)
    lm_arr = (_lib.LevelMeta * max(num_levels, 1))(*[lm for _, lm in lms])
    cat = lambda xs, dt: np.ascontiguousarray(np.concatenate(xs) if xs else np.zeros(0, dt), dt)
    h = C.c_void_p()
    # every array the call reads is bound to a name for the duration of the call
    sym16, cum_c, words_c = (np.ascontiguousarray(symbols, np.uint16), np.ascontiguousarray(cum),
                             np.ascontiguousarray(words))
    l1_c, l2_c = cat(l1s, np.int64), cat(l2s, np.uint16)
    ones_c, zeros_c = cat(ones, np.int64), cat(zeros, np.int64)
    check(lib.wt_tree_from_arrays(C.byref(meta), ptr(sym16), ptr(cum_c), ptr(words_c), lm_arr,
                                  ptr(l1_c), ptr(l2_c), ptr(ones_c), ptr(zeros_c),
                                  _lib.current_device(), C.byref(h)), "wt_tree_from_arrays")
    del sym16, cum_c, words_c, l1_c, l2_c, ones_c, zeros_c
    tree = WaveletTree(_TreeHandle(h), width, symbols.dtype)
    # node tables: structural check against the shape, then the stored ranks
    # against the device's (wtree.py:556-572)
    for l, (starts, vals) in enumerate(node_tables):
        if not np.array_equal(starts, tree.node_starts[l]):
            raise CorruptIndexError(f"node starts mismatch at level {l}")
        recomputed = tree.rs[l].rank0_bulk(cum[starts]) if len(starts) else starts
        if not np.array_equal(vals, recomputed):
            raise CorruptIndexError(f"precomputed node ranks mismatch at level {l}")
    return tree
