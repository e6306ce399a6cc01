"""GPU parity at sizes where every kernel path runs many tiles: full and
partial tiles, single-node and multi-node tiles, LUT levels (level 0 through
the symbol -> code map), u8 / u16 codes.  Every array of the device tree is
compared with the oracle (the numpy restatement pinned to the reference's
golden vectors), then batched queries are checked against the text."""

import io

import numpy as np
import pytest

import oracle as O
from test_parity_gpu import assert_same_structure

pytestmark = pytest.mark.gpu

RNG = np.random.default_rng(20251017)


def _zipf(n, sigma, a=1.2, seed=3):
    r = np.random.default_rng(seed)
    return (np.minimum(r.zipf(a, n), sigma) - 1).astype(np.uint16)


LARGE = {
    "u8_s256_full": lambda: np.random.default_rng(1).integers(0, 256, 1 << 22, dtype=np.uint8),
    "u8_s256_partial": lambda: np.random.default_rng(2).integers(0, 256, (1 << 22) + 777,
                                                                 dtype=np.uint8),
    "u8_s200_lut": lambda: np.random.default_rng(3).integers(0, 200, (1 << 21) + 5,
                                                             dtype=np.uint8),
    "dna": lambda: np.frombuffer(b"ACGT", np.uint8)[
        np.random.default_rng(4).integers(0, 4, (1 << 22) + 13)],
    "u16_s4096": lambda: np.random.default_rng(5).integers(0, 4096, (1 << 21) + 3).astype(np.uint16),
    "u16_zipf_inferred": lambda: _zipf((1 << 21) + 1, 65536),
    "u8_skewed": lambda: np.minimum(np.random.default_rng(6).geometric(0.02, 1 << 21), 255)
                            .astype(np.uint8),
}


@pytest.fixture(scope="module")
def W():
    import paper_2505_03372_b200 as w
    return w


def _check_queries(W, t, text, sigma_syms, m=20000, seed=9):
    r = np.random.default_rng(seed)
    n = len(text)
    pos = r.integers(0, n, m)
    assert np.array_equal(W.access_batch(t, pos), text[pos])
    fa, fr, fs = O.text_answers(text, 1 << (8 * text.dtype.itemsize))
    syms = sigma_syms[r.integers(0, len(sigma_syms), m)].astype(np.int64)
    p = r.integers(0, n + 1, m)
    assert np.array_equal(W.rank_batch(t, syms, p), fr(syms, p))
    occ = {int(s): int(c) for s, c in zip(*np.unique(text, return_counts=True))}
    present = np.array(sorted(occ), np.int64)
    ss = present[r.integers(0, len(present), m)]
    ks = 1 + (r.random(m) * np.array([occ[int(s)] for s in ss])).astype(np.int64)
    assert np.array_equal(W.select_batch(t, ss, ks), fs(ss, ks))


@pytest.mark.parametrize("name", sorted(LARGE))
def test_large_build_and_queries(W, name):
    text = LARGE[name]()
    t = W.construct(text)
    o = O.build(text)
    assert_same_structure(t, o)
    _check_queries(W, t, text, t.alphabet.sorted_symbols)


def test_large_declared_alphabet_16_levels(W):
    """C3z recipe at reduced n: Zipf over a declared 2^16 alphabet -> 16 full
    levels with many multi-node tiles at the deep levels."""
    text = _zipf(1 << 21, 65536, seed=11)
    alpha = np.arange(65536, dtype=np.uint16)
    t = W.construct_with_alphabet(text, alpha)
    o = O.build_with_alphabet(text, alpha)
    assert t.num_levels == 16
    assert_same_structure(t, o)
    _check_queries(W, t, text, alpha)


def test_large_u8_text_u16_codes(W):
    """u8 text with a declared 1000-symbol alphabet: level 0 reads bytes and
    writes 16-bit codes (10 levels)."""
    text = np.random.default_rng(12).integers(0, 256, (1 << 20) + 9, dtype=np.uint8)
    alpha = np.arange(1000, dtype=np.uint16)
    t = W.construct_with_alphabet(text, alpha)
    o = O.build_with_alphabet(text, alpha)
    assert t.num_levels == 10
    assert_same_structure(t, o)


@pytest.mark.parametrize("chunk", [1000, 1 << 16, 1 << 22])
def test_device_query_sort_keeps_answers_and_errors(W, chunk):
    """WT_F_SORT (device sort_queries_by_symbol): same answers in query order,
    same first bad index, for every kind and chunking."""
    text = np.random.default_rng(21).integers(0, 256, (1 << 20) + 17, dtype=np.uint8)
    t = W.construct(text)
    r = np.random.default_rng(22)
    m = 50000
    pos = r.integers(0, len(text), m)
    syms = t.alphabet.sorted_symbols[r.integers(0, t.sigma, m)].astype(np.int64)
    rpos = r.integers(0, len(text) + 1, m)
    occ = np.diff(t.cum_hist)
    ids = r.integers(0, t.sigma, m)
    ks = 1 + (r.random(m) * occ[ids]).astype(np.int64)
    ssym = t.alphabet.sorted_symbols[ids].astype(np.int64)
    for f, args in ((W.access_batch, (pos,)), (W.rank_batch, (syms, rpos)),
                    (W.select_batch, (ssym, ks))):
        a = f(t, *args, chunk_size=chunk)
        b = f(t, *args, chunk_size=chunk, sort=True)
        assert np.array_equal(a, b)
    bad = rpos.copy()
    bad[[777, 31000]] = len(text) + 9
    with pytest.raises(W.BatchError) as e1:
        W.rank_batch(t, syms, bad, chunk_size=chunk, sort=True)
    assert e1.value.index == 777
    # device-resident path
    import torch
    from paper_2505_03372_b200 import _lib
    import ctypes as C
    d_ids = torch.from_numpy(ssym).cuda()
    d_ks = torch.from_numpy(ks).cuda()
    out = torch.empty(m, dtype=torch.int64, device="cuda")
    badi = C.c_int64(-1)
    _lib.check(_lib.lib.wt_tree_query(t.handle, _lib.Q_SELECT, C.c_void_p(d_ids.data_ptr()),
                                      C.c_void_p(d_ks.data_ptr()), C.c_void_p(out.data_ptr()), m, 0,
                                      _lib.F_DEVICE_PTRS | _lib.F_SYMBOLS | _lib.F_SORT, None,
                                      C.byref(badi), None))
    assert badi.value == -1
    assert np.array_equal(out.cpu().numpy(), W.select_batch(t, ssym, ks))


def test_device_query_sort_largest_argument(W):
    """n + 1 = 2^20 + 1 puts rank(c, n) exactly on the top of the 16-bit key
    range: the key must still land in one of the 65536 buckets."""
    text = np.random.default_rng(31).integers(0, 256, 1 << 20, dtype=np.uint8)
    t = W.construct(text)
    syms = t.alphabet.sorted_symbols.astype(np.int64)
    pos = np.full(len(syms), len(text), np.int64)
    want = np.array([(text == s).sum() for s in syms], np.int64)
    assert np.array_equal(W.rank_batch(t, syms, pos, sort=True), want)
    assert np.array_equal(W.rank_batch(t, syms, pos), want)


def test_nccl_replicate_world1(W):
    """The NCCL path of wt_tree_replicate (dlopen'ed NCCL, header + grouped
    broadcasts) at world size 1 -- the only size a one-GPU box can run; the
    multi-rank host logic is covered by tests/test_parallel_cpu.py."""
    import ctypes as C
    from paper_2505_03372_b200 import _lib
    text = np.random.default_rng(41).integers(0, 256, 1 << 20, dtype=np.uint8)
    t = W.construct(text)
    uid = (C.c_uint8 * 128)()
    _lib.check(_lib.lib.wt_nccl_unique_id(uid), "wt_nccl_unique_id")
    out = C.c_void_p()
    ms = C.c_float(-1)
    _lib.check(_lib.lib.wt_tree_replicate(t.handle, uid, 0, 1, _lib.current_device(), C.byref(out),
                                          C.byref(ms)), "wt_tree_replicate")
    assert out.value is None and ms.value >= 0  # the root keeps its own tree
    pos = np.random.default_rng(42).integers(0, len(text), 1000)
    assert np.array_equal(W.access_batch(t, pos), text[pos])


BLOCK_MODE = {
    "u8_s256_full": LARGE["u8_s256_full"],
    "u8_s256_partial": LARGE["u8_s256_partial"],
    "u8_s200_lut": LARGE["u8_s200_lut"],
    "dna": LARGE["dna"],
    "u8_skewed": LARGE["u8_skewed"],
    "one_block": lambda: np.random.default_rng(7).integers(0, 256, 65536, dtype=np.uint8),
    "under_one_block": lambda: np.random.default_rng(8).integers(0, 9, 40000, dtype=np.uint8),
    "blocks_plus_one": lambda: np.random.default_rng(9).integers(0, 256, 3 * 65536 + 1, dtype=np.uint8),
}


@pytest.mark.parametrize("name", sorted(BLOCK_MODE))
def test_level0_block_mode(W, name, monkeypatch):
    """Level 0 of a u8 text in block mode (a warp walks whole L1 blocks, P1 from
    the per-block histograms of K1) -- the default for large texts, forced here
    at test sizes -- gives the oracle's tree."""
    monkeypatch.setenv("WT_BLOCK_MODE", "1")
    text = BLOCK_MODE[name]()
    t = W.construct(text)
    assert_same_structure(t, O.build(text))
    _check_queries(W, t, text, t.alphabet.sorted_symbols, m=5000)


def test_device_query_sort_unaligned_inputs(W):
    """Device-resident batches starting at an odd element (8-byte, not 16-byte
    aligned) and odd lengths through the sorted path."""
    import ctypes as C
    import torch
    from paper_2505_03372_b200 import _lib
    text = np.random.default_rng(51).integers(0, 256, 1 << 20, dtype=np.uint8)
    t = W.construct(text)
    r = np.random.default_rng(52)
    m = 10001
    ids = t.alphabet.sorted_symbols[r.integers(0, t.sigma, m + 1)].astype(np.int64)
    pos = r.integers(0, len(text) + 1, m + 1)
    d_ids = torch.from_numpy(ids).cuda()[1:]
    d_pos = torch.from_numpy(pos).cuda()[1:]
    assert d_pos.data_ptr() % 16 == 8
    out = torch.empty(m, dtype=torch.int64, device="cuda")
    bad = C.c_int64(-1)
    _lib.check(_lib.lib.wt_tree_query(t.handle, _lib.Q_RANK, C.c_void_p(d_ids.data_ptr()),
                                      C.c_void_p(d_pos.data_ptr()), C.c_void_p(out.data_ptr()), m, 0,
                                      _lib.F_DEVICE_PTRS | _lib.F_SYMBOLS | _lib.F_SORT, None,
                                      C.byref(bad), None))
    assert bad.value == -1
    assert np.array_equal(out.cpu().numpy(), W.rank_batch(t, ids[1:], pos[1:]))


@pytest.mark.parametrize("name", ["u16_s4096", "u16_zipf_inferred", "u8_skewed", "dna"])
def test_device_query_sort_other_trees(W, name):
    """The sorted path on u16 / Zipf / skewed / DNA trees: bucket layouts with
    many symbol bits (sigma up to 2^16) and select position estimates from very
    unequal occurrence counts."""
    text = LARGE[name]()
    t = W.construct(text)
    _, fr, fs = O.text_answers(text, 1 << (8 * text.dtype.itemsize))
    r = np.random.default_rng(61)
    m = 30011
    pos = r.integers(0, len(text), m)
    assert np.array_equal(W.access_batch(t, pos, sort=True), text[pos])
    syms = t.alphabet.sorted_symbols[r.integers(0, t.sigma, m)].astype(np.int64)
    p = r.integers(0, len(text) + 1, m)
    assert np.array_equal(W.rank_batch(t, syms, p, sort=True), fr(syms, p))
    occ = np.diff(t.cum_hist)
    ids = np.flatnonzero(occ)[r.integers(0, np.count_nonzero(occ), m)]
    ks = 1 + (r.random(m) * occ[ids]).astype(np.int64)
    ss = t.alphabet.sorted_symbols[ids].astype(np.int64)
    assert np.array_equal(W.select_batch(t, ss, ks, sort=True), fs(ss, ks))


@pytest.mark.parametrize("m", [1, 2, 33, 4097])
def test_device_query_sort_tiny_batches(W, m):
    text = np.random.default_rng(71).integers(0, 256, 100003, dtype=np.uint8)
    t = W.construct(text)
    r = np.random.default_rng(72 + m)
    pos = r.integers(0, len(text), m)
    assert np.array_equal(W.access_batch(t, pos, sort=True), text[pos])
    syms = t.alphabet.sorted_symbols[r.integers(0, t.sigma, m)].astype(np.int64)
    ks = np.ones(m, np.int64)
    _, _, fs = O.text_answers(text, 256)
    assert np.array_equal(W.select_batch(t, syms, ks, sort=True), fs(syms, ks))


def test_hist16_counter_wrap(W):
    """Hot symbols with far more than 32768 occurrences per CTA (the packed
    16-bit shared counters spill many times), two of them in the same counter
    word, next to rare ones: exact histogram, exact rank / select."""
    r = np.random.default_rng(81)
    n = (1 << 25) + 5
    # two hot symbols sharing one 32-bit counter word (40000, 40001) and a
    # third hot one, each far past 32768 per CTA
    text = np.where(r.random(n) < 0.5, 40000, 40001).astype(np.uint16)
    text[r.integers(0, n, n // 5)] = 7
    text[r.integers(0, n, 50000)] = r.integers(0, 65536, 50000).astype(np.uint16)
    t = W.construct(text)
    vals, cnts = np.unique(text, return_counts=True)
    assert np.array_equal(t.alphabet.sorted_symbols, vals)
    assert np.array_equal(np.diff(t.cum_hist), cnts)
    _, fr, fs = O.text_answers(text, 65536)
    syms = np.array([40000, 40001, int(vals[0]), int(vals[-1])] * 250, np.int64)
    pos = r.integers(0, n + 1, len(syms))
    assert np.array_equal(W.rank_batch(t, syms, pos), fr(syms, pos))
    occ = dict(zip(vals.tolist(), cnts.tolist()))
    ks = 1 + (r.random(len(syms)) * np.array([occ[int(s_)] for s_ in syms])).astype(np.int64)
    assert np.array_equal(W.select_batch(t, syms, ks), fs(syms, ks))


@pytest.mark.parametrize("case", ["full", "declared_zipf", "s4096_fallback", "partial_blocks"])
def test_level0_block_mode_u16(W, case, monkeypatch):
    """u16 level 0 in block mode: K1 counts the symbols >= 32768 per L1 block,
    used when the top-bit threshold is 32768 (full or declared 2^16
    alphabets); other thresholds fall back to the counting pass."""
    monkeypatch.setenv("WT_BLOCK_MODE", "1")
    r = np.random.default_rng(91)
    alpha = None
    if case == "full":
        text = r.integers(0, 65536, (1 << 21) + 3).astype(np.uint16)
    elif case == "declared_zipf":
        text = _zipf((1 << 21) + 7, 65536, seed=13)
        alpha = np.arange(65536, dtype=np.uint16)
    elif case == "s4096_fallback":
        text = r.integers(0, 4096, (1 << 21) + 1).astype(np.uint16)
    else:
        text = r.integers(0, 65536, 3 * 65536 + 999).astype(np.uint16)
        alpha = np.arange(65536, dtype=np.uint16)
    if alpha is None:
        t, o = W.construct(text), O.build(text)
    else:
        t, o = W.construct_with_alphabet(text, alpha), O.build_with_alphabet(text, alpha)
    assert_same_structure(t, o)
    _check_queries(W, t, text, t.alphabet.sorted_symbols if alpha is None else alpha, m=4000)


def test_device_query_sort_slices(W, monkeypatch):
    """Device batches above the slice size (2^31 queries in production) are
    sorted slice by slice: same answers and the same first bad index."""
    import ctypes as C
    import torch
    from paper_2505_03372_b200 import _lib
    monkeypatch.setenv("WT_SORT_SLICE", "1000")
    text = np.random.default_rng(101).integers(0, 256, 200003, dtype=np.uint8)
    t = W.construct(text)
    r = np.random.default_rng(102)
    m = 5003
    syms = t.alphabet.sorted_symbols[r.integers(0, t.sigma, m)].astype(np.int64)
    pos = r.integers(0, len(text) + 1, m)
    _, fr, _ = O.text_answers(text, 256)
    d_ids, d_pos = torch.from_numpy(syms).cuda(), torch.from_numpy(pos).cuda()
    out = torch.empty(m, dtype=torch.int64, device="cuda")
    bad = C.c_int64(-1)
    flags = _lib.F_DEVICE_PTRS | _lib.F_SYMBOLS | _lib.F_SORT
    P = lambda x: C.c_void_p(x.data_ptr())
    _lib.check(_lib.lib.wt_tree_query(t.handle, _lib.Q_RANK, P(d_ids), P(d_pos), P(out), m, 0, flags,
                                      None, C.byref(bad), None))
    assert bad.value == -1
    assert np.array_equal(out.cpu().numpy(), fr(syms, pos))
    pos[[3100, 4500]] = len(text) + 7
    d_pos = torch.from_numpy(pos).cuda()
    rc = _lib.lib.wt_tree_query(t.handle, _lib.Q_RANK, P(d_ids), P(d_pos), P(out), m, 0, flags, None,
                                C.byref(bad), None)
    assert bad.value == 3100


@pytest.mark.parametrize("dt,syms", [(np.uint8, (97, 98)), (np.uint16, (1000, 60000)),
                                     (np.uint8, (0, 1))])
def test_single_level_trees(W, dt, syms):
    """sigma = 2: level 0 is the last level (wlast_kernel) -- through the LUT
    for non-identity alphabets -- with full tiles on the TMA ring and a
    partial last tile."""
    r = np.random.default_rng(111)
    text = np.array(syms, dt)[r.integers(0, 2, (1 << 20) + 5)]
    t = W.construct(text)
    assert t.num_levels == 1
    assert_same_structure(t, O.build(text))
    _check_queries(W, t, text, t.alphabet.sorted_symbols, m=3000)


PAIR_CASES = {
    "u8_s256": lambda: np.random.default_rng(31).integers(0, 256, (1 << 22) + 4097, dtype=np.uint8),
    "u8_s4_small": lambda: np.random.default_rng(32).integers(0, 4, 70_001, dtype=np.uint8),
    "dna": lambda: np.frombuffer(b"ACGT", np.uint8)[
        np.random.default_rng(33).integers(0, 4, (1 << 22) + 13)],
    "u8_s16_skewed": lambda: np.minimum(np.random.default_rng(34).geometric(0.3, 1 << 21), 16)
                                .astype(np.uint8) - 1,
    "u16_s65536": lambda: np.random.default_rng(35).integers(0, 65536, (1 << 21) + 9)
                             .astype(np.uint16),
    "u16_s1024_lut": lambda: (np.random.default_rng(36).integers(0, 1024, (1 << 20) + 1)
                              * 37).astype(np.uint16),
    "u16_zipf": lambda: _zipf((1 << 21) + 5, 65536, seed=37),
}


@pytest.mark.parametrize("block", ["0", "1"])
@pytest.mark.parametrize("name", sorted(PAIR_CASES))
def test_pair_mode_matches_level_by_level(W, name, block, monkeypatch):
    """Pair mode (the last two levels in one pass: the last level's bits from
    the staged runs, its L2 / samples from dir_kernel) builds the same index
    as the level-by-level path (WT_PAIR=0), and the oracle's."""
    text = PAIR_CASES[name]()
    monkeypatch.setenv("WT_BLOCK_MODE", block)
    monkeypatch.setenv("WT_PAIR", "1")
    t1 = W.construct(text)
    monkeypatch.setenv("WT_PAIR", "0")
    t0 = W.construct(text)
    b1, b0 = io.BytesIO(), io.BytesIO()
    t1.save(b1)
    t0.save(b0)
    assert b1.getvalue() == b0.getvalue()
    assert_same_structure(t1, O.build(text))
    _check_queries(W, t1, text, t1.alphabet.sorted_symbols, m=5000)
