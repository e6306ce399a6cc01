"""GPU parity: the CUDA path (through the C-ABI) against the reference's golden
vectors and the oracle, bit for bit."""

import hashlib
import io
import json
import os
import struct

import numpy as np
import pytest

import cases as C
import oracle as O

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")
G = json.load(open(os.path.join(GOLD, "golden.json")))
NPZ = np.load(os.path.join(GOLD, "golden.npz"))


@pytest.fixture(scope="module")
def W():
    import paper_2505_03372_b200 as w
    return w


def build(W, case):
    text = C.text_of(case)
    alpha = C.alphabet_of(case)
    params = W.RankSelectParams(l2_bits=case["l2_bits"], sample_rate=case["rate"])
    if alpha is None:
        return W.construct(text, params=params)
    return W.construct_with_alphabet(text, alpha, params=params)


def oracle_tree(case):
    text = C.text_of(case)
    alpha = C.alphabet_of(case)
    if alpha is None:
        return O.build(text, case["l2_bits"], case["rate"])
    return O.build_with_alphabet(text, alpha, case["l2_bits"], case["rate"])


def assert_same_structure(t, o):
    assert (t.n, t.sigma, t.num_levels) == (o.n, o.sigma, o.L)
    assert np.array_equal(t.alphabet.sorted_symbols, o.symbols)
    assert np.array_equal(t.codes.values, o.values) and np.array_equal(t.codes.lens, o.lens)
    assert np.array_equal(t.cum_hist, o.cum)
    assert np.array_equal(t.level_sizes, o.sizes)
    assert np.array_equal(t.bits.region_offsets, o.offsets)
    words = t.bits.words
    assert len(words) == len(o.words)
    for l in range(o.L):
        w0 = int(o.offsets[l]) >> 6
        w1 = w0 + (int(o.sizes[l]) + 63) // 64
        bad = np.flatnonzero(words[w0:w1] != o.words[w0:w1])
        assert len(bad) == 0, f"level {l}: {len(bad)} words differ, first at word {bad[:5]}"
    assert np.array_equal(words, o.words), "padding words differ"
    for l, d in enumerate(o.dirs):
        rs = t.rs[l]
        assert rs.total_ones == d["total_ones"], l
        assert np.array_equal(rs.l1_counts, d["l1"]), f"L1 level {l}"
        assert np.array_equal(rs.l2_counts, d["l2"]), f"L2 level {l}"
        assert np.array_equal(rs.one_samples, d["ones"]), f"one samples level {l}"
        assert np.array_equal(rs.zero_samples, d["zeros"]), f"zero samples level {l}"
        assert np.array_equal(t.node_starts[l], o.node_starts[l])
        assert np.array_equal(t.node_rank0[l], o.node_rank0[l])


@pytest.mark.parametrize("case", C.TREE_CASES, ids=[c["name"] for c in C.TREE_CASES])
def test_build_bit_exact(W, case):
    t = build(W, case)
    o = oracle_tree(case)
    assert_same_structure(t, o)
    buf = io.BytesIO()
    t.save(buf)
    raw = buf.getvalue()
    assert raw == o.save_bytes()
    assert hashlib.sha256(raw).hexdigest() == G["tree"][case["name"]]["save_sha256"]


@pytest.mark.parametrize("case", C.TREE_CASES, ids=[c["name"] for c in C.TREE_CASES])
def test_batch_queries_match_reference(W, case):
    t = build(W, case)
    hist = np.diff(t.cum_hist)
    acc, (rsym, rpos), (ssym, ks) = C.queries_of(t.n, hist, t.alphabet.sorted_symbols, 7, 400)
    name = case["name"]
    a = W.access_batch(t, acc)
    assert a.dtype == NPZ[name + "__access"].dtype
    assert np.array_equal(a, NPZ[name + "__access"])
    assert np.array_equal(W.rank_batch(t, rsym, rpos), NPZ[name + "__rank"])
    assert np.array_equal(W.select_batch(t, ssym, ks), NPZ[name + "__select"])
    # chunking never changes results (test_batch.py:58-79)
    for chunk in (1, 37, 4096):
        assert np.array_equal(W.rank_batch(t, rsym, rpos, chunk_size=chunk), NPZ[name + "__rank"])
    # scalar paths (wtree.py:194-279)
    for j in range(0, len(acc), 97):
        assert t.access(int(acc[j])) == int(NPZ[name + "__access"][j])
        assert t.rank(int(rsym[j]), int(rpos[j])) == int(NPZ[name + "__rank"][j])
    for j in range(0, len(ks), 97):
        assert t.select(int(ssym[j]), int(ks[j])) == int(NPZ[name + "__select"][j])


@pytest.mark.parametrize("case", C.BITS_CASES, ids=[c["name"] for c in C.BITS_CASES])
def test_bit_directory_bit_exact(W, case):
    g = G["bits"][case["name"]]
    bits = C.bits_of(case)
    ba = W.build_bit_array([len(bits)])
    if len(bits):
        ba.fill_region(0, bits)
    idx = W.build_index(ba, 0, W.RankSelectParams(l2_bits=case["l2_bits"],
                                                  sample_rate=case["rate"]))
    buf = io.BytesIO()
    idx.write(buf)
    assert hashlib.sha256(buf.getvalue()).hexdigest() == g["rs_sha256"]
    cs = np.concatenate([[0], np.cumsum(bits, dtype=np.int64)])
    rng = np.random.default_rng(case["seed"] + 1)
    n = len(bits)
    pos = rng.integers(0, n + 1, 300)
    assert np.array_equal(idx.rank1_bulk(pos), cs[pos])
    ones = np.flatnonzero(bits)
    zeros = np.flatnonzero(bits == 0)
    if len(ones):
        k = rng.integers(1, len(ones) + 1, 300)
        assert np.array_equal(idx.select1_bulk(k), ones[k - 1])
    if len(zeros):
        k = rng.integers(1, len(zeros) + 1, 300)
        assert np.array_equal(idx.select0_bulk(k), zeros[k - 1])


def test_worked_example(W):
    t = W.construct(b"dbdcaacbcd")
    assert (t.n, t.sigma, t.num_levels) == (10, 4, 2)
    assert t.cum_hist.tolist() == [0, 2, 4, 7, 10]
    assert [t.bits.get_region_bit(0, j) for j in range(10)] == [1, 0, 1, 1, 0, 0, 1, 0, 1, 1]
    assert [t.bits.get_region_bit(1, j) for j in range(10)] == [1, 0, 0, 1, 1, 1, 0, 0, 0, 1]
    assert t.access(6) == ord("c")
    assert t.rank("c", 6) == 1
    assert t.select("c", 2) == 6
    assert bytes(t.access(i) for i in range(10)) == b"dbdcaacbcd"
    assert W.access_batch(t, [6]).tolist() == [ord("c")]
    assert W.rank_batch(t, [ord("c")], [6]).tolist() == [1]
    assert W.select_batch(t, [ord("c")], [2]).tolist() == [6]


def test_batch_errors_match_reference(W):
    t = W.construct(b"dbdcaacbcd")
    with pytest.raises(W.BatchError) as e:
        W.access_batch(t, [0, 3, 10, -1])
    assert e.value.index == 2 and isinstance(e.value.__cause__, W.PositionError)
    with pytest.raises(W.BatchError) as e:
        W.rank_batch(t, [ord("a"), ord("z"), ord("a")], [0, 1, 11])
    assert e.value.index == 1 and isinstance(e.value.__cause__, W.SymbolError)
    with pytest.raises(W.BatchError) as e:
        W.rank_batch(t, [ord("a"), ord("a")], [10, 11])
    assert e.value.index == 1 and isinstance(e.value.__cause__, W.PositionError)
    with pytest.raises(W.BatchError) as e:
        W.select_batch(t, [ord("a"), ord("c")], [2, 4])
    assert e.value.index == 1 and isinstance(e.value.__cause__, W.OrdinalError)
    # errors in a later chunk still report the global first index
    pos = np.zeros(10000, np.int64)
    pos[7777] = 99
    pos[9000] = -5
    with pytest.raises(W.BatchError) as e:
        W.access_batch(t, pos, chunk_size=1000)
    assert e.value.index == 7777
    with pytest.raises(W.PositionError):
        t.access(10)
    with pytest.raises(W.SymbolError):
        t.rank("z", 0)
    with pytest.raises(W.OrdinalError):
        t.select("a", 3)
    assert W.rank_batch(t, [ord("c")], [10]).tolist() == [3]
    assert len(W.access_batch(t, [])) == 0


def test_staging_never_exceeds_two_chunks(W):
    t = W.construct(np.random.default_rng(3).integers(0, 50, 5000).astype(np.uint8))
    r = W.BatchRunner(t, chunk_size=100)
    r.run(W.QueryBatch("access", np.arange(5000) % t.n))
    # measured by the C pipeline from its CUDA events (not a formula): the
    # most queries resident in the two device slots at once
    assert r.chunks == 50 and r.staging_allocated_records == 200
    assert 100 <= r.staging_peak_records <= 200
    assert r.stage_seconds > 0 and r.process_seconds > 0
    one = W.BatchRunner(t, chunk_size=10_000)
    one.run(W.QueryBatch("access", np.arange(5000) % t.n))
    assert (one.chunks, one.staging_peak_records, one.staging_allocated_records) == (1, 5000, 5000)


def test_build_errors(W):
    with pytest.raises(W.BuildError):
        W.construct(b"")
    with pytest.raises(W.BuildError):
        W.construct(np.array([1.5, 2.0]))
    with pytest.raises(W.BuildError):
        W.construct(np.array([70000, 1]))
    with pytest.raises(W.SymbolError) as e:
        W.construct_with_alphabet(b"abcxa", b"abc")
    assert "position 3" in str(e.value)
    with pytest.raises(W.BuildError):
        W.construct_with_alphabet(b"abc", b"")


def test_save_load_roundtrip(W, tmp_path):
    rng = np.random.default_rng(5)
    for text in (rng.integers(0, 11, 3000).astype(np.uint8),
                 rng.integers(0, 3000, 20000).astype(np.uint16), b"zzzz"):
        t = W.construct(text)
        p = tmp_path / "x.wti"
        W.save(t, p)
        t2 = W.load(p)
        b1, b2 = io.BytesIO(), io.BytesIO()
        t.save(b1)
        t2.save(b2)
        assert b1.getvalue() == b2.getvalue()
        pos = rng.integers(0, t.n, 500)
        assert np.array_equal(W.access_batch(t, pos), W.access_batch(t2, pos))
    raw = p.read_bytes()
    with pytest.raises(W.BadMagicError):
        W.load(io.BytesIO(b"XXXXXXXX" + raw[8:]))
    with pytest.raises(W.TruncatedError):
        W.load(io.BytesIO(raw[:-3]))
    with pytest.raises(W.CorruptIndexError):
        W.load(io.BytesIO(raw + b"\0"))


def test_device_resident_text(W):
    import torch
    rng = np.random.default_rng(9)
    text = rng.integers(0, 256, 1 << 20).astype(np.uint8)
    t_host = W.construct(text)
    t_dev = W.construct(torch.from_numpy(text).cuda())
    b1, b2 = io.BytesIO(), io.BytesIO()
    t_host.save(b1)
    t_dev.save(b2)
    assert b1.getvalue() == b2.getvalue()


def test_load_many_small_trees_roundtrip(W):
    """Regression: load() passed temporaries (np.concatenate results) to the
    C-ABI by address; numpy's small-buffer cache then reused their memory
    before the call read it (found by the reference's own C8 / CLI stats
    tests, run against this package)."""
    rng = np.random.default_rng(1008)
    for k in range(40):
        sigma = int(rng.integers(2, 300))
        n = int(rng.integers(1, 20000))
        text = rng.integers(0, sigma, n).astype(np.uint8 if sigma <= 256 else np.uint16)
        t = W.construct(text)
        buf = io.BytesIO()
        W.save(t, buf)
        blob = buf.getvalue()
        t2 = W.load(io.BytesIO(blob))
        buf2 = io.BytesIO()
        W.save(t2, buf2)
        assert buf2.getvalue() == blob


def test_pinned_result_cache_size_classes_and_cap():
    """Pinned result blocks come in power-of-two classes (a block serves any
    size of its class) and the free lists are capped (the cache
    grew one block per distinct size, without bound)."""
    import gc

    from paper_2505_03372_b200 import _lib
    a = _lib.pinned_empty((3 << 20) // 8, np.int64)      # 3 MiB -> the 4 MiB class
    addr = a.ctypes.data
    del a
    gc.collect()
    b = _lib.pinned_empty((7 << 19) // 8, np.int64)      # 3.5 MiB: same class, same block
    assert b.ctypes.data == addr
    del b
    gc.collect()
    old = _lib.PINNED_CACHE_BYTES
    try:
        _lib.PINNED_CACHE_BYTES = _lib.pinned_cached_bytes()  # no room for more
        c = _lib.pinned_empty((9 << 20) // 8, np.int64)    # a new 16 MiB block
        del c
        gc.collect()
        assert _lib.pinned_cached_bytes() <= _lib.PINNED_CACHE_BYTES  # freed, not cached
    finally:
        _lib.PINNED_CACHE_BYTES = old


@pytest.mark.parametrize("sort", [False, True])
def test_narrow_wire_chunks_mixed_with_wide(W, sort, monkeypatch):
    """Host-buffer batches cross PCIe packed (u16 symbols / u32 arguments,
    wt_capi.cu pack_wire); a chunk holding a value that does not fit crosses
    wide.  Answers and the first bad index are the same either way."""
    monkeypatch.setenv("WT_WIRE_MIN_CHUNK", "1")  # (default: chunks of 2^20 and up)
    rng = np.random.default_rng(11)
    text = rng.integers(0, 200, 50_000).astype(np.uint8)
    t = W.construct(text)
    fa, fr, fs = O.text_answers(text, 256)
    m = 20_000
    c = rng.choice(np.unique(text), m).astype(np.int64)
    p = rng.integers(0, len(text) + 1, m)
    assert np.array_equal(W.rank_batch(t, c, p, chunk_size=3000, sort=sort), fr(c, p))
    occ = np.bincount(text, minlength=256)
    k = 1 + (rng.random(m) * occ[c]).astype(np.int64)
    assert np.array_equal(W.select_batch(t, c, k, chunk_size=3000, sort=sort), fs(c, k))
    pos = rng.integers(0, len(text), m)
    assert np.array_equal(W.access_batch(t, pos, chunk_size=3000, sort=sort), text[pos])
    r = W.BatchRunner(t, 3000, sort=sort)
    assert np.array_equal(r.run(W.QueryBatch("rank", p, c, 3000)), fr(c, p))
    assert r.chunks == 7 and r.narrow_chunks == 7 and r.h2d_bytes == 6 * m
    big = c.copy()
    big[3500] = 1 << 20  # chunk 1 crosses wide (and raises: not in the alphabet)
    with pytest.raises(W.BatchError):
        r.run(W.QueryBatch("rank", p, big, 3000))
    assert r.chunks == 7 and r.narrow_chunks == 6
    monkeypatch.setenv("WT_WIRE_MIN_CHUNK", str(1 << 40))
    assert np.array_equal(r.run(W.QueryBatch("rank", p, c, 3000)), fr(c, p))
    assert r.narrow_chunks == 0 and r.h2d_bytes == 16 * m
    monkeypatch.setenv("WT_WIRE_MIN_CHUNK", "1")
    # a symbol >= 2^16 (wide chunk 4) after an in-range but absent one (narrow chunk 2)
    bad_c = c.copy()
    bad_c[13_000] = 70_000
    bad_c[7_500] = 250
    with pytest.raises(W.BatchError) as e:
        W.rank_batch(t, bad_c, p, chunk_size=3000, sort=sort)
    assert e.value.index == 7_500 and isinstance(e.value.__cause__, W.SymbolError)
    bad_c[7_500] = c[7_500]
    with pytest.raises(W.BatchError) as e:
        W.rank_batch(t, bad_c, p, chunk_size=3000, sort=sort)
    assert e.value.index == 13_000 and isinstance(e.value.__cause__, W.SymbolError)
    # positions / ordinals >= 2^32 and negative ones cross wide and still fail
    bad_p = p.copy()
    bad_p[4_001] = 1 << 33
    bad_p[19_999] = -1
    with pytest.raises(W.BatchError) as e:
        W.rank_batch(t, c, bad_p, chunk_size=3000, sort=sort)
    assert e.value.index == 4_001 and isinstance(e.value.__cause__, W.PositionError)
    bad_k = k.copy()
    bad_k[6_123] = (1 << 32) + 5
    with pytest.raises(W.BatchError) as e:
        W.select_batch(t, c, bad_k, chunk_size=3000, sort=sort)
    assert e.value.index == 6_123 and isinstance(e.value.__cause__, W.OrdinalError)
    bad_pos = pos.copy()
    bad_pos[11_111] = -(1 << 40)
    with pytest.raises(W.BatchError) as e:
        W.access_batch(t, bad_pos, chunk_size=3000, sort=sort)
    assert e.value.index == 11_111 and isinstance(e.value.__cause__, W.PositionError)
