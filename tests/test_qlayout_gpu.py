"""GPU: the query-side layout ("rank lines" + line samples) and the reference
directory written by the build's fused pass (dirq_kernel: one streaming pass
per level) equal

  * a numpy restatement from the level's bits (line i = [ones before bit
    192 i | words 3i .. 3i+2], sel1[j] = line of the (64 j + 1)-th one),
  * the layout of the same index loaded from its saved bytes (load() runs
    qlayout_kernel over the reference directory), and
  * the split path (WT_DIRQ=0: dir_kernel + qlayout_kernel),

at sizes around every boundary the kernel has: one line (192 bits), one CTA
(1024 lines = three L1 blocks), L2 / sample parameters off their defaults."""

import io

import numpy as np
import pytest

import oracle as O
from test_parity_gpu import assert_same_structure

pytestmark = pytest.mark.gpu

QW, QBITS, QSEL = 3, 192, 64


@pytest.fixture(scope="module")
def W():
    import paper_2505_03372_b200 as w
    return w


def _layout(W, t, l):
    from paper_2505_03372_b200 import _lib
    lm = t._lmeta[l]
    n_lines = lm.n_bits // QBITS + 1
    lines = t._get(_lib.A_QLINES, l, 4 * n_lines, np.uint64)
    z = lm.n_bits - lm.total_ones
    s1 = t._get(_lib.A_QSEL1, l, -(-lm.total_ones // QSEL), np.uint32)
    s0 = t._get(_lib.A_QSEL0, l, -(-z // QSEL), np.uint32)
    return lines.reshape(-1, 4), s1, s0


def _expected(W, t, l):
    """numpy restatement of the layout from the level's words."""
    from paper_2505_03372_b200 import _lib
    lm = t._lmeta[l]
    m = int(lm.n_bits)
    words = t._get(_lib.A_WORDS, 0, t._meta.n_words, np.uint64)
    off = int(t._get(_lib.A_REGION_OFFS, 0, t.num_levels, np.int64)[l])
    nw = (m + 63) // 64
    w = words[off // 64: off // 64 + nw]
    n_lines = m // QBITS + 1
    wp = np.zeros(3 * n_lines, np.uint64)
    wp[:nw] = w
    wp = wp.reshape(-1, 3)
    bits = np.unpackbits(w.view(np.uint8), bitorder="little")[:m]
    ones_before_line = np.concatenate([[0], np.cumsum(bits, dtype=np.int64)])[
        np.minimum(np.arange(n_lines) * QBITS, m)]
    lines = np.column_stack([ones_before_line.astype(np.uint64), wp])
    one_pos = np.flatnonzero(bits)
    zero_pos = np.flatnonzero(bits == 0)
    s1 = (one_pos[::QSEL] // QBITS).astype(np.uint32)
    s0 = (zero_pos[::QSEL] // QBITS).astype(np.uint32)
    return lines, s1, s0


def _same_layout(W, a, b):
    for l in range(a.num_levels):
        la, lb = _layout(W, a, l), _layout(W, b, l)
        for x, y, what in zip(la, lb, ("lines", "sel1", "sel0")):
            assert np.array_equal(x, y), f"level {l}: {what} differ"


CASES = {
    "n1": lambda: np.array([7], np.uint8),
    "n191_s2": lambda: np.random.default_rng(1).integers(0, 2, 191, dtype=np.uint8),
    "n192_s2": lambda: np.random.default_rng(2).integers(0, 2, 192, dtype=np.uint8),
    "n193_s3": lambda: np.random.default_rng(3).integers(0, 3, 193, dtype=np.uint8),
    "one_cta_s2": lambda: np.random.default_rng(4).integers(0, 2, 3 * 65536, dtype=np.uint8),
    "one_cta_plus1_s2": lambda: np.random.default_rng(5).integers(0, 2, 3 * 65536 + 1,
                                                                  dtype=np.uint8),
    "u8_s256_partial": lambda: np.random.default_rng(6).integers(0, 256, (1 << 21) + 777,
                                                                 dtype=np.uint8),
    "u8_skewed": lambda: np.minimum(np.random.default_rng(7).geometric(0.05, 1 << 20), 255)
                            .astype(np.uint8),
    "u16_s4096": lambda: np.random.default_rng(8).integers(0, 4096, (1 << 20) + 3)
                            .astype(np.uint16),
    "almost_all_ones": lambda: np.concatenate([[0], np.full(5 * 65536 + 9, 1)]).astype(np.uint8),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_build_layout_matches_restatement_load_and_split_path(W, name, monkeypatch):
    text = CASES[name]()
    t = W.construct(text)
    for l in range(t.num_levels):
        got, exp = _layout(W, t, l), _expected(W, t, l)
        for x, y, what in zip(got, exp, ("lines", "sel1", "sel0")):
            assert np.array_equal(x, y), f"level {l}: {what} differ from the restatement"
    buf = io.BytesIO()
    t.save(buf)
    buf.seek(0)
    _same_layout(W, t, W.load(buf))
    monkeypatch.setenv("WT_DIRQ", "0")
    t0 = W.construct(text)
    _same_layout(W, t, t0)
    b0 = io.BytesIO()
    t0.save(b0)
    assert b0.getvalue() == buf.getvalue()
    assert_same_structure(t, O.build(text))


@pytest.mark.parametrize("l2_bits,rate", [(64, 7), (65536, 1), (1024, 4096), (512, 100)])
def test_build_layout_nondefault_directory(W, l2_bits, rate):
    from paper_2505_03372_b200.rankselect import RankSelectParams
    text = np.random.default_rng(l2_bits + rate).integers(0, 16, 3 * 65536 + 4099, dtype=np.uint8)
    params = RankSelectParams(l2_bits=l2_bits, sample_rate=rate)
    t = W.construct(text, params=params)
    for l in range(t.num_levels):
        got, exp = _layout(W, t, l), _expected(W, t, l)
        for x, y, what in zip(got, exp, ("lines", "sel1", "sel0")):
            assert np.array_equal(x, y), f"level {l}: {what} differ from the restatement"
    assert_same_structure(t, O.build(text, l2_bits=l2_bits, rate=rate))
