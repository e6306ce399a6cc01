"""Pin the oracle (oracle/wt_oracle.py) to the real reference's golden vectors.

Every vector in tests/golden/ was produced by running the reference itself
(tests/golden/make_golden.py).  CPU only.
"""

import hashlib
import json
import os
import zlib

import numpy as np
import pytest

import cases as C
import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")
G = json.load(open(os.path.join(GOLD, "golden.json")))
NPZ = np.load(os.path.join(GOLD, "golden.npz"))


def crc(a):
    return f"{zlib.crc32(np.ascontiguousarray(a).tobytes()):08x}"


def oracle_tree(case):
    text = C.text_of(case)
    alpha = C.alphabet_of(case)
    if alpha is None:
        return O.build(text, case["l2_bits"], case["rate"])
    return O.build_with_alphabet(text, alpha, case["l2_bits"], case["rate"])


@pytest.mark.parametrize("case", C.TREE_CASES, ids=[c["name"] for c in C.TREE_CASES])
def test_tree_case_matches_reference(case):
    g = G["tree"][case["name"]]
    t = oracle_tree(case)
    assert t.sizes.tolist() == g["level_sizes"]
    assert [d["total_ones"] for d in t.dirs] == g["total_ones"]
    assert crc(t.words.astype("<u8")) == g["words_crc"]
    raw = t.save_bytes()
    if "save_file" in g:
        want = open(os.path.join(GOLD, g["save_file"]), "rb").read()
        assert raw == want
    assert hashlib.sha256(raw).hexdigest() == g["save_sha256"]
    # queries through the tree-walking restatement (Alg. 5-8)
    acc, (rsym, rpos), (ssym, ks) = C.queries_of(t.n, t.hist, t.symbols, 7, 400)
    rid = np.searchsorted(t.symbols, rsym)
    sid = np.searchsorted(t.symbols, ssym)
    a = t.symbols[t.access_ids(acc)]
    r = t.rank_ids(rid, rpos)
    s = t.select_ids(sid, ks)
    assert np.array_equal(a, NPZ[case["name"] + "__access"])
    assert str(a.dtype) == g["access_dtype"]
    assert np.array_equal(r, NPZ[case["name"] + "__rank"])
    assert np.array_equal(s, NPZ[case["name"] + "__select"])
    # and the definition-level answers agree
    ids_text = np.searchsorted(t.symbols, np.frombuffer(C.text_of(case), np.uint8)
                               if isinstance(C.text_of(case), bytes) else C.text_of(case))
    fa, fr, fs = O.text_answers(ids_text, t.sigma)
    assert np.array_equal(t.symbols[fa(acc)], a)
    assert np.array_equal(fr(rid, rpos), r)
    assert np.array_equal(fs(sid, ks), s)


@pytest.mark.parametrize("case", C.BITS_CASES, ids=[c["name"] for c in C.BITS_CASES])
def test_bit_directory_matches_reference(case):
    import io
    import struct
    g = G["bits"][case["name"]]
    bits = C.bits_of(case)
    d = O.directory(bits, case["l2_bits"], case["rate"])
    buf = io.BytesIO()
    buf.write(struct.pack("<IIIQQ", O.L1_BITS, case["l2_bits"], case["rate"],
                          d["n_bits"], d["total_ones"]))
    for arr, code in ((d["l1"], "<u8"), (d["l2"], "<u2"), (d["ones"], "<u8"), (d["zeros"], "<u8")):
        buf.write(struct.pack("<Q", len(arr)) + arr.astype(code).tobytes())
    assert hashlib.sha256(buf.getvalue()).hexdigest() == g["rs_sha256"]
    packed = np.packbits(bits, bitorder="little")
    packed = np.concatenate([packed, np.zeros(-len(packed) % 8, np.uint8)])
    assert crc(packed.view("<u8")) == g["words_crc"]


def test_code_tables_match_reference():
    sig = NPZ["code_sigmas"]
    for i, s in enumerate(sig.tolist()):
        v, l, first = O.tree_codes(s)
        got = zlib.crc32(v.astype("<u2").tobytes() + l.astype("u1").tobytes())
        assert got == int(NPZ["code_crc"][i]), s
        assert first == int(NPZ["code_first"][i]), s


def test_worked_example_known_answers():
    # test_wtree.py:41-53 / test_acceptance.py:38-47
    t = O.build(b"dbdcaacbcd")
    assert t.cum.tolist() == [0, 2, 4, 7, 10]
    lv0 = [int(t.words[0] >> j & 1) for j in range(10)]
    assert lv0 == [1, 0, 1, 1, 0, 0, 1, 0, 1, 1]
    w1 = int(t.words[int(t.offsets[1]) >> 6])
    assert [w1 >> j & 1 for j in range(10)] == [1, 0, 0, 1, 1, 1, 0, 0, 0, 1]
    c = int(np.searchsorted(t.symbols, ord("c")))
    assert t.symbols[t.access_ids([6])][0] == ord("c")
    assert t.rank_ids([c], [6])[0] == 1
    assert t.select_ids([c], [2])[0] == 6


def test_bit_level_known_answers():
    # test_rankselect.py:69-77: bits 1011001011 -> rank1(6)=3, select1(4)=6
    bits = np.array([1, 0, 1, 1, 0, 0, 1, 0, 1, 1], np.uint8)
    d = O.directory(bits, 512, 16384)
    packed = np.packbits(bits, bitorder="little")
    w = np.concatenate([packed, np.zeros(6, np.uint8)]).view("<u8")
    lv = O.wt_oracle._Level(w, d, 512, 16384)
    assert lv.rank1(np.array([6]))[0] == 3
    assert lv.select(np.array([4]), True)[0] == 6
    # all-zeros samples at 16384k-1 (test_rankselect.py:36-44)
    z = O.directory(np.zeros(65536 * 2, np.uint8), 512, 16384)
    assert z["zeros"].tolist() == [16384 * k - 1 for k in range(1, 9)]
    # all-ones L2 (test_rankselect.py:47-55)
    o = O.directory(np.ones(2048, np.uint8), 512, 16384)
    assert o["l2"].tolist() == [0, 512, 1024, 1536]
