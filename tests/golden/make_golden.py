"""Generate the golden vectors by running the REAL reference (wtindex 0.1.0).

Run in the build container (the reference only exists there):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``wtindex`` from /root/reference/pkg/src (read-only), builds every
case of ``cases.py`` through the reference's public API and records:

* ``golden.json``   -- per tree case: sha256 of ``save()`` bytes, level sizes,
  cum_hist crc, per-level total_ones, crc32 of every query answer array;
  per bit-vector case: sha256 of ``RankSelectIndex.write`` bytes and answer crcs;
* ``golden.npz``    -- the query answer arrays themselves (small cases) and the
  per-sigma code-table crcs for sigma in CODE_SIGMAS;
* ``save_<case>.bin`` -- full ``save()`` bytes of the small tree cases.

The GPU box never runs this file; the tests read only its outputs.
"""

from __future__ import annotations

import hashlib
import io
import json
import os
import sys
import zlib

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

import wtindex as wt  # noqa: E402
from wtindex.rankselect import RankSelectParams, build_index  # noqa: E402

import cases as C  # noqa: E402

NUM_Q = 400
SAVE_INLINE_MAX = 96 * 1024


def crc(a) -> str:
    return f"{zlib.crc32(np.ascontiguousarray(a).tobytes()):08x}"


def main():
    out = {"tree": {}, "bits": {}}
    arrays = {}
    for case in C.TREE_CASES:
        text = C.text_of(case)
        alpha = C.alphabet_of(case)
        params = RankSelectParams(l2_bits=case["l2_bits"], sample_rate=case["rate"])
        if alpha is None:
            t = wt.construct(text, params=params)
        else:
            t = wt.construct_with_alphabet(text, alpha, params=params)
        buf = io.BytesIO()
        t.save(buf)
        raw = buf.getvalue()
        hist = np.diff(t.cum_hist)
        acc, (rsym, rpos), (ssym, ks) = C.queries_of(
            t.n, hist, t.alphabet.sorted_symbols, case.get("qseed", 7), NUM_Q)
        name = case["name"]
        quirks = {}
        try:
            a = wt.access_batch(t, acc)
        except IndexError as e:
            # reference quirk: access_ids_bulk indexes an empty level region
            # (rankselect.py:146) -- record it and take the scalar answers.
            quirks["access_batch_raises"] = f"IndexError: {e}"
            a = np.array([t.access(int(i)) for i in acc], t.alphabet.sorted_symbols.dtype)
        r = wt.rank_batch(t, rsym, rpos)
        s = wt.select_batch(t, ssym, ks)
        rec = {
            "quirks": quirks,
            "save_sha256": hashlib.sha256(raw).hexdigest(),
            "save_len": len(raw),
            "sigma": int(t.sigma), "levels": int(t.num_levels),
            "width": int(t.symbol_width),
            "level_sizes": [int(x) for x in t.level_sizes],
            "total_ones": [int(rs.total_ones) for rs in t.rs],
            "cum_hist_crc": crc(t.cum_hist.astype("<u8")),
            "words_crc": crc(t.bits.words.astype("<u8")),
            "n_words": int(len(t.bits.words)),
            "access_crc": crc(a), "rank_crc": crc(r), "select_crc": crc(s),
            "access_dtype": str(a.dtype),
        }
        if len(raw) <= SAVE_INLINE_MAX:
            with open(os.path.join(HERE, f"save_{name}.bin"), "wb") as f:
                f.write(raw)
            rec["save_file"] = f"save_{name}.bin"
        arrays[f"{name}__access"] = a
        arrays[f"{name}__rank"] = r
        arrays[f"{name}__select"] = s
        out["tree"][name] = rec
        print(name, rec["save_len"], rec["save_sha256"][:12])

    for case in C.BITS_CASES:
        bits = C.bits_of(case)
        ba = wt.build_bit_array([len(bits)])
        if len(bits):
            ba.fill_region(0, bits)
        params = RankSelectParams(l2_bits=case["l2_bits"], sample_rate=case["rate"])
        idx = build_index(ba, 0, params)
        buf = io.BytesIO()
        idx.write(buf)
        rng = np.random.default_rng(case["seed"] + 1)
        n = len(bits)
        pos = rng.integers(0, n + 1, 300)
        r1 = idx.rank1_bulk(pos)
        k1 = rng.integers(1, idx.total_ones + 1, 300) if idx.total_ones else np.zeros(0, np.int64)
        nz = n - idx.total_ones
        k0 = rng.integers(1, nz + 1, 300) if nz else np.zeros(0, np.int64)
        s1 = idx.select1_bulk(k1)
        s0 = idx.select0_bulk(k0)
        out["bits"][case["name"]] = {
            "rs_sha256": hashlib.sha256(buf.getvalue()).hexdigest(),
            "words_crc": crc(ba.words.astype("<u8")),
            "rank_crc": crc(r1), "select1_crc": crc(s1), "select0_crc": crc(s0),
            "total_ones": int(idx.total_ones),
        }
        print(case["name"], out["bits"][case["name"]]["rs_sha256"][:12])

    code_crc = np.zeros(len(C.CODE_SIGMAS), np.uint32)
    code_first = np.zeros(len(C.CODE_SIGMAS), np.int64)
    for i, s in enumerate(C.CODE_SIGMAS):
        ct = wt.create_codes(s)
        code_crc[i] = zlib.crc32(ct.values.astype("<u2").tobytes() + ct.lens.astype("u1").tobytes())
        code_first[i] = ct.first_coded
    arrays["code_sigmas"] = np.asarray(C.CODE_SIGMAS, np.int64)
    arrays["code_crc"] = code_crc
    arrays["code_first"] = code_first

    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)


if __name__ == "__main__":
    main()
