"""Seeded input recipes shared by the golden generator and the parity tests.

Nothing here imports the reference: texts and query sets are regenerated
from (recipe, seed) with numpy's PCG64, which is bit-stable across hosts.
"""

from __future__ import annotations

import numpy as np


def text_of(case: dict) -> np.ndarray | bytes:
    kind = case["kind"]
    if kind == "bytes":
        return case["data"].encode("latin-1")
    rng = np.random.default_rng(case["seed"])
    n = case["n"]
    dt = np.uint16 if case.get("dtype") == "u16" else np.uint8
    if kind == "uniform":
        return rng.integers(case.get("lo", 0), case["sigma"], n).astype(dt)
    if kind == "zipf":
        return (np.minimum(rng.zipf(case.get("a", 1.2), n), case["sigma"]) - 1).astype(dt)
    if kind == "dna":
        return np.frombuffer(b"ACGT", np.uint8)[rng.integers(0, 4, n)]
    if kind == "sparse":   # few distinct symbols spread over a wide value range
        vals = np.sort(rng.choice(case["range"], case["sigma"], replace=False))
        return vals[rng.integers(0, case["sigma"], n)].astype(dt)
    raise ValueError(kind)


def alphabet_of(case: dict):
    a = case.get("alphabet")
    if a is None:
        return None
    if isinstance(a, str):
        return a.encode("latin-1")
    if isinstance(a, dict):      # {"arange": k, "dtype": ...}
        dt = np.uint16 if a.get("dtype") == "u16" else np.uint8
        return np.arange(a["arange"], dtype=dt)
    return np.asarray(a)


def queries_of(n: int, hist: np.ndarray, sorted_symbols: np.ndarray, seed: int, num: int):
    """(access positions, rank symbols+positions, select symbols+ordinals),
    following the reference CLI generator (cli.py:246-260), in original symbols."""
    rng = np.random.default_rng(seed)
    sigma = len(hist)
    acc = rng.integers(0, n, num)
    rids = rng.integers(0, sigma, num)
    rsym = sorted_symbols[rids].astype(np.int64)
    rpos = rng.integers(0, n + 1, num)
    present = np.flatnonzero(hist > 0)
    sids = present[rng.integers(0, len(present), num)]
    ks = 1 + np.floor(rng.random(num) * hist[sids]).astype(np.int64)
    ssym = sorted_symbols[sids].astype(np.int64)
    # always include the edges the reference tests poke at
    acc = np.concatenate([acc, [0, n - 1]])
    rsym = np.concatenate([rsym, rsym[:1], rsym[:1]])
    rpos = np.concatenate([rpos, [0, n]])
    ssym = np.concatenate([ssym, ssym[:1]])
    ks = np.concatenate([ks, [int(hist[sids[0]])]])
    return acc, (rsym, rpos), (ssym, ks)


def bits_of(case: dict) -> np.ndarray:
    """Bit-vector recipes of the reference tests (helpers.py:19-42)."""
    rng = np.random.default_rng(case["seed"])
    n = case["n"]
    if case["kind"] == "uniform_bits":
        return (rng.random(n) < case["fill"]).astype(np.uint8)
    if case["kind"] == "adversarial_bits":
        pct = case["fill_pct"]
        total = n * pct // 100
        tail_start = n - n * pct // 100
        tail = total * 99 // 100
        head = total - tail
        bits = np.zeros(n, np.uint8)
        tp = rng.choice(n - tail_start, size=min(tail, n - tail_start), replace=False)
        bits[tail_start + tp] = 1
        if tail_start > 0 and head:
            hp = rng.choice(tail_start, size=min(head, tail_start), replace=False)
            bits[hp] = 1
        return bits
    if case["kind"] == "const_bits":
        return np.full(n, case["value"], np.uint8)
    raise ValueError(case["kind"])


# ---------------------------------------------------------------------------
# the case lists
# ---------------------------------------------------------------------------

TREE_CASES: list[dict] = []


def _add(name, **kw):
    kw.setdefault("l2_bits", 512)
    kw.setdefault("rate", 4096)
    TREE_CASES.append({"name": name, **kw})


_add("worked_example", kind="bytes", data="dbdcaacbcd")
_add("single_symbol", kind="bytes", data="zzzzzzzzz")
_add("declared_superset", kind="bytes", data="eeee", alphabet="abcde")
_add("declared_gap", kind="bytes", data="acca", alphabet="abcdefg")
for i, s in enumerate((2, 3, 4, 5, 6, 7, 8, 11, 13, 25, 31, 243, 256)):
    _add(f"u8_s{s}", kind="uniform", sigma=s, n=1000 + 37 * i, seed=100 + i)
for i, n in enumerate((1, 63, 64, 65, 511, 512, 513, 65535, 65536, 65537, 1 << 20)):
    _add(f"bin_n{n}", kind="uniform", sigma=2, n=n, seed=200 + i)
for i, (l2, rate) in enumerate(((64, 16), (128, 100), (2048, 1), (65536, 16384), (512, 3))):
    _add(f"params_l2{l2}_r{rate}", kind="uniform", sigma=6, n=150_000, seed=300 + i,
         l2_bits=l2, rate=rate)
_add("u16_s4096", kind="uniform", sigma=4096, n=5000, seed=400, dtype="u16")
_add("u16_s65536", kind="uniform", sigma=65536, n=1 << 18, seed=401, dtype="u16")
_add("u16_zipf_inferred", kind="zipf", sigma=65536, n=1 << 18, seed=402, dtype="u16")
_add("u16_zipf_declared", kind="zipf", sigma=65536, n=1 << 17, seed=403, dtype="u16",
     alphabet={"arange": 65536, "dtype": "u16"})
_add("u16_sparse", kind="sparse", sigma=1000, range=65536, n=50_000, seed=404, dtype="u16")
_add("u8_text_u16_alphabet", kind="uniform", sigma=200, n=20_000, seed=405,
     alphabet={"arange": 300, "dtype": "u16"})
_add("dna", kind="dna", n=1 << 20, seed=406)
_add("c1_u8_s256", kind="uniform", sigma=256, n=1 << 20, seed=0)
_add("u8_zipf", kind="zipf", sigma=256, n=300_000, seed=407)
_add("u8_lo_skip", kind="uniform", sigma=256, lo=250, n=70_000, seed=408)

BITS_CASES: list[dict] = []
for i, (n, fill) in enumerate(((1, 1.0), (4096, 0.5), (65536 * 3 + 17, 0.5),
                               (1_000_003, 0.01), (1_000_003, 0.99), (200_000, 0.5))):
    for l2, rate in ((512, 16384), (64, 16), (128, 100)):
        BITS_CASES.append({"name": f"uni_{n}_{fill}_{l2}_{rate}", "kind": "uniform_bits",
                           "n": n, "fill": fill, "seed": 500 + i, "l2_bits": l2, "rate": rate})
for i, pct in enumerate((1, 10, 50)):
    BITS_CASES.append({"name": f"adv_{pct}", "kind": "adversarial_bits", "n": 1_000_000,
                       "fill_pct": pct, "seed": 600 + i, "l2_bits": 512, "rate": 16384})
BITS_CASES.append({"name": "zeros", "kind": "const_bits", "n": 65536 * 2 + 5, "value": 0,
                   "seed": 0, "l2_bits": 512, "rate": 16384})
BITS_CASES.append({"name": "ones", "kind": "const_bits", "n": 2048, "value": 1,
                   "seed": 0, "l2_bits": 512, "rate": 16384})

CODE_SIGMAS = list(range(1, 4097)) + [5000, 38158, 40000, 65535, 65536]
