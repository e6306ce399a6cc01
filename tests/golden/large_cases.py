"""Seeded recipes of BASELINE.json's configurations at their full sizes.

Shared by ``make_golden_large.py`` (which runs the REAL reference on them and
records checksums) and the ``-m gpu`` parity tests / ``bench.py`` (which build
the same texts on the B200 and compare).  Nothing here imports the reference.

| name        | BASELINE config | text                                              |
|-------------|-----------------|---------------------------------------------------|
| C1          | configs[0]      | u8, n=2^20, uniform over 256 (numpy PCG64 seed 0) |
| C2          | configs[1]      | u8, n=2^30, uniform over 256 (numpy PCG64 seed 0) |
| C3u         | configs[2]      | u16, n=2^30, uniform over 2^16 (PCG64 seed 0)     |
| C3z         | configs[2]      | u16, n=2^30, Zipf(1.2) ranks truncated at 2^16, declared alphabet arange(2^16) |
| C3z_inf     | configs[2]      | the C3z text, alphabet inferred                   |
| C3r         | configs[2]      | u16, n=2^30, Zipf(1.2) ranks truncated at 38,158: inferred sigma 38,158 -> reduced (non power-of-two) codes, 16 levels |
| C4          | configs[3]      | u8 DNA "ACGT", n=2^32 (PCG64 seed 0, uint8 draws) |

The Zipf texts are NOT drawn with ``numpy.random.Generator.zipf``: that
sampler runs ~190 ns per symbol (200 s for 2^30 on one core), too slow for a
test.  They use a counter-based generator instead, identical on CPU (numpy,
torch) and on the GPU (torch): symbol i = inverse-CDF of the truncated Zipf(1.2)
law (``zipf_cdf``) at u_i = top 53 bits of splitmix64(seed, i) / 2^53.  At
n=2^30 every one of the 65,536 symbols occurs (the rarest expects ~300
occurrences), so C3z's inferred alphabet is the full 2^16 and reduced codes at
this size need the narrower C3r law.
"""

from __future__ import annotations

import numpy as np

GOLDEN = 0x9E3779B97F4A7C15
M1 = 0xBF58476D1CE4E5B9
M2 = 0x94D049BB133111EB
ZIPF_A = 1.2

LARGE = {
    "C1": {"kind": "uniform", "n_log": 20, "sigma": 256, "dtype": "u8", "seed": 0},
    "C2": {"kind": "uniform", "n_log": 30, "sigma": 256, "dtype": "u8", "seed": 0},
    "C3u": {"kind": "uniform", "n_log": 30, "sigma": 65536, "dtype": "u16", "seed": 0},
    "C3z": {"kind": "zipf", "n_log": 30, "sigma": 65536, "dtype": "u16", "seed": 3,
            "declared": True},
    "C3z_inf": {"kind": "zipf", "n_log": 30, "sigma": 65536, "dtype": "u16", "seed": 3},
    "C3r": {"kind": "zipf", "n_log": 30, "sigma": 38158, "dtype": "u16", "seed": 4},
    "C4": {"kind": "dna", "n_log": 32, "sigma": 4, "dtype": "u8", "seed": 0},
}

# query sets per config: cli._bench_queries (cli.py:246-260) with these seeds
QUERY_NUM = {"C1": 100_000}
QUERY_NUM_DEFAULT = 1_000_000
QUERY_SEEDS = {"access": 11, "rank": 12, "select": 13}


def query_num(name: str) -> int:
    return QUERY_NUM.get(name, QUERY_NUM_DEFAULT)


def zipf_cdf(sigma: int, a: float = ZIPF_A) -> np.ndarray:
    """float64 P(X <= k) for k = 1 .. sigma-1 of Zipf(a) on 1, 2, ...;
    the mass above sigma-1 goes to the last symbol (the ``min(zipf, sigma)``
    truncation of SURVEY 8(d))."""
    from scipy.special import zeta
    k = np.arange(1, sigma, dtype=np.float64)
    return np.cumsum(k ** -a) / zeta(a)


def splitmix_np(seed: int, lo: int, hi: int) -> np.ndarray:
    """uint64 splitmix64 outputs for counters [lo, hi) of stream `seed`."""
    with np.errstate(over="ignore"):
        x = (np.arange(lo, hi, dtype=np.uint64) + np.uint64(1)) * np.uint64(GOLDEN) \
            + np.uint64((seed * 0x632BE59BD9B4E019) & 0xFFFFFFFFFFFFFFFF)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(M1)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(M2)
        return x ^ (x >> np.uint64(31))


def _i64(c: int) -> int:
    c &= 0xFFFFFFFFFFFFFFFF
    return c - (1 << 64) if c >= 1 << 63 else c


def splitmix_torch(seed: int, lo: int, hi: int, device):
    """Same as splitmix_np in torch int64 (two's-complement wrap; logical
    shifts by masking)."""
    import torch

    def shr(v, s):
        return (v >> s) & ((1 << (64 - s)) - 1)

    x = torch.arange(lo + 1, hi + 1, dtype=torch.int64, device=device)
    x = x * _i64(GOLDEN) + _i64(seed * 0x632BE59BD9B4E019)
    x = (x ^ shr(x, 30)) * _i64(M1)
    x = (x ^ shr(x, 27)) * _i64(M2)
    return x ^ shr(x, 31)


def zipf_np(seed: int, sigma: int, lo: int, hi: int, cdf=None) -> np.ndarray:
    cdf = zipf_cdf(sigma) if cdf is None else cdf
    u = (splitmix_np(seed, lo, hi) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    return np.searchsorted(cdf, u, side="right").astype(np.uint16)


def zipf_torch(seed: int, sigma: int, n: int, device, chunk: int = 1 << 26):
    import torch
    cdf = torch.from_numpy(zipf_cdf(sigma)).to(device)
    out = torch.empty(n, dtype=torch.int16, device=device)
    for lo in range(0, n, chunk):
        hi = min(n, lo + chunk)
        z = splitmix_torch(seed, lo, hi, device)
        u = ((z >> 11) & ((1 << 53) - 1)).to(torch.float64) * 2.0 ** -53
        s = torch.searchsorted(cdf, u, right=True)
        # values < 2^16 as the int16 holding the same u16 bit pattern: shift
        # into int16's range first (a CUDA int32 -> int16 cast saturates)
        out[lo:hi] = torch.where(s >= 32768, s - 65536, s).to(torch.int16)
    return out


def text_np(name: str) -> np.ndarray:
    """The config's text as a host numpy array (CPU)."""
    c = LARGE[name]
    n = 1 << c["n_log"]
    if c["kind"] == "uniform":
        dt = np.uint16 if c["dtype"] == "u16" else np.uint8
        return np.random.default_rng(c["seed"]).integers(0, c["sigma"], n, dtype=dt)
    if c["kind"] == "dna":
        lut = np.frombuffer(b"ACGT", np.uint8)
        return lut[np.random.default_rng(c["seed"]).integers(0, 4, n, dtype=np.uint8)]
    if c["kind"] == "zipf":
        import torch
        return zipf_torch(c["seed"], c["sigma"], n, "cpu").numpy().view(np.uint16)
    raise ValueError(c["kind"])


def text_device(name: str, device):
    """The config's text as a torch tensor on `device` (u8, or int16 holding
    u16 bit patterns).  Uniform / DNA texts come from numpy (the same PCG64
    stream as text_np); Zipf texts are generated on the device."""
    import torch
    c = LARGE[name]
    if c["kind"] == "zipf":
        return zipf_torch(c["seed"], c["sigma"], 1 << c["n_log"], device)
    a = text_np(name)
    if a.dtype == np.uint16:
        a = a.view(np.int16)
    return torch.from_numpy(a).to(device)


def alphabet_of(name: str):
    c = LARGE[name]
    if c.get("declared"):
        return np.arange(c["sigma"], dtype=np.uint16 if c["dtype"] == "u16" else np.uint8)
    return None


def bench_queries(n: int, hist: np.ndarray, sorted_symbols: np.ndarray, kind: str,
                  num: int, seed: int):
    """cli._bench_queries (cli.py:246-260) restated: (symbols or None, args)
    in original symbols, the reference CLI's exact draws."""
    rng = np.random.default_rng(seed)
    sigma = len(hist)
    if kind == "access":
        return None, rng.integers(0, n, num)
    if kind == "rank":
        ids = rng.integers(0, sigma, num)
        syms = sorted_symbols[ids].astype(np.int64)
        return syms, rng.integers(0, n + 1, num)
    present = np.flatnonzero(hist > 0)
    ids = present[rng.integers(0, len(present), num)]
    ks = 1 + np.floor(rng.random(num) * hist[ids]).astype(np.int64)
    return sorted_symbols[ids].astype(np.int64), ks


def edge_queries(n: int, hist: np.ndarray, sorted_symbols: np.ndarray):
    """rank(c, n) and select(c, occ(c)) for every present symbol c (the 64-bit
    edges: at C4 rank(c, n) counts past 2^30 and positions pass 2^32), plus
    access at 0, n-1 and around every 2^32 boundary below n."""
    present = np.flatnonzero(hist > 0)
    syms = sorted_symbols[present].astype(np.int64)
    acc = [0, n - 1]
    if n > 1 << 31:
        acc += [(1 << 31) - 1, 1 << 31]
    b = 1 << 32
    while b < n:
        acc += [b - 1, b]
        b += 1 << 32
    acc += [n // 2, n - 2] if n > 2 else []
    return (np.asarray(acc, np.int64), (syms, np.full(len(syms), n, np.int64)),
            (syms, hist[present].astype(np.int64)))
