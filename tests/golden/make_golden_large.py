"""Golden checksums at BASELINE.json's full sizes, from the REAL reference.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_large.py C2 [C3u ...]

Imports ``wtindex`` 0.1.0 from /root/reference/pkg/src (the build container)
or, when that is absent, from the unmodified install in baseline/_ref (the GPU
box's host: C4 at n=2^32 needs ~100 GB of host RAM, more than the build
container has).  For each named config of ``large_cases.LARGE`` it builds the
text with the reference's own ``construct`` / ``construct_with_alphabet`` and
records into ``golden_large.json`` (merged per config):

* shape: n, sigma, levels, width, level sizes, per-level total_ones, cum_hist crc;
* per level crc32 of the bit-vector region words, l1 (<i8), l2 (<u2),
  one/zero samples (<i8) and node_rank0 (<i8); crc32 of all words;
* sha256 + length of the ``save()`` bytes (WTIDX001, the whole index);
* crc32 of the reference's answers to ``cli._bench_queries`` (cli.py:246-260)
  batches of ``query_num`` queries per kind through ``BatchRunner.run``, plus
  the full answers to the 64-bit edge queries (``large_cases.edge_queries``).

The tests never import the reference; they read only this file's output.
"""

from __future__ import annotations

import hashlib
import io
import json
import os
import resource
import sys
import time
import zlib

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, HERE)
if os.path.isdir("/root/reference/pkg/src"):
    sys.path.insert(0, "/root/reference/pkg/src")
    REF_FROM = "/root/reference/pkg/src"
else:
    sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
    REF_FROM = "baseline/_ref"

import wtindex as wt  # noqa: E402
import wtindex.cli as wcli  # noqa: E402

import large_cases as LC  # noqa: E402

OUT = os.path.join(HERE, "golden_large.json")


def crc(a, dt=None) -> str:
    a = np.ascontiguousarray(a if dt is None else np.asarray(a).astype(dt))
    return f"{zlib.crc32(memoryview(a).cast('B')):08x}"


def run(name: str, out_path: str) -> dict:
    t0 = time.time()
    text = LC.text_np(name)
    alpha = LC.alphabet_of(name)
    t_text = time.time() - t0
    t0 = time.time()
    workers = os.cpu_count() or 1
    if alpha is None:
        t = wt.construct(text, workers=workers)
    else:
        t = wt.construct_with_alphabet(text, alpha, workers=workers)
    t_build = time.time() - t0
    del text
    print(f"{name}: text {t_text:.1f}s build {t_build:.1f}s sigma={t.sigma}", flush=True)
    levels = []
    for l in range(t.num_levels):
        rs = t.rs[l]
        levels.append({
            "words": crc(t.bits.region_words(l), "<u8"),
            "l1": crc(rs.l1_counts, "<i8"), "l2": crc(rs.l2_counts, "<u2"),
            "ones": crc(rs.one_samples, "<i8"), "zeros": crc(rs.zero_samples, "<i8"),
            "n_ones_samples": int(len(rs.one_samples)),
            "n_zeros_samples": int(len(rs.zero_samples)),
            "node_rank0": crc(t.node_rank0[l], "<i8"),
        })
    buf = io.BytesIO()
    t.save(buf)
    raw = buf.getbuffer()
    save_sha = hashlib.sha256(raw).hexdigest()
    save_len = len(raw)
    del raw, buf
    hist = np.diff(t.cum_hist)
    queries = {}
    for kind, seed in LC.QUERY_SEEDS.items():
        num = LC.query_num(name)
        batch = wcli._bench_queries(t, kind, num, seed)
        # the restated generator must draw the very same queries
        syms, args = LC.bench_queries(t.n, hist, t.alphabet.sorted_symbols, kind, num, seed)
        assert np.array_equal(args, batch.args)
        assert (syms is None and batch.symbols is None) or np.array_equal(syms, batch.symbols)
        tq = time.time()
        res = wt.BatchRunner(t, workers=workers).run(batch)
        dt = time.time() - tq
        queries[kind] = {"seed": seed, "num": num, "crc": crc(res), "dtype": str(res.dtype),
                         "ref_seconds": round(dt, 3)}
        print(f"  {kind}: {num} in {dt:.1f}s crc {queries[kind]['crc']}", flush=True)
    acc, (rs_, rp), (ss, ks) = LC.edge_queries(t.n, hist, t.alphabet.sorted_symbols)
    edges = {
        "access_pos": acc.tolist(),
        "access": [int(t.access(int(i))) for i in acc],
        "rank_n": wt.rank_batch(t, rs_, rp).tolist(),
        "select_last": wt.select_batch(t, ss, ks).tolist(),
    }
    if len(edges["rank_n"]) > 1024:   # sigma = 2^16: keep checksums only
        edges["rank_n"] = crc(np.asarray(edges["rank_n"], np.int64))
        edges["select_last"] = crc(np.asarray(edges["select_last"], np.int64))
    rec = {
        "recipe": LC.LARGE[name], "reference": f"wtindex {wt.__version__} from {REF_FROM}",
        "ref_build_seconds": round(t_build, 1), "ref_workers": workers,
        "ref_peak_rss_gb": round(resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 2**20, 1),
        "n": int(t.n), "sigma": int(t.sigma), "levels": int(t.num_levels),
        "width": int(t.symbol_width),
        "level_sizes": [int(x) for x in t.level_sizes],
        "total_ones": [int(r.total_ones) for r in t.rs],
        "cum_hist_crc": crc(t.cum_hist, "<i8"),
        "hist_max": int(hist.max()), "present": int((hist > 0).sum()),
        "words_crc": crc(t.bits.words, "<u8"), "n_words": int(len(t.bits.words)),
        "per_level": levels, "save_sha256": save_sha, "save_len": save_len,
        "queries": queries, "edges": edges,
    }
    merged = {}
    if os.path.exists(out_path):
        with open(out_path) as f:
            merged = json.load(f)
    merged[name] = rec
    with open(out_path, "w") as f:
        json.dump(merged, f, indent=1, sort_keys=True)
    print(f"{name}: done, save {save_len} B sha {save_sha[:12]}", flush=True)
    return rec


if __name__ == "__main__":
    out = OUT
    names = sys.argv[1:]
    if names and names[0].startswith("--out="):
        out = names[0][6:]
        names = names[1:]
    for nm in names:
        run(nm, out)
