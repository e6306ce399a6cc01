#!/usr/bin/env python
"""Benchmark: wavelet-tree build + batched access/rank/select on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one batch of 1e8 mixed queries (equal thirds access / rank /
select, run as three kind-homogeneous batches exactly like the reference's
BatchRunner) per GPU against the C2 tree (n = 2^30 u8 symbols, sigma = 256),
inputs resident in HBM.  ``value`` = queries/s over all ranks (weak scaling:
every rank answers its own 1e8 against a replica broadcast from rank 0 over
NCCL).  The build of the C2 tree (single GPU, the other half of BASELINE.json's
metric) is timed on rank 0 over the same K/W and reported under "build".

``--impl reference`` times the reference itself (wtindex 0.1.0, installed
unmodified into baseline/_ref; the oracle port when that is absent) on all of
this host's cores for the same metric, on a bounded sample.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("build symbols/sec (GB/s vs HBM peak); "
          "access/rank/select queries/sec at 1/2/4/8 GPUs")
UNIT = "queries/s"

# SURVEY 8(d) random-access sector model, bytes per query for a sigma = 256 tree
# (L = 8): rank step = 64 B (L2 entry + bit sector), access final bit 32 B,
# select step = 96 B (sample + L2 + bit), I/O 16 B access / 24 B rank & select.
SECTOR_BYTES = {"access": 7 * 64 + 32 + 16, "rank": 8 * 64 + 24, "select": 8 * 96 + 24}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def build_alg_bytes(sizes, n, w, c, l2_bits=512, rate=4096):
    """Algorithmic bytes of one build: histogram read, per level
    input read + bit write, partitioned write for l >= 1, directories."""
    b = n * w
    for l, m in enumerate(sizes):
        b += m * ((w if l == 0 else c) + 1 / 8)
        if l >= 1:
            b += m * c
        b += 8 * -(-m // 65536) + 2 * -(-m // l2_bits) + 8 * m / rate
    return b


def level_alg_bytes(sizes, l, w, c, l2_bits=512, rate=4096):
    m = sizes[l]
    b = m * ((w if l == 0 else c) + 1 / 8)
    if l + 1 < len(sizes):
        b += sizes[l + 1] * c
    return b + 8 * -(-m // 65536) + 2 * -(-m // l2_bits) + 8 * m / rate


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()  # the timed region starts once the sampler is live
            while not self.rows and time.time() - t0 < 3.0:
                time.sleep(0.01)
            self.rows.clear()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            t0 = time.time()  # at least one sample from inside the region
            while not self.rows and time.time() - t0 < 1.0:
                time.sleep(0.01)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[4 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args):
    import ctypes as C

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    os.environ["WT_DEVICE"] = str(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2505_03372_b200 as W
    from paper_2505_03372_b200 import _lib

    dev = torch.device("cuda", local)
    n = 1 << args.n_log
    sigma = 256
    hbm, peak_kind = peaks()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---------------- build (rank 0: the single-GPU construction) ----------
    build = None
    tree = None
    text_np = None
    if rank == 0:
        text_np = np.random.default_rng(0).integers(0, sigma, n, dtype=np.uint8)  # C2 recipe
        text_dev = torch.from_numpy(text_np).to(dev)
        for _ in range(args.warmup):
            tree = W.construct(text_dev)
            del tree
        ms, lvl = [], []
        prof = (C.c_float * 32)()
        with Clocks(local) as clk_b:
            for _ in range(args.steps):
                tree = W.construct(text_dev)
                ms.append(tree.build_ms)
                _lib.lib.wt_tree_build_profile(tree.handle, prof, 32)
                lvl.append([prof[i] for i in range(1 + tree.num_levels)])
                if _ < args.steps - 1:
                    del tree
        sizes = [int(x) for x in tree.level_sizes]
        c = 1 if tree.num_levels <= 8 else 2
        t_ms = float(np.mean(ms))
        alg = build_alg_bytes(sizes, n, 1, c)
        lvl = np.mean(np.array(lvl), axis=0)
        dom = int(np.argmax(lvl[1:]))
        dom_alg = level_alg_bytes(sizes, dom, 1, c)
        build = {
            "symbols_per_s": n / (t_ms / 1e3), "ms": t_ms, "ms_all": ms,
            "GB_per_s": alg / (t_ms / 1e3) / 1e9, "alg_bytes": alg,
            "frac_of_hbm": alg / (t_ms / 1e3) / 1e9 / hbm,
            "n": n, "sigma": sigma, "levels": tree.num_levels,
            "ms_histogram_and_plan": float(lvl[0]),
            "ms_per_level": [float(x) for x in lvl[1:]],
            "dominant_kernel": {"name": f"wlevel_kernel (level {dom})", "ms": float(lvl[1 + dom]),
                                "alg_bytes": dom_alg,
                                "GB_per_s": dom_alg / (lvl[1 + dom] / 1e3) / 1e9},
            "clocks": clk_b.summary(),
        }
        del text_dev
        torch.cuda.empty_cache()

    # ---------------- replicate over NCCL --------------------------------------
    replicate = None
    if world > 1:
        from paper_2505_03372_b200 import parallel as par
        tree = par.replicate(tree if rank == 0 else None, device=local)
        replicate = {"ms": max_over_ranks(float(tree.replicate_ms)),
                     "bytes": int(tree.device_bytes)}
        replicate["GB_per_s"] = replicate["bytes"] / (replicate["ms"] / 1e3) / 1e9

    # ---------------- queries ---------------------------------------------------
    m_total = args.queries
    per = [m_total // 3 + (1 if i < m_total % 3 else 0) for i in range(3)]
    g = torch.Generator(device=dev)
    g.manual_seed(1234 + rank)
    occ = torch.from_numpy(np.diff(tree.cum_hist)).to(dev)
    syms = torch.from_numpy(tree.alphabet.sorted_symbols.astype(np.int64)).to(dev)
    present = torch.nonzero(occ > 0).flatten()
    # cli._bench_queries recipe (cli.py:246-260), generated on the device
    q_acc = torch.randint(0, n, (per[0],), generator=g, device=dev, dtype=torch.int64)
    rid = torch.randint(0, sigma, (per[1],), generator=g, device=dev, dtype=torch.int64)
    q_rsym = syms[rid]
    q_rpos = torch.randint(0, n + 1, (per[1],), generator=g, device=dev, dtype=torch.int64)
    sid = present[torch.randint(0, len(present), (per[2],), generator=g, device=dev)]
    q_ssym = syms[sid]
    q_ks = 1 + torch.floor(torch.rand(per[2], generator=g, device=dev, dtype=torch.float64)
                           * occ[sid]).to(torch.int64)
    q_ks = torch.minimum(q_ks, occ[sid])
    o_acc = torch.empty(per[0], dtype=torch.uint8, device=dev)
    o_rank = torch.empty(per[1], dtype=torch.int64, device=dev)
    o_sel = torch.empty(per[2], dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev)
    sptr = C.c_void_p(stream.cuda_stream)
    bad = C.c_int64(-1)
    flags = _lib.F_DEVICE_PTRS | _lib.F_SYMBOLS
    # device sort_queries_by_symbol (WT_F_SORT, the paper's query sorting):
    # every batch is sorted on the device by (symbol, coarse position /
    # ordinal) before the walk; the sort runs inside the timed region.
    sort_kinds = set() if args.no_sort else {"access", "rank", "select"}
    h = tree.handle
    batches = [("access", _lib.Q_ACCESS, None, q_acc, o_acc),
               ("rank", _lib.Q_RANK, q_rsym, q_rpos, o_rank),
               ("select", _lib.Q_SELECT, q_ssym, q_ks, o_sel)]
    kind_name = {b[1]: b[0] for b in batches}

    def launch(kind, ids, a, o):
        fl = flags | (_lib.F_SORT if kind_name[kind] in sort_kinds else 0)
        _lib.check(_lib.lib.wt_tree_query(h, kind, C.c_void_p(ids.data_ptr()) if ids is not None
                                          else None, C.c_void_p(a.data_ptr()),
                                          C.c_void_p(o.data_ptr()), a.numel(), 0, fl, sptr,
                                          C.byref(bad), None), "query")
        if bad.value != -1:
            raise RuntimeError(f"invalid query {bad.value}")

    for _ in range(args.warmup):
        for _, kind, ids, a, o in batches:
            launch(kind, ids, a, o)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    barrier()
    with Clocks(local) as clk:
        for s in range(args.steps):
            evs[s][0].record(stream)
            for j, (_, kind, ids, a, o) in enumerate(batches):
                launch(kind, ids, a, o)
                evs[s][j + 1].record(stream)
        barrier()
    step_ms = [e[0].elapsed_time(e[3]) for e in evs]
    kind_ms = {b[0]: float(np.mean([e[j].elapsed_time(e[j + 1]) for e in evs]))
               for j, b in enumerate(batches)}
    local_ms = float(np.mean(step_ms))
    ms_step = max_over_ranks(local_ms)
    value = world * m_total / (ms_step / 1e3)

    # correctness spot-check of this run's answers (size-independent)
    if rank == 0 and text_np is not None:
        k = min(per[0], 1 << 20)
        got = o_acc[:k].cpu().numpy()
        want = text_np[q_acc[:k].cpu().numpy()]
        assert np.array_equal(got, want), "access answers differ from the text"

    queries = {}
    for name, _, _, a, _ in batches:
        t = kind_ms[name]
        queries[name] = {"queries_per_s": a.numel() / (t / 1e3), "ms": t,
                         "sector_model_bytes_per_query": SECTOR_BYTES[name],
                         "model_GB_per_s": SECTOR_BYTES[name] * a.numel() / (t / 1e3) / 1e9}
    dom = max(kind_ms, key=kind_ms.get)
    dom_q = queries[dom]
    roofline = {"bound": "hbm", "kernel": f"{dom}_kernel",
                "achieved": dom_q["model_GB_per_s"], "peak": hbm, "unit": "GB/s",
                "frac": dom_q["model_GB_per_s"] / hbm, "peak_source": peak_kind,
                "traffic": traffic_from_profiles(f"{dom}_kernel", per[["access", "rank",
                                                                        "select"].index(dom)])}
    if roofline["traffic"]:
        # what the DRAM actually moved for this kind (ncu, profiles/ncu_traffic.json)
        roofline["dram_frac"] = roofline["traffic"] / (dom_q["ms"] / 1e3) / 1e9 / hbm
    roofline["note"] = ("achieved = SURVEY 8(d) sector-model bytes (every step one DRAM sector) / "
                        "the kind's batch time incl. the device sort; sorted batches reuse sectors "
                        "in L2, so frac can pass 1 -- dram_frac is the measured DRAM share")

    # ---------------- end to end through the public API -------------------------
    e2e = None
    if args.e2e:
        pin = lambda t: t.cpu().pin_memory().numpy()
        h_acc, h_rsym, h_rpos, h_ssym, h_ks = map(pin, (q_acc, q_rsym, q_rpos, q_ssym, q_ks))
        chunk = 1 << 21  # 16 chunks per kind: the copy-in / kernel / copy-out pipeline overlaps
        for _ in range(max(2, args.warmup)):  # also fills the pinned result-array cache
            ra = W.access_batch(tree, h_acc, chunk_size=chunk, sort="access" in sort_kinds)
            rr = W.rank_batch(tree, h_rsym, h_rpos, chunk_size=chunk, sort="rank" in sort_kinds)
            rs = W.select_batch(tree, h_ssym, h_ks, chunk_size=chunk, sort="select" in sort_kinds)
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            ra = W.access_batch(tree, h_acc, chunk_size=chunk, sort="access" in sort_kinds)
            rr = W.rank_batch(tree, h_rsym, h_rpos, chunk_size=chunk, sort="rank" in sort_kinds)
            rs = W.select_batch(tree, h_ssym, h_ks, chunk_size=chunk, sort="select" in sort_kinds)
        torch.cuda.synchronize()
        e2e_ms = max_over_ranks((time.perf_counter() - t0) * 1e3 / args.steps)
        assert np.array_equal(ra, o_acc.cpu().numpy()) and np.array_equal(rr, o_rank.cpu().numpy())
        assert np.array_equal(rs, o_sel.cpu().numpy())
        e2e = {"value": world * m_total / (e2e_ms / 1e3), "unit": UNIT, "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": int(per[0] * 8 + (per[1] + per[2]) * 16),
               "d2h_bytes_per_step": int(per[0] * 1 + (per[1] + per[2]) * 8),
               "api": "access_batch / rank_batch / select_batch on pinned numpy arrays"}
        # the bound: PCIe traffic, both directions at once (~70 GB/s measured on
        # the box, tools/e2e_probe.py)
        e2e["pcie_GB_per_s"] = (e2e["h2d_bytes_per_step"] + e2e["d2h_bytes_per_step"]) / (e2e_ms / 1e3) / 1e9

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(seconds=args.cpu_seconds)

    if world > 1:
        dist.barrier()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "int64", "data": "synthetic (seeded PCG64 C2 text; cli._bench_queries "
                                      "query recipe generated on device)",
            "config": {"workload": "C2/C5: n=2^%d u8 text, sigma=256; %d mixed "
                                   "access/rank/select queries per GPU per step "
                                   "(equal thirds, kind-homogeneous batches, each sorted on the "
                                   "device by symbol / position first)"
                                   % (args.n_log, m_total),
                       "n": n, "sigma": sigma, "queries_per_gpu": m_total,
                       "parallelism": f"replicas x{world} (NCCL broadcast)",
                       "l2": "inputs larger than L2 (tree %.2f GB, queries %.2f GB)"
                             % (tree.device_bytes / 1e9, m_total * 16 / 1e9)},
            "queries": queries, "build": build, "replicate": replicate,
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": args.steps * sum(6 if b[0] in sort_kinds else 1 for b in batches),
            "clocks": clk.summary(),
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def traffic_from_profiles(kernel: str, launch_queries: int):
    """dram bytes per launch from the committed ncu capture, scaled to this
    launch's query count (profiles/ncu_traffic.json), else None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            t = json.load(f)[kernel]
        return t["dram_bytes_per_query"] * launch_queries
    except Exception:
        return None


# ---------------------------------------------------------------------------
# CPU side: the reference itself (baseline/_ref), else the oracle port
# ---------------------------------------------------------------------------
_CPU = {}


def _reference_module():
    """The unmodified reference (wtindex 0.1.0) installed into baseline/_ref
    with pip; None when that install is absent."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "wtindex")):
        return None
    if ref not in sys.path:
        sys.path.insert(0, ref)
    import wtindex
    import wtindex.cli
    return wtindex


def _cpu_setup(n_log: int, num: int, seed: int):
    """Build the C2-recipe tree at n = 2^n_log and pre-generate `num` queries
    of each kind with the reference CLI's generator (cli.py:246-260)."""
    text = np.random.default_rng(0).integers(0, 256, 1 << n_log, dtype=np.uint8)
    wt = _reference_module()
    t0 = time.perf_counter()
    if wt is not None:
        tree = wt.construct(text)
        build_s = time.perf_counter() - t0
        qs = {k: wt.cli._bench_queries(tree, k, num, seed) for k in ("access", "rank", "select")}
        kind = "reference"
    else:
        import oracle as O
        tree = O.build(text)
        build_s = time.perf_counter() - t0
        qs = {k: O.bench_queries(tree.n, tree.hist, k, num, seed)
              for k in ("access", "rank", "select")}
        kind = "port"
    _CPU.update(tree=tree, qs=qs, kind=kind, wt=wt)
    return build_s, kind


def _cpu_worker(job):
    """Answer queries [lo, hi) of one kind; returns seconds."""
    kind, lo, hi = job
    tree, q, wt = _CPU["tree"], _CPU["qs"][kind], _CPU["wt"]
    t0 = time.perf_counter()
    if wt is not None:   # the reference's own batch path (batch.py:152-239)
        sub = wt.QueryBatch(kind, q.args[lo:hi], None if q.symbols is None else q.symbols[lo:hi])
        wt.BatchRunner(tree, sub.chunk_size, 1).run(sub)
    else:
        ids, args = q
        ids = None if ids is None else ids[lo:hi]
        if kind == "access":
            tree.access_ids(args[lo:hi])
        elif kind == "rank":
            tree.rank_ids(ids, args[lo:hi])
        else:
            tree.select_ids(ids, args[lo:hi])
    return time.perf_counter() - t0


def cpu_baseline(seconds: float = 20.0, n_log: int = 22):
    """Rank 0 at N=1: the reference on ONE host core, bounded sample."""
    n_q = 30000
    build_s, kind = _cpu_setup(n_log, n_q, 0)
    done, spent = 0, 0.0
    while spent < seconds * 0.5 and done < 3_000_000:
        for k in ("access", "rank", "select"):
            spent += _cpu_worker((k, 0, n_q))
            done += n_q
    what = ("wtindex 0.1.0 (the reference, baseline/_ref) access_batch/rank_batch/select_batch"
            if kind == "reference" else "oracle port (numpy restatement of wtindex)")
    return {"value": done / spent, "unit": UNIT, "cores": 1, "kind": kind,
            "sample": f"{what}, tree n=2^{n_log} sigma=256, {done} mixed queries in "
                      f"{n_q}-query kind-homogeneous batches, 1 process",
            "build_symbols_per_s": (1 << n_log) / build_s}


def run_reference(args):
    """--impl reference: the reference's CPU path on all host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import multiprocessing as mp
    n_log = args.ref_n_log
    procs = os.cpu_count() or 1
    per_proc = args.ref_queries_per_proc
    build_s, kind = _cpu_setup(n_log, procs * per_proc, 7)   # before the pool forks
    ctx = mp.get_context("fork")
    times = []
    with ctx.Pool(procs) as pool:
        for step in range(args.warmup + args.steps):
            jobs = [(k, p * per_proc, (p + 1) * per_proc)
                    for p in range(procs) for k in ("access", "rank", "select")]
            t0 = time.perf_counter()
            pool.map(_cpu_worker, jobs)
            dt = time.perf_counter() - t0
            if step >= args.warmup:
                times.append(dt)
    q = procs * per_proc * 3
    ms = float(np.mean(times)) * 1e3
    value = q / (ms / 1e3)
    what = ("wtindex 0.1.0, the unmodified reference installed in baseline/_ref, through "
            "BatchRunner.run" if kind == "reference" else
            "oracle port (numpy restatement of wtindex; baseline/_ref absent)")
    sample = (f"{what}; tree n=2^{n_log} sigma=256 (C2 recipe) built in {build_s:.1f}s; "
              f"{q} mixed queries per step (cli._bench_queries) over {procs} processes")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": int(os.environ.get("WORLD_SIZE", "1")), "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic (seeded PCG64, cli._bench_queries recipe)",
        "config": {"workload": f"C2 recipe at n=2^{n_log} (bounded CPU sample), mixed "
                               "access/rank/select", "n": 1 << n_log, "sigma": 256},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": procs, "kind": kind,
                         "sample": sample, "build_symbols_per_s": (1 << n_log) / build_s},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n-log", type=int, default=30)
    ap.add_argument("--queries", type=int, default=100_000_000)
    ap.add_argument("--no-e2e", dest="e2e", action="store_false")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-sort", action="store_true", help="no device query sorting")
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--ref-n-log", type=int, default=24)
    ap.add_argument("--ref-queries-per-proc", type=int, default=40000)
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
