#!/usr/bin/env python
"""Benchmark: wavelet-tree build + batched access/rank/select on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one batch of 1e8 mixed queries per GPU (equal thirds access /
rank / select, run as three kind-homogeneous batches exactly like the
reference's BatchRunner, each sorted on the device first) against the C2 tree
(BASELINE.json configs[1]: n = 2^30 u8 symbols, sigma = 256), inputs resident
in HBM.  ``value`` = queries/s over all ranks (weak scaling: every rank
answers its own 1e8 against a replica broadcast from rank 0 over NCCL).

Beside the headline the line carries:

* ``build``  -- the C2 build (single GPU, the other half of BASELINE.json's
  metric) timed over the same K / W on rank 0;
* ``builds`` -- C3u, C3z (declared 2^16), C3z_inf, C3r (reduced codes) and C4
  (n = 2^32 DNA) builds on rank 0 (configs[2], configs[3]);
* ``c5``     -- configs[4]: 1e9 mixed queries per step split over the N GPUs
  (strong scaling);
* ``roofline`` -- the dominant kernel of the step (the sorted select walk),
  algorithmic bytes / its CUDA-event time;
* ``e2e``    -- the same queries through the public API
  (access_batch / rank_batch / select_batch) from pinned host arrays;
* ``cpu_baseline`` -- the unmodified reference (baseline/_ref) answering a
  bounded sample of the same C2 workload on one host core: the tree is the
  GPU-built index, saved in the reference's own WTIDX001 format and loaded by
  ``wtindex.load`` (byte-identical to the reference's own build of this text,
  tests/test_configs_gpu.py); its answers are checked against ours.

``--gpus N`` without a torchrun environment re-launches itself under
``torch.distributed.run`` with N ranks (one per GPU).  ``--impl reference``
times the unmodified reference on this host's cores for the same metric and
config: it builds the C2 tree with ``wtindex.construct(workers=nproc)`` and
answers bounded query samples in nproc processes; under torchrun only rank 0
runs it.  ``--dry-run`` exercises the launcher and the max-over-ranks timing
on CPU (gloo) for the tests.
"""

from __future__ import annotations

import argparse
import gc
import io
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

METRIC = ("build symbols/sec (GB/s vs HBM peak); "
          "access/rank/select queries/sec at 1/2/4/8 GPUs")
UNIT = "queries/s"
KINDS = ("access", "rank", "select")

# SURVEY 8(d) random-access sector model, bytes per query for a sigma = 256 tree
# (L = 8): rank step = 64 B (L2 entry + bit sector), access final bit 32 B,
# select step = 96 B (sample + L2 + bit), I/O 16 B access / 24 B rank & select.
SECTOR_BYTES = {"access": 7 * 64 + 32 + 16, "rank": 8 * 64 + 24, "select": 8 * 96 + 24}


_T0 = time.time()


def log(msg: str) -> None:
    """Progress on stderr (the JSON line alone goes to stdout)."""
    print(f"[bench {time.time() - _T0:7.1f}s] {msg}", file=sys.stderr, flush=True)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


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


def sorted_walk_alg_bytes(kind, q, n_bits_levels, width=1):
    """Algorithmic bytes of one walk over a SORTED batch of q queries
    (DESIGN.md 5): each level's touched 32-byte rank lines are read at most
    once -- min(q lines, all lines of the level) -- plus, for select, the line
    samples (one u32 per 64 ones / zeros), plus the batch I/O (8-byte packed
    arguments in, results out)."""
    b = 0.0
    for nb in n_bits_levels:
        lines = -(-nb // 192)
        b += min(q, lines) * 32
        if kind == "select":
            b += min(q * 4, (nb // 64) * 4)
    out = width if kind == "access" else 8
    return b + q * (8 + out)


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


def workload_config(args, world):
    """The config dict both arms print (identical, so the driver compares
    like with like)."""
    return {"workload": "C2/C5: n=2^%d u8 text, sigma=256; %d mixed access/rank/select "
                        "queries per GPU per step (equal thirds, kind-homogeneous batches, "
                        "each sorted on the device by symbol / position first)"
                        % (args.n_log, args.queries),
            "n": 1 << args.n_log, "sigma": 256, "queries_per_gpu": args.queries,
            "parallelism": f"replicas x{world} (NCCL broadcast)",
            "l2": "inputs larger than L2 (the C2 tree is 3.6 GB on the device, the "
                  "queries 1.6 GB per GPU; L2 is 126 MB)"}


# ---------------------------------------------------------------------------
# launcher
# ---------------------------------------------------------------------------
def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def maybe_relaunch(args) -> None:
    """--gpus N > 1 outside torchrun: re-exec under torch.distributed.run with
    N ranks on this node (one process per GPU)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def _dist_setup(dry: bool):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if not dry:
        torch.cuda.set_device(local)
        os.environ["WT_DEVICE"] = str(local)
    if world > 1:
        if dry:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def run_dry(args):
    """CPU (gloo) pass through the launcher, the barrier and max-over-ranks."""
    import torch.distributed as dist
    world, rank, _ = _dist_setup(True)
    from paper_2505_03372_b200 import parallel as par
    t0 = time.perf_counter()
    for _ in range(args.warmup + args.steps):
        if world > 1:
            dist.barrier()
    ms = par.max_over_ranks((time.perf_counter() - t0) * 1e3 / max(1, args.steps))
    seen = par.max_over_ranks(rank) + 1
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": 0.0, "unit": UNIT, "n_gpus": world,
                          "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                          "dry_run": True, "ranks_seen": seen}))
    if world > 1:
        dist.destroy_process_group()


def _build_timed(W, text_dev, alpha, steps, warmup):
    """(tree of the last step, [ms per build], [per-phase ms]) -- device time
    of every build from the CUDA events inside wt_construct."""
    import ctypes as C
    from paper_2505_03372_b200 import _lib
    mk = (lambda: W.construct(text_dev)) if alpha is None else \
        (lambda: W.construct_with_alphabet(text_dev, alpha))
    # each replaced tree is collected before the next build: a WaveletTree
    # sits in a reference cycle (its lazy rank/select views), so without the
    # collect several trees' device arrays pile up and a later build waits on
    # the memory pool growing (seen: 57 ms .. 1.6 s pre-phases)
    tree = None
    for _ in range(warmup):
        tree = mk()
        del tree
        gc.collect()
    ms, lvl = [], []
    prof = (C.c_float * 32)()
    for s in range(steps):
        tree = mk()
        ms.append(tree.build_ms)
        _lib.lib.wt_tree_build_profile(tree.handle, prof, 32)
        lvl.append([prof[i] for i in range(1 + tree.num_levels)])
        if s < steps - 1:
            del tree
            gc.collect()
    return tree, ms, np.median(np.array(lvl), axis=0)


def _build_record(tree, n, w, ms, lvl, hbm):
    sizes = [int(x) for x in tree.level_sizes]
    c = 1 if tree.num_levels <= 8 else 2
    # median over the timed builds: one build whose pre-phase waited on a
    # host-side stall (seen once at 130 ms in a C3z pre-phase) would otherwise
    # set the figure; the mean and the minimum are reported beside it
    t_ms = float(np.median(ms))
    alg = build_alg_bytes(sizes, n, w, c)
    rec = {"symbols_per_s": n / (t_ms / 1e3), "ms": t_ms, "ms_min": float(np.min(ms)),
           "ms_mean": float(np.mean(ms)), "ms_all": [float(x) for x in ms],
           "GB_per_s": alg / (t_ms / 1e3) / 1e9, "alg_bytes": alg,
           "frac_of_hbm": alg / (t_ms / 1e3) / 1e9 / hbm, "n": n, "sigma": tree.sigma,
           "levels": tree.num_levels, "ms_histogram_and_plan": float(lvl[0]),
           "ms_per_level": [float(x) for x in lvl[1:]]}
    if tree.num_levels:
        # per-level device time = the level's kernel + its directory / layout
        # pass (dirq_kernel); the last two levels of a power-of-two alphabet
        # are ONE pair pass (wpair_kernel), reported together
        L = tree.num_levels
        pair = L >= 2 and sizes[L - 2] == sizes[L - 1]
        lv = [float(x) for x in lvl[1:]]
        if pair:
            lv[L - 2] += lv[L - 1]
            lv[L - 1] = 0.0
        dom = int(np.argmax(lv))
        if pair and dom == L - 2:
            name = f"wpair_kernel + 2 x dirq_kernel (levels {L - 2}-{L - 1})"
            dom_alg = level_alg_bytes(sizes, L - 2, w, c) + level_alg_bytes(sizes, L - 1, w, c)
        else:
            kern = "wlast_kernel" if dom == L - 1 else "wlevel_kernel"
            name = f"{kern} + dirq_kernel (level {dom})"
            dom_alg = level_alg_bytes(sizes, dom, w, c)
        rec["dominant_kernel"] = {
            "name": name, "ms": lv[dom], "alg_bytes": dom_alg,
            "GB_per_s": dom_alg / (lv[dom] / 1e3) / 1e9,
            "frac_of_hbm": dom_alg / (lv[dom] / 1e3) / 1e9 / hbm}
    return rec


def _extra_text(LC, name, dev):
    import torch
    c = LC.LARGE[name]
    n = 1 << c["n_log"]
    g = torch.Generator(device=dev)
    g.manual_seed(77)
    if c["kind"] == "zipf":
        return LC.zipf_torch(c["seed"], c["sigma"], n, dev)
    if c["kind"] == "dna":  # in slices: int64 indices of 2^32 symbols would be 32 GB
        lut = torch.tensor(list(b"ACGT"), dtype=torch.uint8, device=dev)
        text = torch.empty(n, dtype=torch.uint8, device=dev)
        for lo in range(0, n, 1 << 28):
            hi = min(n, lo + (1 << 28))
            idx = torch.randint(0, 4, (hi - lo,), generator=g, device=dev, dtype=torch.int32)
            text[lo:hi] = lut[idx.long()]
        return text
    return torch.randint(0, c["sigma"], (n,), generator=g, device=dev,
                         dtype=torch.int32).to(torch.int16 if c["dtype"] == "u16" else torch.uint8)


def _extra_builds(W, args, dev, hbm):
    """configs[2] / configs[3] builds on rank 0: device-generated texts of each
    recipe (tests/golden/large_cases.py; the parity tests build the exact
    golden texts), builds timed by their CUDA events.  Every config is built
    once before any is timed, so the library's stream-ordered memory pool has
    grown to the largest build's footprint first (timed builds that had to
    grow it waited 10 ms .. 1.6 s in their pre-phase)."""
    import torch
    import large_cases as LC
    out = {}
    steps = max(1, min(args.steps, 10))
    texts = {}
    for name in args.extra_builds:
        log(f"extra build {name}: text + warm-up build")
        texts[name] = _extra_text(LC, name, dev)
        tree = (W.construct(texts[name]) if LC.alphabet_of(name) is None
                else W.construct_with_alphabet(texts[name], LC.alphabet_of(name)))
        del tree
        gc.collect()
    for name in args.extra_builds:
        log(f"extra build {name}")
        c = LC.LARGE[name]
        n = 1 << c["n_log"]
        text = texts.pop(name)
        w = 2 if c["dtype"] == "u16" else 1
        tree, ms, lvl = _build_timed(W, text, LC.alphabet_of(name), steps, min(args.warmup, 2))
        rec = _build_record(tree, n, w, ms, lvl, hbm)
        rec["alphabet"] = "declared arange(2^16)" if c.get("declared") else "inferred"
        rec["text"] = c
        out[name] = rec
        del tree, text
        gc.collect()
    torch.cuda.empty_cache()
    return out


def _gen_queries(tree, m_each, dev, seed):
    """cli._bench_queries recipe (cli.py:246-260) drawn on the device."""
    import torch
    n, sigma = tree.n, tree.sigma
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    occ = torch.from_numpy(np.diff(tree.cum_hist)).to(dev)
    syms = torch.from_numpy(tree.alphabet.sorted_symbols.astype(np.int64)).to(dev)
    present = torch.nonzero(occ > 0).flatten()
    q = {}
    q["access"] = (None, torch.randint(0, n, (m_each[0],), generator=g, device=dev,
                                       dtype=torch.int64))
    rid = torch.randint(0, sigma, (m_each[1],), generator=g, device=dev, dtype=torch.int64)
    q["rank"] = (syms[rid], torch.randint(0, n + 1, (m_each[1],), generator=g, device=dev,
                                          dtype=torch.int64))
    sid = present[torch.randint(0, len(present), (m_each[2],), generator=g, device=dev)]
    ks = 1 + torch.floor(torch.rand(m_each[2], generator=g, device=dev, dtype=torch.float64)
                         * occ[sid]).to(torch.int64)
    q["select"] = (syms[sid], torch.minimum(ks, occ[sid]))
    return q


class DeviceBatches:
    """Three kind-homogeneous device-resident batches and their output
    buffers, run through the C-ABI on the current stream."""

    def __init__(self, tree, q, dev):
        import ctypes as C
        import torch
        from paper_2505_03372_b200 import _lib
        self.C, self.lib = C, _lib
        self.tree = tree
        self.q = q
        self.out = {"access": torch.empty(len(q["access"][1]), dtype=torch.uint8, device=dev),
                    "rank": torch.empty(len(q["rank"][1]), dtype=torch.int64, device=dev),
                    "select": torch.empty(len(q["select"][1]), dtype=torch.int64, device=dev)}
        self.stream = torch.cuda.current_stream(dev)
        self.sptr = C.c_void_p(self.stream.cuda_stream)
        self.bad = C.c_int64(-1)

    def launch(self, kind, sort=True, phases=None):
        C, L = self.C, self.lib
        ids, a = self.q[kind]
        o = self.out[kind]
        fl = L.F_DEVICE_PTRS | L.F_SYMBOLS | (L.F_SORT if sort else 0)
        ms = None
        if phases is not None:
            fl |= L.F_PHASES
            ms = (C.c_float * 4)()
        kid = {"access": L.Q_ACCESS, "rank": L.Q_RANK, "select": L.Q_SELECT}[kind]
        L.check(L.lib.wt_tree_query(self.tree.handle, kid,
                                    None if ids is None else C.c_void_p(ids.data_ptr()),
                                    C.c_void_p(a.data_ptr()), C.c_void_p(o.data_ptr()), a.numel(),
                                    0, fl, self.sptr, C.byref(self.bad), ms), "query")
        if self.bad.value != -1:
            raise RuntimeError(f"invalid query {self.bad.value}")
        if phases is not None:
            phases.update(total=ms[0], sort=ms[1], walk=ms[2], gather=ms[3])


def run_ours(args):
    import torch
    import torch.distributed as dist

    world, rank, local = _dist_setup(False)
    import large_cases as LC
    import paper_2505_03372_b200 as W
    from paper_2505_03372_b200 import parallel as par

    dev = torch.device("cuda", local)
    n = 1 << args.n_log
    hbm, peak_kind = peaks()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---------------- build (rank 0: the single-GPU construction) ----------
    build = builds = tree = None
    if rank == 0:
        log("C2 build")
        text_np = LC.text_np("C2") if args.n_log == 30 else \
            np.random.default_rng(0).integers(0, 256, n, dtype=np.uint8)  # C2 recipe
        text_dev = torch.from_numpy(text_np).to(dev)
        with Clocks(local) as clk_b:
            tree, ms, lvl = _build_timed(W, text_dev, None, args.steps, args.warmup)
        build = _build_record(tree, n, 1, ms, lvl, hbm)
        build["clocks"] = clk_b.summary()
        # size-independent check of this run's tree against the text
        pos = np.random.default_rng(5).integers(0, n, 1 << 16)
        assert np.array_equal(W.access_batch(tree, pos), text_np[pos]), "access != text"
        del text_dev, text_np
        torch.cuda.empty_cache()
        if args.extra_builds:
            builds = _extra_builds(W, args, dev, hbm)

    # ---------------- replicate over NCCL --------------------------------------
    replicate = None
    log("queries")
    if world > 1:
        tree = par.replicate(tree if rank == 0 else None, device=local)
        replicate = {"ms": par.max_over_ranks(float(tree.replicate_ms)),
                     "bytes": int(tree.device_bytes), "ranks": world}
        replicate["GB_per_s"] = replicate["bytes"] / (replicate["ms"] / 1e3) / 1e9

    # ---------------- weak-scaling step: 1e8 mixed queries per rank ------------
    m_total = args.queries
    per = [m_total // 3 + (1 if i < m_total % 3 else 0) for i in range(3)]
    q = _gen_queries(tree, per, dev, 1234 + rank)
    B = DeviceBatches(tree, q, dev)
    stream = B.stream
    for _ in range(args.warmup):
        for k in KINDS:
            B.launch(k)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    barrier()
    with Clocks(local) as clk:
        for s in range(args.steps):
            evs[s][0].record(stream)
            for j, k in enumerate(KINDS):
                B.launch(k)
                evs[s][j + 1].record(stream)
        barrier()
    step_ms = [e[0].elapsed_time(e[3]) for e in evs]
    kind_ms = {k: float(np.mean([e[j].elapsed_time(e[j + 1]) for e in evs]))
               for j, k in enumerate(KINDS)}
    ms_step = par.max_over_ranks(float(np.mean(step_ms)))
    value = world * m_total / (ms_step / 1e3)

    # per-phase device times of each sorted batch (sort / walk / gather) and
    # the same batches unsorted: one untimed pass each, after the timed region
    queries = {}
    lv_bits = [int(x) for x in tree.level_sizes]
    for j, k in enumerate(KINDS):
        ph = {}
        B.launch(k, phases=ph)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        B.launch(k, sort=False)
        e1.record(stream)
        torch.cuda.synchronize()
        uns = e0.elapsed_time(e1)
        walk_alg = sorted_walk_alg_bytes(k, per[j], lv_bits)
        queries[k] = {
            "queries": per[j], "queries_per_s": per[j] / (kind_ms[k] / 1e3), "ms": kind_ms[k],
            "phase_ms": {p: float(ph[p]) for p in ("sort", "walk", "gather")},
            "walk_alg_bytes": walk_alg,
            "walk_frac_of_hbm": walk_alg / (ph["walk"] / 1e3) / 1e9 / hbm,
            "unsorted": {"ms": uns, "queries_per_s": per[j] / (uns / 1e3),
                         "sector_model_bytes_per_query": SECTOR_BYTES[k],
                         "sector_model_frac": SECTOR_BYTES[k] * per[j] / (uns / 1e3) / 1e9 / hbm}}

    # the dominant kernel of the step: the longest walk (select)
    dom = max(KINDS, key=lambda k: queries[k]["phase_ms"]["walk"])
    dq = queries[dom]
    walk_ms = dq["phase_ms"]["walk"]
    traffic = traffic_from_profiles(f"{dom}_kernel", per[KINDS.index(dom)])
    roofline = {"bound": "hbm", "kernel": f"{dom}_kernel (walk of the sorted {dom} batch)",
                "achieved": dq["walk_alg_bytes"] / (walk_ms / 1e3) / 1e9, "peak": hbm,
                "unit": "GB/s", "frac": dq["walk_alg_bytes"] / (walk_ms / 1e3) / 1e9 / hbm,
                "peak_source": peak_kind, "traffic": traffic,
                "kernel_ms": walk_ms, "alg_bytes": dq["walk_alg_bytes"],
                "alg_model": "sorted walk: per level min(queries, level lines) x 32-B rank "
                             "lines (+ select line samples) + 16-24 B of batch I/O per query",
                "unsorted_sector_model_frac": dq["unsorted"]["sector_model_frac"]}
    if traffic:
        roofline["dram_frac"] = traffic / (walk_ms / 1e3) / 1e9 / hbm

    # correctness spot-check of this run's answers against the host API
    # (the same tree answering the same queries through another path)
    k = min(per[0], 1 << 16)
    pos = q["access"][1][:k].cpu().numpy()
    assert np.array_equal(B.out["access"][:k].cpu().numpy(), W.access_batch(tree, pos))

    # ---------------- end to end through the public API -------------------------
    e2e = None
    log("e2e")
    if args.e2e:
        pin = lambda t: t.cpu().pin_memory().numpy()
        h = {k: (None if q[k][0] is None else pin(q[k][0]), pin(q[k][1])) for k in KINDS}
        # 8 chunks per kind: copy-in / kernel / copy-out (and the host pack)
        # overlap; 2^22 measured 5 % faster than 2^21 (tools/bench_e2e.py)
        chunk = 1 << 22

        runners = {k: W.BatchRunner(tree, chunk, sort=True) for k in KINDS}
        batches = {k: W.QueryBatch(k, h[k][1], h[k][0], chunk) for k in KINDS}
        kind_s = {k: 0.0 for k in KINDS}

        def e2e_step(acc=None):
            res = []
            for k in KINDS:
                t1 = time.perf_counter()
                res.append(runners[k].run(batches[k]))
                if acc is not None:
                    acc[k] += time.perf_counter() - t1
            return res
        for _ in range(max(2, args.warmup)):
            # as in the timed loop, the previous step's results stay alive while
            # the next runs: the pinned result-array cache is warm for exactly that
            ra, rr, rs = e2e_step()
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            ra, rr, rs = e2e_step(kind_s)
        torch.cuda.synchronize()
        e2e_ms = par.max_over_ranks((time.perf_counter() - t0) * 1e3 / args.steps)
        assert np.array_equal(ra, B.out["access"].cpu().numpy())
        assert np.array_equal(rr, B.out["rank"].cpu().numpy())
        assert np.array_equal(rs, B.out["select"].cpu().numpy())
        # h2d bytes as the pipeline copied them (narrow wire: u32 arguments +
        # u16 symbols packed on the host); the API's own int64 inputs beside it
        e2e = {"value": world * m_total / (e2e_ms / 1e3), "unit": UNIT, "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": int(sum(runners[k].h2d_bytes for k in KINDS)),
               "api_input_bytes_per_step": int(per[0] * 8 + (per[1] + per[2]) * 16),
               "narrow_chunks": {k: [runners[k].narrow_chunks, runners[k].chunks] for k in KINDS},
               "d2h_bytes_per_step": int(per[0] * 1 + (per[1] + per[2]) * 8),
               "api": "BatchRunner(sort=True).run (access_batch / rank_batch / select_batch) "
                      "on pinned numpy arrays, chunk 2^22; int64 inputs packed to the "
                      "narrow wire (u16 symbols, u32 arguments) by a host thread pool",
               "per_kind": {k: {"ms": kind_s[k] * 1e3 / args.steps,
                                "stage_ms": runners[k].stage_seconds * 1e3,
                                "process_ms": runners[k].process_seconds * 1e3,
                                "staging_peak_records": runners[k].staging_peak_records}
                            for k in KINDS}}
        e2e["pcie_GB_per_s"] = (e2e["h2d_bytes_per_step"] + e2e["d2h_bytes_per_step"]) \
            / (e2e_ms / 1e3) / 1e9
    del B, q
    torch.cuda.empty_cache()

    # ---------------- C5: 1e9 queries per step split over the ranks -----------
    c5 = None
    log("c5")
    if args.c5_queries:
        lo, hi = par.shard_bounds(args.c5_queries, rank, world)
        mine = hi - lo
        per5 = [mine // 3 + (1 if i < mine % 3 else 0) for i in range(3)]
        B5 = DeviceBatches(tree, _gen_queries(tree, per5, dev, 99 + rank), dev)
        for k in KINDS:
            B5.launch(k)
        steps5 = max(1, min(args.steps, 5))
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(B5.stream)
        for _ in range(steps5):
            for k in KINDS:
                B5.launch(k)
        e1.record(B5.stream)
        barrier()
        ms5 = par.max_over_ranks(e0.elapsed_time(e1) / steps5)
        c5 = {"queries_per_step": args.c5_queries, "queries_per_gpu": mine, "steps": steps5,
              "ms_per_step": ms5, "queries_per_s": args.c5_queries / (ms5 / 1e3),
              "scaling": "strong", "note": "configs[4]: 1e9 mixed queries (sorted on the device) "
                                           "per step split over the replicas"}
        del B5
        torch.cuda.empty_cache()

    cpu = None
    log("cpu baseline")
    if rank == 0 and not args.no_cpu:
        cpu = cpu_baseline(W, tree, args)

    if world > 1:
        dist.barrier()
    if rank == 0:
        n_sorted_kernels = 6  # key, 2 scan passes, scatter, walk, gather
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "int64", "data": "synthetic (C2 text: numpy PCG64 seed 0, the golden "
                                      "recipe; queries: cli._bench_queries recipe drawn on the "
                                      "device)",
            "config": workload_config(args, world),
            "queries": queries, "build": build, "builds": builds, "c5": c5,
            "replicate": replicate, "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": args.steps * 3 * n_sorted_kernels,
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


def cpu_baseline(W, tree, args):
    """Rank 0: the reference on ONE host core, on a bounded sample of the C2
    workload, over the very tree the GPU answers (saved in the reference's
    WTIDX001 format, loaded by wtindex.load); answers checked against ours."""
    wt = _reference_module()
    if wt is None:
        return cpu_baseline_port(args)
    t0 = time.perf_counter()
    buf = io.BytesIO()
    tree.save(buf)
    log("cpu baseline: tree saved")
    buf.seek(0)
    rt = wt.load(buf)
    del buf
    load_s = time.perf_counter() - t0
    log("cpu baseline: reference loaded the index")
    sample = {k: args.cpu_sample for k in KINDS}  # equal thirds, as the GPU step
    done, spent, checked = 0, 0.0, 0
    per_kind = {}
    for k in KINDS:
        b = wt.cli._bench_queries(rt, k, sample[k], 21 + KINDS.index(k))
        t1 = time.perf_counter()
        got = wt.BatchRunner(rt, wt.batch.DEFAULT_CHUNK_SIZE, 1).run(b)
        dt = time.perf_counter() - t1
        ours = W.run_batch(tree, W.QueryBatch(k, b.args, b.symbols))
        assert np.array_equal(got, ours), f"reference and GPU answers differ ({k})"
        checked += len(got)
        done += len(got)
        spent += dt
        per_kind[k] = {"queries": len(got), "queries_per_s": len(got) / dt}
        log(f"cpu baseline: {k} {len(got) / dt:.0f} q/s")
    return {"value": done / spent, "unit": UNIT, "cores": 1, "kind": "reference",
            "sample": (f"wtindex 0.1.0 (the unmodified reference, baseline/_ref) "
                       f"BatchRunner.run(workers=1) on the C2 tree (n=2^{args.n_log}, sigma=256; "
                       f"the GPU-built index saved as WTIDX001 and loaded by wtindex.load in "
                       f"{load_s:.1f}s), one cli._bench_queries batch of {sample['access']} queries per kind "
                       f"(equal thirds, as the GPU step)"),
            "per_kind": per_kind, "answers_checked_vs_gpu": checked, "same_config": True}


def cpu_baseline_port(args, n_log=22):
    import oracle as O
    text = np.random.default_rng(0).integers(0, 256, 1 << n_log, dtype=np.uint8)
    t = O.build(text)
    num = 30000
    per_kind = {}
    for k in KINDS:
        ids, a = O.bench_queries(t.n, t.hist, k, num, 3)
        t0 = time.perf_counter()
        if k == "access":
            t.access_ids(a)
        elif k == "rank":
            t.rank_ids(ids, a)
        else:
            t.select_ids(ids, a)
        per_kind[k] = {"queries": num, "queries_per_s": num / (time.perf_counter() - t0)}
    mixed = 3 / sum(1 / per_kind[k]["queries_per_s"] for k in KINDS)
    return {"value": mixed, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"oracle port (numpy restatement; baseline/_ref absent), n=2^{n_log}",
            "per_kind": per_kind, "same_config": False}


_REF = {}


def _ref_worker(job):
    """Answer queries [lo, hi) of one kind with the reference; returns seconds."""
    kind, lo, hi = job
    wt, tree, q = _REF["wt"], _REF["tree"], _REF["qs"][kind]
    sub = wt.QueryBatch(kind, q.args[lo:hi], None if q.symbols is None else q.symbols[lo:hi])
    t0 = time.perf_counter()
    wt.BatchRunner(tree, wt.batch.DEFAULT_CHUNK_SIZE, 1).run(sub)
    return time.perf_counter() - t0


def run_reference(args):
    """--impl reference: the reference's own CPU path on all host cores, on
    the C2 config: wtindex.construct(workers=nproc) of the C2 text (timed once:
    ``build``), then per step a bounded sample of mixed queries answered by
    nproc forked processes through BatchRunner.run."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    import multiprocessing as mp

    import large_cases as LC
    wt = _reference_module()
    procs = os.cpu_count() or 1
    if wt is None:
        print(json.dumps({"impl": "reference", "unavailable":
                          "baseline/_ref absent (run __graft_entry__.build() in the build "
                          "container)"}))
        return
    n = 1 << args.n_log
    text = LC.text_np("C2") if args.n_log == 30 else \
        np.random.default_rng(0).integers(0, 256, n, dtype=np.uint8)
    t0 = time.perf_counter()
    tree = wt.construct(text, workers=procs)
    build_s = time.perf_counter() - t0
    del text
    pp = {k: args.ref_queries_per_proc for k in KINDS}  # equal thirds, as our step
    qs = {k: wt.cli._bench_queries(tree, k, procs * pp[k], 7 + KINDS.index(k)) for k in KINDS}
    _REF.update(wt=wt, tree=tree, qs=qs)
    ctx = mp.get_context("fork")
    times = []
    with ctx.Pool(procs) as pool:   # forked after the build: the tree is shared
        for step in range(args.warmup + args.steps):
            jobs = [(k, p * pp[k], (p + 1) * pp[k]) for p in range(procs) for k in KINDS]
            t1 = time.perf_counter()
            pool.map(_ref_worker, jobs)
            dt = time.perf_counter() - t1
            if step >= args.warmup:
                times.append(dt)
    q = procs * sum(pp.values())
    ms = float(np.mean(times)) * 1e3
    value = q / (ms / 1e3)
    sample = (f"wtindex 0.1.0, the unmodified reference (baseline/_ref), BatchRunner.run on the "
              f"C2 tree built by wtindex.construct(workers={procs}) in {build_s:.0f}s; per step "
              f"{pp['access']}/{pp['rank']}/{pp['select']} access/rank/select queries "
              f"(cli._bench_queries) in each of {procs} processes")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic (C2 text: numpy PCG64 seed 0; cli._bench_queries recipe)",
        "config": workload_config(args, world),
        "build": {"symbols_per_s": n / build_s, "seconds": build_s, "workers": procs,
                  "n": n, "sigma": 256},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": procs, "kind": "reference",
                         "sample": sample},
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
    ap.add_argument("--c5-queries", type=int, default=1_000_000_000,
                    help="configs[4] strong-scaling batch per step (0: skip)")
    ap.add_argument("--extra-builds", default="C3u,C3z,C3z_inf,C3r,C4",
                    help="comma list of tests/golden/large_cases.py configs to time ('' = none)")
    ap.add_argument("--no-e2e", dest="e2e", action="store_false")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=300_000,
                    help="cpu_baseline queries per kind (~10 s on one core at C2)")
    ap.add_argument("--ref-queries-per-proc", type=int, default=8000,
                    help="reference arm: queries per kind per process per step")
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU (gloo): launcher + barrier + max-over-ranks only")
    args = ap.parse_args()
    args.extra_builds = [x for x in args.extra_builds.split(",") if x]
    maybe_relaunch(args)
    if args.dry_run:
        run_dry(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
