"""Multi-GPU host logic (paper_2505_03372_b200.parallel) on CPU: world-size-2
gloo groups in forked processes.  The device engine is replaced by a stand-in
tree answering from the text (a test double with the WaveletTree.query
contract); the logic under test is the sharding, the error semantics across
shards, the unique-id broadcast, the gather order and the timing reduction."""

import multiprocessing as mp
import os
import socket
import traceback

import numpy as np
import pytest

from paper_2505_03372_b200 import BatchError, OrdinalError, PositionError, QueryBatch, SymbolError
from paper_2505_03372_b200 import parallel as par
from paper_2505_03372_b200.alphabet import AlphabetMap

Q_ACCESS, Q_RANK, Q_SELECT = 0, 1, 2


class TextTree:
    """Answers batches straight from the text (stand-in for the device tree)."""

    def __init__(self, text):
        self.text = np.asarray(text)
        self.n = len(self.text)
        syms = np.unique(self.text)
        self.alphabet = AlphabetMap(syms)
        self.occ = {int(s): int((self.text == s).sum()) for s in syms}

    def occurrences(self, c):
        return self.occ.get(int(c), 0)

    def query(self, kind, ids, args, *, symbols=False, access_ids=False, chunk=0, sort=False,
              out=None, stats=None):
        args = np.asarray(args, np.int64)
        if out is None:
            out = np.zeros(len(args), np.int64 if kind else self.text.dtype)
        assert len(out) == len(args) and out.dtype == (np.int64 if kind else self.text.dtype)
        for i, a in enumerate(args):
            if kind == Q_ACCESS:
                if not 0 <= a < self.n:
                    return out, i
                out[i] = self.text[a]
                continue
            c = int(ids[i])
            if c not in self.occ:
                return out, i
            if kind == Q_RANK:
                if not 0 <= a <= self.n:
                    return out, i
                out[i] = int((self.text[:a] == c).sum())
            else:
                if not 1 <= a <= self.occ[c]:
                    return out, i
                out[i] = int(np.flatnonzero(self.text == c)[a - 1])
        return out, -1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(world, fn, *args):
    port = _free_port()
    ctx = mp.get_context("fork")
    q = ctx.Queue()
    procs = [ctx.Process(target=_entry, args=(r, world, port, q, fn, args)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, ok, val = q.get(timeout=120)
        res[r] = (ok, val)
    for p in procs:
        p.join(timeout=60)
    for r, (ok, val) in sorted(res.items()):
        assert ok, f"rank {r}: {val}"
    return [res[r][1] for r in range(world)]


def _entry(rank, world, port, q, fn, args):
    try:
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        try:
            val = fn(rank, world, *args)
        finally:
            dist.destroy_process_group()
        q.put((rank, True, val))
    except Exception:
        q.put((rank, False, traceback.format_exc()))


@pytest.mark.parametrize("world", [1, 2, 3, 8])
@pytest.mark.parametrize("m", [0, 1, 7, 8, 1000, 10**8 + 3])
def test_shard_bounds_partition(world, m):
    b = [par.shard_bounds(m, r, world) for r in range(world)]
    assert b[0][0] == 0 and b[-1][1] == m
    for (lo, hi), (lo2, _) in zip(b, b[1:]):
        assert hi == lo2
    sizes = [hi - lo for lo, hi in b]
    assert max(sizes) - min(sizes) <= 1


def _w_basic(rank, world):
    uid = par.share_bytes(bytes(range(128)) if rank == 0 else None, 128)
    mx = par.max_over_ranks(float(rank + 1))
    mn = par.min_over_ranks(10 - rank)
    with par.SharedResult(11, np.int64) as res:
        lo, hi = par.shard_bounds(11, rank, world)
        res.slice(lo, hi)[:] = np.arange(lo, hi) * 10   # this rank's slice only
        import torch.distributed as dist
        dist.barrier()
        g = res.array.tolist()
    return uid, mx, mn, g


def test_uid_broadcast_reductions_and_shared_result_world2():
    out = _run(2, _w_basic)
    for uid, mx, mn, g in out:
        assert uid == bytes(range(128))
        assert mx == 2.0 and mn == 9
        assert g == [10 * i for i in range(11)]


def _w_shared_name_unique(rank, world):
    a = par.SharedResult(5, np.uint8)
    b = par.SharedResult(5, np.uint8)
    names = (a.shm.name, b.shm.name)
    a.close()
    b.close()
    return names


def test_shared_results_are_distinct_blocks():
    (a0, b0), (a1, b1) = _run(2, _w_shared_name_unique)
    assert a0 == a1 and b0 == b1 and a0 != b0


TEXT = np.random.default_rng(5).integers(0, 12, 400).astype(np.uint8)


def _w_sharded(rank, world, kind, args, syms):
    tree = TextTree(TEXT)
    return par.run_sharded(tree, QueryBatch(kind, args, syms)).tolist()


def _w_sharded_out(rank, world, kind, args, syms):
    """Caller-owned shared result: every rank reads the whole batch's answers
    from the one array after run_sharded returns."""
    tree = TextTree(TEXT)
    with par.SharedResult(len(args), par.result_dtype(tree, kind)) as res:
        got = par.run_sharded(tree, QueryBatch(kind, args, syms), out=res)
        assert got is res.array
        return got.tolist()


def test_run_sharded_equals_single_rank():
    r = np.random.default_rng(1)
    pos = r.integers(0, len(TEXT), 101)
    syms = np.unique(TEXT)[r.integers(0, len(np.unique(TEXT)), 101)]
    rpos = r.integers(0, len(TEXT) + 1, 101)
    occ = np.array([(TEXT == s).sum() for s in syms])
    ks = 1 + (r.random(101) * occ).astype(np.int64)
    one = TextTree(TEXT)
    for kind, args, s in (("access", pos, None), ("rank", rpos, syms), ("select", ks, syms)):
        want = one.query({"access": 0, "rank": 1, "select": 2}[kind], s, args)[0].tolist()
        for got in _run(2, _w_sharded, kind, args, s):
            assert got == want
        for got in _run(3, _w_sharded_out, kind, args, s):
            assert got == want


def _w_error(rank, world, kind, args, syms):
    tree = TextTree(TEXT)
    try:
        par.run_sharded(tree, QueryBatch(kind, args, syms))
    except BatchError as e:
        return e.index, type(e.__cause__).__name__
    return None


@pytest.mark.parametrize("bad_at", [3, 60])  # in rank 0's shard / in rank 1's shard
def test_first_bad_query_index_is_global(bad_at):
    args = np.arange(100) % len(TEXT)
    args[bad_at] = len(TEXT) + 5            # PositionError
    args[bad_at + 30 if bad_at + 30 < 100 else 99] = -1
    for idx, cause in _run(2, _w_error, "access", args, None):
        assert idx == bad_at and cause == PositionError.__name__
    syms = np.full(100, int(TEXT[0]))
    ks = np.ones(100, np.int64)
    ks[bad_at] = 10**6                        # OrdinalError
    for idx, cause in _run(2, _w_error, "select", ks, syms):
        assert idx == bad_at and cause == OrdinalError.__name__
    syms2 = syms.copy()
    syms2[bad_at] = 250                       # SymbolError (not in the alphabet)
    for idx, cause in _run(2, _w_error, "rank", np.ones(100, np.int64), syms2):
        assert idx == bad_at and cause == SymbolError.__name__
