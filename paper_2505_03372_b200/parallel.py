"""Multi-GPU queries: replicas of one tree, independent query shards.

The reference has no multi-process code; the north star asks for
construction on one GPU and query batches sharded over the GPUs of a box, each
holding a replica broadcast over NVLink.  One process per GPU
(``torch.distributed``; ``torchrun`` sets RANK / WORLD_SIZE / LOCAL_RANK):

* ``replicate(tree_or_None)`` -- rank 0 passes its built tree, the others
  ``None``; the NCCL unique id (128 bytes) travels over the process group, the
  tree's arrays over one grouped ``ncclBroadcast`` inside
  ``wt_tree_replicate`` (C-ABI); every rank returns a device-resident replica;
* ``shard_bounds(m, rank, world)`` -- the contiguous slice of a batch a rank
  answers (no data-path collective: the shards are independent);
* ``SharedResult`` -- ONE host array for a whole batch's answers, shared by
  the ranks of the node (POSIX shared memory, page-locked on every rank with
  ``wt_host_register``): each rank's device copies its answers straight into
  its own disjoint slice, so results never pass through a collective;
* ``run_sharded(tree, batch)`` -- one kind-homogeneous ``QueryBatch`` answered
  by all ranks, each its shard, into a ``SharedResult``; the first invalid
  query of the WHOLE batch is found with one 8-byte MIN all-reduce and raised
  on every rank as the reference's ``BatchError(index, cause)``
  (batch.py:112-148);
* ``max_over_ranks(x)`` -- the timing reduction bench.py reports.

Everything but ``replicate`` is host logic, exercised with world-size-2
``gloo`` groups on CPU (tests/test_parallel_cpu.py).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .batch import BatchRunner, QueryBatch

_KIND_ID = {"access": _lib.Q_ACCESS, "rank": _lib.Q_RANK, "select": _lib.Q_SELECT}
_NO_ERROR = np.iinfo(np.int64).max


def _dist():
    import torch.distributed as dist
    return dist


def _is_multi(group=None) -> bool:
    dist = _dist()
    return dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1


def _collective_device(group=None):
    """The device collectives of `group` run on: CUDA for NCCL, else CPU."""
    import torch
    dist = _dist()
    if dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def shard_bounds(m: int, rank: int, world: int) -> tuple[int, int]:
    """[lo, hi) of query indices for `rank`: contiguous, disjoint, covering
    [0, m), sizes differing by at most one."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    base, extra = divmod(int(m), world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def share_bytes(payload: bytes | None, nbytes: int, group=None, src: int = 0) -> bytes:
    """Broadcast a small fixed-size byte string from `src` (a uint8 tensor
    broadcast: the NCCL unique id, a shared-memory name)."""
    import torch
    dist = _dist()
    buf = torch.zeros(nbytes, dtype=torch.uint8)
    if dist.get_rank() == src:
        raw = bytes(payload)
        if len(raw) > nbytes:
            raise ValueError(f"payload of {len(raw)} bytes exceeds {nbytes}")
        buf[:len(raw)] = torch.frombuffer(bytearray(raw), dtype=torch.uint8)
    dev = _collective_device(group)
    t = buf.to(dev)
    dist.broadcast(t, src=src, group=group)
    return bytes(t.cpu().numpy().tobytes())


def max_over_ranks(x: float, group=None) -> float:
    """Max of a per-rank scalar (device-timed step times are reported as the
    max over ranks)."""
    if not _is_multi(group):
        return float(x)
    import torch
    dist = _dist()
    t = torch.tensor([float(x)], dtype=torch.float64, device=_collective_device(group))
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def min_over_ranks(x: int, group=None) -> int:
    if not _is_multi(group):
        return int(x)
    import torch
    dist = _dist()
    t = torch.tensor([int(x)], dtype=torch.int64, device=_collective_device(group))
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    return int(t.item())


class SharedResult:
    """One result array for a whole batch, shared by the ranks of a node.

    Rank 0 creates a POSIX shared-memory block of ``m`` elements and
    broadcasts its name (a few bytes; the answers themselves never enter a
    collective); every rank maps it, page-locks it (``wt_host_register``, so
    its device->host copies are DMA into its slice) and writes only
    ``array[lo:hi]`` of its shard.  After ``run_sharded`` returns, every
    rank sees all answers in query order.  Close on every rank (rank 0
    unlinks after a barrier)."""

    def __init__(self, m: int, dtype, group=None, register: bool = True):
        from multiprocessing import shared_memory
        dist = _dist()
        self.group = group
        self.dtype = np.dtype(dtype)
        self.m = int(m)
        self.rank = dist.get_rank() if _is_multi(group) else 0
        nbytes = max(1, self.m * self.dtype.itemsize)
        if self.rank == 0:
            self.shm = shared_memory.SharedMemory(create=True, size=nbytes)
            name = self.shm.name.encode()
        else:
            name = None
        if _is_multi(group):
            name = share_bytes(name, 64, group).rstrip(b"\0")
        if self.rank != 0:
            self.shm = shared_memory.SharedMemory(name=name.decode())
            try:  # the creator owns the block: no tracker unlink from this rank
                from multiprocessing import resource_tracker
                resource_tracker.unregister(self.shm._name, "shared_memory")
            except Exception:
                pass
        self.array = np.ndarray(self.m, self.dtype, buffer=self.shm.buf)
        self._addr = self.array.ctypes.data if self.m else 0
        self._registered = False
        if register and self.m:
            self._registered = _lib.lib.wt_host_register(C.c_void_p(self._addr),
                                                         self.m * self.dtype.itemsize) == 0
        self._closed = False

    def slice(self, lo: int, hi: int) -> np.ndarray:
        return self.array[lo:hi]

    def close(self):
        if self._closed:
            return
        self._closed = True
        if self._registered:
            _lib.lib.wt_host_unregister(C.c_void_p(self._addr))
        del self.array
        if _is_multi(self.group):
            _dist().barrier(group=self.group)
        self.shm.close()
        if self.rank == 0:
            self.shm.unlink()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def replicate(tree, device: int | None = None, group=None):
    """NCCL-broadcast rank 0's tree to every rank; returns this rank's replica
    (rank 0 gets its own tree back)."""
    dist = _dist()
    if not _is_multi(group):
        return tree
    rank, world = dist.get_rank(), dist.get_world_size(group)
    if rank == 0 and tree is None:
        raise ValueError("rank 0 must pass the built tree")
    uid = (C.c_uint8 * 128)()
    if rank == 0:
        _lib.check(_lib.lib.wt_nccl_unique_id(uid), "wt_nccl_unique_id")
    raw = share_bytes(bytes(uid) if rank == 0 else None, 128, group)
    uid = (C.c_uint8 * 128).from_buffer_copy(raw)
    out = C.c_void_p()
    ms = C.c_float(0)
    dev = _lib.current_device() if device is None else int(device)
    _lib.check(_lib.lib.wt_tree_replicate(tree.handle if rank == 0 else None, uid, rank, world,
                                          dev, C.byref(out), C.byref(ms)), "wt_tree_replicate")
    if rank == 0:
        tree.replicate_ms = float(ms.value)
        return tree
    from .wtree import WaveletTree, _TreeHandle
    meta = _lib.Meta()
    _lib.check(_lib.lib.wt_tree_meta(out, C.byref(meta)), "wt_tree_meta")
    rep = WaveletTree(_TreeHandle(out), int(meta.symbol_width),
                      np.uint8 if meta.symbol_width == 1 else np.uint16)
    rep.replicate_ms = float(ms.value)
    return rep


def result_dtype(tree, kind: str):
    return tree.alphabet.sorted_symbols.dtype if kind == "access" else np.dtype(np.int64)


def run_sharded(tree, batch: QueryBatch, group=None, out: SharedResult | None = None,
                sort: bool = False) -> np.ndarray:
    """Answer one kind-homogeneous batch across the group.

    Each rank answers ``shard_bounds(len(batch), rank, world)`` on its own
    replica, its device copying the answers into its slice of ``out`` (a
    ``SharedResult``; one is made -- and closed -- when ``out`` is None, and
    the answers are returned as a private copy).  Validation has the
    reference's semantics over the WHOLE batch: the smallest invalid query
    index of any shard (one MIN all-reduce) is raised on every rank as
    ``BatchError(index, cause)``."""
    from .errors import BatchError
    dist = _dist()
    multi = _is_multi(group)
    rank = dist.get_rank() if multi else 0
    world = dist.get_world_size(group) if multi else 1
    m = len(batch)
    lo, hi = shard_bounds(m, rank, world)
    own = out is None
    res = SharedResult(m, result_dtype(tree, batch.kind), group) if own else out
    try:
        bad = -1
        if hi > lo:
            syms = None if batch.symbols is None else batch.symbols[lo:hi]
            _, bad = tree.query(_KIND_ID[batch.kind], syms, batch.args[lo:hi], symbols=True,
                                chunk=min(batch.chunk_size, hi - lo), sort=sort,
                                out=res.slice(lo, hi))
        first = min_over_ranks(lo + bad if bad >= 0 else _NO_ERROR, group)
        if first != _NO_ERROR:
            # every rank holds the whole batch: the cause is derived locally
            raise BatchError(first, BatchRunner(tree)._cause(batch, first))
        if multi:
            dist.barrier(group=group)  # every slice has landed
        return res.array.copy() if own else res.array
    finally:
        if own:
            res.close()
