"""Multi-GPU queries: replicas of one tree, independent query shards.

The reference has no multi-process code; the north star asks for
construction on one GPU and query batches sharded over the GPUs of a box, each
holding a replica broadcast over NVLink.  One process per GPU
(``torch.distributed``; ``torchrun`` sets RANK / WORLD_SIZE / LOCAL_RANK):

* ``replicate(tree_or_None)`` -- rank 0 passes its built tree, the others
  ``None``; the NCCL unique id travels over the process group, the tree's
  arrays over ``ncclBroadcast`` inside ``wt_tree_replicate`` (C-ABI); every
  rank returns a device-resident replica;
* ``shard_bounds(m, rank, world)`` -- the contiguous slice of a batch a rank
  answers (no data-path collective: the shards are independent);
* ``gather(local, m, group)`` -- optional: concatenate the ranks' answers in
  rank order (all-gather), so every rank sees the whole batch's result;
* ``run_sharded(tree, batch)`` -- one kind-homogeneous ``QueryBatch`` answered
  by all ranks, each its shard, gathered in query order;
* ``max_over_ranks(x)`` -- the timing reduction bench.py reports.

Everything here but ``replicate`` is plain host logic and is exercised with a
world-size-2 ``gloo`` group on CPU (tests/test_parallel_cpu.py).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .batch import QueryBatch, run_batch


def _dist():
    import torch.distributed as dist
    return dist


def shard_bounds(m: int, rank: int, world: int) -> tuple[int, int]:
    """[lo, hi) of query indices for `rank`: contiguous, disjoint, covering
    [0, m), sizes differing by at most one."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    base, extra = divmod(int(m), world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def share_bytes(payload: bytes | None, group=None, src: int = 0) -> bytes:
    """Broadcast a small byte string (the NCCL unique id) from `src`."""
    dist = _dist()
    obj = [payload if dist.get_rank() == src else None]
    dist.broadcast_object_list(obj, src=src, group=group)
    return obj[0]


def max_over_ranks(x: float, group=None, device=None) -> float:
    """Max of a per-rank scalar (device-timed step times are reported as the
    max over ranks)."""
    dist = _dist()
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(x)
    import torch
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def gather(local: np.ndarray, m: int, group=None) -> np.ndarray:
    """All-gather the ranks' shard results into one array in query order."""
    dist = _dist()
    world = dist.get_world_size(group)
    if world == 1:
        return local
    parts = [None] * world
    dist.all_gather_object(parts, np.ascontiguousarray(local), group=group)
    out = np.concatenate(parts) if parts else local[:0]
    if len(out) != m:
        raise RuntimeError(f"gathered {len(out)} answers for a batch of {m}")
    return out


def replicate(tree, device: int | None = None, group=None):
    """NCCL-broadcast rank 0's tree to every rank; returns this rank's replica
    (rank 0 gets its own tree back)."""
    dist = _dist()
    rank, world = dist.get_rank(), dist.get_world_size(group)
    if world == 1:
        return tree
    if rank == 0 and tree is None:
        raise ValueError("rank 0 must pass the built tree")
    uid = (C.c_uint8 * 128)()
    if rank == 0:
        _lib.check(_lib.lib.wt_nccl_unique_id(uid), "wt_nccl_unique_id")
    raw = share_bytes(bytes(uid) if rank == 0 else None, group)
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


def run_sharded(tree, batch: QueryBatch, group=None, gather_all: bool = True) -> np.ndarray:
    """Answer one kind-homogeneous batch across the group: each rank runs its
    shard through the single-GPU BatchRunner (same validation and error
    semantics: a BatchError carries the index in the WHOLE batch), results
    gathered in query order."""
    from .errors import BatchError
    dist = _dist()
    rank, world = dist.get_rank(), dist.get_world_size(group)
    lo, hi = shard_bounds(len(batch), rank, world)
    sub = QueryBatch(batch.kind, batch.args[lo:hi],
                     None if batch.symbols is None else batch.symbols[lo:hi], batch.chunk_size)
    err = None
    try:
        local = run_batch(tree, sub)
    except BatchError as e:  # first bad query of this shard, as a whole-batch index
        err = (lo + e.index, e)
        local = None
    errs = [None] * world
    dist.all_gather_object(errs, None if err is None else (err[0], type(err[1].__cause__).__name__,
                                                           str(err[1].__cause__)), group=group)
    bad = [e for e in errs if e is not None]
    if bad:
        first = min(bad)
        if err is not None and err[0] == first[0]:
            raise BatchError(first[0], err[1].__cause__) from err[1].__cause__
        from . import errors as E
        cause = getattr(E, first[1], E.Error)(first[2])
        raise BatchError(first[0], cause) from cause
    return gather(local, len(batch), group) if gather_all else local
