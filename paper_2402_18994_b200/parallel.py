"""Data-parallel decomposition of the training step (host-side rules).

The engine (engine.cu, snn_train_epochs_from / bench.py) and the tests share
these rules:

* the epoch permutation is the reference's (optimize.hpp:266-268), cut into
  global batches of B_global = B_local * world (drop remainder, data.hpp:190);
* rank r takes the contiguous slice [r*B_local, (r+1)*B_local) of each global
  batch;
* every rank scales the CE cotangent by 1/B_global (objective.hpp:104), so the
  SUM over ranks of the local gradients is the full-batch gradient;
* the loss numerator (sum of lse - logit_y) and the hit count ride in the same
  allreduce as the gradient; StepResult = (sum / B_global, hits / B_global);
* with the NCCL tail every rank applies the identical Adam update to the
  identical reduced gradient; with the peer tail each parameter is updated by
  exactly one owner rank and copied to the others -- either way the parameter
  replicas stay bit-identical.

Two device tails implement the exchange (engine.cu):

* "peer" (default, owner-computes): every rank's k_reduce writes its local
  buffer (gradient, loss numerator, hits, regularizer values) into an
  IPC-exported exchange buffer and raises flag A on every rank; rank r owns
  the flat parameter slice [r n / W, (r+1) n / W) (`owner_slice`):
  k_peer_owner waits for all A flags, sums its slice over the ranks' buffers by
  peer loads over NVLink in ascending rank order (`peer_sum`), runs Adam on it
  (m / v sharded with the owner, ZeRO-1 style) and raises flag B; k_peer_gather
  waits for all B flags and copies every slice from its owner.  Each rank reads
  about 2 n (W-1)/W floats per step -- O(n), not O(W n);
* "nccl": k_reduce, ncclAllReduce (sum), k_adam.
"""
from __future__ import annotations

import numpy as np


def global_batches(perm: np.ndarray, b_global: int) -> int:
    return len(perm) // b_global


def shard_rows(perm: np.ndarray, batch: int, rank: int, world: int, b_local: int) -> np.ndarray:
    """Rows of global batch `batch` owned by `rank`."""
    gb = b_local * world
    start = batch * gb + rank * b_local
    return np.asarray(perm[start:start + b_local])


def owner_slice(n: int, rank: int, world: int) -> tuple[int, int]:
    """[lo, hi) of the flat parameters rank `rank` updates (kernels.cuh peer_slice_lo)."""
    return n * rank // world, n * (rank + 1) // world


def peer_sum(buffers):
    """k_peer_adam's reduction: float32 sum of the ranks' buffers, ascending rank
    order, starting from 0 -- the same bits on every rank."""
    acc = np.zeros_like(np.asarray(buffers[0], np.float32))
    for b in buffers:
        acc = (acc + np.asarray(b, np.float32)).astype(np.float32)
    return acc


def exchange_handles(handle: bytes, rank: int, world: int, dist) -> list:
    """All-gather every rank's 64-byte exchange-buffer handle, in rank order."""
    if len(handle) != 64:
        raise ValueError("peer handle must be 64 bytes")
    got = [None] * world
    dist.all_gather_object(got, (rank, bytes(handle)))
    if [r for r, _ in got] != list(range(world)):
        raise RuntimeError(f"handle exchange out of order: {[r for r, _ in got]}")
    return [h for _, h in got]


def setup_data_parallel(eng, rank: int, world: int, dist, tail: str = "peer") -> None:
    """Join `eng` to the data-parallel group: tail "peer" (exchange buffers over
    NVLink peer memory) or "nccl" (ncclAllReduce)."""
    if tail == "peer":
        eng.peer_open(rank, world, exchange_handles(eng.peer_handle(), rank, world, dist))
    elif tail == "nccl":
        from .engine import Engine
        uid = [Engine.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        eng.comm_init(uid[0], rank, world)
    else:
        raise ValueError(f"unknown data-parallel tail {tail!r}")


def combine_tail(loss_sums, hits, b_global: int):
    """StepResult from the allreduced (loss numerator, hit count)."""
    return float(np.float32(sum(loss_sums)) / np.float32(b_global)), float(sum(hits)) / b_global
