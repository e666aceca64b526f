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
* every rank applies the identical Adam update to the identical reduced
  gradient, so parameter replicas stay bit-identical.
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


def combine_tail(loss_sums, hits, b_global: int):
    """StepResult from the allreduced (loss numerator, hit count)."""
    return float(np.float32(sum(loss_sums)) / np.float32(b_global)), float(sum(hits)) / b_global
