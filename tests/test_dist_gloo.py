"""Multi-process (gloo, world_size 2, CPU) checks of the data-parallel step.

Each rank runs the CPU oracle on its shard of every global batch with the CE
cotangent scaled by 1/B_global (here: the rank's gradient of its local mean
loss times B_local/B_global), allreduces (sum) gradient + loss numerator +
hits, and applies Adam.  The result must equal single-process full-batch
training, and the replicas must stay bit-identical.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as tmp

from oracle.pyoracle import Lib, Net, State
from paper_2402_18994_b200.parallel import shard_rows

NET = Net(inp=30, hidden=(16, 12), classes=5, unroll=4)
B_LOCAL, WORLD, T, N, STEPS = 4, 2, 19, 24, 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _data(orc):
    x, y = orc.synth_raster(NET.classes, N, T, NET.inp, 3)
    return orc.pack_time(x), y


def _worker(rank, port, out):
    import torch
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    orc = Lib("orc")
    pk, y = _data(orc)
    st = State(orc.init(NET, orc.key_child(orc.key_from_seed(0), 0)) * np.float32(3.0))
    perm = orc.permutation(orc.key_child(orc.key_child(orc.key_from_seed(0), 1), 0), N)
    b_global = B_LOCAL * WORLD
    losses = []
    for step in range(STEPS):
        rows = shard_rows(perm, step, rank, WORLD, B_LOCAL)
        o = orc.forward_backward(NET, st.params, pk[rows], T, y[rows])
        scale = np.float32(B_LOCAL) / np.float32(b_global)
        local = np.concatenate([o["grads"] * scale,
                                [np.float32(o["loss"]) * np.float32(B_LOCAL), o["acc"] * B_LOCAL]])
        buf = torch.from_numpy(local.astype(np.float32))
        dist.all_reduce(buf, op=dist.ReduceOp.SUM)
        red = buf.numpy()
        g = red[:-2].copy()
        losses.append(float(red[-2]) / b_global)
        st.step = orc.adam(st.params, g, st.m, st.v, st.step)
    out[rank] = (st.params.copy(), losses)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_gloo_matches_single_process(orc):
    port = _free_port()
    mgr = tmp.Manager()
    out = mgr.dict()
    tmp.spawn(_worker, args=(port, out), nprocs=WORLD, join=True)
    p0, l0 = out[0]
    p1, l1 = out[1]
    assert np.array_equal(p0, p1), "replicas diverged"
    assert l0 == l1
    # single process, full global batches
    pk, y = _data(orc)
    st = State(orc.init(NET, orc.key_child(orc.key_from_seed(0), 0)) * np.float32(3.0))
    perm = orc.permutation(orc.key_child(orc.key_child(orc.key_from_seed(0), 1), 0), N)
    b_global = B_LOCAL * WORLD
    for step in range(STEPS):
        rows = perm[step * b_global:(step + 1) * b_global]
        o = orc.forward_backward(NET, st.params, pk[rows], T, y[rows])
        assert abs(o["loss"] - l0[step]) <= 1e-5 * abs(o["loss"])
        st.step = orc.adam(st.params, o["grads"], st.m, st.v, st.step)
    rel = np.linalg.norm(p0 - st.params) / np.linalg.norm(st.params)
    assert rel <= 1e-6, rel


def test_shard_rows_partition_the_global_batch():
    perm = np.random.default_rng(0).permutation(64)
    for world in (1, 2, 4, 8):
        b_local = 8 // world if world <= 8 else 1
        rows = np.concatenate([shard_rows(perm, 1, r, world, b_local) for r in range(world)])
        assert np.array_equal(rows, perm[8:16])


def _peer_worker(rank, port, out):
    """The owner-computes peer tail's rules on the CPU: every rank publishes its local
    buffer; rank r sums ITS slice (parallel.owner_slice) over all ranks' buffers in
    ascending rank order (parallel.peer_sum, what k_peer_owner's peer loads see),
    runs Adam on that slice only (m / v sharded with the owner), and every rank then
    gathers the updated slices from their owners (k_peer_gather)."""
    import torch
    from paper_2402_18994_b200.parallel import exchange_handles, owner_slice, peer_sum
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    # handle exchange: rank order, 64 bytes each
    hs = exchange_handles(bytes([rank + 1]) * 64, rank, WORLD, dist)
    assert hs == [bytes([q + 1]) * 64 for q in range(WORLD)]
    orc = Lib("orc")
    pk, y = _data(orc)
    st = State(orc.init(NET, orc.key_child(orc.key_from_seed(0), 0)) * np.float32(3.0))
    perm = orc.permutation(orc.key_child(orc.key_child(orc.key_from_seed(0), 1), 0), N)
    b_global = B_LOCAL * WORLD
    losses = []
    for step in range(STEPS):
        rows = shard_rows(perm, step, rank, WORLD, B_LOCAL)
        o = orc.forward_backward(NET, st.params, pk[rows], T, y[rows])
        scale = np.float32(B_LOCAL) / np.float32(b_global)
        local = np.concatenate([o["grads"] * scale,
                                [np.float32(o["loss"]) * np.float32(B_LOCAL), o["acc"] * B_LOCAL]])
        bufs = [torch.zeros(local.size) for _ in range(WORLD)]
        dist.all_gather(bufs, torch.from_numpy(local.astype(np.float32)))
        n = st.params.size
        lo, hi = owner_slice(n, rank, WORLD)
        red = peer_sum([b.numpy()[lo:hi] for b in bufs])          # my slice only
        tail = peer_sum([b.numpy()[n:] for b in bufs])             # loss numerator, hits
        losses.append(float(tail[0]) / b_global)
        mine = st.params[lo:hi].copy()
        m, v = st.m[lo:hi].copy(), st.v[lo:hi].copy()
        orc.adam(mine, red.copy(), m, v, st.step)
        st.m[lo:hi], st.v[lo:hi] = m, v                             # only the owner's are valid
        st.step += 1
        sl = [None] * WORLD
        dist.all_gather_object(sl, mine)
        st.params = np.concatenate(sl).astype(np.float32)
    out[rank] = (st.params.copy(), losses)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_peer_tail_rules_match_single_process(orc):
    port = _free_port()
    mgr = tmp.Manager()
    out = mgr.dict()
    tmp.spawn(_peer_worker, args=(port, out), nprocs=WORLD, join=True)
    p0, l0 = out[0]
    p1, l1 = out[1]
    assert np.array_equal(p0, p1), "replicas diverged"
    assert l0 == l1
    pk, y = _data(orc)
    st = State(orc.init(NET, orc.key_child(orc.key_from_seed(0), 0)) * np.float32(3.0))
    perm = orc.permutation(orc.key_child(orc.key_child(orc.key_from_seed(0), 1), 0), N)
    b_global = B_LOCAL * WORLD
    for step in range(STEPS):
        rows = perm[step * b_global:(step + 1) * b_global]
        o = orc.forward_backward(NET, st.params, pk[rows], T, y[rows])
        assert abs(o["loss"] - l0[step]) <= 1e-5 * abs(o["loss"])
        st.step = orc.adam(st.params, o["grads"], st.m, st.v, st.step)
    assert np.linalg.norm(p0 - st.params) / np.linalg.norm(st.params) <= 1e-6


def test_peer_sum_is_rank_ordered_float32():
    from paper_2402_18994_b200.parallel import peer_sum
    bufs = [np.array([1e8, 1.0], np.float32), np.array([1.0, 1e8], np.float32),
            np.array([-1e8, -1e8], np.float32)]
    got = peer_sum(bufs)
    want = np.array([(np.float32(1e8) + np.float32(1.0)) - np.float32(1e8),
                     (np.float32(1.0) + np.float32(1e8)) - np.float32(1e8)], np.float32)
    assert got.dtype == np.float32 and np.array_equal(got, want)
