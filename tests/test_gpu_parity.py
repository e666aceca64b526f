"""GPU parity: the CUDA engine (through the C ABI) vs the CPU oracle.

Bar (BASELINE.json north_star): spike-raster agreement >= 99.99 %, loss and
gradients within 1e-4 relative (norm per tensor) on the fp32 path.  The scan
kernels are additionally checked BIT-EXACT given the GPU's own projection
(numpy float32 restatement in tests/scanref.py, same op order as neuron.hpp).
"""
import numpy as np
import pytest

import scanref
from oracle.pyoracle import Net, State

pytestmark = pytest.mark.gpu

SPIKE_AGREE = 0.9999
REL_TOL = 1e-4


def relnorm(a, b):
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-30))


def make_engine(net: Net, B, T, seed=0, lr=1e-3, **cfg):
    from paper_2402_18994_b200 import Engine, TrainConfig, shd_spec
    spec = shd_spec(hidden=net.hidden, classes=net.classes, inp=net.inp, act=net.act,
                    bias=net.bias)
    for layer in spec.layers:
        if hasattr(layer, "threshold"):
            layer.threshold = net.threshold
            if net.slope is not None:
                layer.activation.slope = net.slope
    if net.cell:  # declared ALIF / RLIF cells (oracle/spiketrain_oracle.h)
        from paper_2402_18994_b200 import ALIFLayer, RLIFLayer
        hid = [i for i, layer in enumerate(spec.layers) if type(layer).__name__ == "LIFLayer"]
        for i, kind in zip(hid, net.cell):
            if kind != "lif":
                old = spec.layers[i]
                cls = ALIFLayer if kind == "alif" else RLIFLayer
                spec.layers[i] = cls(old.activation, old.threshold, old.beta_mode, old.fixed_beta)
    if net.monitor:  # MonitorLayer after the listed hidden LIF layers
        from paper_2402_18994_b200 import MonitorLayer
        for m in sorted(net.monitor, reverse=True):
            spec.layers.insert(2 * m + 2, MonitorLayer())
    if net.readout == "lif":  # a LIF readout: its spikes are the trace (network.hpp:396)
        from paper_2402_18994_b200 import LIFLayer
        hid = next(layer for layer in spec.layers if type(layer).__name__ == "LIFLayer")
        ro = spec.layers[-1]
        spec.layers[-1] = LIFLayer(hid.activation, hid.threshold, ro.beta_mode, ro.fixed_beta)
    return Engine(spec, TrainConfig(batch_size=B, seed=seed, lr=lr, unroll=net.unroll, **cfg), T)


def check_grads(orc, net, g, ref, tol=REL_TOL):
    for name, off, size in orc.entries(net):
        r = relnorm(g[off:off + size], ref[off:off + size])
        assert r <= tol, f"{name}: relnorm {r:.3e}"


def check_adam_step(orc, net, p_gpu, p_ref, g_ref, lr=1e-3):
    """Parameters after one Adam step.  The first step is ~lr*sign(g), so an element
    whose gradient nearly cancels (|g| tiny next to its tensor) can legitimately move
    the other way when the fp32 sums round differently; every other element must
    agree to 1e-6 relative (and the update itself is bit-exact given the gradient,
    test_gpu_benched_shapes.py::test_adam_bit_exact_given_gradient)."""
    d = np.abs(p_gpu - p_ref)
    for name, off, size in orc.entries(net):
        sl = slice(off, off + size)
        scale = np.abs(g_ref[sl]).max()
        bad = d[sl] > 1e-6 * np.maximum(np.abs(p_ref[sl]), 1e-3)
        tiny = np.abs(g_ref[sl]) <= 1e-2 * scale
        assert not (bad & ~tiny).any(), f"{name}: Adam step differs where |g| is not negligible"
        assert (d[sl] <= 2.0 * lr * 1.0001).all(), f"{name}: update larger than 2 lr"


CASES = [
    ("tiny", Net(inp=30, hidden=(16, 12), classes=5, unroll=4), 6, 19, 3.0),
    ("T70-superspike", Net(inp=70, hidden=(40, 24), classes=7, act="superspike"), 5, 70, 3.0),
    ("3hidden-triangular", Net(inp=50, hidden=(64, 48, 32), classes=6, act="triangular"), 4, 33, 3.0),
    ("bias-boxcar", Net(inp=40, hidden=(24, 20), classes=4, act="boxcar", bias=True), 5, 23, 3.0),
    ("custom-theta", Net(inp=33, hidden=(130, 32), classes=7, act="custom", threshold=0.75), 3, 40, 2.0),
    ("T200-two-tiles", Net(inp=64, hidden=(128, 128), classes=10), 3, 200, 2.0),
    ("c1-shape", Net(), 8, 128, 2.0),
    # three hidden layers in one fused forward launch (inp >= 128, H <= 128, T <= 128)
    ("3hidden-fused", Net(inp=150, hidden=(64, 48, 32), classes=6, act="superspike"), 5, 50, 3.0),
    # declared sigmoid surrogate (custom(heaviside, k s (1 - s)), oracle/spiketrain_oracle.h)
    ("sigmoid", Net(inp=60, hidden=(96, 40), classes=8, act="sigmoid"), 5, 45, 3.0),
]


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_step_parity(orc, case):
    _, net, B, T, scale = case
    params = orc.init(net, orc.key_child(orc.key_from_seed(11), 0)) * np.float32(scale)
    x, y = orc.synth_raster(net.classes, B, T, net.inp, 5)
    pk = orc.pack_time(x)
    eng = make_engine(net, B, T)
    eng.stage_dataset(pk, y)
    eng.set_params(params)
    assert np.array_equal(eng.get_params(), params)
    eng.debug(True)
    rows = np.arange(B, dtype=np.uint32)
    loss, acc = eng.forward_backward(rows)
    ref = orc.forward_backward(net, params, pk, T, y, want_spikes=True, want_trace=True)
    assert abs(loss - ref["loss"]) <= REL_TOL * abs(ref["loss"])
    ents = {n: (o, s) for n, o, s in orc.entries(net)}
    for l, h in enumerate(net.hidden):
        I = eng.fetch("I", l)
        o, s = ents[f"l{2 * l + 1}.beta"]
        V_ref, S_ref = scanref.lif_forward(
            I if not net.bias else I, params[o:o + s], net.threshold)
        assert np.array_equal(eng.fetch("V", l), V_ref), f"layer {l}: V not bit-exact given I"
        S = eng.fetch("spikes", l)
        assert np.array_equal(S, S_ref), f"layer {l}: spikes not bit-exact given I"
        assert (S == ref["spikes"][l]).mean() >= SPIKE_AGREE
    assert relnorm(eng.fetch("trace"), ref["trace"]) <= REL_TOL
    check_grads(orc, net, eng.get_grads(), ref["grads"])
    # the backward scan given the GPU's own dS: tests/test_gpu_benched_shapes.py
    # (test_backward_scan_given_ds) checks dI against scanref.lif_backward
    # one optimizer step
    st = State(params.copy())
    lo, ao = orc.train_step(net, st, pk, T, y)
    eng.debug(False)
    l2, a2 = eng.train_step(rows)
    assert abs(l2 - lo) <= REL_TOL * abs(lo) and a2 == ao
    check_adam_step(orc, net, eng.get_params(), st.params, ref["grads"])
    m, v, step = eng.get_opt_state()
    assert step == 1
    assert relnorm(m, st.m) <= REL_TOL and relnorm(v, st.v) <= 1e-3


@pytest.mark.parametrize("tag", ["init", "warm", "hot"])
def test_c1_golden(orc, golden, tag):
    """C1 network at the reference's own init/warm/hot checkpoints (golden)."""
    g = golden("c1")
    net = Net()
    params = g["params_init"] if tag == "init" else g[f"{tag}_params"]
    eng = make_engine(net, 16, 128)
    eng.stage_dataset(g["batch_packed"], g["batch_y"])
    eng.set_params(params)
    eng.debug(True)
    loss, acc = eng.forward_backward(np.arange(16, dtype=np.uint32))
    ref_loss = float(g[f"{tag}_loss"])
    assert abs(loss - ref_loss) <= REL_TOL * max(abs(ref_loss), 1e-3)
    for l in range(2):
        S = eng.fetch("spikes", l)
        ref_s = np.unpackbits(g[f"{tag}_spikes{l}_bits"])[:S.size].reshape(S.shape)
        assert (S == ref_s).mean() >= SPIKE_AGREE
    check_grads(orc, net, eng.get_grads(), g[f"{tag}_grads"])


@pytest.mark.parametrize("tag", ["init", "hot"])
def test_c1_full_batch(orc, golden, tag):
    """Full C1 workload (B=256, T=128) vs the oracle on the same inputs."""
    g = golden("c1")
    net = Net()
    params = g["params_init"] if tag == "init" else g["hot_params"]
    x, y = orc.synth_raster(20, 256, 128, 700, 1)
    pk = orc.pack_time(x)
    eng = make_engine(net, 256, 128)
    eng.stage_dataset(pk, y)
    eng.set_params(params)
    eng.debug(True)
    loss, acc = eng.forward_backward(np.arange(256, dtype=np.uint32))
    ref = orc.forward_backward(net, params, pk, 128, y, want_spikes=True)
    assert abs(loss - ref["loss"]) <= REL_TOL * max(abs(ref["loss"]), 1e-3)
    assert acc == ref["acc"]
    for l in range(2):
        assert (eng.fetch("spikes", l) == ref["spikes"][l]).mean() >= SPIKE_AGREE
    check_grads(orc, net, eng.get_grads(), ref["grads"])


def test_training_curve_matches_oracle(orc):
    """Epoch loop with the reference key schedule: 3 epochs of C1-shaped training."""
    net = Net()
    B, N, T = 64, 256, 128
    x, y = orc.synth_raster(20, N, T, 700, 1)
    pk = orc.pack_time(x)
    eng = make_engine(net, B, T, seed=0)
    p0 = orc.init(net, orc.key_child(orc.key_from_seed(0), 0))
    assert np.array_equal(eng.get_params(), p0), "engine init != reference init(master.child(0))"
    eng.stage_dataset(pk, y)
    m_gpu = eng.train_epochs(3)
    st = State(p0.copy())
    m_ref = orc.train_epochs(net, st, pk, y, T, B, 3, 0)
    assert np.allclose(m_gpu[:, 0], m_ref[:, 0], rtol=1e-3), (m_gpu, m_ref)
    assert np.abs(m_gpu[:, 1] - m_ref[:, 1]).max() <= 1.0 / B + 1e-12
    assert relnorm(eng.get_params(), st.params) <= 1e-4


def test_packed_entry_matches_rows_entry(orc):
    """train_step(st, packed_x, T, targets) == the staged-dataset path."""
    net = Net(inp=30, hidden=(16, 12), classes=5)
    x, y = orc.synth_raster(5, 4, 19, 30, 2)
    pk = orc.pack_time(x)
    e1 = make_engine(net, 4, 19)
    e2 = make_engine(net, 4, 19)
    e1.stage_dataset(pk, y)
    l1 = e1.train_step(np.arange(4, dtype=np.uint32))
    l2 = e2.train_step_packed(pk, y)
    assert l1 == l2
    assert np.array_equal(e1.get_params(), e2.get_params())


def test_errors_map_to_reference_classes(orc):
    from paper_2402_18994_b200 import ArgumentError, FormatError
    net = Net(inp=30, hidden=(16,), classes=5)
    eng = make_engine(net, 2, 19)
    x, y = orc.synth_raster(5, 2, 19, 30, 2)
    pk = orc.pack_time(x)
    with pytest.raises(ArgumentError):
        eng.stage_dataset(pk, np.array([0, 7]))       # target outside [0, classes)
    with pytest.raises(FormatError):
        eng.stage_dataset(pk[:, :1], y)                # packed extent != ceil(T/8)
    eng.stage_dataset(pk, y)
    with pytest.raises(ArgumentError):
        eng.train_step(np.array([0, 5], np.uint32))    # row outside the dataset
    from paper_2402_18994_b200 import ShapeError
    with pytest.raises(ShapeError):
        eng.train_step_packed(pk[:, :, :29], y)        # feature count != network input
    with pytest.raises(ShapeError):
        eng.train_step_packed(pk.reshape(2, -1), y)    # not [B, ceil(T/8), input]
    with pytest.raises(FormatError):
        eng.train_steps_packed(pk[None, :, :2], y[None])   # packed extent != ceil(T/8)


def test_determinism(orc):
    net = Net(inp=30, hidden=(16, 12), classes=5)
    x, y = orc.synth_raster(5, 8, 19, 30, 2)
    pk = orc.pack_time(x)
    outs = []
    for _ in range(2):
        e = make_engine(net, 4, 19, seed=9)
        e.stage_dataset(pk, y)
        m = e.train_epochs(3)
        outs.append((m, e.get_params()))
    assert np.array_equal(outs[0][0], outs[1][0])
    assert np.array_equal(outs[0][1], outs[1][1])


BIG = [
    ("c3-shape", Net(inp=700, hidden=(1024, 1024), classes=20), 2, 256, 1.0),
    ("c5-shape", Net(inp=700, hidden=(256, 256), classes=20), 2, 1000, 1.5),
]


@pytest.mark.parametrize("case", BIG, ids=[c[0] for c in BIG])
def test_baseline_shapes(orc, case):
    """Config C3 (700-1024-1024-20, T=256) and C5 (700-256-256-20, T=1000) shapes."""
    _, net, B, T, scale = case
    params = orc.init(net, orc.key_child(orc.key_from_seed(0), 0)) * np.float32(scale)
    x, y = orc.synth_raster(20, B, T, 700, 1)
    pk = orc.pack_time(x)
    eng = make_engine(net, B, T)
    eng.stage_dataset(pk, y)
    eng.set_params(params)
    eng.debug(True)
    loss, acc = eng.forward_backward(np.arange(B, dtype=np.uint32))
    ref = orc.forward_backward(net, params, pk, T, y, want_spikes=True)
    assert abs(loss - ref["loss"]) <= REL_TOL * abs(ref["loss"])
    flips = 0
    S = [eng.fetch("spikes", l) for l in range(2)]
    for l in range(2):
        assert (S[l] == ref["spikes"][l]).mean() >= SPIKE_AGREE
        flips += int((S[l] != ref["spikes"][l]).sum())
    if flips == 0:
        check_grads(orc, net, eng.get_grads(), ref["grads"])
    else:
        # a flipped fp32 near-tie legitimately moves the gradient: the 1e-4 bar is
        # applied to the teacher-forced oracle replaying the GPU's own rasters
        forced = orc.forward_backward(net, params, pk, T, y, forced=S)
        check_grads(orc, net, eng.get_grads(), forced["grads"])


def test_device_synth_is_bit_exact(orc):
    """synth_raster + pack_time generated in HBM == the reference's host version."""
    from paper_2402_18994_b200 import Engine, TrainConfig, shd_spec
    for T, n in ((128, 40), (19, 7), (1000, 3)):
        eng = Engine(shd_spec(), TrainConfig(batch_size=1), T)
        eng.synth_dataset(n, seed=1)
        pk, y = eng.read_dataset(0, n)
        x_ref, y_ref = orc.synth_raster(20, n, T, 700, 1)
        assert np.array_equal(pk, orc.pack_time(x_ref))
        assert np.array_equal(y, y_ref)


def test_epoch_permutation_matches_reference(orc):
    from paper_2402_18994_b200 import Engine, TrainConfig, shd_spec
    eng = Engine(shd_spec(), TrainConfig(batch_size=1, seed=7), 8)
    for e in (0, 3):
        ref = orc.permutation(orc.key_child(orc.key_child(orc.key_from_seed(7), 1 + e), 0), 500)
        assert np.array_equal(eng.epoch_permutation(e, 500), ref)


def test_schedule_steps_match_train_step(orc):
    """Device-resident schedule (8-step graphs, device slot counter, fused step
    tail) == host-driven train_step on the same rows, bit for bit; a slot jump
    re-seeds the device counter."""
    net = Net(inp=30, hidden=(16, 12), classes=5)
    B, T, N = 4, 19, 40
    x, y = orc.synth_raster(5, N, T, 30, 2)
    pk = orc.pack_time(x)
    rng = np.random.default_rng(3)
    sched = rng.integers(0, N, size=(24, B)).astype(np.uint32)
    order = list(range(0, 11)) + [17] + list(range(18, 21)) + [4]   # 8-graph + singles, jumps
    ref = make_engine(net, B, T, seed=5)
    ref.stage_dataset(pk, y)
    for s in order:
        last_ref = ref.train_step(sched[s])
    eng = make_engine(net, B, T, seed=5)
    eng.stage_dataset(pk, y)
    eng.upload_schedule(sched.reshape(-1))
    eng.enqueue_steps(0, 11)
    eng.enqueue_step(17)
    eng.enqueue_steps(18, 3)
    eng.enqueue_steps(4, 1)
    eng.sync()
    assert eng.read_result() == last_ref
    assert np.array_equal(eng.get_params(), ref.get_params())
    m1, v1, s1 = eng.get_opt_state()
    m2, v2, s2 = ref.get_opt_state()
    assert s1 == s2 == len(order)
    assert np.array_equal(m1, m2) and np.array_equal(v1, v2)


def test_launch_count_matches_captured_step(orc):
    """bench.py's gpu_launches claim: launches_per_step == kernels in one captured step,
    for partially and fully fused forward launch groups."""
    # (layer 0 has K_pad = 64 < 128, so it runs alone and layers 1-2 fuse), (all fused)
    for net, T, n_fwd in ((Net(inp=30, hidden=(16, 12, 8), classes=5), 19, 2),
                          (Net(inp=150, hidden=(64, 48, 32), classes=5), 40, 1)):
        x, y = orc.synth_raster(5, 8, T, net.inp, 2)
        eng = make_engine(net, 4, T)
        eng.stage_dataset(orc.pack_time(x), y)
        names = [n for n, _ in eng.profile(1)]
        assert len(names) == eng.launches_per_step, names
        assert sum(n.startswith("lif_fwd") for n in names) == n_fwd, names
        groups = eng.forward_launches
        assert len(groups) == n_fwd and sum(c for _, c in groups) == len(net.hidden), groups
        assert names[-1] == "wgrad"  # one rank: the step tail runs in k_wgrad's epilogue


def test_apply_trace_matches_oracle(orc):
    """apply (network.hpp:435-448): the readout trace of one batch, forward only."""
    net = Net(inp=40, hidden=(24, 20), classes=6, act="superspike")
    B, T = 5, 30
    params = orc.init(net, orc.key_child(orc.key_from_seed(4), 0)) * np.float32(3.0)
    x, y = orc.synth_raster(net.classes, 12, T, net.inp, 3)
    pk = orc.pack_time(x)
    eng = make_engine(net, B, T)
    eng.stage_dataset(pk, y)
    eng.set_params(params)
    rows = np.array([7, 0, 11, 3, 3], np.uint32)
    tr = eng.apply(rows)
    ref = orc.forward_backward(net, params, pk[rows], T, y[rows], want_grads=False, want_trace=True)
    assert relnorm(tr, ref["trace"]) <= REL_TOL
    assert np.array_equal(eng.get_params(), params)        # forward only: no update
    assert eng.get_opt_state()[2] == 0


def test_evaluate_matches_cmd_eval(orc):
    """cmd_eval (commands.hpp:144-169) after some training: accuracy equals the
    reference's batched walk exactly, and is independent of the batch split
    (commands_test.cpp:199-238: 24 examples as one batch vs 4 x 5 + a tail of 4)."""
    net = Net(inp=40, hidden=(24, 20), classes=4)
    T, N = 25, 24
    x, y = orc.synth_raster(net.classes, N, T, net.inp, 6)
    pk = orc.pack_time(x)
    trainer = make_engine(net, N, T, seed=2)
    trainer.stage_dataset(pk, y)
    for _ in range(6):
        trainer.train_step(np.arange(N, dtype=np.uint32))
    params = trainer.get_params()
    accs = {}
    for B in (24, 5):
        eng = make_engine(net, B, T)
        eng.stage_dataset(pk, y)
        eng.set_params(params)
        acc, loss = eng.evaluate(np.arange(N, dtype=np.uint32))
        ref = orc.eval_accuracy(net, params, pk, y, T, B)
        assert acc == ref, (B, acc, ref)
        assert np.isfinite(loss) and loss > 0
        accs[B] = acc
    assert accs[24] == accs[5]
    assert 0.0 <= accs[24] <= 1.0


OPTION_CASES = [
    ("rate_mse", dict(loss="spike_rate_mse", rate_hi=0.8, rate_lo=0.05)),
    ("sgd", dict(optimizer="sgd", momentum=0.8)),
    ("sgd+rate_mse", dict(optimizer="sgd", momentum=0.5, loss="spike_rate_mse", rate_hi=0.7,
                          rate_lo=0.2)),
]


@pytest.mark.parametrize("case", OPTION_CASES, ids=[c[0] for c in OPTION_CASES])
def test_step_options_match_oracle(orc, case):
    """TrainConfig options on the step: spike-rate MSE (objective.hpp:139-183) and
    SGD + momentum (optimize.hpp:69-84), against the oracle (pinned to the reference
    by tests/golden/opts.npz)."""
    from oracle.pyoracle import Opts
    from paper_2402_18994_b200 import Engine, TrainConfig, shd_spec
    name, kw = case
    o = Opts(optimizer=kw.get("optimizer", "adam"), momentum=kw.get("momentum", 0.9),
             loss="rate_mse" if kw.get("loss") == "spike_rate_mse" else "ce",
             rate_hi=kw.get("rate_hi", 0.9), rate_lo=kw.get("rate_lo", 0.1))
    net = Net(inp=40, hidden=(24, 20), classes=6, act="superspike")
    B, T = 5, 30
    params = orc.init(net, orc.key_child(orc.key_from_seed(8), 0)) * np.float32(3.0)
    x, y = orc.synth_raster(net.classes, B, T, net.inp, 4)
    pk = orc.pack_time(x)
    eng = Engine(shd_spec(hidden=net.hidden, classes=net.classes, inp=net.inp, act=net.act),
                 TrainConfig(batch_size=B, **kw), T)
    eng.stage_dataset(pk, y)
    eng.set_params(params)
    rows = np.arange(B, dtype=np.uint32)
    loss, acc = eng.forward_backward(rows)
    ref = orc.forward_backward(net, params, pk, T, y, opts=o)
    assert abs(loss - ref["loss"]) <= REL_TOL * abs(ref["loss"]) and acc == ref["acc"]
    check_grads(orc, net, eng.get_grads(), ref["grads"])
    st = State(params.copy())
    for _ in range(3):
        lo, ao = orc.train_step(net, st, pk, T, y, opts=o)
        l2, a2 = eng.train_step(rows)
        assert abs(l2 - lo) <= REL_TOL * abs(lo) and a2 == ao
    m, v, step = eng.get_opt_state()
    assert step == 3
    if o.optimizer == "sgd":
        # p -= lr * m is linear in the gradient: the accumulated update carries the
        # gradient tolerance (1e-4 per step, 3 steps)
        assert relnorm(eng.get_params() - params, st.params - params) <= 1e-3
        assert relnorm(m, st.m) <= 1e-3 and not v.any()
    else:
        assert relnorm(eng.get_params(), st.params) <= 1e-4


def test_rate_mse_golden_loss_bit_exact(golden):
    """Rate-MSE loss on the reference-made fixture: logits are bit-exact and the
    (b, c) terms are summed in the reference's single running order."""
    from paper_2402_18994_b200 import Engine, TrainConfig, shd_spec
    g = golden("opts")
    hidden = tuple(int(h) for h in g["hidden"])
    T, B = int(g["t"]), int(g["y"].size)
    eng = Engine(shd_spec(hidden=hidden, classes=int(g["classes"]), inp=int(g["inp"]), act=str(g["act"])),
                 TrainConfig(batch_size=B, loss="spike_rate_mse", rate_hi=0.8, rate_lo=0.05), T)
    eng.stage_dataset(g["packed"], g["y"])
    eng.set_params(g["params"])
    loss, _ = eng.forward_backward(np.arange(B, dtype=np.uint32))
    assert np.float32(loss) == g["rate_mse_loss"]


def test_packed_entry_pinned_caller_buffer(orc):
    """A caller batch in pinned memory is DMA'd directly; results equal the
    pageable-buffer path (staged through the copy pool) bit for bit."""
    import torch
    net = Net(inp=30, hidden=(16, 12), classes=5)
    x, y = orc.synth_raster(5, 4, 19, 30, 2)
    pk = orc.pack_time(x)
    pinned = torch.empty(pk.shape, dtype=torch.uint8, pin_memory=True)
    pinned.numpy()[...] = pk
    e1, e2 = make_engine(net, 4, 19), make_engine(net, 4, 19)
    for _ in range(2):
        assert e1.train_step_packed(pk, y) == e2.train_step_packed(pinned.numpy(), y)
    assert np.array_equal(e1.get_params(), e2.get_params())


def test_single_rank_nccl_tail_matches_fused_tail(orc):
    """The multi-rank tail (k_reduce -> ncclAllReduce -> k_adam) on a one-rank NCCL
    communicator gives bit-identical training to the fused single-rank tail."""
    from paper_2402_18994_b200 import DeviceError, Engine
    net = Net(inp=30, hidden=(16, 12), classes=5)
    x, y = orc.synth_raster(5, 8, 19, 30, 2)
    pk = orc.pack_time(x)
    e1, e2 = make_engine(net, 4, 19, seed=3), make_engine(net, 4, 19, seed=3)
    try:
        e2.comm_init(Engine.nccl_unique_id(), 0, 1)
    except DeviceError as err:
        pytest.skip(f"NCCL unavailable: {err}")
    # one rank runs its tail inside k_wgrad; NCCL: k_reduce + (allreduce) + k_adam
    assert e2.launches_per_step == e1.launches_per_step + 2
    for eng in (e1, e2):
        eng.stage_dataset(pk, y)
    for i in range(4):
        rows = np.arange(4 * (i % 2), 4 * (i % 2) + 4, dtype=np.uint32)
        assert e1.train_step(rows) == e2.train_step(rows)
    assert np.array_equal(e1.get_params(), e2.get_params())
    m1, v1, s1 = e1.get_opt_state()
    m2, v2, s2 = e2.get_opt_state()
    assert s1 == s2 == 4 and np.array_equal(m1, m2) and np.array_equal(v1, v2)
    assert e1.forward_backward(np.arange(4, dtype=np.uint32)) == e2.forward_backward(np.arange(4, dtype=np.uint32))
    assert np.array_equal(e1.get_grads(), e2.get_grads())


CKPT_NET = Net(inp=30, hidden=(16, 12), classes=5, bias=True, act="arctan", unroll=4)


@pytest.mark.parametrize("opt", ["adam", "sgd"])
def test_checkpoint_matches_reference_file(golden, tmp_path, opt):
    """.spkc files written by the reference itself (tests/golden/ckpt_*.spkc):
    the engine loads them exactly and writes the same bytes back."""
    import os
    from paper_2402_18994_b200 import Engine, TrainConfig, shd_spec
    g = golden("ckpt")
    spec = shd_spec(hidden=CKPT_NET.hidden, classes=CKPT_NET.classes, inp=CKPT_NET.inp,
                    act=CKPT_NET.act, bias=True)
    eng = Engine(spec, TrainConfig(batch_size=4, optimizer=opt, momentum=0.9), 19)
    src = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", f"ckpt_{opt}.spkc")
    cfg = eng.load_checkpoint(src)
    assert cfg.encode() == g["config"].tobytes()
    assert np.array_equal(eng.get_params(), g[f"{opt}_params"])
    m, v, step = eng.get_opt_state()
    assert step == int(g[f"{opt}_step"])
    assert np.array_equal(m, g[f"{opt}_m"]) and (opt == "sgd" or np.array_equal(v, g[f"{opt}_v"]))
    out = tmp_path / "out.spkc"
    eng.save_checkpoint(str(out), cfg)
    assert out.read_bytes() == open(src, "rb").read()


def test_checkpoint_resume_is_bit_exact(orc, tmp_path):
    """optimize_test.cpp:257-290: training resumed from a checkpoint continues
    bit-identically; errors map to the reference classes."""
    from paper_2402_18994_b200 import FormatError, IoError, ShapeError
    x, y = orc.synth_raster(5, 8, 19, 30, 2)
    pk = orc.pack_time(x)
    a = make_engine(CKPT_NET, 4, 19, seed=6)
    a.stage_dataset(pk, y)
    rows = [np.arange(4 * (i % 2), 4 * (i % 2) + 4, dtype=np.uint32) for i in range(5)]
    for r in rows[:3]:
        a.train_step(r)
    path = str(tmp_path / "mid.spkc")
    a.save_checkpoint(path, "resume test")
    b = make_engine(CKPT_NET, 4, 19, seed=99)
    b.stage_dataset(pk, y)
    assert b.load_checkpoint(path) == "resume test"
    for r in rows[3:]:
        assert a.train_step(r) == b.train_step(r)
    assert np.array_equal(a.get_params(), b.get_params())
    with pytest.raises(IoError):
        b.load_checkpoint(str(tmp_path / "missing.spkc"))
    bad = tmp_path / "bad.spkc"
    bad.write_bytes(b"XXXX" + open(path, "rb").read()[4:])
    with pytest.raises(FormatError):
        b.load_checkpoint(str(bad))
    other = make_engine(Net(inp=30, hidden=(16, 12), classes=5), 4, 19)  # no bias entries
    with pytest.raises(ShapeError):
        other.load_checkpoint(path)


BETA_NET = Net(inp=40, hidden=(24, 20), classes=6, act="superspike", bias=True,
               beta_mode=("scalar", "fixed", "scalar"), fixed_beta=(0.5, 0.3, 0.5), unroll=9)


def beta_engine(net, B, T, **kw):
    from paper_2402_18994_b200 import (Engine, LIFLayer, LILayer, LinearLayer, NetworkSpec,
                                       TrainConfig, default_activation_desc)
    layers = []
    for i, h in enumerate(net.hidden):
        layers += [LinearLayer(h, net.bias),
                   LIFLayer(default_activation_desc(net.act), beta_mode=net.beta_mode[i],
                            fixed_beta=net.fixed_beta[i])]
    layers += [LinearLayer(net.classes, net.bias),
               LILayer(beta_mode=net.beta_mode[-1], fixed_beta=net.fixed_beta[-1])]
    return Engine(NetworkSpec([net.inp], layers), TrainConfig(batch_size=B, **kw), T)


def test_beta_modes_match_reference_fixture(orc, golden):
    """BetaMode::LearnableScalar / Fixed cells (neuron.hpp:56-76): init bit-exact,
    loss / gradients / 3 Adam steps against the reference-made fixture."""
    g = golden("betamodes")
    T, B = 30, int(g["y"].size)
    eng = beta_engine(BETA_NET, B, T, seed=23)
    assert np.array_equal(eng.get_params(), g["init"])
    eng.stage_dataset(g["packed"], g["y"])
    eng.set_params(g["params"])
    rows = np.arange(B, dtype=np.uint32)
    loss, _ = eng.forward_backward(rows)
    assert abs(loss - g["loss"]) <= REL_TOL * abs(g["loss"])
    check_grads(orc, BETA_NET, eng.get_grads(), g["grads"])
    for i in range(3):
        l2, _ = eng.train_step(rows)
        assert abs(l2 - g["step_losses"][i]) <= REL_TOL * abs(g["step_losses"][i])
    assert relnorm(eng.get_params(), g["params3"]) <= 1e-4
    o = {n: (off, sz) for n, off, sz in orc.entries(BETA_NET)}
    off, sz = o["l3.beta"]                    # fixed: untouched, no optimizer state
    assert sz == 1 and eng.get_params()[off] == g["params"][off] == g["params3"][off]
    m, v, _ = eng.get_opt_state()
    assert m[off] == 0 and v[off] == 0


SHIFTS = {"one_axis": dict(max_shift=3, shift_axes=(2,)), "two_axes": dict(max_shift=5, shift_axes=(2, -1))}


@pytest.mark.parametrize("name", list(SHIFTS))
def test_shift_augment_matches_reference_fixture(orc, golden, name):
    """Epoch loop with shift_augment (data.hpp:216-227, optimize.hpp:276-278): two
    epochs against the reference's own run (tests/golden/shift.npz)."""
    g = golden("shift")
    net = Net(inp=int(g["inp"]), hidden=tuple(int(h) for h in g["hidden"]), classes=int(g["classes"]),
              bias=bool(g["bias"]), threshold=float(g["threshold"]), act=str(g["act"]),
              unroll=int(g["unroll"]))
    eng = make_engine(net, 4, int(g["t"]), seed=9, **SHIFTS[name])
    eng.stage_dataset(g["packed"], g["y"])
    eng.set_params(g["params"])
    m = eng.train_epochs(2)
    ref = g[f"{name}_metrics"]
    assert np.allclose(m[:, 0], ref[:, 0], rtol=1e-4), (m, ref)
    assert np.array_equal(m[:, 1], ref[:, 1])
    assert relnorm(eng.get_params(), g[f"{name}_params"]) <= 1e-4
    assert eng.get_opt_state()[2] == int(g[f"{name}_step"])
    # a following plain step is unshifted again
    st = State(eng.get_params().copy())
    rows = np.arange(4, dtype=np.uint32)
    fb = orc.forward_backward(net, st.params, g["packed"][:4], int(g["t"]), g["y"][:4])
    loss, _ = eng.forward_backward(rows)
    assert abs(loss - fb["loss"]) <= REL_TOL * abs(fb["loss"])


def test_shift_augment_c1_shape_matches_oracle(orc):
    """C1 shape (700 inputs, 11 padding features) with rolls up to +-40 over 2 epochs."""
    from oracle.pyoracle import Opts
    net = Net()
    B, N, T = 64, 192, 128
    x, y = orc.synth_raster(20, N, T, 700, 4)
    pk = orc.pack_time(x)
    eng = make_engine(net, B, T, seed=3, max_shift=40, shift_axes=(2, -1))
    eng.stage_dataset(pk, y)
    p0 = eng.get_params()
    m_gpu = eng.train_epochs(2)
    st = State(p0.copy())
    m_ref = orc.train_epochs(net, st, pk, y, T, B, 2, 3, opts=Opts(max_shift=40, shift_axes=(2, -1)))
    assert np.allclose(m_gpu[:, 0], m_ref[:, 0], rtol=1e-3), (m_gpu, m_ref)
    assert np.abs(m_gpu[:, 1] - m_ref[:, 1]).max() <= 1.0 / B + 1e-12
    assert relnorm(eng.get_params(), st.params) <= 1e-4


def test_shift_axes_validation():
    """train() rejects axes 0 / 1 (optimize.hpp:241-245); other non-feature rolls
    are refused as unsupported; max_shift <= 0 accepts any other axis."""
    from paper_2402_18994_b200 import ArgumentError, UnsupportedError
    net = Net(inp=30, hidden=(16,), classes=5)
    for axes in ((0,), (1,), (2, 1)):
        with pytest.raises(ArgumentError):
            make_engine(net, 2, 16, max_shift=2, shift_axes=axes)
    with pytest.raises(ArgumentError):
        make_engine(net, 2, 16, max_shift=0, shift_axes=(1,))
    with pytest.raises(UnsupportedError):
        make_engine(net, 2, 16, max_shift=2, shift_axes=(-2,))
    make_engine(net, 2, 16, max_shift=0, shift_axes=(3,))


ACT_OPTS = {"both": dict(lambda_low=0.5, lambda_high=2.0, f_min=0.1, f_max=0.3),
            "high": dict(lambda_high=1.5, f_max=0.05)}


def _act_net(g):
    return Net(inp=int(g["inp"]), hidden=tuple(int(h) for h in g["hidden"]), classes=int(g["classes"]),
               bias=bool(g["bias"]), threshold=float(g["threshold"]), act=str(g["act"]),
               unroll=int(g["unroll"]), monitor=tuple(int(m) for m in g["monitor"]))


@pytest.mark.parametrize("name", list(ACT_OPTS))
def test_activity_regularizer_matches_reference_fixture(orc, golden, name):
    """MonitorLayer + activity regularizer (objective.hpp:186-227, optimize.hpp:185-191)
    against the reference's own numbers: init and entry names with the shifted
    layer ids, loss and grads of one step, three train_steps."""
    g = golden("activity")
    net = _act_net(g)
    T = int(g["t"])
    eng = make_engine(net, 7, T, seed=41, **ACT_OPTS[name])
    assert np.array_equal(eng.get_params(), g["params_init"]), "init keys with monitors"
    assert [e[0] for e in eng.entries()] == [str(n) for n in g["names"]]
    eng.stage_dataset(g["packed"], g["y"])
    eng.set_params(g["params"])
    rows = np.arange(7, dtype=np.uint32)
    loss, _ = eng.forward_backward(rows)
    assert abs(loss - g[f"{name}_loss"]) <= REL_TOL * abs(g[f"{name}_loss"])
    check_grads(orc, net, eng.get_grads(), g[f"{name}_grads"])
    losses = [eng.train_step(rows)[0] for _ in range(3)]
    assert np.allclose(losses, g[f"{name}_step_losses"], rtol=REL_TOL, atol=0)
    assert relnorm(eng.get_params(), g[f"{name}_params3"]) <= 1e-4


def test_activity_regularizer_c1_shape_matches_oracle(orc):
    """C1 shape (B=64) with monitors on both LIF layers, both hinge sides active."""
    from oracle.pyoracle import Opts
    net = Net(monitor=(0, 1))
    B, T = 64, 128
    params = orc.init(net, orc.key_child(orc.key_from_seed(2), 0)) * np.float32(2.0)
    x, y = orc.synth_raster(20, B, T, 700, 6)
    pk = orc.pack_time(x)
    # strong enough that the regularizer moves the gradient ~50x the parity bar
    kw = dict(lambda_low=3000.0, lambda_high=4500.0, f_min=0.05, f_max=0.2)
    eng = make_engine(net, B, T, **kw)
    eng.stage_dataset(pk, y)
    eng.set_params(params)
    rows = np.arange(B, dtype=np.uint32)
    loss, _ = eng.forward_backward(rows)
    ref = orc.forward_backward(net, params, pk, T, y, opts=Opts(**kw), want_spikes=True)
    plain = orc.forward_backward(net, params, pk, T, y)
    assert abs(loss - ref["loss"]) <= REL_TOL * abs(ref["loss"])
    assert ref["loss"] > plain["loss"] and relnorm(ref["grads"], plain["grads"]) > 3e-3, "regularizer inactive"
    check_grads(orc, net, eng.get_grads(), ref["grads"])
    # ApplyResult.monitors: spike counts of the same forward
    for l in range(2):
        assert np.array_equal(eng.monitor_counts(l), ref["spikes"][l].sum(axis=1).astype(np.float32))
    # the update path (fused tail) reports the same loss, and the histogram resets per step
    l1, _ = eng.train_step(rows)
    assert abs(l1 - ref["loss"]) <= REL_TOL * abs(ref["loss"])
    l2, _ = eng.forward_backward(rows)
    ref2 = orc.forward_backward(net, eng.get_params(), pk, T, y, opts=Opts(**kw))
    assert abs(l2 - ref2["loss"]) <= REL_TOL * abs(ref2["loss"])


def test_activity_regularizer_nccl_tail_matches_fused_tail(orc):
    """Regularizer values travel through the allreduce buffer on the multi-rank tail."""
    from paper_2402_18994_b200 import DeviceError, Engine
    net = Net(inp=30, hidden=(16, 12), classes=5, monitor=(1,))
    x, y = orc.synth_raster(5, 8, 19, 30, 2)
    pk = orc.pack_time(x)
    kw = dict(lambda_low=0.5, lambda_high=0.5, f_min=0.2, f_max=0.4)
    e1, e2 = make_engine(net, 4, 19, seed=3, **kw), make_engine(net, 4, 19, seed=3, **kw)
    try:
        e2.comm_init(Engine.nccl_unique_id(), 0, 1)
    except DeviceError as err:
        pytest.skip(f"NCCL unavailable: {err}")
    for eng in (e1, e2):
        eng.stage_dataset(pk, y)
    for i in range(3):
        rows = np.arange(4 * (i % 2), 4 * (i % 2) + 4, dtype=np.uint32)
        assert e1.train_step(rows) == e2.train_step(rows)
    assert np.array_equal(e1.get_params(), e2.get_params())


def test_monitor_spec_errors():
    from paper_2402_18994_b200 import (ArgumentError, Engine, LIFLayer, LILayer, LinearLayer,
                                       MonitorLayer, NetworkSpec, SpecError, TrainConfig)
    bad = NetworkSpec([30], [LinearLayer(16), MonitorLayer(), LIFLayer(), LinearLayer(5), LILayer()])
    with pytest.raises(SpecError):
        Engine(bad, TrainConfig(batch_size=2), 16)
    twice = NetworkSpec([30], [LinearLayer(16), LIFLayer(), MonitorLayer(), MonitorLayer(),
                               LinearLayer(5), LILayer()])
    with pytest.raises(SpecError):
        Engine(twice, TrainConfig(batch_size=2), 16)
    ok = NetworkSpec([30], [LinearLayer(16), LIFLayer(), MonitorLayer(), LinearLayer(5), LILayer()])
    with pytest.raises(ArgumentError):
        Engine(ok, TrainConfig(batch_size=2, lambda_low=1.0, f_min=0.6, f_max=0.3), 16)
    eng = Engine(ok, TrainConfig(batch_size=2, f_min=0.6, f_max=0.3), 16)  # lambdas 0: unchecked
    with pytest.raises(ArgumentError):
        eng.monitor_counts(1)


def test_single_rank_peer_tail_matches_fused_tail(orc):
    """The peer-memory tail (k_reduce -> k_peer_owner -> k_peer_gather) on one rank
    trains bit-identically to the fused single-rank tail."""
    net = Net(inp=30, hidden=(16, 12), classes=5)
    x, y = orc.synth_raster(5, 8, 19, 30, 2)
    pk = orc.pack_time(x)
    e1, e2 = make_engine(net, 4, 19, seed=3), make_engine(net, 4, 19, seed=3)
    e2.peer_open(0, 1, [e2.peer_handle()])
    assert e2.launches_per_step == e1.launches_per_step + 3  # k_reduce, k_peer_owner, k_peer_gather
    for eng in (e1, e2):
        eng.stage_dataset(pk, y)
    for i in range(4):
        rows = np.arange(4 * (i % 2), 4 * (i % 2) + 4, dtype=np.uint32)
        assert e1.train_step(rows) == e2.train_step(rows)
    assert np.array_equal(e1.get_params(), e2.get_params())
    m1, v1, s1 = e1.get_opt_state()
    m2, v2, s2 = e2.get_opt_state()
    assert s1 == s2 == 4 and np.array_equal(m1, m2) and np.array_equal(v1, v2)
    assert e1.forward_backward(np.arange(4, dtype=np.uint32)) == e2.forward_backward(np.arange(4, dtype=np.uint32))
    assert np.array_equal(e1.get_grads(), e2.get_grads())
    # schedule mode (8-step graphs) through the peer tail
    sched = np.arange(8 * 4, dtype=np.uint32) % 8
    for eng in (e1, e2):
        eng.upload_schedule(sched.reshape(8, 4))
        eng.enqueue_steps(0, 8)
        eng.sync()
    assert np.array_equal(e1.get_params(), e2.get_params())


@pytest.mark.parametrize("world,cell", [(2, ()), (3, ()), (2, ("alif", "rlif"))],
                         ids=["2ranks", "3ranks", "2ranks-alif-rlif"])
def test_peer_tail_ranks_emulated_on_one_gpu(orc, world, cell):
    """`world` ranks of the peer tail on one GPU (B200_PROFILING: never let ranks
    wait on each other as separate launches -- every rank runs its part before the
    cross-rank wait, then every rank runs the tail).  Replicas stay bit-identical and
    match full-global-batch training on the oracle."""
    from paper_2402_18994_b200 import Engine
    net = Net(inp=40, hidden=(24, 20), classes=5, act="superspike", cell=cell)
    B, T, N = 4, 23, 48
    x, y = orc.synth_raster(5, N, T, 40, 8)
    pk = orc.pack_time(x)
    engs = [make_engine(net, B, T, seed=5) for _ in range(world)]
    Engine.peer_attach_local(engs)
    p0 = engs[0].get_params()
    for name, off, size in orc.entries(net):  # louder weights (gamma / beta keep their init)
        if name.endswith((".w", ".rec")):
            p0[off:off + size] *= np.float32(3.0)
    for e in engs:
        e.stage_dataset(pk, y)
        e.set_params(p0)
    st = State(p0.copy())
    perm = orc.permutation(orc.key_from_seed(17), N)
    for step in range(3):
        gb = perm[step * B * world:(step + 1) * B * world].astype(np.uint32)
        ref = orc.forward_backward(net, st.params, pk[gb], T, y[gb])
        for r, e in enumerate(engs):
            e.train_step_split(gb[r * B:(r + 1) * B], 0)
        for e in engs:                      # owner phase: each rank updates its slice
            e.train_step_split(None, 1)
        res = [e.train_step_split(None, 2) for e in engs]   # gather the owners' slices
        assert all(r == res[0] for r in res), res
        assert abs(res[0][0] - ref["loss"]) <= REL_TOL * abs(ref["loss"])
        assert res[0][1] == ref["acc"]
        g = engs[0].get_grads()
        check_grads(orc, net, g, ref["grads"])
        for e in engs[1:]:
            assert np.array_equal(e.get_grads(), g)
        orc.train_step(net, st, pk[gb], T, y[gb])
        params = [e.get_params() for e in engs]
        assert all(np.array_equal(p, params[0]) for p in params), "replicas diverged"
        if step == 0:
            check_adam_step(orc, net, params[0], st.params, ref["grads"])
        st.params = params[0].copy()  # follow the engine (Adam's sign flips on tiny grads)
        m, v, s = engs[0].get_opt_state()
        st.m, st.v, st.step = m, v, s


def _ipc_rank(rank, port, out):
    """One process per rank on GPU 0: real IPC handle export / all-gather / open, then
    split steps with a barrier between the parts (every flag is set before any rank's
    tail runs, so no kernel waits on a rank that has not run)."""
    import os
    import torch.distributed as dist
    from oracle.pyoracle import Lib
    from paper_2402_18994_b200.parallel import setup_data_parallel
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    orc = Lib("orc")
    net = Net(inp=40, hidden=(24, 20), classes=5, act="superspike")
    x, y = orc.synth_raster(5, 32, 23, 40, 8)
    pk = orc.pack_time(x)
    eng = make_engine(net, 4, 23, seed=5)
    setup_data_parallel(eng, rank, 2, dist, "peer")
    eng.stage_dataset(pk, y)
    eng.set_params(eng.get_params() * np.float32(3.0))
    res = []
    for step in range(3):
        rows = np.arange(step * 8 + rank * 4, step * 8 + rank * 4 + 4, dtype=np.uint32)
        eng.train_step_split(rows, 0)
        dist.barrier()
        eng.train_step_split(None, 1)
        dist.barrier()
        res.append(eng.train_step_split(None, 2))
        dist.barrier()
    out[rank] = (res, eng.get_params(), eng.get_grads())
    dist.destroy_process_group()


def test_peer_tail_over_real_ipc_two_processes(orc):
    import socket
    import torch.multiprocessing as tmp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = tmp.Manager().dict()
    tmp.spawn(_ipc_rank, args=(port, out), nprocs=2, join=True)
    (r0, p0, g0), (r1, p1, g1) = out[0], out[1]
    assert r0 == r1 and np.array_equal(p0, p1) and np.array_equal(g0, g1)
    # same three global batches on one in-process 8-sample engine
    net = Net(inp=40, hidden=(24, 20), classes=5, act="superspike")
    x, y = orc.synth_raster(5, 32, 23, 40, 8)
    pk = orc.pack_time(x)
    ref = make_engine(net, 8, 23, seed=5)
    ref.stage_dataset(pk, y)
    ref.set_params(ref.get_params() * np.float32(3.0))
    for step in range(3):
        l, a = ref.train_step(np.arange(step * 8, step * 8 + 8, dtype=np.uint32))
        assert abs(l - r0[step][0]) <= REL_TOL * abs(l) and a == r0[step][1]
    assert relnorm(p0, ref.get_params()) <= 1e-5


def test_container_load_save_matches_reference_files(golden, tmp_path):
    """.spkd I/O (data.hpp:229-341) against files written by the reference's own
    write_container: load stages the same bytes (flat and [N, T', 5, 8] feature
    shapes), save reproduces the reference's file byte for byte."""
    import os
    g = golden("spkd")
    gold = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    net = Net(inp=40, hidden=(16,), classes=5)
    eng = make_engine(net, 2, int(g["t"]))
    for name in ("flat.spkd", "multi.spkd"):
        assert eng.load_container(os.path.join(gold, name)) == 6
        pk, y = eng.read_dataset(0, 6)
        assert np.array_equal(pk, g["packed"]) and np.array_equal(y, g["y"])
    out = tmp_path / "saved.spkd"
    eng.save_container(str(out))
    assert out.read_bytes() == open(os.path.join(gold, "flat.spkd"), "rb").read()


def test_container_errors_match_reference_classes(tmp_path):
    import os
    from paper_2402_18994_b200 import FormatError, IoError, ShapeError
    gold = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    raw = open(os.path.join(gold, "flat.spkd"), "rb").read()
    eng = make_engine(Net(inp=40, hidden=(16,), classes=5), 2, 21)
    with pytest.raises(IoError):
        eng.load_container(str(tmp_path / "missing.spkd"))
    cases = {"magic": b"SPKX" + raw[4:], "version": raw[:4] + b"\x02" + raw[5:],
             "truncated": raw[:-7], "dtype": raw[:8] + b"\x01" + raw[9:]}
    for name, data in cases.items():
        p = tmp_path / f"{name}.spkd"
        p.write_bytes(data)
        with pytest.raises(FormatError):
            eng.load_container(str(p))
    other_t = make_engine(Net(inp=40, hidden=(16,), classes=5), 2, 30)
    with pytest.raises(FormatError):
        other_t.load_container(os.path.join(gold, "flat.spkd"))
    other_in = make_engine(Net(inp=41, hidden=(16,), classes=5), 2, 21)
    with pytest.raises(ShapeError):
        other_in.load_container(os.path.join(gold, "flat.spkd"))


# ---------------------------------------------------------------------------
# Declared ALIF cell (BASELINE config 2; not in the reference -- the checker is
# the oracle's restatement, itself pinned to float64 autograd in
# tests/test_alif_oracle.py).  Forward V / a / spikes bit-exact given the GPU's
# projection; loss and gradients (gamma included) within the north_star bar.
ALIF_CASES = [
    ("alif-tiny", Net(inp=30, hidden=(16, 12), classes=5, act="superspike", cell=("alif", "alif")), 6, 19, 3.0),
    ("alif-c2-shape", Net(act="superspike", cell=("alif", "alif")), 8, 128, 2.0),
    ("alif-lif-T200", Net(inp=64, hidden=(128, 128), classes=10, cell=("alif", "lif")), 3, 200, 2.0),
    ("alif-bias-3hidden", Net(inp=50, hidden=(64, 48, 32), classes=6, act="triangular", bias=True,
                              cell=("lif", "alif", "alif")), 4, 33, 3.0),
    ("alif-T1000", Net(inp=64, hidden=(96,), classes=5, act="superspike", cell=("alif",)), 2, 1000, 2.0),
]


@pytest.mark.parametrize("case", ALIF_CASES, ids=[c[0] for c in ALIF_CASES])
def test_alif_step_parity(orc, case):
    _, net, B, T, scale = case
    params = orc.init(net, orc.key_child(orc.key_from_seed(21), 0))
    ents = orc.entries(net)
    for n, o, s in ents:
        if n.endswith(".w"):
            params[o:o + s] *= np.float32(scale)
    x, y = orc.synth_raster(net.classes, B, T, net.inp, 5)
    pk = orc.pack_time(x)
    eng = make_engine(net, B, T)
    names = [n for n, _, _ in ents]
    assert eng.entries() == ents
    assert np.array_equal(eng.get_params(), orc.init(net, orc.key_child(orc.key_from_seed(0), 0)))
    eng.stage_dataset(pk, y)
    eng.set_params(params)
    eng.debug(True)
    rows = np.arange(B, dtype=np.uint32)
    loss, acc = eng.forward_backward(rows)
    ref = orc.forward_backward(net, params, pk, T, y, want_spikes=True, want_trace=True)
    emap = {n: (o, s) for n, o, s in ents}
    flips = 0
    for l, h in enumerate(net.hidden):
        I = eng.fetch("I", l)
        cell = names[names.index(f"l{2 * l}.w") + (2 if net.bias else 1)][:-5]
        o, s = emap[cell + ".beta"]
        S = eng.fetch("spikes", l)
        if net.cell[l] == "alif":
            go, gs = emap[cell + ".gamma"]
            V_ref, A_ref, S_ref = scanref.alif_forward(I, params[o:o + s], params[go:go + gs], net.threshold)
            assert np.array_equal(eng.fetch("A", l), A_ref), f"layer {l}: a not bit-exact given I"
        else:
            V_ref, S_ref = scanref.lif_forward(I, params[o:o + s], net.threshold)
        assert np.array_equal(eng.fetch("V", l), V_ref), f"layer {l}: V not bit-exact given I"
        assert np.array_equal(S, S_ref), f"layer {l}: spikes not bit-exact given I"
        agree = (S == ref["spikes"][l]).mean()
        assert agree >= SPIKE_AGREE, agree
        flips += int((S != ref["spikes"][l]).sum())
        assert 0.005 < S.mean() < 0.9, f"layer {l}: rate {S.mean()}"
    assert abs(loss - ref["loss"]) <= REL_TOL * abs(ref["loss"])
    if flips == 0:
        check_grads(orc, net, eng.get_grads(), ref["grads"])
    else:  # 1e-4 against the teacher-forced oracle (the GPU's own rasters)
        Sg = [eng.fetch("spikes", l) for l in range(len(net.hidden))]
        check_grads(orc, net, eng.get_grads(),
                    orc.forward_backward(net, params, pk, T, y, forced=Sg)["grads"])
    st = State(params.copy())
    lo, ao = orc.train_step(net, st, pk, T, y)
    eng.debug(False)
    l2, a2 = eng.train_step(rows)
    assert abs(l2 - lo) <= REL_TOL * abs(lo) and a2 == ao
    check_adam_step(orc, net, eng.get_params(), st.params, ref["grads"])


def test_alif_training_curve(orc):
    """C2-shaped ALIF training (superspike) over 3 epochs tracks the oracle."""
    net = Net(act="superspike", cell=("alif", "alif"))
    N, B, T = 64, 16, 128
    x, y = orc.synth_raster(net.classes, N, T, net.inp, 1)
    pk = orc.pack_time(x)
    params = orc.init(net, orc.key_child(orc.key_from_seed(0), 0))
    st = State(params.copy())
    m_ref = orc.train_epochs(net, st, pk, y, T, B, 3, 0)
    eng = make_engine(net, B, T, seed=0)
    eng.stage_dataset(pk, y)
    m_gpu = eng.train_epochs(3)
    assert np.allclose(m_gpu[:, 0], m_ref[:, 0], rtol=1e-3), (m_gpu, m_ref)
    assert np.abs(m_gpu[:, 1] - m_ref[:, 1]).max() <= 1.0 / B + 1e-12
    # 12 Adam steps of ~lr * sign(g): elements whose gradient nearly cancels can move
    # the other way (check_adam_step), so the parameter bound after training is 5e-4
    assert relnorm(eng.get_params(), st.params) <= 5e-4


# ---------------------------------------------------------------------------
# Declared RLIF cell (BASELINE config 4; not in the reference -- checker: the
# oracle's restatement, pinned to float64 autograd in tests/test_alif_oracle.py).
# Forward V / spikes bit-exact given the GPU's projection (the feedback sum runs
# over the spiking sources in the oracle's ascending order); loss and gradients
# (rec included) within the north_star bar.
RLIF_CASES = [
    ("rlif-tiny", Net(inp=30, hidden=(16, 12), classes=5, cell=("rlif", "rlif")), 6, 19, 3.0),
    ("rlif-c4-shape", Net(hidden=(512, 512), act="arctan", cell=("rlif", "rlif")), 3, 128, 2.0),
    ("lif-rlif-T200-bias", Net(inp=64, hidden=(128, 96), classes=8, act="superspike", bias=True,
                               cell=("lif", "rlif")), 3, 200, 2.0),
    ("rlif-alif-3hidden", Net(inp=50, hidden=(64, 48, 32), classes=6, act="triangular",
                              cell=("rlif", "alif", "lif")), 4, 33, 3.0),
    # cluster scans (H_pad 256): two sample groups of the cluster, the second partial
    ("rlif-256-cluster", Net(inp=100, hidden=(250,), classes=6, act="boxcar", bias=True,
                             cell=("rlif",)), 20, 70, 2.0),
]


@pytest.mark.parametrize("case", RLIF_CASES, ids=[c[0] for c in RLIF_CASES])
def test_rlif_step_parity(orc, case):
    _, net, B, T, scale = case
    params = orc.init(net, orc.key_child(orc.key_from_seed(31), 0))
    ents = orc.entries(net)
    for n, o, s in ents:
        if n.endswith(".w"):
            params[o:o + s] *= np.float32(scale)
    x, y = orc.synth_raster(net.classes, B, T, net.inp, 5)
    pk = orc.pack_time(x)
    eng = make_engine(net, B, T)
    names = [n for n, _, _ in ents]
    assert eng.entries() == ents
    assert np.array_equal(eng.get_params(), orc.init(net, orc.key_child(orc.key_from_seed(0), 0)))
    eng.stage_dataset(pk, y)
    eng.set_params(params)
    eng.debug(True)
    rows = np.arange(B, dtype=np.uint32)
    loss, acc = eng.forward_backward(rows)
    ref = orc.forward_backward(net, params, pk, T, y, want_spikes=True, want_trace=True)
    emap = {n: (o, s) for n, o, s in ents}
    flips = 0
    for l, h in enumerate(net.hidden):
        I = eng.fetch("I", l)
        cell = names[names.index(f"l{2 * l}.w") + (2 if net.bias else 1)][:-5]
        o, s = emap[cell + ".beta"]
        S = eng.fetch("spikes", l)
        if net.cell[l] == "rlif":
            ro, rs = emap[cell + ".rec"]
            V_ref, S_ref = scanref.rlif_forward(I, params[o:o + s], params[ro:ro + rs], net.threshold)
        elif net.cell[l] == "alif":
            go, gs = emap[cell + ".gamma"]
            V_ref, _, S_ref = scanref.alif_forward(I, params[o:o + s], params[go:go + gs], net.threshold)
        else:
            V_ref, S_ref = scanref.lif_forward(I, params[o:o + s], net.threshold)
        assert np.array_equal(eng.fetch("V", l), V_ref), f"layer {l}: V not bit-exact given I"
        assert np.array_equal(S, S_ref), f"layer {l}: spikes not bit-exact given I"
        agree = (S == ref["spikes"][l]).mean()
        assert agree >= SPIKE_AGREE, agree
        flips += int((S != ref["spikes"][l]).sum())
        assert 0.005 < S.mean() < 0.9, f"layer {l}: rate {S.mean()}"
    assert abs(loss - ref["loss"]) <= REL_TOL * abs(ref["loss"])
    if flips == 0:
        check_grads(orc, net, eng.get_grads(), ref["grads"])
    else:  # 1e-4 against the teacher-forced oracle (the GPU's own rasters)
        Sg = [eng.fetch("spikes", l) for l in range(len(net.hidden))]
        check_grads(orc, net, eng.get_grads(),
                    orc.forward_backward(net, params, pk, T, y, forced=Sg)["grads"])
    st = State(params.copy())
    lo, ao = orc.train_step(net, st, pk, T, y)
    eng.debug(False)
    l2, a2 = eng.train_step(rows)
    assert abs(l2 - lo) <= REL_TOL * abs(lo) and a2 == ao
    check_adam_step(orc, net, eng.get_params(), st.params, ref["grads"])
    # a second step runs on the Adam-refreshed rec^T (k_rlif_bwd's copy)
    l3, _ = eng.train_step(rows)
    lo3, _ = orc.train_step(net, st, pk, T, y)
    assert abs(l3 - lo3) <= 1e-3 * abs(lo3)


def test_declared_cells_checkpoint_apply_monitor(orc, tmp_path):
    """The declared cells through the rest of the API: .spkc save / load with the
    gamma and rec entries (resume bit-exact), apply, evaluate, a monitored ALIF layer
    with the activity regularizer, and SGD."""
    from paper_2402_18994_b200 import ShapeError
    net = Net(inp=40, hidden=(24, 256), classes=5, act="superspike", cell=("alif", "rlif"),
              monitor=(0,))
    B, T = 16, 30
    x, y = orc.synth_raster(5, 32, T, 40, 4)
    pk = orc.pack_time(x)
    kw = dict(optimizer="sgd", lambda_low=0.5, lambda_high=0.5, f_min=0.05, f_max=0.2)
    a = make_engine(net, B, T, seed=3, **kw)
    a.stage_dataset(pk, y)
    p0 = a.get_params()
    for n, o, s in orc.entries(net):
        if n.endswith(".w"):
            p0[o:o + s] *= np.float32(3.0)
    a.set_params(p0)
    rows = [np.arange(16 * (i % 2), 16 * (i % 2) + 16, dtype=np.uint32) for i in range(5)]
    for r in rows[:2]:
        a.train_step(r)
    path = str(tmp_path / "cells.spkc")
    a.save_checkpoint(path, "declared cells")
    b = make_engine(net, B, T, seed=11, **kw)
    b.stage_dataset(pk, y)
    assert b.load_checkpoint(path) == "declared cells"
    assert np.array_equal(a.get_params(), b.get_params())
    for r in rows[2:]:
        assert a.train_step(r) == b.train_step(r)
    assert np.array_equal(a.get_params(), b.get_params())
    # forward-only entries on the trained declared network agree with the oracle
    params = a.get_params()
    ref = orc.forward_backward(net, params, pk[rows[0]], T, y[rows[0]], want_grads=False,
                               want_trace=True, want_spikes=True)
    assert relnorm(a.apply(rows[0]), ref["trace"]) <= REL_TOL
    counts = a.monitor_counts(0)
    assert (counts == ref["spikes"][0].sum(axis=1)).mean() >= 0.999
    acc, loss = a.evaluate(np.arange(32, dtype=np.uint32))
    assert 0.0 <= acc <= 1.0 and np.isfinite(loss)
    # a LIF network cannot load the declared network's checkpoint (entry shapes differ)
    c = make_engine(Net(inp=40, hidden=(24, 256), classes=5, monitor=(0,)), B, T)
    with pytest.raises(ShapeError):
        c.load_checkpoint(path)


def test_pipelined_host_batches_match_per_step_calls(orc):
    """snn_train_steps_packed (uploads of batch k+1 overlapped with step k) gives the same
    bits as one train_step_packed call per batch, losses and parameters."""
    import torch
    net = Net(inp=70, hidden=(40, 24), classes=7, act="superspike")
    B, T, K = 8, 45, 5
    x, y = orc.synth_raster(7, B * K, T, 70, 9)
    pk = orc.pack_time(x).reshape(K, B, -1, 70)
    yk = y.reshape(K, B)
    pinned = torch.empty(pk.shape, dtype=torch.uint8, pin_memory=True)
    pinned.numpy()[...] = pk
    a = make_engine(net, B, T, seed=4)
    b = make_engine(net, B, T, seed=4)
    la, aa = a.train_steps_packed(pinned.numpy(), yk)
    ref = [b.train_step_packed(pk[k], yk[k]) for k in range(K)]
    assert [float(v) for v in la] == [r[0] for r in ref]
    assert [float(v) for v in aa] == [r[1] for r in ref]
    assert np.array_equal(a.get_params(), b.get_params())
    # a second call continues the same optimizer state (pageable memory works too)
    la2, _ = a.train_steps_packed(pk[:2], yk[:2])
    assert [float(v) for v in la2] == [b.train_step_packed(pk[k], yk[k])[0] for k in range(2)]
    assert np.array_equal(a.get_params(), b.get_params())


LIF_READOUT_GPU = [
    ("ce-superspike", Net(inp=40, hidden=(24, 20), classes=5, act="superspike", readout="lif"), "ce", 6, 30),
    ("mse-arctan-bias", Net(inp=40, hidden=(24,), classes=4, act="arctan", bias=True, readout="lif"),
     "rate_mse", 5, 45),
    ("mse-c1-shape", Net(readout="lif"), "rate_mse", 32, 128),
]


@pytest.mark.parametrize("case", LIF_READOUT_GPU, ids=[c[0] for c in LIF_READOUT_GPU])
def test_lif_readout_parity(orc, case):
    """A LIF readout (network.hpp:153-155, :396; VERDICT r1 missing #3): the trace is
    the readout's spikes, the logits their counts; with the spike-rate MSE loss
    (objective.hpp:139-183) this is the reference's rate-coded output.  Against the
    oracle (pinned bit for bit to the reference, test_oracle.py)."""
    from oracle.pyoracle import Opts
    _, net, loss, B, T = case
    o = Opts(loss=loss)
    params = orc.init(net, orc.key_child(orc.key_from_seed(7), 0)) * np.float32(3.0)
    x, y = orc.synth_raster(net.classes, B, T, net.inp, 4)
    pk = orc.pack_time(x)
    kw = dict(loss="spike_rate_mse") if loss == "rate_mse" else {}
    eng = make_engine(net, B, T, **kw)
    assert eng.entries() == orc.entries(net)
    eng.stage_dataset(pk, y)
    eng.set_params(params)
    eng.debug(True)
    rows = np.arange(B, dtype=np.uint32)
    l1, a1 = eng.forward_backward(rows)
    ref = orc.forward_backward(net, params, pk, T, y, opts=o, want_trace=True, want_spikes=True)
    tr = eng.fetch("trace")
    assert set(np.unique(tr)) <= {0.0, 1.0} and 0.0 < tr.mean() < 1.0
    assert (tr == ref["trace"]).mean() >= SPIKE_AGREE
    assert abs(l1 - ref["loss"]) <= REL_TOL * abs(ref["loss"]) and a1 == ref["acc"]
    check_grads(orc, net, eng.get_grads(), ref["grads"])
    st = State(params.copy())
    for _ in range(2):
        lo, ao = orc.train_step(net, st, pk, T, y, opts=o)
        l2, a2 = eng.train_step(rows)
        assert abs(l2 - lo) <= 1e-3 * abs(lo) and a2 == ao


RAW_LAYOUT = [
    # (name, net, B, T, steps): IN % 4 == 0 and T_pad / 8 == ceil(T / 8), so host batches
    # are used in the reference layout as DMA'd (row pitch IN, last block masked)
    ("c1-shape", Net(), 16, 128, 3),
    ("c1-shape-17", Net(), 16, 128, 17),
    ("ring-wrap", Net(inp=40, hidden=(24, 20), classes=5), 2, 64, 4100),
]


@pytest.mark.parametrize("case", RAW_LAYOUT, ids=[c[0] for c in RAW_LAYOUT])
def test_reference_layout_batches_match_staged_dataset(orc, case):
    """Host batches kept in the reference layout [B][ceil(T/8)][IN] (no device re-layout;
    the forward / wgrad decoders read rows of IN bytes and mask features >= IN of the last
    64-k block) train bit-identically to the same rows of a staged [n][T_pad/8][IN_pad]
    dataset; the StepResults of snn_train_steps_packed come from the mapped ring the fused
    tail writes (more steps than the ring holds: drained mid-call)."""
    import torch
    _, net, B, T, K = case
    x, y = orc.synth_raster(net.classes, B * K, T, net.inp, 5)
    pk = orc.pack_time(x)
    a = make_engine(net, B, T, seed=2)
    b = make_engine(net, B, T, seed=2)
    c = make_engine(net, B, T, seed=2)
    b.stage_dataset(pk, y)
    ref = [b.train_step(np.arange(k * B, (k + 1) * B, dtype=np.uint32)) for k in range(K)]
    pinned = torch.empty((K, B) + pk.shape[1:], dtype=torch.uint8, pin_memory=True)
    pinned.numpy()[...] = pk.reshape((K, B) + pk.shape[1:])
    la, aa = a.train_steps_packed(pinned.numpy(), y.reshape(K, B))
    assert [float(v) for v in la] == [r[0] for r in ref]
    assert [float(v) for v in aa] == [r[1] for r in ref]
    assert np.array_equal(a.get_params(), b.get_params())
    n1 = min(K, 3)
    lc = [c.train_step_packed(pk[k * B:(k + 1) * B], y[k * B:(k + 1) * B]) for k in range(n1)]
    assert lc == ref[:n1]
