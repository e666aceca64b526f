"""Pins the plain-C oracle against the reference (CPU only).

* golden vectors in tests/golden/ were produced by the unmodified reference
  (tests/gen_golden.py -> oracle/_ref); the oracle must reproduce them BIT FOR
  BIT (same fp32 operation order, -ffp-contract=off, same libm);
* known-answer tests restated from the reference's own suite
  (data_test.cpp:26-44, optimize_test.cpp:82-95, rng_test.cpp);
* when oracle/_ref is present (this container), randomized configurations are
  compared live against the reference.
"""
import os

import numpy as np
import pytest

from oracle.pyoracle import Lib, Net, State, have_ref


def _net(g):
    return Net(inp=int(g["net_inp"]), hidden=tuple(int(h) for h in g["net_hidden"]),
               classes=int(g["net_classes"]), bias=bool(g["net_bias"]),
               threshold=float(g["net_threshold"]), act=str(g["net_act"]),
               unroll=int(g["net_unroll"]))


def test_rng_golden(orc, golden):
    g = golden("rng")
    k = orc.key_from_seed(42)
    assert np.uint64(k) == g["seed42_word"]
    assert [orc.key_bits(k, i) for i in range(8)] == g["bits"].tolist()
    assert [orc.key_child(k, i) for i in range(8)] == g["child"].tolist()
    assert [orc.uniform01(k, i) for i in range(8)] == g["uniform"].tolist()
    assert np.array_equal(orc.permutation(orc.key_child(k, 3), 50), g["perm"])
    assert np.array_equal(orc.truncated_normal(orc.key_child(k, 4), 64, 0.5, 0.25),
                          g["tnorm"])


def test_permutation_is_a_permutation(orc):
    p = orc.permutation(orc.key_from_seed(3), 1000)
    assert sorted(p.tolist()) == list(range(1000))


def test_pack_msb_first_kat(orc):
    # data_test.cpp:26-38: T=10, spikes at t 0,3,8,9 -> 0x90, 0xC0
    x = np.zeros((1, 10, 1), np.uint8)
    x[0, [0, 3, 8, 9], 0] = 1
    pk = orc.pack_time(x)
    assert pk.shape == (1, 2, 1)
    assert pk[0, 0, 0] == 0x90 and pk[0, 1, 0] == 0xC0
    # data_test.cpp:40-44: trailing pad bits stay zero
    assert orc.pack_time(np.ones((1, 3, 1), np.uint8))[0, 0, 0] == 0xE0


def test_pack_roundtrip(orc):
    rng = np.random.default_rng(0)
    for t in (1, 7, 8, 9, 19, 128, 131):
        x = (rng.random((3, t, 5)) < 0.3).astype(np.uint8)
        assert np.array_equal(orc.unpack_time(orc.pack_time(x), t), x)


def test_adam_first_step_moves_by_lr(orc):
    # optimize_test.cpp:82-95 (fp32 here)
    p = np.array([1.0, -2.0], np.float32)
    g = np.array([0.5, -3.0], np.float32)
    m, v = np.zeros(2, np.float32), np.zeros(2, np.float32)
    assert orc.adam(p, g, m, v, 0, lr=1e-3) == 1
    assert p[0] == pytest.approx(1.0 - 1e-3, rel=1e-6)
    assert p[1] == pytest.approx(-2.0 + 1e-3, rel=1e-6)


def test_adam_matches_scalar_reference(orc):
    # optimize_test.cpp:24-36 ScalarAdam, 25 steps (fp32 vs f64 textbook)
    rng = np.random.default_rng(700)
    p = rng.standard_normal(3).astype(np.float32)
    pref = p.astype(np.float64)
    m, v = np.zeros(3, np.float32), np.zeros(3, np.float32)
    mr, vr = np.zeros(3), np.zeros(3)
    step = 0
    for s in range(1, 26):
        g = rng.standard_normal(3).astype(np.float32)
        step = orc.adam(p, g, m, v, step, lr=1e-3)
        mr = 0.9 * mr + 0.1 * g
        vr = 0.999 * vr + 0.001 * g.astype(np.float64) ** 2
        pref = pref - 1e-3 * (mr / (1 - 0.9 ** s)) / (np.sqrt(vr / (1 - 0.999 ** s)) + 1e-8)
        assert np.allclose(p, pref, rtol=0, atol=2e-6)
    assert step == 25


def test_tiny_golden_bit_exact(orc, golden):
    g = golden("tiny")
    net = _net(g)
    t = int(g["t"])
    out = orc.forward_backward(net, g["params"], g["packed"], t, g["y"],
                               want_spikes=True, want_trace=True)
    assert out["loss"] == float(g["loss"])
    assert out["acc"] == float(g["acc"])
    assert np.array_equal(out["trace"], g["trace"])
    assert np.array_equal(out["spikes"][0], g["spikes0"])
    assert np.array_equal(out["spikes"][1], g["spikes1"])
    assert np.array_equal(out["grads"], g["grads"])
    st = State(g["params"].copy())
    loss, _ = orc.train_step(net, st, g["packed"], t, g["y"])
    assert loss == float(g["step_loss"])
    assert np.array_equal(st.params, g["step_params"])
    assert np.array_equal(st.m, g["step_m"]) and np.array_equal(st.v, g["step_v"])
    st2 = State(g["params"].copy())
    metrics = orc.train_epochs(net, st2, g["packed"], g["y"], t, 4, 3, 7)
    assert np.array_equal(metrics, g["epochs_metrics"])
    assert np.array_equal(st2.params, g["epochs_params"])
    assert st2.step == int(g["epochs_step"])


@pytest.mark.parametrize("tag", ["init", "warm", "hot"])
def test_c1_golden_bit_exact(orc, golden, tag):
    g = golden("c1")
    net = _net(g)
    params = g["params_init"] if tag == "init" else g[f"{tag}_params"]
    out = orc.forward_backward(net, params, g["batch_packed"], 128, g["batch_y"],
                               want_spikes=True, want_trace=True)
    assert out["loss"] == float(g[f"{tag}_loss"])
    assert out["acc"] == float(g[f"{tag}_acc"])
    assert np.array_equal(out["trace"], g[f"{tag}_trace"])
    assert np.array_equal(np.packbits(out["spikes"][0]), g[f"{tag}_spikes0_bits"])
    assert np.array_equal(np.packbits(out["spikes"][1]), g[f"{tag}_spikes1_bits"])
    assert np.array_equal(out["grads"], g[f"{tag}_grads"])


def test_c1_init_params_golden(orc, golden):
    g = golden("c1")
    master = orc.key_from_seed(0)
    p = orc.init(_net(g), orc.key_child(master, 0))
    assert np.array_equal(p, g["params_init"])
    names = [e[0] for e in orc.entries(_net(g))]
    assert names == ["l0.w", "l1.beta", "l2.w", "l3.beta", "l4.w", "l5.beta"]
    assert p.size == 108820


@pytest.mark.slow
def test_c1_warm_checkpoint_golden(orc, golden):
    """Re-train the warm checkpoint (12 steps at C1) and match bit for bit."""
    g = golden("c1")
    net = _net(g)
    x, y = orc.synth_raster(20, 1024, 128, 700, 1)
    pk = orc.pack_time(x)
    import hashlib
    assert hashlib.sha256(pk.tobytes()).digest() == g["dataset_packed_sha"].tobytes()
    st = State(g["params_init"].copy())
    metrics = orc.train_epochs(net, st, pk, y, 128, 256, 3, 0)
    assert np.array_equal(metrics, g["warm_metrics"])
    assert np.array_equal(st.params, g["warm_params"])
    assert st.step == int(g["warm_step"])


CONFIGS = [
    Net(inp=30, hidden=(16, 12), classes=5, unroll=4),
    Net(inp=30, hidden=(16,), classes=5, bias=True, act="superspike", unroll=3),
    Net(inp=40, hidden=(24, 20, 8), classes=4, bias=True, act="triangular", unroll=5),
    Net(inp=40, hidden=(24, 20), classes=4, act="boxcar", unroll=7),
    Net(inp=40, hidden=(24, 20), classes=4, act="custom", unroll=1),
    Net(inp=33, hidden=(64, 32), classes=7, act="arctan", threshold=0.75, unroll=32),
]


@pytest.mark.skipif(not have_ref(), reason="oracle/_ref needs /root/reference")
@pytest.mark.parametrize("cfg", range(len(CONFIGS)))
def test_oracle_vs_reference_live(orc, cfg):
    ref = Lib("ref")
    net = CONFIGS[cfg]
    assert orc.entries(net) == ref.entries(net)
    key = orc.key_from_seed(100 + cfg)
    p = orc.init(net, key)
    assert np.array_equal(p, ref.init(net, key))
    p = p * np.float32(3.0)
    B, T = 10, 23
    x, y = orc.synth_raster(net.classes, B, T, net.inp, 9 + cfg)
    pk = orc.pack_time(x)
    a = orc.forward_backward(net, p, pk, T, y, want_spikes=True, want_trace=True)
    b = ref.forward_backward(net, p, pk, T, y, want_spikes=True, want_trace=True)
    assert a["loss"] == b["loss"] and a["acc"] == b["acc"]
    assert np.array_equal(a["trace"], b["trace"])
    for s1, s2 in zip(a["spikes"], b["spikes"]):
        assert np.array_equal(s1, s2)
    assert np.array_equal(a["grads"], b["grads"])
    s1, s2 = State(p.copy()), State(p.copy())
    m1 = orc.train_epochs(net, s1, pk, y, T, 3, 2, 5)
    m2 = ref.train_epochs(net, s2, pk, y, T, 3, 2, 5)
    assert np.array_equal(m1, m2) and np.array_equal(s1.params, s2.params)


def _opts_case():
    from oracle.pyoracle import Opts
    g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "opts.npz"))
    net = Net(inp=int(g["inp"]), hidden=tuple(int(h) for h in g["hidden"]), classes=int(g["classes"]),
              bias=bool(g["bias"]), threshold=float(g["threshold"]), act=str(g["act"]),
              unroll=int(g["unroll"]))
    opts = {"rate_mse": Opts(loss="rate_mse", rate_hi=0.8, rate_lo=0.05),
            "sgd": Opts(optimizer="sgd", momentum=0.8)}
    return g, net, opts


@pytest.mark.parametrize("name", ["rate_mse", "sgd"])
def test_opts_golden_bit_exact(orc, name):
    """Spike-rate MSE loss (objective.hpp:139-183) and SGD + momentum
    (optimize.hpp:69-84): the C restatement equals fixtures made by the reference."""
    g, net, opts = _opts_case()
    o, T = opts[name], int(g["t"])
    fb = orc.forward_backward(net, g["params"], g["packed"], T, g["y"], opts=o)
    assert fb["loss"] == g[f"{name}_loss"]
    assert np.array_equal(fb["grads"], g[f"{name}_grads"])
    st = State(g["params"].copy())
    losses = [orc.train_step(net, st, g["packed"], T, g["y"], opts=o)[0] for _ in range(3)]
    assert np.array_equal(np.array(losses, np.float32), g[f"{name}_step_losses"])
    assert np.array_equal(st.params, g[f"{name}_params3"])
    assert np.array_equal(st.m, g[f"{name}_m3"]) and np.array_equal(st.v, g[f"{name}_v3"])


@pytest.mark.skipif(not have_ref(), reason="oracle/_ref needs /root/reference")
@pytest.mark.parametrize("cfg", range(3))
def test_opts_vs_reference_live(orc, cfg):
    from oracle.pyoracle import Opts
    net = CONFIGS[cfg]
    ref = Lib("ref")
    p = orc.init(net, orc.key_from_seed(300 + cfg)) * np.float32(3.0)
    B, T = 6, 21
    x, y = orc.synth_raster(net.classes, B, T, net.inp, 31 + cfg)
    pk = orc.pack_time(x)
    for o in (Opts(loss="rate_mse", rate_hi=0.7, rate_lo=0.2), Opts(optimizer="sgd", momentum=0.5),
              Opts(optimizer="sgd", loss="rate_mse")):
        a = orc.forward_backward(net, p, pk, T, y, opts=o)
        b = ref.forward_backward(net, p, pk, T, y, opts=o)
        assert a["loss"] == b["loss"] and np.array_equal(a["grads"], b["grads"])
        s1, s2 = State(p.copy()), State(p.copy())
        for _ in range(2):
            assert orc.train_step(net, s1, pk, T, y, opts=o) == ref.train_step(net, s2, pk, T, y, opts=o)
        assert np.array_equal(s1.params, s2.params) and np.array_equal(s1.m, s2.m)


BETA_NET = Net(inp=40, hidden=(24, 20), classes=6, act="superspike", bias=True,
               beta_mode=("scalar", "fixed", "scalar"), fixed_beta=(0.5, 0.3, 0.5), unroll=9)


def test_beta_modes_golden_bit_exact(orc, golden):
    """LearnableScalar / Fixed beta (neuron.hpp:56-76, autodiff.hpp:191-205 for the
    broadcast gradient): the C restatement equals reference-made fixtures."""
    g = golden("betamodes")
    assert np.array_equal(orc.init(BETA_NET, orc.key_child(orc.key_from_seed(23), 0)), g["init"])
    fb = orc.forward_backward(BETA_NET, g["params"], g["packed"], 30, g["y"], want_trace=True)
    assert fb["loss"] == g["loss"] and np.array_equal(fb["grads"], g["grads"])
    assert np.array_equal(fb["trace"], g["trace"])
    st = State(g["params"].copy())
    losses = [orc.train_step(BETA_NET, st, g["packed"], 30, g["y"])[0] for _ in range(3)]
    assert np.array_equal(np.array(losses, np.float32), g["step_losses"])
    assert np.array_equal(st.params, g["params3"]) and np.array_equal(st.m, g["m3"])
    assert np.array_equal(st.v, g["v3"])


@pytest.mark.skipif(not have_ref(), reason="oracle/_ref needs /root/reference")
@pytest.mark.parametrize("modes", [("scalar", "scalar", "fixed"), ("fixed", "per_neuron", "scalar")])
def test_beta_modes_vs_reference_live(orc, modes):
    from oracle.pyoracle import Opts
    ref = Lib("ref")
    net = Net(inp=30, hidden=(16, 12), classes=5, beta_mode=modes, fixed_beta=(0.6, 0.4, 0.8), unroll=5)
    assert orc.entries(net) == ref.entries(net)
    key = orc.key_from_seed(41)
    p = orc.init(net, key)
    assert np.array_equal(p, ref.init(net, key))
    p = p * np.float32(2.5)
    x, y = orc.synth_raster(5, 6, 23, 30, 12)
    pk = orc.pack_time(x)
    a = orc.forward_backward(net, p, pk, 23, y)
    b = ref.forward_backward(net, p, pk, 23, y)
    assert a["loss"] == b["loss"] and np.array_equal(a["grads"], b["grads"])
    for o in (Opts(), Opts(optimizer="sgd")):
        s1, s2 = State(p.copy()), State(p.copy())
        for _ in range(2):
            assert orc.train_step(net, s1, pk, 23, y, opts=o) == ref.train_step(net, s2, pk, 23, y, opts=o)
        assert np.array_equal(s1.params, s2.params) and np.array_equal(s1.m, s2.m)


def _shift_case():
    from oracle.pyoracle import Opts
    g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "shift.npz"))
    net = Net(inp=int(g["inp"]), hidden=tuple(int(h) for h in g["hidden"]), classes=int(g["classes"]),
              bias=bool(g["bias"]), threshold=float(g["threshold"]), act=str(g["act"]),
              unroll=int(g["unroll"]))
    opts = {"one_axis": Opts(max_shift=3, shift_axes=(2,)),
            "two_axes": Opts(max_shift=5, shift_axes=(2, -1))}
    return g, net, opts


@pytest.mark.parametrize("name", ["one_axis", "two_axes"])
def test_shift_augment_golden_bit_exact(orc, name):
    """shift_augment in the epoch loop (data.hpp:216-227, optimize.hpp:241-280):
    the C restatement reproduces the reference's 2-epoch run bit for bit."""
    g, net, opts = _shift_case()
    st = State(g["params"].copy())
    metrics = orc.train_epochs(net, st, g["packed"], g["y"], int(g["t"]), 4, 2, 9, opts=opts[name])
    assert np.array_equal(metrics, g[f"{name}_metrics"])
    assert np.array_equal(st.params, g[f"{name}_params"])
    assert np.array_equal(st.m, g[f"{name}_m"]) and np.array_equal(st.v, g[f"{name}_v"])
    assert st.step == int(g[f"{name}_step"])
    # the shift is not a no-op: an unshifted run ends elsewhere
    st0 = State(g["params"].copy())
    orc.train_epochs(net, st0, g["packed"], g["y"], int(g["t"]), 4, 2, 9)
    assert not np.array_equal(st0.params, st.params)


@pytest.mark.skipif(not have_ref(), reason="oracle/_ref not built")
def test_shift_augment_live_vs_reference(orc):
    """Same check against the reference's own train() on other shapes."""
    from oracle.pyoracle import Opts
    ref = Lib("ref")
    net = Net(inp=33, hidden=(16, 9), classes=4, bias=False, act="arctan", unroll=2)
    p = orc.init(net, orc.key_from_seed(5)) * np.float32(3.0)
    x, y = orc.synth_raster(4, 11, 17, 33, 3)
    pk = orc.pack_time(x)
    for o in (Opts(max_shift=7, shift_axes=(-1,)), Opts(max_shift=40, shift_axes=(2, 2, -1)),
              Opts(max_shift=0, shift_axes=(2,))):
        s1, s2 = State(p.copy()), State(p.copy())
        m1 = orc.train_epochs(net, s1, pk, y, 17, 3, 2, 11, opts=o)
        m2 = ref.train_epochs(net, s2, pk, y, 17, 3, 2, 11, opts=o)
        assert np.array_equal(m1, m2) and np.array_equal(s1.params, s2.params)


@pytest.mark.parametrize("axes,max_shift", [((0,), 2), ((1,), 2), ((2, 1), 2), ((1,), 0)])
def test_shift_augment_rejects_batch_and_time_axes(orc, axes, max_shift):
    """train() refuses axes 0 / 1 even when no shift happens (optimize.hpp:241-245)."""
    from oracle.pyoracle import Opts
    g, net, _ = _shift_case()
    libs = [orc] + ([Lib("ref")] if have_ref() else [])
    for lib in libs:
        with pytest.raises(ValueError):
            lib.train_epochs(net, State(g["params"].copy()), g["packed"], g["y"], int(g["t"]), 4, 1,
                             9, opts=Opts(max_shift=max_shift, shift_axes=axes))


def test_shift_augment_nonpositive_max_shift_is_identity(orc):
    """max_shift <= 0 never reaches shift_augment (optimize.hpp:276): same run as none."""
    from oracle.pyoracle import Opts
    g, net, _ = _shift_case()
    base = State(g["params"].copy())
    orc.train_epochs(net, base, g["packed"], g["y"], int(g["t"]), 4, 1, 9)
    for o in (Opts(max_shift=0, shift_axes=(2,)), Opts(max_shift=-3, shift_axes=(2,)),
              Opts(max_shift=0, shift_axes=(3,))):
        st = State(g["params"].copy())
        orc.train_epochs(net, st, g["packed"], g["y"], int(g["t"]), 4, 1, 9, opts=o)
        assert np.array_equal(st.params, base.params)


def _activity_case():
    from oracle.pyoracle import Opts
    g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "activity.npz"))
    net = Net(inp=int(g["inp"]), hidden=tuple(int(h) for h in g["hidden"]), classes=int(g["classes"]),
              bias=bool(g["bias"]), threshold=float(g["threshold"]), act=str(g["act"]),
              unroll=int(g["unroll"]), monitor=tuple(int(m) for m in g["monitor"]))
    opts = {"both": Opts(lambda_low=0.5, lambda_high=2.0, f_min=0.1, f_max=0.3),
            "high": Opts(lambda_high=1.5, f_max=0.05)}
    return g, net, opts


def test_monitor_layer_ids_golden(orc):
    """Monitors take normalised layer ids: entry names and init keys of every later
    layer move up (network.hpp:231-286), exactly as the reference's."""
    g, net, _ = _activity_case()
    assert [n for n, _, _ in orc.entries(net)] == [str(n) for n in g["names"]]
    assert np.array_equal(orc.init(net, orc.key_child(orc.key_from_seed(41), 0)), g["params_init"])


@pytest.mark.parametrize("name", ["both", "high"])
def test_activity_regularizer_golden_bit_exact(orc, name):
    """Activity regularizer on two monitors (objective.hpp:186-227): loss, grads and
    three train_steps equal the reference's fixture bit for bit."""
    g, net, opts = _activity_case()
    o, T = opts[name], int(g["t"])
    fb = orc.forward_backward(net, g["params"], g["packed"], T, g["y"], opts=o)
    assert fb["loss"] == g[f"{name}_loss"]
    assert np.array_equal(fb["grads"], g[f"{name}_grads"])
    plain = orc.forward_backward(net, g["params"], g["packed"], T, g["y"])
    assert fb["loss"] != plain["loss"] and not np.array_equal(fb["grads"], plain["grads"])
    st = State(g["params"].copy())
    losses = [orc.train_step(net, st, g["packed"], T, g["y"], opts=o)[0] for _ in range(3)]
    assert np.array_equal(np.array(losses, np.float32), g[f"{name}_step_losses"])
    assert np.array_equal(st.params, g[f"{name}_params3"])


@pytest.mark.skipif(not have_ref(), reason="oracle/_ref not built")
def test_activity_regularizer_live_vs_reference(orc):
    from oracle.pyoracle import Opts
    ref = Lib("ref")
    net = Net(inp=40, hidden=(24, 20, 8), classes=4, bias=True, monitor=(0, 2), act="boxcar", unroll=5)
    key = orc.key_child(orc.key_from_seed(4), 0)
    p = orc.init(net, key)
    assert np.array_equal(p, ref.init(net, key)) and orc.entries(net) == ref.entries(net)
    p = p * np.float32(3.0)
    x, y = orc.synth_raster(4, 7, 21, 40, 2)
    pk = orc.pack_time(x)
    for o in (Opts(lambda_low=0.5, lambda_high=2.0, f_min=0.1, f_max=0.3),
              Opts(lambda_low=3.0, f_min=0.9, loss="rate_mse"), Opts(lambda_low=1.0, optimizer="sgd")):
        a = orc.forward_backward(net, p, pk, 21, y, opts=o)
        b = ref.forward_backward(net, p, pk, 21, y, opts=o)
        assert a["loss"] == b["loss"] and np.array_equal(a["grads"], b["grads"])


def test_activity_regularizer_rejects_bad_band(orc):
    """need 0 <= f_min <= f_max <= 1 once a lambda is set (objective.hpp:191-192)."""
    from oracle.pyoracle import Opts
    g, net, _ = _activity_case()
    for o in (Opts(lambda_low=1.0, f_min=0.5, f_max=0.2), Opts(lambda_high=1.0, f_max=1.5)):
        with pytest.raises(ValueError):
            orc.forward_backward(net, g["params"], g["packed"], int(g["t"]), g["y"], opts=o)
    # lambdas zero: the band is never checked (the regularizer is not called)
    orc.forward_backward(net, g["params"], g["packed"], int(g["t"]), g["y"],
                         opts=Opts(f_min=0.5, f_max=0.2))


@pytest.mark.skipif(not have_ref(), reason="oracle/_ref not built")
def test_container_fixtures_read_back_by_reference():
    """tests/golden/*.spkd are the reference's write_container output; its own
    read_container returns the packed bytes and labels of spkd.npz."""
    gold = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    g = np.load(os.path.join(gold, "spkd.npz"))
    ref = Lib("ref")
    for name in ("flat.spkd", "multi.spkd"):
        pk, y, t = ref.read_container(os.path.join(gold, name), 4096, 64)
        assert t == int(g["t"]) and np.array_equal(y, g["y"])
        assert np.array_equal(pk[:g["packed"].size], g["packed"].ravel())


ACT_NAMES = ("custom", "superspike", "triangular", "arctan", "boxcar", "sigmoid")


@pytest.mark.parametrize("act", ACT_NAMES)
def test_surrogate_golden_bit_exact(orc, golden, act):
    """g(x) of every surrogate == the reference's own tape (spike() over
    register_custom) bit for bit; sigmoid is the declared custom() backward
    (spiketrain_oracle.h ORC_ACT_SIGMOID), fixture tests/golden/surrogates.npz."""
    g = golden("surrogates")
    assert np.array_equal(orc.surrogate(act, g["x"]), g[act])
    assert np.array_equal(orc.surrogate(act, g["x"], slope=5.0, aux=0.25), g[act + "_k5"])


@pytest.mark.skipif(not have_ref(), reason="oracle/_ref needs /root/reference")
def test_surrogate_vs_reference_tape_live(orc):
    ref = Lib("ref")
    x = np.random.default_rng(3).normal(0, 2, 5000).astype(np.float32)
    for act in ACT_NAMES:
        assert np.array_equal(orc.surrogate(act, x), ref.surrogate(act, x)), act


def test_sigmoid_surrogate_is_dsigmoid():
    """The declared formula is d/dx sigmoid(kx), finite everywhere."""
    from oracle.pyoracle import Lib as _L
    o = _L("orc")
    x = np.linspace(-5, 5, 1001).astype(np.float32)
    k = 25.0
    s = 1.0 / (1.0 + np.exp(-k * x.astype(np.float64)))
    np.testing.assert_allclose(o.surrogate("sigmoid", x), k * s * (1 - s), rtol=1e-5, atol=2e-6)  # f32 tails round s to 1
    big = np.array([1e4, -1e4, 80.0, -80.0], np.float32)
    assert np.isfinite(o.surrogate("sigmoid", big)).all()


THREAD_NETS = [
    ("lif", Net(inp=40, hidden=(24, 20), classes=4, bias=True, act="superspike", unroll=5)),
    ("alif", Net(inp=40, hidden=(24, 20), classes=4, cell=("alif", "lif"), unroll=7)),
    ("rlif", Net(inp=40, hidden=(24, 20), classes=4, cell=("rlif", "alif"), act="sigmoid")),
]


@pytest.mark.parametrize("case", THREAD_NETS, ids=[c[0] for c in THREAD_NETS])
def test_threads_are_bit_identical(case):
    """orc_set_threads(n) splits output elements only: any n gives the same bits."""
    _, net = case
    o = Lib("orc")
    p = o.init(net, o.key_child(o.key_from_seed(4), 0)) * np.float32(3.0)
    x, y = o.synth_raster(net.classes, 13, 29, net.inp, 2)
    pk = o.pack_time(x)
    outs = []
    for n in (1, 3, 8):
        o.set_threads(n)
        outs.append(o.forward_backward(net, p, pk, 29, y, want_spikes=True, want_trace=True))
    o.set_threads(1)
    for r in outs[1:]:
        assert r["loss"] == outs[0]["loss"]
        assert np.array_equal(r["grads"], outs[0]["grads"])
        assert np.array_equal(r["trace"], outs[0]["trace"])


@pytest.mark.parametrize("case", THREAD_NETS, ids=[c[0] for c in THREAD_NETS])
def test_forced_with_own_spikes_is_identity(orc, case):
    """Teacher forcing with the oracle's own rasters reproduces the free run bit
    for bit; forcing a different raster changes it (the mode is live)."""
    _, net = case
    p = orc.init(net, orc.key_child(orc.key_from_seed(4), 0)) * np.float32(3.0)
    x, y = orc.synth_raster(net.classes, 7, 29, net.inp, 2)
    pk = orc.pack_time(x)
    free = orc.forward_backward(net, p, pk, 29, y, want_spikes=True, want_trace=True, want_v=True)
    assert sum(int(s.sum()) for s in free["spikes"]) > 0
    forced = orc.forward_backward(net, p, pk, 29, y, want_spikes=True, want_trace=True,
                                  want_v=True, forced=free["spikes"])
    assert forced["loss"] == free["loss"]
    assert np.array_equal(forced["grads"], free["grads"])
    for a, b in zip(forced["spikes"], free["spikes"]):
        assert np.array_equal(a, b)
    flip = [s.copy() for s in free["spikes"]]
    flip[0][0, 3, :] ^= 1
    other = orc.forward_backward(net, p, pk, 29, y, want_spikes=True, forced=flip)
    assert np.array_equal(other["spikes"][0], flip[0])
    assert not np.array_equal(other["grads"], free["grads"])


LIF_READOUT = [
    ("ce-superspike", Net(inp=40, hidden=(24, 20), classes=5, act="superspike", readout="lif", unroll=7), "ce"),
    ("mse-arctan-bias", Net(inp=40, hidden=(24,), classes=4, act="arctan", bias=True, readout="lif"), "rate_mse"),
    ("mse-triangular-scalar", Net(inp=33, hidden=(16, 12), classes=6, act="triangular", readout="lif",
                                  beta_mode=("per_neuron", "per_neuron", "scalar")), "rate_mse"),
]


@pytest.mark.skipif(not have_ref(), reason="oracle/_ref needs /root/reference")
@pytest.mark.parametrize("case", LIF_READOUT, ids=[c[0] for c in LIF_READOUT])
def test_lif_readout_bit_exact_vs_reference(orc, case):
    """A network ending in a LIF readout (network.hpp:153-155): its spikes are the
    trace (:396).  The restatement equals the reference bit for bit: loss, trace,
    every gradient, and 2 epochs of training."""
    from oracle.pyoracle import Opts
    _, net, loss = case
    ref = Lib("ref")
    o = Opts(loss=loss)
    p = orc.init(net, orc.key_child(orc.key_from_seed(3), 0)) * np.float32(3.0)
    assert np.array_equal(p, ref.init(net, ref.key_child(ref.key_from_seed(3), 0)) * np.float32(3.0))
    x, y = orc.synth_raster(net.classes, 12, 30, net.inp, 2)
    pk = orc.pack_time(x)
    a = orc.forward_backward(net, p, pk, 30, y, opts=o, want_trace=True, want_spikes=True)
    b = ref.forward_backward(net, p, pk, 30, y, opts=o, want_trace=True, want_spikes=True)
    assert a["loss"] == b["loss"] and a["acc"] == b["acc"]
    assert np.array_equal(a["trace"], b["trace"]) and set(np.unique(a["trace"])) <= {0.0, 1.0}
    assert 0.0 < a["trace"].mean() < 1.0
    assert np.array_equal(a["grads"], b["grads"])
    s1, s2 = State(p.copy()), State(p.copy())
    m1 = orc.train_epochs(net, s1, pk, y, 30, 4, 2, 5, opts=o)
    m2 = ref.train_epochs(net, s2, pk, y, 30, 4, 2, 5, opts=o)
    assert np.array_equal(m1, m2) and np.array_equal(s1.params, s2.params)
