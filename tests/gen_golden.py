"""Generate tests/golden/*.npz from the REFERENCE ITSELF (oracle/_ref).

Run here (needs /root/reference to build oracle/_ref):
    python tests/gen_golden.py
The fixtures pin the plain-C oracle (oracle/liboracle.so) on machines where the
reference is absent (the GPU box).  Every array comes from ref_* entry points,
i.e. from the unmodified spiketrain headers.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.pyoracle import Lib, Net, State, have_ref  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")

TINY = Net(inp=30, hidden=(16, 12), classes=5, act="arctan", unroll=4)
C1 = Net()  # 700-128-128-20, arctan k=2, nobias, unroll 32


def net_dict(n: Net) -> dict:
    return dict(inp=n.inp, hidden=np.array(n.hidden), classes=n.classes,
                bias=int(n.bias), threshold=n.threshold, act=n.act,
                unroll=n.unroll)


def tiny(ref: Lib):
    key = ref.key_child(ref.key_from_seed(5), 0)
    p = ref.init(TINY, key) * np.float32(3.0)  # scale for activity
    x, y = ref.synth_raster(5, 12, 19, 30, 3)
    pk = ref.pack_time(x)
    out = ref.forward_backward(TINY, p, pk, 19, y, want_spikes=True, want_trace=True)
    st = State(p.copy())
    l1, a1 = ref.train_step(TINY, st, pk, 19, y)
    st2 = State(p.copy())
    metrics = ref.train_epochs(TINY, st2, pk, y, 19, 4, 3, 7)
    np.savez_compressed(
        os.path.join(GOLD, "tiny.npz"), **{f"net_{k}": v for k, v in net_dict(TINY).items()},
        params=p, packed=pk, y=y, t=19, loss=out["loss"], acc=out["acc"],
        grads=out["grads"], trace=out["trace"],
        spikes0=out["spikes"][0], spikes1=out["spikes"][1],
        step_params=st.params, step_m=st.m, step_v=st.v, step_loss=l1,
        epochs_params=st2.params, epochs_metrics=metrics, epochs_step=st2.step)


def c1(ref: Lib):
    """C1 shape: init and warm (3 epochs x 4 steps at N=1024, B=256, seed 0)."""
    master = ref.key_from_seed(0)
    p_init = ref.init(C1, ref.key_child(master, 0))
    x, y = ref.synth_raster(20, 1024, 128, 700, 1)
    pk = ref.pack_time(x)
    st = State(p_init.copy())
    metrics = ref.train_epochs(C1, st, pk, y, 128, 256, 3, 0)
    # "hot": resume the warm state for 9 more epochs (epoch keys restart at 0
    # on resume, optimize.hpp:258) -> hidden rates of several percent.
    hot = st.copy()
    hot_metrics = ref.train_epochs(C1, hot, pk, y, 128, 256, 9, 0)
    # evaluation batch: first 16 examples of the dataset (labels 0..15)
    bx, by = pk[:16], y[:16]
    res = {}
    for tag, params in (("init", p_init), ("warm", st.params), ("hot", hot.params)):
        o = ref.forward_backward(C1, params, bx, 128, by, want_spikes=True, want_trace=True)
        res[tag] = o
    np.savez_compressed(
        os.path.join(GOLD, "c1.npz"), **{f"net_{k}": v for k, v in net_dict(C1).items()},
        params_init=p_init, warm_params=st.params, warm_m=st.m, warm_v=st.v,
        warm_step=st.step, warm_metrics=metrics, batch_packed=bx, batch_y=by,
        hot_params=hot.params, hot_step=hot.step, hot_metrics=hot_metrics,
        dataset_packed_sha=np.frombuffer(__import__("hashlib").sha256(pk.tobytes()).digest(), np.uint8),
        **{f"{t}_{k}": v for t, o in res.items() for k, v in (
            ("loss", o["loss"]), ("acc", o["acc"]), ("grads", o["grads"]),
            ("trace", o["trace"]),
            ("spikes0_bits", np.packbits(o["spikes"][0])),
            ("spikes1_bits", np.packbits(o["spikes"][1])))})
    print("warm metrics", metrics.tolist(), "hot", hot_metrics.tolist())
    for tag in res:
        print(tag, "rates", [float(s.mean()) for s in res[tag]["spikes"]])


def rng_kats(ref: Lib):
    k = ref.key_from_seed(42)
    vals = dict(
        seed42_word=np.uint64(k),
        bits=np.array([ref.key_bits(k, i) for i in range(8)], np.uint64),
        child=np.array([ref.key_child(k, i) for i in range(8)], np.uint64),
        uniform=np.array([ref.uniform01(k, i) for i in range(8)], np.float64),
        perm=ref.permutation(ref.key_child(k, 3), 50),
        tnorm=ref.truncated_normal(ref.key_child(k, 4), 64, 0.5, 0.25))
    np.savez_compressed(os.path.join(GOLD, "rng.npz"), **vals)


OPTS_NET = Net(inp=40, hidden=(24, 20), classes=6, act="superspike", unroll=7)
OPTS = {"rate_mse": dict(loss="rate_mse", rate_hi=0.8, rate_lo=0.05),
        "sgd": dict(optimizer="sgd", momentum=0.8)}


def opts_fixture(ref: Lib):
    """TrainConfig options on the step: spike-rate MSE loss (objective.hpp:139-183)
    and SGD with momentum (optimize.hpp:69-84), 3 train_steps each."""
    from oracle.pyoracle import Opts
    key = ref.key_child(ref.key_from_seed(21), 0)
    p = ref.init(OPTS_NET, key) * np.float32(3.0)
    x, y = ref.synth_raster(6, 7, 30, 40, 13)
    pk = ref.pack_time(x)
    vals = dict(params=p, packed=pk, y=y, t=30, **net_dict(OPTS_NET))
    for name, kw in OPTS.items():
        o = Opts(**kw)
        fb = ref.forward_backward(OPTS_NET, p, pk, 30, y, opts=o)
        st = State(p.copy())
        losses = [ref.train_step(OPTS_NET, st, pk, 30, y, opts=o)[0] for _ in range(3)]
        vals.update({f"{name}_loss": np.float32(fb["loss"]), f"{name}_grads": fb["grads"],
                     f"{name}_step_losses": np.array(losses, np.float32),
                     f"{name}_params3": st.params, f"{name}_m3": st.m, f"{name}_v3": st.v})
    np.savez_compressed(os.path.join(GOLD, "opts.npz"), **vals)


ACT_NET = Net(inp=40, hidden=(24, 20), classes=5, act="superspike", unroll=4, monitor=(0, 1))
ACT_OPTS = {"both": dict(lambda_low=0.5, lambda_high=2.0, f_min=0.1, f_max=0.3),
            "high": dict(lambda_high=1.5, f_max=0.05)}


def activity_fixture(ref: Lib):
    """MonitorLayer after both LIF layers (network.hpp:57, :415-420) and the
    activity regularizer (objective.hpp:186-227, optimize.hpp:185-191).  The
    monitors shift the normalised layer ids, so entry names and init keys are
    part of the fixture."""
    from oracle.pyoracle import Opts
    key = ref.key_child(ref.key_from_seed(41), 0)
    p_init = ref.init(ACT_NET, key)
    p = p_init * np.float32(3.0)
    x, y = ref.synth_raster(5, 7, 30, 40, 23)
    pk = ref.pack_time(x)
    names = np.array([n for n, _, _ in ref.entries(ACT_NET)])
    vals = dict(params_init=p_init, params=p, packed=pk, y=y, t=30, names=names,
                monitor=np.array(ACT_NET.monitor), **net_dict(ACT_NET))
    for name, kw in ACT_OPTS.items():
        o = Opts(**kw)
        fb = ref.forward_backward(ACT_NET, p, pk, 30, y, opts=o)
        st = State(p.copy())
        losses = [ref.train_step(ACT_NET, st, pk, 30, y, opts=o)[0] for _ in range(3)]
        vals.update({f"{name}_loss": np.float32(fb["loss"]), f"{name}_grads": fb["grads"],
                     f"{name}_step_losses": np.array(losses, np.float32),
                     f"{name}_params3": st.params})
    np.savez_compressed(os.path.join(GOLD, "activity.npz"), **vals)


def container_fixture(ref: Lib):
    """.spkd containers written by the reference's write_container (data.hpp:229-293):
    a flat [N, ceil(T/8), 40] dataset and the same bytes as [N, ceil(T/8), 5, 8]."""
    x, y = ref.synth_raster(5, 6, 21, 40, 29)
    pk = ref.pack_time(x)
    ref.write_container(os.path.join(GOLD, "flat.spkd"), pk, 21, y)
    ref.write_container(os.path.join(GOLD, "multi.spkd"), pk.reshape(6, 3, 5, 8), 21, y)
    np.savez_compressed(os.path.join(GOLD, "spkd.npz"), packed=pk, y=y, t=21)


SHIFT_NET = Net(inp=40, hidden=(24,), classes=5, bias=True, act="superspike", unroll=3)
SHIFT_OPTS = {"one_axis": dict(max_shift=3, shift_axes=(2,)),
              "two_axes": dict(max_shift=5, shift_axes=(2, -1))}


def shift_fixture(ref: Lib):
    """shift_augment inside the epoch loop (data.hpp:216-227 called from
    optimize.hpp:241-280): every batch rolled along the feature axis by the sum
    of per-axis randint(child(epoch_key, 1 + b), axis, -max_shift, max_shift)."""
    from oracle.pyoracle import Opts
    key = ref.key_child(ref.key_from_seed(33), 0)
    p = ref.init(SHIFT_NET, key) * np.float32(3.0)
    x, y = ref.synth_raster(5, 14, 20, 40, 17)
    pk = ref.pack_time(x)
    vals = dict(params=p, packed=pk, y=y, t=20, **net_dict(SHIFT_NET))
    for name, kw in SHIFT_OPTS.items():
        st = State(p.copy())
        metrics = ref.train_epochs(SHIFT_NET, st, pk, y, 20, 4, 2, 9, opts=Opts(**kw))
        vals.update({f"{name}_metrics": metrics, f"{name}_params": st.params,
                     f"{name}_m": st.m, f"{name}_v": st.v, f"{name}_step": np.uint64(st.step)})
    np.savez_compressed(os.path.join(GOLD, "shift.npz"), **vals)


CKPT_NET = Net(inp=30, hidden=(16, 12), classes=5, bias=True, act="arctan", unroll=4)
CKPT_CONFIG = "# spiketrain run config (fixture)\nnet = 30-16-12-5 lif arctan bias\nlr = 1e-3\n"


def checkpoint_fixture(ref: Lib):
    """.spkc files written by the reference (optimize.hpp:334-366) after 2 steps with
    Adam and with SGD, plus the state they hold (ckpt.npz)."""
    from oracle.pyoracle import Opts
    key = ref.key_child(ref.key_from_seed(17), 0)
    p = ref.init(CKPT_NET, key) * np.float32(3.0)
    x, y = ref.synth_raster(5, 6, 19, 30, 8)
    pk = ref.pack_time(x)
    vals = dict(config=np.frombuffer(CKPT_CONFIG.encode(), np.uint8), **net_dict(CKPT_NET))
    for opt in ("adam", "sgd"):
        st = State(p.copy())
        for _ in range(2):
            ref.train_step(CKPT_NET, st, pk, 19, y, opts=Opts(optimizer=opt, momentum=0.9))
        ref.write_checkpoint(CKPT_NET, st.params, st.m, st.v, st.step, opt, CKPT_CONFIG,
                             os.path.join(GOLD, f"ckpt_{opt}.spkc"))
        vals.update({f"{opt}_params": st.params, f"{opt}_m": st.m, f"{opt}_v": st.v,
                     f"{opt}_step": np.int64(st.step)})
    np.savez_compressed(os.path.join(GOLD, "ckpt.npz"), **vals)


BETA_NET = Net(inp=40, hidden=(24, 20), classes=6, act="superspike", bias=True,
               beta_mode=("scalar", "fixed", "scalar"), fixed_beta=(0.5, 0.3, 0.5), unroll=9)


def beta_modes_fixture(ref: Lib):
    """BetaMode::LearnableScalar / Fixed cells (neuron.hpp:56-76): init, one
    forward/backward and 3 Adam steps, from the reference."""
    key = ref.key_child(ref.key_from_seed(23), 0)
    p0 = ref.init(BETA_NET, key)
    p = p0 * np.float32(2.0)
    x, y = ref.synth_raster(6, 5, 30, 40, 3)
    pk = ref.pack_time(x)
    fb = ref.forward_backward(BETA_NET, p, pk, 30, y, want_trace=True)
    st = State(p.copy())
    losses = [ref.train_step(BETA_NET, st, pk, 30, y)[0] for _ in range(3)]
    np.savez_compressed(os.path.join(GOLD, "betamodes.npz"), init=p0, params=p, packed=pk, y=y,
                        loss=np.float32(fb["loss"]), grads=fb["grads"], trace=fb["trace"],
                        step_losses=np.array(losses, np.float32), params3=st.params, m3=st.m,
                        v3=st.v)


def surrogate_fixture(ref: Lib):
    """g(x) of every surrogate through the reference's own tape (spike() over
    register_custom, surrogate.hpp:124-129): the five catalogue entries via
    make_activation and the declared sigmoid via custom(heaviside, bwd)."""
    x = np.concatenate([np.linspace(-3, 3, 601, dtype=np.float32),
                        np.array([0.0, -0.0, 1e-8, -1e-8, 40.0, -40.0, 1e4, -1e4], np.float32)])
    out = {"x": x}
    for act in ("custom", "superspike", "triangular", "arctan", "boxcar", "sigmoid"):
        out[act] = ref.surrogate(act, x)
        out[act + "_k5"] = ref.surrogate(act, x, slope=5.0, aux=0.25)
    np.savez_compressed(os.path.join(GOLD, "surrogates.npz"), **out)


if __name__ == "__main__":
    if not have_ref():
        Lib.__init__  # noqa: B018
        from oracle.pyoracle import build
        build()
    if not have_ref():
        sys.exit("oracle/_ref not buildable here (no /root/reference)")
    os.makedirs(GOLD, exist_ok=True)
    ref = Lib("ref")
    only = sys.argv[1] if len(sys.argv) > 1 else None  # e.g. "opts": one fixture
    if only in (None, "rng"):
        rng_kats(ref)
    if only in (None, "tiny"):
        tiny(ref)
    if only in (None, "c1"):
        c1(ref)
    if only in (None, "opts"):
        opts_fixture(ref)
    if only in (None, "ckpt"):
        checkpoint_fixture(ref)
    if only in (None, "spkd"):
        container_fixture(ref)
    if only in (None, "activity"):
        activity_fixture(ref)
    if only in (None, "shift"):
        shift_fixture(ref)
    if only in (None, "betamodes"):
        beta_modes_fixture(ref)
    if only in (None, "surrogates"):
        surrogate_fixture(ref)
    print("golden fixtures written to", GOLD)
