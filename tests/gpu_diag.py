"""Verbose GPU-vs-oracle diagnostics (run on the B200 box, prints a report).

    python tests/gpu_diag.py [--big]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle.pyoracle import Lib, Net  # noqa: E402
import scanref  # noqa: E402
from paper_2402_18994_b200 import Engine, TrainConfig, shd_spec  # noqa: E402


def relnorm(a, b):
    return float(np.linalg.norm(a.astype(np.float64) - b) / max(np.linalg.norm(b.astype(np.float64)), 1e-30))


def run(net: Net, B, T, seed, scale=1.0, params=None, n_ex=None, label=""):
    orc = Lib("orc")
    spec = shd_spec(hidden=net.hidden, classes=net.classes, inp=net.inp, act=net.act, bias=net.bias)
    eng = Engine(spec, TrainConfig(batch_size=B, seed=0, unroll=net.unroll), T)
    if params is None:
        params = orc.init(net, orc.key_child(orc.key_from_seed(seed), 0)) * np.float32(scale)
    n_ex = n_ex or B
    x, y = orc.synth_raster(net.classes, n_ex, T, net.inp, seed + 1)
    pk = orc.pack_time(x)
    eng.stage_dataset(pk, y)
    eng.set_params(params)
    back = eng.get_params()
    print(f"[{label}] params roundtrip exact: {np.array_equal(back, params)}")
    eng.debug(True)
    rows = np.arange(B, dtype=np.uint32)
    t0 = time.time()
    loss, acc = eng.forward_backward(rows)
    print(f"[{label}] gpu fwd_bwd {time.time()-t0:.3f}s loss {loss!r} acc {acc}")
    ref = orc.forward_backward(net, params, pk[:B], T, y[:B], want_spikes=True, want_trace=True,
                               want_v=True)
    print(f"[{label}] orc loss {ref['loss']!r} acc {ref['acc']}  rel {abs(loss-ref['loss'])/abs(ref['loss']):.3e}")
    # layer-wise
    X = orc.unpack_time(pk[:B], T).astype(np.float64)
    ents = {n: (o, s) for n, o, s in orc.entries(net)}
    A = X
    for l, h in enumerate(net.hidden):
        o, s = ents[f"l{2*l}.w"]
        W = params[o:o + s].reshape(-1, h).astype(np.float64)
        I_true = A @ W
        I_gpu = eng.fetch("I", l)
        err = np.abs(I_gpu - I_true).max()
        print(f"[{label}] L{l} I max abs err {err:.3e} (scale {np.abs(I_true).max():.3e})")
        ob, sb = ents[f"l{2*l+1}.beta"]
        V_ref, S_ref = scanref.lif_forward(I_gpu, params[ob:ob + sb], net.threshold)
        V_gpu = eng.fetch("V", l)
        S_gpu = eng.fetch("spikes", l)
        print(f"[{label}] L{l} scan-given-I exact: V {np.array_equal(V_gpu, V_ref)} "
              f"S {np.array_equal(S_gpu, S_ref)}; spike agreement vs oracle "
              f"{(S_gpu == ref['spikes'][l]).mean()*100:.5f}% rate {S_gpu.mean():.4f}")
        A = S_gpu.astype(np.float64)
    tr = eng.fetch("trace")
    print(f"[{label}] trace rel {relnorm(tr, ref['trace']):.3e}")
    for l in range(len(net.hidden)):
        dS = eng.fetch("dS", l)
        print(f"[{label}] L{l} dS finite {np.isfinite(dS).all()} absmax {np.abs(dS).max():.3e}")
    g = eng.get_grads()
    for name, o, s in orc.entries(net):
        print(f"[{label}] grad {name:8s} relnorm {relnorm(g[o:o+s], ref['grads'][o:o+s]):.3e}"
              f"  |g| {np.linalg.norm(ref['grads'][o:o+s]):.3e}")
    # one Adam step vs oracle
    from oracle.pyoracle import State
    st = State(params.copy())
    lo, _ = orc.train_step(net, st, pk[:B], T, y[:B])
    eng.debug(False)
    l2, _ = eng.train_step(rows)
    p2 = eng.get_params()
    print(f"[{label}] after 1 step: loss {l2!r} vs {lo!r}; param relnorm {relnorm(p2, st.params):.3e}"
          f" max abs {np.abs(p2 - st.params).max():.3e}")
    eng.close()


if __name__ == "__main__":
    run(Net(inp=30, hidden=(16, 12), classes=5, unroll=4), B=6, T=19, seed=5, scale=3.0, label="tiny")
    run(Net(inp=70, hidden=(40, 24), classes=7, act="superspike"), B=5, T=70, seed=9, scale=3.0,
        label="small-T70")
    run(Net(), B=16, T=128, seed=0, scale=1.0, label="c1-init-B16")
    if "--big" in sys.argv:
        run(Net(), B=256, T=128, seed=0, scale=2.0, label="c1-B256-x2")
