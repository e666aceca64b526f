"""The drop-in proof (VERDICT r1 "compiled reference-side drop-in").

tests/dropin/train_swap is the reference's OWN train() (optimize.hpp:237-299,
compiled from the unmodified headers) with train_step<float> swapped for the
B200 engine by include/spiketrain_b200_adapter.hpp (an explicit specialization;
not one line of the reference changes).  Against the pure reference
(oracle/_ref: the same headers, CPU train_step) on the same .spkd container, the
epoch metrics and the final parameters must agree within the north_star bar.
"""
import os
import subprocess

import numpy as np
import pytest

from oracle.pyoracle import Lib, Net, State, have_ref

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "dropin", "_build", "train_swap")

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not os.path.exists(BIN) or not have_ref(),
                    reason="drop-in binary / oracle/_ref not built (need /root/reference at build time)")
@pytest.mark.parametrize("act", ["arctan", "superspike"])
def test_reference_train_with_gpu_step(tmp_path, act):
    ref = Lib("ref")
    T, N, B, E, H = 128, 256, 64, 3, 128
    x, y = ref.synth_raster(20, N, T, 700, 1)
    pk = ref.pack_time(x)
    data = str(tmp_path / "data.spkd")
    ref.write_container(data, pk, T, y)
    out = str(tmp_path / "out.bin")
    r = subprocess.run([BIN, data, str(H), act, str(E), str(B), "0", out], capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    net = Net(hidden=(H, H), act=act)
    n = ref.param_count(net)
    raw = open(out, "rb").read()
    metrics = np.frombuffer(raw[:16 * E], np.float64).reshape(E, 2)
    params = np.frombuffer(raw[16 * E:16 * E + 4 * n], np.float32)
    step = int(np.frombuffer(raw[16 * E + 4 * n:], np.uint64)[0])
    # the pure reference: same spec, config, seed and container
    st = State(ref.init(net, ref.key_child(ref.key_from_seed(0), 0)))
    m_ref = ref.train_epochs(net, st, pk, y, T, B, E, 0)
    print(f"{act}: reference {m_ref.tolist()}\n  swapped {metrics.tolist()}")
    assert step == st.step == E * (N // B)
    assert np.allclose(metrics[:, 0], m_ref[:, 0], rtol=1e-3), (metrics, m_ref)
    assert np.abs(metrics[:, 1] - m_ref[:, 1]).max() <= 1.0 / B + 1e-12
    rel = np.linalg.norm(params - st.params) / np.linalg.norm(st.params)
    assert rel <= 1e-4, rel
