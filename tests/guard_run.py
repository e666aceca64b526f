"""Out-of-bounds write sweep (run with SNN_GUARD=1; tests/test_gpu_guards.py).

compute-sanitizer is not available on this GPU pool, so every device buffer is
allocated with 4 KB of a known pattern past its end and checked after each case:
train steps, forward/backward, apply, evaluate and the schedule graphs across the
kernel variants (fused / unfused forward, ragged widths, multi-tile T, ALIF, RLIF
on all three reverse-scan paths, LIF readout, monitors, bias, fast GEMM modes,
the peer tail with emulated ranks)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle.pyoracle import Lib, Net  # noqa: E402
from test_gpu_parity import make_engine  # noqa: E402

assert os.environ.get("SNN_GUARD") == "1", "run with SNN_GUARD=1"
orc = Lib("orc")
CASES = [
    ("c1", Net(), 64, 128, {}),
    ("c1-bf16x2", Net(), 64, 128, dict(gemm_planes=2)),
    ("ragged-3hidden-bias", Net(inp=50, hidden=(130, 48, 33), classes=7, bias=True), 5, 37, {}),
    ("T200-two-tiles", Net(inp=64, hidden=(128, 128), classes=10), 3, 200, {}),
    ("T1000", Net(inp=700, hidden=(256, 256), classes=20), 2, 1000, {}),
    ("wide-1024", Net(inp=700, hidden=(1024, 1024), classes=20), 2, 256, {}),
    ("alif", Net(act="superspike", cell=("alif", "alif")), 40, 128, {}),
    ("rlif-512-tc", Net(inp=700, hidden=(512, 512), classes=20, cell=("rlif", "rlif")), 50, 128, {}),
    ("rlif-250-cluster", Net(inp=60, hidden=(250, 40), classes=5, cell=("rlif", "lif")), 11, 40, {}),
    ("rlif-small", Net(inp=30, hidden=(40, 24), classes=5, cell=("rlif", "alif")), 4, 25, {}),
    ("lif-readout-mse", Net(inp=40, hidden=(24,), classes=4, bias=True, readout="lif"), 5, 45,
     dict(loss="spike_rate_mse")),
    ("monitor-reg", Net(inp=40, hidden=(24, 20), classes=5, monitor=(0, 1)), 6, 30,
     dict(lambda_low=1.0, lambda_high=1.0, f_min=0.05, f_max=0.3)),
    ("sigmoid-sgd", Net(inp=64, hidden=(96, 40), classes=8, act="sigmoid"), 5, 45,
     dict(optimizer="sgd", momentum=0.5)),
]
total = 0
for name, net, B, T, cfg in CASES:
    x, y = orc.synth_raster(net.classes, 3 * B, T, net.inp, 2)
    pk = orc.pack_time(x)
    eng = make_engine(net, B, T, **cfg)
    eng.stage_dataset(pk, y)
    eng.set_params(eng.get_params() * np.float32(2.0))
    rows = np.arange(B, dtype=np.uint32)
    eng.train_step(rows)
    eng.forward_backward(rows + B)
    eng.apply(rows)
    eng.evaluate(np.arange(3 * B, dtype=np.uint32))
    eng.upload_schedule(np.arange(8 * B, dtype=np.uint32) % (3 * B))
    eng.enqueue_steps(0, 8)
    eng.sync()
    eng.train_step_packed(pk[:B], y[:B])
    n = eng.check_guards()
    total += n
    print(f"{name}: {n} buffers clean", flush=True)
    eng.close()
# the peer tail with 2 emulated ranks (owner phase + gather write remote-mapped memory)
from paper_2402_18994_b200 import Engine  # noqa: E402
net = Net(inp=40, hidden=(24, 20), classes=5)
x, y = orc.synth_raster(5, 16, 23, 40, 8)
pk = orc.pack_time(x)
engs = [make_engine(net, 4, 23, seed=5) for _ in range(2)]
Engine.peer_attach_local(engs)
for e in engs:
    e.stage_dataset(pk, y)
for step in range(2):
    for r, e in enumerate(engs):
        e.train_step_split(np.arange(r * 4, r * 4 + 4, dtype=np.uint32), 0)
    for e in engs:
        e.train_step_split(None, 1)
    for e in engs:
        e.train_step_split(None, 2)
print(f"peer tail: {engs[0].check_guards()} buffers clean")
print(f"GUARDS OK ({total} buffer checks)")
