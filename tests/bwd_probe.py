"""Backward-kernel phase clocks (clocks-only debug mode) at a given config:
[gemm, compose, chain, replay, combine, end] cycles per CTA (median / max), the
first t-tile only; e.g. PROBE_CFG=c3w for the wide 700-1024-1024-20 layers."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import WORKLOADS  # noqa: E402
from paper_2402_18994_b200 import Engine, TrainConfig, shd_spec  # noqa: E402
w = WORKLOADS[os.environ.get("PROBE_CFG", "c3w")]
B = int(os.environ.get("PROBE_B", str(w["B"])))
eng = Engine(shd_spec(hidden=w["hidden"], classes=w["classes"], inp=w["inp"], act=w["act"]),
             TrainConfig(batch_size=B, seed=0, gemm_planes=int(os.environ.get("PROBE_PLANES", "3"))), w["T"])
eng.synth_dataset(2 * B, seed=1)
rows = np.arange(B, dtype=np.uint32)
for _ in range(20):
    eng.train_step(rows)
eng.debug(2)
eng.train_step(rows)
clk = eng.fetch("clk")
L = len(w["hidden"])
for l in reversed(range(L)):
    c = clk[1 + L + l]
    v = c[:, 14] > 0
    d = np.diff(c[v][:, :7], axis=1)
    print(f"bwd{l} CTAs {v.sum()} [gemm, compose, chain, replay, combine, end] median",
          np.median(d, 0).astype(int).tolist(), "max", d.max(0).tolist())
