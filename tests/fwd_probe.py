"""Phase clocks of the fused forward (debug mode, C1): per CTA
[GEMM0 (start -> layer-0 accumulator ready), scan0, GEMM1 wait, scan1] cycles,
and the backward kernels' phases [GEMM, compose, chain, replay, tail]."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2402_18994_b200 import Engine, TrainConfig, shd_spec
B = int(os.environ.get("PROBE_B", "256"))
eng = Engine(shd_spec(), TrainConfig(batch_size=B, seed=0, gemm_planes=int(os.environ.get("PROBE_PLANES", "3"))), 128)
eng.synth_dataset(16384, seed=1)
rows = np.arange(B, dtype=np.uint32)
for _ in range(int(os.environ.get("PROBE_TRAIN", "300"))):   # trained-like spike rates
    eng.train_step(rows)
eng.debug(2)  # clock stamps only
for _ in range(2):
    eng.train_step(rows)
clk = eng.fetch("clk")
c = clk[1][: B // 2]
d = np.stack([c[:, 8] - c[:, 0], c[:, 9] - c[:, 8], c[:, 10] - c[:, 9], c[:, 11] - c[:, 10]], 1)
print("fwd CTAs", len(c), "[GEMM0, scan0, GEMM1 wait, scan1] median", np.median(d, 0).astype(int).tolist(),
      "max", d.max(0).tolist())
for l in (1, 0):
    c = clk[3 + l][:B]
    d = np.diff(c[:, :7], axis=1)
    print(f"bwd{l} [gemm, compose, chain, replay, combine, end] median", np.median(d, 0).astype(int).tolist())
c = clk[0][:B]
print("readout phases", np.median(np.diff(c[:, :8], axis=1), 0).astype(int).tolist())
eng.debug(True)
eng.train_step(rows)
for l in range(2):
    print(f"layer {l} spike rate {eng.fetch('spikes', l).mean():.3f}")
if os.environ.get("PROBE_KB"):
    # MMA-warp time stamps at each k-block's full-barrier pass (clk[16 + it])
    c = eng.fetch("clk")[1][: B // 2]
    kbt = c[:, 16:16 + 11].astype(np.int64)
    print("k-block issue deltas (median)", np.median(np.diff(kbt, axis=1), 0).astype(int).tolist(),
          "first after start", int(np.median(kbt[:, 0] - c[:, 0])))
