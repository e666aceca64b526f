import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2402_18994_b200 import Engine, TrainConfig, shd_spec
eng = Engine(shd_spec(), TrainConfig(batch_size=256, seed=0), 128)
eng.synth_dataset(16384, seed=1)
eng.debug(True)  # clocks + debug tensors
rows = np.arange(256, dtype=np.uint32)
for _ in range(3):
    eng.forward_backward(rows)
clk = eng.fetch("clk")
d = np.diff(clk, axis=1)
print("phase cycles (median over CTAs):", np.median(d, axis=0).astype(int).tolist())
print("phase cycles (max):", d.max(axis=0).tolist())
print("start spread:", int(clk[:, 0].max() - clk[:, 0].min()), "end spread", int(clk[:, 7].max() - clk[:, 0].min()))
