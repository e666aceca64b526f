"""One C1 training step (and one forward/backward) for compute-sanitizer runs:
    compute-sanitizer --tool memcheck|racecheck|synccheck python tests/sanitize_step.py
Small dataset (512 examples) so the sanitized synth stays short."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2402_18994_b200 import Engine, TrainConfig, shd_spec
cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
cell = {"c1": "lif", "c2": "alif", "c4": "rlif"}[cfg]
hid = (512, 512) if cfg == "c4" else (128, 128)
B = 64 if cfg == "c4" else 256
eng = Engine(shd_spec(hidden=hid, cell=cell, act="superspike" if cfg == "c2" else "arctan"),
             TrainConfig(batch_size=B, seed=0), 128)
eng.synth_dataset(512, seed=1)
rows = np.arange(B, dtype=np.uint32)
print("train_step", eng.train_step(rows))
print("forward_backward", eng.forward_backward(rows))
print("train_step", eng.train_step(rows + 1))
eng.close()
print("sanitize_step ok")
