"""H2D bandwidth of the 2.87 MB C1 host batch, alone and while training steps run
(engine schedule steps on the engine stream, copies on a torch side stream)."""
import os, sys, time
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2402_18994_b200 import Engine, TrainConfig, shd_spec

nbytes = 256 * 16 * 700
pin = torch.empty((64, nbytes), dtype=torch.uint8, pin_memory=True)
dev = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
side = torch.cuda.Stream()
def copies(n=64):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(side):
        e0.record()
        for i in range(n):
            dev.copy_(pin[i], non_blocking=True)
        e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) * 1e3 / n
copies()
print(f"alone: {copies():.1f} us per batch")
B = 256
eng = Engine(shd_spec(), TrainConfig(batch_size=B, seed=0), 128)
eng.synth_dataset(4096, seed=1)
rows = np.arange(B, dtype=np.uint32)
eng.upload_schedule(np.tile(rows, 512))
eng.enqueue_steps(0, 8); eng.sync()
eng.enqueue_steps(0, 512)      # ~65 ms of training on the engine stream
time.sleep(0.002)
print(f"under load: {copies():.1f} us per batch")
eng.sync()
