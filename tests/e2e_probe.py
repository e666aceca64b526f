"""Host<->device costs of one e2e step (2.87 MB packed C1 batch)."""
import os, sys, time
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2402_18994_b200 import Engine, TrainConfig, shd_spec

nbytes = 256 * 16 * 700
x = np.random.default_rng(0).integers(0, 255, nbytes, dtype=np.uint8)
dev = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
pin = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
pn = pin.numpy()
torch.cuda.synchronize()

def t(fn, n=50):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e6

print(f"pageable H2D      {t(lambda: dev.copy_(torch.from_numpy(x), non_blocking=False)):.1f} us")
print(f"host memcpy->pin  {t(lambda: np.copyto(pn, x)):.1f} us")
print(f"pinned H2D        {t(lambda: dev.copy_(pin, non_blocking=True)):.1f} us")
print(f"os.cpu_count      {os.cpu_count()}")

eng = Engine(shd_spec(), TrainConfig(batch_size=256, seed=0), 128)
eng.synth_dataset(4096, seed=1)
pk, y = eng.read_dataset(0, 256)
eng.train_step_packed(pk, y)
print(f"train_step_packed {t(lambda: eng.train_step_packed(pk, y), 100):.1f} us/step")
import ctypes
t0 = time.perf_counter()
for _ in range(400):
    eng.train_step_packed(pk, y)
print(f"python loop {(time.perf_counter() - t0) / 400 * 1e6:.1f} us/step")
