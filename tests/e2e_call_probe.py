"""Per-call cost of snn_train_steps_packed (C1, pinned host batches): wall time per
call of n steps against n device steps, and the same with the call's pieces timed."""
import os, sys, time
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2402_18994_b200 import Engine, TrainConfig, shd_spec

B, n = 256, int(os.environ.get("PROBE_N", "64"))
eng = Engine(shd_spec(), TrainConfig(batch_size=B, seed=0), 128)
eng.synth_dataset(4096, seed=1)
pk, y = eng.read_dataset(0, 4096)
batches = torch.empty((n, B) + pk.shape[1:], dtype=torch.uint8, pin_memory=True).numpy()
labels = np.zeros((n, B), np.int64)
for k in range(n):
    j = k % (4096 // B)
    batches[k] = pk[j * B:(j + 1) * B]
    labels[k] = y[j * B:(j + 1) * B]
for _ in range(3):
    eng.train_steps_packed(batches, labels)
rows = np.arange(B, dtype=np.uint32)
eng.train_step(rows)
torch.cuda.synchronize()
calls = 20
t0 = time.perf_counter()
for _ in range(calls):
    eng.train_steps_packed(batches, labels)
dt = (time.perf_counter() - t0) / calls
print(f"train_steps_packed: {dt * 1e6:.0f} us per call of {n} = {dt / n * 1e6:.2f} us/step")
# device-side reference: the same n steps as 8-step schedule graphs
eng.upload_schedule(np.tile(rows, n))
eng.enqueue_steps(0, n)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(calls):
    eng.enqueue_steps(0, n)
    eng.sync()
dt2 = (time.perf_counter() - t0) / calls
print(f"schedule steps (device-resident batches): {dt2 * 1e6:.0f} us per {n} = {dt2 / n * 1e6:.2f} us/step")
