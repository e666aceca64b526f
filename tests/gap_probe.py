"""Where do the per-step microseconds outside the kernels go?  Times the schedule path
(8-step graphs) with fresh permuted rows of a 16384-example dataset vs the same 256
rows every step, and one-step graphs, all with CUDA events on the engine stream."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2402_18994_b200 import Engine, TrainConfig, shd_spec

eng = Engine(shd_spec(), TrainConfig(batch_size=256, seed=0), 128)
eng.synth_dataset(16384, seed=1)
stream = torch.cuda.ExternalStream(eng.stream)
N = 800
rng = np.random.default_rng(0)
fresh = np.concatenate([rng.permutation(16384)[:256] for _ in range(N)]).astype(np.uint32)
same = np.tile(np.arange(256, dtype=np.uint32), N)


def timed(fn, n):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    fn()
    e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1) * 1e3 / n


for name, rows in (("fresh rows", fresh), ("same rows", same)):
    eng.upload_schedule(rows)
    eng.enqueue_steps(0, 64)
    eng.sync()
    us = timed(lambda: eng.enqueue_steps(64, N - 64), N - 64)
    print(f"{name:12s} 8-step graphs: {us:.1f} us/step")
eng.upload_schedule(fresh)
eng.enqueue_steps(0, 16)
eng.sync()
us = timed(lambda: [eng.enqueue_step(16 + i) for i in range(400)], 400)
print(f"{'fresh rows':12s} 1-step graphs: {us:.1f} us/step")

# timeline of the last step of an 8-step graph vs a 1-step graph (debug stamps)
L = 2
def tl(tag):
    clk = eng.fetch("clk")
    spans = []
    t0 = None
    out = []
    for name, slot in (("fwd", 1), ("readout", 0), ("bwd1", 1 + L + 1), ("bwd0", 1 + L), ("wgrad", 1 + 2 * L), ("tail", 2 + 2 * L)):
        c = clk[slot]
        v = c[:, 14] > 0
        if not v.any():
            continue
        st, en = c[v, 14].min(), c[v, 15].max()
        if t0 is None:
            t0 = st
        out.append(f"{name} {(st - t0) / 1e3:.1f}-{(en - t0) / 1e3:.1f}")
    print(tag, " | ".join(out))
eng.debug(True)
eng.upload_schedule(fresh)
eng.enqueue_steps(0, 8); eng.sync()
eng.enqueue_steps(8, 8); eng.sync()
tl("8-step graph, last step:")
eng.enqueue_steps(16, 1); eng.sync()
eng.enqueue_steps(17, 1); eng.sync()
tl("1-step graph:          ")
eng.debug(False)

# spike rates and readout phases of the trained network
eng.debug(True)
eng.enqueue_steps(18, 1); eng.sync()
for l in range(L):
    print(f"layer {l} spike rate {eng.fetch('spikes', l).mean():.3f}")
c = eng.fetch("clk")[0][:256]
d = np.diff(c[:, :8], axis=1)
print("readout phases (trained)", np.median(d, axis=0).astype(int).tolist())
eng.debug(False)
