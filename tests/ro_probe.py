"""Readout (K4) per-CTA phase clocks in the trained regime (clocks-only debug mode):
[W+spikes load, projection, LI scan, CE, reverse, -, dI3 planes] cycles, median / p90 / max,
and the CTA start / end spread (globaltimer)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2402_18994_b200 import Engine, TrainConfig, shd_spec
B = 256
eng = Engine(shd_spec(), TrainConfig(batch_size=B, seed=0), 128)
eng.synth_dataset(16384, seed=1)
perm = eng.epoch_permutation(0, 16384)
sched = np.concatenate([perm[(i * B) % 16384:(i * B) % 16384 + B] for i in range(1200)]).astype(np.uint32)
eng.upload_schedule(sched)
if os.environ.get("PROBE_LOAD"):   # A/B builds: the same trained state (and rasters) for each
    eng.load_checkpoint(os.environ["PROBE_LOAD"])
else:
    eng.enqueue_steps(0, 1192)
    eng.sync()
    if os.environ.get("PROBE_SAVE"):
        eng.save_checkpoint(os.environ["PROBE_SAVE"])
eng.debug(2)
eng.enqueue_steps(1192, 8)
eng.sync()
clk = eng.fetch("clk")[0][:B]
d = np.diff(clk[:, :8], axis=1)
tot = clk[:, 7] - clk[:, 0]
for name, f in (("median", np.median), ("p90", lambda x, axis: np.percentile(x, 90, axis=axis)), ("max", np.max)):
    print(f"{name:6s}", f(d, axis=0).astype(int).tolist(), int(f(tot, axis=0)))
gt = clk[:, 14:16]
t0 = gt[:, 0].min()
print(f"start spread {(gt[:, 0].max() - t0) / 1e3:.1f} us; end {(gt[:, 1].min() - t0) / 1e3:.1f}..{(gt[:, 1].max() - t0) / 1e3:.1f} us")
slow = np.argsort(tot)[-5:]
print("slowest CTAs", slow.tolist(), d[slow].tolist())
eng.debug(True)
eng.enqueue_steps(1192, 1)
eng.sync()
s1 = eng.fetch("spikes", 1)
per = s1.sum(axis=(1, 2))
print("layer-1 spikes per sample: median", int(np.median(per)), "max", int(per.max()), "rate", s1.mean())
# per-step spike counts: a warp of the projection walks 16 steps, its loop runs the
# max over them; a CTA's projection phase is its slowest warp
cnt = s1.sum(axis=2)  # [B, T]
T = cnt.shape[1]
wmax = cnt[:, :T - T % 16].reshape(B, -1, 16).max(axis=2)
print("per-step spikes: mean", cnt.mean(), "max", cnt.max(), "| per-warp max: median",
      np.median(wmax), "| per-CTA max warp-max: median", np.median(wmax.max(1)))
print("corr(projection cycles, CTA max warp-max)", np.corrcoef(d[:, 1], wmax.max(1))[0, 1],
      "cycles per warp-max spike", np.median(d[:, 1] / np.maximum(wmax.max(1), 1)))
# per-warp end of the projection (clk[16 + warp]) relative to the phase start (clk[1])
pw = clk[:, 16:24] - clk[:, 1:2]
print("projection end per warp (median over CTAs)", np.median(pw, axis=0).astype(int).tolist(),
      "max", pw.max(axis=0).tolist())
