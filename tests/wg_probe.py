"""Phase clocks of k_wgrad with the fused step tail (debug mode, C1): per CTA
[prologue, first stage, MMA loop, commit->epilogue, TMEM->smem staging,
vector entries, loss, TMA store drain, tile wait, first partial load, first chunk
sum+Adam] in cycles."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2402_18994_b200 import Engine, TrainConfig, shd_spec
eng = Engine(shd_spec(), TrainConfig(batch_size=256, seed=0, gemm_planes=int(os.environ.get("PROBE_PLANES", "3"))), 128)
eng.synth_dataset(16384, seed=1)
eng.debug(2)  # clock stamps only
rows = np.arange(256, dtype=np.uint32)
for _ in range(3):
    eng.train_step(rows)
clk = eng.fetch("clk")
L = 2
c = clk[1 + 2 * L]
valid = c[:, 6] > 0
c = c[valid]
cols = [(1, 0), (2, 1), (3, 2), (4, 3), (10, 4), (11, 10), (8, 11), (9, 8), (12, 9), (13, 12)]
d = np.stack([c[:, a] - c[:, b] for a, b in cols], 1)
print("wgrad CTAs", valid.sum())
print("  [prologue, first-stage, mma-loop, commit->epi, staging+vec, loss, store-drain, tile-wait, load, sum+adam] cycles")
print("  median", np.median(d, 0).astype(int).tolist())
print("  max   ", d.max(0).tolist())
gt = c[:, 6:8]
t0 = gt[:, 0].min()
print(f"  start spread {(gt[:, 0].max() - t0) / 1e3:.1f} us, end {(gt[:, 1].min() - t0) / 1e3:.1f}..{(gt[:, 1].max() - t0) / 1e3:.1f} us")
for blk in (0, 52, 53, 105, 106, 126, 127, len(c) - 1):
    if blk < len(c):
        print("  cta", blk, d[blk].tolist(), f"start {(gt[blk, 0] - t0) / 1e3:.1f} us")
if os.environ.get("PROBE_ALL"):
    tot = c[:, 13] - c[:, 0]
    for blk in range(len(c)):
        print(f"  {blk:3d} loop {d[blk, 2]:6d} epi {int(c[blk, 13] - c[blk, 4]):6d} total {int(tot[blk]):6d} "
              f"end {(gt[blk, 1] - t0) / 1e3:5.1f} us")
if os.environ.get("PROBE_ALL"):
    # absolute arrival on the tile counter (globaltimer start + clock64 delta at ~1.965 GHz)
    arr = (gt[:, 0] - t0) / 1e3 + (c[:, 8] - c[:, 0]) / 1965.0
    for lo, hi in ((0, 54), (54, 108), (108, 129), (129, len(c))):
        o = np.argsort(arr[lo:hi])[::-1][:4] + lo
        print(f"  CTAs [{lo},{hi}) latest arrivals", [(int(i), round(float(arr[i]), 1)) for i in o],
              "median", round(float(np.median(arr[lo:hi])), 1))
if os.environ.get("PROBE_LAYERS"):
    # per-layer loop / total cycles (layer ranges from the engine's split plan)
    info = eng.wgrad_plan() if hasattr(eng, "wgrad_plan") else None
    loop = c[:, 3] - c[:, 2]
    tot = c[:, 13] - c[:, 0]
    edges = [int(x) for x in os.environ["PROBE_LAYERS"].split(",")]
    for lo, hi in zip(edges[:-1], edges[1:]):
        print(f"  CTAs [{lo},{hi}) loop median {int(np.median(loop[lo:hi]))} max {int(loop[lo:hi].max())}"
              f"  total median {int(np.median(tot[lo:hi]))} max {int(tot[lo:hi].max())}")
