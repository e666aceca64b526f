"""Phase timestamps (clock64) of the readout, forward and backward kernels (debug mode)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2402_18994_b200 import Engine, TrainConfig, shd_spec
BATCH = int(os.environ.get("PROBE_B", "256"))
eng = Engine(shd_spec(), TrainConfig(batch_size=BATCH, seed=0), 128)
eng.synth_dataset(16384, seed=1)
eng.debug(True)
rows = np.arange(BATCH, dtype=np.uint32)
for _ in range(3):
    eng.train_step(rows)
clk = eng.fetch("clk")
L = 2
names = ["readout"] + [f"fwd{l}" for l in range(L)] + [f"bwd{l}" for l in range(L)]
for s, name in enumerate(names):
    c = clk[s, :256]
    n = 8 if name == "readout" else (4 if name.startswith("fwd") else 7)
    d = np.diff(c[:, :n], axis=1)
    print(f"{name:8s} phase cycles median {np.median(d, axis=0).astype(int).tolist()} max {d.max(axis=0).tolist()} total med {int(np.median(c[:, n-1]-c[:, 0]))}")
for s, name in ((1, "fwd0"), (2, "fwd1")):
    c = clk[s]
    valid = c[:, 6] > 0
    if not valid.any():
        continue
    st, en = c[valid, 6], c[valid, 7]
    t0 = st.min()
    print(f"{name}: CTAs {valid.sum()}  start spread {(st.max()-t0)/1e3:.1f} us  end spread {(en.min()-t0)/1e3:.1f}..{(en.max()-t0)/1e3:.1f} us  per-CTA median {np.median(en-st)/1e3:.1f} us")
c = clk[1 + 2 * L]
valid = c[:, 6] > 0
c = c[valid]
d = np.stack([c[:, 1] - c[:, 0], c[:, 2] - c[:, 1], c[:, 3] - c[:, 2], c[:, 4] - c[:, 3], c[:, 5] - c[:, 4]], 1)
print("wgrad CTAs", valid.sum(), "[prologue, first-stage, mma-loop, commit->epi, epilogue] median", np.median(d, 0).astype(int).tolist(), "max", d.max(0).tolist())
gt = c[:, 6:8]; t0 = gt[:, 0].min()
print(f"wgrad start spread {(gt[:,0].max()-t0)/1e3:.1f} us, end {(gt[:,1].min()-t0)/1e3:.1f}..{(gt[:,1].max()-t0)/1e3:.1f} us; clock {np.median((c[:,5]-c[:,0])/((gt[:,1]-gt[:,0])*1e-3)):.0f} MHz")
for blk in (0, 60, 119, 125, 140, 147):
    if blk < len(c): print("  cta", blk, (c[blk, 1:6] - c[blk, 0:5]).tolist())
c = clk[1][:128]
g = c[:, 1] - c[:, 0]
sm = c[:, 4]
order = np.argsort(g)
print("fwd0 GEMM-phase cycles by CTA (fastest 6 / slowest 10): ", [(int(i), int(sm[i]), int(g[i])) for i in order[:6]], [(int(i), int(sm[i]), int(g[i])) for i in order[-10:]])
print("  slow (> 1.5x median) CTA ids:", sorted(np.where(g > 1.5 * np.median(g))[0].tolist()))
print("  smids of slow:", sorted(sm[g > 1.5 * np.median(g)].tolist()))

# timeline of one replay (globaltimer slots 14/15), kernels in launch order
order = [f"fwd{l}" for l in range(L)] + ["readout"] + [f"bwd{l}" for l in reversed(range(L))] + ["wgrad", "tail"]
slot = {"readout": 0, "wgrad": 1 + 2 * L, "tail": 2 + 2 * L, **{f"fwd{l}": 1 + l for l in range(L)}, **{f"bwd{l}": 1 + L + l for l in range(L)}}
t0 = None
for name in order:
    c = clk[slot[name]]
    v = c[:, 14] > 0
    if not v.any():
        print(f"TL {name:8s} (fused into another launch)")
        continue
    st, en = c[v, 14], c[v, 15]
    if t0 is None: t0 = st.min()
    print(f"TL {name:8s} ctas {v.sum():4d} start {(st.min()-t0)/1e3:7.1f} .. {(st.max()-t0)/1e3:7.1f}  end {(en.min()-t0)/1e3:7.1f} .. {(en.max()-t0)/1e3:7.1f} us  span {(en.max()-st.min())/1e3:6.1f}  cta med {np.median(en-st)/1e3:5.1f}")

# forward layer-0 per-k-block stage readiness (MMA thread), cycles from CTA start
c = clk[1][:max(1, BATCH // 2)]
for blk in sorted({0, min(64, BATCH // 2 - 1)}):
    print(f"fwd0 cta {blk}: kblock ready", (c[blk, 16:16 + 11] - c[blk, 0]).tolist(), " scan start", int(c[blk, 1] - c[blk, 0]))
