"""Profiling driver: C1 engine, W warm-up steps, then P profiled steps.

    ncu ... python tests/prof_step.py [--warmup 3] [--steps 1] [--config c1]
Kernels per step: see Engine.launches_per_step (synth is launched once first).
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import WORKLOADS  # noqa: E402
from paper_2402_18994_b200 import Engine, TrainConfig, shd_spec  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--config", default="c1")
    args = ap.parse_args()
    w = WORKLOADS[args.config]
    eng = Engine(shd_spec(hidden=w["hidden"], classes=w["classes"], inp=w["inp"], act=w["act"],
                          cell=w.get("cell", "lif")),
                 TrainConfig(batch_size=w["B"], seed=0), w["T"])
    eng.synth_dataset(w["n_data"], seed=1)
    perm = eng.epoch_permutation(0, w["n_data"])
    n = args.warmup + args.steps
    rows = np.concatenate([perm[i * w["B"]:(i + 1) * w["B"]] for i in range(n)])
    eng.upload_schedule(rows)
    for i in range(n):
        eng.enqueue_step(i)
    eng.sync()
    print("launches/step", eng.launches_per_step, "loss", eng.read_result())


if __name__ == "__main__":
    main()
