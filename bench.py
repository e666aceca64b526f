#!/usr/bin/env python
"""bench.py -- SNN train samples/s (fwd + bwd + Adam, SHD shape) on B200.

Default: N=1, configuration C1 of BASELINE.json (700-128-128-20 LIF, T=128,
batch 256, arctan surrogate, integral CE + Adam).  One "step" = one full
train_step over one batch drawn from an HBM-resident synthetic dataset that
is larger than L2 (16384 examples, 184 MB staged), fresh rows every step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (data-parallel; started bare with
                                                         --gpus N it launches the N ranks itself)

Prints ONE JSON line on rank 0.  The `reference` arm times the reference's own
CPU train_step (oracle/_ref, built from /root/reference) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

E2E_CHUNK = int(os.environ.get("SNN_E2E_CHUNK", "64"))  # host batches per snn_train_steps_packed call in the e2e leg
METRIC = "SNN train samples/sec (fwd+bwd+Adam, SHD shape) at 1/2/4/8 B200 vs CPU ref"
UNIT = "samples/s"

WORKLOADS = {
    # name: input, hidden, classes, T, per-GPU batch, surrogate, dataset examples
    "c1": dict(inp=700, hidden=(128, 128), classes=20, T=128, B=256, act="arctan", n_data=16384,
               desc="SHD-shaped 700-128-128-20 LIF, T=128, batch 256/GPU, arctan k=2, "
                    "integral-CE + Adam, nobias"),
    "c2": dict(inp=700, hidden=(128, 128), classes=20, T=128, B=1024, act="superspike",
               cell="alif", n_data=16384,
               desc="SHD-shaped 700-128-128-20 ALIF (declared cell, oracle/spiketrain_oracle.h), "
                    "T=128, batch 1024/GPU, superspike k=25, integral-CE + Adam, nobias"),
    # BASELINE configs[2]: global batch 4096 sharded over the N GPUs (strong scaling)
    "c3": dict(inp=700, hidden=(1024, 1024), classes=20, T=256, B=4096, global_batch=True,
               act="arctan", n_data=16384,
               desc="wide 700-1024-1024-20 LIF, T=256, global batch 4096 sharded over the GPUs"),
    "c3w": dict(inp=700, hidden=(1024, 1024), classes=20, T=256, B=512, act="arctan", n_data=8192,
                desc="wide 700-1024-1024-20 LIF, T=256, batch 512/GPU (weak scaling)"),
    "c4": dict(inp=700, hidden=(512, 512), classes=20, T=128, B=256, act="arctan", cell="rlif",
               n_data=8192,
               desc="recurrent 700-512-512-20 RLIF (declared cell, oracle/spiketrain_oracle.h), "
                    "T=128, batch 256/GPU (B unstated in BASELINE; SURVEY §8), arctan k=2"),
    "c5": dict(inp=700, hidden=(256, 256), classes=20, T=1000, B=512, act="arctan", n_data=2048,
               desc="long-sequence 700-256-256-20 LIF, T=1000, batch 512/GPU"),
}


def peaks():
    """(HBM GB/s, dense bf16 TFLOP/s burst, source): the burst figures, since each
    kernel is timed alone (a few tens of us) inside the profiling graph."""
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        p = json.load(open(path))
        return float(p["hbm_gbs"]), float(p["bf16_tflops"]), "measured (MEASURED_PEAKS.json hbm_gbs, bf16_tflops burst)"
    except Exception:
        return 6650.0, 1590.0, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clocks + throttle reasons during the timed region: NVML polled every 2 ms
    on a thread, plus explicit samples (`mark()`) taken while the enqueued steps
    are running, so even a region of a few ms carries samples."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4}

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._h = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
        except Exception:
            self._h = None
        return self

    def mark(self):
        if self._h is None:
            return
        try:
            nv = self._nv
            self.samples.append((nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM),
                                 nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)))
        except Exception:
            pass

    def _poll(self):
        while not self._stop.wait(0.002):
            self.mark()

    def __exit__(self, *a):
        self._stop.set()
        if self._h is not None:
            self.thread.join(1.0)

    def summary(self):
        sm = [s for s, _ in self.samples]
        reasons = sorted({n for _, r in self.samples for n, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": getattr(self, "max_mhz", None), "reasons": reasons,
                "samples": len(sm), "source": "NVML (2 ms poll + samples while the steps run)"}


# ------------------------------------------------------------------ roofline
def algorithmic(name: str, w: dict, n_params: int, fwd_groups=None, B=None):
    """Algorithmic work per launch from SURVEY.md §8(d)'s per-unit figures:
    {"tensor": flops, "hbm": bytes} (either may be 0).  A fused GEMM + scan launch
    carries both; the binding one is the larger fraction of its peak.
    fwd_groups: Engine.forward_launches -- a fused forward launch does every layer
    it covers."""
    B = B or w["B"]
    T, C = w["T"], w["classes"]
    dims = [w["inp"], *w["hidden"], C]
    alif = w.get("cell") == "alif"
    base, _, idx = name.partition("[")
    l = int(idx.rstrip("]")) if idx else 0
    if base == "lif_fwd":
        # GEMM: I = A W over all T, 2 B T K N flop per layer.  Scan: 8.125 B per
        # neuron-step (I f32 in, V f32 out, 1 spike bit; ALIF +4 B for a), plus the
        # first layer's packed input bits (1 bit per (b, t, i))
        n = dict(fwd_groups or []).get(l, 1)
        fl = sum(2.0 * B * T * dims[j] * dims[j + 1] for j in range(l, l + n))
        by = sum((12.125 if alif else 8.125) * B * T * dims[j + 1] for j in range(l, l + n))
        by += B * T * dims[l] / 8.0 if l == 0 else 0.0
        return {"tensor": fl, "hbm": by}
    if base == "wgrad":              # dW = A^T dI, every Linear layer in one launch
        return {"tensor": sum(2.0 * B * T * dims[j] * dims[j + 1] for j in range(len(dims) - 1)),
                "hbm": 0.0}
    if base == "lif_bwd":            # dS GEMM (layers >= 1 get dS from the next layer) + reverse scan
        return {"tensor": 2.0 * B * T * dims[l + 1] * dims[l + 2],
                "hbm": (16.0 if alif else 12.0) * B * T * dims[l + 1]}
    if base == "readout":            # LI fwd 4 B + bwd 4 B per readout element
        return {"tensor": 0.0, "hbm": 8.0 * B * T * C}
    if base == "rlif_fwd":           # recurrent scan: read I, write V (+ spike bits) per neuron-step
        return {"tensor": 0.0, "hbm": 8.125 * B * T * dims[l + 1]}
    if base == "rlif_bwd":           # recurrent reverse scan (+ the per-step rec product, 2 H^2 / sample-step)
        return {"tensor": 2.0 * B * T * dims[l + 1] ** 2, "hbm": 12.0 * B * T * dims[l + 1]}
    if base == "ds":                 # dS GEMM only (RLIF layers)
        return {"tensor": 2.0 * B * T * dims[l + 1] * dims[l + 2], "hbm": 0.0}
    if base in ("adam", "reduce_adam", "peer_adam"):  # Adam: 28 B / param
        return {"tensor": 0.0, "hbm": 28.0 * n_params}
    return {"tensor": 0.0, "hbm": 0.0}


def roofline_of(k: dict, hbm_peak: float, tf_peak: float) -> dict:
    """Both fractions of one launch (burst peaks: a kernel timed alone); the
    binding one is the larger."""
    sec = k["ms"] / 1e3
    out = {}
    if k["work"]["tensor"] > 0:
        a = k["work"]["tensor"] / sec / 1e12
        out["tensor"] = {"achieved": a, "peak": tf_peak, "unit": "TFLOP/s", "frac": a / tf_peak,
                         "work_per_launch": k["work"]["tensor"]}
    if k["work"]["hbm"] > 0:
        a = k["work"]["hbm"] / sec / 1e9
        out["hbm"] = {"achieved": a, "peak": hbm_peak, "unit": "GB/s", "frac": a / hbm_peak,
                      "work_per_launch": k["work"]["hbm"]}
    return out


SPAN_STEPS = 8


def kernel_spans(eng, w: dict, first_slot: int) -> dict:
    """Per-kernel in-graph spans (ms) of the last step of an 8-step graph replayed with
    clock stamps on (debug level 2: the kernels keep their production paths and each
    CTA stores its globaltimer once past its dependency wait, and at its end): span =
    last CTA end - first CTA start (so a kernel launched early by PDL is not charged
    for the time it waits on its predecessor).
    Slots: readout 0, forward launch starting at layer l 1 + l, backward of layer l
    1 + L + l, wgrad (+ the one-rank tail) 1 + 2 L."""
    L = len(w["hidden"])
    try:
        eng.debug(2)
        eng.enqueue_steps(first_slot, SPAN_STEPS)
        eng.sync()
        clk = eng.fetch("clk")
    except Exception:
        return {}
    finally:
        try:
            eng.debug(False)
        except Exception:
            pass
    slots = {"readout": 0, "wgrad": 1 + 2 * L}
    for l in range(L):
        slots[f"lif_fwd[{l}]"] = 1 + l
        slots[f"lif_bwd[{l}]"] = 1 + L + l
    out = {}
    for name, sl in slots.items():
        c = clk[sl]
        v = c[:, 14] > 0
        if v.any():
            out[name] = float(c[v, 15].max() - c[v, 14].min()) / 1e6
    return out


def ncu_traffic(kernel: str):
    """dram bytes per launch for `kernel` from the committed ncu summary, if any."""
    for fn in sorted(os.listdir(os.path.join(ROOT, "profiles")) if os.path.isdir(
            os.path.join(ROOT, "profiles")) else [], reverse=True):
        if fn.endswith("_ncu.json"):
            try:
                d = json.load(open(os.path.join(ROOT, "profiles", fn)))
                if kernel in d.get("dram_bytes_per_launch", {}):
                    return d["dram_bytes_per_launch"][kernel]
            except Exception:
                pass
    return None


# ------------------------------------------------------------ CPU baseline
def _cpu_net(w):
    """The reference network of workload w.  The reference has LIF cells only
    (SPEC.md:373, :382), so an ALIF workload is timed on its LIF stand-in of the
    same shape and surrogate -- labelled in the sample string."""
    from oracle.pyoracle import Net
    return Net(inp=w["inp"], hidden=tuple(w["hidden"]), classes=w["classes"], act=w["act"])


def _cpu_label(w, b):
    cell = {"alif": "LIF stand-in for ALIF (no ALIF in the reference)",
            "rlif": "LIF stand-in for RLIF (no recurrent cell in the reference)"}.get(w.get("cell"), "LIF")
    return (f"{b} examples/step of the workload shape ({w['inp']}-" + "-".join(map(str, w["hidden"])) +
            f"-{w['classes']}, T={w['T']}, {w['act']}, {cell}, init regime)")


def _ref_worker(args):
    which, w, n_examples, steps, warmup, seed, q = args
    from oracle.pyoracle import Lib, State
    lib = Lib(which)
    net = _cpu_net(w)
    x, y = lib.synth_raster(w["classes"], n_examples, w["T"], w["inp"], seed)
    pk = lib.pack_time(x)
    st = State(lib.init(net, lib.key_child(lib.key_from_seed(0), 0)))
    for _ in range(warmup):
        lib.train_step(net, st, pk, w["T"], y)
    t0 = time.perf_counter()
    for _ in range(steps):
        lib.train_step(net, st, pk, w["T"], y)
    q.put((n_examples * steps, time.perf_counter() - t0))


def cpu_reference(w: dict, steps: int, warmup: int, workers: int, per_step_budget_s: float):
    """Reference CPU train_step on `workers` host cores (independent replicas).

    Each step of each worker is a bounded sample of workload w: b examples (b sized
    so the whole run fits the budget) at the workload's network shape and T."""
    from oracle.pyoracle import Lib, State, have_ref
    which = "ref" if have_ref() else "orc"
    kind = "reference" if which == "ref" else "port"
    lib = Lib(which)
    # calibrate the per-example cost on one core
    net = _cpu_net(w)
    x, y = lib.synth_raster(w["classes"], 2, w["T"], w["inp"], 1)
    pk = lib.pack_time(x)
    st = State(lib.init(net, lib.key_child(lib.key_from_seed(0), 0)))
    t0 = time.perf_counter()
    lib.train_step(net, st, pk, w["T"], y)
    per_ex = (time.perf_counter() - t0) / 2
    b = int(max(1, min(w["B"], per_step_budget_s / max(per_ex, 1e-6))))
    ctx = mp.get_context("fork")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ref_worker, args=((which, w, b, steps, warmup, 1 + i, q),))
             for i in range(workers)]
    t0 = time.perf_counter()
    for p in procs:
        p.start()
    res = [q.get() for _ in procs]
    wall = time.perf_counter() - t0
    for p in procs:
        p.join()
    samples = sum(r[0] for r in res)
    slowest = max(r[1] for r in res)
    value = samples / slowest
    return dict(value=value, unit=UNIT, cores=workers, kind=kind,
                sample=f"{workers} x replica train_step on " + _cpu_label(w, b) +
                       f", {steps} timed + {warmup} warm-up steps each", wall_s=wall,
                examples_per_step=b,
                ms_per_step=1e3 * slowest / max(steps, 1))


def host_cpu() -> dict:
    model = None
    try:
        for ln in subprocess.run(["lscpu"], capture_output=True, text=True).stdout.splitlines():
            if ln.startswith("Model name:"):
                model = ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return {"nproc": os.cpu_count(), "model": model}


def cpu_baseline_single(w: dict, seconds: float = 12.0, params=None, regime="init"):
    """Bounded single-core sample for our arm's cpu_baseline key.  params: the
    regime's parameters (None = the reference init, seed 0).  The reference skips
    zero inputs (ops.hpp:168, :216), so a spiking (warm) network costs it more."""
    from oracle.pyoracle import Lib, State, have_ref
    which = "ref" if have_ref() else "orc"
    lib = Lib(which)
    net = _cpu_net(w)
    b = 32
    x, y = lib.synth_raster(w["classes"], b, w["T"], w["inp"], 1)
    pk = lib.pack_time(x)
    st = State(lib.init(net, lib.key_child(lib.key_from_seed(0), 0)) if params is None
               else np.array(params, np.float32))
    lib.train_step(net, st, pk, w["T"], y)
    n, t0 = 0, time.perf_counter()
    while True:
        lib.train_step(net, st, pk, w["T"], y)
        n += 1
        el = time.perf_counter() - t0
        if el >= seconds or n >= 200:
            break
    return dict(value=b * n / el, unit=UNIT, cores=1,
                kind="reference" if which == "ref" else "port",
                sample=f"{n} train_steps of " + _cpu_label(w, b).replace("init regime", f"{regime} regime")
                       + f" on 1 host core, {el:.1f} s")


# ------------------------------------------------------------------ main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c1", choices=sorted(WORKLOADS))
    ap.add_argument("--e2e-steps", type=int, default=256)
    ap.add_argument("--profile-steps", type=int, default=20)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--gemm-planes", type=int, default=3, choices=[1, 2, 3],
                    help="bf16 operand planes per real GEMM operand: 3 = the fp32 path (default), "
                         "2 = fast bf16x2 mode, 1 = bf16 (separate lines, own tolerances)")
    args = ap.parse_args()
    warmup = max(3, args.warmup)
    w = WORKLOADS[args.config]

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        # started bare with --gpus N: launch the N ranks ourselves (one process per GPU)
        import socket
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
               f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if w.get("global_batch"):
        if w["B"] % world:
            raise SystemExit(f"{args.config}: global batch {w['B']} not divisible by {world} ranks")
        w = dict(w, B=w["B"] // world)
    scaling = "strong" if w.get("global_batch") else "weak"
    config = {"workload": f"{args.config}: {w['desc']}", "global_batch": w["B"] * world,
              "seq_len": w["T"], "network": f"{w['inp']}-" + "-".join(map(str, w["hidden"])) +
              f"-{w['classes']}", "parallelism": f"dp{world}",
              "l2": f"HBM-resident dataset of {w['n_data']} examples "
                    f"({w['n_data'] * (w['T'] // 8) * ((w['inp'] + 63) // 64 * 64) / 1e6:.0f} MB "
                    f"staged) > 126 MB L2; fresh permuted rows every step, no L2 flush"}
    if world > 1:
        config["dp_tail"] = os.environ.get("SNN_DP_TAIL", "peer")  # gradient exchange (parallel.py)
    dtype = {3: "f32", 2: "bf16x2", 1: "bf16"}[args.gemm_planes]
    if args.gemm_planes != 3:
        config["gemm_mode"] = (f"{dtype}: {args.gemm_planes} bf16 plane(s) per real GEMM operand "
                               "(fast mode; tolerance in DESIGN.md)")

    if args.impl == "reference":
        if rank != 0:
            return
        workers = max(1, os.cpu_count() or 1)
        budget = 150.0 / (args.steps + warmup)
        r = cpu_reference(w, args.steps, warmup, workers, budget)
        line = {"impl": "reference", "metric": METRIC, "value": r["value"], "unit": UNIT,
                "n_gpus": args.gpus, "steps": args.steps, "warmup": warmup,
                "ms_per_step": r["ms_per_step"], "higher_is_better": True, "scaling": scaling,
                "vs_baseline": None, "dtype": "f32", "data": "synthetic (synth_raster seed 1)",
                "config": config,
                "cpu_baseline": {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")},
                "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    import torch
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2402_18994_b200 import Engine, TrainConfig, shd_spec
    spec = shd_spec(hidden=w["hidden"], classes=w["classes"], inp=w["inp"], act=w["act"],
                    cell=w.get("cell", "lif"))
    B = w["B"]
    eng = Engine(spec, TrainConfig(batch_size=B, seed=0, lr=1e-3, gemm_planes=args.gemm_planes), w["T"],
                 device=local)
    if world > 1:
        # gradient exchange: peer-memory tail (default) or NCCL (SNN_DP_TAIL=nccl)
        from paper_2402_18994_b200.parallel import setup_data_parallel
        tail = os.environ.get("SNN_DP_TAIL", "peer")
        if tail == "peer":
            # the peer tail maps every rank's buffer over NVLink; every rank takes the same
            # decision from the (symmetric) peer-access matrix of the node's GPUs
            # (multi-node jobs always take NCCL: IPC handles do not cross nodes)
            n_local = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
            if n_local != world or not all(torch.cuda.can_device_access_peer(i, j)
                                           for i in range(n_local) for j in range(n_local) if i != j):
                tail = "nccl"
        config["dp_tail"] = tail
        setup_data_parallel(eng, rank, world, dist, tail)
    n_data = w["n_data"]
    eng.synth_dataset(n_data, seed=1)
    # schedule: the reference epoch shuffle, this rank's contiguous slice of each global batch
    gb = B * world
    per_epoch = n_data // gb
    total = warmup + args.steps + SPAN_STEPS  # + the clock-stamped replay (kernel_spans)
    rows = np.empty((total, B), np.uint32)
    e = 0
    s = 0
    while s < total:
        perm = eng.epoch_permutation(e, n_data)
        for bi in range(per_epoch):
            if s >= total:
                break
            rows[s] = perm[bi * gb + rank * B: bi * gb + (rank + 1) * B]
            s += 1
        e += 1
    eng.upload_schedule(rows.reshape(-1))
    stream = torch.cuda.ExternalStream(eng.stream)

    def barrier():
        if dist is not None:
            dist.barrier()

    eng.enqueue_steps(0, warmup)
    eng.sync()
    barrier()
    torch.cuda.synchronize()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        # hold the stream with a ~25 ms device spin so the start event fires only after
        # the whole timed region is enqueued: host-side stalls (GIL hand-off to the
        # sampler thread) stay out of the device-timed region
        with torch.cuda.stream(stream):
            torch.cuda._sleep(50_000_000)
        t_start.record(stream)
        eng.enqueue_steps(warmup, args.steps)
        clocks.mark()                      # the enqueued steps are running now
        t_end.record(stream)
        eng.sync()
        torch.cuda.synchronize()
    barrier()
    ms = t_start.elapsed_time(t_end)
    if dist is not None:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    loss, acc = eng.read_result()
    ranks = None
    if dist is not None:
        # proof of participation: every rank's device, step counter and replica checksum
        # (the data-parallel replicas must be bit-identical)
        p = eng.get_params()
        mine = {"rank": rank, "device": torch.cuda.get_device_name(local), "local_rank": local,
                "steps_done": int(eng.get_opt_state()[2]),
                "param_checksum": float(np.float64(p.astype(np.float64).sum()))}
        allr = [None] * world
        dist.all_gather_object(allr, mine)
        ranks = {"world": world, "tail": config.get("dp_tail"), "per_rank": allr,
                 "replicas_identical": len({r["param_checksum"] for r in allr}) == 1}
    ms_per_step = ms / args.steps
    value = gb * args.steps / (ms / 1e3)

    # --- end to end through the public API with HOST buffers (pinned H2D in, loss/acc out)
    packed_host, labels_host = eng.read_dataset(0, min(n_data, 4 * B))
    # the caller's host batches live in pinned (page-locked) memory, as the e2e
    # protocol states; the engine DMAs them directly (no staging copy)
    pinned = torch.empty(packed_host.shape, dtype=torch.uint8, pin_memory=True)
    pinned.numpy()[...] = packed_host
    packed_host = pinned.numpy()
    nb = packed_host.shape[0] // B
    for i in range(3):
        eng.train_step_packed(packed_host[(i % nb) * B:(i % nb + 1) * B],
                              labels_host[(i % nb) * B:(i % nb + 1) * B])
    barrier()
    t0 = time.perf_counter()
    for i in range(args.e2e_steps):
        k = i % nb
        eng.train_step_packed(packed_host[k * B:(k + 1) * B], labels_host[k * B:(k + 1) * B])
    sync_s = time.perf_counter() - t0
    # the train() form over host batches: snn_train_steps_packed uploads batch k+1 while
    # step k runs; every step's batch is DMA'd from pinned memory and every StepResult
    # read back inside the timed region (calls of E2E_CHUNK steps)
    chunk = max(2, min(E2E_CHUNK, args.e2e_steps, (64 * 256) // B))  # bounds the pinned batch set
    seq = np.arange(chunk) % nb
    stream_batches = torch.empty((chunk, B) + tuple(packed_host.shape[1:]), dtype=torch.uint8,
                                 pin_memory=True).numpy()
    for c, k in enumerate(seq):
        stream_batches[c] = packed_host[k * B:(k + 1) * B]
    stream_labels = np.stack([labels_host[k * B:(k + 1) * B] for k in seq])
    eng.train_steps_packed(stream_batches, stream_labels)  # warm: builds the host-batch graph
    barrier()
    calls = max(1, args.e2e_steps // chunk)
    t0 = time.perf_counter()
    for _ in range(calls):
        eng.train_steps_packed(stream_batches, stream_labels)
    e2e_s = time.perf_counter() - t0
    if dist is not None:
        t = torch.tensor([e2e_s, sync_s], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s, sync_s = float(t[0].item()), float(t[1].item())
    e2e_value = gb * calls * chunk / e2e_s
    sync_value = gb * args.e2e_steps / sync_s
    h2d = int(packed_host[:B].nbytes + 8 * B)
    d2h = 4 + 8

    # --- per-kernel device times (graph with event nodes) -> roofline of the dominant kernel
    prof = eng.profile(args.profile_steps)
    spans = kernel_spans(eng, w, warmup + args.steps)
    hbm_peak, tf_peak, peak_src = peaks()
    kernels = []
    for name, kms in prof:
        # in-graph span (first CTA start .. last CTA end, globaltimer) when stamped;
        # else the event-graph time (which adds a launch and a drain per kernel)
        k = {"name": name, "ms": spans.get(name, kms), "ms_event_graph": kms,
             "timing": "in-graph span" if name in spans else "event graph",
             "work": algorithmic(name, w, eng.n_params, eng.forward_launches, B)}
        k["roofline"] = roofline_of(k, hbm_peak, tf_peak)
        kernels.append(k)
    dom = max(kernels, key=lambda k: k["ms"])
    both = dom["roofline"]
    bound = max(both, key=lambda b: both[b]["frac"])
    roofline = {"kernel": dom["name"], "bound": bound, "achieved": both[bound]["achieved"],
                "peak": both[bound]["peak"], "unit": both[bound]["unit"],
                "frac": both[bound]["frac"], "traffic": ncu_traffic(dom["name"]),
                "peak_source": peak_src, "work_per_launch": both[bound]["work_per_launch"],
                "share_of_step": dom["ms"] / sum(k["ms"] for k in kernels),
                "fractions": {b: round(v["frac"], 4) for b, v in both.items()}}

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": dtype,
            "data": "synthetic (synth_raster seed 1, generated in HBM bit-identical to the "
                    "reference), random-init weights (reference init, seed 0)",
            "config": config, "clocks": clocks.summary(),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h,
                    "path": f"snn_train_steps_packed (train() over host batches, {chunk} per call): "
                            "every step's pinned host batch (reference layout) -> H2D on a copy stream "
                            "into the step's device slot (used in place when ceil(T/8) = T_pad/8 and "
                            "input % 4 == 0, else re-laid out there), overlapped with the previous "
                            "step's graph; every step's loss/acc written by its own tail into mapped "
                            "host memory (12 B D2H); one host sync per call",
                    "per_step_call": {"value": sync_value, "unit": UNIT,
                                      "path": "snn_train_step_packed: H2D, step graph, loss/acc "
                                              "into mapped host memory, host sync every step"}},
            "gpu_launches": eng.launches_per_step * args.steps,
            **({"ranks": ranks} if ranks is not None else {}),
            "roofline": roofline,
            "kernels": [{"name": k["name"], "ms": round(k["ms"], 5), "timing": k["timing"],
                         "ms_event_graph": round(k["ms_event_graph"], 5),
                         **{b: round(v["frac"], 4) for b, v in k["roofline"].items()}}
                        for k in kernels],
            "final_loss": loss, "final_acc": acc}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_single(w)
        line["cpu_baseline"]["host"] = host_cpu()
        gold = os.path.join(ROOT, "tests", "golden", "c1.npz")
        if args.config == "c1" and os.path.exists(gold):
            # warm regime: the reference's own C1 checkpoint after 3 epochs
            warm = cpu_baseline_single(w, params=np.load(gold)["warm_params"], regime="warm")
            line["cpu_baseline"]["warm"] = {k: warm[k] for k in ("value", "unit", "cores", "sample")}
    if rank == 0:
        print(json.dumps(line))
    eng.close()
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
