"""ctypes binding for the CPU checker libraries -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg import
this module.  It loads either the plain-C restatement (``oracle/liboracle.so``,
prefix ``orc_``) or the reference driver (``oracle/_ref/libspiketrain_ref.so``,
prefix ``ref_``); both export the interface in ``spiketrain_oracle.h``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libspiketrain_ref.so")

# "sigmoid" is DECLARED (not in the reference catalogue; spiketrain_oracle.h):
# custom(heaviside, d/dx sigmoid(kx)), k = 25 by default
ACTS = {"custom": 0, "superspike": 1, "triangular": 2, "arctan": 3, "boxcar": 4,
        "sigmoid": 5}
DEFAULT_SLOPE = {"custom": (0.0, 0.0), "superspike": (25.0, 0.0),
                 "triangular": (0.5, 0.0), "arctan": (2.0, 0.0),
                 "boxcar": (2.0, 0.5), "sigmoid": (25.0, 0.0)}


class _Net(C.Structure):
    _fields_ = [("in_", C.c_int), ("n_hidden", C.c_int),
                ("hidden", C.c_int * 8), ("classes", C.c_int),
                ("bias", C.c_int), ("threshold", C.c_float), ("act", C.c_int),
                ("slope", C.c_float), ("aux", C.c_float), ("unroll", C.c_int),
                ("beta_mode", C.c_int * 9), ("fixed_beta", C.c_float * 9),
                ("monitor", C.c_int * 8), ("cell", C.c_int * 8), ("readout_lif", C.c_int)]

# hidden cell kinds: "lif" (neuron.hpp:127-136) | "alif" | "rlif" (declared
# restatements, spiketrain_oracle.h -- not in the reference)
CELLS = {"lif": 0, "alif": 1, "rlif": 2}

BETA_MODES = {"per_neuron": 0, "scalar": 1, "fixed": 2}


class _Opts(C.Structure):
    _fields_ = [("optimizer", C.c_int), ("momentum", C.c_float), ("loss", C.c_int),
                ("rate_hi", C.c_float), ("rate_lo", C.c_float), ("max_shift", C.c_int),
                ("n_shift_axes", C.c_int), ("shift_axes", C.c_int * 4),
                ("f_min", C.c_float), ("f_max", C.c_float), ("lambda_low", C.c_float),
                ("lambda_high", C.c_float)]


@dataclass
class Opts:
    """TrainConfig options on the step (optimize.hpp:113-131): optimizer 'adam' |
    'sgd' (+ momentum), loss 'ce' (integral CE) | 'rate_mse' (+ rate targets)."""
    optimizer: str = "adam"
    momentum: float = 0.9
    loss: str = "ce"
    rate_hi: float = 0.9
    rate_lo: float = 0.1
    max_shift: int = 0          # shift_augment (epoch loop only)
    shift_axes: tuple = ()
    f_min: float = 0.0          # activity regularizer (both lambdas 0 = off)
    f_max: float = 1.0
    lambda_low: float = 0.0
    lambda_high: float = 0.0

    def c(self) -> _Opts:
        o = _Opts(1 if self.optimizer == "sgd" else 0, self.momentum,
                  1 if self.loss == "rate_mse" else 0, self.rate_hi, self.rate_lo,
                  self.max_shift, len(self.shift_axes))
        o.f_min, o.f_max = self.f_min, self.f_max
        o.lambda_low, o.lambda_high = self.lambda_low, self.lambda_high
        for i, a in enumerate(self.shift_axes):
            o.shift_axes[i] = a
        return o


@dataclass
class Net:
    """Linear->LIF stack + Linear->LI readout (network.hpp:23-60)."""
    inp: int = 700
    hidden: tuple = (128, 128)
    classes: int = 20
    bias: bool = False
    threshold: float = 1.0
    act: str = "arctan"
    slope: float | None = None
    aux: float | None = None
    unroll: int = 32
    # BetaMode per cell (hidden LIF layers, then the LI readout): "per_neuron" |
    # "scalar" (LearnableScalar) | "fixed"; fixed_beta per cell (default 0.5)
    beta_mode: tuple = ()
    fixed_beta: tuple = ()
    # hidden LIF layers followed by a MonitorLayer (indices into hidden)
    monitor: tuple = ()
    # cell kind per hidden layer ("lif" | "alif"); missing entries are "lif"
    cell: tuple = ()
    # readout cell: "li" (default) or "lif" (network.hpp:153-155, :396)
    readout: str = "li"

    def c(self) -> _Net:
        s, a = DEFAULT_SLOPE[self.act]
        n = _Net()
        n.in_ = self.inp
        n.n_hidden = len(self.hidden)
        for i, h in enumerate(self.hidden):
            n.hidden[i] = h
        n.classes = self.classes
        n.bias = int(self.bias)
        n.threshold = self.threshold
        n.act = ACTS[self.act]
        n.slope = s if self.slope is None else self.slope
        n.aux = a if self.aux is None else self.aux
        n.unroll = self.unroll
        for i in range(len(self.hidden) + 1):
            n.beta_mode[i] = BETA_MODES[self.beta_mode[i]] if i < len(self.beta_mode) else 0
            n.fixed_beta[i] = self.fixed_beta[i] if i < len(self.fixed_beta) else 0.5
        for i in self.monitor:
            n.monitor[i] = 1
        for i, c in enumerate(self.cell):
            n.cell[i] = CELLS[c]
        n.readout_lif = 1 if self.readout == "lif" else 0
        return n


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _ptr(a, t):
    return a.ctypes.data_as(C.POINTER(t)) if a is not None else None


class Lib:
    """One of the two checker libraries."""

    def __init__(self, which: str = "orc"):
        path = ORACLE_SO if which == "orc" else REF_SO
        if not os.path.exists(path):
            build()
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = C.CDLL(path)
        self.p = which + "_"
        L = self.lib
        f = lambda n: getattr(L, self.p + n)  # noqa: E731
        f("key_from_seed").restype = C.c_uint64
        f("key_from_seed").argtypes = [C.c_uint64]
        f("key_child").restype = C.c_uint64
        f("key_child").argtypes = [C.c_uint64, C.c_uint64]
        f("key_bits").restype = C.c_uint64
        f("key_bits").argtypes = [C.c_uint64, C.c_uint64]
        f("uniform01").restype = C.c_double
        f("uniform01").argtypes = [C.c_uint64, C.c_uint64]
        f("param_count").restype = C.c_size_t
        f("entry_count").restype = C.c_int
        f("forward_backward").restype = C.c_int
        f("forward_backward_ex").restype = C.c_int
        f("train_step").restype = C.c_int
        f("train_step_ex").restype = C.c_int
        f("train_epochs").restype = C.c_int
        f("train_epochs_ex").restype = C.c_int
        self._f = f
        if hasattr(L, self.p + "forward_backward_forced"):
            f("forward_backward_forced").restype = C.c_int

    def set_threads(self, n: int) -> None:
        """Host threads for big shapes (the C restatement only; bit-identical for any n)."""
        fn = getattr(self.lib, self.p + "set_threads", None)
        if fn is not None:
            fn(C.c_int(int(n)))

    def surrogate(self, act: str, x, slope=None, aux=None):
        """g(x) elementwise; for the ref library through the reference's own tape."""
        s, a = DEFAULT_SLOPE[act]
        x = np.ascontiguousarray(x, np.float32)
        out = np.zeros_like(x)
        self._f("surrogate")(C.c_int(ACTS[act]), C.c_float(s if slope is None else slope),
                             C.c_float(a if aux is None else aux), _ptr(x, C.c_float),
                             C.c_size_t(x.size), _ptr(out, C.c_float))
        return out

    # ---- rng -----------------------------------------------------------
    def key_from_seed(self, s):
        return self._f("key_from_seed")(s)

    def key_child(self, k, i):
        return self._f("key_child")(k, i)

    def key_bits(self, k, c):
        return self._f("key_bits")(k, c)

    def uniform01(self, k, c):
        return self._f("uniform01")(k, c)

    def permutation(self, key, n):
        out = np.zeros(n, np.uint64)
        self._f("permutation")(C.c_uint64(key), C.c_size_t(n), _ptr(out, C.c_uint64))
        return out

    def truncated_normal(self, key, n, mean, sd):
        out = np.zeros(n, np.float32)
        self._f("truncated_normal")(C.c_uint64(key), C.c_size_t(n), C.c_float(mean),
                                    C.c_float(sd), _ptr(out, C.c_float))
        return out

    # ---- data ----------------------------------------------------------
    def synth_raster(self, classes, n, t, f, seed):
        x = np.zeros((n, t, f), np.uint8)
        y = np.zeros(n, np.int64)
        self._f("synth_raster")(C.c_size_t(classes), C.c_size_t(n), C.c_size_t(t),
                                C.c_size_t(f), C.c_uint64(seed), _ptr(x, C.c_uint8),
                                _ptr(y, C.c_int64))
        return x, y

    def pack_time(self, x):
        n, t, f = x.shape
        x = np.ascontiguousarray(x, np.uint8)
        out = np.zeros((n, (t + 7) // 8, f), np.uint8)
        self._f("pack_time")(_ptr(x, C.c_uint8), C.c_size_t(n), C.c_size_t(t),
                             C.c_size_t(f), _ptr(out, C.c_uint8))
        return out

    def unpack_time(self, packed, t):
        n, _, f = packed.shape
        packed = np.ascontiguousarray(packed, np.uint8)
        out = np.zeros((n, t, f), np.uint8)
        self._f("unpack_time")(_ptr(packed, C.c_uint8), C.c_size_t(n), C.c_size_t(t),
                               C.c_size_t(f), _ptr(out, C.c_uint8))
        return out

    # ---- network -------------------------------------------------------
    def param_count(self, net: Net) -> int:
        n = net.c()
        return self._f("param_count")(C.byref(n))

    def entries(self, net: Net):
        n = net.c()
        cnt = self._f("entry_count")(C.byref(n))
        offs = (C.c_size_t * cnt)()
        sizes = (C.c_size_t * cnt)()
        names = ((C.c_char * 16) * cnt)()
        self._f("entry_layout")(C.byref(n), offs, sizes, names)
        return [(names[i].value.decode(), offs[i], sizes[i]) for i in range(cnt)]

    def init(self, net: Net, key: int):
        n = net.c()
        p = np.zeros(self.param_count(net), np.float32)
        self._f("init")(C.byref(n), C.c_uint64(key), _ptr(p, C.c_float))
        return p

    def forward_backward(self, net: Net, params, packed, t, targets,
                         want_grads=True, want_spikes=False, want_trace=False,
                         want_v=False, opts: "Opts | None" = None, forced=None):
        """forced: optional list of per-layer u8 rasters [B,T,H] (teacher forcing,
        orc_forward_backward_forced; the C restatement only)."""
        n = net.c()
        oc = opts.c() if opts is not None else None
        B = packed.shape[0]
        params = np.ascontiguousarray(params, np.float32)
        packed = np.ascontiguousarray(packed, np.uint8)
        targets = np.ascontiguousarray(targets, np.int64)
        loss = C.c_float()
        acc = C.c_double()
        grads = np.zeros_like(params) if want_grads else None
        nsp = B * t * sum(net.hidden)
        spikes = np.zeros(nsp, np.uint8) if want_spikes else None
        vtr = np.zeros(nsp, np.float32) if want_v else None
        trace = np.zeros((B, t, net.classes), np.float32) if want_trace else None
        if forced is None:
            rc = self._f("forward_backward_ex")(
                C.byref(n), C.byref(oc) if oc is not None else None, _ptr(params, C.c_float),
                _ptr(packed, C.c_uint8),
                C.c_size_t(B), C.c_size_t(t), _ptr(targets, C.c_int64), C.byref(loss),
                C.byref(acc), _ptr(grads, C.c_float), _ptr(spikes, C.c_uint8),
                _ptr(vtr, C.c_float), _ptr(trace, C.c_float))
        else:
            fr = np.ascontiguousarray(np.concatenate(
                [np.asarray(f, np.uint8).reshape(-1) for f in forced]))
            assert fr.size == nsp, "forced rasters must cover every hidden layer"
            rc = self._f("forward_backward_forced")(
                C.byref(n), C.byref(oc) if oc is not None else None, _ptr(params, C.c_float),
                _ptr(packed, C.c_uint8), C.c_size_t(B), C.c_size_t(t),
                _ptr(targets, C.c_int64), _ptr(fr, C.c_uint8), C.byref(loss),
                C.byref(acc), _ptr(grads, C.c_float), _ptr(spikes, C.c_uint8),
                _ptr(vtr, C.c_float), _ptr(trace, C.c_float))
        if rc != 0:
            raise ValueError(f"forward_backward failed rc={rc}")
        out = {"loss": loss.value, "acc": acc.value}
        if want_grads:
            out["grads"] = grads
        if want_spikes:
            sp, off = [], 0
            for h in net.hidden:
                sp.append(spikes[off:off + B * t * h].reshape(B, t, h))
                off += B * t * h
            out["spikes"] = sp
        if want_v:
            vs, off = [], 0
            for h in net.hidden:
                vs.append(vtr[off:off + B * t * h].reshape(B, t, h))
                off += B * t * h
            out["v"] = vs
        if want_trace:
            out["trace"] = trace
        return out

    def eval_accuracy(self, net: Net, params, packed, y, t, batch) -> float:
        """cmd_eval (commands.hpp:144-169): batches of `batch` rows (the last one
        short), integral_accuracy per batch (objective.hpp:118-134, computed by the
        oracle in the reference order) accumulated as correct += acc * nb, / n."""
        n = packed.shape[0]
        correct = 0.0
        for lo in range(0, n, batch):
            hi = min(n, lo + batch)
            r = self.forward_backward(net, params, packed[lo:hi], t, y[lo:hi], want_grads=False)
            correct += r["acc"] * float(hi - lo)
        return correct / float(n)

    def write_container(self, path: str, packed, original_t: int, labels) -> None:
        """Reference write_container (data.hpp:272-293); ref library only."""
        packed = np.ascontiguousarray(packed, np.uint8)
        shape = np.array(packed.shape, np.uint64)
        f = self._f("write_container")
        f.restype = C.c_int
        rc = f(path.encode(), _ptr(packed, C.c_uint8), _ptr(shape, C.c_uint64), C.c_int(packed.ndim),
               C.c_uint32(original_t), _ptr(np.ascontiguousarray(labels, np.int64), C.c_int64))
        if rc != 0:
            raise ValueError("write_container failed")

    def read_container(self, path: str, cap: int, n_cap: int):
        """Reference read_container (data.hpp:295-339); ref library only."""
        packed = np.zeros(cap, np.uint8)
        labels = np.zeros(n_cap, np.int64)
        t, n = C.c_uint32(), C.c_uint64()
        f = self._f("read_container")
        f.restype = C.c_int
        rc = f(path.encode(), _ptr(packed, C.c_uint8), C.c_size_t(cap), _ptr(labels, C.c_int64),
               C.c_size_t(n_cap), C.byref(t), C.byref(n))
        if rc != 0:
            raise ValueError(f"read_container failed rc={rc}")
        return packed, labels[:n.value], t.value

    def write_checkpoint(self, net: Net, params, m, v, step: int, optimizer: str,
                         config_text: str, path: str) -> None:
        """Reference write_checkpoint (optimize.hpp:334-366); ref library only."""
        n = net.c()
        f = self._f("write_checkpoint")
        f.restype = C.c_int
        rc = f(C.byref(n), _ptr(np.ascontiguousarray(params, np.float32), C.c_float),
               _ptr(np.ascontiguousarray(m, np.float32), C.c_float),
               _ptr(np.ascontiguousarray(v, np.float32), C.c_float), C.c_uint64(step),
               C.c_int(1 if optimizer == "sgd" else 0), config_text.encode(), path.encode())
        if rc != 0:
            raise ValueError("write_checkpoint failed")

    def adam(self, p, g, m, v, step, lr=1e-3, b1=0.9, b2=0.999, eps=1e-8):
        st = C.c_uint64(step)
        self._f("adam")(_ptr(p, C.c_float), _ptr(g, C.c_float), _ptr(m, C.c_float),
                        _ptr(v, C.c_float), C.c_size_t(p.size), C.byref(st),
                        C.c_float(lr), C.c_float(b1), C.c_float(b2), C.c_float(eps))
        return st.value

    def train_step(self, net: Net, state: "State", packed, t, targets, lr=1e-3,
                   opts: "Opts | None" = None):
        n = net.c()
        oc = opts.c() if opts is not None else None
        packed = np.ascontiguousarray(packed, np.uint8)
        targets = np.ascontiguousarray(targets, np.int64)
        loss = C.c_float()
        acc = C.c_double()
        st = C.c_uint64(state.step)
        rc = self._f("train_step_ex")(
            C.byref(n), C.byref(oc) if oc is not None else None,
            _ptr(state.params, C.c_float), _ptr(state.m, C.c_float),
            _ptr(state.v, C.c_float), C.byref(st), _ptr(packed, C.c_uint8),
            C.c_size_t(packed.shape[0]), C.c_size_t(t), _ptr(targets, C.c_int64),
            C.c_float(lr), C.byref(loss), C.byref(acc))
        if rc != 0:
            raise ValueError("train_step failed")
        state.step = st.value
        return loss.value, acc.value

    def train_epochs(self, net: Net, state: "State", packed, y, t, batch, epochs,
                     seed, lr=1e-3, opts: "Opts" = None):
        n = net.c()
        packed = np.ascontiguousarray(packed, np.uint8)
        y = np.ascontiguousarray(y, np.int64)
        metrics = np.zeros((epochs, 2), np.float64)
        st = C.c_uint64(state.step)
        o = (opts or Opts()).c()
        rc = self._f("train_epochs_ex")(
            C.byref(n), C.byref(o), _ptr(state.params, C.c_float), _ptr(state.m, C.c_float),
            _ptr(state.v, C.c_float), C.byref(st), _ptr(packed, C.c_uint8),
            _ptr(y, C.c_int64), C.c_size_t(packed.shape[0]), C.c_size_t(t),
            C.c_size_t(batch), C.c_size_t(epochs), C.c_uint64(seed), C.c_float(lr),
            _ptr(metrics, C.c_double))
        if rc != 0:
            raise ValueError("train_epochs failed")
        state.step = st.value
        return metrics


@dataclass
class State:
    params: np.ndarray
    m: np.ndarray = field(default=None)
    v: np.ndarray = field(default=None)
    step: int = 0

    def __post_init__(self):
        self.params = np.ascontiguousarray(self.params, np.float32)
        if self.m is None:
            self.m = np.zeros_like(self.params)
        if self.v is None:
            self.v = np.zeros_like(self.params)

    def copy(self) -> "State":
        return State(self.params.copy(), self.m.copy(), self.v.copy(), self.step)


def have_ref() -> bool:
    return os.path.exists(REF_SO)
