"""Python mirror of the reference's training-step API over the engine's C ABI.

Names follow spiketrain (network.hpp, optimize.hpp, surrogate.hpp, errors.hpp):
NetworkSpec / LinearLayer / LIFLayer / LILayer / ActivationDesc / TrainConfig,
train_step, train; errors are raised as the reference's exception classes.
Every call goes through include/snn_engine.h into libsnn_b200.so (sm_100a).
There is no CPU fallback: without the library or a B200 the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from .build import LIB, build, needs_build

# ----------------------------------------------------------------- errors
class Error(RuntimeError):
    """spiketrain::Error (errors.hpp:9-11)."""


class ShapeError(Error): ...
class ArgumentError(Error): ...
class ContractError(Error): ...
class StateError(Error): ...
class FormatError(Error): ...
class IoError(Error): ...
class SpecError(Error): ...
class ConfigError(Error): ...
class UnsupportedError(Error): ...
class DeviceError(Error):
    """No usable B200 / CUDA failure (the engine never falls back to the CPU)."""


_STATUS = {1: ShapeError, 2: ArgumentError, 3: ContractError, 4: StateError, 5: FormatError,
           6: IoError, 7: SpecError, 8: ConfigError, 9: UnsupportedError, 10: DeviceError}

# ------------------------------------------------------------- spec types
# "sigmoid" is DECLARED (not in the reference catalogue): the
# custom(heaviside, k s (1 - s)) backward of oracle/spiketrain_oracle.h
ACTIVATIONS = {"custom": 0, "superspike": 1, "triangular": 2, "arctan": 3, "boxcar": 4,
               "sigmoid": 5}


@dataclass
class ActivationDesc:
    """surrogate.hpp:134-138; defaults per default_activation_desc (:150-157)."""
    name: str = "superspike"
    slope: float = 25.0
    aux: float = 0.0


def default_activation_desc(name: str) -> ActivationDesc:
    table = {"custom": (0.0, 0.0), "superspike": (25.0, 0.0), "triangular": (0.5, 0.0),
             "arctan": (2.0, 0.0), "boxcar": (2.0, 0.5), "sigmoid": (25.0, 0.0)}
    if name not in table:
        raise ArgumentError(f"unknown activation: {name}")
    return ActivationDesc(name, *table[name])


@dataclass
class LinearLayer:
    out: int
    bias: bool = True


@dataclass
class LIFLayer:
    activation: ActivationDesc = field(default_factory=ActivationDesc)
    threshold: float = 1.0
    beta_mode: str = "per_neuron"   # BetaMode: "per_neuron" | "scalar" | "fixed" (neuron.hpp:24)
    fixed_beta: float = 0.5


@dataclass
class ALIFLayer(LIFLayer):
    """Adaptive-threshold LIF -- a DECLARED cell, not in the reference (SPEC.md:373,
    :382): threshold theta + a, reset by it, a' = a*clip01(gamma) + (1-clip01(gamma))*s,
    with a per-neuron "l{id}.gamma" entry after "l{id}.beta" (Spyx's ALIF in the
    reference's LIF op order; checker: oracle/spiketrain_oracle.h).  gamma is always
    per neuron and trainable; beta_mode applies to beta."""


@dataclass
class RLIFLayer(LIFLayer):
    """Recurrent LIF -- a DECLARED cell, not in the reference (feed-forward only,
    network.hpp:16): fb_j = sum_i s_i rec[i][j] over the step's spiking
    neurons, v' = (((v*bc) + I) + fb) - s*theta, with an "l{id}.rec" [H][H] entry after
    "l{id}.beta" (Spyx's RLIF in the reference's LIF op order; checker:
    oracle/spiketrain_oracle.h).  Width <= 1024."""


@dataclass
class LILayer:
    beta_mode: str = "per_neuron"
    fixed_beta: float = 0.5


@dataclass
class MonitorLayer:
    """Spike counts of the LIF layer before it (network.hpp:57); feeds the activity
    regularizer and ApplyResult.monitors.  Takes a normalised layer id."""


@dataclass
class NetworkSpec:
    input_shape: Sequence[int]
    layers: list


@dataclass
class TrainConfig:
    """optimize.hpp:116-133 (the fields the training step consumes)."""
    epochs: int = 100
    batch_size: int = 64
    lr: float = 1e-3
    seed: int = 0
    unroll: int = 32
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    optimizer: str = "adam"              # OptimizerKind: "adam" | "sgd" (optimize.hpp:22)
    momentum: float = 0.9                # SGD only
    loss: str = "integral_crossentropy"  # LossKind: | "spike_rate_mse" (optimize.hpp:23)
    rate_hi: float = 0.9                 # rate-MSE targets
    rate_lo: float = 0.1
    max_shift: int = 0                   # shift augmentation on packed batches
    shift_axes: tuple = ()               # feature axis only (2 or -1); 0 / 1 rejected
    f_min: float = 0.0                   # activity regularizer; zero lambdas disable it
    f_max: float = 1.0
    lambda_low: float = 0.0
    lambda_high: float = 0.0
    gemm_planes: int = 3                 # engine option (not in the reference): 3 = fp32 path,
                                         # 2 = fast bf16x2 planes, 1 = bf16 (snn_engine.h)


ABI_VERSION = 8  # SNN_ABI_VERSION in include/snn_engine.h


class _NetDesc(C.Structure):
    _fields_ = [("input", C.c_int32), ("n_hidden", C.c_int32), ("hidden", C.c_int32 * 8),
                ("classes", C.c_int32), ("bias", C.c_int32), ("threshold", C.c_float),
                ("activation", C.c_int32), ("slope", C.c_float), ("aux", C.c_float),
                ("beta_mode", C.c_int32 * 9), ("fixed_beta", C.c_float * 9),
                ("monitor", C.c_int32 * 8), ("cell", C.c_int32 * 8), ("readout_lif", C.c_int32)]


BETA_MODES = {"per_neuron": 0, "scalar": 1, "fixed": 2}


class _TrainCfg(C.Structure):
    _fields_ = [("batch_size", C.c_int32), ("time_steps", C.c_int32), ("lr", C.c_float),
                ("beta1", C.c_float), ("beta2", C.c_float), ("eps", C.c_float),
                ("seed", C.c_uint64), ("unroll", C.c_int32), ("optimizer", C.c_int32),
                ("momentum", C.c_float), ("loss", C.c_int32), ("rate_hi", C.c_float),
                ("rate_lo", C.c_float), ("max_shift", C.c_int32), ("n_shift_axes", C.c_int32),
                ("shift_axes", C.c_int32 * 4), ("f_min", C.c_float), ("f_max", C.c_float),
                ("lambda_low", C.c_float), ("lambda_high", C.c_float), ("gemm_planes", C.c_int32)]


def normalize(spec: NetworkSpec) -> dict:
    """Map a NetworkSpec onto the engine's feed-forward family, validating like
    normalize() (network.hpp:125-157).  Supported: [Linear, LIF]*k, Linear, LI | LIF."""
    if not spec.input_shape:
        raise SpecError("network: input shape not declared")
    if not spec.layers:
        raise SpecError("network: no layers")
    last = spec.layers[-1]
    if not isinstance(last, (LIFLayer, LILayer)):
        raise SpecError("network must end in a lif or li readout")
    inp = int(np.prod(spec.input_shape))
    layers, monitor = [], []
    for i, layer in enumerate(spec.layers):
        if isinstance(layer, MonitorLayer):  # network.hpp:139-144
            if not layers or not isinstance(layers[-1], LIFLayer) or (monitor and monitor[-1] == len(layers)):
                raise SpecError(f"layer {i}: monitor must follow a lif layer")
            monitor.append(len(layers))
            continue
        layers.append(layer)
    monitor = [m // 2 - 1 for m in monitor]  # index of the hidden LIF block
    if len(layers) < 4 or len(layers) % 2:
        raise UnsupportedError("engine supports [Linear, LIF]*k + Linear + LI")
    hidden, act, thr, bias, modes, fixed, cells = [], None, None, None, [], [], []
    for i in range(0, len(layers) - 2, 2):
        lin, cell = layers[i], layers[i + 1]
        if not isinstance(lin, LinearLayer) or not isinstance(cell, LIFLayer):
            raise UnsupportedError(f"layer {i}: expected Linear + LIF")
        if cell.beta_mode not in BETA_MODES:
            raise ArgumentError(f"unknown beta mode: {cell.beta_mode}")
        if act is not None and (cell.activation != act or cell.threshold != thr):
            raise UnsupportedError("all LIF layers must share activation and threshold")
        if bias is not None and lin.bias != bias:
            raise UnsupportedError("all Linear layers must share the bias flag")
        act, thr, bias = cell.activation, cell.threshold, lin.bias
        hidden.append(int(lin.out))
        modes.append(cell.beta_mode)
        cells.append("alif" if isinstance(cell, ALIFLayer) else
                     "rlif" if isinstance(cell, RLIFLayer) else "lif")
        fixed.append(float(cell.fixed_beta))
    lin, cell = layers[-2], layers[-1]
    readout_lif = isinstance(cell, LIFLayer)  # network.hpp:153-155: a LIF readout's spikes are the trace
    if not isinstance(lin, LinearLayer) or not isinstance(cell, (LILayer, LIFLayer)):
        raise UnsupportedError("readout must be Linear + LI or Linear + LIF")
    if readout_lif:
        if isinstance(cell, (ALIFLayer, RLIFLayer)):
            raise UnsupportedError("readout must be a LIF or LI cell")
        if cell.activation != act or cell.threshold != thr:
            raise UnsupportedError("all LIF layers must share activation and threshold")
    if lin.bias != bias:
        raise UnsupportedError("all Linear layers must share the bias flag")
    if act.name not in ACTIVATIONS:
        raise ArgumentError(f"unknown activation: {act.name}")
    if cell.beta_mode not in BETA_MODES:
        raise ArgumentError(f"unknown beta mode: {cell.beta_mode}")
    return dict(input=inp, hidden=hidden, classes=int(lin.out), bias=bool(bias),
                threshold=float(thr), activation=act.name, slope=float(act.slope),
                aux=float(act.aux), beta_mode=modes + [cell.beta_mode],
                fixed_beta=fixed + [float(cell.fixed_beta)], monitor=monitor, cell=cells,
                readout_lif=bool(readout_lif))


def shd_spec(hidden=(128, 128), classes=20, inp=700, act="arctan", bias=False,
             cell="lif") -> NetworkSpec:
    """The BASELINE network: 700-H1-H2-20, LIF, arctan k=2, nobias;
    cell="alif" gives BASELINE config 2's adaptive-threshold variant."""
    layers = []
    kind = {"lif": LIFLayer, "alif": ALIFLayer, "rlif": RLIFLayer}[cell]
    for h in hidden:
        layers += [LinearLayer(h, bias), kind(default_activation_desc(act))]
    layers += [LinearLayer(classes, bias), LILayer()]
    return NetworkSpec([inp], layers)


# ---------------------------------------------------------------- library
_lib = None


def lib() -> C.CDLL:
    """Load libsnn_b200.so (built in-tree).  Fails loudly if it cannot be built."""
    global _lib
    if _lib is not None:
        return _lib
    if needs_build():
        build()
    lib = os.environ.get("SNN_B200_LIB") or LIB  # A/B builds of the same sources
    if not os.path.exists(lib):
        raise DeviceError(f"{lib} missing: the CUDA engine is required (no CPU fallback)")
    L = C.CDLL(lib, mode=C.RTLD_GLOBAL)
    # struct layouts below must match the library (SNN_B200_ABI_ANY: timing A/B of an
    # older build whose structs are a prefix of these -- never for results)
    if L.snn_abi_version() != ABI_VERSION and not os.environ.get("SNN_B200_ABI_ANY"):
        raise DeviceError(f"{lib}: ABI {L.snn_abi_version()} != {ABI_VERSION}; rebuild")
    L.snn_last_error.restype = C.c_char_p
    L.snn_last_error.argtypes = [C.c_void_p]
    L.snn_stream.restype = C.c_void_p
    L.snn_stream.argtypes = [C.c_void_p]
    L.snn_launches_per_step.restype = C.c_int32
    L.snn_launches_per_step.argtypes = [C.c_void_p]
    L.snn_forward_launch_layers.restype = C.c_int32
    L.snn_forward_launch_layers.argtypes = [C.c_void_p, C.c_int32, C.POINTER(C.c_int32)]
    for name in ("snn_engine_create", "snn_param_count", "snn_entry_count", "snn_entry_info",
                 "snn_set_params", "snn_get_params", "snn_init_params", "snn_get_opt_state",
                 "snn_set_opt_state", "snn_get_grads", "snn_stage_dataset", "snn_train_step",
                 "snn_train_step_packed", "snn_train_steps_packed", "snn_forward_backward", "snn_train_epochs",
                 "snn_upload_schedule", "snn_enqueue_step", "snn_enqueue_steps", "snn_evaluate", "snn_apply", "snn_save_checkpoint", "snn_load_checkpoint", "snn_sync", "snn_read_result",
                 "snn_nccl_unique_id", "snn_comm_init", "snn_debug_enable", "snn_debug_fetch",
                 "snn_synth_dataset", "snn_epoch_permutation", "snn_profile_steps",
                 "snn_read_dataset", "snn_monitor_counts", "snn_peer_handle", "snn_peer_open",
                 "snn_peer_attach_local", "snn_train_step_split", "snn_load_container",
                 "snn_save_container"):
        if hasattr(L, name) or not os.environ.get("SNN_B200_ABI_ANY"):
            getattr(L, name).restype = C.c_int
    L.snn_launch_name.restype = C.c_char_p
    L.snn_launch_name.argtypes = [C.c_void_p, C.c_int32]
    L.snn_engine_destroy.restype = None
    L.snn_engine_destroy.argtypes = [C.c_void_p]
    _lib = L
    return L


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


class Engine:
    """One training state (TrainState, optimize.hpp:135-141) resident on one GPU."""

    def __init__(self, spec: NetworkSpec, cfg: TrainConfig, time_steps: int, device: int = 0):
        d = normalize(spec)
        self.desc = d
        self.spec, self.cfg, self.time_steps = spec, cfg, int(time_steps)
        n = _NetDesc()
        n.input = d["input"]
        n.n_hidden = len(d["hidden"])
        if n.n_hidden > 8:
            raise UnsupportedError("at most 8 hidden layers")
        for i, h in enumerate(d["hidden"]):
            n.hidden[i] = h
        n.classes = d["classes"]
        n.bias = int(d["bias"])
        n.threshold = d["threshold"]
        n.activation = ACTIVATIONS[d["activation"]]
        n.slope = d["slope"]
        n.aux = d["aux"]
        for i, (bm, fb) in enumerate(zip(d["beta_mode"], d["fixed_beta"])):
            n.beta_mode[i] = BETA_MODES[bm]
            n.fixed_beta[i] = fb
        for m in d["monitor"]:
            n.monitor[m] = 1
        for i, k in enumerate(d["cell"]):
            n.cell[i] = {"lif": 0, "alif": 1, "rlif": 2}[k]
        n.readout_lif = int(d["readout_lif"])
        c = _TrainCfg()
        c.batch_size = int(cfg.batch_size)
        c.time_steps = int(time_steps)
        c.lr = float(cfg.lr)
        c.beta1, c.beta2, c.eps = float(cfg.beta1), float(cfg.beta2), float(cfg.eps)
        c.seed = int(cfg.seed)
        c.unroll = int(cfg.unroll)
        if cfg.optimizer not in ("adam", "sgd"):
            raise ArgumentError(f"train_step: unknown optimizer {cfg.optimizer!r}")
        if cfg.loss not in ("integral_crossentropy", "spike_rate_mse"):
            raise ArgumentError(f"train_step: unknown loss kind {cfg.loss!r}")
        c.optimizer = 1 if cfg.optimizer == "sgd" else 0
        c.momentum = float(cfg.momentum)
        c.loss = 1 if cfg.loss == "spike_rate_mse" else 0
        c.rate_hi, c.rate_lo = float(cfg.rate_hi), float(cfg.rate_lo)
        axes = tuple(int(a) for a in cfg.shift_axes)
        if len(axes) > 4:
            raise ArgumentError("train: at most 4 shift axes")
        c.max_shift, c.n_shift_axes = int(cfg.max_shift), len(axes)
        c.f_min, c.f_max = float(cfg.f_min), float(cfg.f_max)
        c.lambda_low, c.lambda_high = float(cfg.lambda_low), float(cfg.lambda_high)
        c.gemm_planes = int(cfg.gemm_planes)
        for i, a in enumerate(axes):
            c.shift_axes[i] = a
        self._L = lib()
        h = C.c_void_p()
        self._h = None
        self._check(self._L.snn_engine_create(C.byref(n), C.byref(c), int(device), C.byref(h)),
                    create=True)
        self._h = h
        cnt = C.c_size_t()
        self._check(self._L.snn_param_count(self._h, C.byref(cnt)))
        self.n_params = cnt.value
        self.batch_size = int(cfg.batch_size)

    # -------------------------------------------------------------- utils
    def _check(self, rc: int, create: bool = False):
        if rc == 0:
            return
        msg = self._L.snn_last_error(None if create else self._h)
        msg = msg.decode() if msg else f"status {rc}"
        raise _STATUS.get(rc, Error)(msg)

    def close(self):
        if self._h is not None:
            self._L.snn_engine_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    # ---------------------------------------------------------- parameters
    def entries(self):
        cnt = C.c_int32()
        self._check(self._L.snn_entry_count(self._h, C.byref(cnt)))
        out = []
        for i in range(cnt.value):
            name = C.create_string_buffer(16)
            off, size, tr = C.c_size_t(), C.c_size_t(), C.c_int32()
            self._check(self._L.snn_entry_info(self._h, i, name, C.byref(off), C.byref(size),
                                               C.byref(tr)))
            out.append((name.value.decode(), off.value, size.value))
        return out

    def get_params(self) -> np.ndarray:
        out = np.empty(self.n_params, np.float32)
        self._check(self._L.snn_get_params(self._h, _p(out, C.c_float), C.c_size_t(out.size)))
        return out

    def set_params(self, params: np.ndarray):
        p = np.ascontiguousarray(params, np.float32)
        self._check(self._L.snn_set_params(self._h, _p(p, C.c_float), C.c_size_t(p.size)))

    def init_params(self, key_word: int):
        self._check(self._L.snn_init_params(self._h, C.c_uint64(key_word)))

    def get_grads(self) -> np.ndarray:
        out = np.empty(self.n_params, np.float32)
        self._check(self._L.snn_get_grads(self._h, _p(out, C.c_float), C.c_size_t(out.size)))
        return out

    def get_opt_state(self):
        m = np.empty(self.n_params, np.float32)
        v = np.empty(self.n_params, np.float32)
        st = C.c_uint64()
        self._check(self._L.snn_get_opt_state(self._h, _p(m, C.c_float), _p(v, C.c_float),
                                              C.byref(st), C.c_size_t(m.size)))
        return m, v, st.value

    def set_opt_state(self, m, v, step: int):
        m = np.ascontiguousarray(m, np.float32)
        v = np.ascontiguousarray(v, np.float32)
        self._check(self._L.snn_set_opt_state(self._h, _p(m, C.c_float), _p(v, C.c_float),
                                              C.c_uint64(step), C.c_size_t(m.size)))

    # ---------------------------------------------------------------- data
    def stage_dataset(self, packed: np.ndarray, labels: np.ndarray):
        packed = np.ascontiguousarray(packed, np.uint8)
        labels = np.ascontiguousarray(labels, np.int64)
        if packed.ndim != 3 or packed.shape[1] != (self.time_steps + 7) // 8:
            raise FormatError(f"packed extent {packed.shape} inconsistent with T={self.time_steps}")
        if packed.shape[0] != labels.shape[0]:
            raise ArgumentError("label count mismatch")
        self._check(self._L.snn_stage_dataset(self._h, _p(packed, C.c_uint8),
                                              C.c_size_t(packed.shape[0]), _p(labels, C.c_int64)))
        self.n_examples = packed.shape[0]

    def synth_dataset(self, n: int, seed: int = 1):
        """synth_raster(classes, n, T, {input}, seed) generated in HBM (commands.hpp:50-86)."""
        self._check(self._L.snn_synth_dataset(self._h, C.c_size_t(n), C.c_uint64(seed)))
        self.n_examples = n

    def read_dataset(self, start: int, n: int):
        """Rows [start, start+n) of the staged dataset in the reference packed layout."""
        packed = np.empty((n, (self.time_steps + 7) // 8, self.desc["input"]), np.uint8)
        labels = np.empty(n, np.int64)
        self._check(self._L.snn_read_dataset(self._h, C.c_size_t(start), C.c_size_t(n),
                                             _p(packed, C.c_uint8), _p(labels, C.c_int64)))
        return packed, labels

    def epoch_permutation(self, epoch: int, n: int) -> np.ndarray:
        out = np.empty(n, np.uint32)
        self._check(self._L.snn_epoch_permutation(self._h, C.c_size_t(epoch), _p(out, C.c_uint32),
                                                  C.c_size_t(n)))
        return out

    # ---------------------------------------------------------------- steps
    def train_step(self, rows) -> tuple[float, float]:
        r = np.ascontiguousarray(rows, np.uint32)
        if r.size != self.batch_size:
            raise ArgumentError(f"targets: {r.size} rows for batch {self.batch_size}")
        loss, acc = C.c_float(), C.c_double()
        self._check(self._L.snn_train_step(self._h, _p(r, C.c_uint32), C.byref(loss), C.byref(acc)))
        return loss.value, acc.value

    def forward_backward(self, rows) -> tuple[float, float]:
        r = np.ascontiguousarray(rows, np.uint32)
        if r.size != self.batch_size:
            raise ArgumentError(f"targets: {r.size} rows for batch {self.batch_size}")
        loss, acc = C.c_float(), C.c_double()
        self._check(self._L.snn_forward_backward(self._h, _p(r, C.c_uint32), C.byref(loss),
                                                 C.byref(acc)))
        return loss.value, acc.value

    def _check_packed(self, packed_x: np.ndarray, time_axis: int):
        """Full shape check before the C ABI reads B * ceil(T/8) * input bytes per step:
        [..., B, ceil(T/8), input] with exactly time_axis + 2 dims (unpack_time's
        FormatError for the time extent, data.hpp:131-134; ShapeError otherwise)."""
        if packed_x.ndim != time_axis + 2:
            raise ShapeError(f"packed batch: {packed_x.ndim} dims, need {time_axis + 2}")
        if packed_x.shape[time_axis] != (self.time_steps + 7) // 8:
            raise FormatError(f"unpack_time: packed extent {packed_x.shape[time_axis]} "
                              f"inconsistent with T={self.time_steps}")
        if packed_x.shape[time_axis + 1] != self.desc["input"]:
            raise ShapeError(f"packed batch: {packed_x.shape[time_axis + 1]} features, "
                             f"the network takes {self.desc['input']}")

    def train_step_packed(self, packed_x: np.ndarray, targets) -> tuple[float, float]:
        """train_step(st, packed_x, T, targets) (optimize.hpp:152-156)."""
        packed_x = np.ascontiguousarray(packed_x, np.uint8)
        t = np.ascontiguousarray(targets, np.int64)
        self._check_packed(packed_x, 1)
        if packed_x.shape[0] != self.batch_size or t.size != self.batch_size:
            raise ArgumentError(f"targets: {t.size} labels for batch {packed_x.shape[0]}")
        loss, acc = C.c_float(), C.c_double()
        self._check(self._L.snn_train_step_packed(self._h, _p(packed_x, C.c_uint8),
                                                  _p(t, C.c_int64), C.byref(loss), C.byref(acc)))
        return loss.value, acc.value

    def train_steps_packed(self, packed_x: np.ndarray, targets) -> tuple[np.ndarray, np.ndarray]:
        """train() over host batches with pipelined uploads: packed_x [n_steps, B, ceil(T/8),
        input] (pinned memory overlaps the copies), targets [n_steps, B] -> per-step
        (losses, accuracies); same results as n_steps train_step_packed calls."""
        packed_x = np.ascontiguousarray(packed_x, np.uint8)
        t = np.ascontiguousarray(targets, np.int64)
        n = packed_x.shape[0]
        self._check_packed(packed_x, 2)
        if packed_x.shape[1] != self.batch_size or t.shape != (n, self.batch_size):
            raise ArgumentError("train_steps_packed: need [n_steps, B, ceil(T/8), input] and [n_steps, B]")
        losses = np.zeros(n, np.float32)
        accs = np.zeros(n, np.float64)
        self._check(self._L.snn_train_steps_packed(self._h, _p(packed_x, C.c_uint8), _p(t, C.c_int64),
                                                   C.c_size_t(n), _p(losses, C.c_float),
                                                   _p(accs, C.c_double)))
        return losses, accs

    def train_epochs(self, epochs: int) -> np.ndarray:
        metrics = np.zeros((epochs, 2), np.float64)
        self._check(self._L.snn_train_epochs(self._h, C.c_size_t(epochs), _p(metrics, C.c_double)))
        return metrics

    # ------------------------------------------------------------- async path
    def upload_schedule(self, rows: np.ndarray):
        r = np.ascontiguousarray(rows, np.uint32)
        self._check(self._L.snn_upload_schedule(self._h, _p(r, C.c_uint32),
                                                C.c_size_t(r.size // self.batch_size)))

    def enqueue_step(self, slot: int):
        self._check(self._L.snn_enqueue_step(self._h, C.c_size_t(slot)))

    def enqueue_steps(self, first_slot: int, n_steps: int):
        """Schedule slots [first_slot, first_slot + n_steps), 8 steps per graph launch."""
        self._check(self._L.snn_enqueue_steps(self._h, C.c_size_t(first_slot), C.c_size_t(n_steps)))

    # ------------------------------------------------------------ evaluation
    def evaluate(self, rows) -> tuple[float, float]:
        """cmd_eval (commands.hpp:144-169) over dataset `rows`: (accuracy, mean loss)."""
        r = np.ascontiguousarray(rows, np.uint32)
        acc, loss = C.c_double(), C.c_double()
        self._check(self._L.snn_evaluate(self._h, _p(r, C.c_uint32), C.c_size_t(r.size),
                                         C.byref(acc), C.byref(loss)))
        return acc.value, loss.value

    def apply(self, rows) -> np.ndarray:
        """apply (network.hpp:435-448) on one batch of rows: readout trace [B, T, C]."""
        r = np.ascontiguousarray(rows, np.uint32)
        out = np.empty((self.batch_size, self.time_steps, self.desc["classes"]), np.float32)
        self._check(self._L.snn_apply(self._h, _p(r, C.c_uint32), _p(out, C.c_float),
                                      C.c_size_t(out.size)))
        return out

    def load_container(self, path: str) -> int:
        """read_container (data.hpp:295-339) of a .spkd file, staged in HBM; returns N."""
        n = C.c_size_t()
        self._check(self._L.snn_load_container(self._h, str(path).encode(), C.byref(n)))
        return n.value

    def save_container(self, path: str):
        """write_container (data.hpp:272-293) of the staged dataset."""
        self._check(self._L.snn_save_container(self._h, str(path).encode()))

    def monitor_counts(self, layer: int) -> np.ndarray:
        """ApplyResult.monitors entry of the monitor after hidden LIF `layer`: spike
        counts [B, H] of the last forward (neuron.hpp:106-114)."""
        if layer not in self.desc["monitor"]:
            raise ArgumentError(f"hidden layer {layer} has no monitor")
        out = np.empty((self.batch_size, self.desc["hidden"][layer]), np.float32)
        self._check(self._L.snn_monitor_counts(self._h, C.c_int32(layer), _p(out, C.c_float),
                                               C.c_size_t(out.size)))
        return out

    # ------------------------------------------------------------ checkpoints
    def save_checkpoint(self, path: str, config_text: str = ""):
        """write_checkpoint (optimize.hpp:334-366) of the device state, .spkc bit-exact."""
        cfg = config_text.encode()
        self._check(self._L.snn_save_checkpoint(self._h, os.fsencode(path), cfg, C.c_size_t(len(cfg))))

    def load_checkpoint(self, path: str) -> str:
        """read_checkpoint (optimize.hpp:376-436) into the engine; returns the config text."""
        n = C.c_size_t()
        buf = C.create_string_buffer((1 << 20) + 1)  # the format caps config text at 1 MiB
        self._check(self._L.snn_load_checkpoint(self._h, os.fsencode(path), buf,
                                                C.c_size_t(len(buf)), C.byref(n)))
        return buf.raw[:n.value].decode()

    def sync(self):
        self._check(self._L.snn_sync(self._h))

    def read_result(self):
        loss, acc = C.c_float(), C.c_double()
        self._check(self._L.snn_read_result(self._h, C.byref(loss), C.byref(acc)))
        return loss.value, acc.value

    @property
    def stream(self) -> int:
        return int(self._L.snn_stream(self._h) or 0)

    def profile(self, steps: int = 5):
        """[(launch name, mean device ms)] for one step (graph with event nodes)."""
        ms = np.zeros(64, np.float64)
        n = C.c_int32()
        self._check(self._L.snn_profile_steps(self._h, int(steps), _p(ms, C.c_double), 64,
                                              C.byref(n)))
        return [(self._L.snn_launch_name(self._h, i).decode(), float(ms[i])) for i in range(n.value)]

    @property
    def launches_per_step(self) -> int:
        return int(self._L.snn_launches_per_step(self._h))

    @property
    def forward_launches(self) -> list[tuple[int, int]]:
        """[(first hidden layer, layer count)] per forward launch of a step."""
        out, i, first = [], 0, C.c_int32()
        while True:
            n = int(self._L.snn_forward_launch_layers(self._h, i, C.byref(first)))
            if n == 0:
                return out
            out.append((int(first.value), n))
            i += 1

    # ---------------------------------------------------------- multi-GPU
    @staticmethod
    def nccl_unique_id() -> bytes:
        L = lib()
        buf = (C.c_uint8 * 128)()
        rc = L.snn_nccl_unique_id(buf)
        if rc != 0:
            raise DeviceError((L.snn_last_error(None) or b"").decode())
        return bytes(buf)

    def comm_init(self, uid: bytes, rank: int, world: int):
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        self._check(self._L.snn_comm_init(self._h, buf, int(rank), int(world)))

    # peer-memory data parallelism (the default multi-GPU tail; see snn_engine.h)
    def peer_handle(self) -> bytes:
        """This rank's exchange buffer as a 64-byte IPC handle."""
        buf = (C.c_uint8 * 64)()
        self._check(self._L.snn_peer_handle(self._h, buf))
        return bytes(buf)

    def peer_open(self, rank: int, world: int, handles):
        """Map every rank's exchange buffer (handles in rank order, from peer_handle)."""
        if len(handles) != world or any(len(h) != 64 for h in handles):
            raise ArgumentError("peer_open: one 64-byte handle per rank")
        buf = (C.c_uint8 * (64 * world)).from_buffer_copy(b"".join(handles))
        self._check(self._L.snn_peer_open(self._h, int(rank), int(world), buf))

    @staticmethod
    def peer_attach_local(engines):
        """Test hook: engines of one GPU as ranks 0..n-1 of the peer tail (drive them
        with train_step_split so no kernel waits on a rank that has not run)."""
        L = lib()
        arr = (C.c_void_p * len(engines))(*[e._h.value for e in engines])
        rc = L.snn_peer_attach_local(arr, len(engines))
        if rc != 0:
            engines[0]._check(rc)

    def train_step_split(self, rows, part: int):
        """part 0: forward .. local reduction (synchronised); part 1: owner phase
        (this rank's parameter slice, synchronised); part 2: gather -> (loss, accuracy)."""
        loss, acc = C.c_float(), C.c_double()
        r = np.ascontiguousarray(rows, np.uint32) if rows is not None else None
        self._check(self._L.snn_train_step_split(self._h, _p(r, C.c_uint32) if r is not None else None,
                                                 int(part), C.byref(loss), C.byref(acc)))
        return loss.value, acc.value

    # ---------------------------------------------------------- diagnostics
    def debug(self, on=True):
        """True / 1: capture tensors + clock stamps; 2: clock stamps only."""
        self._check(self._L.snn_debug_enable(self._h, 2 if on == 2 else int(bool(on))))

    def check_guards(self) -> int:
        """SNN_GUARD=1: verify the out-of-bounds guard bytes of every device buffer
        (raises ContractError on an overwrite); returns the number checked."""
        n = C.c_int32()
        self._check(self._L.snn_debug_check_guards(self._h, C.byref(n)))
        return n.value

    def fetch(self, which: str, layer: int = 0) -> np.ndarray:
        idx = {"I": 0, "V": 1, "spikes": 2, "trace": 3, "dS": 4, "clk": 5, "A": 6, "dI": 7}[which]
        B, T = self.batch_size, self.time_steps
        if which == "clk":  # rows per slot: engine.cu clk_region()
            tiles = max([4] + [(h + 127) // 128 for h in self.desc["hidden"]])
            out = np.empty((3 + 2 * len(self.desc["hidden"]), max(B * tiles, 4096), 48), np.int64)
        elif which == "trace" or (which == "dI" and layer == len(self.desc["hidden"])):
            out = np.empty((B, T, self.desc["classes"]), np.float32)
        else:
            H = self.desc["hidden"][layer]
            out = np.empty((B, T, H), np.uint8 if which == "spikes" else np.float32)
        self._check(self._L.snn_debug_fetch(self._h, idx, int(layer),
                                            out.ctypes.data_as(C.c_void_p), C.c_size_t(out.nbytes)))
        return out


def train_step(engine: Engine, packed_x, original_t: int, targets):
    """Free-function form of optimize.hpp:152-156."""
    if original_t != engine.time_steps:
        raise FormatError(f"unpack_time: packed extent inconsistent with T={original_t}")
    return engine.train_step_packed(packed_x, targets)
