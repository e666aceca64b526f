"""B200-native SNN training engine (drop-in for spiketrain's train_step).

The compute path is libsnn_b200.so (hand-written sm_100a CUDA, tcgen05/TMEM/TMA)
behind the C ABI in include/snn_engine.h; this package is the Python mirror of
the reference interface used by the tests and bench.py.
"""
from .engine import (  # noqa: F401
    ActivationDesc, ALIFLayer, ArgumentError, ConfigError, ContractError, DeviceError, Engine, Error,
    FormatError, IoError, LIFLayer, LILayer, LinearLayer, MonitorLayer, NetworkSpec, RLIFLayer, ShapeError,
    SpecError,
    StateError, TrainConfig, UnsupportedError, default_activation_desc, lib, normalize,
    shd_spec, train_step,
)
