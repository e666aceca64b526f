"""CPU-side checks of the C-ABI library: it builds for sm_100a, loads, exports
every symbol include/snn_engine.h declares, and refuses to run without a GPU
(no CPU fallback).  No compute calls."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "snn_engine.h")).read()
    return sorted(set(re.findall(r"\b(snn_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2402_18994_b200.build import build
    return build()


def test_exports_every_declared_symbol(libpath):
    lib = C.CDLL(libpath)
    missing = [s for s in header_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert len(header_symbols()) >= 25


def test_sass_is_blackwell_native(libpath):
    out = subprocess.run(["cuobjdump", "-sass", libpath], capture_output=True, text=True).stdout
    assert "UTCHMMA" in out          # tcgen05.mma
    assert "UTMALDG" in out          # TMA tensor loads
    assert "LDTM" in out             # tcgen05.ld (TMEM -> registers)
    assert "HMMA" not in out.replace("UTCHMMA", "")  # no legacy mma.sync path
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", libpath], capture_output=True,
                                       text=True).stdout


def test_no_gpu_means_device_error():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2402_18994_b200 import DeviceError, Engine, TrainConfig, shd_spec
    with pytest.raises(DeviceError):
        Engine(shd_spec(), TrainConfig(batch_size=4), 128)


def test_spec_validation_mirrors_reference():
    from paper_2402_18994_b200 import (LIFLayer, LILayer, LinearLayer, NetworkSpec, SpecError,
                                       UnsupportedError, normalize, shd_spec)
    d = normalize(shd_spec())
    assert d["hidden"] == [128, 128] and d["classes"] == 20 and d["input"] == 700
    with pytest.raises(SpecError):
        normalize(NetworkSpec([], [LinearLayer(4), LILayer()]))
    with pytest.raises(SpecError):
        normalize(NetworkSpec([4], [LinearLayer(4)]))
    # a LIF readout (network.hpp:153-155, :396) is supported; it must share the
    # hidden layers' threshold and surrogate
    d = normalize(NetworkSpec([4], [LinearLayer(4), LIFLayer(), LinearLayer(3), LIFLayer()]))
    assert d["readout_lif"] and d["classes"] == 3
    assert not normalize(shd_spec())["readout_lif"]
    with pytest.raises(UnsupportedError):
        normalize(NetworkSpec([4], [LinearLayer(4), LIFLayer(), LinearLayer(3), LIFLayer(threshold=0.5)]))
    with pytest.raises(SpecError):
        normalize(NetworkSpec([4], [LinearLayer(4), LIFLayer(), LinearLayer(3)]))
