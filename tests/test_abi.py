"""The C-ABI library loads and exports every symbol include/desklm_cuda.h
declares (no compute calls -- this runs on the CPU-only builder)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "desklm_cuda.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(dl_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_header_symbols():
    from paper_1502_00512_b200 import _lib
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.EXPORTS)


def test_library_is_sm100a():
    so = os.path.join(ROOT, "paper_1502_00512_b200", "libdesklm_cuda.so")
    data = open(so, "rb").read()
    assert b"sm_100a" in data or b"sm_100" in data


def test_errors_without_gpu_are_reported_not_crashes():
    import paper_1502_00512_b200 as dl
    from paper_1502_00512_b200 import _lib
    lib = _lib.load()
    assert lib.dl_version().startswith(b"desklm-b200")
    h = C.c_void_p()
    assert lib.dl_create(C.byref(h), 0, 0, 4, 0, 0) == _lib.DL_EINVAL
    assert lib.dl_create(C.byref(h), 0, 16, 4, 7, 0) == _lib.DL_EINVAL
    assert lib.dl_create(C.byref(h), 0, 10, 4, 0, 1) == _lib.DL_EINVAL  # bf16 needs %8
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if not has_gpu:
        with pytest.raises((dl.DeviceError, ValueError)):
            dl.GpuRnn(16, 8)


def test_config_validation_mirrors_reference():
    from paper_1502_00512_b200 import TrainConfig
    TrainConfig(mode=1).validate()
    TrainConfig(mode=0).validate()  # NCE (LossMode::kNce, the reference default)
    for bad in (dict(nstate=0), dict(noffset=0), dict(eta=0.0), dict(rho=1.0), dict(eps=0.0),
                dict(clip=0.0), dict(max_epochs=0), dict(divergence_factor=1.0),
                dict(valid_limit=-1), dict(valid_shards=0), dict(init_range=0.0),
                dict(threads=0), dict(mode=2), dict(mode=0, nce_k=0)):
        with pytest.raises(ValueError):
            TrainConfig(**dict(dict(mode=1), **bad)).validate()


def test_bottleneck_argument_errors_without_gpu():
    """dl_bn_create validates like the BottleneckParams constructor
    (compress.hpp:66-74) before touching the device."""
    from paper_1502_00512_b200 import _lib
    lib = _lib.load()
    h = C.c_void_p()
    assert lib.dl_bn_create(C.byref(h), 0, 0, 4, 2, 0, 0) == _lib.DL_EINVAL
    assert lib.dl_bn_create(C.byref(h), 0, 16, 4, 8, 0, 0) == _lib.DL_EINVAL  # P > H
    assert b"P must not exceed H" in lib.dl_bn_last_error(None)
    assert lib.dl_bn_create(C.byref(h), 0, 16, 8, 4, 0, 1) == _lib.DL_EINVAL  # bf16 needs %8
    assert lib.dl_bn_create(C.byref(h), 0, 16, 8, 8, 3, 0) == _lib.DL_EINVAL  # act


def test_library_loaded_before_torch_leaves_torch_importable():
    """The library and libtorch_cuda must share one libnccl.so.2: loaded
    first, the library must not pin an older NCCL that leaves torch's
    symbols unresolved (Makefile NCCL_LIB)."""
    import subprocess
    import sys
    code = ("from paper_1502_00512_b200 import _lib; _lib.load()\n"
            "import torch, torch.distributed\n"
            "print('ok')\n")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]
