"""The C-ABI library builds for sm_100a, loads, and exports every entry point
declared in include/rnngraph_b200.h (no compute: this runs without a GPU)."""
from __future__ import annotations

import ctypes
import os
import re
import shutil

import pytest

from paper_1503_02852_b200 import _lib

HEADER = os.path.join(_lib.REPO, "include", "rnngraph_b200.h")


def _declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:int|const char\*)\s+(rgb_\w+)\(", text, flags=re.M)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(_lib.LIB_PATH):
        if shutil.which("nvcc") is None:
            pytest.skip("library not built and nvcc unavailable")
        _lib.build()
    return _lib.lib()


def test_header_and_binding_agree():
    assert _declared() == sorted(_lib.EXPORTS)


def test_every_declared_symbol_is_exported(lib):
    for name in _declared():
        assert hasattr(lib, name), name
    assert lib.rgb_abi_version() == 1


def test_no_cpu_fallback_without_sm100(lib):
    """Plan creation must fail loudly when no sm_100 device is visible."""
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is visible")
    except ImportError:
        pass
    h = ctypes.c_void_p()
    words = (ctypes.c_int32 * 40)()
    rc = lib.rgb_plan_create(ctypes.cast(words, ctypes.c_void_p), 40, ctypes.byref(h))
    assert rc == _lib.RGB_ERR_CUDA
    assert b"device" in lib.rgb_last_error()


def test_sass_is_sm100(lib):
    """The fatbin holds sm_100a SASS (cuobjdump), not PTX for a JIT fallback."""
    if shutil.which("cuobjdump") is None:
        pytest.skip("cuobjdump unavailable")
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_set_tc_precision_validates_mode_without_gpu():
    import paper_1503_02852_b200 as P
    with pytest.raises(ValueError):
        P.set_tc_precision("fp16")
