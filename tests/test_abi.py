"""The C-ABI library: builds, loads, exports exactly what include/tnb.h declares,
and fails loudly (no CPU fallback) when there is no GPU. No compute on CPU."""
import ctypes
import os
import re

import pytest

from paper_2401_01921_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "tnb.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tnb_[a-z0-9_]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert declared_symbols() == sorted(_lib.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = _lib.lib()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.tnb_version() == 100


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out.replace("sm_100a", ""))


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    n = _lib.device_count()
    assert n == 0
    with pytest.raises(_lib.EngineUnavailable):
        _lib.permute(0, 0, 8, [2, 3], [1, 0], None)
    with pytest.raises(_lib.EngineUnavailable):
        _lib.contract_dense(0, 0, [2, 2], [0, 1], 0, 0, [2, 2], [0, 1], [1], [0], 0, 0, None)
    from paper_2401_01921_b200 import dense
    with pytest.raises(_lib.EngineUnavailable):
        dense.zeros([2, 2])


def test_last_error_message_is_set():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(_lib.EngineUnavailable) as e:
        _lib.permute(0, 0, 8, [2, 3], [1, 0], None)
    assert "no CUDA device" in str(e.value)
