"""CPU-side checks of the C-ABI boundary: the library loads, exports every
symbol include/znn_cuda.h declares, and fails loudly (status 2, no CPU
fallback) when there is no CUDA device."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "znn_cuda.h")).read()
    return sorted(set(re.findall(r"\b(znn_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_1510_06706_b200 import _lib
    L = _lib.lib()
    declared = header_symbols()
    assert len(declared) >= 40
    for name in declared:
        assert hasattr(L, name), name
    assert sorted(_lib.EXPORTS) == declared


def test_version_and_device_count():
    from paper_1510_06706_b200 import _lib
    L = _lib.lib()
    assert b"sm_100a" in L.znn_version()
    assert L.znn_device_count() >= 0


def test_no_cpu_fallback_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1510_06706_b200 import Context, ZnnError
    with pytest.raises(ZnnError) as e:
        Context(0)
    assert e.value.status == 2
    assert "no CPU fallback" in str(e.value)


def test_sass_is_sm100a():
    """The shipped .so carries sm_100a SASS only (no PTX JIT path to other archs)."""
    import subprocess
    so = os.path.join(ROOT, "paper_1510_06706_b200", "libznn_cuda.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
