"""The C-ABI library: builds, loads and exports every symbol the header declares (no GPU)."""

import ctypes
import os
import re

import pytest

from conftest import ROOT, gpu_available

HEADER = os.path.join(ROOT, "include", "momentcp_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(mcp_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_reference_boundary():
    syms = declared_symbols()
    for needed in ("mcp_create", "mcp_destroy", "mcp_load_obs", "mcp_fg", "mcp_fg_packed",
                   "mcp_ttsv_batch", "mcp_data_norm_sq", "mcp_fg_partial_device",
                   "mcp_fg_finish_device", "mcp_last_error"):
        assert needed in syms


def test_library_exports_every_declared_symbol():
    from paper_1911_03813_b200 import _native

    lib = _native.load_library()
    for name in declared_symbols():
        assert hasattr(lib, name), f"{name} declared in the header but not exported"
        assert name in _native.SIGNATURES, f"{name} has no ctypes signature"
    assert lib.mcp_abi_version() == 1


def test_library_links_only_system_runtime():
    # statically linked cudart: the .so must not depend on torch's CUDA libraries
    from paper_1911_03813_b200 import _native

    import subprocess

    out = subprocess.run(["ldd", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "libtorch" not in out and "libc10" not in out


@pytest.mark.skipif(gpu_available(), reason="checks the no-GPU failure mode")
def test_create_fails_loudly_without_gpu():
    from paper_1911_03813_b200 import _native

    lib = _native.load_library()
    h = ctypes.c_void_p()
    rc = lib.mcp_create(ctypes.byref(h), 0)
    assert rc == _native.MCP_ERR_CUDA
    assert lib.mcp_last_error(None)  # a message, not silence
    with pytest.raises(RuntimeError):
        _native.Context(0)


def test_sass_uses_fp64_tensor_path():
    """K1/K5 lower to DMMA (the FP64 tensor-core instruction), not scalar DFMA loops."""
    import shutil
    import subprocess

    from paper_1911_03813_b200 import _native

    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    sass = subprocess.run([tool, "-sass", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "DMMA.8x8x4" in sass
    assert "sm_100a" in subprocess.run([tool, "-lelf", _native.LIB_PATH], capture_output=True,
                                       text=True).stdout or "sm_100" in sass
