"""CPU: the C-ABI library loads and exports every symbol include/bosp_b200.h declares
(no compute without a GPU)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "bosp_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = set(re.findall(r"\b(bosp_[A-Za-z0-9_]+)\s*\(", text))
    # typedef'd function-pointer names are not symbols
    names -= {"bosp_host_apply_fn", "bosp_device_apply_fn"}
    return sorted(names)


def test_header_declares_core_entry_points():
    syms = declared_symbols()
    for s in ("bosp_solve", "bosp_op_csr", "bosp_op_dense", "bosp_op_callback", "bosp_biorth",
              "bosp_block_inner", "bosp_cg_solve"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_2506_08355_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        pytest.fail("libbosp_b200.so not built: run __graft_entry__.build()")
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert sorted(_lib.EXPORTED) == declared_symbols()


def test_library_is_sm100a_only():
    """The fatbin carries sm_100a SASS (DMMA for the fp64 contractions), no PTX fallback."""
    import shutil
    import subprocess
    from paper_2506_08355_b200 import _lib
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([exe, "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run([exe, "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "DMMA" in sass


def test_no_gpu_call_fails_loudly_without_device():
    """Without a GPU the product path must raise, never fall back to CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np
    from paper_2506_08355_b200 import bosp
    with pytest.raises(bosp.BospError):
        bosp.LinearOperator.identity(4).apply(np.ones((4, 1)))
    with pytest.raises(bosp.BospError):
        bosp.LinearOperator.from_dense(np.eye(4))
    with pytest.raises(bosp.BospError):
        bosp.block_inner(None, np.ones((5, 2)), np.ones((5, 2)))
