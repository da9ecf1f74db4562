"""The drop-in boundary: liblinedg_b200.so loads without a GPU and exports
every entry point include/linedg_b200.h declares; without a device the
library refuses to create a context (no CPU fallback)."""
import ctypes as C
import os
import re
import subprocess

import pytest

from paper_1204_1533_b200 import CONFIGS, _abi
from paper_1204_1533_b200._abi import gpu_lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "linedg_b200.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ldg_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_reconstructed_api():
    names = declared()
    for n in ("ldg_create", "ldg_residual", "ldg_gradient", "ldg_residual_uq", "ldg_jacobian_assemble",
              "ldg_bsr_spmv", "ldg_split_matvec", "ldg_export_blocks", "ldg_last_error", "ldg_destroy"):
        assert n in names


def test_library_exports_every_declared_symbol():
    lib = gpu_lib()
    for name in declared():
        assert hasattr(lib, name), f"{name} not exported"
    out = subprocess.run(["nm", "-D", "--defined-only", os.path.join(ROOT, "paper_1204_1533_b200",
                                                                   "liblinedg_b200.so")],
                         capture_output=True, text=True).stdout
    for name in declared():
        assert re.search(rf"\bT {name}\b", out), name
    # the library carries sm_100a code
    sass = subprocess.run(["cuobjdump", "--list-elf", os.path.join(ROOT, "paper_1204_1533_b200",
                                                                   "liblinedg_b200.so")],
                          capture_output=True, text=True).stdout
    assert "sm_100a" in sass


def test_python_mirror_binds_all_symbols():
    assert set(_abi.GPU_SYMBOLS) <= set(declared())


def test_no_device_means_no_context():
    import torch

    if torch.cuda.is_available():
        pytest.skip("device present")
    case, _ = CONFIGS[1].build(n=2)
    ph = CONFIGS[1].physics.to_c()
    h = C.c_void_p()
    st = gpu_lib().ldg_create(case.setup_ptr, C.byref(ph), None, C.byref(h))
    assert st == _abi.LDG_ERR_CUDA
    assert b"no CUDA device" in gpu_lib().ldg_last_error(None)
