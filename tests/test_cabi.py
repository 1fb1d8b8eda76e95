"""The drop-in boundary (include/et_runtime.h): the C-ABI library loads and
exports every declared entry point; without a GPU it fails loudly."""

import ctypes
import os
import re

import paper_2604_13327_b200 as pkg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    text = open(os.path.join(ROOT, "include", "et_runtime.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(et_[a-z_]+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(pkg.LIBRARY_PATH)
    names = declared()
    assert len(names) >= 14, names
    for n in names:
        assert hasattr(lib, n), n


def test_abi_version_and_struct_sizes():
    lib = ctypes.CDLL(pkg.LIBRARY_PATH)
    assert lib.et_abi_version() == 1
    from paper_2604_13327_b200 import etsim
    from paper_2604_13327_b200.ops import EtOp

    assert ctypes.sizeof(EtOp) == etsim.OP_BYTES == 176


def test_no_device_is_reported_not_faked():
    import torch

    if torch.cuda.is_available():
        return
    lib = ctypes.CDLL(pkg.LIBRARY_PATH)
    n = ctypes.c_int(-1)
    assert lib.et_device_count(ctypes.byref(n)) == 6  # ET_ERR_NO_DEVICE
    assert n.value == 0
