"""The C-ABI library loads and exports every declared symbol (CPU only)."""

import os
import re
import subprocess

import pytest

from paper_2305_13479_b200 import _native
from paper_2305_13479_b200.errors import SolverBackendError

HEADER = os.path.join(os.path.dirname(__file__), "..", "include", "teccl_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(teccl_[a-z0-9_]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert declared_symbols() == sorted(_native.EXPORTED)


def test_library_exports_every_declared_symbol():
    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("libteccl_b200.so not built (run __graft_entry__.build())")
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (teccl_[a-z0-9_]+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing


def test_library_loads_and_reports_version():
    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("libteccl_b200.so not built")
    lib = _native.load()
    assert b"sm_100a" in lib.teccl_version()


def test_no_device_fails_loudly():
    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("libteccl_b200.so not built")
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(SolverBackendError):
        _native.Context(0)


def test_missing_library_fails_loudly(tmp_path):
    with pytest.raises(SolverBackendError):
        _native.load(str(tmp_path / "nope.so"))
