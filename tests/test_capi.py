"""CPU tests of the C ABI boundary: every function declared in include/scb.h is bound in
paper_2605_13928_b200/_lib.py and exported by libscb_b200.so; host-only entry points and the
error path work without a GPU."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "scb.h")


def header_functions():
    txt = open(HEADER).read()
    return set(re.findall(r"SCB_API\s+[\w\s\*]+?\b(scb_\w+)\s*\(", txt))


@pytest.fixture(scope="module")
def lib():
    from paper_2605_13928_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        subprocess.run(["make", "-j8", "-C", os.path.join(ROOT, "paper_2605_13928_b200", "csrc")], check=True)
    return ctypes.CDLL(_lib.LIB_PATH)


def test_header_and_binding_agree():
    from paper_2605_13928_b200 import _lib
    declared = header_functions()
    assert len(declared) >= 20
    assert declared == set(_lib.SIGNATURES), (declared ^ set(_lib.SIGNATURES))


def test_library_exports_every_declared_symbol(lib):
    for name in sorted(header_functions()):
        assert hasattr(lib, name), name


def test_binding_loads_and_host_entry_points(lib):
    from paper_2605_13928_b200 import _lib
    L = _lib.load()
    assert L.scb_abi_version() == 1
    assert L.scb_hvg_tiles(2000) == 1
    assert L.scb_hvg_tiles(25000) == 2
    assert _lib.launch_count() >= 0


def test_error_path_without_device(lib):
    """No GPU in this container: context creation must fail loudly with a message (no CPU fallback)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2605_13928_b200 import _lib
    with pytest.raises(_lib.ScbError) as e:
        _lib.context(0)
    assert "scb_ctx_create" in str(e.value)


def test_null_argument_rejected(lib):
    from paper_2605_13928_b200 import _lib
    L = _lib.load()
    rc = L.scb_gram(None, None, 0, 128, None, None)
    assert rc == -1
    assert b"null" in L.scb_last_error()
