"""The C-ABI library loads and exports every symbol include/hf.h declares (CPU only;
no compute calls).  Also checks argument validation that needs no GPU."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hf.h")


def declared_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(hf_[a-z0-9_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def hf():
    from paper_2203_08395_b200 import build
    build.build()
    from paper_2203_08395_b200 import hf as _hf
    return _hf


def test_header_declares_the_north_star_calls():
    syms = declared_symbols()
    for name in ("hf_graph_create", "hf_levelize", "hf_propagate_forward",
                 "hf_propagate_backward", "hf_run_batch"):
        assert name in syms


def test_library_exports_every_declared_symbol(hf):
    lib = ctypes.CDLL(hf.LIB_PATH)
    syms = declared_symbols()
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert sorted(hf.EXPORTS) == syms
    out = subprocess.run(["nm", "-D", "--defined-only", hf.LIB_PATH], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r"\bT (hf_[a-z0-9_]+)$", out, flags=re.M))
    assert set(syms) <= exported


def test_library_is_sm100a(hf):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", hf.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_strings_and_version(hf):
    assert hf.hf_version() == 101
    assert hf._status_name(3) == "HF_ERR_CYCLE"
    assert hf._status_name(0) == "HF_OK"


def test_invalid_args_without_gpu(hf):
    import numpy as np
    with pytest.raises(hf.HFError) as ei:
        hf.hf_graph_create(-1, 0, np.zeros(1, np.int32), None)
    assert ei.value.status == hf.HF_ERR_INVALID_ARG
    out = ctypes.c_void_p()
    st = hf._lib.hf_graph_create(3, 2, None, None, None, None, None, 0, None, ctypes.byref(out))
    assert st == hf.HF_ERR_INVALID_ARG
    assert hf._lib.hf_graph_destroy(None) == hf.HF_OK
    assert hf._lib.hf_sync(None) == hf.HF_ERR_INVALID_ARG
    assert hf._lib.hf_levelize(None, None, None, None, None) == hf.HF_ERR_INVALID_ARG
