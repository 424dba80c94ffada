"""The C-ABI library loads on a CPU-only host and exports every symbol declared in
include/promptcache_b200.h; device entry points fail loudly (no CPU fallback)."""
import ctypes
import os
import re

import pytest

import paper_2311_04934_b200 as pcb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "promptcache_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pcb_[a-z0-9_]+)\s*\(", text)))


def test_every_declared_symbol_is_exported():
    lib = ctypes.CDLL(pcb.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 50
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_library_is_sm100a():
    # the product library carries sm_100a tcgen05 code (UTCHMMA / UTMALDG in SASS)
    import shutil
    import subprocess

    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    out = subprocess.run(["cuobjdump", "-sass", pcb.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", pcb.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in out and ("UTMALDG" in out or "UBLKCP" in out)


def test_no_cpu_fallback_without_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    with pytest.raises(pcb.PromptCacheError) as ei:
        pcb.Model({"n_layers": 1}, dtype=pcb.BF16)
    assert ei.value.code == "CudaError"


def test_version_string():
    assert b"sm_100a" in pcb.lib().pcb_version()
