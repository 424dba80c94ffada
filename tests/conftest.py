import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


def _ensure_built():
    lib = os.path.join(ROOT, "paper_2311_04934_b200", "lib", "libpcb200.so")
    if not os.path.exists(lib):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_2311_04934_b200", "csrc"), "-j8"], check=True)
    if not os.path.exists(os.path.join(ROOT, "oracle", "liboracle.so")):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "oracle"], check=True)


_ensure_built()


@pytest.fixture(scope="session")
def host_golden():
    with open(os.path.join(GOLDEN, "host.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def numeric_golden():
    with open(os.path.join(GOLDEN, "numeric.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def ref():
    """The compiled reference (oracle/_ref); skipped when it was not built here."""
    from oracle.oracle import Ref, ref_available

    if not ref_available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    Ref.lib()
    return Ref
