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


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    """Greedy-token parity accounting (report how many cases used the tie exemption)."""
    from tests.util import GREEDY, RELS, SEQ

    if not GREEDY["checked"] and not SEQ["checked"]:
        return
    tr = terminalreporter
    tr.write_sep("-", "greedy-token parity")
    tr.write_line(f"first tokens compared: {GREEDY['checked']}, identical: {GREEDY['identical']}, "
                  f"tie-exempt: {len(GREEDY['exempt'])}")
    for e in GREEDY["exempt"]:
        tr.write_line(f"  exempt {e}")
    if SEQ["checked"]:
        tr.write_line(f"bf16 decoded sequences compared: {SEQ['checked']}, diverged after the first token: "
                      f"{len(SEQ['diverged'])}")
        for e in SEQ["diverged"][:20]:
            tr.write_line(f"  {e}")
    if RELS:
        tr.write_line("bf16 logits rel-err vs the reference at Llama-2-7B width (bar 2e-2):")
        for k, v in RELS.items():
            tr.write_line(f"  {k}: {v:.2e}")


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
