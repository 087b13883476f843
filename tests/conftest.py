import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def _ensure_built():
    """Builds the oracle libraries and the CUDA library when missing (the
    GPU box receives prebuilt files; /root/reference only exists here)."""
    oracle_lib = os.path.join(ROOT, "oracle", "_ref", "liboracle.so")
    ref_lib = os.path.join(ROOT, "oracle", "_ref", "libpolarmg_ref.so")
    cuda_lib = os.path.join(ROOT, "paper_2507_03812_b200", "lib", "libpolarmg_b200.so")
    if not os.path.exists(oracle_lib):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "oracle"], check=True)
    if not os.path.exists(ref_lib) and os.path.isdir("/root/reference/proj/core"):
        subprocess.run(["make", "-j8", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)
    if not os.path.exists(cuda_lib):
        subprocess.run(["make", "-j4", "-C", os.path.join(ROOT, "paper_2507_03812_b200")],
                       check=True)


_ensure_built()


def have_ref():
    return os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libpolarmg_ref.so"))


requires_ref = pytest.mark.skipif(not have_ref(), reason="oracle/_ref not built")
