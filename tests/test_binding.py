"""The C++ drop-in binding of INTEGRATION.md (include/polarmg_b200.hpp),
compiled against the reference's own headers and driven next to a reference
polarmg::MultigridSolver by tests/binding_demo.cpp (oracle/_ref/binding_demo,
built by `make -C oracle binding` / __graft_entry__.build()).
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEMO = os.path.join(ROOT, "oracle", "_ref", "binding_demo")


@pytest.mark.skipif(not os.path.isdir("/root/reference/proj/core/include"),
                    reason="reference headers only exist in the build container")
def test_binding_compiles():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "binding"], check=True)
    assert os.access(DEMO, os.X_OK)


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(DEMO), reason="binding_demo not built")
def test_binding_solves_bitwise():
    """Manufactured problems (Take V/W, Give V, FMG + extrapolation) solved by
    the reference and by the B200 library through the binding: same cycle
    counts, Take solutions bitwise, Give within 1e-10."""
    out = subprocess.run([DEMO], capture_output=True, text=True, timeout=600)
    print(out.stdout, out.stderr)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "all ok" in out.stdout
