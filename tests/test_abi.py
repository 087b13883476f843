"""C ABI checks that need no GPU: the library loads, exports every symbol
include/polarmg_b200.h declares, its struct layouts match the ctypes mirror,
the host-only hierarchy logic reproduces the reference, and device entry
points fail loudly (status + message, no crash) when no GPU is present."""
import ctypes as C
import os
import re
import subprocess
import tempfile

import numpy as np
import pytest

from conftest import ROOT
import paper_2507_03812_b200 as pmg
from paper_2507_03812_b200 import solver as S
from oracle.oracle import OracleSolver, config_case, Case

HEADER = os.path.join(ROOT, "include", "polarmg_b200.h")


def declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(pmg_[a-z_]+)\s*\(", txt)))


def test_exports_every_declared_symbol():
    lib = pmg.load_library()
    names = declared()
    assert len(names) >= 25
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(S.EXPORTED) == names


def test_struct_layout_matches_header():
    src = r'''
#include <stdio.h>
#include <stddef.h>
#include "polarmg_b200.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu\n", sizeof(pmg_geometry), sizeof(pmg_problem), sizeof(pmg_grid),
         sizeof(pmg_settings), sizeof(pmg_report));
  printf("%zu %zu %zu\n", offsetof(pmg_grid, pair_tolerance), offsetof(pmg_settings, reference_order),
         offsetof(pmg_report, device_bytes));
  return 0;
}'''
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "t.c")
        open(c, "w").write(src)
        exe = os.path.join(d, "t")
        subprocess.run(["gcc", "-I", os.path.dirname(HEADER), c, "-o", exe], check=True)
        out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split()
    sizes = [int(x) for x in out]
    assert sizes[:5] == [C.sizeof(S._Geometry), C.sizeof(S._Problem), C.sizeof(S._Grid),
                         C.sizeof(S._Settings), C.sizeof(S._Report)]
    assert sizes[5:] == [S._Grid.pair_tolerance.offset, S._Settings.reference_order.offset,
                         S._Report.device_bytes.offset]


def test_default_settings_are_the_reference_defaults():
    lib = pmg.load_library()
    st = S._Settings()
    lib.pmg_default_settings(C.byref(st))
    ref = pmg.MultigridSettings()  # multigrid.hpp:32-51 defaults
    assert st.pre_smoothing == ref.pre_smoothing == 1
    assert st.max_iterations == ref.max_iterations == 150
    assert st.relative_tolerance == ref.relative_tolerance == 1e-8
    assert st.absolute_tolerance == ref.absolute_tolerance == -1.0
    assert st.fmg_iterations == 2 and st.cycle == 0 and st.reference_order == 1


@pytest.mark.parametrize("k", [0, 1, 2, 3])
def test_host_hierarchy_matches_reference(k):
    geom, prob, grid, st, _ = pmg.baseline_config(k)
    levels = pmg.grid_hierarchy(grid)
    O = OracleSolver(config_case(k, max_iterations=0))
    assert levels == [tuple(x) for x in O.levels]


def test_config4_hierarchy():
    _, _, grid, _, _ = pmg.baseline_config(4)
    lv = pmg.grid_hierarchy(grid)
    assert len(lv) == 12 and lv[0] == (8193, 8192, 1304) and lv[-1][:2] == (5, 4)


def test_grid_errors():
    with pytest.raises(ValueError, match="radial spacings violate the pairing constraint"):
        pmg.grid_hierarchy(pmg.PolarGrid.uniform(1e-5, 1.3, 4097, 4096))
    with pytest.raises(ValueError, match="inner radius must be positive"):
        pmg.grid_hierarchy(pmg.PolarGrid.uniform(0.0, 1.3, 17, 16))


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU failure path")
def test_create_fails_loudly_without_gpu():
    geom, prob, grid, st, _ = pmg.baseline_config(0)
    with pytest.raises((pmg.PmgError, ValueError)) as ei:
        pmg.MultigridSolver(geom, prob, grid, st)
    assert "CUDA" in str(ei.value) or "device" in str(ei.value)


def test_invalid_settings_rejected_before_device():
    geom, prob, grid, st, _ = pmg.baseline_config(0)
    st.extrapolation = True
    st.max_levels = 1  # config.cpp:179-181
    with pytest.raises(ValueError, match="extrapolation requires at least two levels"):
        pmg.MultigridSolver(geom, prob, grid, st)
    st.extrapolation = False
    st.max_levels = 0
    st.fmg_iterations = 0  # config.cpp:175-176
    with pytest.raises(ValueError, match="FMG_iterations"):
        pmg.MultigridSolver(geom, prob, grid, st)
    st.fmg_iterations = 2
    st.pre_smoothing = -1
    with pytest.raises(ValueError, match="preSmoothingSteps"):
        pmg.MultigridSolver(geom, prob, grid, st)
