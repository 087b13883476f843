"""The five BASELINE.json configurations as solver inputs.

Common: R0 = 1e-5, Rmax = 1.3, AcrossOrigin, Dirichlet u = 0 on ring n_r-1,
alpha = exp(-tanh((r/1.3 - 0.5)/0.1)) (Zoni, r_p = 0.5, delta_r = 0.1),
V(1,1), weighted-l2 norm, relative tolerance 1e-10, max 200 cycles, u0 = 0.
Seeded u* ~ U(-1,1) from std::mt19937(20240611 [+ section]); f = A_take u*.
"""
from __future__ import annotations

import numpy as np

from .solver import GeometryMap, MultigridSettings, PolarGrid, ProblemCase

SEED = 20240611


def baseline_config(k: int, **settings_over):
    """Returns (geometry, problem, grid, settings, meta) of BASELINE config k."""
    prob = ProblemCase("Zoni", "InverseAlpha", rmax=1.3, alpha_jump=0.5, delta_r=0.1)
    st = MultigridSettings(stencil_mode="Take", cycle="V", relative_tolerance=1e-10,
                           max_iterations=200)
    meta = {"n_sections": 1}
    if k == 0:
        geom = GeometryMap("CirclePolar", 0.0, 0.0)
        prob.beta_coeff = "Zero"
        grid = PolarGrid.uniform(1e-5, 1.3, 257, 256)
        st.stencil_mode = "Give"
    elif k == 1:
        geom = GeometryMap("Shafranov", 0.3, 0.2)
        grid = PolarGrid.uniform(1e-5, 1.3, 1025, 1024)
    elif k == 2:
        geom = GeometryMap("Czarny", 0.3, 1.4)
        # PolarGrid::uniform(1e-5,1.3,4097,4096) fails the reference's 1e-12
        # pairing check: use the divideBy2 route.
        grid = PolarGrid.build(1e-5, 1.3, 8, 8, 0, 4)
    elif k == 3:
        geom = GeometryMap("Shafranov", 0.3, 0.2)
        grid = PolarGrid.uniform(1e-5, 1.3, 513, 512)
        meta["n_sections"] = 256
    elif k == 4:
        geom = GeometryMap("Czarny", 0.3, 1.4)
        # 8193x8192 needs a roundoff-scaled pairing tolerance
        grid = PolarGrid.uniform(1e-5, 1.3, 8193, 8192, pair_tolerance=1e-9)
    else:
        raise ValueError(f"unknown config {k}")
    for key, v in settings_over.items():
        setattr(st, key, v)
    return geom, prob, grid, st, meta


def section_scales(n_sections: int = 256, seed: int = SEED + 1000003) -> np.ndarray:
    """Config 3 alpha scales c_i ~ U(0.5, 2): std::mt19937(seed) with
    libstdc++ uniform_real_distribution<double> (generate_canonical<double,53>:
    two 32-bit draws per value), in section order."""
    rs = np.random.RandomState(seed)
    raw = rs.randint(0, 2**32, size=2 * n_sections, dtype=np.uint32).astype(np.float64)
    c = (raw[0::2] + raw[1::2] * 4294967296.0) / 18446744073709551616.0
    c = np.where(c >= 1.0, np.nextafter(1.0, 0.0), c)
    return c * 1.5 + 0.5
