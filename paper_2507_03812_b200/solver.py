"""Host-side mirror of the reference ``polarmg::MultigridSolver`` API over the
C ABI of ``include/polarmg_b200.h`` (lib/libpolarmg_b200.so).

The reference surface (multigrid.hpp:86-151) is::

    MultigridSolver(GeometryMap, ProblemCase, PolarGrid, MultigridSettings)
    ConvergenceReport solve();  solution();  num_levels();  grid(l);  op(l) ...

Here the same names take small dataclasses with the reference's field names
and defaults.  There is no CPU fallback: constructing a solver without the
built CUDA library, or without a CUDA device, raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PMG_LIB") or os.path.join(_HERE, "lib", "libpolarmg_b200.so")

PMG_OK, PMG_EINVAL, PMG_ERUNTIME, PMG_ECUDA, PMG_ENOTCONV = 0, 1, 2, 3, 4
LAYOUT_NODE, LAYOUT_CANONICAL = 0, 1

GEOMETRY = {"CirclePolar": 0, "Shafranov": 1, "Czarny": 2}
STENCIL = {"Take": 0, "Give": 1}
CYCLE = {"V": 0, "W": 1, "F": 2}
NORM = {"weighted-l2": 0, "euclidean": 1, "infinity": 2}
BOUNDARY = {"AcrossOrigin": 0, "InteriorDirichlet": 1}

# kernel classes of pmg_time_kernel / pmg_profile_read
KERNEL_KINDS = {"residual": 0, "circle": 1, "radial": 2, "smooth": 3, "restrict": 4,
                "prolongate": 5, "coarse": 6, "norm": 7, "other": 8}


class PmgError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class _Geometry(C.Structure):
    _fields_ = [("kind", C.c_int), ("kappa_eps", C.c_double), ("delta_e", C.c_double),
                ("x0", C.c_double), ("y0", C.c_double)]


class _Problem(C.Structure):
    _fields_ = [("alpha_coeff", C.c_int), ("beta_coeff", C.c_int), ("rmax", C.c_double),
                ("alpha_jump", C.c_double), ("delta_r", C.c_double), ("alpha_scale", C.c_double),
                ("solution", C.c_int)]


class _Grid(C.Structure):
    _fields_ = [("mode", C.c_int), ("R0", C.c_double), ("Rmax", C.c_double), ("n_r", C.c_int),
                ("n_theta", C.c_int), ("nr_exp", C.c_int), ("ntheta_exp", C.c_int),
                ("anisotropic_factor", C.c_int), ("divide_by_2", C.c_int),
                ("radii", C.POINTER(C.c_double)), ("angles", C.POINTER(C.c_double)),
                ("pair_tolerance", C.c_double)]


class _Settings(C.Structure):
    _fields_ = [("stencil_mode", C.c_int), ("boundary_mode", C.c_int), ("cache_profile", C.c_int),
                ("cache_geometry", C.c_int), ("max_levels", C.c_int), ("pre_smoothing", C.c_int),
                ("post_smoothing", C.c_int), ("cycle", C.c_int), ("extrapolation", C.c_int),
                ("fmg", C.c_int), ("fmg_iterations", C.c_int), ("fmg_cycle", C.c_int),
                ("norm_type", C.c_int), ("max_iterations", C.c_int),
                ("absolute_tolerance", C.c_double), ("relative_tolerance", C.c_double),
                ("max_threads", C.c_int), ("verbose", C.c_int), ("reference_order", C.c_int)]


class _Report(C.Structure):
    _fields_ = [("converged", C.c_int), ("iterations", C.c_int), ("fine_cycles_total", C.c_int),
                ("num_residuals", C.c_int), ("reduction_factor_mean", C.c_double),
                ("initial_residual", C.c_double), ("final_residual", C.c_double),
                ("setup_seconds", C.c_double), ("solve_seconds", C.c_double),
                ("device_bytes", C.c_size_t), ("exact_error_weighted", C.c_double),
                ("exact_error_infinity", C.c_double)]


_dp = C.POINTER(C.c_double)
_lib = None

# every symbol include/polarmg_b200.h declares (checked by tests)
EXPORTED = [
    "pmg_last_error", "pmg_version", "pmg_default_settings", "pmg_create", "pmg_create_batch",
    "pmg_destroy", "pmg_grid_hierarchy", "pmg_num_levels", "pmg_num_sections", "pmg_level_info", "pmg_level_grid",
    "pmg_set_rhs", "pmg_get_rhs", "pmg_set_rhs_device", "pmg_seeded_rhs", "pmg_assemble_rhs",
    "pmg_exact_errors", "pmg_solve", "pmg_get_solution",
    "pmg_solution_device", "pmg_apply", "pmg_residual", "pmg_smooth", "pmg_sweep",
    "pmg_restrict", "pmg_prolongate", "pmg_coarse_solve", "pmg_norm", "pmg_launch_count",
    "pmg_time_kernel", "pmg_profile_enable", "pmg_profile_read",
]


def load_library(path: str = LIB_PATH):
    """Loads the CUDA library; raises when it is not built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build the CUDA extension first "
            "(`make -C paper_2507_03812_b200` or __graft_entry__.build()); "
            "there is no CPU fallback")
    lib = C.CDLL(path)
    vp = C.c_void_p
    lib.pmg_last_error.restype = C.c_char_p
    lib.pmg_version.restype = C.c_char_p
    lib.pmg_default_settings.argtypes = [C.POINTER(_Settings)]
    lib.pmg_default_settings.restype = None
    lib.pmg_create.argtypes = [C.POINTER(_Geometry), C.POINTER(_Problem), C.POINTER(_Grid),
                               C.POINTER(_Settings), C.c_int, vp, C.POINTER(vp)]
    lib.pmg_create_batch.argtypes = [C.POINTER(_Geometry), C.POINTER(_Problem), C.POINTER(_Grid),
                                     C.POINTER(_Settings), C.c_int, _dp, C.c_int, vp,
                                     C.POINTER(vp)]
    lib.pmg_destroy.argtypes = [vp]
    lib.pmg_grid_hierarchy.argtypes = [C.POINTER(_Grid), C.c_int, C.c_int, C.POINTER(C.c_int),
                                       C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]
    lib.pmg_num_levels.argtypes = [vp, C.POINTER(C.c_int)]
    lib.pmg_num_sections.argtypes = [vp, C.POINTER(C.c_int)]
    lib.pmg_level_info.argtypes = [vp, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                   C.POINTER(C.c_int)]
    lib.pmg_level_grid.argtypes = [vp, C.c_int, _dp, _dp]
    lib.pmg_set_rhs.argtypes = [vp, _dp, C.c_int]
    lib.pmg_set_rhs_device.argtypes = [vp, vp]
    lib.pmg_get_rhs.argtypes = [vp, _dp, C.c_int]
    lib.pmg_seeded_rhs.argtypes = [vp, C.c_uint, _dp, C.c_int]
    lib.pmg_solve.argtypes = [vp, C.POINTER(_Report), _dp, C.c_int]
    lib.pmg_assemble_rhs.argtypes = [vp]
    lib.pmg_exact_errors.argtypes = [vp, _dp, _dp]
    lib.pmg_get_solution.argtypes = [vp, _dp, C.c_int]
    lib.pmg_solution_device.argtypes = [vp, C.POINTER(vp)]
    lib.pmg_apply.argtypes = [vp, C.c_int, _dp, _dp]
    lib.pmg_residual.argtypes = [vp, C.c_int, _dp, _dp, _dp]
    lib.pmg_smooth.argtypes = [vp, C.c_int, _dp, _dp]
    lib.pmg_sweep.argtypes = [vp, C.c_int, C.c_int, C.c_int, _dp, _dp]
    lib.pmg_restrict.argtypes = [vp, C.c_int, _dp, _dp]
    lib.pmg_prolongate.argtypes = [vp, C.c_int, _dp, _dp, C.c_int]
    lib.pmg_coarse_solve.argtypes = [vp, _dp, _dp]
    lib.pmg_norm.argtypes = [vp, C.c_int, _dp, C.c_long, _dp]
    lib.pmg_launch_count.argtypes = [vp, C.POINTER(C.c_longlong)]
    lib.pmg_time_kernel.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int, _dp]
    lib.pmg_profile_enable.argtypes = [vp, C.c_int]
    lib.pmg_profile_read.argtypes = [vp, C.c_int, _dp, C.POINTER(C.c_longlong)]
    _lib = lib
    return lib


def _check(rc: int):
    if rc != PMG_OK:
        msg = _lib.pmg_last_error().decode()
        if rc == PMG_EINVAL:
            raise ValueError(msg)
        raise PmgError(rc, msg)


def _arr(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a: np.ndarray):
    return a.ctypes.data_as(_dp)


# ----------------------------------------------------------------- inputs
@dataclass
class GeometryMap:
    """GeometryMap(kind, kappa_eps, delta_e, x0, y0) -- geometry.hpp:35-77."""
    kind: str = "Czarny"
    kappa_eps: float = 0.3
    delta_e: float = 1.4
    x0: float = 0.0
    y0: float = 0.0


@dataclass
class ProblemCase:
    """ProblemCase(alpha_coeff, beta_coeff, solution, rmax, alpha_jump, delta_r) --
    problem.hpp:47-94.  ``solution`` "None" (the RHS is supplied: set_rhs / seeded_rhs)
    or "Polar" (PolarOscillation, problem.cpp:48-72: assemble_rhs, FMG, exact errors)."""
    alpha_coeff: str = "Zoni"  # "Poisson" | "Zoni"
    beta_coeff: str = "InverseAlpha"  # "Zero" | "InverseAlpha"
    rmax: float = 1.3
    alpha_jump: float = 0.7
    delta_r: float = 0.05
    alpha_scale: float = 1.0
    solution: str = "None"  # "None" | "Polar"


@dataclass
class PolarGrid:
    """Grid recipe: ``uniform(R0, Rmax, n_r, n_theta)`` (polar_grid.cpp:99-113),
    ``build(R0, Rmax, nr_exp, ntheta_exp, anisotropic_factor, divideBy2)``
    (polar_grid.cpp:131-178) or explicit radii/angles."""
    mode: int = 0
    R0: float = 1e-5
    Rmax: float = 1.3
    n_r: int = 0
    n_theta: int = 0
    nr_exp: int = 0
    ntheta_exp: int = 0
    anisotropic_factor: int = 0
    divide_by_2: int = 0
    radii: Optional[np.ndarray] = None
    angles: Optional[np.ndarray] = None
    pair_tolerance: float = 1e-12

    @staticmethod
    def uniform(R0: float, Rmax: float, n_r: int, n_theta: int, pair_tolerance: float = 1e-12):
        return PolarGrid(0, R0, Rmax, n_r, n_theta, pair_tolerance=pair_tolerance)

    @staticmethod
    def build(R0: float, Rmax: float, nr_exp: int, ntheta_exp: int, anisotropic_factor: int = 0,
              divide_by_2: int = 0, pair_tolerance: float = 1e-12):
        return PolarGrid(1, R0, Rmax, 0, 0, nr_exp, ntheta_exp, anisotropic_factor, divide_by_2,
                         pair_tolerance=pair_tolerance)

    @staticmethod
    def explicit(radii: Sequence[float], angles: Sequence[float], pair_tolerance: float = 1e-12):
        r, a = _arr(radii), _arr(angles)
        return PolarGrid(2, float(r[0]), float(r[-1]), len(r), len(a), radii=r, angles=a,
                         pair_tolerance=pair_tolerance)


@dataclass
class MultigridSettings:
    """MultigridSettings -- multigrid.hpp:32-51 (same names and defaults)."""
    stencil_mode: str = "Take"
    boundary_mode: str = "AcrossOrigin"
    cache_profile: bool = True
    cache_geometry: bool = False
    max_levels: int = 0
    pre_smoothing: int = 1
    post_smoothing: int = 1
    cycle: str = "V"
    extrapolation: bool = False
    fmg: bool = False
    fmg_iterations: int = 2
    fmg_cycle: str = "F"
    norm_type: str = "weighted-l2"
    max_iterations: int = 150
    absolute_tolerance: float = -1.0
    relative_tolerance: float = 1e-8
    max_threads: int = 0
    verbose: bool = False
    # extension: line solves reproduce the reference's sequential substitution
    # bit for bit (default; False = faster chunked scans, roundoff-level drift)
    reference_order: bool = True


@dataclass
class ConvergenceReport:
    """ConvergenceReport -- multigrid.hpp:55-68."""
    converged: bool = False
    iterations: int = 0
    fine_cycles_total: int = 0
    residual_norms: List[float] = field(default_factory=list)
    reduction_factor_mean: float = 0.0
    setup_seconds: float = 0.0
    solve_seconds: float = 0.0  # device time (CUDA events) of the solve window
    device_bytes: int = 0
    exact_error_weighted: float = -1.0  # -1 without a manufactured solution
    exact_error_infinity: float = -1.0


def _grid_struct(grid: "PolarGrid", keep: list):
    gr = _Grid(grid.mode, grid.R0, grid.Rmax, grid.n_r, grid.n_theta, grid.nr_exp,
               grid.ntheta_exp, grid.anisotropic_factor, grid.divide_by_2, None, None,
               grid.pair_tolerance)
    if grid.mode == 2:
        r, a = _arr(grid.radii), _arr(grid.angles)
        keep += [r, a]
        gr.radii, gr.angles = _p(r), _p(a)
    return gr


def grid_hierarchy(grid: "PolarGrid", max_levels: int = 0):
    """[(n_r, n_theta, split), ...] of the level chain (host only, no GPU)."""
    lib = load_library()
    keep: list = []
    gr = _grid_struct(grid, keep)
    cap = 64
    L = C.c_int()
    nr, nt, sp = (C.c_int * cap)(), (C.c_int * cap)(), (C.c_int * cap)()
    _check(lib.pmg_grid_hierarchy(C.byref(gr), max_levels, cap, C.byref(L), nr, nt, sp))
    return [(nr[i], nt[i], sp[i]) for i in range(min(L.value, cap))]


def _lookup(table, key, what):
    if isinstance(key, int):
        return key
    if key not in table:
        raise ValueError(f"unknown {what} '{key}'")
    return table[key]


class MultigridSolver:
    """B200 drop-in for ``polarmg::MultigridSolver`` (one or a batch of sections).

    ``n_sections > 1`` builds one batched solver over independent problems that
    share the grid (config 3), section i with alpha scaled by ``alpha_scales[i]``.
    """

    def __init__(self, geometry: GeometryMap, problem: ProblemCase, grid: PolarGrid,
                 settings: MultigridSettings, n_sections: int = 1,
                 alpha_scales: Optional[Sequence[float]] = None, device: int = 0,
                 stream: Optional[int] = None):
        self._lib = load_library()
        self.settings = settings
        g = _Geometry(_lookup(GEOMETRY, geometry.kind, "geometry"), geometry.kappa_eps,
                      geometry.delta_e, geometry.x0, geometry.y0)
        p = _Problem({"Poisson": 0, "Zoni": 1}[problem.alpha_coeff] if isinstance(
            problem.alpha_coeff, str) else problem.alpha_coeff,
            {"Zero": 0, "InverseAlpha": 1}[problem.beta_coeff] if isinstance(
                problem.beta_coeff, str) else problem.beta_coeff,
            problem.rmax, problem.alpha_jump, problem.delta_r, problem.alpha_scale,
            _lookup({"None": 0, "Polar": 1, "PolarOscillation": 1}, problem.solution, "problem"))
        self._keep = []
        gr = _grid_struct(grid, self._keep)
        s = _Settings(_lookup(STENCIL, settings.stencil_mode, "stencilDistributionMethod"),
                      _lookup(BOUNDARY, settings.boundary_mode, "boundary mode"),
                      int(settings.cache_profile), int(settings.cache_geometry),
                      settings.max_levels, settings.pre_smoothing, settings.post_smoothing,
                      _lookup(CYCLE, settings.cycle, "cycle type"), int(settings.extrapolation),
                      int(settings.fmg), settings.fmg_iterations,
                      _lookup(CYCLE, settings.fmg_cycle, "cycle type"),
                      _lookup(NORM, settings.norm_type, "residualNormType"),
                      settings.max_iterations, settings.absolute_tolerance,
                      settings.relative_tolerance, settings.max_threads, int(settings.verbose),
                      int(settings.reference_order))
        h = C.c_void_p()
        scales = None
        if alpha_scales is not None:
            sc = _arr(alpha_scales)
            if len(sc) != n_sections:
                raise ValueError("alpha_scales must have n_sections entries")
            self._keep.append(sc)
            scales = _p(sc)
        _check(self._lib.pmg_create_batch(C.byref(g), C.byref(p), C.byref(gr), C.byref(s),
                                          n_sections, scales, device,
                                          C.c_void_p(stream) if stream else None, C.byref(h)))
        self._h = h
        nl = C.c_int()
        _check(self._lib.pmg_num_levels(self._h, C.byref(nl)))
        self._levels = [self._level_info(l) for l in range(nl.value)]
        self.n_sections = n_sections
        self._last_report: Optional[List[ConvergenceReport]] = None

    # -- lifetime
    def close(self):
        if getattr(self, "_h", None):
            self._lib.pmg_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- hierarchy inspection (multigrid.hpp:99-108)
    def _level_info(self, level):
        nr, nt, sp = C.c_int(), C.c_int(), C.c_int()
        _check(self._lib.pmg_level_info(self._h, level, C.byref(nr), C.byref(nt), C.byref(sp)))
        return nr.value, nt.value, sp.value

    def num_levels(self) -> int:
        return len(self._levels)

    def level_shape(self, level: int = 0):
        """(n_r, n_theta, split) of a level."""
        return self._levels[level]

    def grid(self, level: int = 0):
        nr, nt, _ = self._levels[level]
        r, a = np.zeros(nr), np.zeros(nt)
        _check(self._lib.pmg_level_grid(self._h, level, _p(r), _p(a)))
        return r, a

    def n(self, level: int = 0) -> int:
        nr, nt, _ = self._levels[level]
        return nr * nt

    # -- right-hand side and solve
    def set_rhs(self, f, layout: int = LAYOUT_NODE):
        f = _arr(f)
        if f.size != self.n_sections * self.n(0):
            raise ValueError("rhs has the wrong size")
        _check(self._lib.pmg_set_rhs(self._h, _p(f), layout))

    def get_rhs(self, layout: int = LAYOUT_NODE) -> np.ndarray:
        f = np.zeros(self.n_sections * self.n(0))
        _check(self._lib.pmg_get_rhs(self._h, _p(f), layout))
        return f

    def set_rhs_device(self, ptr: int):
        _check(self._lib.pmg_set_rhs_device(self._h, C.c_void_p(ptr)))

    def seeded_rhs(self, seed: int, layout: int = LAYOUT_NODE, return_ustar: bool = False):
        """u* ~ U(-1,1) from std::mt19937(seed + section); f = A_take u* on the device."""
        us = np.zeros(self.n_sections * self.n(0)) if return_ustar else None
        _check(self._lib.pmg_seeded_rhs(self._h, seed, _p(us) if us is not None else None,
                                        layout))
        return us

    def solve(self) -> ConvergenceReport:
        """MultigridSolver::solve() (multigrid.cpp:298-357) on the current RHS.
        Returns the report of section 0; all sections in ``reports``."""
        reps = (_Report * self.n_sections)()
        cap = self.settings.max_iterations + 1
        hist = np.zeros(self.n_sections * cap)
        rc = self._lib.pmg_solve(self._h, reps, _p(hist), cap)
        if rc not in (PMG_OK, PMG_ENOTCONV):
            _check(rc)
        out = []
        for b in range(self.n_sections):
            r = reps[b]
            out.append(ConvergenceReport(
                converged=bool(r.converged), iterations=r.iterations,
                fine_cycles_total=r.fine_cycles_total,
                residual_norms=list(hist[b * cap: b * cap + r.num_residuals]),
                reduction_factor_mean=r.reduction_factor_mean, setup_seconds=r.setup_seconds,
                solve_seconds=r.solve_seconds, device_bytes=int(r.device_bytes),
                exact_error_weighted=r.exact_error_weighted,
                exact_error_infinity=r.exact_error_infinity))
        self._last_report = out
        return out[0]

    def assemble_rhs(self):
        """f = DiscreteOperator::assemble_rhs of the finest level (stencil.cpp:307-353),
        on the device; then solve() is the reference's MultigridSolver::solve()."""
        _check(self._lib.pmg_assemble_rhs(self._h))

    def exact_errors(self):
        """MultigridSolver::exact_errors() (multigrid.cpp:277-296) per section."""
        w = np.zeros(self.n_sections)
        inf = np.zeros(self.n_sections)
        _check(self._lib.pmg_exact_errors(self._h, _p(w), _p(inf)))
        return w, inf

    @property
    def reports(self) -> List[ConvergenceReport]:
        return self._last_report or []

    def solution(self, layout: int = LAYOUT_NODE) -> np.ndarray:
        u = np.zeros(self.n_sections * self.n(0))
        _check(self._lib.pmg_get_solution(self._h, _p(u), layout))
        return u

    def solution_device_ptr(self) -> int:
        p = C.c_void_p()
        _check(self._lib.pmg_solution_device(self._h, C.byref(p)))
        return p.value

    # -- operator seams (stencil.hpp:108-113, smoother.hpp:51-53, interpolation.hpp:27-36)
    def apply(self, u, level: int = 0):
        u = _arr(u)
        y = np.zeros_like(u)
        _check(self._lib.pmg_apply(self._h, level, _p(u), _p(y)))
        return y

    def residual(self, u, f, level: int = 0):
        u, f = _arr(u), _arr(f)
        r = np.zeros_like(u)
        _check(self._lib.pmg_residual(self._h, level, _p(u), _p(f), _p(r)))
        return r

    def smooth(self, u, f, level: int = 0):
        u = np.array(u, dtype=np.float64, copy=True)
        _check(self._lib.pmg_smooth(self._h, level, _p(u), _p(_arr(f))))
        return u

    def sweep(self, u, f, kind: int, parity: int, level: int = 0):
        u = np.array(u, dtype=np.float64, copy=True)
        _check(self._lib.pmg_sweep(self._h, level, kind, parity, _p(u), _p(_arr(f))))
        return u

    def restrict(self, fine, level: int = 0):
        fine = _arr(fine)
        c = np.zeros(self.n_sections * self.n(level + 1))
        _check(self._lib.pmg_restrict(self._h, level, _p(fine), _p(c)))
        return c

    def prolongate(self, coarse, fine=None, level: int = 0, add: bool = False):
        out = np.zeros(self.n_sections * self.n(level)) if fine is None else np.array(
            fine, dtype=np.float64, copy=True)
        _check(self._lib.pmg_prolongate(self._h, level, _p(_arr(coarse)), _p(out), int(add)))
        return out

    def coarse_solve(self, f):
        u = np.zeros(self.n_sections * self.n(self.num_levels() - 1))
        _check(self._lib.pmg_coarse_solve(self._h, _p(_arr(f)), _p(u)))
        return u

    def norm(self, v, norm_type: str = "weighted-l2") -> float:
        v = _arr(v)
        out = C.c_double()
        _check(self._lib.pmg_norm(self._h, NORM[norm_type], _p(v), v.size, C.byref(out)))
        return out.value

    # -- measurement
    def launch_count(self) -> int:
        c = C.c_longlong()
        _check(self._lib.pmg_launch_count(self._h, C.byref(c)))
        return c.value

    def time_kernel(self, kind: str, level: int = 0, reps: int = 10, flush_l2: bool = True) -> float:
        ms = C.c_double()
        _check(self._lib.pmg_time_kernel(self._h, KERNEL_KINDS[kind], level, reps, int(flush_l2),
                                         C.byref(ms)))
        return ms.value

    def profile(self, on: bool):
        _check(self._lib.pmg_profile_enable(self._h, int(on)))

    def profile_read(self, kind: str):
        ms, n = C.c_double(), C.c_longlong()
        _check(self._lib.pmg_profile_read(self._h, KERNEL_KINDS[kind], C.byref(ms), C.byref(n)))
        return ms.value, n.value
