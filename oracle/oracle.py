"""TEST INFRASTRUCTURE ONLY -- ctypes front-ends of the two CPU checkers.

* ``RefSolver``    -> oracle/_ref/libpolarmg_ref.so, the unmodified reference
  polarmg core (+ ref_shim.cpp).  Used to pin the C restatement, to generate
  the committed golden fixtures, and as bench.py's CPU baseline.
* ``OracleSolver`` -> oracle/_ref/liboracle.so, the plain-C restatement in
  polarmg_oracle.c (each function cites the reference file:line it follows).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module.  The product package
(paper_2507_03812_b200) never does.

All vectors are in the reference's NodeIndexing order (polar_grid.hpp:17-37)
unless a function says otherwise.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
REF_LIB = os.path.join(_HERE, "_ref", "libpolarmg_ref.so")
ORACLE_LIB = os.path.join(_HERE, "_ref", "liboracle.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)

GEOMETRY = {"CirclePolar": 0, "Shafranov": 1, "Czarny": 2}
MODE = {"Take": 0, "Give": 1}
CYCLE = {"V": 0, "W": 1, "F": 2}
NORM = {"weighted-l2": 0, "euclidean": 1, "infinity": 2}


def _ptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_dp)


@dataclass
class Case:
    """One solver configuration (the BASELINE.json config vocabulary)."""

    geometry: str = "Czarny"
    kappa_eps: float = 0.3
    delta_e: float = 1.4
    alpha_coeff: int = 1  # 0 Poisson, 1 Zoni
    beta_coeff: int = 1  # 0 Zero, 1 InverseAlpha
    rmax: float = 1.3
    alpha_jump: float = 0.5
    delta_r: float = 0.1
    alpha_scale: float = 1.0
    grid_mode: int = 0  # 0 uniform(R0,Rmax,a,b); 1 build_grid(nr_exp=a, ntheta_exp=b)
    R0: float = 1e-5
    a: int = 17
    b: int = 16
    aniso: int = 0
    divide_by_2: int = 0
    pair_tol: float = 1e-12
    stencil_mode: str = "Take"
    boundary_mode: int = 0  # 0 AcrossOrigin, 1 InteriorDirichlet
    max_levels: int = 0
    pre: int = 1
    post: int = 1
    cycle: str = "V"
    norm_type: str = "weighted-l2"
    max_iterations: int = 200
    abs_tol: float = -1.0
    rel_tol: float = 1e-10
    threads: int = 0
    solution: int = 0  # 0 None, 1 PolarOscillation (problem.hpp:32-44)
    fmg: int = 0
    fmg_iterations: int = 2
    fmg_cycle: str = "F"
    extrapolation: int = 0
    extra: dict = field(default_factory=dict)

    def args(self):
        return (
            GEOMETRY[self.geometry], self.kappa_eps, self.delta_e,
            self.alpha_coeff, self.beta_coeff, self.rmax, self.alpha_jump,
            self.delta_r, self.alpha_scale, self.grid_mode, self.R0, self.a,
            self.b, self.aniso, self.divide_by_2, self.pair_tol,
            MODE[self.stencil_mode], self.boundary_mode, self.max_levels,
            self.pre, self.post, CYCLE[self.cycle], NORM[self.norm_type],
            self.max_iterations, self.abs_tol, self.rel_tol, self.threads,
        )


_CREATE_ARGTYPES = [
    C.c_int, C.c_double, C.c_double, C.c_int, C.c_int, C.c_double, C.c_double,
    C.c_double, C.c_double, C.c_int, C.c_double, C.c_int, C.c_int, C.c_int,
    C.c_int, C.c_double, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
    C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, C.POINTER(C.c_void_p),
]


def _bind(lib, prefix):
    getattr(lib, prefix + "last_error").restype = C.c_char_p
    getattr(lib, prefix + "create").argtypes = _CREATE_ARGTYPES
    getattr(lib, prefix + "destroy").argtypes = [C.c_void_p]
    getattr(lib, prefix + "num_levels").argtypes = [C.c_void_p]
    getattr(lib, prefix + "level_info").argtypes = [C.c_void_p, C.c_int, _ip, _ip, _ip]
    getattr(lib, prefix + "level_grid").argtypes = [C.c_void_p, C.c_int, _dp, _dp]
    getattr(lib, prefix + "apply").argtypes = [C.c_void_p, C.c_int, C.c_int, _dp, _dp]
    getattr(lib, prefix + "residual").argtypes = [C.c_void_p, C.c_int, C.c_int, _dp, _dp, _dp]
    getattr(lib, prefix + "smooth").argtypes = [C.c_void_p, C.c_int, _dp, _dp]
    getattr(lib, prefix + "sweep").argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, _dp, _dp]
    getattr(lib, prefix + "restrict").argtypes = [C.c_void_p, C.c_int, _dp, _dp]
    getattr(lib, prefix + "prolongate").argtypes = [C.c_void_p, C.c_int, _dp, _dp, C.c_int]
    getattr(lib, prefix + "coarse_solve").argtypes = [C.c_void_p, _dp, _dp]
    getattr(lib, prefix + "seeded_field").argtypes = [C.c_void_p, C.c_uint, _dp]
    getattr(lib, prefix + "solve").argtypes = [C.c_void_p, _dp, _dp, _dp, _ip, _ip, _dp, _dp]
    getattr(lib, prefix + "row").argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, _ip, _dp, _ip]
    getattr(lib, prefix + "level_coeffs").argtypes = [C.c_void_p, C.c_int, _dp, _dp, _dp, _dp, _dp, _dp]
    getattr(lib, prefix + "set_extra").argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int]
    getattr(lib, prefix + "assemble_rhs").argtypes = [C.c_void_p, C.c_int, _dp]
    getattr(lib, prefix + "exact_errors").argtypes = [C.c_void_p, _dp, _dp, _dp]
    native = [C.c_void_p, _dp, _dp, _ip, _ip, _ip, _dp, _dp, _dp]
    getattr(lib, prefix + "solve_native").argtypes = native + ([_dp] if prefix == "ref_" else [])


_LIBS: dict = {}


def _load(path, prefix):
    if path not in _LIBS:
        if not os.path.exists(path):
            raise FileNotFoundError(
                f"{path} is not built; run `make -C oracle` (or __graft_entry__.build())")
        lib = C.CDLL(path)
        _bind(lib, prefix)
        _LIBS[path] = lib
    return _LIBS[path]


class _Solver:
    """Common driver of the reference shim and the C restatement (same ABI)."""

    _path = ""
    _prefix = ""

    def __init__(self, case: Case):
        self.lib = _load(self._path, self._prefix)
        self.case = case
        h = C.c_void_p()
        self._fn("set_extra")(case.solution, case.fmg, case.fmg_iterations, CYCLE[case.fmg_cycle],
                              case.extrapolation)
        self._check(self._fn("create")(*case.args(), C.byref(h)))
        self.h = h
        self.num_levels = self._fn("num_levels")(self.h)
        self.levels = [self.level_info(l) for l in range(self.num_levels)]

    def _fn(self, name):
        return getattr(self.lib, self._prefix + name)

    def _check(self, rc):
        if rc != 0:
            msg = self._fn("last_error")().decode()
            raise (ValueError if rc == 1 else RuntimeError)(msg)

    def __del__(self):
        if getattr(self, "h", None):
            self._fn("destroy")(self.h)
            self.h = None

    def level_info(self, level):
        nr, nt, sp = C.c_int(), C.c_int(), C.c_int()
        self._check(self._fn("level_info")(self.h, level, C.byref(nr), C.byref(nt), C.byref(sp)))
        return nr.value, nt.value, sp.value

    def n(self, level=0):
        nr, nt, _ = self.levels[level]
        return nr * nt

    def level_grid(self, level=0):
        nr, nt, _ = self.levels[level]
        r, a = np.zeros(nr), np.zeros(nt)
        self._check(self._fn("level_grid")(self.h, level, _ptr(r), _ptr(a)))
        return r, a

    def level_coeffs(self, level=0):
        nr, nt, _ = self.levels[level]
        arrs = [np.zeros(nr * nt) for _ in range(4)]
        al, be = np.zeros(nr), np.zeros(nr)
        self._check(self._fn("level_coeffs")(self.h, level, *[_ptr(x) for x in arrs], _ptr(al), _ptr(be)))
        return arrs + [al, be]

    def row(self, level, s, t):
        cols = (C.c_int * 10)()
        vals = (C.c_double * 10)()
        cnt = C.c_int()
        self._check(self._fn("row")(self.h, level, s, t, cols, vals, C.byref(cnt)))
        return list(cols[: cnt.value]), list(vals[: cnt.value])

    def apply(self, u, level=0, mode=None):
        y = np.zeros(self.n(level))
        m = MODE[mode or self.case.stencil_mode]
        self._check(self._fn("apply")(self.h, level, m, _ptr(np.ascontiguousarray(u, np.float64)), _ptr(y)))
        return y

    def residual(self, u, f, level=0, mode=None):
        r = np.zeros(self.n(level))
        m = MODE[mode or self.case.stencil_mode]
        self._check(self._fn("residual")(self.h, level, m, _ptr(np.ascontiguousarray(u, np.float64)),
                                          _ptr(np.ascontiguousarray(f, np.float64)), _ptr(r)))
        return r

    def smooth(self, u, f, level=0):
        u = np.array(u, dtype=np.float64, copy=True)
        self._check(self._fn("smooth")(self.h, level, _ptr(u), _ptr(np.ascontiguousarray(f, np.float64))))
        return u

    def sweep(self, u, f, kind, parity, level=0):
        """kind 0 = circle sweep, 1 = radial sweep (smoother.cpp:95-142)."""
        u = np.array(u, dtype=np.float64, copy=True)
        self._check(self._fn("sweep")(self.h, level, kind, parity, _ptr(u),
                                       _ptr(np.ascontiguousarray(f, np.float64))))
        return u

    def restrict(self, fine, level=0):
        c = np.zeros(self.n(level + 1))
        self._check(self._fn("restrict")(self.h, level, _ptr(np.ascontiguousarray(fine, np.float64)), _ptr(c)))
        return c

    def prolongate(self, coarse, fine=None, level=0, add=False):
        out = np.zeros(self.n(level)) if fine is None else np.array(fine, dtype=np.float64, copy=True)
        self._check(self._fn("prolongate")(self.h, level, _ptr(np.ascontiguousarray(coarse, np.float64)),
                                            _ptr(out), 1 if add else 0))
        return out

    def coarse_solve(self, f):
        u = np.zeros(self.n(self.num_levels - 1))
        self._check(self._fn("coarse_solve")(self.h, _ptr(np.ascontiguousarray(f, np.float64)), _ptr(u)))
        return u

    def seeded_field(self, seed):
        u = np.zeros(self.n(0))
        self._check(self._fn("seeded_field")(self.h, seed, _ptr(u)))
        return u

    def seeded_rhs(self, seed):
        """u* ~ U(-1,1) (mt19937(seed), canonical order, outer ring 0); f = A_take u*."""
        ustar = self.seeded_field(seed)
        return ustar, self.apply(ustar, 0, "Take")

    def solve(self, f):
        n = self.n(0)
        u = np.zeros(n)
        hist = np.zeros(self.case.max_iterations + 1)
        it, conv = C.c_int(), C.c_int()
        red, sec = C.c_double(), C.c_double()
        self._check(self._fn("solve")(self.h, _ptr(np.ascontiguousarray(f, np.float64)), _ptr(u),
                                       _ptr(hist), C.byref(it), C.byref(conv), C.byref(red), C.byref(sec)))
        return {
            "u": u,
            "iterations": it.value,
            "converged": bool(conv.value),
            "residual_norms": hist[: it.value + 1].copy(),
            "reduction_factor_mean": red.value,
            "seconds": sec.value,
        }


    def assemble_rhs(self, level=0):
        """DiscreteOperator::assemble_rhs (stencil.cpp:326-353) of a level."""
        b = np.zeros(self.n(level))
        self._check(self._fn("assemble_rhs")(self.h, level, _ptr(b)))
        return b

    def exact_errors(self, u):
        w, inf = C.c_double(), C.c_double()
        self._check(self._fn("exact_errors")(self.h, _ptr(np.ascontiguousarray(u, np.float64)),
                                              C.byref(w), C.byref(inf)))
        return w.value, inf.value

    def solve_native(self):
        """MultigridSolver::solve() itself (multigrid.cpp:298-357)."""
        u = np.zeros(self.n(0))
        hist = np.zeros(self.case.max_iterations + 1)
        it, fc, conv = C.c_int(), C.c_int(), C.c_int()
        red, ew, ei, sec = C.c_double(), C.c_double(), C.c_double(), C.c_double()
        args = [self.h, _ptr(u), _ptr(hist), C.byref(it), C.byref(fc), C.byref(conv),
                C.byref(red), C.byref(ew), C.byref(ei)]
        if self._prefix == "ref_":
            args.append(C.byref(sec))
        self._check(self._fn("solve_native")(*args))
        return {
            "u": u,
            "iterations": it.value,
            "fine_cycles_total": fc.value,
            "converged": bool(conv.value),
            "residual_norms": hist[: it.value + 1].copy(),
            "reduction_factor_mean": red.value,
            "exact_error_weighted": ew.value,
            "exact_error_infinity": ei.value,
        }


class RefSolver(_Solver):
    _path = REF_LIB
    _prefix = "ref_"


class OracleSolver(_Solver):
    _path = ORACLE_LIB
    _prefix = "orc_"


def canonical_to_node(split: int, nr: int, nt: int) -> np.ndarray:
    """perm[c] = NodeIndexing index of canonical node c = s*nt + t."""
    s = np.repeat(np.arange(nr), nt)
    t = np.tile(np.arange(nt), nr)
    return np.where(s < split, s * nt + t, split * nt + t * (nr - split) + (s - split))


# --- the five BASELINE.json configs --------------------------
SEED = 20240611


def config_case(k: int, **over) -> Case:
    base = dict(alpha_coeff=1, alpha_jump=0.5, delta_r=0.1, rmax=1.3, R0=1e-5, rel_tol=1e-10,
                max_iterations=200)
    if k == 0:
        c = Case(geometry="CirclePolar", kappa_eps=0.0, delta_e=0.0, beta_coeff=0, a=257, b=256,
                 stencil_mode="Give", **base)
    elif k == 1:
        c = Case(geometry="Shafranov", kappa_eps=0.3, delta_e=0.2, beta_coeff=1, a=1025, b=1024, **base)
    elif k == 2:
        c = Case(geometry="Czarny", kappa_eps=0.3, delta_e=1.4, beta_coeff=1, grid_mode=1, a=8, b=8,
                 divide_by_2=4, **base)
    elif k == 3:
        c = Case(geometry="Shafranov", kappa_eps=0.3, delta_e=0.2, beta_coeff=1, a=513, b=512, **base)
    elif k == 4:
        c = Case(geometry="Czarny", kappa_eps=0.3, delta_e=1.4, beta_coeff=1, a=8193, b=8192,
                 pair_tol=1e-9, **base)
    else:
        raise ValueError(k)
    for key, v in over.items():
        setattr(c, key, v)
    return c


def section_scales(n_sections: int = 256, seed: int = SEED + 1000003) -> np.ndarray:
    """Config 3's alpha scales c_i ~ U(0.5, 2) from mt19937(seed) in section order
    (std::uniform_real_distribution<double> semantics, see mt_uniform)."""
    return 0.5 + 1.5 * mt_canonical(seed, n_sections)


def mt_canonical(seed: int, count: int) -> np.ndarray:
    """libstdc++ generate_canonical<double,53>(mt19937(seed)): two 32-bit draws
    per value, (lo + hi * 2^32) / 2^64."""
    rs = np.random.RandomState(seed)
    raw = rs.randint(0, 2**32, size=2 * count, dtype=np.uint32).astype(np.float64)
    lo, hi = raw[0::2], raw[1::2]
    v = (lo + hi * 4294967296.0) / 18446744073709551616.0
    return np.where(v >= 1.0, np.nextafter(1.0, 0.0), v)
