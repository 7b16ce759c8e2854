"""TEST INFRASTRUCTURE ONLY — ctypes wrapper over oracle/liboracle.so (the CPU oracle).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
import this module. The product package (paper_1604_07163_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

MAX_PARTS = 64
POISSON7, VARCOEF7 = 0, 1
EST_REFERENCE, EST_LANCZOS = 0, 1
REASONS = ["rtol", "atol", "max_its", "fixed_its_done", "diverged"]


class Header(C.Structure):
    _fields_ = [
        ("dim", C.c_int),
        ("np", C.c_int64 * 3),
        ("dof", C.c_int),
        ("pg", C.c_int * 3),
        ("off", (C.c_int64 * (MAX_PARTS + 1)) * 3),
    ]

    def offsets(self, axis):
        return [int(self.off[axis][p]) for p in range(self.pg[axis] + 1)]

    def n_ranks(self):
        return self.pg[0] * self.pg[1] * self.pg[2]

    def n(self):
        return int(self.np[0] * self.np[1] * self.np[2] * self.dof)


class MGCfg(C.Structure):
    _fields_ = [
        ("kind", C.c_int),
        ("np", C.c_int64 * 3),
        ("nlevels", C.c_int),
        ("smooth_its", C.c_int),
        ("est_mode", C.c_int),
        ("zero_coarse_bc", C.c_int),
        ("seed_k", C.c_uint64),
        ("n_spheres", C.c_int),
        ("k_in", C.c_double),
        ("cheb_lo_fac", C.c_double),
        ("cheb_hi_fac", C.c_double),
        ("galerkin", C.c_int),
    ]


class ElCfg(C.Structure):
    _fields_ = [("np", C.c_int64 * 3), ("nlevels", C.c_int), ("smooth_its", C.c_int), ("est_mode", C.c_int),
                ("seed_e", C.c_uint64), ("nu", C.c_double)]


class Report(C.Structure):
    _fields_ = [("reason", C.c_int), ("iterations", C.c_int), ("norm0", C.c_double),
                ("norm_final", C.c_double)]


_lib = None


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        D = C.POINTER(C.c_double)
        I64 = C.POINTER(C.c_int64)
        L.orc_hashed_uniform.restype = C.c_double
        L.orc_hashed_uniform.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_splitmix64.restype = C.c_uint64
        L.orc_splitmix64.argtypes = [C.c_uint64]
        L.orc_choose_proc_grid.argtypes = [C.c_int, C.c_int, I64, C.POINTER(C.c_int)]
        L.orc_build_header.argtypes = [C.c_int, C.c_int, I64, C.c_int, C.POINTER(C.c_int), C.POINTER(Header)]
        L.orc_coarsen_header.argtypes = [C.POINTER(Header), C.POINTER(Header)]
        L.orc_global_index.restype = C.c_int64
        L.orc_global_index.argtypes = [C.POINTER(Header), C.c_int64, C.c_int64, C.c_int64, C.c_int]
        L.orc_global_to_natural.restype = C.c_int64
        L.orc_global_to_natural.argtypes = [C.POINTER(Header), C.c_int64]
        L.orc_natural_to_global.restype = C.c_int64
        L.orc_natural_to_global.argtypes = [C.POINTER(Header), C.c_int64]
        L.orc_layout_offsets.argtypes = [C.POINTER(Header), I64]
        L.orc_split_strided.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_int)]
        L.orc_repartition.argtypes = [C.POINTER(Header), C.c_int, C.POINTER(C.c_int), C.POINTER(Header)]
        L.orc_prefusion_layout.argtypes = [C.POINTER(Header), C.c_int, C.POINTER(C.c_int), C.c_int, I64]
        L.orc_build_permutation.argtypes = [C.POINTER(Header), C.POINTER(Header), I64]
        L.orc_mg_create.restype = C.c_void_p
        L.orc_mg_create.argtypes = [C.POINTER(MGCfg)]
        L.orc_mg_destroy.argtypes = [C.c_void_p]
        L.orc_mg_level_n.restype = C.c_int64
        L.orc_mg_level_n.argtypes = [C.c_void_p, C.c_int, I64]
        L.orc_mg_bounds.argtypes = [C.c_void_p, C.c_int, D, D]
        L.orc_mg_coeff.argtypes = [C.c_void_p, C.c_int, D]
        L.orc_mg_stencil27.argtypes = [C.c_void_p, C.c_int, D]
        L.orc_rhs.argtypes = [I64, C.c_uint64, D]
        L.orc_fill_random.argtypes = [C.c_int64, C.c_uint64, D]
        for fn in ("orc_apply", "orc_jacobi", "orc_smooth", "orc_restrict", "orc_prolong_add", "orc_vcycle"):
            getattr(L, fn).argtypes = [C.c_void_p, C.c_int, D, D]
        L.orc_coarse_solve.argtypes = [C.c_void_p, D, D]
        L.orc_estimate.argtypes = [C.c_void_p, C.c_int, C.c_int, D, D]
        L.orc_dot.restype = C.c_double
        L.orc_dot.argtypes = [C.c_int64, D, D]
        L.orc_mgcg_solve.argtypes = [C.c_void_p, D, D, C.c_double, C.c_double, C.c_int, D, C.POINTER(Report)]
        L.orc_estimate_dense.restype = C.c_double
        L.orc_estimate_dense.argtypes = [C.c_int, D, C.c_int, C.c_int]
        L.orc_el_kref.argtypes = [C.c_double, D]
        L.orc_el_create.restype = C.c_void_p
        L.orc_el_create.argtypes = [C.POINTER(ElCfg)]
        L.orc_el_destroy.argtypes = [C.c_void_p]
        L.orc_el_level_nv.restype = C.c_int64
        L.orc_el_level_nv.argtypes = [C.c_void_p, C.c_int]
        L.orc_el_bounds.argtypes = [C.c_void_p, C.c_int, D, D]
        L.orc_el_elements.argtypes = [C.c_void_p, C.c_int, D]
        for fn in ("orc_el_apply", "orc_el_jacobi", "orc_el_smooth", "orc_el_restrict", "orc_el_prolong_add",
                   "orc_el_vcycle"):
            getattr(L, fn).argtypes = [C.c_void_p, C.c_int, D, D]
        L.orc_el_coarse_solve.argtypes = [C.c_void_p, D, D]
        L.orc_el_rhs.argtypes = [I64, D]
        L.orc_el_solve.argtypes = [C.c_void_p, D, D, C.c_double, C.c_double, C.c_int, D, C.POINTER(Report)]
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _ip64(a):
    return a.ctypes.data_as(C.POINTER(C.c_int64))


# ---------------------------------------------------------------- grid maps
def hashed_uniform(seed, index):
    return lib().orc_hashed_uniform(seed, index)


def choose_proc_grid(size, dim, np3):
    npa = np.array(np3, dtype=np.int64)
    pg = (C.c_int * 3)()
    if lib().orc_choose_proc_grid(size, dim, _ip64(npa), pg):
        return None
    return tuple(pg)


def build_header(size, np3, dof=1, hint=None, dim=3):
    h = Header()
    npa = np.array(np3, dtype=np.int64)
    hp = (C.c_int * 3)(*hint) if hint is not None else None
    if lib().orc_build_header(size, dim, _ip64(npa), dof, hp, C.byref(h)):
        raise ValueError("over-decomposed / invalid header")
    return h


def coarsen_header(h):
    out = Header()
    if lib().orc_coarsen_header(C.byref(h), C.byref(out)):
        return None
    return out


def layout_offsets(h):
    off = np.zeros(h.n_ranks() + 1, dtype=np.int64)
    lib().orc_layout_offsets(C.byref(h), _ip64(off))
    return off


def global_to_natural(h, g):
    return lib().orc_global_to_natural(C.byref(h), g)


def natural_to_global(h, n):
    return lib().orc_natural_to_global(C.byref(h), n)


def split_strided(n, r):
    mm = (C.c_int * n)()
    m = lib().orc_split_strided(n, r, mm)
    return list(mm[:m])


def repartition(h, sub_size, override=(0, 0, 0)):
    out = Header()
    ov = (C.c_int * 3)(*override)
    if lib().orc_repartition(C.byref(h), sub_size, ov, C.byref(out)):
        raise ValueError("repartition rejected")
    return out


def prefusion_layout(newh, parent_size, member_map):
    mm = (C.c_int * len(member_map))(*member_map)
    off = np.zeros(parent_size + 1, dtype=np.int64)
    lib().orc_prefusion_layout(C.byref(newh), parent_size, mm, len(member_map), _ip64(off))
    return off


def build_permutation(oldh, newh):
    q = np.zeros(oldh.n(), dtype=np.int64)
    lib().orc_build_permutation(C.byref(oldh), C.byref(newh), _ip64(q))
    return q


# ---------------------------------------------------------------- numerics
class MG:
    """1-rank MG hierarchy (level 0 = coarsest, LU)."""

    def __init__(self, np3, nlevels, kind=POISSON7, smooth_its=2, est_mode=EST_LANCZOS,
                 zero_coarse_bc=0, seed_k=7, n_spheres=32, k_in=1e4, galerkin=False):
        cfg = MGCfg()
        cfg.kind = kind
        cfg.np = (C.c_int64 * 3)(*np3)
        cfg.nlevels = nlevels
        cfg.smooth_its = smooth_its
        cfg.est_mode = est_mode
        cfg.zero_coarse_bc = zero_coarse_bc
        cfg.seed_k = seed_k
        cfg.n_spheres = n_spheres
        cfg.k_in = k_in
        cfg.cheb_lo_fac, cfg.cheb_hi_fac = 0.1, 1.1
        cfg.galerkin = int(galerkin)
        self.cfg = cfg
        self.nlevels = nlevels
        self.h = lib().orc_mg_create(C.byref(cfg))
        if not self.h:
            raise ValueError("cannot coarsen")

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_mg_destroy(self.h)
            self.h = None

    def level_shape(self, level):
        n = np.zeros(3, dtype=np.int64)
        lib().orc_mg_level_n(self.h, level, _ip64(n))
        return tuple(int(v) for v in n)

    def level_size(self, level):
        s = self.level_shape(level)
        return s[0] * s[1] * s[2]

    def bounds(self, level):
        lo, hi = C.c_double(), C.c_double()
        lib().orc_mg_bounds(self.h, level, C.byref(lo), C.byref(hi))
        return lo.value, hi.value

    def coeff(self, level):
        out = np.zeros(self.level_size(level))
        lib().orc_mg_coeff(self.h, level, _dp(out))
        return out

    def stencil27(self, level):
        out = np.zeros(27 * self.level_size(level))
        if not lib().orc_mg_stencil27(self.h, level, _dp(out)):
            return None
        return out.reshape(27, -1)

    def _lv(self, fn, level, x, out=None):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros(self.level_size(level)) if out is None else out
        getattr(lib(), fn)(self.h, level, _dp(x), _dp(y))
        return y

    def apply(self, level, x):
        return self._lv("orc_apply", level, x)

    def jacobi(self, level, x):
        return self._lv("orc_jacobi", level, x)

    def smooth(self, level, b, x0=None):
        x = np.zeros(self.level_size(level)) if x0 is None else np.array(x0, dtype=np.float64)
        return self._lv("orc_smooth", level, b, x)

    def restrict(self, fine_level, r):
        r = np.ascontiguousarray(r, dtype=np.float64)
        out = np.zeros(self.level_size(fine_level - 1))
        lib().orc_restrict(self.h, fine_level, _dp(r), _dp(out))
        return out

    def prolong_add(self, fine_level, xc, xf):
        xc = np.ascontiguousarray(xc, dtype=np.float64)
        xf = np.array(xf, dtype=np.float64)
        lib().orc_prolong_add(self.h, fine_level, _dp(xc), _dp(xf))
        return xf

    def vcycle(self, level, b):
        return self._lv("orc_vcycle", level, b)

    def coarse_solve(self, b):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.zeros(self.level_size(0))
        lib().orc_coarse_solve(self.h, _dp(b), _dp(x))
        return x

    def estimate(self, level, mode):
        lo, hi = C.c_double(), C.c_double()
        lib().orc_estimate(self.h, level, mode, C.byref(lo), C.byref(hi))
        return lo.value, hi.value

    def solve(self, b, rtol=1e-8, atol=1e-50, max_its=10000, x0=None):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.zeros_like(b) if x0 is None else np.array(x0, dtype=np.float64)
        hist = np.zeros(max_its + 1)
        rep = Report()
        lib().orc_mgcg_solve(self.h, _dp(b), _dp(x), rtol, atol, max_its, _dp(hist), C.byref(rep))
        return x, {"reason": REASONS[rep.reason], "iterations": rep.iterations, "norm0": rep.norm0,
                   "norm_final": rep.norm_final, "history": hist[: rep.iterations + 1].copy()}


def rhs(np3, seed):
    n = int(np3[0] * np3[1] * np3[2])
    b = np.zeros(n)
    npa = np.array(np3, dtype=np.int64)
    lib().orc_rhs(_ip64(npa), seed, _dp(b))
    return b


def fill_random(n, seed):
    x = np.zeros(n)
    lib().orc_fill_random(n, seed, _dp(x))
    return x


def dot(x, y):
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    return lib().orc_dot(x.size, _dp(x), _dp(y))


def estimate_dense(A, jacobi=False, mode=EST_LANCZOS):
    A = np.ascontiguousarray(A, dtype=np.float64)
    return lib().orc_estimate_dense(A.shape[0], _dp(A), int(jacobi), mode)


# ---------------------------------------------------------------- Q1 elasticity (tmg_elast_oracle.c)
def el_kref(nu=0.3):
    K = np.zeros(576)
    lib().orc_el_kref(nu, _dp(K))
    return K.reshape(24, 24)


def el_rhs(np3):
    n = int(np3[0] * np3[1] * np3[2])
    b = np.zeros(3 * n)
    npa = np.array(np3, dtype=np.int64)
    lib().orc_el_rhs(_ip64(npa), _dp(b))
    return b


class ElastMG:
    """Q1 elasticity MG hierarchy (3 interleaved dofs per vertex; level 0 = coarsest, LU)."""

    def __init__(self, np3, nlevels, smooth_its=2, est_mode=EST_LANCZOS, seed_e=11, nu=0.3):
        cfg = ElCfg()
        cfg.np = (C.c_int64 * 3)(*np3)
        cfg.nlevels, cfg.smooth_its, cfg.est_mode, cfg.seed_e, cfg.nu = nlevels, smooth_its, est_mode, seed_e, nu
        self.cfg = cfg
        self.nlevels = nlevels
        self.np3 = tuple(np3)
        self.h = lib().orc_el_create(C.byref(cfg))

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_el_destroy(self.h)
            self.h = None

    def level_nv(self, level):
        return int(lib().orc_el_level_nv(self.h, level))

    def level_size(self, level):
        return 3 * self.level_nv(level)

    def bounds(self, level):
        lo, hi = C.c_double(), C.c_double()
        lib().orc_el_bounds(self.h, level, C.byref(lo), C.byref(hi))
        return lo.value, hi.value

    def elements(self, level):
        n = round(self.level_nv(level) ** (1 / 3))
        out = np.zeros((n - 1) ** 3)
        lib().orc_el_elements(self.h, level, _dp(out))
        return out

    def _lv(self, fn, level, x, out=None):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros(self.level_size(level)) if out is None else out
        getattr(lib(), fn)(self.h, level, _dp(x), _dp(y))
        return y

    def apply(self, level, x):
        return self._lv("orc_el_apply", level, x)

    def jacobi(self, level, x):
        return self._lv("orc_el_jacobi", level, x)

    def smooth(self, level, b, x0=None):
        x = np.zeros(self.level_size(level)) if x0 is None else np.array(x0, dtype=np.float64)
        return self._lv("orc_el_smooth", level, b, x)

    def restrict(self, fine_level, r):
        r = np.ascontiguousarray(r, dtype=np.float64)
        out = np.zeros(self.level_size(fine_level - 1))
        lib().orc_el_restrict(self.h, fine_level, _dp(r), _dp(out))
        return out

    def prolong_add(self, fine_level, xc, xf):
        xc = np.ascontiguousarray(xc, dtype=np.float64)
        xf = np.array(xf, dtype=np.float64)
        lib().orc_el_prolong_add(self.h, fine_level, _dp(xc), _dp(xf))
        return xf

    def vcycle(self, level, b):
        return self._lv("orc_el_vcycle", level, b)

    def coarse_solve(self, b):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.zeros(self.level_size(0))
        lib().orc_el_coarse_solve(self.h, _dp(b), _dp(x))
        return x

    def solve(self, b, rtol=1e-6, atol=1e-50, max_its=10000, x0=None):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.zeros_like(b) if x0 is None else np.array(x0, dtype=np.float64)
        hist = np.zeros(max_its + 1)
        rep = Report()
        lib().orc_el_solve(self.h, _dp(b), _dp(x), rtol, atol, max_its, _dp(hist), C.byref(rep))
        return x, {"reason": REASONS[rep.reason], "iterations": rep.iterations, "norm0": rep.norm0,
                   "norm_final": rep.norm_final, "history": hist[: rep.iterations + 1].copy()}
