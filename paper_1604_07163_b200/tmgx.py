"""Python mirror of the reference's solver / preconditioner surface over the tmgx C-ABI.

The reference (arxiv 1604.07163 re-creation, /root/reference/proj/core) exposes, for this
path, KrylovConfig / SolveReport / SolverNode (solver.hpp:27-93), Preconditioner::apply
(preconditioner.hpp:17-32), the grid maps of grid.hpp and Comm::split_strided
(comm.hpp:57-71). The same names, argument meanings and error classes are kept here; every
call goes through include/tmgx.h into the in-tree sm_100a library. There is no CPU fallback:
if libtmgx.so is missing or no GPU is present, the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
MAX_AXIS_PARTS = 64
MAX_TELESCOPE = 4
JOB_TOKEN_BYTES = 33

POISSON7, VARCOEF7_HARMONIC = 0, 1
EST_REFERENCE, EST_LANCZOS = 0, 1
KSP_CG, KSP_PREONLY = 2, 5
REASONS = ["rtol", "atol", "max_its", "fixed_its_done", "diverged"]


# ----------------------------------------------------------------- errors (common.hpp:16-34)
class Error(RuntimeError):
    """tmg::Error"""


class ConfigError(Error):
    """tmg::ConfigError (CLI exit 1)"""


class CudaError(Error):
    """CUDA / cross-process transport failure (C-ABI status 3)"""


# ----------------------------------------------------------------- ctypes structs
class Header(C.Structure):
    _fields_ = [("dim", C.c_int), ("np", C.c_int64 * 3), ("dof", C.c_int), ("pg", C.c_int * 3),
                ("off", (C.c_int64 * (MAX_AXIS_PARTS + 1)) * 3)]


class _Problem(C.Structure):
    _fields_ = [("kind", C.c_int), ("np", C.c_int64 * 3), ("pg_hint", C.c_int * 3), ("seed_k", C.c_uint64),
                ("n_spheres", C.c_int), ("k_in", C.c_double)]


class _Stage(C.Structure):
    _fields_ = [("level", C.c_int), ("reduction_factor", C.c_int), ("override_", C.c_int * 3)]


class _MG(C.Structure):
    _fields_ = [("nlevels", C.c_int), ("smooth_its", C.c_int), ("est_mode", C.c_int),
                ("cheb_bounds", C.POINTER(C.c_double)), ("n_telescope", C.c_int),
                ("telescope", _Stage * MAX_TELESCOPE), ("galerkin", C.c_int)]


class _Ksp(C.Structure):
    _fields_ = [("method", C.c_int), ("rtol", C.c_double), ("atol", C.c_double), ("max_its", C.c_int),
                ("zero_initial_guess", C.c_int)]


class _Report(C.Structure):
    _fields_ = [("reason", C.c_int), ("iterations", C.c_int), ("norm0", C.c_double), ("norm_final", C.c_double),
                ("t_solve_s", C.c_double), ("kernel_launches", C.c_int64)]


class _Counters(C.Structure):
    _fields_ = [("kernel_launches", C.c_int64), ("halo_bytes_sent", C.c_int64),
                ("telescope_bytes_sent", C.c_int64), ("allreduces", C.c_int64)]


# Every function include/tmgx.h declares (checked by tests/test_capi_symbols.py).
EXPORTS = [
    "tmgx_choose_proc_grid", "tmgx_grid_header", "tmgx_coarsen_header", "tmgx_layout_offsets",
    "tmgx_global_to_natural", "tmgx_natural_to_global", "tmgx_split_strided", "tmgx_repartition_header",
    "tmgx_prefusion_layout", "tmgx_permutation", "tmgx_job_token", "tmgx_world_create",
    "tmgx_world_destroy", "tmgx_world_local_ranks", "tmgx_solver_create", "tmgx_solver_destroy",
    "tmgx_solver_level_info", "tmgx_solver_bounds", "tmgx_fill_rhs", "tmgx_solve", "tmgx_solve_seeded",
    "tmgx_pc_apply", "tmgx_level_apply", "tmgx_level_smooth", "tmgx_level_residual_restrict",
    "tmgx_level_prolong_add", "tmgx_coarse_solve", "tmgx_telescope_gather", "tmgx_telescope_scatter",
    "tmgx_get_counters", "tmgx_parity_build", "tmgx_last_error", "tmgx_bench_kernel", "tmgx_plan_summary",
    "tmgx_node_selftest", "tmgx_exchange_timing", "tmgx_level_profile",
    "tmgx_options_create", "tmgx_options_destroy", "tmgx_options_parse", "tmgx_options_parse_file_text",
    "tmgx_options_set", "tmgx_options_get", "tmgx_options_serialize", "tmgx_options_unused",
    "tmgx_options_resolve", "tmgx_solver_from_options", "tmgx_telescope_timing",
    "tmgx_elast_create", "tmgx_elast_create_mg", "tmgx_elast_destroy", "tmgx_elast_kref", "tmgx_elast_level_info", "tmgx_elast_rhs",
    "tmgx_elast_level_apply", "tmgx_elast_level_smooth", "tmgx_elast_pc_apply", "tmgx_elast_solve",
    "tmgx_elast_bench_apply",
]

_libs = {}


def lib_path(parity=False):
    if not parity and os.environ.get("TMGX_LIB"):  # tuning experiments: an alternative in-tree build
        return os.path.join(HERE, os.environ["TMGX_LIB"])
    return os.path.join(HERE, "libtmgx_parity.so" if parity else "libtmgx.so")


def load(parity: bool = False):
    """Loads the in-tree sm_100a library (fails loudly if it has not been built)."""
    if parity in _libs:
        return _libs[parity]
    path = lib_path(parity)
    if not os.path.exists(path):
        raise Error(f"{path} not built: run python -c 'import __graft_entry__; __graft_entry__.build()'")
    L = C.CDLL(path)
    P, D, I64 = C.POINTER, C.POINTER(C.c_double), C.POINTER(C.c_int64)
    H = P(Header)
    sig = {
        "tmgx_choose_proc_grid": [C.c_int, C.c_int, I64, P(C.c_int)],
        "tmgx_grid_header": [C.c_int, C.c_int, I64, C.c_int, P(C.c_int), H],
        "tmgx_coarsen_header": [H, H],
        "tmgx_layout_offsets": [H, I64],
        "tmgx_global_to_natural": [H, C.c_int64],
        "tmgx_natural_to_global": [H, C.c_int64],
        "tmgx_split_strided": [C.c_int, C.c_int, P(C.c_int), P(C.c_int)],
        "tmgx_repartition_header": [C.c_int, C.c_int, P(C.c_int), H],
        "tmgx_prefusion_layout": [H, C.c_int, P(C.c_int), C.c_int, I64],
        "tmgx_permutation": [H, H, C.c_int64, C.c_int64, I64],
        "tmgx_job_token": [C.c_char_p],
        "tmgx_world_create": [C.c_int, C.c_int, C.c_int, C.c_int, C.c_char_p, P(C.c_void_p)],
        "tmgx_world_destroy": [C.c_void_p],
        "tmgx_world_local_ranks": [C.c_void_p, P(C.c_int), P(C.c_int)],
        "tmgx_solver_create": [C.c_void_p, P(_Problem), P(_MG), P(C.c_void_p)],
        "tmgx_solver_destroy": [C.c_void_p],
        "tmgx_solver_level_info": [C.c_void_p, C.c_int, H, I64],
        "tmgx_solver_bounds": [C.c_void_p, C.c_int, D, D],
        "tmgx_fill_rhs": [C.c_void_p, C.c_uint64, D],
        "tmgx_solve": [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, P(_Ksp), D, P(_Report)],
        "tmgx_solve_seeded": [C.c_void_p, C.c_uint64, C.c_void_p, P(_Ksp), D, P(_Report)],
        "tmgx_pc_apply": [C.c_void_p, D, D],
        "tmgx_level_apply": [C.c_void_p, C.c_int, D, D],
        "tmgx_level_smooth": [C.c_void_p, C.c_int, D, D],
        "tmgx_level_residual_restrict": [C.c_void_p, C.c_int, D, D, D],
        "tmgx_level_prolong_add": [C.c_void_p, C.c_int, D, D],
        "tmgx_coarse_solve": [C.c_void_p, D, D],
        "tmgx_telescope_gather": [C.c_void_p, C.c_int, D, D],
        "tmgx_telescope_scatter": [C.c_void_p, C.c_int, D, D],
        "tmgx_get_counters": [C.c_void_p, P(_Counters)],
        "tmgx_level_profile": [C.c_void_p, C.c_int, C.c_int, P(C.c_int), P(C.c_int), P(C.c_int64), P(C.c_int),
                               P(C.c_double), P(C.c_int64)],
        "tmgx_bench_kernel": [C.c_void_p, C.c_int, C.c_int, C.c_int, D, D],
        "tmgx_plan_summary": [C.c_int, C.c_int, C.c_int, P(_Problem), P(_MG), I64, C.c_int, P(C.c_int)],
        "tmgx_node_selftest": [C.c_char_p, C.c_int, C.c_int, C.c_int, I64],
        "tmgx_exchange_timing": [C.c_void_p, C.c_int, C.c_int, P(C.c_double), P(C.c_int64)],
        "tmgx_options_create": [P(C.c_void_p)],
        "tmgx_options_destroy": [C.c_void_p],
        "tmgx_options_parse": [C.c_void_p, C.c_int, P(C.c_char_p)],
        "tmgx_options_parse_file_text": [C.c_void_p, C.c_char_p],
        "tmgx_options_set": [C.c_void_p, C.c_char_p, C.c_char_p],
        "tmgx_options_get": [C.c_void_p, C.c_char_p, C.c_char_p, C.c_int, P(C.c_int)],
        "tmgx_options_serialize": [C.c_void_p, C.c_char_p, C.c_int],
        "tmgx_options_unused": [C.c_void_p, C.c_char_p, C.c_int],
        "tmgx_options_resolve": [C.c_void_p, C.c_char_p, C.c_char_p, P(_MG), P(_Ksp), C.c_char_p, C.c_int],
        "tmgx_telescope_timing": [C.c_void_p, C.c_int, C.c_int, D, D, I64],
        "tmgx_elast_create": [C.c_void_p, I64, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_double, P(C.c_void_p)],
        "tmgx_elast_create_mg": [C.c_void_p, I64, P(_MG), C.c_uint64, C.c_double, P(C.c_void_p)],
        "tmgx_elast_destroy": [C.c_void_p],
        "tmgx_elast_kref": [C.c_double, D],
        "tmgx_elast_level_info": [C.c_void_p, C.c_int, I64, D, D],
        "tmgx_elast_rhs": [C.c_void_p, D],
        "tmgx_elast_level_apply": [C.c_void_p, C.c_int, D, D],
        "tmgx_elast_level_smooth": [C.c_void_p, C.c_int, D, D],
        "tmgx_elast_pc_apply": [C.c_void_p, D, D],
        "tmgx_elast_solve": [C.c_void_p, C.c_void_p, C.c_void_p, P(_Ksp), D, P(_Report)],
        "tmgx_elast_bench_apply": [C.c_void_p, C.c_int, D, D, D],
        "tmgx_solver_from_options": [C.c_void_p, P(_Problem), C.c_void_p, C.c_char_p, C.c_char_p, P(C.c_void_p),
                                     P(_Ksp)],
    }
    sig["tmgx_repartition_header"] = [H, C.c_int, P(C.c_int), H]
    for name, args in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = C.c_int
    L.tmgx_global_to_natural.restype = C.c_int64
    L.tmgx_natural_to_global.restype = C.c_int64
    L.tmgx_last_error.restype = C.c_char_p
    L.tmgx_parity_build.restype = C.c_int
    _libs[parity] = L
    return L


def _check(L, rc):
    if rc == 0 or rc == 2:
        return rc
    msg = L.tmgx_last_error().decode()
    if rc == 1:
        raise ConfigError(msg)
    if rc == 3:
        raise CudaError(msg)
    raise Error(msg)


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _i64(a):
    return a.ctypes.data_as(C.POINTER(C.c_int64))


# ----------------------------------------------------------------- grid maps (grid.hpp)
@dataclass
class GridHeader:
    """GridHeader (grid.hpp:41-79)."""
    npoints: tuple
    proc_grid: tuple
    axis_offsets: tuple
    dim: int = 3
    dof: int = 1

    def _c(self):
        h = Header()
        h.dim, h.dof = self.dim, self.dof
        for a in range(3):
            h.np[a] = self.npoints[a]
            h.pg[a] = self.proc_grid[a]
            for p, v in enumerate(self.axis_offsets[a]):
                h.off[a][p] = v
        return h

    @staticmethod
    def _from(h):
        return GridHeader(tuple(int(v) for v in h.np), tuple(int(v) for v in h.pg),
                          tuple(tuple(int(h.off[a][p]) for p in range(h.pg[a] + 1)) for a in range(3)),
                          int(h.dim), int(h.dof))

    def n_ranks(self):
        return self.proc_grid[0] * self.proc_grid[1] * self.proc_grid[2]

    def n_unknowns(self):
        return self.npoints[0] * self.npoints[1] * self.npoints[2] * self.dof

    def box(self, rank):
        pg = self.proc_grid
        pc = (rank % pg[0], (rank // pg[0]) % pg[1], rank // (pg[0] * pg[1]))
        return (tuple(self.axis_offsets[a][pc[a]] for a in range(3)),
                tuple(self.axis_offsets[a][pc[a] + 1] for a in range(3)))

    def layout(self):
        L = load()
        off = np.zeros(self.n_ranks() + 1, dtype=np.int64)
        _check(L, L.tmgx_layout_offsets(C.byref(self._c()), _i64(off)))
        return off

    def global_to_natural(self, g):
        return load().tmgx_global_to_natural(C.byref(self._c()), g)

    def natural_to_global(self, n):
        return load().tmgx_natural_to_global(C.byref(self._c()), n)


def choose_proc_grid(size, dim, npoints):
    L = load()
    npa = np.array(npoints, dtype=np.int64)
    pg = (C.c_int * 3)()
    _check(L, L.tmgx_choose_proc_grid(size, dim, _i64(npa), pg))
    return tuple(pg)


def create_grid_header(size, npoints, dof=1, hint=None, dim=3):
    """create_grid's header (grid.cpp:256-292)."""
    L = load()
    npa = np.array(npoints, dtype=np.int64)
    h = Header()
    hp = (C.c_int * 3)(*hint) if hint is not None else None
    _check(L, L.tmgx_grid_header(size, dim, _i64(npa), dof, hp, C.byref(h)))
    return GridHeader._from(h)


def coarsen(h: GridHeader):
    L = load()
    out = Header()
    _check(L, L.tmgx_coarsen_header(C.byref(h._c()), C.byref(out)))
    return GridHeader._from(out)


@dataclass
class SplitResult:
    """SplitResult (comm.hpp:57-71)."""
    member_map: List[int]
    reduction_factor: int
    parent_size: int

    def is_member(self, parent_rank):
        return parent_rank % self.reduction_factor == 0

    def group_begin(self, m):
        return self.member_map[m]

    def group_end(self, m):
        return self.member_map[m + 1] if m + 1 < len(self.member_map) else self.parent_size


def split_strided(n, r):
    L = load()
    mm = (C.c_int * max(n, 1))()
    cnt = C.c_int()
    _check(L, L.tmgx_split_strided(n, r, mm, C.byref(cnt)))
    return SplitResult(list(mm[: cnt.value]), r, n)


def repartition_onto(h: GridHeader, split: SplitResult, override=(None, None, None)):
    """repartition_onto's header (grid.cpp:433-493)."""
    L = load()
    ov = (C.c_int * 3)(*[0 if o is None else o for o in override])
    out = Header()
    _check(L, L.tmgx_repartition_header(C.byref(h._c()), len(split.member_map), ov, C.byref(out)))
    return GridHeader._from(out)


def prefusion_layout(new_h: GridHeader, split: SplitResult):
    L = load()
    mm = (C.c_int * len(split.member_map))(*split.member_map)
    off = np.zeros(split.parent_size + 1, dtype=np.int64)
    _check(L, L.tmgx_prefusion_layout(C.byref(new_h._c()), split.parent_size, mm, len(split.member_map), _i64(off)))
    return off


def build_permutation(old_h: GridHeader, new_h: GridHeader, row_begin=0, row_end=None):
    """Columns of P-hat for old-layout rows [row_begin, row_end) (grid.cpp:582-599)."""
    L = load()
    if row_end is None:
        row_end = old_h.n_unknowns()
    cols = np.zeros(row_end - row_begin, dtype=np.int64)
    _check(L, L.tmgx_permutation(C.byref(old_h._c()), C.byref(new_h._c()), row_begin, row_end, _i64(cols)))
    return cols


# ----------------------------------------------------------------- solver surface
@dataclass
class KrylovConfig:
    """KrylovConfig (solver.hpp:27-37) restricted to this path (cg / preonly)."""
    method: str = "cg"
    rtol: float = 1e-8
    atol: float = 1e-50
    max_its: int = 10000
    initial_guess_nonzero: bool = True  # False: x is output only (x0 = 0, not uploaded)


@dataclass
class SolveReport:
    """SolveReport (solver.hpp:39-52)."""
    reason: str
    iterations: int
    residual_history: List[float]
    norm_kind: str = "preconditioned residual 2-norm"
    note: str = ""
    t_solve_s: float = 0.0
    kernel_launches: int = 0

    def converged(self):
        return self.reason in ("rtol", "atol", "fixed_its_done")


@dataclass
class Problem:
    """assemble_problem spec."""
    npoints: tuple = (65, 65, 65)
    kind: int = POISSON7
    proc_grid_hint: Optional[tuple] = None
    seed_k: int = 7
    n_spheres: int = 32
    k_in: float = 1e4


@dataclass
class TelescopeStage:
    level: int
    reduction_factor: int
    repart_da_processors: tuple = (None, None, None)


@dataclass
class MGConfig:
    """pc_mg: levels, Chebyshev(Jacobi) V(m,m), estimator mode, telescope stages, LU coarse."""
    nlevels: int = 5
    smooth_its: int = 2
    est_mode: int = EST_LANCZOS
    cheb_bounds: Optional[Sequence[float]] = None
    telescope: List[TelescopeStage] = field(default_factory=list)
    galerkin: bool = False  # -pc_mg_galerkin: 2^-3 P^T A P coarse operators (27-point)


# ----------------------------------------------------------------- options
class OptionsDatabase:
    """Prefix-keyed options database (the reference's missing options.cpp): ordered
    key -> string map with the leading dash stripped, flags stored as "true", later
    insertions winning, and used-key tracking. Backed by the C++ host layer of libtmgx."""

    def __init__(self, tokens: Optional[Sequence[str]] = None, parity: bool = False):
        self.L = load(parity)
        h = C.c_void_p()
        _check(self.L, self.L.tmgx_options_create(C.byref(h)))
        self.h = h
        if tokens:
            self.parse(tokens)

    def __del__(self):
        if getattr(self, "h", None):
            self.L.tmgx_options_destroy(self.h)
            self.h = None

    def parse(self, tokens: Sequence[str]):
        """parse(argv); ConfigError on a malformed token (with its position)."""
        arr = (C.c_char_p * max(len(tokens), 1))(*[t.encode() for t in tokens])
        _check(self.L, self.L.tmgx_options_parse(self.h, len(tokens), arr))
        return self

    def parse_file_text(self, text: str):
        _check(self.L, self.L.tmgx_options_parse_file_text(self.h, text.encode()))
        return self

    @classmethod
    def from_file(cls, path: str, parity: bool = False):
        with open(path) as f:
            return cls(parity=parity).parse_file_text(f.read())

    def set(self, key: str, value: str = "true"):
        _check(self.L, self.L.tmgx_options_set(self.h, key.encode(), str(value).encode()))
        return self

    def get(self, key: str) -> Optional[str]:
        buf = C.create_string_buffer(4096)
        found = C.c_int()
        _check(self.L, self.L.tmgx_options_get(self.h, key.encode(), buf, len(buf), C.byref(found)))
        return buf.value.decode() if found.value else None

    def _lines(self, fn) -> List[str]:
        n = 1 << 16
        while True:
            buf = C.create_string_buffer(n)
            rc = fn(self.h, buf, n)
            if rc == 0:
                v = buf.value.decode()
                return v.split("\n") if v else []
            if n > (1 << 26):
                _check(self.L, rc)
            n *= 4

    def serialize(self) -> List[str]:
        """Tokens that reparse to an equal database."""
        out = []
        for ln in self._lines(self.L.tmgx_options_serialize):
            out.append(ln)
        return out

    def unused(self) -> List[str]:
        return self._lines(self.L.tmgx_options_unused)

    def items(self):
        t = self.serialize()
        return [(t[i][1:], t[i + 1]) for i in range(0, len(t), 2)]


@dataclass
class ResolvedTree:
    ksp: KrylovConfig
    mg: MGConfig
    describe: str


def resolve_solver_tree(db: OptionsDatabase, prefix: str = "", default_ksp: Optional[str] = None) -> ResolvedTree:
    """build_solver_tree resolved onto the GPU hierarchy, host only: the fused
    level ladder (N1 + N2 - 1 levels), telescope stages, smoother and outer KSP."""
    mg, ksp = _MG(), _Ksp()
    buf = C.create_string_buffer(1 << 16)
    _check(db.L, db.L.tmgx_options_resolve(db.h, prefix.encode(), default_ksp.encode() if default_ksp else None,
                                           C.byref(mg), C.byref(ksp), buf, len(buf)))
    stages = []
    for t in range(mg.n_telescope):
        st = mg.telescope[t]
        ov = tuple(int(st.override_[a]) or None for a in range(3))
        stages.append(TelescopeStage(int(st.level), int(st.reduction_factor), ov))
    cfg = MGConfig(nlevels=mg.nlevels, smooth_its=mg.smooth_its, est_mode=mg.est_mode, telescope=stages,
                   galerkin=bool(mg.galerkin))
    method = {KSP_CG: "cg", KSP_PREONLY: "preonly"}[ksp.method]
    return ResolvedTree(KrylovConfig(method, ksp.rtol, ksp.atol, ksp.max_its, not ksp.zero_initial_guess), cfg,
                        buf.value.decode())


def build_solver_tree(db: OptionsDatabase, world: "World", problem: "Problem", prefix: str = "",
                      default_ksp: Optional[str] = None):
    """Instantiate the GPU solver from the options (KSP/PC tree).
    Returns (SolverNode, KrylovConfig for SolverNode.solve)."""
    r = resolve_solver_tree(db, prefix, default_ksp)
    return SolverNode(world, problem, r.mg), r.ksp


def job_token(parity=False):
    """A fresh node-local rendezvous name for a multi-process World (make it on one process and
    pass it to the others)."""
    L = load(parity)
    buf = C.create_string_buffer(JOB_TOKEN_BYTES)
    _check(L, L.tmgx_job_token(buf))
    return buf.value.decode()


class World:
    """spawn_world analog: n_ranks reference ranks over nproc processes (one GPU each)."""

    def __init__(self, n_ranks=1, nproc=1, proc=0, device=0, job: Optional[str] = None, parity=False):
        self.L = load(parity)
        self.parity = parity
        self.h = C.c_void_p()
        jb = job.encode() if job else None
        _check(self.L, self.L.tmgx_world_create(n_ranks, nproc, proc, device, jb, C.byref(self.h)))
        f, e = C.c_int(), C.c_int()
        self.L.tmgx_world_local_ranks(self.h, C.byref(f), C.byref(e))
        self.local_ranks = (f.value, e.value)
        self.n_ranks, self.nproc, self.proc = n_ranks, nproc, proc

    def close(self):
        if self.h:
            self.L.tmgx_world_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _c_problem(problem: Problem):
    p = _Problem()
    p.kind = problem.kind
    for a in range(3):
        p.np[a] = problem.npoints[a]
        p.pg_hint[a] = problem.proc_grid_hint[a] if problem.proc_grid_hint else 0
    p.seed_k, p.n_spheres, p.k_in = problem.seed_k, problem.n_spheres, problem.k_in
    return p


def _c_mg(mg: MGConfig):
    m = _MG()
    m.nlevels, m.smooth_its, m.est_mode = mg.nlevels, mg.smooth_its, mg.est_mode
    m.galerkin = int(mg.galerkin)
    bounds = None
    if mg.cheb_bounds is not None:
        bounds = np.ascontiguousarray(mg.cheb_bounds, dtype=np.float64)
        m.cheb_bounds = _dp(bounds)
    m.n_telescope = len(mg.telescope)
    for t, st in enumerate(mg.telescope):
        m.telescope[t].level = st.level
        m.telescope[t].reduction_factor = st.reduction_factor
        for a in range(3):
            o = st.repart_da_processors[a]
            m.telescope[t].override_[a] = 0 if o is None else o
    return m, bounds


def plan_summary(n_ranks, nproc, proc, problem: Problem, mg: MGConfig, max_records=100000):
    """Host-only: the halo / telescope plans process `proc` would build (tmgx_plan_summary).
    Returns a list of (plan_id, kind, peer, count, checksum, level); kind 0 send, 1 recv, 2 local."""
    L = load()
    p = _c_problem(problem)
    m, _keep = _c_mg(mg)
    out = np.zeros(6 * max_records, dtype=np.int64)
    n = C.c_int()
    _check(L, L.tmgx_plan_summary(n_ranks, nproc, proc, C.byref(p), C.byref(m), _i64(out), max_records,
                                  C.byref(n)))
    return [tuple(int(v) for v in out[6 * i: 6 * i + 6]) for i in range(n.value)]


def node_selftest(job, nproc, proc, rounds=50):
    """Host-only: join the node-local process group `job` and run its barrier / allgather
    self-check (tmgx_node_selftest). Returns (sum of gathered indices, consistent rounds)."""
    L = load()
    out = np.zeros(2, dtype=np.int64)
    _check(L, L.tmgx_node_selftest(job.encode(), nproc, proc, rounds, _i64(out)))
    return int(out[0]), int(out[1])


class SolverNode:
    """SolverNode (solver.hpp:72-93): CG + MG(Chebyshev-Jacobi, telescope, LU) on tmgx."""

    def __init__(self, world: World, problem: Problem, mg: MGConfig):
        self.world, self.problem, self.mg = world, problem, mg
        self.L = world.L
        p = _c_problem(problem)
        m, self._bounds = _c_mg(mg)
        self.h = C.c_void_p()
        _check(self.L, self.L.tmgx_solver_create(world.h, C.byref(p), C.byref(m), C.byref(self.h)))

    @classmethod
    def create(cls, world, problem, mg):
        return cls(world, problem, mg)

    def close(self):
        if self.h:
            self.L.tmgx_solver_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # --- introspection
    def telescope_timing(self, stage=0, reps=20):
        """(T_setup s, T_apply s, bytes per apply) of telescope stage `stage` (Table 1)."""
        ts, ta, by = C.c_double(), C.c_double(), C.c_int64()
        _check(self.L, self.L.tmgx_telescope_timing(self.h, stage, reps, C.byref(ts), C.byref(ta), C.byref(by)))
        return ts.value, ta.value, by.value

    def exchange_timing(self, level, reps=50):
        """(us per halo exchange of `level`, bytes this process sends per exchange); collective."""
        us, by = C.c_double(), C.c_int64()
        _check(self.L, self.L.tmgx_exchange_timing(self.h, level, reps, C.byref(us), C.byref(by)))
        return us.value, by.value

    def level_info(self, level):
        h = Header()
        n = C.c_int64()
        _check(self.L, self.L.tmgx_solver_level_info(self.h, level, C.byref(h), C.byref(n)))
        return GridHeader._from(h), n.value

    def local_size(self, level=None):
        return self.level_info(self.mg.nlevels - 1 if level is None else level)[1]

    def bounds(self, level):
        lo, hi = C.c_double(), C.c_double()
        _check(self.L, self.L.tmgx_solver_bounds(self.h, level, C.byref(lo), C.byref(hi)))
        return lo.value, hi.value

    def counters(self):
        c = _Counters()
        self.L.tmgx_get_counters(self.h, C.byref(c))
        return {k: getattr(c, k) for k, _ in _Counters._fields_}

    def rhs(self, seed):
        b = np.zeros(self.local_size())
        _check(self.L, self.L.tmgx_fill_rhs(self.h, seed, _dp(b)))
        return b

    # --- solve (krylov_solve)
    def _ksp(self, cfg: KrylovConfig):
        k = _Ksp()
        k.method = {"cg": KSP_CG, "preonly": KSP_PREONLY}.get(cfg.method, -1)
        if k.method < 0:
            raise ConfigError(f"unknown ksp_type '{cfg.method}' on this path (valid: cg, preonly)")
        k.rtol, k.atol, k.max_its = cfg.rtol, cfg.atol, cfg.max_its
        k.zero_initial_guess = 0 if cfg.initial_guess_nonzero else 1
        return k

    def _report(self, rep, hist, cfg):
        n = rep.iterations + 1 if cfg.method == "cg" else 0
        return SolveReport(REASONS[rep.reason], rep.iterations, list(hist[:n]),
                           note="cg breakdown" if rep.reason == 4 else "", t_solve_s=rep.t_solve_s,
                           kernel_launches=rep.kernel_launches)

    def solve(self, b, x=None, cfg: KrylovConfig = KrylovConfig()):
        """Host arrays (numpy) in this process's rank-block local order; x is the initial guess
        and receives the solution."""
        b = np.ascontiguousarray(b, dtype=np.float64)
        if x is None:
            x = np.zeros_like(b)
        k = self._ksp(cfg)
        hist = np.zeros(cfg.max_its + 1)
        rep = _Report()
        _check(self.L, self.L.tmgx_solve(self.h, b.ctypes.data, x.ctypes.data, 0, C.byref(k), _dp(hist),
                                         C.byref(rep)))
        return x, self._report(rep, hist, cfg)

    def solve_ptr(self, b_ptr, x_ptr, on_device, cfg: KrylovConfig = KrylovConfig()):
        """Raw pointers (e.g. torch pinned host or device tensors)."""
        k = self._ksp(cfg)
        hist = np.zeros(cfg.max_its + 1)
        rep = _Report()
        _check(self.L, self.L.tmgx_solve(self.h, C.c_void_p(b_ptr), C.c_void_p(x_ptr), int(on_device), C.byref(k),
                                         _dp(hist), C.byref(rep)))
        return self._report(rep, hist, cfg)

    def solve_seeded(self, seed, x_dev_ptr=None, cfg: KrylovConfig = KrylovConfig()):
        k = self._ksp(cfg)
        hist = np.zeros(cfg.max_its + 1)
        rep = _Report()
        _check(self.L, self.L.tmgx_solve_seeded(self.h, seed, C.c_void_p(x_dev_ptr) if x_dev_ptr else None,
                                                C.byref(k), _dp(hist), C.byref(rep)))
        return self._report(rep, hist, cfg)

    # --- Preconditioner::apply and level primitives
    def pc_apply(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros_like(x)
        _check(self.L, self.L.tmgx_pc_apply(self.h, _dp(x), _dp(y)))
        return y

    def level_apply(self, level, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros_like(x)
        _check(self.L, self.L.tmgx_level_apply(self.h, level, _dp(x), _dp(y)))
        return y

    def level_smooth(self, level, b, x0=None):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.zeros_like(b) if x0 is None else np.array(x0, dtype=np.float64)
        _check(self.L, self.L.tmgx_level_smooth(self.h, level, _dp(b), _dp(x)))
        return x

    def residual_restrict(self, fine_level, b, x):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.ascontiguousarray(x, dtype=np.float64)
        bc = np.zeros(self.level_info(fine_level - 1)[1])
        _check(self.L, self.L.tmgx_level_residual_restrict(self.h, fine_level, _dp(b), _dp(x), _dp(bc)))
        return bc

    def prolong_add(self, fine_level, xc, xf):
        xc = np.ascontiguousarray(xc, dtype=np.float64)
        xf = np.array(xf, dtype=np.float64)
        _check(self.L, self.L.tmgx_level_prolong_add(self.h, fine_level, _dp(xc), _dp(xf)))
        return xf

    def coarse_solve(self, b):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.zeros_like(b)
        _check(self.L, self.L.tmgx_coarse_solve(self.h, _dp(b), _dp(x)))
        return x

    def level_profile(self, reps=10):
        """Per-node V-cycle profile (tmgx_level_profile): list of dicts {node, kind, npoints,
        ranks, us, peer_bytes}, node 0 = finest."""
        mx = 64
        n = C.c_int()
        kind, ranks = (C.c_int * mx)(), (C.c_int * mx)()
        npts = (C.c_int64 * (3 * mx))()
        us, by = (C.c_double * mx)(), (C.c_int64 * mx)()
        _check(self.L, self.L.tmgx_level_profile(self.h, reps, mx, C.byref(n), kind, npts, ranks, us, by))
        names = {0: "smooth", 1: "telescope", 2: "coarse"}
        return [{"node": i, "kind": names.get(kind[i], str(kind[i])), "npoints": list(npts[3 * i:3 * i + 3]),
                 "ranks": ranks[i], "us": us[i], "peer_bytes": by[i]} for i in range(n.value)]

    def bench_kernel(self, which, level, iters=20):
        """(ms per launch, algorithmic bytes per launch) for kernel `which` on `level`."""
        ms, by = C.c_double(), C.c_double()
        _check(self.L, self.L.tmgx_bench_kernel(self.h, which, level, iters, C.byref(ms), C.byref(by)))
        return ms.value, by.value

    def telescope_gather(self, stage, x_parent, n_sub):
        x_parent = np.ascontiguousarray(x_parent, dtype=np.float64)
        out = np.zeros(n_sub)
        _check(self.L, self.L.tmgx_telescope_gather(self.h, stage, _dp(x_parent), _dp(out)))
        return out

    def telescope_scatter(self, stage, y_sub, n_parent):
        y_sub = np.ascontiguousarray(y_sub, dtype=np.float64)
        out = np.zeros(n_parent)
        _check(self.L, self.L.tmgx_telescope_scatter(self.h, stage, _dp(y_sub), _dp(out)))
        return out


# ----------------------------------------------------------------- ordering helpers
def rank_block_to_natural(h: GridHeader, ranks=None):
    """Index array: natural index of each entry of the concatenated local slices of `ranks`
    (default: all ranks) in rank-block order (grid.cpp:61-82)."""
    if ranks is None:
        ranks = range(h.n_ranks())
    out = []
    for r in ranks:
        lo, hi = h.box(r)
        k, j, i = np.meshgrid(np.arange(lo[2], hi[2]), np.arange(lo[1], hi[1]), np.arange(lo[0], hi[0]),
                              indexing="ij")
        out.append((i + h.npoints[0] * (j + h.npoints[1] * k)).ravel())
    return np.concatenate(out) if out else np.zeros(0, dtype=np.int64)


# ----------------------------------------------------------------- Q1 elasticity (configs[4])
def elast_kref(nu=0.3, parity=False):
    """24x24 reference stiffness of the unit-cube Q1 element (E = 1), host computed."""
    L = load(parity)
    K = np.zeros(576)
    _check(L, L.tmgx_elast_kref(nu, _dp(K)))
    return K.reshape(24, 24)


class ElastSolver:
    """Q1 hexahedral elasticity MG-CG (tmgx_elast.cu): N^3 vertices x 3 dofs, log-uniform E per
    element, clamped x = 0, body force (0, 0, -1), point-block Jacobi Chebyshev V(m,m),
    rediscretised coarse levels, LU on level 0. The levels are split into the world's boxes
    like the scalar path and may be telescoped (`telescope`: TelescopeStage list; cfg5 is 8
    boxes with reduction factor 8 at level 3). Vectors in the level's global natural vertex
    order with 3 interleaved dofs; each process reads / writes its own boxes' entries."""

    def __init__(self, world: World, npoints, nlevels, smooth_its=2, est_mode=EST_LANCZOS, seed_e=11, nu=0.3,
                 telescope: Optional[Sequence[TelescopeStage]] = None, cheb_bounds=None):
        self.world, self.L = world, world.L
        self.nlevels = nlevels
        npa = np.array(npoints, dtype=np.int64)
        h = C.c_void_p()
        if cheb_bounds is not None and len(cheb_bounds) != 2 * nlevels:
            raise ConfigError(f"elasticity: cheb_bounds needs 2 * nlevels = {2 * nlevels} values")
        mg = MGConfig(nlevels=nlevels, smooth_its=smooth_its, est_mode=est_mode, cheb_bounds=cheb_bounds,
                      telescope=list(telescope or []))
        m, _keep = _c_mg(mg)
        _check(self.L, self.L.tmgx_elast_create_mg(world.h, _i64(npa), C.byref(m), seed_e, nu, C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            self.L.tmgx_elast_destroy(self.h)
            self.h = None

    def level_shape(self, level):
        n = np.zeros(3, dtype=np.int64)
        lo, hi = C.c_double(), C.c_double()
        _check(self.L, self.L.tmgx_elast_level_info(self.h, level, _i64(n), C.byref(lo), C.byref(hi)))
        return tuple(int(v) for v in n)

    def level_size(self, level):
        s = self.level_shape(level)
        return 3 * s[0] * s[1] * s[2]

    def bounds(self, level):
        n = np.zeros(3, dtype=np.int64)
        lo, hi = C.c_double(), C.c_double()
        _check(self.L, self.L.tmgx_elast_level_info(self.h, level, _i64(n), C.byref(lo), C.byref(hi)))
        return lo.value, hi.value

    def rhs(self):
        b = np.zeros(self.level_size(self.nlevels - 1))
        _check(self.L, self.L.tmgx_elast_rhs(self.h, _dp(b)))
        return b

    def level_apply(self, level, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros_like(x)
        _check(self.L, self.L.tmgx_elast_level_apply(self.h, level, _dp(x), _dp(y)))
        return y

    def level_smooth(self, level, b, x0=None):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.zeros_like(b) if x0 is None else np.array(x0, dtype=np.float64)
        _check(self.L, self.L.tmgx_elast_level_smooth(self.h, level, _dp(b), _dp(x)))
        return x

    def pc_apply(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros_like(x)
        _check(self.L, self.L.tmgx_elast_pc_apply(self.h, _dp(x), _dp(y)))
        return y

    def solve(self, b, x=None, cfg: KrylovConfig = KrylovConfig(rtol=1e-6)):
        b = np.ascontiguousarray(b, dtype=np.float64)
        if x is None:
            x = np.zeros_like(b)
        k = SolverNode._ksp(None, cfg)
        hist = np.zeros(cfg.max_its + 1)
        rep = _Report()
        _check(self.L, self.L.tmgx_elast_solve(self.h, b.ctypes.data, x.ctypes.data, C.byref(k), _dp(hist),
                                               C.byref(rep)))
        return x, SolverNode._report(None, rep, hist, cfg)

    def bench_apply(self, iters=20):
        ms, by, fl = C.c_double(), C.c_double(), C.c_double()
        _check(self.L, self.L.tmgx_elast_bench_apply(self.h, iters, C.byref(ms), C.byref(by), C.byref(fl)))
        return ms.value, by.value, fl.value

    def solve_ptr(self, b_ptr, x_ptr, cfg: KrylovConfig = KrylovConfig(rtol=1e-6)):
        k = SolverNode._ksp(None, cfg)
        hist = np.zeros(cfg.max_its + 1)
        rep = _Report()
        _check(self.L, self.L.tmgx_elast_solve(self.h, C.c_void_p(b_ptr), C.c_void_p(x_ptr), C.byref(k), _dp(hist),
                                               C.byref(rep)))
        return SolverNode._report(None, rep, hist, cfg)
