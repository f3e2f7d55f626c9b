"""B200-native adaptive BDDC (arXiv 0910.5863) -- Python mirror of the C ABI.

The product is the in-tree shared library `libbddc_b200.so` (C++ host layer +
sm_100a CUDA kernels, `include/bddc_b200.h`).  This module binds it with
ctypes and mirrors the reference library's interface for the hot path
(`/root/reference/proj/core/include/bddc/*.hpp`): structure summary, constraint
sets, `enrich_constraints`, the BDDC preconditioner, the interface (Schur)
problem, `pcg`, and the experiment rows.  There is no CPU fallback: loading
fails loudly when the library is missing, and every compute call raises when
no CUDA device is present.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field
from pathlib import Path
from typing import List, Optional, Sequence

import numpy as np

__all__ = ["load_library", "Problem", "BDDC", "Row", "BddcError", "EXPORTS", "emit_table"]

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "libbddc_b200.so"

# Status codes (include/bddc_b200.h; reference types.hpp:21-63)
STATUS = {0: "OK", 1: "Error", 2: "NotPositiveDefinite", 3: "DegenerateElement",
          4: "CornerSelectionFailed", 5: "NullspaceInclusionViolated", 6: "SingularGram",
          7: "NotAdjacent", 8: "BadProblemSpec", 9: "MaxIterationsExceeded", 10: "CudaError",
          11: "Unsupported"}


class BddcError(RuntimeError):
    """Raised for a non-zero status; `.kind` is the reference exception name."""

    def __init__(self, code: int, message: str):
        super().__init__("%s: %s" % (STATUS.get(code, "Error"), message))
        self.code = code
        self.kind = STATUS.get(code, "Error")


class _Problem(C.Structure):
    _fields_ = [("subdomains", C.c_int * 3), ("elements_per_edge", C.c_int), ("physics", C.c_int),
                ("n_materials", C.c_int), ("material_id", C.POINTER(C.c_int)),
                ("conductivity", C.POINTER(C.c_double)), ("youngs", C.POINTER(C.c_double)),
                ("poisson", C.POINTER(C.c_double)), ("n_regions", C.c_int),
                ("region_box", C.POINTER(C.c_int)), ("region_material", C.POINTER(C.c_int)),
                ("n_dirichlet", C.c_int), ("dirichlet_face", C.POINTER(C.c_int)),
                ("dirichlet_components", C.POINTER(C.c_int)), ("n_loads", C.c_int),
                ("load_face", C.POINTER(C.c_int)), ("load_traction", C.POINTER(C.c_double)),
                ("load_flux", C.POINTER(C.c_double)), ("body_force", C.c_double * 3),
                ("source", C.c_double), ("tolerance", C.c_double), ("max_iterations", C.c_int),
                ("element_scale", C.POINTER(C.c_double))]


class _Structure(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("dofs", "free_dofs", "interface_dofs", "corners",
                                         "classification_corners", "edges", "faces",
                                         "coarse_space_dim", "subdomains", "w_dim", "elements")]


class _PcgResult(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("relative_residual", C.c_double),
                ("condition_estimate", C.c_double), ("converged", C.c_int)]


class _StepOut(C.Structure):
    _fields_ = [("seconds", C.c_double), ("setup_seconds", C.c_double), ("solve_seconds", C.c_double),
                ("h2d_bytes", C.c_double), ("d2h_bytes", C.c_double), ("launches", C.c_int64),
                ("constraint_rows", C.c_int64), ("omega_tilde", C.c_double), ("iterations", C.c_int64),
                ("kappa", C.c_double), ("converged", C.c_int), ("leaf_factor_seconds", C.c_double),
                ("leaf_flops", C.c_double)]


class _Row(C.Structure):
    _fields_ = [("omega_tilde", C.c_double), ("constraint_rows", C.c_int64), ("kappa", C.c_double),
                ("iterations", C.c_int64), ("converged", C.c_int),
                ("seconds_analysis", C.c_double), ("seconds_factorization", C.c_double),
                ("seconds_iterations", C.c_double), ("seconds_total", C.c_double),
                ("seconds_eigen", C.c_double), ("seconds_preconditioner", C.c_double),
                ("root_size", C.c_int64)]


P = C.c_void_p
D = C.POINTER(C.c_double)
I64 = C.POINTER(C.c_int64)
EXPORTS = {
    "bddc_b200_last_error": (C.c_char_p, []),
    "bddc_b200_device_count": (C.c_int, []),
    "bddc_b200_set_device": (C.c_int, [C.c_int]),
    "bddc_b200_create": (C.c_int, [C.POINTER(_Problem), C.POINTER(P)]),
    "bddc_b200_create_config": (C.c_int, [C.c_int, C.c_uint64, C.POINTER(C.c_int), C.c_int, C.POINTER(P)]),
    "bddc_b200_destroy": (None, [P]),
    "bddc_b200_structure_get": (C.c_int, [P, C.POINTER(_Structure)]),
    "bddc_b200_interface_dofs": (C.c_int, [P, I64]),
    "bddc_b200_subdomain_dim": (C.c_int, [P, C.c_int, I64]),
    "bddc_b200_local_to_wc": (C.c_int, [P, C.c_int, I64]),
    "bddc_b200_global_dof": (C.c_int, [P, C.c_int, I64]),
    "bddc_b200_element_scale": (C.c_int, [P, D]),
    "bddc_b200_subdomain_matrix": (C.c_int, [P, C.c_int, I64, I64, I64, D, D]),
    "bddc_b200_leaf_front": (C.c_int, [P, C.c_int, I64, D, I64]),
    "bddc_b200_nccl_unique_id": (C.c_int, [C.c_char_p]),
    "bddc_b200_shard_nccl": (C.c_int, [P, C.c_char_p, C.c_int, C.c_int, C.POINTER(C.c_int)]),
    "bddc_b200_shard_loopback": (C.c_int, [P, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int)]),
    "bddc_b200_subdomain_lattice": (C.c_int, [P, I64]),
    "bddc_b200_primal_tree_plan": (C.c_int, [P, C.POINTER(C.c_int), C.c_int, C.c_int, C.c_int, I64, I64, I64, I64,
                                            C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int),
                                            C.POINTER(C.c_int)]),
    "bddc_b200_halo_plan": (C.c_int, [P, C.POINTER(C.c_int), C.c_int, C.c_int, I64, I64, C.POINTER(C.c_int),
                                      C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int),
                                      C.POINTER(C.c_int)]),
    "bddc_b200_glob_count": (C.c_int, [P, I64]),
    "bddc_b200_glob_info": (C.c_int, [P, C.c_int, C.POINTER(C.c_int), I64, I64]),
    "bddc_b200_glob_nodes": (C.c_int, [P, C.c_int, I64, I64]),
    "bddc_b200_constraints_arithmetic": (C.c_int, [P, C.c_int, C.c_int]),
    "bddc_b200_constraint_rows": (C.c_int, [P, I64]),
    "bddc_b200_constraint_count": (C.c_int, [P, I64]),
    "bddc_b200_constraint_get": (C.c_int, [P, C.c_int, C.POINTER(C.c_int), I64, D]),
    "bddc_b200_analysis": (C.c_int, [P]),
    "bddc_b200_enrich": (C.c_int, [P, C.c_double, C.c_int, C.c_int, C.c_int, C.c_int, D]),
    "bddc_b200_pair_count": (C.c_int, [P, I64]),
    "bddc_b200_pair_report": (C.c_int, [P, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                        C.POINTER(C.c_int), D, C.POINTER(C.c_int), I64, D]),
    "bddc_b200_setup_preconditioner": (C.c_int, [P]),
    "bddc_b200_setup_preconditioner_t": (C.c_int, [P, C.c_double]),
    "bddc_b200_stabilization_t": (C.c_int, [P, D]),
    "bddc_b200_stabilized": (C.c_int, [P, I64, I64, I64, I64, D]),
    "bddc_b200_export_matrix_market": (C.c_int, [P, C.c_char_p]),
    "bddc_b200_glob_transform": (C.c_int, [P, C.c_int, C.POINTER(C.c_int), I64, D]),
    "bddc_b200_constraints_clear": (C.c_int, [P]),
    "bddc_b200_constraint_add": (C.c_int, [P, C.c_int, D, C.c_int64, C.c_int, C.POINTER(C.c_int)]),
    "bddc_b200_interface_size": (C.c_int, [P, I64]),
    "bddc_b200_schur_apply": (C.c_int, [P, D, D]),
    "bddc_b200_precond_apply": (C.c_int, [P, D, D]),
    "bddc_b200_restrict_residual": (C.c_int, [P, D, D]),
    "bddc_b200_coarse_solve": (C.c_int, [P, D, D]),
    "bddc_b200_prolong": (C.c_int, [P, D, D]),
    "bddc_b200_operator_times": (C.c_int, [P, C.c_int, D]),
    "bddc_b200_rhs": (C.c_int, [P, D]),
    "bddc_b200_recover": (C.c_int, [P, D, D]),
    "bddc_b200_pcg": (C.c_int, [P, D, D, C.c_double, C.c_int, C.c_int, C.POINTER(_PcgResult), D, D]),
    "bddc_b200_run_item": (C.c_int, [P, C.c_char_p, C.c_double, C.c_int, C.c_int, C.c_int,
                                     C.POINTER(_Row)]),
    "bddc_b200_times": (C.c_int, [P, D]),
    "bddc_b200_step": (C.c_int, [P, C.c_char_p, C.c_double, C.c_int, C.c_int, C.c_int, C.c_int, D,
                                 C.c_void_p]),
    "bddc_b200_launch_count": (C.c_int64, []),
    "bddc_b200_lanczos": (C.c_int, [D, D, C.c_int64, D]),
}

_lib = None


def load_library(build: bool = False):
    """Load `libbddc_b200.so` (building it first when asked).  Fails loudly."""
    global _lib
    if _lib is not None:
        return _lib
    if build or not LIB_PATH.exists():
        from . import build as _build
        _build.build()
    if not LIB_PATH.exists():
        raise ImportError("libbddc_b200.so is missing; run paper_0910_5863_b200/build.py")
    lib = C.CDLL(str(LIB_PATH))
    for name, (res, args) in EXPORTS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _check(rc: int):
    if rc != 0:
        raise BddcError(rc, _lib.bddc_b200_last_error().decode())


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(D)


def _iptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int))


FACES = {"xmin": 0, "xmax": 1, "ymin": 2, "ymax": 3, "zmin": 4, "zmax": 5}


@dataclass
class Problem:
    """ProblemSpec (`problem.hpp:43-53`) plus the per-element coefficient extension."""
    subdomains: Sequence[int] = (1, 1, 1)
    elements_per_edge: int = 1
    physics: str = "scalar"
    materials: dict = field(default_factory=lambda: {0: (1.0, 1.0, 0.3)})  # id -> (k, E, nu)
    regions: list = field(default_factory=list)       # (lo(3), hi(3), material)
    dirichlet: list = field(default_factory=list)     # (face, (bool, bool, bool))
    loads: list = field(default_factory=list)         # (face, traction(3), flux)
    body_force: Sequence[float] = (0.0, 0.0, 0.0)
    source: float = 0.0
    tolerance: float = 1e-8
    max_iterations: int = 500
    element_scale: Optional[np.ndarray] = None

    @staticmethod
    def cube(subdomains, elements_per_edge, physics, clamp=True, clamp_face="xmin",
             load_face="xmax") -> "Problem":
        """`tests/support.hpp:32-48`."""
        p = Problem(tuple(subdomains), elements_per_edge, physics)
        if clamp:
            p.dirichlet.append((clamp_face, (True, True, True)))
        p.loads.append((load_face, (0.0, 0.0, -1.0), 1.0))
        return p


@dataclass
class Row:
    """ResultRow (`experiment.hpp:37-46`)."""
    label: str
    omega_tilde: float
    constraint_rows: int
    kappa: float
    iterations: int
    converged: bool
    seconds_analysis: float
    seconds_factorization: float
    seconds_iterations: float
    seconds_total: float
    seconds_eigen: float = 0.0
    seconds_preconditioner: float = 0.0
    root_size: int = 0


def lanczos_condition_estimate(alphas, betas) -> float:
    """`pcg.cpp:11-26` through the library's host implementation."""
    lib = load_library()
    a = np.ascontiguousarray(alphas, dtype=np.float64)
    b = np.ascontiguousarray(betas, dtype=np.float64)
    k = C.c_double()
    _check(lib.bddc_b200_lanczos(_dptr(a), _dptr(b), len(a), C.byref(k)))
    return k.value


def emit_table(rows: List[Row], fmt="csv", include_times=True) -> str:
    """`experiment.cpp:222-278` (kappa to 4 significant digits)."""
    header = ["mode_or_tau", "omega_tilde", "Nc", "kappa", "it"]
    if include_times:
        header += ["analysis_s", "factorization_s", "iterations_s", "total_s"]
    body = []
    for r in rows:
        cells = [r.label, "" if math.isnan(r.omega_tilde) else "%.4g" % r.omega_tilde,
                 str(r.constraint_rows), "%.4g" % r.kappa,
                 str(r.iterations) + ("" if r.converged else "*")]
        if include_times:
            cells += ["%.3f" % x for x in (r.seconds_analysis, r.seconds_factorization,
                                          r.seconds_iterations, r.seconds_total)]
        body.append(cells)
    if fmt == "csv":
        return "".join(",".join(c) + "\n" for c in [header] + body)
    line = lambda cells: "|" + "".join(" %s |" % c for c in cells) + "\n"
    return line(header) + line(["---"] * len(header)) + "".join(line(c) for c in body)


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (rank 0), to be broadcast to the other ranks."""
    buf = C.create_string_buffer(128)
    _check(load_library().bddc_b200_nccl_unique_id(buf))
    return buf.raw


class BDDC:
    """One problem instance: host substructuring + the device engine."""

    def __init__(self, problem: Optional[Problem] = None, *, config: Optional[int] = None,
                 seed: int = 20091030, subdomains=None, elements_per_edge: int = 0):
        lib = load_library()
        self._lib = lib
        h = P()
        if config is not None:
            sub = (C.c_int * 3)(*subdomains) if subdomains is not None else None
            _check(lib.bddc_b200_create_config(config, seed, sub, elements_per_edge, C.byref(h)))
        else:
            _check(lib.bddc_b200_create(C.byref(self._pack(problem)), C.byref(h)))
        self._h = h

    def _pack(self, p: Problem) -> _Problem:
        s = _Problem()
        s.subdomains[:] = list(p.subdomains)
        s.elements_per_edge = p.elements_per_edge
        s.physics = 0 if p.physics == "scalar" else 1
        keep = []

        def arr(vals, ctype):
            a = np.ascontiguousarray(np.array(vals, dtype=ctype))
            keep.append(a)
            return a.ctypes.data_as(C.POINTER(C.c_int if ctype == np.int32 else C.c_double))

        ids = sorted(p.materials)
        s.n_materials = len(ids)
        s.material_id = arr(ids, np.int32)
        s.conductivity = arr([p.materials[i][0] for i in ids], np.float64)
        s.youngs = arr([p.materials[i][1] for i in ids], np.float64)
        s.poisson = arr([p.materials[i][2] for i in ids], np.float64)
        s.n_regions = len(p.regions)
        s.region_box = arr([v for lo, hi, _ in p.regions for a in range(3) for v in (lo[a], hi[a])] or [0],
                           np.int32)
        s.region_material = arr([m for _, _, m in p.regions] or [0], np.int32)
        s.n_dirichlet = len(p.dirichlet)
        s.dirichlet_face = arr([FACES[f] for f, _ in p.dirichlet] or [0], np.int32)
        s.dirichlet_components = arr([int(c) for _, cs in p.dirichlet for c in cs] or [0], np.int32)
        s.n_loads = len(p.loads)
        s.load_face = arr([FACES[f] for f, _, _ in p.loads] or [0], np.int32)
        s.load_traction = arr([t for _, tr, _ in p.loads for t in tr] or [0.0], np.float64)
        s.load_flux = arr([fl for _, _, fl in p.loads] or [0.0], np.float64)
        s.body_force[:] = list(p.body_force)
        s.source = p.source
        s.tolerance = p.tolerance
        s.max_iterations = p.max_iterations
        if p.element_scale is not None:
            s.element_scale = arr(p.element_scale, np.float64)
        self._keep = keep
        return s

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            self._lib.bddc_b200_destroy(h)
            self._h = None

    # --- sharding over GPUs ------------------------------------
    def lattice(self):
        d = np.empty(3, dtype=np.int64)
        _check(self._lib.bddc_b200_subdomain_lattice(self._h, d.ctypes.data_as(I64)))
        return tuple(int(x) for x in d)

    def shard(self, rank: int, world: int, owner=None, backend: str = "nccl", nccl_id: bytes = None,
              group: int = 0):
        """Shard this handle: `owner` (default shard.partition of the lattice)
        assigns substructures to ranks.  backend "nccl" needs the id from
        nccl_unique_id() on rank 0, shared by the caller (torch.distributed);
        "loopback" pairs handles of one process driven by separate threads."""
        from . import shard as _shard
        if owner is None:
            owner = _shard.partition(self.lattice(), world)
        own = np.ascontiguousarray(np.asarray(owner, dtype=np.int32))
        self._owner = own
        ptr = own.ctypes.data_as(C.POINTER(C.c_int))
        if backend == "nccl":
            if nccl_id is None or len(nccl_id) != 128:
                raise ValueError("nccl backend needs the 128-byte id from nccl_unique_id()")
            _check(self._lib.bddc_b200_shard_nccl(self._h, nccl_id, rank, world, ptr))
        elif backend == "loopback":
            _check(self._lib.bddc_b200_shard_loopback(self._h, group, rank, world, ptr))
        else:
            raise ValueError("backend must be 'nccl' or 'loopback'")

    # --- structure and index maps (host) -----------------------------------
    def halo_plan(self, owner, rank: int, world: int) -> dict:
        """The sharded engine's interface halo of `rank` (host only): peers,
        per-peer shared interface dofs, touched and owned masks."""
        own = np.ascontiguousarray(owner, dtype=np.int32)
        ip = lambda a: a.ctypes.data_as(C.POINTER(C.c_int))  # noqa: E731
        npeer, nsh = C.c_int64(), C.c_int64()
        _check(self._lib.bddc_b200_halo_plan(self._h, ip(own), rank, world, C.byref(npeer), C.byref(nsh),
                                             None, None, None, None, None))
        n = self.structure()["interface_dofs"]
        peers = np.empty(max(npeer.value, 1), dtype=np.int32)
        off = np.empty(npeer.value + 1, dtype=np.int32)
        sh = np.empty(max(nsh.value, 1), dtype=np.int32)
        touched = np.empty(n, dtype=np.int32)
        owned = np.empty(n, dtype=np.int32)
        _check(self._lib.bddc_b200_halo_plan(self._h, ip(own), rank, world, C.byref(npeer), C.byref(nsh), ip(peers),
                                             ip(off), ip(sh), ip(touched), ip(owned)))
        peers = peers[:npeer.value]
        return {"peers": peers.tolist(), "touched": touched.astype(bool), "owned": owned.astype(bool),
                "shared": {int(p): sh[off[k]:off[k + 1]].copy() for k, p in enumerate(peers)}}

    def primal_tree_plan(self, owner, rank: int, world: int, depth: int) -> dict:
        """Primal-tree plan of `rank` (host only): the top front's unknowns and,
        deepest level first, the unknowns each of the rank's own fronts
        eliminates (the distributed tree of the sharded engine; world 1 = the
        single-GPU plan)."""
        own = np.ascontiguousarray(owner, dtype=np.int32)
        ip = lambda a: a.ctypes.data_as(C.POINTER(C.c_int))  # noqa: E731
        d, nt, nf, no = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        args = (self._h, ip(own), rank, world, depth, C.byref(d), C.byref(nt), C.byref(nf), C.byref(no))
        _check(self._lib.bddc_b200_primal_tree_plan(*args, None, None, None, None))
        top = np.empty(max(nt.value, 1), dtype=np.int32)
        level = np.empty(max(nf.value, 1), dtype=np.int32)
        ptr = np.empty(nf.value + 1, dtype=np.int32)
        fown = np.empty(max(no.value, 1), dtype=np.int32)
        _check(self._lib.bddc_b200_primal_tree_plan(*args, ip(top), ip(level), ip(ptr), ip(fown)))
        return {"depth": d.value, "top": top[:nt.value].copy(),
                "fronts": [(int(level[f]), fown[ptr[f]:ptr[f + 1]].copy()) for f in range(nf.value)]}

    def structure(self) -> dict:
        s = _Structure()
        _check(self._lib.bddc_b200_structure_get(self._h, C.byref(s)))
        return {n: getattr(s, n) for n, _ in _Structure._fields_}

    def interface_dofs(self) -> np.ndarray:
        n = self.structure()["interface_dofs"]
        out = np.empty(n, dtype=np.int64)
        _check(self._lib.bddc_b200_interface_dofs(self._h, out.ctypes.data_as(I64)))
        return out

    def _sub_array(self, fn, s):
        dim = C.c_int64()
        _check(self._lib.bddc_b200_subdomain_dim(self._h, s, C.byref(dim)))
        out = np.empty(dim.value, dtype=np.int64)
        _check(fn(self._h, s, out.ctypes.data_as(I64)))
        return out

    def local_to_wc(self, s) -> np.ndarray:
        return self._sub_array(self._lib.bddc_b200_local_to_wc, s)

    def global_dof(self, s) -> np.ndarray:
        return self._sub_array(self._lib.bddc_b200_global_dof, s)

    def element_scale(self) -> np.ndarray:
        out = np.empty(self.structure()["elements"])
        _check(self._lib.bddc_b200_element_scale(self._h, _dptr(out)))
        return out

    def subdomain_matrix(self, s):
        """(scipy.sparse.csr_matrix, load) of substructure s."""
        import scipy.sparse as sp
        nnz = C.c_int64()
        _check(self._lib.bddc_b200_subdomain_matrix(self._h, s, C.byref(nnz), None, None, None, None))
        dim = C.c_int64()
        _check(self._lib.bddc_b200_subdomain_dim(self._h, s, C.byref(dim)))
        ptr = np.empty(dim.value + 1, dtype=np.int64)
        idx = np.empty(nnz.value, dtype=np.int64)
        val = np.empty(nnz.value)
        load = np.empty(dim.value)
        _check(self._lib.bddc_b200_subdomain_matrix(self._h, s, C.byref(nnz), ptr.ctypes.data_as(I64),
                                                    idx.ctypes.data_as(I64), _dptr(val), _dptr(load)))
        return sp.csr_matrix((val, idx, ptr), shape=(dim.value, dim.value)), load

    def leaf_front(self, s):
        """(dense front ld x ld as assembled on the device, position of each local dof)."""
        ld = C.c_int64()
        _check(self._lib.bddc_b200_leaf_front(self._h, s, C.byref(ld), None, None))
        dim = C.c_int64()
        _check(self._lib.bddc_b200_subdomain_dim(self._h, s, C.byref(dim)))
        front = np.empty(ld.value * ld.value)
        pos = np.empty(dim.value, dtype=np.int64)
        _check(self._lib.bddc_b200_leaf_front(self._h, s, C.byref(ld), _dptr(front), pos.ctypes.data_as(I64)))
        return front.reshape(ld.value, ld.value).T, pos

    def globs(self):
        n = C.c_int64()
        _check(self._lib.bddc_b200_glob_count(self._h, C.byref(n)))
        out = []
        for g in range(n.value):
            kind, nn, ns = C.c_int(), C.c_int64(), C.c_int64()
            _check(self._lib.bddc_b200_glob_info(self._h, g, C.byref(kind), C.byref(nn), C.byref(ns)))
            nodes = np.empty(nn.value, dtype=np.int64)
            subs = np.empty(ns.value, dtype=np.int64)
            _check(self._lib.bddc_b200_glob_nodes(self._h, g, nodes.ctypes.data_as(I64),
                                                   subs.ctypes.data_as(I64)))
            out.append((("corner", "edge", "face")[kind.value], nodes.tolist(), tuple(subs.tolist())))
        return out

    # --- constraints (constraints.cpp) --------------------------------------
    def arithmetic_constraints(self, edge_globs: bool, face_globs: bool):
        _check(self._lib.bddc_b200_constraints_arithmetic(self._h, int(edge_globs), int(face_globs)))

    def constraint_rows(self) -> int:
        r = C.c_int64()
        _check(self._lib.bddc_b200_constraint_rows(self._h, C.byref(r)))
        return r.value

    def constraints(self):
        n = C.c_int64()
        _check(self._lib.bddc_b200_constraint_count(self._h, C.byref(n)))
        out = []
        for a in range(n.value):
            g, nw = C.c_int(), C.c_int64()
            _check(self._lib.bddc_b200_constraint_get(self._h, a, C.byref(g), C.byref(nw), None))
            w = np.empty(nw.value)
            _check(self._lib.bddc_b200_constraint_get(self._h, a, C.byref(g), C.byref(nw), _dptr(w)))
            out.append((g.value, w))
        return out

    # --- device path ---------------------------------------------------------
    def analysis(self):
        _check(self._lib.bddc_b200_analysis(self._h))

    def enrich(self, tau=10.0, max_vectors=15, keep_edge=False, fixed_count=-1,
               indicator_only=False) -> float:
        om = C.c_double()
        _check(self._lib.bddc_b200_enrich(self._h, tau, max_vectors, int(keep_edge), fixed_count,
                                          int(indicator_only), C.byref(om)))
        return om.value

    def pair_reports(self):
        n = C.c_int64()
        _check(self._lib.bddc_b200_pair_count(self._h, C.byref(n)))
        out = []
        for k in range(n.value):
            si, sj, enf, sat = C.c_int(), C.c_int(), C.c_int(), C.c_int()
            om, ne = C.c_double(), C.c_int64()
            _check(self._lib.bddc_b200_pair_report(self._h, k, C.byref(si), C.byref(sj), C.byref(enf),
                                                   C.byref(om), C.byref(sat), C.byref(ne), None))
            ev = np.empty(ne.value)
            _check(self._lib.bddc_b200_pair_report(self._h, k, C.byref(si), C.byref(sj), C.byref(enf),
                                                   C.byref(om), C.byref(sat), C.byref(ne), _dptr(ev)))
            out.append(dict(si=si.value, sj=sj.value, enforced=enf.value, omega_next=om.value,
                            saturated=bool(sat.value), eigenvalues=ev))
        return out

    def setup_preconditioner(self, t: float = -1.0):
        """BddcPreconditioner(systems, maps, averaging, cov, t) (bddc_operator.cpp:38-50)."""
        _check(self._lib.bddc_b200_setup_preconditioner_t(self._h, t))

    def stabilization_t(self) -> float:
        t = C.c_double()
        _check(self._lib.bddc_b200_stabilization_t(self._h, C.byref(t)))
        return t.value

    def stabilized(self):
        """The stabilized operator A~ (scipy CSR, full symmetric), formed on the host."""
        import scipy.sparse as sp
        n, nnz = C.c_int64(), C.c_int64()
        _check(self._lib.bddc_b200_stabilized(self._h, C.byref(n), C.byref(nnz), None, None, None))
        ptr = np.empty(n.value + 1, dtype=np.int64)
        idx = np.empty(nnz.value, dtype=np.int64)
        val = np.empty(nnz.value)
        _check(self._lib.bddc_b200_stabilized(self._h, C.byref(n), C.byref(nnz), ptr.ctypes.data_as(I64),
                                              idx.ctypes.data_as(I64), _dptr(val)))
        return sp.csr_matrix((val, idx, ptr), shape=(n.value, n.value))

    def glob_transform(self, glob: int):
        """(rank, t) of the glob under the current constraint set (transform.cpp:51-90)."""
        r, n = C.c_int(), C.c_int64()
        _check(self._lib.bddc_b200_glob_transform(self._h, glob, C.byref(r), C.byref(n), None))
        t = np.empty((n.value, n.value))
        _check(self._lib.bddc_b200_glob_transform(self._h, glob, C.byref(r), C.byref(n), _dptr(t)))
        return r.value, t

    def export_matrix_market(self, stem: str):
        _check(self._lib.bddc_b200_export_matrix_market(self._h, stem.encode()))

    def clear_constraints(self):
        _check(self._lib.bddc_b200_constraints_clear(self._h))

    def add_average(self, glob: int, weights, adaptive: bool = False) -> bool:
        """add_average (constraints.cpp:61-76): True when kept by the rank filter."""
        w = np.ascontiguousarray(weights, dtype=np.float64)
        kept = C.c_int()
        _check(self._lib.bddc_b200_constraint_add(self._h, glob, _dptr(w), len(w), int(adaptive), C.byref(kept)))
        return bool(kept.value)

    @property
    def interface_size(self) -> int:
        n = C.c_int64()
        _check(self._lib.bddc_b200_interface_size(self._h, C.byref(n)))
        return n.value

    def schur_apply(self, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty_like(x)
        _check(self._lib.bddc_b200_schur_apply(self._h, _dptr(x), _dptr(y)))
        return y

    def precond_apply(self, r: np.ndarray) -> np.ndarray:
        r = np.ascontiguousarray(r, dtype=np.float64)
        z = np.empty_like(r)
        _check(self._lib.bddc_b200_precond_apply(self._h, _dptr(r), _dptr(z)))
        return z

    def restrict_residual(self, r: np.ndarray) -> np.ndarray:
        """`BddcPreconditioner::restrict_residual` (`bddc_operator.cpp:52-68`): interface -> W^c."""
        r = np.ascontiguousarray(r, dtype=np.float64)
        wc = np.empty(self.structure()["coarse_space_dim"])
        _check(self._lib.bddc_b200_restrict_residual(self._h, _dptr(r), _dptr(wc)))
        return wc

    def coarse_solve(self, wc_residual: np.ndarray) -> np.ndarray:
        """`BddcPreconditioner::coarse_solve` (`bddc_operator.cpp:70-85`): W^c -> W^c."""
        w = np.ascontiguousarray(wc_residual, dtype=np.float64)
        out = np.empty_like(w)
        _check(self._lib.bddc_b200_coarse_solve(self._h, _dptr(w), _dptr(out)))
        return out

    def prolong(self, wc: np.ndarray) -> np.ndarray:
        """`BddcPreconditioner::prolong` (`bddc_operator.cpp:87-99`): W^c -> interface."""
        w = np.ascontiguousarray(wc, dtype=np.float64)
        z = np.empty(self.interface_size)
        _check(self._lib.bddc_b200_prolong(self._h, _dptr(w), _dptr(z)))
        return z

    def operator_times(self, reps: int = 10) -> dict:
        """Device-timed Schur and preconditioner applications (seconds per
        application) with the preconditioner's stages and algorithmic bytes."""
        out = np.zeros(13)
        _check(self._lib.bddc_b200_operator_times(self._h, reps, _dptr(out)))
        keys = ("schur", "precond", "restrict", "leaf_fwd", "tree_fwd", "root", "tree_bwd", "leaf_bwd",
                "prolong", "sum_copies", "schur_bytes", "precond_bytes", "leaf_sweep_bytes")
        return dict(zip(keys, out.tolist()))

    def rhs(self) -> np.ndarray:
        out = np.empty(self.interface_size)
        _check(self._lib.bddc_b200_rhs(self._h, _dptr(out)))
        return out

    def recover(self, u_interface: np.ndarray) -> np.ndarray:
        u_interface = np.ascontiguousarray(u_interface, dtype=np.float64)
        out = np.empty(self.structure()["free_dofs"])
        _check(self._lib.bddc_b200_recover(self._h, _dptr(u_interface), _dptr(out)))
        return out

    def pcg(self, b: Optional[np.ndarray] = None, tolerance=1e-8, max_iterations=500,
            preconditioned_residual=False):
        """Returns (x, iterations, relres, kappa, converged, alphas, betas)."""
        n = self.interface_size
        x = np.empty(n)
        res = _PcgResult()
        al = np.empty(max_iterations + 1)
        be = np.empty(max_iterations + 1)
        bp = None
        if b is not None:
            b = np.ascontiguousarray(b, dtype=np.float64)
            bp = _dptr(b)
        rc = self._lib.bddc_b200_pcg(self._h, bp, _dptr(x), tolerance, max_iterations,
                                     int(preconditioned_residual), C.byref(res), _dptr(al), _dptr(be))
        if rc not in (0, 9):
            _check(rc)
        it = res.iterations
        return dict(x=x, iterations=it, relative_residual=res.relative_residual,
                    condition_estimate=res.condition_estimate, converged=bool(res.converged),
                    alphas=al[:it].copy(), betas=be[:it].copy())

    def run_item(self, mode: str, tau: float = 10.0, max_vectors: int = 15, keep_edge=False,
                 base_faces=False) -> Row:
        """One work item of `run_items` (`experiment.cpp:143-205`)."""
        r = _Row()
        _check(self._lib.bddc_b200_run_item(self._h, mode.encode(), tau, max_vectors, int(keep_edge),
                                            int(base_faces), C.byref(r)))
        label = ("inf" if math.isinf(tau) else "%.4g" % tau) if mode == "adaptive" else mode
        return Row(label, r.omega_tilde, r.constraint_rows, r.kappa, r.iterations, bool(r.converged),
                   r.seconds_analysis, r.seconds_factorization, r.seconds_iterations, r.seconds_total,
                   r.seconds_eigen, r.seconds_preconditioner, r.root_size)

    def times(self) -> dict:
        out = np.zeros(11)
        _check(self._lib.bddc_b200_times(self._h, _dptr(out)))
        keys = ("analysis", "eigen", "preconditioner", "pcg", "leaf_flops", "leaf_front_bytes",
                "schur_bytes", "root_size", "leaf_factor", "pcg_iterations", "pcg_bytes_per_iteration")
        return dict(zip(keys, out.tolist()))

    def step(self, mode: str, tau: float = 10.0, max_vectors: int = 15, keep_edge=False,
             base_faces=False, e2e=False, u_free: Optional[np.ndarray] = None) -> dict:
        """One device-timed pass of the hot path (see `bddc_b200_step`)."""
        o = _StepOut()
        up = _dptr(u_free) if u_free is not None else None
        _check(self._lib.bddc_b200_step(self._h, mode.encode(), tau, max_vectors, int(keep_edge),
                                        int(base_faces), int(e2e), up, C.byref(o)))
        return {n: getattr(o, n) for n, _ in _StepOut._fields_}

    @staticmethod
    def launch_count() -> int:
        return load_library().bddc_b200_launch_count()
