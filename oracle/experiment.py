"""Oracle: the experiment driver, result tables, and the BASELINE.json configs.

Restates `core/src/experiment.cpp` (modes, phase timers, table format) and
`tests/support.hpp` (fixtures).  The seeded coefficient fields for configs 2-5
follow the generator specified in DESIGN.md ("Synthetic inputs"); the C++
product host implements the same generator bit-for-bit (checked by
tests/test_host_parity.py).  TEST INFRASTRUCTURE ONLY (see oracle/__init__).
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import fem
from .adaptive import EnrichmentOptions, enrich_constraints
from .bddc import BddcPreconditioner, pcg
from .constraints import ConstraintSet, arithmetic_constraints, change_of_variables
from .fem import (DirichletSpec, LoadSpec, Material, ProblemSpec, apply_dirichlet,
                  assemble_subdomains, build_cube_mesh, decompose_cube)
from .globs import CORNER, EDGE, FACE, classify_globs, select_corners
from .spaces import AveragingOperator, HarmonicExtension, InterfaceProblem, build_embeddings

MODES = ("c", "c+e", "c+e+f", "c+e+f-3eigv", "adaptive")


@dataclass
class Pipeline:
    """`tests/support.hpp:80-100`."""
    spec: ProblemSpec
    mesh: fem.Mesh
    deco: fem.Decomposition
    dmap: fem.DofMap
    systems: list
    globset: object
    maps: object
    classification_corners: int = 0


def build_pipeline(spec: ProblemSpec, promote_corners=True) -> Pipeline:
    """`experiment.cpp:116-128` / `support.hpp:89-100`."""
    mesh = build_cube_mesh(spec.subdomains, spec.elements_per_edge, spec.physics, spec.regions)
    deco = decompose_cube(mesh, spec.subdomains)
    dmap = apply_dirichlet(mesh, spec.dirichlet)
    systems = assemble_subdomains(mesh, deco, dmap, spec)
    gs = classify_globs(mesh, deco)
    ccount = gs.classification_corner_count
    if promote_corners:
        select_corners(gs, mesh, deco)
    maps = build_embeddings(systems, dmap.free_count, gs, dmap)
    return Pipeline(spec, mesh, deco, dmap, systems, gs, maps, ccount)


def cube_spec(subdomains, elements_per_edge, physics, clamp=True, clamp_face="xmin",
              load_face="xmax") -> ProblemSpec:
    """`tests/support.hpp:32-48`."""
    spec = ProblemSpec(subdomains=tuple(subdomains), elements_per_edge=elements_per_edge,
                       physics=physics)
    if clamp:
        spec.dirichlet.append(DirichletSpec(clamp_face, (True, True, True)))
    spec.loads.append(LoadSpec(load_face, (0.0, 0.0, -1.0), 1.0))
    return spec


def constraint_set_for(p: Pipeline, mode: str, base_faces=False) -> ConstraintSet:
    """`experiment.cpp:150-153`: the adaptive base is c+e unless base_faces."""
    edges = mode != "c"
    faces = mode == "c+e+f" or (mode in ("adaptive", "c+e+f-3eigv") and base_faces)
    return arithmetic_constraints(p.globset, p.dmap, edges, faces)


@dataclass
class ResultRow:
    """`experiment.hpp:37-46`."""
    label: str
    omega_tilde: float = float("nan")
    constraint_rows: int = 0
    kappa: float = 1.0
    iterations: int = 0
    converged: bool = True
    seconds_analysis: float = 0.0
    seconds_factorization: float = 0.0
    seconds_iterations: float = 0.0
    seconds_total: float = 0.0
    # extras for parity checks
    pcg: object = None
    outcome: object = None
    constraints: object = None


def tau_label(tau: float) -> str:
    """`experiment.cpp:50-56`: precision(4) general format."""
    if math.isinf(tau):
        return "inf"
    return "%.4g" % tau


def solve_item(p: Pipeline, mode: str, tau: float = 10.0, max_vectors=15, keep_edge=False,
               base_faces=False, analysis=None, log=None) -> ResultRow:
    """One work item of `experiment.cpp:143-205`."""
    t0 = time.perf_counter()
    if analysis is None:
        harmonic = HarmonicExtension(p.systems, p.maps)
        averaging = AveragingOperator(p.systems, p.maps)
        interface = InterfaceProblem(p.systems, p.maps, harmonic)
    else:
        harmonic, averaging, interface = analysis
    t_an = time.perf_counter() - t0
    row = ResultRow(tau_label(tau) if mode == "adaptive" else mode)
    t1 = time.perf_counter()
    cs = constraint_set_for(p, mode, base_faces)
    if mode in ("adaptive", "c+e+f-3eigv"):
        opts = EnrichmentOptions(tau=tau, max_vectors=max_vectors, keep_edge_constraints=keep_edge)
        if mode == "c+e+f-3eigv":
            opts = EnrichmentOptions(fixed_count=3, keep_edge_constraints=keep_edge)
        row.outcome = enrich_constraints(cs, p.globset, p.dmap, p.systems, p.maps, opts)
        row.omega_tilde = row.outcome.omega_tilde
    row.constraint_rows = cs.row_count(p.globset)
    row.constraints = cs
    cov = change_of_variables(cs, p.globset, p.dmap, p.maps)
    prec = BddcPreconditioner(p.systems, p.maps, averaging, cov, -1.0)
    row.seconds_factorization = time.perf_counter() - t1
    t2 = time.perf_counter()
    res = pcg(interface.apply, prec.apply, interface.rhs(), p.spec.tolerance,
              p.spec.max_iterations, log=log)
    row.seconds_iterations = time.perf_counter() - t2
    row.kappa, row.iterations, row.converged, row.pcg = (res.condition_estimate, res.iterations,
                                                         res.converged, res)
    row.seconds_analysis = t_an
    row.seconds_total = t_an + row.seconds_factorization + row.seconds_iterations
    return row


def run_experiment(spec: ProblemSpec, modes, tau_list=(), max_vectors=15, keep_edge=False,
                   base_faces=False):
    """`experiment.cpp:109-220`."""
    items = []
    for m in modes:
        if m not in MODES:
            raise ValueError("unknown constraint mode '%s'" % m)
        if m == "adaptive":
            if not tau_list:
                raise ValueError("adaptive mode requires a nonempty tau list")
            items += [(m, t) for t in tau_list]
        else:
            items.append((m, 0.0))
    if not items:
        raise ValueError("no constraint modes requested")
    t0 = time.perf_counter()
    p = build_pipeline(spec)
    analysis = (HarmonicExtension(p.systems, p.maps), AveragingOperator(p.systems, p.maps))
    analysis = analysis + (InterfaceProblem(p.systems, p.maps, analysis[0]),)
    t_an = time.perf_counter() - t0
    rows = []
    for m, tau in items:
        r = solve_item(p, m, tau, max_vectors, keep_edge, base_faces, analysis)
        r.seconds_analysis = t_an
        r.seconds_total = t_an + r.seconds_factorization + r.seconds_iterations
        rows.append(r)
    return p, rows


def emit_table(rows, fmt="csv", include_times=True) -> str:
    """`experiment.cpp:222-278`."""
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


# --- BASELINE.json configs -------------------

_M64 = (1 << 64) - 1


class SplitMix64:
    """splitmix64; identical to the C++ host generator."""

    def __init__(self, seed: int):
        self.state = seed & _M64

    def next(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & _M64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
        return z ^ (z >> 31)

    def uniform(self) -> float:
        return (self.next() >> 11) * (1.0 / 9007199254740992.0)

    def normal(self) -> float:
        u1 = 1.0 - self.uniform()
        u2 = self.uniform()
        return math.sqrt(-2.0 * math.log(u1)) * math.cos(2.0 * math.pi * u2)


CONFIG_SEED = 20091030


def element_scale_for(config: int, ne, seed: int = CONFIG_SEED) -> Optional[np.ndarray]:
    """Per-element coefficient multipliers for BASELINE.json configs 2-5."""
    nx, ny, nz = ne
    if config == 1:
        return None
    rng = SplitMix64(seed)
    if config == 2:
        col = np.zeros((ny, nx), dtype=bool)
        for j in range(ny):
            for i in range(nx):
                col[j, i] = rng.uniform() < 0.1
        scale = np.where(col, 1e6, 1.0)
        return np.broadcast_to(scale[None, :, :], (nz, ny, nx)).ravel().copy()
    if config == 3:
        n = nx * ny * nz
        return np.array([math.exp(2.0 * rng.normal()) for _ in range(n)])
    if config == 4:
        spheres = []
        for _ in range(20):
            cx, cy, cz = rng.uniform(), rng.uniform(), rng.uniform()
            r = 0.05 + 0.05 * rng.uniform()
            spheres.append((cx, cy, cz, r))
        k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
        x = (i.ravel() + 0.5) / nx
        y = (j.ravel() + 0.5) / ny
        z = (k.ravel() + 0.5) / nz
        inside = np.zeros(x.shape, dtype=bool)
        for cx, cy, cz, r in spheres:
            dx, dy, dz = x - cx, y - cy, z - cz
            inside |= (dx * dx + dy * dy + dz * dz) < r * r
        return np.where(inside, 1e4, 1.0)
    if config == 5:
        k = np.arange(nx * ny * nz) // (nx * ny)
        return np.where((k // 3) % 2 == 1, 1e5, 1.0)
    raise ValueError("unknown config %d" % config)


@dataclass
class ConfigSpec:
    config: int
    spec: ProblemSpec
    mode: str
    tau: float = 10.0
    max_vectors: int = 15
    base_faces: bool = False


def baseline_config(config: int, seed: int = CONFIG_SEED, subdomains=None,
                    elements_per_edge=None) -> ConfigSpec:
    """BASELINE.json `configs[config-1]` (optionally shrunk for parity tests)."""
    table = {1: ((3, 3, 3), 8, fem.SCALAR), 2: ((3, 3, 3), 8, fem.SCALAR),
             3: ((8, 8, 8), 10, fem.SCALAR), 4: ((6, 6, 6), 8, fem.ELASTICITY),
             5: ((12, 12, 12), 8, fem.ELASTICITY)}
    subs, epe, phys = table[config]
    subs = tuple(subdomains) if subdomains is not None else subs
    epe = elements_per_edge if elements_per_edge is not None else epe
    spec = ProblemSpec(subdomains=subs, elements_per_edge=epe, physics=phys)
    spec.dirichlet.append(DirichletSpec("xmin", (True, True, True)))
    if phys == fem.SCALAR:
        spec.source = 1.0
    else:
        spec.materials = {0: Material(1.0, 1.0, 0.3)}
        spec.body_force = (0.0, 0.0, -1.0)
    ne = tuple(s * epe for s in subs)
    spec.element_scale = element_scale_for(config, ne, seed)
    if config == 1:
        return ConfigSpec(1, spec, "c+e+f")
    if config == 2:
        return ConfigSpec(2, spec, "adaptive", tau=10.0, max_vectors=10)
    if config == 3:
        return ConfigSpec(3, spec, "adaptive", tau=5.0, max_vectors=15)
    if config == 4:
        return ConfigSpec(4, spec, "adaptive", tau=10.0, max_vectors=15, base_faces=True)
    return ConfigSpec(5, spec, "adaptive", tau=10.0, max_vectors=15)
