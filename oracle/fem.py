"""Oracle: structured mesh, decomposition, Dirichlet elimination, Q1 assembly.

Restates `core/src/mesh.cpp`, `core/src/assemble.cpp` and the `ProblemSpec`
of `core/include/bddc/problem.hpp`.  TEST INFRASTRUCTURE ONLY (see oracle/__init__).

Extension (SURVEY.md section 5 "gaps"): `ProblemSpec.element_scale`, an optional
per-element multiplier of the material coefficient (conductivity or Young's
modulus).  The reference would express it as one material per element through
its `ElementMatrixCache` (`assemble.cpp:145-169`); stiffness is linear in the
coefficient, so scaling the per-material element matrix is the same operator.
"""
from __future__ import annotations

import dataclasses
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

import numpy as np
import scipy.sparse as sp

SCALAR, ELASTICITY = "scalar", "elasticity"
FACES = ("xmin", "xmax", "ymin", "ymax", "zmin", "zmax")


def components(physics: str) -> int:
    """`types.hpp:16`."""
    return 1 if physics == SCALAR else 3


@dataclass
class Material:
    """`mesh.hpp:17-21`."""
    conductivity: float = 1.0
    youngs: float = 1.0
    poisson: float = 0.3


@dataclass
class MaterialRegion:
    """Half-open element box, `mesh.hpp:25-30`."""
    lo: Tuple[int, int, int] = (0, 0, 0)
    hi: Tuple[int, int, int] = (0, 0, 0)
    material: int = 0


@dataclass
class DirichletSpec:
    """`problem.hpp:23-26`."""
    face: str = "xmin"
    constrained: Tuple[bool, bool, bool] = (True, True, True)


@dataclass
class LoadSpec:
    """`problem.hpp:28-32`."""
    face: str = "xmax"
    traction: Tuple[float, float, float] = (0.0, 0.0, 0.0)
    flux: float = 0.0


@dataclass
class ProblemSpec:
    """`problem.hpp:43-53` plus the per-element coefficient extension."""
    subdomains: Tuple[int, int, int] = (1, 1, 1)
    elements_per_edge: int = 1
    physics: str = SCALAR
    materials: Dict[int, Material] = field(default_factory=lambda: {0: Material()})
    regions: List[MaterialRegion] = field(default_factory=list)
    dirichlet: List[DirichletSpec] = field(default_factory=list)
    loads: List[LoadSpec] = field(default_factory=list)
    body_force: Tuple[float, float, float] = (0.0, 0.0, 0.0)
    source: float = 0.0
    tolerance: float = 1e-8
    max_iterations: int = 500
    element_scale: Optional[np.ndarray] = None   # extension, length = element count


@dataclass
class Mesh:
    """`mesh.hpp:34-51`.  Node ids are x-fastest (`mesh.hpp:48-50`)."""
    physics: str
    nodes_per_axis: Tuple[int, int, int]
    elements_per_axis: Tuple[int, int, int]
    h: float
    coords: np.ndarray          # (nodes, 3)
    elements: np.ndarray        # (elements, 8) VTK hexahedron order
    element_material: np.ndarray

    @property
    def node_count(self) -> int:
        return self.coords.shape[0]

    @property
    def element_count(self) -> int:
        return self.elements.shape[0]

    @property
    def total_dofs(self) -> int:
        return self.node_count * components(self.physics)

    def node_id(self, i, j, k):
        nx, ny, _ = self.nodes_per_axis
        return (k * ny + j) * nx + i


def build_cube_mesh(subdomains, elements_per_edge, physics, regions=()) -> Mesh:
    """`mesh.cpp:9-50`: unit-cube subdomains, h = 1/elements_per_edge."""
    if elements_per_edge < 1:
        raise ValueError("elements per subdomain edge must be >= 1")
    h = 1.0 / elements_per_edge
    ne = tuple(int(s) * elements_per_edge for s in subdomains)
    npa = tuple(n + 1 for n in ne)
    k, j, i = np.meshgrid(np.arange(npa[2]), np.arange(npa[1]), np.arange(npa[0]), indexing="ij")
    coords = np.stack([i.ravel() * h, j.ravel() * h, k.ravel() * h], axis=1)
    ek, ej, ei = np.meshgrid(np.arange(ne[2]), np.arange(ne[1]), np.arange(ne[0]), indexing="ij")
    ei, ej, ek = ei.ravel(), ej.ravel(), ek.ravel()

    def nid(a, b, c):
        return (c * npa[1] + b) * npa[0] + a

    elements = np.stack([nid(ei, ej, ek), nid(ei + 1, ej, ek), nid(ei + 1, ej + 1, ek),
                         nid(ei, ej + 1, ek), nid(ei, ej, ek + 1), nid(ei + 1, ej, ek + 1),
                         nid(ei + 1, ej + 1, ek + 1), nid(ei, ej + 1, ek + 1)], axis=1)
    mat = np.zeros(len(ei), dtype=np.int64)
    for r in regions:  # later regions win (`mesh.cpp:41-46`)
        inside = ((ei >= r.lo[0]) & (ei < r.hi[0]) & (ej >= r.lo[1]) & (ej < r.hi[1]) &
                  (ek >= r.lo[2]) & (ek < r.hi[2]))
        mat[inside] = r.material
    return Mesh(physics, npa, ne, h, coords, elements.astype(np.int64), mat)


@dataclass
class Decomposition:
    """`mesh.hpp:54-59`."""
    subdomains_per_axis: Tuple[int, int, int]
    subdomain_count: int
    element_subdomain: np.ndarray
    node_subdomains: List[Tuple[int, ...]]   # sorted per node


def decompose_cube(mesh: Mesh, subdomains) -> Decomposition:
    """`mesh.cpp:52-82`."""
    ne = mesh.elements_per_axis
    for a in range(3):
        if ne[a] % subdomains[a]:
            raise ValueError("element grid does not tile the requested subdomains")
    per = [ne[a] // subdomains[a] for a in range(3)]
    e = np.arange(mesh.element_count)
    i, j, k = e % ne[0], (e // ne[0]) % ne[1], e // (ne[0] * ne[1])
    esub = (k // per[2] * subdomains[1] + j // per[1]) * subdomains[0] + i // per[0]
    # node -> sorted set of subdomains of its elements
    pairs = np.unique(np.stack([mesh.elements.ravel(), np.repeat(esub, 8)], axis=1), axis=0)
    node_subs: List[list] = [[] for _ in range(mesh.node_count)]
    for n, s in pairs:
        node_subs[n].append(int(s))
    return Decomposition(tuple(subdomains), int(np.prod(subdomains)), esub,
                         [tuple(x) for x in node_subs])


# --- element matrices (`assemble.cpp:11-99`) --------------------------------

_KXI = np.array([-1, 1, 1, -1, -1, 1, 1, -1], dtype=float)
_KETA = np.array([-1, -1, 1, 1, -1, -1, 1, 1], dtype=float)
_KZETA = np.array([-1, -1, -1, -1, 1, 1, 1, 1], dtype=float)


def _gauss_2x2x2():
    g = 1.0 / np.sqrt(3.0)
    return [(a * g, b * g, c * g, 1.0) for a in (-1, 1) for b in (-1, 1) for c in (-1, 1)]


def _shape_gradients_ref(xi, eta, zeta):
    d = np.empty((8, 3))
    d[:, 0] = 0.125 * _KXI * (1 + eta * _KETA) * (1 + zeta * _KZETA)
    d[:, 1] = 0.125 * (1 + xi * _KXI) * _KETA * (1 + zeta * _KZETA)
    d[:, 2] = 0.125 * (1 + xi * _KXI) * (1 + eta * _KETA) * _KZETA
    return d


def _isotropic_tensor(m: Material):
    lam = m.youngs * m.poisson / ((1 + m.poisson) * (1 - 2 * m.poisson))
    mu = m.youngs / (2 * (1 + m.poisson))
    c = np.zeros((6, 6))
    for a in range(3):
        for b in range(3):
            c[a, b] = lam
        c[a, a] = lam + 2 * mu
        c[3 + a, 3 + a] = mu
    return c


def element_stiffness(corners: np.ndarray, material: Material, physics: str) -> np.ndarray:
    """`assemble.cpp:60-99`: trilinear hexahedron, 2x2x2 Gauss."""
    ncomp = components(physics)
    ke = np.zeros((8 * ncomp, 8 * ncomp))
    ct = _isotropic_tensor(material)
    for xi, eta, zeta, w in _gauss_2x2x2():
        dref = _shape_gradients_ref(xi, eta, zeta)
        jac = corners.T @ dref
        det = np.linalg.det(jac)
        if det <= 0:
            raise ValueError("element with nonpositive Jacobian determinant")
        grad = dref @ np.linalg.inv(jac)
        if physics == SCALAR:
            ke += material.conductivity * w * det * (grad @ grad.T)
        else:
            b = np.zeros((6, 24))
            for i in range(8):
                dx, dy, dz = grad[i]
                b[0, 3 * i], b[1, 3 * i + 1], b[2, 3 * i + 2] = dx, dy, dz
                b[3, 3 * i], b[3, 3 * i + 1] = dy, dx
                b[4, 3 * i + 1], b[4, 3 * i + 2] = dz, dy
                b[5, 3 * i], b[5, 3 * i + 2] = dz, dx
            ke += w * det * (b.T @ ct @ b)
    return ke


@dataclass
class DofMap:
    """`assemble.hpp:23-30`: node*ncomp+c -> free dof id or -1."""
    dofs_per_node: int
    free_count: int
    dof: np.ndarray

    def at(self, node, comp):
        return self.dof[node * self.dofs_per_node + comp]


def _on_face(mesh: Mesh, face: str):
    nx, ny, nz = mesh.nodes_per_axis
    n = np.arange(mesh.node_count)
    i, j, k = n % nx, (n // nx) % ny, n // (nx * ny)
    return {"xmin": i == 0, "xmax": i == nx - 1, "ymin": j == 0, "ymax": j == ny - 1,
            "zmin": k == 0, "zmax": k == nz - 1}[face]


def apply_dirichlet(mesh: Mesh, dirichlet) -> DofMap:
    """`assemble.cpp:101-141`: free dofs numbered node-major, component fastest."""
    nc = components(mesh.physics)
    fixed = np.zeros(mesh.node_count * nc, dtype=bool)
    for d in dirichlet:
        on = np.nonzero(_on_face(mesh, d.face))[0]
        for c in range(nc):
            if d.constrained[c]:
                fixed[on * nc + c] = True
    dof = np.full(mesh.node_count * nc, -1, dtype=np.int64)
    dof[~fixed] = np.arange(int((~fixed).sum()))
    return DofMap(nc, int((~fixed).sum()), dof)


@dataclass
class SubdomainSystem:
    """`assemble.hpp:41-51`."""
    subdomain: int
    nodes: np.ndarray
    global_dof: np.ndarray
    node_comp: np.ndarray
    stiffness: sp.csr_matrix     # full symmetric
    load: np.ndarray

    @property
    def dim(self):
        return len(self.global_dof)


_FACE_LOCAL_NODES = {"xmin": (0, 3, 7, 4), "xmax": (1, 2, 6, 5), "ymin": (0, 1, 5, 4),
                     "ymax": (3, 2, 6, 7), "zmin": (0, 1, 2, 3), "zmax": (4, 5, 6, 7)}


def _element_on_face(mesh: Mesh, e: np.ndarray, face: str):
    ne = mesh.elements_per_axis
    i, j, k = e % ne[0], (e // ne[0]) % ne[1], e // (ne[0] * ne[1])
    return {"xmin": i == 0, "xmax": i == ne[0] - 1, "ymin": j == 0, "ymax": j == ne[1] - 1,
            "zmin": k == 0, "zmax": k == ne[2] - 1}[face]


def element_matrices(mesh: Mesh, spec: ProblemSpec):
    """Per-material element matrix cache (`assemble.cpp:145-169`, congruent elements)."""
    cache = {}
    corners = mesh.coords[mesh.elements[0]]
    for mid in np.unique(mesh.element_material):
        if int(mid) not in spec.materials:
            raise ValueError("element references unknown material %d" % mid)
        cache[int(mid)] = element_stiffness(corners, spec.materials[int(mid)], mesh.physics)
    return cache


def assemble_subdomains(mesh: Mesh, deco: Decomposition, dmap: DofMap,
                        spec: ProblemSpec) -> List[SubdomainSystem]:
    """`assemble.cpp:202-292`: local numbering nodes ascending x components."""
    nc = components(mesh.physics)
    cache = element_matrices(mesh, spec)
    scale = spec.element_scale
    systems = []
    order = np.argsort(deco.element_subdomain, kind="stable")
    bounds = np.searchsorted(deco.element_subdomain[order], np.arange(deco.subdomain_count + 1))
    ed = 8 * nc
    ai, bi = np.meshgrid(np.arange(ed), np.arange(ed), indexing="ij")
    for s in range(deco.subdomain_count):
        elems = order[bounds[s]:bounds[s + 1]]
        conn = mesh.elements[elems]
        nodes = np.unique(conn)
        nodecomp = (nodes[:, None] * nc + np.arange(nc)[None, :]).ravel()
        free = dmap.dof[nodecomp] >= 0
        nodecomp = nodecomp[free]
        gdof = dmap.dof[nodecomp]
        n_local = len(gdof)
        # node*nc+c -> local id (nodecomp is ascending; `assemble.cpp:222-230`)
        enc = (conn[:, :, None] * nc + np.arange(nc)[None, None, :]).reshape(len(elems), ed)
        pos = np.minimum(np.searchsorted(nodecomp, enc), n_local - 1)
        local = np.where(nodecomp[pos] == enc, pos, -1).astype(np.int64)
        rows, cols, vals = [], [], []
        load = np.zeros(n_local)
        mats = mesh.element_material[elems]
        for mid in np.unique(mats):
            sel = np.nonzero(mats == mid)[0]
            ke = cache[int(mid)]
            la = local[sel][:, ai]          # (m, ed, ed)
            lb = local[sel][:, bi]
            keep = (la >= 0) & (lb >= 0) & (lb >= la)
            v = np.broadcast_to(ke, la.shape)
            if scale is not None:
                v = v * scale[elems[sel]][:, None, None]
            rows.append(la[keep]); cols.append(lb[keep]); vals.append(v[keep])
        upper = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                              shape=(n_local, n_local)).tocsr()
        upper.sum_duplicates()
        full = (upper + sp.triu(upper, k=1).T).tocsr()
        full.sort_indices()
        # body force / source: h^3/8 per element node (`assemble.cpp:260-269`)
        cell = mesh.h ** 3 / 8.0
        for c in range(nc):
            dens = spec.source if mesh.physics == SCALAR else spec.body_force[c]
            if dens != 0.0:
                lc = local[:, np.arange(8) * nc + c].ravel()
                np.add.at(load, lc[lc >= 0], dens * cell)
        # surface loads (`assemble.cpp:271-283`)
        for ls in spec.loads:
            on = _element_on_face(mesh, elems, ls.face)
            qa = mesh.h * mesh.h / 4.0
            for c in range(nc):
                t = ls.flux if mesh.physics == SCALAR else ls.traction[c]
                if t == 0.0:
                    continue
                fn = np.array(_FACE_LOCAL_NODES[ls.face]) * nc + c
                lc = local[on][:, fn].ravel()
                np.add.at(load, lc[lc >= 0], t * qa)
        systems.append(SubdomainSystem(s, nodes, gdof, nodecomp, full, load))
    return systems


def global_matrix(systems: List[SubdomainSystem], free_count: int) -> sp.csr_matrix:
    """`assemble.cpp:316-327` (subassembly sum)."""
    rows, cols, vals = [], [], []
    for sys in systems:
        c = sys.stiffness.tocoo()
        rows.append(sys.global_dof[c.row]); cols.append(sys.global_dof[c.col]); vals.append(c.data)
    return sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                         shape=(free_count, free_count)).tocsr()


def global_rhs(systems, free_count) -> np.ndarray:
    """`assemble.cpp:329-335`."""
    f = np.zeros(free_count)
    for sys in systems:
        np.add.at(f, sys.global_dof, sys.load)
    return f
