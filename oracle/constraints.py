"""Oracle: glob averages, rank filter, change of variables, group projector.

Restates `core/src/constraints.cpp` and `core/src/transform.cpp`.
TEST INFRASTRUCTURE ONLY (see oracle/__init__).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp

from .fem import DofMap, Mesh
from .globs import CORNER, EDGE, FACE, Glob, GlobSet
from .linalg import SingularGram, pivoted_qr
from .spaces import EmbeddingMaps


@dataclass
class GlobAverage:
    """`constraints.hpp:23-27`."""
    glob: int
    weights: np.ndarray
    provenance: str = "arithmetic"


@dataclass
class ConstraintSet:
    """`constraints.hpp:32-37`, `constraints.cpp:11-23`."""
    averages: List[GlobAverage] = field(default_factory=list)

    def row_count(self, gs: GlobSet) -> int:
        return sum(len(gs.globs[a.glob].subdomains) - 1 for a in self.averages)

    def by_glob(self, n_globs):
        out = [[] for _ in range(n_globs)]
        for i, a in enumerate(self.averages):
            out[a.glob].append(i)
        return out

    def copy(self):
        return ConstraintSet([GlobAverage(a.glob, a.weights.copy(), a.provenance)
                              for a in self.averages])


def glob_free_dofs(glob: Glob, dmap: DofMap) -> np.ndarray:
    """`constraints.cpp:25-32`: node-major, Dirichlet dofs skipped."""
    out = []
    for node in glob.nodes:
        for c in range(dmap.dofs_per_node):
            g = dmap.at(node, c)
            if g >= 0:
                out.append(g)
    return np.array(out, dtype=np.int64)


def arithmetic_constraints(gs: GlobSet, dmap: DofMap, edge_globs: bool,
                           face_globs: bool) -> ConstraintSet:
    """`constraints.cpp:34-59`: one unit average per component."""
    cs = ConstraintSet()
    for gi, g in enumerate(gs.globs):
        if g.kind == CORNER or (g.kind == EDGE and not edge_globs) or \
                (g.kind == FACE and not face_globs):
            continue
        comps = [c for node in g.nodes for c in range(dmap.dofs_per_node)
                 if dmap.at(node, c) >= 0]
        if not comps:
            continue
        comps = np.array(comps)
        for c in range(dmap.dofs_per_node):
            w = (comps == c).astype(float)
            if not w.any():
                continue
            cs.averages.append(GlobAverage(gi, w, "arithmetic"))
    return cs


def add_average(cs: ConstraintSet, avg: GlobAverage) -> bool:
    """`constraints.cpp:61-76`: pivoted-QR rank filter against the glob's averages."""
    if not np.any(avg.weights != 0.0):
        return False
    existing = [a.weights for a in cs.averages if a.glob == avg.glob]
    if existing:
        stack = np.column_stack(existing + [avg.weights])
        if pivoted_qr(stack).rank <= len(existing):
            return False
    cs.averages.append(avg)
    return True


def _wc_index(maps: EmbeddingMaps, g: int, s: int) -> int:
    for cs_, cl in maps.dof_copies[g]:
        if cs_ == s:
            return int(maps.local_to_wc[cs_][cl])
    raise RuntimeError("glob dof has no copy in its sharing substructure")


def constraint_matrix(cs: ConstraintSet, gs: GlobSet, dmap: DofMap,
                      maps: EmbeddingMaps) -> sp.csr_matrix:
    """`constraints.cpp:89-116`: rows ordered glob, average, sharer."""
    rows, cols, vals = [], [], []
    row = 0
    bg = cs.by_glob(len(gs.globs))
    for gi, g in enumerate(gs.globs):
        if not bg[gi]:
            continue
        dofs = glob_free_dofs(g, dmap)
        anchor = g.subdomains[0]
        for ai in bg[gi]:
            w = cs.averages[ai].weights
            for other in g.subdomains[1:]:
                for t in range(len(w)):
                    if w[t] == 0.0:
                        continue
                    rows += [row, row]
                    cols += [_wc_index(maps, dofs[t], anchor), _wc_index(maps, dofs[t], other)]
                    vals += [w[t], -w[t]]
                row += 1
    return sp.csr_matrix((vals, (rows, cols)), shape=(row, maps.wc_dim))


# --- transform.cpp -----------------------------------------------------------

@dataclass
class GlobTransform:
    """`transform.hpp:20-27`."""
    glob: int
    rank: int
    h: np.ndarray
    t: np.ndarray
    explicit_slots: List[int]


def build_glob_transform(glob: int, avg_rows: np.ndarray) -> GlobTransform:
    """`transform.cpp:51-90`."""
    r_in, n = avg_rows.shape
    qr = pivoted_qr(avg_rows)
    if qr.rank < r_in:
        raise SingularGram("dependent averages slipped past the rank filter")
    r = qr.rank
    u = qr.r[:r, :r]
    v = qr.r[:r, r:]
    h_perm = np.zeros((n, n))
    h_perm[:r, :r] = u
    h_perm[:r, r:] = v
    h_perm[r:, r:] = np.eye(n - r)
    u_inv = sla.solve_triangular(u, np.eye(r), lower=False)
    t_perm = np.zeros((n, n))
    t_perm[:r, :r] = u_inv
    t_perm[:r, r:] = -u_inv @ v
    t_perm[r:, r:] = np.eye(n - r)
    h = np.zeros((n, n))
    t = np.zeros((n, n))
    for i in range(n):
        h[:, qr.perm[i]] = h_perm[:, i]
        t[qr.perm[i], :] = t_perm[i, :]
    return GlobTransform(glob, r, h, t, list(range(r)))


@dataclass
class ChangeOfVariables:
    """`transform.hpp:47-55`."""
    glob_transforms: List[GlobTransform]
    basis: List[sp.csr_matrix]
    groups: List[List[int]]


def change_of_variables(cs: ConstraintSet, gs: GlobSet, dmap: DofMap,
                        maps: EmbeddingMaps) -> ChangeOfVariables:
    """`transform.cpp:94-149`."""
    bg = cs.by_glob(len(gs.globs))
    n_sub = len(maps.local_to_wc)
    trip = [([], [], []) for _ in range(n_sub)]
    covered = [np.zeros(len(m), dtype=bool) for m in maps.local_to_wc]
    gts, groups = [], []
    for gi, g in enumerate(gs.globs):
        if not bg[gi]:
            continue
        dofs = glob_free_dofs(g, dmap)
        n = len(dofs)
        avg_rows = np.stack([cs.averages[a].weights for a in bg[gi]])
        gt = build_glob_transform(gi, avg_rows)
        gts.append(gt)
        nz_a, nz_b = np.nonzero(gt.t != 0.0)
        for s in g.subdomains:
            local = np.array([next(cl for cs_, cl in maps.dof_copies[d] if cs_ == s) for d in dofs])
            covered[s][local] = True
            trip[s][0].append(local[nz_a]); trip[s][1].append(local[nz_b])
            trip[s][2].append(gt.t[nz_a, nz_b])
        for k in range(gt.rank):
            gdof = dofs[gt.explicit_slots[k]]
            grp = []
            for s in g.subdomains:
                for cs_, cl in maps.dof_copies[gdof]:
                    if cs_ == s:
                        grp.append(int(maps.local_to_wc[s][cl]))
            groups.append(grp)
    basis = []
    for s in range(n_sub):
        dim = len(covered[s])
        idn = np.nonzero(~covered[s])[0]
        r = np.concatenate(trip[s][0] + [idn]) if trip[s][0] else idn
        c = np.concatenate(trip[s][1] + [idn]) if trip[s][1] else idn
        v = np.concatenate(trip[s][2] + [np.ones(len(idn))]) if trip[s][2] else np.ones(len(idn))
        basis.append(sp.csr_matrix((v, (r, c)), shape=(dim, dim)))
    return ChangeOfVariables(gts, basis, groups)


class GroupProjector:
    """`transform.cpp:12-46`: each group replaced by its mean."""

    def __init__(self, groups, dim):
        seen = np.zeros(dim, dtype=bool)
        for g in groups:
            if seen[g].any():
                raise SingularGram("transformed equality groups overlap")
            seen[g] = True
        self.groups, self.dim = groups, dim
        self.flat = [np.array(g, dtype=np.int64) for g in groups]

    def apply(self, v):
        for g in self.flat:
            v[g] = v[g].sum() / len(g)
        return v

    def matrix(self):
        rows, cols, vals = [], [], []
        grouped = np.zeros(self.dim, dtype=bool)
        for g in self.flat:
            grouped[g] = True
            a, b = np.meshgrid(g, g, indexing="ij")
            rows.append(a.ravel()); cols.append(b.ravel())
            vals.append(np.full(a.size, 1.0 / len(g)))
        idn = np.nonzero(~grouped)[0]
        rows.append(idn); cols.append(idn); vals.append(np.ones(len(idn)))
        return sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                             shape=(self.dim, self.dim))


def transformed_constraint_matrix(cov: ChangeOfVariables, maps: EmbeddingMaps):
    """`transform.cpp:151-164`."""
    rows, cols, vals = [], [], []
    row = 0
    for g in cov.groups:
        for m in g[1:]:
            rows += [row, row]; cols += [g[0], m]; vals += [1.0, -1.0]
            row += 1
    return sp.csr_matrix((vals, (rows, cols)), shape=(row, maps.wc_dim))
