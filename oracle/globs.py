"""Oracle: interface globs and deterministic corner selection.

Restates `core/src/globs.cpp`.  TEST INFRASTRUCTURE ONLY (see oracle/__init__).
"""
from __future__ import annotations

from collections import deque
from dataclasses import dataclass, field
from typing import List, Tuple

import numpy as np

from .fem import SCALAR, Decomposition, Mesh

CORNER, EDGE, FACE = "corner", "edge", "face"
_RANK = {CORNER: 0, EDGE: 1, FACE: 2}


@dataclass
class Glob:
    """`globs.hpp:18-22`."""
    kind: str
    nodes: List[int]
    subdomains: Tuple[int, ...]


@dataclass
class GlobSet:
    """`globs.hpp:24-44`: corners first, then edges, then faces."""
    globs: List[Glob] = field(default_factory=list)
    classification_corner_count: int = 0

    def count(self, kind):
        return sum(1 for g in self.globs if g.kind == kind)

    def corner_nodes(self):
        return [g.nodes[0] for g in self.globs if g.kind == CORNER]


def _grid_neighbors(mesh: Mesh, node: int):
    """`globs.cpp:21-34`: 6-neighbourhood in the fixed order -x,+x,-y,+y,-z,+z."""
    nx, ny, nz = mesh.nodes_per_axis
    i, j, k = node % nx, (node // nx) % ny, node // (nx * ny)
    out = []
    if i > 0: out.append(node - 1)
    if i + 1 < nx: out.append(node + 1)
    if j > 0: out.append(node - nx)
    if j + 1 < ny: out.append(node + nx)
    if k > 0: out.append(node - nx * ny)
    if k + 1 < nz: out.append(node + nx * ny)
    return out


def _sort_canonical(globs: List[Glob]):
    """`globs.cpp:38-44`."""
    globs.sort(key=lambda g: (_RANK[g.kind], g.nodes[0]))


def _strict_superset(big, small):
    return len(big) > len(small) and set(small).issubset(big)


def classify_globs(mesh: Mesh, deco: Decomposition) -> GlobSet:
    """`globs.cpp:61-99`: group by sharing set (std::map order), BFS components."""
    groups = {}
    for n, subs in enumerate(deco.node_subdomains):
        if len(subs) >= 2:
            groups.setdefault(subs, []).append(n)
    out = GlobSet()
    for sharers in sorted(groups):
        nodes = groups[sharers]
        pending = set(nodes)
        for seed in nodes:
            if seed not in pending:
                continue
            members = []
            frontier = deque([seed])
            pending.discard(seed)
            while frontier:
                n = frontier.popleft()
                members.append(n)
                for nb in _grid_neighbors(mesh, n):
                    if nb in pending:
                        pending.discard(nb)
                        frontier.append(nb)
            members.sort()
            if len(sharers) == 2:
                kind = FACE
            elif len(members) == 1:
                kind = CORNER
            else:
                kind = EDGE
            out.globs.append(Glob(kind, members, sharers))
    out.classification_corner_count = out.count(CORNER)
    _sort_canonical(out.globs)
    return out


class _CornerSelection:
    """`globs.cpp:103-250`."""

    def __init__(self, gs: GlobSet, mesh: Mesh, deco: Decomposition):
        self.gs, self.mesh, self.deco = gs, mesh, deco
        self.corners = [g.nodes[0] for g in gs.globs if g.kind == CORNER]

    def run(self):
        self.promote_edge_endpoints()
        self.repair_pairs()
        self.gs.globs = [g for g in self.gs.globs if g.nodes]
        _sort_canonical(self.gs.globs)

    def promote(self, source: int, node: int):
        self.gs.globs[source].nodes.remove(node)
        self.gs.globs.append(Glob(CORNER, [node], self.deco.node_subdomains[node]))
        self.corners.append(node)

    def in_glob_neighbors(self, members, node):
        return sum(1 for nb in _grid_neighbors(self.mesh, node) if nb in members)

    def promote_edge_endpoints(self):
        n_globs = len(self.gs.globs)
        for gi in range(n_globs):
            g = self.gs.globs[gi]
            if g.kind != EDGE:
                continue
            members = set(g.nodes)
            promoted = []
            for node in g.nodes:
                if self.in_glob_neighbors(members, node) > 1:
                    continue
                bigger = any(_strict_superset(self.deco.node_subdomains[nb], g.subdomains)
                             for nb in _grid_neighbors(self.mesh, node))
                if not bigger:
                    promoted.append(node)
            for node in promoted:
                self.promote(gi, node)

    def shared_corners(self, pair):
        return [c for c in self.corners if set(pair).issubset(self.deco.node_subdomains[c])]

    def pinned(self, shared):
        if self.mesh.physics == SCALAR:
            return len(shared) > 0
        if len(shared) < 3:
            return False
        p0 = self.mesh.coords[shared[0]]
        for a in range(1, len(shared)):
            u = self.mesh.coords[shared[a]] - p0
            for b in range(a + 1, len(shared)):
                v = self.mesh.coords[shared[b]] - p0
                cx = u[1] * v[2] - u[2] * v[1]
                cy = u[2] * v[0] - u[0] * v[2]
                cz = u[0] * v[1] - u[1] * v[0]
                if cx * cx + cy * cy + cz * cz > 1e-16:
                    return True
        return False

    def promote_candidates(self, glob, candidates, pair):
        candidates = list(candidates)
        while candidates:
            shared = self.shared_corners(pair)
            if self.pinned(shared):
                return
            ranked = []
            for node in candidates:
                dmin = float("inf")
                for c in shared:
                    d = self.mesh.coords[node] - self.mesh.coords[c]
                    dmin = min(dmin, float(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]))
                ranked.append((dmin, node))
            ranked.sort(key=lambda t: (-t[0], t[1]))
            top = ranked[0][0]
            group = [node for d, node in ranked
                     if d == top or abs(d - top) <= 1e-9 * max(1.0, top)]
            for node in group:
                self.promote(glob, node)
                candidates.remove(node)

    def repair_pairs(self):
        faces = [gi for gi, g in enumerate(self.gs.globs) if g.kind == FACE]
        faces.sort(key=lambda gi: (self.gs.globs[gi].subdomains, self.gs.globs[gi].nodes[0]))
        for gi in faces:
            pair = self.gs.globs[gi].subdomains
            if self.pinned(self.shared_corners(pair)):
                continue
            nodes = self.gs.globs[gi].nodes
            members = set(nodes)
            rim = [n for n in nodes if self.in_glob_neighbors(members, n) <= 2]
            self.promote_candidates(gi, rim, pair)
            if not self.pinned(self.shared_corners(pair)):
                self.promote_candidates(gi, list(self.gs.globs[gi].nodes), pair)
            if not self.pinned(self.shared_corners(pair)):
                raise RuntimeError("cannot pin substructure pair %d,%d" % (pair[0], pair[1]))


def select_corners(gs: GlobSet, mesh: Mesh, deco: Decomposition):
    """`globs.cpp:252-254`."""
    _CornerSelection(gs, mesh, deco).run()
