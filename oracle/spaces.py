"""Oracle: product-space embeddings, weighted averaging, harmonic extension,
and the interface (Schur) problem.

Restates `core/src/spaces.cpp` and `core/src/schur.cpp`.
TEST INFRASTRUCTURE ONLY (see oracle/__init__).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Tuple

import numpy as np
import scipy.sparse as sp

from .fem import DofMap, SubdomainSystem
from .globs import GlobSet
from .linalg import Factorization


@dataclass
class EmbeddingMaps:
    """`spaces.hpp:23-43`."""
    w_offset: np.ndarray
    w_dim: int
    dof_copies: List[List[Tuple[int, int]]]
    interface_dofs: np.ndarray
    global_to_interface: np.ndarray
    corner_dof_count: int
    wc_dim: int
    local_to_wc: List[np.ndarray]
    local_is_corner: List[np.ndarray]
    corner_dof_of_global: np.ndarray

    @property
    def interface_count(self):
        return len(self.interface_dofs)


def build_embeddings(systems: List[SubdomainSystem], free_count: int, gs: GlobSet,
                     dmap: DofMap) -> EmbeddingMaps:
    """`spaces.cpp:9-56`."""
    n_sub = len(systems)
    dims = np.array([s.dim for s in systems], dtype=np.int64)
    w_offset = np.concatenate([[0], np.cumsum(dims)[:-1]]).astype(np.int64)
    copies = [[] for _ in range(free_count)]
    for s, sys in enumerate(systems):        # ascending subdomain
        for l, g in enumerate(sys.global_dof):
            copies[g].append((s, l))
    ncopies = np.array([len(c) for c in copies])
    interface = np.nonzero(ncopies >= 2)[0].astype(np.int64)
    g2i = np.full(free_count, -1, dtype=np.int64)
    g2i[interface] = np.arange(len(interface))
    corner_of = np.full(free_count, -1, dtype=np.int64)
    count = 0
    for node in gs.corner_nodes():
        for c in range(dmap.dofs_per_node):
            g = dmap.at(node, c)
            if g < 0:
                continue
            corner_of[g] = count
            count += 1
    wc = count
    l2wc, is_corner = [], []
    for sys in systems:
        cor = corner_of[sys.global_dof]
        m = np.empty(sys.dim, dtype=np.int64)
        nc = cor < 0
        m[~nc] = cor[~nc]
        m[nc] = wc + np.arange(int(nc.sum()))
        wc += int(nc.sum())
        l2wc.append(m)
        is_corner.append(~nc)
    return EmbeddingMaps(w_offset, int(dims.sum()), copies, interface, g2i, count, wc,
                         l2wc, is_corner, corner_of)


class AveragingOperator:
    """`spaces.cpp:71-106`: weights = A_s(l,l) / sum over copies."""

    def __init__(self, systems, maps: EmbeddingMaps):
        self.maps = maps
        diags = [s.stiffness.diagonal() for s in systems]
        self.weights = []
        rows, cols, vals = [], [], []
        for g, copies in enumerate(maps.dof_copies):
            w = [diags[s][l] for s, l in copies]
            tot = 0.0
            for x in w:
                tot += x
            w = [x / tot for x in w]
            self.weights.append(w)
            for (s, l), x in zip(copies, w):
                rows.append(g); cols.append(maps.w_offset[s] + l); vals.append(x)
        # E as a sparse matrix (global x W); E^T distributes
        self.e = sp.csr_matrix((vals, (rows, cols)), shape=(len(maps.dof_copies), maps.w_dim))
        self.et = self.e.T.tocsr()

    def average(self, w):
        return self.e @ w

    def distribute(self, u):
        return self.et @ u


class HarmonicExtension:
    """`spaces.cpp:108-177`: interior = single-copy local dofs."""

    def __init__(self, systems, maps: EmbeddingMaps):
        self.maps = maps
        self.interior, self.boundary, self.coupling, self.factor = [], [], [], []
        for sys in systems:
            ncop = np.array([len(maps.dof_copies[g]) for g in sys.global_dof])
            b = np.nonzero(ncop >= 2)[0]
            i = np.nonzero(ncop < 2)[0]
            a = sys.stiffness
            self.interior.append(i)
            self.boundary.append(b)
            self.coupling.append(a[i][:, b].tocsr())
            self.factor.append(Factorization(a[i][:, i]))

    def interior_solve(self, s, b):
        return self.factor[s].solve(b)


class InterfaceProblem:
    """`schur.cpp:12-75`."""

    def __init__(self, systems, maps: EmbeddingMaps, harmonic: HarmonicExtension):
        self.systems, self.maps, self.h = systems, maps, harmonic
        self.bidx = [maps.global_to_interface[sys.global_dof[harmonic.boundary[s]]]
                     for s, sys in enumerate(systems)]

    @property
    def size(self):
        return self.maps.interface_count

    def apply(self, u):
        out = np.zeros(self.size)
        for s, sys in enumerate(self.systems):
            x = np.zeros(sys.dim)
            bnd, inn = self.h.boundary[s], self.h.interior[s]
            x[bnd] = u[self.bidx[s]]
            if len(inn):
                x[inn] = self.h.interior_solve(s, -(self.h.coupling[s] @ x[bnd]))
            y = sys.stiffness @ x
            np.add.at(out, self.bidx[s], y[bnd])
        return out

    def rhs(self):
        out = np.zeros(self.size)
        for s, sys in enumerate(self.systems):
            bnd, inn = self.h.boundary[s], self.h.interior[s]
            fold = np.zeros(len(bnd))
            if len(inn):
                fold = self.h.coupling[s].T @ self.h.interior_solve(s, sys.load[inn])
            np.add.at(out, self.bidx[s], sys.load[bnd] - fold)
        return out

    def recover(self, u_interface):
        u = np.zeros(len(self.maps.dof_copies))
        u[self.maps.interface_dofs] = u_interface
        for s, sys in enumerate(self.systems):
            bnd, inn = self.h.boundary[s], self.h.interior[s]
            if not len(inn):
                continue
            xb = u_interface[self.bidx[s]]
            xi = self.h.interior_solve(s, sys.load[inn] - self.h.coupling[s] @ xb)
            u[sys.global_dof[inn]] = xi
        return u
