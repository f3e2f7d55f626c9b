"""Oracle: stabilized transformed operator, BDDC preconditioner, PCG, Lanczos.

Restates `core/src/bddc_operator.cpp` and `core/src/pcg.cpp`.
TEST INFRASTRUCTURE ONLY (see oracle/__init__).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, List, Optional

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp

from .constraints import ChangeOfVariables, GroupProjector
from .linalg import Factorization, pruned
from .spaces import AveragingOperator, EmbeddingMaps


def assemble_transformed_operator(systems, maps: EmbeddingMaps, cov: ChangeOfVariables):
    """`bddc_operator.cpp:7-23`: K = sum_s R^cT T_s^T A_s T_s R^c (upper, mirrored)."""
    rows, cols, vals = [], [], []
    for s, sys in enumerate(systems):
        b = cov.basis[s]
        local = (b.T @ sys.stiffness @ b).tocoo()
        r = maps.local_to_wc[s][local.row]
        c = maps.local_to_wc[s][local.col]
        keep = r <= c
        rows.append(r[keep]); cols.append(c[keep]); vals.append(local.data[keep])
    upper = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                          shape=(maps.wc_dim, maps.wc_dim)).tocsr()
    upper.sum_duplicates()
    return (upper + sp.triu(upper, k=1).T).tocsr()


def stabilize(k: sp.csr_matrix, projector: sp.csr_matrix, t: float, prune: bool = True):
    """`bddc_operator.cpp:25-36`: P K P + t (I - P), symmetrized and pruned.
    `prune=False` is NOT the reference: it keeps the entries below
    1e-12 max|entry| (used only to obtain the mathematically intended operator
    where the reference's pruning makes the factorization fail)."""
    if t <= 0:
        t = float(k.diagonal().max())
    n = k.shape[0]
    m = projector @ k @ projector + t * (sp.identity(n, format="csr") - projector)
    sym = 0.5 * (m.T + m)
    return (pruned(sym) if prune else sp.csr_matrix(sym)), t


class BddcPreconditioner:
    """`bddc_operator.cpp:38-103`."""

    def __init__(self, systems, maps: EmbeddingMaps, averaging: AveragingOperator,
                 cov: ChangeOfVariables, t: float = -1.0, prune: bool = True):
        self.systems, self.maps, self.avg, self.cov = systems, maps, averaging, cov
        self.projector = GroupProjector(cov.groups, maps.wc_dim)
        self.transformed = assemble_transformed_operator(systems, maps, cov)
        self.stabilized, self.t = stabilize(self.transformed, self.projector.matrix(), t, prune)
        self.factor = Factorization(self.stabilized)
        self.bt = [b.T.tocsr() for b in cov.basis]

    def restrict_residual(self, r_interface):
        m = self.maps
        u = np.zeros(len(m.dof_copies))
        u[m.interface_dofs] = r_interface
        w = self.avg.distribute(u)
        wc = np.zeros(m.wc_dim)
        for s, sys in enumerate(self.systems):
            y = self.bt[s] @ w[m.w_offset[s]:m.w_offset[s] + sys.dim]
            np.add.at(wc, m.local_to_wc[s], y)
        return self.projector.apply(wc)

    def coarse_solve(self, wc_residual):
        rhs = self.projector.apply(wc_residual.copy())
        x = self.projector.apply(self.factor.solve(rhs))
        residual = self.projector.apply(self.transformed @ x)
        residual = rhs - residual
        corr = self.projector.apply(self.factor.solve(residual))
        return x + corr

    def prolong(self, wc_corr):
        m = self.maps
        w = np.empty(m.w_dim)
        for s, sys in enumerate(self.systems):
            z = wc_corr[m.local_to_wc[s]]
            w[m.w_offset[s]:m.w_offset[s] + sys.dim] = self.cov.basis[s] @ z
        return self.avg.average(w)[m.interface_dofs]

    def apply(self, r):
        return self.prolong(self.coarse_solve(self.restrict_residual(r)))


def lanczos_condition_estimate(alphas, betas) -> float:
    """`pcg.cpp:11-26`."""
    n = len(alphas)
    if n == 0:
        return 1.0
    diag = np.empty(n)
    sub = np.empty(max(n - 1, 0))
    diag[0] = 1.0 / alphas[0]
    for j in range(1, n):
        diag[j] = 1.0 / alphas[j] + betas[j - 1] / alphas[j - 1]
        sub[j - 1] = np.sqrt(betas[j - 1]) / alphas[j - 1]
    ev = sla.eigh_tridiagonal(diag, sub, eigvals_only=True) if n > 1 else diag
    lo, hi = ev.min(), ev.max()
    return hi / lo if lo > 0 else float("inf")


@dataclass
class PcgResult:
    """`pcg.hpp:28-34`."""
    x: np.ndarray
    iterations: int = 0
    relative_residual: float = 0.0
    alphas: List[float] = field(default_factory=list)
    betas: List[float] = field(default_factory=list)
    condition_estimate: float = 1.0
    converged: bool = True


def pcg(op: Callable, prec: Callable, b: np.ndarray, tolerance=1e-8, max_iterations=500,
        preconditioned_residual=False, log=None) -> PcgResult:
    """`pcg.cpp:28-77`: zero initial guess; MaxIterationsExceeded -> converged=False."""
    res = PcgResult(np.zeros_like(b))
    r = b.copy()
    z = prec(r)
    p = z.copy()
    rz = float(r @ z)
    true_ref = float(np.linalg.norm(b))
    prec_ref = np.sqrt(max(rz, 0.0))
    ref = prec_ref if preconditioned_residual else true_ref
    if ref == 0.0:
        return res

    def current():
        return (np.sqrt(max(rz, 0.0)) if preconditioned_residual else np.linalg.norm(r)) / ref

    res.relative_residual = current()
    for _ in range(max_iterations):
        if res.relative_residual <= tolerance:
            break
        q = op(p)
        alpha = rz / float(p @ q)
        res.x += alpha * p
        r -= alpha * q
        z = prec(r)
        rz_next = float(r @ z)
        beta = rz_next / rz
        p = z + beta * p
        res.alphas.append(alpha)
        res.betas.append(beta)
        rz = rz_next
        res.iterations += 1
        res.relative_residual = current()
        if log is not None:
            log.append(res.relative_residual)
    res.converged = res.relative_residual <= tolerance
    res.condition_estimate = lanczos_condition_estimate(res.alphas, res.betas)
    return res
