"""Oracle: dense kernels and direct factorization.

Restates `core/src/dense_eig.cpp` (column-pivoted Householder QR with the
reference's tie and sign rules; the symmetric generalized eigensolver modulo
null(rhs)) and `core/src/sparse.cpp` (factorize, pruned).  Eigen's
`SelfAdjointEigenSolver` is replaced by LAPACK (`numpy.linalg.eigh`) and
`SimplicialLLT` by a dense Cholesky (small) or SuperLU (large).
TEST INFRASTRUCTURE ONLY (see oracle/__init__).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp
import scipy.sparse.linalg as spla


class NotPositiveDefinite(RuntimeError):
    """`types.hpp:25-28`."""


class NullspaceInclusionViolated(RuntimeError):
    """`types.hpp:46-49`."""


class SingularGram(RuntimeError):
    """`types.hpp:51-54`."""


@dataclass
class PivotedQr:
    """`dense_eig.hpp:20-29`: A P = Q R, perm[k] = original column at slot k."""
    q: np.ndarray
    r: np.ndarray
    perm: List[int]
    rank: int


def pivoted_qr(a: np.ndarray, rel_drop_tol: float = 1e-8) -> PivotedQr:
    """`dense_eig.cpp:17-75`."""
    a = np.array(a, dtype=float, copy=True)
    m, n = a.shape
    q = np.eye(m)
    r = a
    perm = list(range(n))
    steps = min(m, n)
    for k in range(steps):
        best = k
        best_norm = np.linalg.norm(r[k:, k])
        for j in range(k + 1, n):
            nj = np.linalg.norm(r[k:, j])
            if nj > best_norm:  # strict: ties keep the earliest column
                best, best_norm = j, nj
        if best != k:
            r[:, [k, best]] = r[:, [best, k]]
            perm[k], perm[best] = perm[best], perm[k]
        if best_norm == 0.0:
            break
        x = r[k:, k].copy()
        v = x.copy()
        alpha = (-1.0 if x[0] >= 0 else 1.0) * np.linalg.norm(x)
        v[0] -= alpha
        vsq = float(v @ v)
        if vsq > 0:
            block = r[k:, k:]
            block -= np.outer((2.0 / vsq) * v, v @ block)
            qblock = q[:, k:]
            qblock -= np.outer(qblock @ v, (2.0 / vsq) * v)
        r[k, k] = alpha
        r[k + 1:, k] = 0.0
        if r[k, k] < 0:
            r[k, k:] = -r[k, k:]
            q[:, k] = -q[:, k]
    d0 = abs(r[0, 0]) if m and n else 0.0
    rank = 0
    for k in range(steps):
        if abs(r[k, k]) > rel_drop_tol * d0 and d0 > 0:
            rank += 1
        else:
            break
    return PivotedQr(q, r, perm, rank)


@dataclass
class EigenReport:
    """`dense_eig.hpp:34-39`."""
    eigenvalues: np.ndarray
    eigenvectors: np.ndarray
    requested: int
    rhs_nullity: int


def generalized_eig_sym(lhs, rhs, k, null_rel_tol=1e-9, inclusion_rel_tol=1e-6) -> EigenReport:
    """`dense_eig.cpp:77-126`: top-k of lhs w = lambda rhs w modulo null(rhs)."""
    n = rhs.shape[0]
    d, v = np.linalg.eigh(rhs)          # ascending, like SelfAdjointEigenSolver
    dmax = max(d[-1], 0.0) if n else 0.0
    null_cut = null_rel_tol * (dmax if dmax > 0 else 1.0)
    nullity = 0
    while nullity < n and d[nullity] <= null_cut:
        nullity += 1
    lhs_scale = max(np.linalg.norm(lhs), 1e-300)
    for j in range(nullity):
        if np.linalg.norm(lhs @ v[:, j]) > inclusion_rel_tol * lhs_scale:
            raise NullspaceInclusionViolated("null(rhs) not in null(lhs)")
    r = n - nullity
    if r == 0 or k == 0:
        return EigenReport(np.zeros(0), np.zeros((n, 0)), k, nullity)
    vr = v[:, nullity:]
    isq = 1.0 / np.sqrt(d[nullity:])
    b = isq[:, None] * (vr.T @ lhs @ vr) * isq[None, :]
    b = 0.5 * (b + b.T)
    ev, ew = np.linalg.eigh(b)
    take = min(k, r)
    vals = np.maximum(ev[::-1][:take], 0.0)
    vecs = vr @ (isq[:, None] * ew[:, ::-1][:, :take])
    return EigenReport(vals, vecs, k, nullity)


class Factorization:
    """`sparse.hpp:55-66` / `sparse.cpp:55-92`: definite factorization handle."""

    def __init__(self, a, dense_limit=4000):
        self.n = a.shape[0]
        if sp.issparse(a) and self.n > dense_limit:
            self.lu = spla.splu(sp.csc_matrix(a), permc_spec="MMD_AT_PLUS_A",
                                diag_pivot_thresh=0.0, options={"SymmetricMode": True})
            d = self.lu.U.diagonal()
            if np.any(d <= 0):
                raise NotPositiveDefinite("factorize: matrix is not positive definite")
            self.c = None
        else:
            dense = a.toarray() if sp.issparse(a) else np.asarray(a)
            try:
                self.c = sla.cho_factor(dense, lower=True, check_finite=False)
            except np.linalg.LinAlgError as e:
                raise NotPositiveDefinite("factorize: matrix is not positive definite") from e
            if self.n and not np.all(np.diag(self.c[0]) > 0):
                raise NotPositiveDefinite("factorize: matrix is not positive definite")
            self.lu = None

    def solve(self, b):
        if self.n == 0:
            return np.zeros_like(b)
        if self.c is not None:
            return sla.cho_solve(self.c, b, check_finite=False)
        return self.lu.solve(b)


def pruned(m: sp.spmatrix, rel_tol=1e-12) -> sp.csr_matrix:
    """`sparse.cpp:98-108`."""
    m = sp.csr_matrix(m, copy=True)
    amax = np.abs(m.data).max() if m.nnz else 0.0
    cut = rel_tol * (amax if amax > 0 else 1.0)
    m.data[np.abs(m.data) <= cut] = 0.0
    m.eliminate_zeros()
    return m
