"""Oracle: pair spaces, admissible bases, pair eigenproblems, enrichment.

Restates `core/src/pair.cpp` and `core/src/adaptive.cpp`.
TEST INFRASTRUCTURE ONLY (see oracle/__init__).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np
import scipy.linalg as sla

from .constraints import ConstraintSet, GlobAverage, add_average, glob_free_dofs
from .globs import CORNER, EDGE, FACE, GlobSet
from .linalg import EigenReport, Factorization, generalized_eig_sym, pivoted_qr


def face_pairs(gs: GlobSet):
    """`adaptive.cpp:12-20`."""
    return sorted({(g.subdomains[0], g.subdomains[1]) for g in gs.globs if g.kind == FACE})


def _local_of(maps, g, s):
    for cs, cl in maps.dof_copies[g]:
        if cs == s:
            return cl
    raise RuntimeError("dof has no copy in the requested substructure")


def local_schur(sys, keep):
    """`pair.cpp:32-63`: dense Schur complement of A_s onto the listed local dofs."""
    keep = np.asarray(keep, dtype=np.int64)
    mask = np.ones(sys.dim, dtype=bool)
    mask[keep] = False
    rest = np.nonzero(mask)[0]
    a = sys.stiffness
    akk = a[keep][:, keep].toarray()
    if len(rest) == 0:
        return akk
    ark = a[rest][:, keep].toarray()
    f = Factorization(a[rest][:, rest])
    return akk - ark.T @ f.solve(ark)


@dataclass
class PairSpace:
    """`pair.hpp:16-38`: [corner | shared_i | shared_j | outer_i outer_j]."""
    si: int
    sj: int
    shared_globs: List[int]
    corner_globals: np.ndarray
    noncorner_globals: np.ndarray
    slot_glob: np.ndarray
    outer_globals: np.ndarray
    rho_i: np.ndarray
    schur: np.ndarray
    n_outer_i: int = 0

    @property
    def n_corner(self): return len(self.corner_globals)

    @property
    def n_shared(self): return len(self.noncorner_globals)

    @property
    def n_outer(self): return len(self.outer_globals)

    @property
    def dim(self): return self.n_corner + 2 * self.n_shared + self.n_outer

    def average_copies(self, v):
        """`pair.cpp:12-21` (columns of a matrix are averaged independently)."""
        out = np.array(v, copy=True)
        nc, nf = self.n_corner, self.n_shared
        rho = self.rho_i if v.ndim == 1 else self.rho_i[:, None]
        mean = rho * v[nc:nc + nf] + (1.0 - rho) * v[nc + nf:nc + 2 * nf]
        out[nc:nc + nf] = mean
        out[nc + nf:nc + 2 * nf] = mean
        return out


def build_pair(systems, maps, gs: GlobSet, dmap, si, sj) -> PairSpace:
    """`pair.cpp:67-146`."""
    shared_globs, corner, noncorner, slot_glob = [], [], [], []
    for gi, g in enumerate(gs.globs):
        if si in g.subdomains and sj in g.subdomains:
            dofs = glob_free_dofs(g, dmap)
            if g.kind == CORNER:
                corner.extend(dofs)
            else:
                shared_globs.append(gi)
                noncorner.extend(dofs)
                slot_glob.extend([gi] * len(dofs))
    if not corner and not noncorner:
        raise RuntimeError("substructures %d and %d share no interface dofs" % (si, sj))
    outer = ([], [])
    for g in gs.globs:
        hi, hj = si in g.subdomains, sj in g.subdomains
        if hi == hj:
            continue
        outer[0 if hi else 1].extend(glob_free_dofs(g, dmap))
    nc, nf = len(corner), len(noncorner)
    rho = np.empty(nf)
    di_all = systems[si].stiffness.diagonal()
    dj_all = systems[sj].stiffness.diagonal()
    for t, g in enumerate(noncorner):
        di = di_all[_local_of(maps, g, si)]
        dj = dj_all[_local_of(maps, g, sj)]
        rho[t] = di / (di + dj)
    dim = nc + 2 * nf + len(outer[0]) + len(outer[1])
    schur = np.zeros((dim, dim))
    for side, s in enumerate((si, sj)):
        outer_base = 0 if side == 0 else len(outer[0])
        keep = [_local_of(maps, g, s) for g in corner]
        slot = list(range(nc))
        keep += [_local_of(maps, g, s) for g in noncorner]
        slot += [nc + (0 if side == 0 else nf) + t for t in range(nf)]
        keep += [_local_of(maps, g, s) for g in outer[side]]
        slot += [nc + 2 * nf + outer_base + t for t in range(len(outer[side]))]
        ss = local_schur(systems[s], keep)
        slot = np.array(slot)
        schur[np.ix_(slot, slot)] += ss
    return PairSpace(si, sj, shared_globs, np.array(corner, dtype=np.int64),
                     np.array(noncorner, dtype=np.int64), np.array(slot_glob, dtype=np.int64),
                     np.array(outer[0] + outer[1], dtype=np.int64), rho, schur, len(outer[0]))


def glob_kernel(rows: Optional[np.ndarray], n: int) -> np.ndarray:
    """Kernel of a glob's installed averages (`pair.cpp:167-188`)."""
    if rows is None:
        return np.eye(n)
    qr = pivoted_qr(rows)
    r = qr.rank
    kernel = np.zeros((n, n - r))
    if n > r:
        u = qr.r[:r, :r]
        v = qr.r[:r, r:]
        top = -sla.solve_triangular(u, v, lower=False)
        for a in range(r):
            kernel[qr.perm[a], :] = top[a, :]
        for a in range(r, n):
            kernel[qr.perm[a], a - r] = 1.0
    return kernel


def pair_admissible_basis(pair: PairSpace, cs: ConstraintSet, gs: GlobSet, dmap) -> np.ndarray:
    """`pair.cpp:148-209`."""
    nc, nf, d = pair.n_corner, pair.n_shared, pair.dim
    bg = cs.by_glob(len(gs.globs))
    cols = []
    for t in range(nc):
        c = np.zeros(d); c[t] = 1.0; cols.append(c)
    base = 0
    for gi in pair.shared_globs:
        n = len(glob_free_dofs(gs.globs[gi], dmap))
        for t in range(n):
            c = np.zeros(d); c[nc + base + t] = 1.0; c[nc + nf + base + t] = 1.0; cols.append(c)
        rows = np.stack([cs.averages[a].weights for a in bg[gi]]) if bg[gi] else None
        kernel = glob_kernel(rows, n)
        for k in range(kernel.shape[1]):
            c = np.zeros(d)
            c[nc + base:nc + base + n] = kernel[:, k]
            c[nc + nf + base:nc + nf + base + n] = -kernel[:, k]
            cols.append(c)
        base += n
    for t in range(pair.n_outer):
        c = np.zeros(d); c[nc + 2 * nf + t] = 1.0; cols.append(c)
    return np.column_stack(cols) if cols else np.zeros((d, 0))


@dataclass
class PairSolve:
    space: PairSpace
    admissible: np.ndarray
    eig: EigenReport


def solve_pair(cs, gs, dmap, systems, maps, si, sj, request, inclusion_rel_tol=1e-6) -> PairSolve:
    """`adaptive.cpp:30-47`.  `inclusion_rel_tol` is the reference's 1e-6
    (dense_eig.cpp:77-126); `inf` disables its nullspace-inclusion throw (NOT the
    reference -- used only to record what the reference would select on the
    pairs where it throws, tests/golden/make_fullsize.py)."""
    space = build_pair(systems, maps, gs, dmap, si, sj)
    z = pair_admissible_basis(space, cs, gs, dmap)
    jump = z - space.average_copies(z)
    s_jump = space.schur @ jump
    lhs = jump.T @ s_jump
    rhs = z.T @ (space.schur @ z)
    eig = generalized_eig_sym(lhs, rhs, min(request, z.shape[1]), inclusion_rel_tol=inclusion_rel_tol)
    return PairSolve(space, z, eig)


def jump_functional(pair: PairSpace, w):
    """`adaptive.cpp:51-58`."""
    d = pair.schur @ (w - pair.average_copies(w))
    nc, nf = pair.n_corner, pair.n_shared
    return (1.0 - pair.rho_i) * d[nc:nc + nf] - pair.rho_i * d[nc + nf:nc + 2 * nf]


@dataclass
class EnrichmentOptions:
    """`adaptive.hpp:24-29`."""
    tau: float = 10.0
    max_vectors: int = 15
    keep_edge_constraints: bool = False
    fixed_count: int = -1


@dataclass
class PairReport:
    """`adaptive.hpp:14-22`."""
    si: int
    sj: int
    eigenvalues: np.ndarray
    enforced: int = 0
    omega_next: float = 0.0
    saturated: bool = False
    kept: int = 0
    dropped: int = 0
    functionals: List[np.ndarray] = field(default_factory=list)


@dataclass
class EnrichmentOutcome:
    pairs: List[PairReport] = field(default_factory=list)
    omega_tilde: float = 0.0
    kept: int = 0
    dropped: int = 0


def _count_above(values, tau):
    k = 0
    while k < len(values) and values[k] > tau:
        k += 1
    return k


def pair_candidates(sol: PairSolve, gs, dmap, opts: EnrichmentOptions, tau_mode=True):
    """The per-pair part of `adaptive.cpp:72-115`: selection count, omega_next,
    saturation, and the split/normalized functional pieces (before the rank
    filter of `add_average`) in the reference's order.  Independent of every
    other pair (all pairs are solved against the same base, `adaptive.cpp:133`)."""
    lam = sol.eig.eigenvalues
    rep = PairReport(sol.space.si, sol.space.sj, lam.copy())
    pieces = []
    if not tau_mode:
        rep.omega_next = float(lam[0]) if len(lam) else 0.0
        return rep, pieces
    if opts.fixed_count >= 0:
        rep.enforced = min(opts.fixed_count, len(lam))
    else:
        rep.enforced = min(_count_above(lam, opts.tau), opts.max_vectors)
    rep.omega_next = float(lam[rep.enforced]) if rep.enforced < len(lam) else 0.0
    rep.saturated = rep.omega_next > opts.tau and opts.fixed_count < 0
    for m in range(rep.enforced):
        func = jump_functional(sol.space, sol.admissible @ sol.eig.eigenvectors[:, m])
        rep.functionals.append(func)
        scale = np.linalg.norm(func)
        base_slot = 0
        for gi in sol.space.shared_globs:
            n = len(glob_free_dofs(gs.globs[gi], dmap))
            piece = func[base_slot:base_slot + n].copy()
            base_slot += n
            if np.linalg.norm(piece) <= 1e-12 * scale:
                continue
            if gs.globs[gi].kind == EDGE and not opts.keep_edge_constraints:
                continue
            top = int(np.argmax(np.abs(piece)))
            nrm = np.linalg.norm(piece)
            piece /= -nrm if piece[top] < 0 else nrm
            pieces.append((gi, piece))
    return rep, pieces


def install_pieces(enrich_into: ConstraintSet, rep: PairReport, pieces):
    """`adaptive.cpp:104-111`: each piece through the rank filter, in order."""
    for gi, piece in pieces:
        if add_average(enrich_into, GlobAverage(gi, piece, "adaptive")):
            rep.kept += 1
        else:
            rep.dropped += 1


def run_pairs(enrich_into, base, gs, dmap, systems, maps, opts, request):
    """`adaptive.cpp:66-125`."""
    out = EnrichmentOutcome()
    for si, sj in face_pairs(gs):
        sol = solve_pair(base, gs, dmap, systems, maps, si, sj, request)
        rep, pieces = pair_candidates(sol, gs, dmap, opts, enrich_into is not None)
        if enrich_into is not None:
            install_pieces(enrich_into, rep, pieces)
        out.omega_tilde = max(out.omega_tilde, rep.omega_next)
        out.kept += rep.kept
        out.dropped += rep.dropped
        out.pairs.append(rep)
    return out


def enrich_constraints(cs: ConstraintSet, gs, dmap, systems, maps, opts: EnrichmentOptions):
    """`adaptive.cpp:129-137`: every pair solved against the same base."""
    base = cs.copy()
    request = (opts.fixed_count if opts.fixed_count >= 0 else opts.max_vectors) + 1
    return run_pairs(cs, base, gs, dmap, systems, maps, opts, request)


def pair_indicator(cs, gs, dmap, systems, maps):
    """`adaptive.cpp:139-144`."""
    return run_pairs(None, cs, gs, dmap, systems, maps, EnrichmentOptions(), 1)
