"""Oracle work item with the face pairs farmed out to worker processes.

TEST INFRASTRUCTURE ONLY (see oracle/__init__): used by bench.py's CPU legs
(`cpu_baseline`, `--impl reference` on all host cores) and by
tests/golden/make_fullsize.py.  The arithmetic is `experiment.solve_item`'s:
every pair is solved against the same base (`adaptive.cpp:133`), so the
pairs are independent; their functional pieces are installed through the rank
filter sequentially in the reference's pair order (`adaptive.cpp:72-115`),
which yields exactly `enrich_constraints`' constraint set.  The reference
itself is serial; the parallel split is over the
independent units SPEC.md allows (pairs).
"""
from __future__ import annotations

import multiprocessing as mp
import time

from .adaptive import EnrichmentOptions, EnrichmentOutcome, PairReport, face_pairs, install_pieces
from .bddc import BddcPreconditioner, pcg
from .constraints import change_of_variables
from .experiment import ResultRow, constraint_set_for, tau_label
from .spaces import AveragingOperator, HarmonicExtension, InterfaceProblem

_W = {}
_LIMIT = []


def _init_worker():
    """One BLAS thread per worker process (the pairs are the parallel axis)."""
    from threadpoolctl import threadpool_limits
    _LIMIT.append(threadpool_limits(limits=1))


def _pair_task(k):
    from .adaptive import pair_candidates, solve_pair
    w = _W
    si, sj = w["pairs"][k]
    t0 = time.perf_counter()
    sol = solve_pair(w["base"], w["p"].globset, w["p"].dmap, w["p"].systems, w["p"].maps, si, sj, w["request"])
    rep, pieces = pair_candidates(sol, w["p"].globset, w["p"].dmap, w["opts"])
    return k, rep, pieces, time.perf_counter() - t0, sol.space.dim


def solve_pairs(p, base, opts: EnrichmentOptions, workers: int, progress=None):
    """Per-pair reports and pieces of every face pair, in pair order:
    [(rep, pieces, seconds, dim)]."""
    pairs = face_pairs(p.globset)
    request = (opts.fixed_count if opts.fixed_count >= 0 else opts.max_vectors) + 1
    _W.update(p=p, base=base, opts=opts, pairs=pairs, request=request)
    res = [None] * len(pairs)
    if workers <= 1:
        for k in range(len(pairs)):
            res[k] = _pair_task(k)[1:]
        return res
    with mp.get_context("fork").Pool(workers, initializer=_init_worker) as pool:
        for i, out in enumerate(pool.imap_unordered(_pair_task, range(len(pairs)), chunksize=2)):
            res[out[0]] = out[1:]
            if progress and (i + 1) % 100 == 0:
                progress(i + 1, len(pairs))
    return res


def enrich_parallel(cs, p, opts: EnrichmentOptions, workers: int) -> EnrichmentOutcome:
    """`enrich_constraints` (adaptive.cpp:129-137) with the pairs in parallel."""
    base = cs.copy()
    out = EnrichmentOutcome()
    for rep, pieces, _, _ in solve_pairs(p, base, opts, workers):
        rep = PairReport(rep.si, rep.sj, rep.eigenvalues, rep.enforced, rep.omega_next, rep.saturated)
        install_pieces(cs, rep, pieces)
        out.omega_tilde = max(out.omega_tilde, rep.omega_next)
        out.kept += rep.kept
        out.dropped += rep.dropped
        out.pairs.append(rep)
    return out


def solve_item_parallel(p, mode: str, tau=10.0, max_vectors=15, base_faces=False, workers=1) -> ResultRow:
    """`experiment.solve_item` (experiment.cpp:143-205) with parallel pairs."""
    t0 = time.perf_counter()
    harmonic = HarmonicExtension(p.systems, p.maps)
    averaging = AveragingOperator(p.systems, p.maps)
    interface = InterfaceProblem(p.systems, p.maps, harmonic)
    row = ResultRow(tau_label(tau) if mode == "adaptive" else mode)
    row.seconds_analysis = time.perf_counter() - t0
    t1 = time.perf_counter()
    cs = constraint_set_for(p, mode, base_faces)
    if mode == "adaptive":
        row.outcome = enrich_parallel(cs, p, EnrichmentOptions(tau=tau, max_vectors=max_vectors), workers)
        row.omega_tilde = row.outcome.omega_tilde
    row.constraint_rows = cs.row_count(p.globset)
    row.constraints = cs
    cov = change_of_variables(cs, p.globset, p.dmap, p.maps)
    prec = BddcPreconditioner(p.systems, p.maps, averaging, cov, -1.0)
    row.seconds_factorization = time.perf_counter() - t1
    t2 = time.perf_counter()
    res = pcg(interface.apply, prec.apply, interface.rhs(), p.spec.tolerance, p.spec.max_iterations)
    row.seconds_iterations = time.perf_counter() - t2
    row.kappa, row.iterations, row.converged, row.pcg = (res.condition_estimate, res.iterations,
                                                         res.converged, res)
    row.seconds_total = row.seconds_analysis + row.seconds_factorization + row.seconds_iterations
    return row
