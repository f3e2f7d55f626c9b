"""Full-size oracle fixtures for BASELINE.json configs 3, 4 and 5.

Run in the build container (CPU only, hours for cfg5; pairs are solved in
parallel worker processes, one BLAS thread each):

    python tests/golden/make_fullsize.py 3 4 5 [--workers 8]

For each config it runs the oracle's full adaptive selection
(`oracle.adaptive`, restating `adaptive.cpp:66-137`): every face pair is solved
against the same base set (`adaptive.cpp:133`), so the pairs are independent
and are farmed out to workers; the functional pieces are then installed through
the rank filter (`constraints.cpp:61-76`) sequentially in the reference's pair
order, which gives exactly `enrich_constraints`' constraint set.  For configs 3
and 4 it then runs the oracle's preconditioner and PCG on that set
(`bddc_operator.cpp:38-103`, `pcg.cpp:28-77`) three times: unperturbed, and
with the preconditioner output perturbed by 1e-13 relative noise (two seeds),
which measures the roundoff floor of the Lanczos estimate on this config.

Written to tests/golden/fullsize_cfg<c>.npz (small: per-pair reports, per-glob
subspace sketches, CG coefficients, the interface solution):

  si, sj, enforced, omega_next, saturated, kept, dropped, n_eig, eigenvalues
  glob_ids, glob_counts         number of averages per glob (every glob that has one)
  sketch_globs, sketch          subspace sketch of each face glob's averages (sketch())
  constraint_rows, omega_tilde
  pcg_* (cfg3, cfg4)            iterations, alphas, betas, kappa, relres log,
                                interface solution x, energy u^T A u, and the
                                perturbed runs' iterations / kappa
The GPU tests read only these files (the box has no oracle time budget for
full-size eigenproblems).  Seeds: BASELINE seed 20091030 (oracle.experiment).
"""
from __future__ import annotations

import argparse
import json
import os
import pickle
import sys
import time
from pathlib import Path

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")
os.environ.setdefault("MKL_NUM_THREADS", "1")

import numpy as np  # noqa: E402

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
from fullsize_sketch import glob_summary  # noqa: E402  (this directory)


# --- worker state (set before the pool forks) ---------------------------------
_W = {}


def _pair_task(k):
    from oracle.adaptive import pair_candidates, solve_pair
    from oracle.linalg import NullspaceInclusionViolated
    w = _W
    si, sj = w["pairs"][k]
    t0 = time.perf_counter()
    raised = ""
    args = (w["base"], w["p"].globset, w["p"].dmap, w["p"].systems, w["p"].maps, si, sj, w["request"])
    try:
        sol = solve_pair(*args)
    except NullspaceInclusionViolated as e:
        # the reference's generalized_eig_sym throws here (dense_eig.cpp:100-106):
        # a near-null direction of rhs (below 1e-9 max) that lhs does not annihilate
        # to 1e-6.  Record it, and what the reference would compute without the throw.
        raised = "NullspaceInclusionViolated: " + str(e)
        sol = solve_pair(*args, inclusion_rel_tol=float("inf"))
    rep, pieces = pair_candidates(sol, w["p"].globset, w["p"].dmap, w["opts"])
    return k, rep.eigenvalues, rep.enforced, rep.omega_next, rep.saturated, pieces, \
        time.perf_counter() - t0, sol.space.dim, raised


def _pcg_task(seed):
    from oracle.bddc import pcg
    w = _W
    prec = w["prec"].apply
    if seed >= 0:
        rng = np.random.default_rng(seed)
        prec = lambda v: w["prec"].apply(v) * (1 + 1e-13 * rng.standard_normal(len(v)))  # noqa: E731
    log = []
    t0 = time.perf_counter()
    r = pcg(w["itf"].apply, prec, w["rhs"], w["tol"], w["maxit"], log=log)
    return seed, r, log, time.perf_counter() - t0


def make(config: int, workers: int, pcg_runs: bool, shrink=None, suffix=""):
    import multiprocessing as mp
    from oracle import fem
    from oracle.adaptive import EnrichmentOptions, PairReport, face_pairs, install_pieces
    from oracle.bddc import BddcPreconditioner
    from oracle.constraints import change_of_variables
    from oracle.linalg import NotPositiveDefinite
    from oracle.experiment import baseline_config, build_pipeline, constraint_set_for
    from oracle.spaces import AveragingOperator, HarmonicExtension, InterfaceProblem

    t0 = time.perf_counter()
    cfg = baseline_config(config, **(shrink or {}))
    p = build_pipeline(cfg.spec)
    base = constraint_set_for(p, cfg.mode, cfg.base_faces)
    opts = EnrichmentOptions(tau=cfg.tau, max_vectors=cfg.max_vectors)
    pairs = face_pairs(p.globset)
    print("cfg%d: pipeline %.1fs, %d pairs" % (config, time.perf_counter() - t0, len(pairs)), flush=True)
    _W.update(p=p, base=base, opts=opts, pairs=pairs, request=cfg.max_vectors + 1)
    res = [None] * len(pairs)
    t1 = time.perf_counter()
    ctx = mp.get_context("fork")
    cache = Path(os.environ.get("FULLSIZE_CACHE", "/tmp")) / ("fullsize_pairs_cfg%d%s.pkl" % (config, suffix))
    if cache.exists():  # per-pair results of an earlier run of this script (scratch, not committed)
        res = [tuple(r) + ("",) * (9 - len(r)) for r in pickle.loads(cache.read_bytes())]
    else:
        with ctx.Pool(workers) as pool:
            for i, out in enumerate(pool.imap_unordered(_pair_task, range(len(pairs)), chunksize=2)):
                res[out[0]] = out
                if (i + 1) % 100 == 0:
                    print("  %d/%d pairs, %.0fs" % (i + 1, len(pairs), time.perf_counter() - t1), flush=True)
        cache.write_bytes(pickle.dumps(res))
    pair_cpu = sum(r[6] for r in res)
    raised = np.array([bool(r[8]) for r in res])
    if raised.any():
        print("cfg%d: %d pairs raise in the reference's eigensolver, e.g." % (config, raised.sum()),
              [(pairs[k], res[k][8]) for k in np.nonzero(raised)[0][:3]], flush=True)
    print("cfg%d: pairs %.0fs wall, %.0fs single-thread CPU" % (config, time.perf_counter() - t1, pair_cpu),
          flush=True)
    cs = base.copy()
    reps = []
    for (k, lam, enf, om, sat, pieces, _, _, _), (si, sj) in zip(res, pairs):
        rep = PairReport(si, sj, lam, enf, om, sat)
        install_pieces(cs, rep, pieces)
        reps.append(rep)
    globs = [g.kind for g in p.globset.globs]
    ids, counts, faces, sk = glob_summary([(a.glob, a.weights) for a in cs.averages], globs)
    n_eig = np.array([len(r.eigenvalues) for r in reps], dtype=np.int64)
    eig = np.zeros((len(reps), max(1, n_eig.max())))
    for i, r in enumerate(reps):
        eig[i, :len(r.eigenvalues)] = r.eigenvalues
    out = dict(
        si=np.array([r.si for r in reps], dtype=np.int64), sj=np.array([r.sj for r in reps], dtype=np.int64),
        enforced=np.array([r.enforced for r in reps], dtype=np.int64),
        omega_next=np.array([r.omega_next for r in reps]),
        saturated=np.array([r.saturated for r in reps], dtype=bool),
        kept=np.array([r.kept for r in reps], dtype=np.int64),
        dropped=np.array([r.dropped for r in reps], dtype=np.int64),
        n_eig=n_eig, eigenvalues=eig, pair_dim=np.array([r[7] for r in res], dtype=np.int64),
        glob_ids=ids, glob_counts=counts, sketch_globs=faces, sketch=sk,
        constraint_rows=np.int64(cs.row_count(p.globset)),
        omega_tilde=np.float64(max(r.omega_next for r in reps)),
        pair_cpu_seconds=np.float64(pair_cpu), raised=raised)
    meta = dict(config=config, seed=20091030, pairs=len(pairs), constraint_rows=int(out["constraint_rows"]),
                omega_tilde=float(out["omega_tilde"]), adaptive_rows=int(sum(r.kept for r in reps)),
                pair_cpu_seconds=pair_cpu, pairs_raising=int(raised.sum()))
    if pcg_runs:
        t2 = time.perf_counter()
        h = HarmonicExtension(p.systems, p.maps)
        itf = InterfaceProblem(p.systems, p.maps, h)
        cov = change_of_variables(cs, p.globset, p.dmap, p.maps)
        avg = AveragingOperator(p.systems, p.maps)
        attempts = [("reference (t = max diag K, entries <= 1e-12 max pruned)", dict()),
                    ("t = max diag K, unpruned", dict(prune=False))]
        prec, meta["stabilization"] = None, []
        for label, kw in attempts:
            try:
                prec = BddcPreconditioner(p.systems, p.maps, avg, cov, **kw)
                meta["stabilization"].append(label + ": factorized")
                break
            except NotPositiveDefinite as e:
                # bddc_operator.cpp:25-50: the reference factors the PRUNED stabilized
                # operator.  When the change of variables makes
                # max|entry| ~1e10, the 1e-12 relative prune drops O(1e-2) couplings
                # of the soft dofs and the factorization fails: the reference itself
                # raises NotPositiveDefinite here.  Pi A~^{-1} Pi of the unpruned
                # operator is the mathematically intended preconditioner.
                meta["stabilization"].append(label + ": " + str(e))
                print("cfg%d: %s failed (%s)" % (config, label, e), flush=True)
        if prec is None:
            raise RuntimeError("no stabilization factorized")
        print("cfg%d: preconditioner %.0fs" % (config, time.perf_counter() - t2), flush=True)
        _W.update(prec=prec, itf=itf, rhs=itf.rhs(), tol=cfg.spec.tolerance, maxit=cfg.spec.max_iterations)
        with ctx.Pool(3) as pool:
            runs = {seed: (r, log, dt) for seed, r, log, dt in pool.map(_pcg_task, [-1, 1, 2])}
        r, log, dt = runs[-1]
        u = itf.recover(r.x)
        a = fem.global_matrix(p.systems, p.dmap.free_count)
        out.update(pcg_iterations=np.int64(r.iterations), pcg_alphas=np.array(r.alphas),
                   pcg_betas=np.array(r.betas), pcg_kappa=np.float64(r.condition_estimate),
                   pcg_relres=np.array(log), pcg_x=r.x, pcg_energy=np.float64(u @ (a @ u)),
                   pcg_seconds=np.float64(dt),
                   pert_iterations=np.array([runs[s][0].iterations for s in (1, 2)], dtype=np.int64),
                   pert_kappa=np.array([runs[s][0].condition_estimate for s in (1, 2)]))
        meta.update(iterations=r.iterations, kappa=r.condition_estimate, pcg_seconds=dt,
                    pert_iterations=out["pert_iterations"].tolist(), pert_kappa=out["pert_kappa"].tolist())
    np.savez_compressed(HERE / ("fullsize_cfg%d%s.npz" % (config, suffix)), **out)
    (HERE / ("fullsize_cfg%d%s.json" % (config, suffix))).write_text(json.dumps(meta, indent=1) + "\n")
    print("cfg%d:" % config, json.dumps(meta), flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", type=int, nargs="+")
    ap.add_argument("--workers", type=int, default=os.cpu_count())
    ap.add_argument("--no-pcg", action="store_true")
    ap.add_argument("--dry", action="store_true", help="3x3x3 H/h=3 versions (quick check of the script)")
    a = ap.parse_args()
    for c in a.configs:
        if a.dry:
            make(c, a.workers, not a.no_pcg, dict(subdomains=(3, 3, 3), elements_per_edge=3), "_dry")
        else:
            make(c, a.workers, pcg_runs=(c in (3, 4) and not a.no_pcg))
