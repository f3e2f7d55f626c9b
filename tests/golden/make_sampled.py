"""Pair-sampled full-size oracle fixture for BASELINE.json config 5.

cfg5 has 4752 face pairs of dimension up to 2304: its complete oracle
selection does not fit the build container's time.  The reference solves every
pair against the same base set (`adaptive.cpp:133`) and a face glob is touched
by its own pair only, so a pair's report and the averages installed on its face
glob are independent of all other pairs.  This script solves a deterministic
sample of pairs at FULL size with the oracle (`oracle.adaptive.solve_pair`,
restating `adaptive.cpp:30-125`) -- pairs next to the Dirichlet face, floating
pairs in the interior, pairs on the outer boundary, and x-, y- and z-normal
faces (the material layers cut the x- and y-normal ones) -- and writes
tests/golden/sampled_cfg5.npz:

  si, sj, enforced, omega_next, saturated, n_eig, eigenvalues, pair_dim,
  face_glob, kept, sketch (subspace sketch of the averages installed on the
  pair's face glob, golden/fullsize_sketch.py)

    python tests/golden/make_sampled.py [--config 5] [--pairs 36] [--workers 8]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")

import numpy as np  # noqa: E402

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
sys.path.insert(0, str(HERE))
from fullsize_sketch import SKETCH_K, sketch  # noqa: E402
import make_fullsize as mf  # noqa: E402  (worker state and the per-pair task)


def choose(pairs, lattice, count):
    """A deterministic sample covering the pair categories."""
    nx, ny, nz = lattice

    def coord(s):
        return s % nx, (s // nx) % ny, s // (nx * ny)

    cats = {}
    for k, (si, sj) in enumerate(pairs):
        a, b = coord(si), coord(sj)
        axis = [i for i in range(3) if a[i] != b[i]][0]
        dirichlet = a[0] == 0  # the lower substructure touches the clamped face x = 0
        outer = any(c in (0, m - 1) for c, m in zip(a, lattice)) or any(c in (0, m - 1) for c, m in zip(b, lattice))
        cats.setdefault((axis, "dirichlet" if dirichlet else "outer" if outer else "interior"), []).append(k)
    rng = np.random.default_rng(20091030)
    picked = []
    keys = sorted(cats)
    while len(picked) < count:
        for key in keys:
            if cats[key] and len(picked) < count:
                picked.append(cats[key].pop(int(rng.integers(len(cats[key])))))
    return sorted(picked)


def main():
    import multiprocessing as mp
    from oracle.adaptive import EnrichmentOptions, PairReport, face_pairs, install_pieces
    from oracle.experiment import baseline_config, build_pipeline, constraint_set_for
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--pairs", type=int, default=36)
    ap.add_argument("--workers", type=int, default=os.cpu_count())
    a = ap.parse_args()
    t0 = time.perf_counter()
    cfg = baseline_config(a.config)
    p = build_pipeline(cfg.spec)
    base = constraint_set_for(p, cfg.mode, cfg.base_faces)
    opts = EnrichmentOptions(tau=cfg.tau, max_vectors=cfg.max_vectors)
    pairs = face_pairs(p.globset)
    sample = choose(pairs, cfg.spec.subdomains, a.pairs)
    print("cfg%d: pipeline %.1fs, %d of %d pairs sampled" % (a.config, time.perf_counter() - t0, len(sample),
                                                             len(pairs)), flush=True)
    mf._W.update(p=p, base=base, opts=opts, pairs=pairs, request=cfg.max_vectors + 1)
    t1 = time.perf_counter()
    with mp.get_context("fork").Pool(a.workers) as pool:
        res = {out[0]: out for out in pool.imap_unordered(mf._pair_task, sample)}
    print("pairs %.0fs wall" % (time.perf_counter() - t1), flush=True)
    n = len(sample)
    eig = np.zeros((n, cfg.max_vectors + 1))
    out = dict(pair_index=np.array(sample, dtype=np.int64), si=np.zeros(n, np.int64), sj=np.zeros(n, np.int64),
               enforced=np.zeros(n, np.int64), omega_next=np.zeros(n), saturated=np.zeros(n, bool),
               n_eig=np.zeros(n, np.int64), eigenvalues=eig, pair_dim=np.zeros(n, np.int64),
               face_glob=np.full(n, -1, np.int64), kept=np.zeros(n, np.int64), sketch=np.zeros((n, SKETCH_K)),
               raised=np.zeros(n, bool))
    for q, k in enumerate(sample):
        _, lam, enf, om, sat, pieces, _, dim, raised = res[k]
        si, sj = pairs[k]
        cs = base.copy()
        n_base = len(cs.averages)
        rep = PairReport(si, sj, lam, enf, om, sat)
        install_pieces(cs, rep, pieces)
        new = cs.averages[n_base:]
        out["si"][q], out["sj"][q], out["enforced"][q], out["omega_next"][q] = si, sj, enf, om
        out["saturated"][q], out["n_eig"][q], out["pair_dim"][q], out["raised"][q] = sat, len(lam), dim, bool(raised)
        eig[q, :len(lam)] = lam
        out["kept"][q] = len(new)
        face = sorted({av.glob for av in new})
        assert len(face) <= 1, face  # edge pieces are dropped: only the pair's face glob
        if face:
            out["face_glob"][q] = face[0]
            out["sketch"][q] = sketch(face[0], np.stack([av.weights for av in new]))
    np.savez_compressed(HERE / ("sampled_cfg%d.npz" % a.config), **out)
    meta = dict(config=a.config, seed=20091030, pairs_total=len(pairs), pairs_sampled=n,
                enforced=out["enforced"].tolist(), pairs_raising=int(out["raised"].sum()),
                seconds=time.perf_counter() - t0)
    (HERE / ("sampled_cfg%d.json" % a.config)).write_text(json.dumps(meta, indent=1) + "\n")
    print(json.dumps(meta), flush=True)


if __name__ == "__main__":
    main()
