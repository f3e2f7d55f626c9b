"""Subspace sketches of constraint sets (shared by make_fullsize.py and
tests/test_fullsize_parity.py)."""
import numpy as np

SKETCH_K = 3


def sketch(glob: int, rows: np.ndarray) -> np.ndarray:
    """Basis-independent fingerprint of the span of a glob's averages: for
    seeded Gaussian g_k, h_k (seed = glob id), (g_k^T Q Q^T h_k)/(|g_k| |h_k|)
    with Q an orthonormal basis of the rows.  Equal spans give equal sketches
    whatever vectors span them (degenerate eigenvalues)."""
    rows = np.atleast_2d(np.asarray(rows, dtype=float))
    n = rows.shape[1]
    q, _ = np.linalg.qr(rows.T)
    rng = np.random.default_rng(1_000_003 + glob)
    g = rng.standard_normal((n, SKETCH_K))
    h = rng.standard_normal((n, SKETCH_K))
    return np.einsum("ik,ik->k", q.T @ g, q.T @ h) / (np.linalg.norm(g, axis=0) * np.linalg.norm(h, axis=0))


def glob_summary(averages, globs):
    """(glob ids with averages, counts, face-glob ids, sketches) of a constraint
    list given as [(glob, weights)]."""
    by = {}
    for g, w in averages:
        by.setdefault(int(g), []).append(np.asarray(w, dtype=float))
    ids = np.array(sorted(by), dtype=np.int64)
    counts = np.array([len(by[g]) for g in ids], dtype=np.int64)
    faces = [g for g in ids if globs[g] == "face"]
    sk = np.array([sketch(g, np.stack(by[g])) for g in faces]).reshape(-1, SKETCH_K)
    return ids, counts, np.array(faces, dtype=np.int64), sk
