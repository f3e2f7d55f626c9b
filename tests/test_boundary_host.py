"""Boundary entry points that run on the host side of the C ABI (CPU only):
caller-built constraint sets through add_average (constraints.cpp:61-76), the
stabilized operator and its t (bddc_operator.cpp:7-36), and the
export_directory Matrix Market dumps (experiment.cpp:172-178,
matrix_market.cpp:12-38), each against the oracle."""
import numpy as np
import pytest
import scipy.io
import scipy.sparse as sp

import paper_0910_5863_b200 as pb
from oracle import fem
from oracle.bddc import assemble_transformed_operator, stabilize
from oracle.constraints import (GlobAverage, GroupProjector, add_average, arithmetic_constraints,
                                change_of_variables, glob_free_dofs, transformed_constraint_matrix)
from oracle.experiment import build_pipeline, cube_spec


def test_dependent_averages_rejected_independent_kept():
    """tests/test_constraints.cpp:102-121."""
    b = pb.BDDC(pb.Problem.cube((1, 1, 2), 2, "scalar", clamp=False))
    b.arithmetic_constraints(True, True)
    got = b.constraints()
    assert len(got) == 1
    face, w = got[0]
    n = len(w)
    assert not b.add_average(face, 2.0 * np.ones(n))
    assert len(b.constraints()) == 1
    assert b.add_average(face, np.linspace(0.0, 1.0, n))
    assert len(b.constraints()) == 2 and b.constraint_rows() == 2
    with pytest.raises(pb.BddcError):
        b.add_average(face, np.ones(n + 1))  # wrong length for the glob


def random_set(p, rng):
    """test_constraints.cpp:83-100: c+e+f plus one random average per glob."""
    cs = arithmetic_constraints(p.globset, p.dmap, True, True)
    extra = []
    for g, glob in enumerate(p.globset.globs):
        if glob.kind == "corner":
            continue
        w = rng.standard_normal(len(glob_free_dofs(glob, p.dmap)))
        extra.append((g, w))
    return cs, extra


def test_caller_constraint_set_matches_oracle():
    p = build_pipeline(cube_spec((2, 2, 2), 2, fem.ELASTICITY))
    cs, extra = random_set(p, np.random.default_rng(21))
    b = pb.BDDC(pb.Problem.cube((2, 2, 2), 2, "elasticity"))
    b.clear_constraints()
    for a in cs.averages:
        assert b.add_average(a.glob, a.weights)
    for g, w in extra:
        assert b.add_average(g, w) == add_average(cs, GlobAverage(g, w, "adaptive"))
    got = b.constraints()
    assert len(got) == len(cs.averages)
    for (g, w), a in zip(got, cs.averages):
        assert g == a.glob and np.array_equal(w, a.weights)
    assert b.constraint_rows() == cs.row_count(p.globset)


def test_exact_integer_transform():
    """tests/test_constraints.cpp:123-142 on the product's host layer: unit
    averages give t = [1, -1, ..., -1] over the identity."""
    b = pb.BDDC(pb.Problem.cube((2, 2, 2), 3, "scalar", clamp=False))
    b.arithmetic_constraints(True, True)
    globs = sorted({g for g, _ in b.constraints()})
    assert globs
    for g in globs:
        r, t = b.glob_transform(g)
        n = t.shape[0]
        ref = np.eye(n)
        ref[0, 1:] = -1.0
        assert r == 1 and np.array_equal(t, ref), g


def test_glob_transforms_match_oracle_without_ties():
    """transform.cpp:51-90 against the oracle for arithmetic (integer, tie rules
    exact) and random averages.  Random rows on top of the component averages
    produce column-norm ties that only roundoff breaks (the reference's pivot
    order is then implementation-defined); the span, and so the preconditioner,
    does not depend on it.  Compared: exact equality for the arithmetic sets,
    and t^{-1}'s first rank rows spanning the averages for the random set."""
    p = build_pipeline(cube_spec((2, 2, 2), 3, fem.ELASTICITY))
    b = pb.BDDC(pb.Problem.cube((2, 2, 2), 3, "elasticity"))
    cs = arithmetic_constraints(p.globset, p.dmap, True, True)
    b.arithmetic_constraints(True, True)
    for gt in change_of_variables(cs, p.globset, p.dmap, p.maps).glob_transforms:
        r, t = b.glob_transform(gt.glob)
        assert r == gt.rank and np.array_equal(t, gt.t), gt.glob
    cs, extra = random_set(p, np.random.default_rng(5))
    for g, w in extra:
        add_average(cs, GlobAverage(g, w, "adaptive"))
    b.clear_constraints()
    for a in cs.averages:
        b.add_average(a.glob, a.weights)
    for gt in change_of_variables(cs, p.globset, p.dmap, p.maps).glob_transforms:
        r, t = b.glob_transform(gt.glob)
        assert r == gt.rank
        rows = np.stack([a.weights for a in cs.averages if a.glob == gt.glob])
        # the explicit coordinates of t^{-1} are the averages: rows @ t = [I_r | 0] up to basis
        h = np.linalg.inv(t)[:r]
        assert np.linalg.matrix_rank(np.vstack([h, rows]), tol=1e-8) == r


@pytest.mark.parametrize("mode", ["c+e", "c+e+f"])
def test_stabilized_operator_and_t(mode):
    p = build_pipeline(cube_spec((2, 2, 2), 3, fem.ELASTICITY))
    b = pb.BDDC(pb.Problem.cube((2, 2, 2), 3, "elasticity"))
    cs = arithmetic_constraints(p.globset, p.dmap, True, mode == "c+e+f")
    b.arithmetic_constraints(True, mode == "c+e+f")
    cov = change_of_variables(cs, p.globset, p.dmap, p.maps)
    k = assemble_transformed_operator(p.systems, p.maps, cov)
    ref, t = stabilize(k, GroupProjector(cov.groups, p.maps.wc_dim).matrix(), -1.0)
    assert abs(b.stabilization_t() - t) <= 1e-12 * t
    got = b.stabilized()
    assert got.shape == ref.shape
    d = abs(got - ref)
    assert d.max() <= 1e-11 * abs(ref).max()


def test_matrix_market_export(tmp_path):
    p = build_pipeline(cube_spec((2, 2, 2), 2, fem.SCALAR))
    cs = arithmetic_constraints(p.globset, p.dmap, True, True)
    cov = change_of_variables(cs, p.globset, p.dmap, p.maps)
    k = assemble_transformed_operator(p.systems, p.maps, cov)
    ref, _ = stabilize(k, GroupProjector(cov.groups, p.maps.wc_dim).matrix(), -1.0)
    b = pb.BDDC(pb.Problem.cube((2, 2, 2), 2, "scalar"))
    b.arithmetic_constraints(True, True)
    stem = str(tmp_path / "c+e+f")
    b.export_matrix_market(stem)
    head = open(stem + "_stabilized.mtx").readline()
    assert head.strip() == "%%MatrixMarket matrix coordinate real symmetric"
    a = scipy.io.mmread(stem + "_stabilized.mtx")
    assert abs(sp.csr_matrix(a) - ref).max() <= 1e-11 * abs(ref).max()
    d = sp.csr_matrix(scipy.io.mmread(stem + "_constraints.mtx"))
    dref = transformed_constraint_matrix(cov, p.maps)
    assert d.shape == dref.shape and abs(d - dref).max() == 0.0
