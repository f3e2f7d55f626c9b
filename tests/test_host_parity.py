"""The C++ host layer reproduces the reference's index maps, globs, coefficient
fields, substructure matrices and constraint sets exactly (checked against
the independent Python oracle; CPU only)."""
import numpy as np
import pytest

import paper_0910_5863_b200 as pb
from oracle import fem
from oracle.constraints import arithmetic_constraints
from oracle.experiment import baseline_config, build_pipeline, cube_spec

CASES = [
    ("clamped 2x2x2 H/h=4 elasticity", cube_spec((2, 2, 2), 4, fem.ELASTICITY),
     lambda: pb.BDDC(pb.Problem.cube((2, 2, 2), 4, "elasticity"))),
    ("floating 2x2x2 H/h=4 elasticity", cube_spec((2, 2, 2), 4, fem.ELASTICITY, clamp=False),
     lambda: pb.BDDC(pb.Problem.cube((2, 2, 2), 4, "elasticity", clamp=False))),
    ("planar 2x2x1 scalar", cube_spec((2, 2, 1), 4, fem.SCALAR, clamp=False),
     lambda: pb.BDDC(pb.Problem.cube((2, 2, 1), 4, "scalar", clamp=False))),
    ("planar 2x2x1 elasticity", cube_spec((2, 2, 1), 4, fem.ELASTICITY, clamp=False),
     lambda: pb.BDDC(pb.Problem.cube((2, 2, 1), 4, "elasticity", clamp=False))),
    ("stacked 1x1x2", cube_spec((1, 1, 2), 2, fem.SCALAR, clamp=False),
     lambda: pb.BDDC(pb.Problem.cube((1, 1, 2), 2, "scalar", clamp=False))),
    ("cfg1", baseline_config(1).spec, lambda: pb.BDDC(config=1)),
    ("cfg2", baseline_config(2).spec, lambda: pb.BDDC(config=2)),
    ("cfg3 shrunk", baseline_config(3, subdomains=(3, 3, 3), elements_per_edge=4).spec,
     lambda: pb.BDDC(config=3, subdomains=(3, 3, 3), elements_per_edge=4)),
    ("cfg4 shrunk", baseline_config(4, subdomains=(3, 3, 3), elements_per_edge=3).spec,
     lambda: pb.BDDC(config=4, subdomains=(3, 3, 3), elements_per_edge=3)),
    ("cfg5 shrunk", baseline_config(5, subdomains=(3, 3, 3), elements_per_edge=3).spec,
     lambda: pb.BDDC(config=5, subdomains=(3, 3, 3), elements_per_edge=3)),
]


@pytest.mark.parametrize("name,spec,make", CASES, ids=[c[0] for c in CASES])
def test_index_maps_and_globs(name, spec, make):
    p = build_pipeline(spec)
    b = make()
    st = b.structure()
    assert st["free_dofs"] == p.dmap.free_count
    assert st["interface_dofs"] == p.maps.interface_count
    assert st["coarse_space_dim"] == p.maps.wc_dim
    assert st["classification_corners"] == p.classification_corners
    assert np.array_equal(b.interface_dofs(), p.maps.interface_dofs)
    globs = b.globs()
    assert len(globs) == len(p.globset.globs)
    for (k, nodes, subs), g in zip(globs, p.globset.globs):
        assert (k, nodes, subs) == (g.kind, list(g.nodes), tuple(g.subdomains))
    for s in range(len(p.systems)):
        assert np.array_equal(b.global_dof(s), p.systems[s].global_dof)
        assert np.array_equal(b.local_to_wc(s), p.maps.local_to_wc[s])


@pytest.mark.parametrize("name,spec,make", CASES, ids=[c[0] for c in CASES])
def test_substructure_matrices_and_loads(name, spec, make):
    p = build_pipeline(spec)
    b = make()
    if spec.element_scale is not None:
        assert np.array_equal(b.element_scale(), spec.element_scale)  # bitwise: same generator
    for s in range(len(p.systems)):
        a, load = b.subdomain_matrix(s)
        ref = p.systems[s].stiffness
        diff = abs(a - ref)
        assert diff.max() <= 1e-13 * abs(ref).max()
        assert np.allclose(load, p.systems[s].load, rtol=1e-13, atol=1e-15)


@pytest.mark.parametrize("edges,faces", [(True, False), (True, True), (False, False)])
def test_arithmetic_constraints(edges, faces):
    spec = cube_spec((2, 2, 2), 4, fem.ELASTICITY)
    p = build_pipeline(spec)
    b = pb.BDDC(pb.Problem.cube((2, 2, 2), 4, "elasticity"))
    b.arithmetic_constraints(edges, faces)
    cs = arithmetic_constraints(p.globset, p.dmap, edges, faces)
    assert b.constraint_rows() == cs.row_count(p.globset)
    got = b.constraints()
    assert len(got) == len(cs.averages)
    for (g, w), a in zip(got, cs.averages):
        assert g == a.glob and np.array_equal(w, a.weights)
