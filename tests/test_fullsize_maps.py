"""Full-size index maps of BASELINE configs 3, 4 and 5 (CPU only).

north_star: "the interface/index maps are identical" on all five configs.
The C++ host layer's maps for the full-size problems -- globs (kind, node list,
sharers, in the reference's order, `globs.cpp:61-256`), corner promotion,
the interface numbering and the per-substructure global-dof and W^c embeddings
(`spaces.cpp:9-56`), and the base constraint set (`constraints.cpp:34-59`) --
are compared element for element with the oracle's `build_pipeline`.  No
factorization is involved, so even cfg5 (2.7M free dofs, 1728 substructures)
takes well under a minute.
"""
import numpy as np
import pytest

import paper_0910_5863_b200 as pb
from oracle.experiment import baseline_config, build_pipeline, constraint_set_for


@pytest.fixture(scope="module", params=[3, 4, 5], ids=["cfg3", "cfg4", "cfg5"])
def both(request):
    cfg = baseline_config(request.param)
    return request.param, cfg, build_pipeline(cfg.spec), pb.BDDC(config=request.param)


def test_structure_and_interface(both):
    c, cfg, p, b = both
    st = b.structure()
    assert st["free_dofs"] == p.dmap.free_count
    assert st["interface_dofs"] == p.maps.interface_count
    assert st["coarse_space_dim"] == p.maps.wc_dim
    assert st["classification_corners"] == p.classification_corners
    assert st["subdomains"] == len(p.systems)
    assert np.array_equal(b.interface_dofs(), p.maps.interface_dofs)
    if cfg.spec.element_scale is not None:
        assert np.array_equal(b.element_scale(), cfg.spec.element_scale)


def test_globs(both):
    c, cfg, p, b = both
    globs = b.globs()
    assert len(globs) == len(p.globset.globs)
    for (k, nodes, subs), g in zip(globs, p.globset.globs):
        assert (k, nodes, subs) == (g.kind, list(g.nodes), tuple(g.subdomains))


def test_embeddings(both):
    c, cfg, p, b = both
    for s in range(len(p.systems)):
        assert np.array_equal(b.global_dof(s), p.systems[s].global_dof), s
        assert np.array_equal(b.local_to_wc(s), p.maps.local_to_wc[s]), s


def test_base_constraints(both):
    c, cfg, p, b = both
    cs = constraint_set_for(p, cfg.mode, cfg.base_faces)
    b.arithmetic_constraints(True, cfg.base_faces)
    assert b.constraint_rows() == cs.row_count(p.globset)
    got = b.constraints()
    assert len(got) == len(cs.averages)
    for (g, w), a in zip(got, cs.averages):
        assert g == a.glob and np.array_equal(w, a.weights)
