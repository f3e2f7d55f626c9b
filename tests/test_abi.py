"""The C-ABI library loads, exports every symbol include/bddc_b200.h declares,
maps the reference's error taxonomy onto status codes, and has no CPU
fallback (CPU only; no compute calls need a GPU here)."""
import re
from pathlib import Path

import numpy as np
import pytest

import paper_0910_5863_b200 as pb

HEADER = Path(__file__).resolve().parents[1] / "include" / "bddc_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(bddc_b200_\w+)\s*\(", text)))


def test_every_declared_symbol_is_exported(lib):
    names = declared_symbols()
    assert len(names) >= 30
    for n in names:
        assert hasattr(lib, n), n
    # and the Python mirror binds all of them
    assert set(names) <= set(pb.EXPORTS), set(names) - set(pb.EXPORTS)


def test_library_is_the_in_tree_build(lib):
    assert Path(lib._name).resolve().parent == Path(pb.__file__).resolve().parent


def test_bad_problem_spec_maps_to_status_code():
    with pytest.raises(pb.BddcError) as e:
        pb.BDDC(pb.Problem((1, 1, 1), 0, "scalar"))
    assert e.value.kind == "BadProblemSpec"
    with pytest.raises(pb.BddcError) as e:
        pb.BDDC(pb.Problem((2, 1, 1), 2, "elasticity", materials={0: (1.0, 1.0, 0.5)}))
    assert e.value.kind == "BadProblemSpec"  # nu must lie in (0, 0.5) (problem.cpp:185)
    with pytest.raises(pb.BddcError) as e:
        pb.BDDC(config=7)
    assert e.value.kind == "BadProblemSpec"


def test_unknown_mode_is_rejected():
    b = pb.BDDC(pb.Problem.cube((2, 2, 1), 2, "scalar"))
    with pytest.raises(pb.BddcError) as e:
        b.run_item("corners")
    assert e.value.kind == "BadProblemSpec"


def test_host_lanczos_estimate():
    """pcg.cpp:11-26 in the C++ host layer: CG on diag(1..10) gives kappa = 10."""
    from oracle.bddc import pcg
    d = np.arange(1.0, 11.0)
    r = pcg(lambda v: d * v, lambda v: v, np.ones(10), 1e-12, 50)
    k = pb.lanczos_condition_estimate(r.alphas, r.betas)
    assert abs(k - 10.0) <= 1e-6 * 10.0
    assert pb.lanczos_condition_estimate([], []) == 1.0


def test_no_cpu_fallback(lib):
    if lib.bddc_b200_device_count() > 0:
        pytest.skip("a CUDA device is present")
    b = pb.BDDC(pb.Problem.cube((2, 2, 1), 2, "scalar"))
    with pytest.raises(pb.BddcError) as e:
        b.analysis()
    assert e.value.kind == "CudaError"
    with pytest.raises(pb.BddcError):
        b.step("c+e")
