"""A plain C program (tests/c/integration.c) compiled against
include/bddc_b200.h and linked with libbddc_b200.so runs the INTEGRATION.md
sequence -- the binding a reference maintainer would write, checked by the C
compiler instead of by ctypes.  CPU: compile, link, host-only calls, and the
device call fails with BDDC_B200_CUDA_ERROR.  GPU: the reference's PCG loop
(pcg.cpp:28-77) over the schur_apply / precond_apply seams agrees with the
device-resident PCG and with the oracle."""
import subprocess
from pathlib import Path

import pytest

import paper_0910_5863_b200 as pb

REPO = Path(__file__).resolve().parents[1]
SRC = REPO / "tests" / "c" / "integration.c"


@pytest.fixture(scope="module")
def exe(tmp_path_factory, lib):
    out = tmp_path_factory.mktemp("cint") / "integration"
    libdir = Path(lib._name).resolve().parent
    cmd = ["gcc", "-std=c99", "-Wall", "-Werror", "-O1", "-I", str(REPO / "include"), str(SRC), "-o", str(out),
           "-L", str(libdir), "-l:libbddc_b200.so", "-Wl,-rpath," + str(libdir), "-lm"]
    subprocess.check_call(cmd)
    return out


def run(exe, arg):
    p = subprocess.run([str(exe), arg], capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, (p.returncode, p.stdout, p.stderr)
    return dict(line.split(" ", 1) for line in p.stdout.strip().splitlines())


def test_c_program_links_and_runs_host_calls(exe, lib):
    out = run(exe, "host")
    b = pb.BDDC(pb.Problem.cube((2, 2, 2), 2, "elasticity"))
    st = b.structure()
    assert int(out["free_dofs"]) == st["free_dofs"]
    assert int(out["interface_dofs"]) == st["interface_dofs"]
    assert int(out["subdomains"]) == 8
    # add_average (constraints.cpp:61-76): the repeated average is dropped by the rank filter
    assert out["kept"] == "1 0"
    assert int(out["rows"]) == 1
    if lib.bddc_b200_device_count() == 0:
        assert int(out["analysis_rc"]) == 10  # BDDC_B200_CUDA_ERROR: no CPU fallback


@pytest.mark.gpu
def test_c_program_device_sequence_matches_oracle(exe):
    from oracle import fem
    from oracle.experiment import build_pipeline, cube_spec, solve_item
    out = run(exe, "device")
    ref = solve_item(build_pipeline(cube_spec((2, 2, 2), 2, fem.ELASTICITY)), "adaptive", 10.0, 15)
    assert int(out["constraint_rows"]) == ref.constraint_rows
    assert abs(float(out["omega_tilde"]) - ref.omega_tilde) <= 1e-6 * ref.omega_tilde
    # the reference's host PCG over the two seams and the device PCG
    assert abs(int(out["host_pcg_iterations"]) - ref.iterations) <= 1
    assert abs(int(out["device_pcg_iterations"]) - ref.iterations) <= 1
    assert float(out["host_vs_device_solution"]) <= 1e-7
    assert abs(float(out["device_pcg_kappa"]) - ref.kappa) <= 1e-6 * ref.kappa
    assert abs(float(out["lanczos_kappa"]) - float(out["device_pcg_kappa"])) <= 1e-12 * ref.kappa
    assert int(out["converged"]) == 1
    assert int(out["row_constraint_rows"]) == ref.constraint_rows
    assert abs(int(out["row_iterations"]) - ref.iterations) <= 1
    assert int(out["capped_rc"]) == 9 and int(out["capped_iterations"]) == 2
