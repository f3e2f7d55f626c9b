"""CPU oracle for the adaptive-BDDC hot path -- TEST INFRASTRUCTURE ONLY.

This package is a numpy/scipy restatement of the reference C++ library
(`/root/reference/proj/core/src/*.cpp`, arXiv 0910.5863 "Adaptive BDDC in
three dimensions").  Every function cites the reference file:line it follows.

Rules:
  * Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline /
    `--impl reference` leg may import this package, and only as the checker or
    the timed CPU baseline.  The product path (`paper_0910_5863_b200`) never
    imports it and fails loudly when its CUDA library is missing.
  * The reference cannot be built here (Eigen3, doctest, CLI11 and
    google-benchmark are absent).  Eigen >= 3.3 (version
    unpinned, `core/CMakeLists.txt:1`) is replaced by LAPACK through
    numpy/scipy: `SimplicialLLT` -> scipy SuperLU / dense Cholesky,
    `SelfAdjointEigenSolver` -> `numpy.linalg.eigh`.  Both compute the same
    mathematical objects; results agree to roundoff.
  * Parity is pinned against the reference's own known answers: the golden
    table `tests/data/structural_cube.csv` and the structural integers of
    `tests/test_substructuring.cpp`, `test_experiment.cpp`,
    `test_constraints.cpp`, `test_adaptive.cpp` (see tests/test_oracle_pins.py).
"""
