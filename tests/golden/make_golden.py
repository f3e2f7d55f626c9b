"""Regenerate the golden fixtures from the reference's own test data.

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
It copies the reference's golden table (proj/tests/data/structural_cube.csv,
compared byte-for-byte by proj/tests/test_experiment.cpp:184-194) and records
the structural known answers its test suites assert, with their sources.
The GPU box has no /root/reference: the tests read only these files.
"""
import json
import shutil
from pathlib import Path

HERE = Path(__file__).resolve().parent
REF = Path("/root/reference/proj/tests")

shutil.copyfile(REF / "data" / "structural_cube.csv", HERE / "structural_cube.csv")

# Structural known answers (file:line of the reference assertion each one pins)
PINS = {
    "floating_222_h4_elasticity": {"dofs": 2187, "corners": 7, "edges": 6, "faces": 12,
                                   "classification_corners": 1, "w_dim": 3000, "wc_dim": 2925,
                                   "interface": 651, "src": "test_substructuring.cpp:57-81"},
    "clamped_222_h4_elasticity": {"dofs": 2187, "free": 1944, "interface": 600, "corners": 7,
                                  "classification_corners": 1, "edges": 6, "faces": 12, "wc_dim": 2634,
                                  "rows_ce": 54, "src": "test_experiment.cpp:75-95"},
    "floating_222_h3_scalar": {"corners": 7, "edges": 6, "faces": 12, "w_dim": 512, "wc_dim": 487,
                               "src": "test_substructuring.cpp:83-91"},
    "planar_221_h4_elasticity": {"corners": 10, "edges": 1, "faces": 4, "wc_dim": 1458,
                                 "src": "test_substructuring.cpp:93-101"},
    "planar_221_h4_scalar": {"corners": 2, "edges": 1, "faces": 4, "src": "test_substructuring.cpp:103-107"},
    "stacked_112_h2_elasticity": {"faces_before": 1, "face_nodes": 9, "corners_after": 4, "w_dim": 162,
                                  "interface": 27, "corner_dofs": 12, "wc_dim": 150,
                                  "src": "test_substructuring.cpp:36-55"},
    "edge_rows_222_h4": {"edge_averages": 18, "rows_e": 54, "rows_ef": 90, "src": "test_constraints.cpp:60-70"},
    "pair_112_h2_scalar": {"n_corner": 4, "n_shared": 5, "dim": 14, "src": "test_adaptive.cpp:126-137"},
    "acceptance_c3": {"dofs": 7803, "kappa_lo": 22.64, "kappa_hi": 33.96, "it_lo": 10, "it_hi": 16,
                      "src": "acceptance/acceptance_main.cpp:130-151"},
    "lanczos_diag_1_10": {"iterations": 10, "kappa": 10.0, "src": "test_solver.cpp:147-159"},
    "table_format": {"csv": "mode_or_tau,omega_tilde,Nc,kappa,it\nc+e,,54,7.298,15\n",
                     "markdown": "| mode_or_tau | omega_tilde | Nc | kappa | it |\n| --- | --- | --- | --- | --- |\n"
                                 "| 10 | 9.639 | 54 | 7.298 | 15* |\n",
                     "src": "test_experiment.cpp:145-170"},
}
(HERE / "structural_pins.json").write_text(json.dumps(PINS, indent=1) + "\n")
print("wrote", HERE / "structural_cube.csv", HERE / "structural_pins.json")
