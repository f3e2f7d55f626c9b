"""Device-timed preconditioner stages with the two front-sweep schedules
(BDDC_B200_SWEEP=dag|cluster) on the BASELINE configs (one B200)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0910_5863_b200 as pb  # noqa: E402

MODES = {3: ("adaptive", 5.0, 15, False), 4: ("adaptive", 10.0, 15, True), 5: ("adaptive", 10.0, 15, False)}
for c in [int(a) for a in sys.argv[1:]] or [3, 4]:
    b = pb.BDDC(config=c)
    mode, tau, maxv, bf = MODES[c]
    for sweep in ("cluster", "dag", "cluster", "dag"):
        os.environ["BDDC_B200_SWEEP"] = sweep
        out = b.step(mode, tau, maxv, base_faces=bf)
        ops = b.operator_times(20)
        print(json.dumps({"config": c, "sweep": sweep, "step_ms": out["seconds"] * 1e3, "it": out["iterations"],
                          "kappa": out["kappa"], "precond_ms": ops["precond"] * 1e3,
                          "leaf_fwd_ms": ops["leaf_fwd"] * 1e3, "leaf_bwd_ms": ops["leaf_bwd"] * 1e3,
                          "tree_fwd_ms": ops["tree_fwd"] * 1e3, "tree_bwd_ms": ops["tree_bwd"] * 1e3,
                          "leaf_fwd_gbs": ops["leaf_sweep_bytes"] / ops["leaf_fwd"] / 1e9,
                          "leaf_bwd_gbs": ops["leaf_sweep_bytes"] / ops["leaf_bwd"] / 1e9,
                          "precond_gbs": ops["precond_bytes"] / ops["precond"] / 1e9}), flush=True)
