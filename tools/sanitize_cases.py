"""Small problems that exercise every persistent / dataflow kernel, for
compute-sanitizer (racecheck, synccheck, memcheck): k_chol_dag in chunked and
plain mode, the dataflow sweeps, k_pcg_persistent, the graph PCG, k_syevx."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0910_5863_b200 as pb  # noqa: E402

cases = [
    # 8 substructures: chunked k_chol_dag, explicit leaves, persistent PCG, adaptive pairs (k_syevx)
    ("el222h2 adaptive", lambda: pb.BDDC(pb.Problem.cube((2, 2, 2), 2, "elasticity")), "adaptive", {}),
    # plain-mode k_chol_dag, dataflow leaf sweeps, primal tree, graph PCG
    ("sc333h3 c+e+f plain", lambda: pb.BDDC(pb.Problem.cube((3, 3, 3), 3, "scalar")), "c+e+f",
     {"BDDC_B200_DAGW": "0", "BDDC_B200_LEAF": "factor", "BDDC_B200_ROOT_DEPTH": "1", "BDDC_B200_PCG": "graph"}),
]
for name, make, mode, env in cases:
    for k, v in env.items():
        os.environ[k] = v
    row = make().run_item(mode, 10.0, 15)
    for k in env:
        del os.environ[k]
    print(name, row.constraint_rows, row.iterations, row.kappa, flush=True)
