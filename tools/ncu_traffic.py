#!/usr/bin/env python
"""DRAM traffic of one leaf factorization / one operator application (ncu).

The bench line's `roofline.traffic` is the DRAM bytes of the dominant kernel
family per launch.  This script runs one phase of the engine twice (the first
warms caches and buffers) and reports the launch window of the second run, so
ncu can capture exactly that window:

    python tools/ncu_traffic.py --config 4 --phase leaf --count   # {"skip": S, "count": C}
    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \\
        --clock-control none -s S -c C --csv --log-file gpurun_out/traffic_leaf_cfg4.csv \\
        python tools/ncu_traffic.py --config 4 --phase leaf
    python tools/ncu_traffic.py --summarise gpurun_out/traffic_leaf_cfg4.csv --config 4 --phase leaf \\
        --out profiles/r01_traffic.json

Phases: `leaf` = Engine::analysis (leaf front assembly + batched partial
Cholesky: A_II eliminated, S_s formed); `apply` = one Schur apply + one
preconditioner apply (the PCG iteration's operators) after a full adaptive
setup.  No timing is taken from the ncu run (cold, serialised launches).
"""
import argparse
import collections
import csv
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

MODES = {1: ("c+e+f", 10.0, 15, False), 2: ("adaptive", 10.0, 10, False), 3: ("adaptive", 5.0, 15, False),
         4: ("adaptive", 10.0, 15, True), 5: ("adaptive", 10.0, 15, False)}


def run(cfg, phase):
    import numpy as np
    import paper_0910_5863_b200 as pb
    b = pb.BDDC(config=cfg)
    if phase == "leaf":
        b.analysis()
        l0 = pb.BDDC.launch_count()
        b.analysis()
    else:
        mode, tau, maxv, faces = MODES[cfg]
        b.run_item(mode, tau, maxv, base_faces=faces)
        x = np.random.default_rng(0).standard_normal(b.interface_size)
        b.schur_apply(x)
        b.precond_apply(x)
        l0 = pb.BDDC.launch_count()
        b.schur_apply(x)
        b.precond_apply(x)
    l1 = pb.BDDC.launch_count()
    return l0, l1 - l0


def summarise(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    per = collections.defaultdict(lambda: collections.defaultdict(float))
    names = {}
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        key = d["ID"]
        names[key] = d["Kernel Name"].split("(")[0].replace("b200::<unnamed>::", "")
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9,
                 "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3}.get(unit, 1.0)
        per[key][d["Metric Name"]] += v * scale
    tot = collections.defaultdict(float)
    by_kernel = collections.defaultdict(lambda: [0, 0.0])
    for k, m in per.items():
        for n, v in m.items():
            tot[n] += v
        by_kernel[names[k]][0] += 1
        by_kernel[names[k]][1] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    return {"launches": len(per), "dram_bytes_read": tot["dram__bytes_read.sum"],
            "dram_bytes_write": tot["dram__bytes_write.sum"],
            "serialised_seconds": tot["gpu__time_duration.sum"],
            "by_kernel_bytes": {k: v[1] for k, v in sorted(by_kernel.items(), key=lambda x: -x[1][1])[:12]}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--phase", choices=["leaf", "apply"], default="leaf")
    ap.add_argument("--count", action="store_true")
    ap.add_argument("--summarise")
    ap.add_argument("--out")
    args = ap.parse_args()
    if args.summarise:
        s = summarise(args.summarise)
        s["source"] = os.path.basename(args.summarise)
        print(json.dumps(s, indent=1))
        if args.out:
            data = json.load(open(args.out)) if os.path.exists(args.out) else {}
            data["cfg%d_%s" % (args.config, args.phase)] = s
            json.dump(data, open(args.out, "w"), indent=1, sort_keys=True)
        return
    skip, count = run(args.config, args.phase)
    if args.count:
        print(json.dumps({"skip": skip, "count": count}))


if __name__ == "__main__":
    main()
