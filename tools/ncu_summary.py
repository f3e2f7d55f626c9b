#!/usr/bin/env python
"""Text summary of an ncu report (`ncu --set full ... -o X`) for profiles/.

    python tools/ncu_summary.py X.ncu-rep [--kernel REGEX] [--top N]

Prints, per profiled kernel launch, the headline metrics (duration, cycles,
occupancy, IPC, memory throughput, DRAM bytes) and the SASS lines with the most
warp-stall samples.
"""
import argparse
import csv
import io
import subprocess

KEYS = ["Duration", "Elapsed Cycles", "SM Frequency", "Grid Size", "Block Size", "Registers Per Thread",
        "Dynamic Shared Memory Per Block", "Theoretical Occupancy", "Achieved Occupancy", "Executed Ipc Active",
        "Issue Slots Busy", "Warp Cycles Per Issued Instruction", "Memory Throughput", "DRAM Throughput",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Compute (SM) Throughput"]


def ncu_csv(args):
    out = subprocess.run(["ncu"] + args, capture_output=True, text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--kernel", default=None)
    ap.add_argument("--top", type=int, default=12)
    a = ap.parse_args()
    sel = ["--kernel-name", "regex:" + a.kernel] if a.kernel else []
    rows = ncu_csv(["-i", a.report, "--page", "details", "--csv"] + sel)
    h = rows[0]
    ik, iid, im, iu, iv = (h.index(x) for x in ("Kernel Name", "ID", "Metric Name", "Metric Unit", "Metric Value"))
    seen = {}
    for r in rows[1:]:
        if r[im] in KEYS:
            seen.setdefault((r[iid], r[ik]), {})[r[im]] = "%s %s" % (r[iv], r[iu])
    dram = ncu_csv(["-i", a.report, "--page", "raw", "--csv", "--metrics",
                    "dram__bytes_read.sum,dram__bytes_write.sum"] + sel)
    if len(dram) > 2:
        hd = dram[0]
        for r in dram[2:]:
            key = (r[hd.index("ID")], r[hd.index("Kernel Name")])
            for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                if m in hd and key in seen:
                    seen[key][m] = "%s %s" % (r[hd.index(m)], dram[1][hd.index(m)])
    for (kid, name), m in seen.items():
        print("== launch %s: %s" % (kid, name))
        for k in KEYS + ["dram__bytes_read.sum", "dram__bytes_write.sum"]:
            if k in m:
                print("  %-36s %s" % (k, m[k]))
    src = ncu_csv(["-i", a.report, "--page", "source", "--csv", "--print-source=sass"] + sel)
    blocks, cur = [], None
    for r in src:
        if r and r[0] == "Kernel Name":
            cur = {"name": r[1], "rows": []}
            blocks.append(cur)
        elif r and r[0] == "Address":
            cur["hdr"] = r
        elif cur is not None and r and r[0].startswith("0x"):
            cur["rows"].append(r)
    for b in blocks[:1] if blocks else []:
        hd = b["hdr"]
        isamp, isrc = hd.index("Warp Stall Sampling (All Samples)"), hd.index("Source")
        tot = sum(float(r[isamp] or 0) for r in b["rows"]) or 1.0
        base = int(b["rows"][0][0], 16)
        print("== top stall SASS lines (%s, %d samples)" % (b["name"][:60], tot))
        for r in sorted(b["rows"], key=lambda r: -float(r[isamp] or 0))[:a.top]:
            print("  +0x%05x %5.1f%%  %s" % (int(r[0], 16) - base, 100 * float(r[isamp] or 0) / tot, r[isrc].strip()[:70]))


if __name__ == "__main__":
    main()
