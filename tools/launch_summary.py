"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import collections
import csv
import sys


def summarise(path, top=25):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0].replace("b200::<unnamed>::", "")[:48]
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "")
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1e-3)
        agg[name][0] += 1
        agg[name][1] += v * scale
    tot = sum(v[1] for v in agg.values())
    out = ["%-48s %7s %12s %6s" % ("kernel", "launches", "total_us", "share")]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        out.append("%-48s %7d %12.1f %5.1f%%" % (k, v[0], v[1], 100 * v[1] / tot))
    out.append("total %.1f us over %d launches" % (tot, sum(v[0] for v in agg.values())))
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
