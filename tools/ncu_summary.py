"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch)."""
import csv
import sys
from collections import defaultdict


def load(path):
    rows, hdr = [], None
    for r in csv.reader(open(path)):
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] == "gpu__time_duration.sum":
                rows.append(d)
    return rows


def summary(path, top=40, key_len=70):
    rows = load(path)
    agg = defaultdict(lambda: [0, 0.0, ""])
    for d in rows:
        name = d["Kernel Name"][:key_len] + " grid=" + d["Grid Size"]
        scale = 1e-3 if d["Metric Unit"] == "ns" else (1.0 if d["Metric Unit"] == "us" else 1e3)
        agg[name][0] += 1
        agg[name][1] += float(d["Metric Value"].replace(",", "")) * scale
    tot = sum(v[1] for v in agg.values())
    out = ["%d launches, %.1f us total" % (len(rows), tot)]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        out.append("%10.1f us %6d x %8.2f us %5.1f%%  %s" % (v[1], v[0], v[1] / v[0], 100 * v[1] / tot, k))
    return "\n".join(out)


if __name__ == "__main__":
    print(summary(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40))
