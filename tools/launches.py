"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import collections
import csv
import sys


def load(path):
    hdr, out = None, []
    for r in csv.reader(open(path)):
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                out.append((int(d["ID"]), d["Kernel Name"], float(d["Metric Value"])))
    return out


if __name__ == "__main__":
    rows = load(sys.argv[1])
    skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    rows = rows[skip:]
    agg = collections.OrderedDict()
    for _, name, ns in rows:
        short = name.split("(")[0].replace("hadis::", "")
        agg.setdefault(short, [0, 0.0])
        agg[short][0] += 1
        agg[short][1] += ns
    total = sum(v[1] for v in agg.values())
    for k, (c, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:48s} {c:4d} {ns/1e3:12.1f} us {100*ns/total:6.2f}%")
    print(f"{'TOTAL':48s} {len(rows):4d} {total/1e3:12.1f} us")
