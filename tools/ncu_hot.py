"""Hottest SASS instructions (warp-stall samples) of one kernel in an ncu report:
python tools/ncu_hot.py report.ncu-rep kernel_regex [top]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kern,
                      "--print-source", "sass,cuda"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
recs = []
for r in rows:
    if "Address" in r and "Source" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        try:
            recs.append((int(d["Warp Stall Sampling (All Samples)"]), d["Address"], d["Source"][:90],
                         d.get("Instructions Executed", "")))
        except ValueError:
            pass
tot = sum(r[0] for r in recs) or 1
for s, a, src, ie in sorted(recs, reverse=True)[:top]:
    print(f"{100*s/tot:5.1f}% {a[-5:]} {ie:>10s}  {src}")
