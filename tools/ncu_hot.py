"""Hottest SASS instructions (warp-stall samples) of one kernel in an ncu report:
python tools/ncu_hot.py report.ncu-rep kernel_regex [top]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kern,
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if "Address" in r and "Source" in r)
H = {h: i for i, h in enumerate(hdr)}
recs, seen = [], set()
for r in rows[rows.index(hdr) + 1:]:
    if len(r) != len(hdr) or r[H["Address"]] in seen:
        continue
    seen.add(r[H["Address"]])
    try:
        recs.append((int(r[H["Warp Stall Sampling (All Samples)"]]), r[H["Address"]][-5:],
                     int(r[H["Instructions Executed"]] or 0), r[H["Source"]].strip()))
    except ValueError:
        pass
tot = sum(x[0] for x in recs) or 1
print(f"total samples {tot}, instructions {sum(x[2] for x in recs)}")
for smp, a, ie, src in sorted(recs, reverse=True)[:top]:
    print(f"{100 * smp / tot:5.1f}% {a} {ie:>11d}  {src[:90]}")
