"""c5 allocation search alone (for ncu): the c2 table on the device, 1000
(demand, SLO) points, with empty queues and with U(0, 40) backlogs.
python tools/k5_run.py [--iters 3]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_00642_b200 import synth  # noqa: E402
from paper_2509_00642_b200.planner import DeviceRows  # noqa: E402
from paper_2509_00642_b200.profiler import GridProfiler  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=3)
a = ap.parse_args()
cfg = synth.CONFIGS["c2"]
pool, h, noise, scores = synth.records(cfg)
dt = GridProfiler(pool, h, scores).run(cfg.thresholds)
cat = cfg.catalog()
dr = DeviceRows.from_device_table(dt, pool, cat)
lams, slos, _ = synth.replan_points(1000)
P = len(lams)
d_lam = torch.tensor(lams, dtype=torch.float64, device="cuda")
d_slo = torch.tensor(slos, dtype=torch.float64, device="cuda")
d_w = torch.full((P,), cfg.workers, dtype=torch.int32, device="cuda")
qs = [torch.zeros((P, len(cat.variants)), dtype=torch.float64, device="cuda"),
      torch.from_numpy(np.random.default_rng(3).uniform(0, 40, (P, len(cat.variants)))).cuda()]
for q in qs:
    for _ in range(a.iters):
        dr.launch(d_lam, d_slo, d_w, q, 1.5)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
ev[0].record()
dr.launch(d_lam, d_slo, d_w, qs[0], 1.5)
ev[1].record()
dr.launch(d_lam, d_slo, d_w, qs[1], 1.5)
ev[2].record()
torch.cuda.synchronize()
print(f"rows {dt.n_rows}: 1000 points {ev[0].elapsed_time(ev[1]):.3f} ms (no queues), "
      f"{ev[1].elapsed_time(ev[2]):.3f} ms (U(0,40) backlogs)")
