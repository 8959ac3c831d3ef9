"""Minimal driver for ncu: build a config's records and run the device
pipeline `--runs` times (first run also grows capacities)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2509_00642_b200 import synth  # noqa: E402
from paper_2509_00642_b200.profiler import GridProfiler  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--runs", type=int, default=2)
ap.add_argument("--solve", action="store_true")
a = ap.parse_args()
cfg = synth.CONFIGS[a.config]
pool, h, noise, scores = synth.records(cfg)
prof = GridProfiler(pool, h, scores)
plan = prof.plan(cfg.thresholds)
for r in range(a.runs):
    dt = prof.finish(prof.launch(plan))
    print("run", r, dt.stats, flush=True)
torch.cuda.synchronize()
