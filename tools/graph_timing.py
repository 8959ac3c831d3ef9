"""Where does a table build's wall time go?  Times, on one config:
  replay+finish  -- what bench.py's timed loop does per step
  replay only    -- K graph replays back to back, one sync at the end
  eager only     -- K eager launches back to back, one sync at the end
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2509_00642_b200 import synth  # noqa: E402
from paper_2509_00642_b200.profiler import GridProfiler  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--steps", type=int, default=20)
a = ap.parse_args()
cfg = synth.CONFIGS[a.config]
pool, h, noise, scores = synth.records(cfg)
prof = GridProfiler(pool, h, scores)
plan = prof.plan(cfg.thresholds)
print("stats", prof.finish(prof.launch(plan)).stats, flush=True)
rep = prof.graph(plan)
for _ in range(3):
    rep()


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(a.steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.steps, (time.perf_counter() - t0) * 1e3 / a.steps


for name, fn in (("replay+finish", rep), ("replay only", rep.launch),
                 ("eager only", lambda: prof.launch(plan)), ("replay+finish", rep),
                 ("replay only", rep.launch)):
    dev_ms, wall_ms = timed(fn)
    print(f"{name:14s} device {dev_ms:.3f} ms  wall {wall_ms:.3f} ms", flush=True)
