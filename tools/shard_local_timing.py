"""Local build time of each rank's shard of an N-way c4 split, on one GPU
(what every rank of `bench.py --gpus N` replays before the all-gather):
python tools/shard_local_timing.py --world 8"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_00642_b200 import synth  # noqa: E402
from paper_2509_00642_b200.profiler import GridProfiler, pair_list  # noqa: E402
from paper_2509_00642_b200.sharding import shard_light_groups  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--world", type=int, default=8)
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--rank", type=int, default=-1, help="only this rank's shard")
a = ap.parse_args()
cfg = synth.CONFIGS[a.config]
pool, h, noise, scores = synth.records(cfg)
pairs = pair_list(pool)
d_h = torch.from_numpy(h).cuda()
for rank in range(a.world) if a.rank < 0 else [a.rank]:
    _, mine = shard_light_groups(pairs, a.world, rank)
    slots = sorted({i for i, _ in mine})
    prof = GridProfiler(pool, d_h, torch.from_numpy(np.ascontiguousarray(scores[slots])).cuda(),
                        slots=slots)
    plan = prof.plan(cfg.thresholds, pairs=mine)
    dt = prof.run(cfg.thresholds, pairs=mine)
    rep = prof.graph(plan)
    for _ in range(3):
        rep()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        rep()
    e1.record()
    torch.cuda.synchronize()
    print(f"rank {rank}/{a.world}: {len(mine)} pairs, light models {slots}, rows {dt.n_rows}, "
          f"local build {e0.elapsed_time(e1) / a.steps:.3f} ms", flush=True)
    del prof, rep
    torch.cuda.empty_cache()
