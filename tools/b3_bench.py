"""Time the record-store stages alone (B0-B2 plan, B3 scatter, K1) on a
config's synthetic records: python tools/b3_bench.py [--config c4] [--iters 20].
Library variant via HADIS_LIB_VARIANT (see csrc/Makefile `variant`)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2509_00642_b200 import _lib, synth  # noqa: E402
from paper_2509_00642_b200.profiler import GridProfiler  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--k", type=int, default=0, help="threshold-grid size override")
a = ap.parse_args()
cfg = synth.CONFIGS[a.config]
if a.k:
    import dataclasses
    cfg = dataclasses.replace(cfg, k=a.k)
pool, h, noise, scores = synth.records(cfg)
prof = GridProfiler(pool, h, scores)
plan = prof.plan(cfg.thresholds)
lib, p = prof.lib, _lib.ptr
hfix, bs, rplan = prof._bucket_store(plan.n_light)
sc = prof.scores[plan.slot0:plan.slot0 + plan.n_light]
U, n, L = plan.U, prof.n, plan.n_light
bins = (U + 1) * (U + 1) * L
cnt = torch.empty(bins, dtype=torch.int32, device="cuda")
hs = torch.empty(bins, dtype=torch.int64, device="cuda")
scanned = torch.empty((U + 1) * L, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream().cuda_stream


def stage(i):
    if i == 0:
        _lib.check(lib.hadis_records_plan(p(prof.h), n, p(plan.d_u), U, prof.shift, p(prof.bad),
                                          p(rplan), rplan.numel(), st), "plan")
    elif i == 1:
        _lib.check(lib.hadis_records_scatter(p(prof.h), p(sc), n, L, p(plan.d_u), U, prof.shift,
                                             p(hfix), p(bs), p(rplan), rplan.numel(), st),
                   "scatter")
    elif i == 2:
        _lib.check(lib.hadis_bin_hist_rows(p(hfix), p(bs), n, L, U, p(rplan), p(cnt), p(hs),
                                           p(scanned), st), "k1")
    else:
        _lib.check(lib.hadis_hist_scan(p(cnt), p(hs), L, U, p(scanned), st), "k2")


for _ in range(3):
    for i in range(4):
        stage(i)
torch.cuda.synchronize()
ev = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(a.iters)]
for it in range(a.iters):
    for i in range(4):
        ev[it][i].record()
        stage(i)
    ev[it][4].record()
torch.cuda.synchronize()
names = ("plan", "scatter", "k1", "k2")
algo = {"plan": 8 * n, "scatter": 8 * n * (1 + L), "k1": 16 * n * ((L + 3) // 4), "k2": 24 * (U + 1) * (U + 1) * L}
for i, nm in enumerate(names):
    ts = sorted(e[i].elapsed_time(e[i + 1]) for e in ev)
    med = ts[len(ts) // 2]
    print(f"{os.environ.get('HADIS_LIB_VARIANT', 'main'):>10} K={cfg.k} {nm:8s} median {med * 1e3:8.1f} us "
          f"min {ts[0] * 1e3:8.1f} us  {algo[nm] / med / 1e6:7.0f} GB/s algorithmic")
