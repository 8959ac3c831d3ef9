import cProfile, pstats, sys, os, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2509_00642_b200 import synth
from paper_2509_00642_b200.profiler import GridProfiler
cfg = synth.CONFIGS["c4"]
pool, h, noise, scores = synth.records(cfg)
prof = GridProfiler(pool, h, scores)
plan = prof.plan(cfg.thresholds)
for _ in range(3): prof.finish(prof.launch(plan))
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5): st = prof.launch(plan)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host launch {1e3*(t1-t0)/5:.2f} ms/launch, device drain {1e3*(t2-t1):.2f} ms")
pr = cProfile.Profile(); pr.enable()
for _ in range(5): st = prof.launch(plan)
pr.disable(); torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
