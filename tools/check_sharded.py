"""Run under torchrun: the pair-sharded multi-rank table (one all-gather merge)
must equal the single-process table row for row.  Ranks may share one GPU
when HADIS_DIST_BACKEND=gloo (the NVLink/NCCL path needs one GPU per rank)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2509_00642_b200 import synth  # noqa: E402
from paper_2509_00642_b200.profiler import GridProfiler, light_scores  # noqa: E402
from paper_2509_00642_b200.sharding import FIELDS, profile_sharded, solve_sharded  # noqa: E402


def main():
    backend = os.environ.get("HADIS_DIST_BACKEND", "nccl")
    local = int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dist.init_process_group(backend)
    cfg = synth.Config("chk", 8, 200_000, 64, 1e-3)
    pool, h, noise, scores = synth.records(cfg, seed=5)
    prof = GridProfiler(pool, h, scores)
    pairs, merged = profile_sharded(prof, cfg.thresholds, dist)
    # the same through ShardedTable with a CUDA graph per rank, two steps
    from paper_2509_00642_b200.sharding import ShardedTable
    st = ShardedTable(pool, prof.h, prof.scores, cfg.thresholds, dist)
    for _ in range(2):
        again = st.step()
    for f in FIELDS:
        assert torch.equal(again[f], merged[f]), f
    if dist.get_rank() == 0:
        single = prof.run(cfg.thresholds)
        for f in FIELDS:
            a = merged[f].cpu().numpy()
            b = getattr(single, f).cpu().numpy().astype(a.dtype)
            assert np.array_equal(a, b), f
    # c5-style allocation search sharded over the points
    from paper_2509_00642_b200.planner import solve_many
    from paper_2509_00642_b200.profiler import rows_from_device
    table_rows = rows_from_device(prof.run(cfg.thresholds), pool, cfg.thresholds)
    cat = cfg.catalog()
    lams = [0.1 * (i + 1) for i in range(97)] + [0.0, 500.0]
    slos = [(15.0, 30.0, 60.0, 90.0)[i % 4] for i in range(len(lams))]
    plans = solve_sharded(table_rows, cat, lams, None, 8, slos, 1.5, dist=dist)
    if dist.get_rank() == 0:
        want = solve_many(table_rows, cat, lams, None, 8, slos, 1.5)
        assert len(plans) == len(want)
        for a, b in zip(plans, want):
            assert (a.row, a.workers, a.batches, a.path_latency_s, a.infeasible) == \
                (b.row, b.workers, b.batches, b.path_latency_s, b.infeasible)
        print(f"sharded OK: world={dist.get_world_size()} rows={len(merged['pair'])} "
              f"pairs={len(pairs)} plans={len(plans)}", flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
