# One GPU call: tests, full bench line, launch list, ncu --set full of the top kernels.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/smi.txt
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$? >> gpurun_out/gpu_tests.log
timeout 600 python bench.py > gpurun_out/bench_full.log 2>&1; echo rc=$? >> gpurun_out/bench_full.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches.csv python tools/profile_run.py --runs 2 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bucket_scatter|row_hist_kernel|scan_cols|filter_kernel|bucket_min_kernel|decide_kernel|group_cands|emit_rows" -c 8 -o gpurun_out/prof_round python tools/profile_run.py --runs 1 > gpurun_out/ncu_round.log 2>&1
