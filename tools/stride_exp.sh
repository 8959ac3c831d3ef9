mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$? >> gpurun_out/gpu_tests.log
timeout 300 python tools/graph_timing.py --steps 10 > gpurun_out/gt.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 45 --csv --log-file gpurun_out/launches.csv python tools/profile_run.py --runs 1 > /dev/null 2>&1
