mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$? >> gpurun_out/gpu_tests.log
timeout 300 python tools/profile_run.py --runs 2 > gpurun_out/prof.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --no-allocation > gpurun_out/bench.log 2>&1; echo rc=$? >> gpurun_out/bench.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python tools/profile_run.py --runs 2 > /dev/null 2>&1
