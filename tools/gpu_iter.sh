# One GPU call for an optimisation step: GPU tests, bench line (no CPU legs), launch list.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$? >> gpurun_out/gpu_tests.log
timeout 300 python bench.py --no-cpu-baseline --no-allocation > gpurun_out/bench.log 2>&1; echo rc=$? >> gpurun_out/bench.log
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches.csv python tools/profile_run.py --runs 2 > /dev/null 2>&1
