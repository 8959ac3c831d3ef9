# Time build variants on the GPU box: bash tools/variant_timing.sh "" "-DFOO=1" ...
# Each argument is passed to make as EXTRA nvcc flags; per variant: graph-replay
# time (tools/graph_timing.py) and the top kernels of one ncu launch list.
mkdir -p gpurun_out
: > gpurun_out/variants.log
for v in "$@"; do
  echo "== variant '$v'" >> gpurun_out/variants.log
  (cd paper_2509_00642_b200/csrc && rm -f ../libhadis_b200.so && make EXTRA="$v" > /dev/null 2>&1)
  timeout 300 python tools/graph_timing.py --steps 10 2>&1 | grep -v eager | head -3 >> gpurun_out/variants.log
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 45 --csv \
    --log-file gpurun_out/variant_launches.csv python tools/profile_run.py --runs 1 > /dev/null 2>&1
  python tools/launches.py gpurun_out/variant_launches.csv 2>/dev/null | head -8 >> gpurun_out/variants.log
done
(cd paper_2509_00642_b200/csrc && make -B > /dev/null 2>&1)
