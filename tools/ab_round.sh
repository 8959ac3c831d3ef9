# A/B of library variants (csrc/Makefile `variant`): per variant the graph-replay
# step time (tools/graph_timing.py) and one ncu launch list of the top kernels.
# VARIANTS="a b" bash tools/ab_round.sh   (main = the in-tree library)
mkdir -p gpurun_out
: > gpurun_out/ab.log
for v in main $VARIANTS; do
  V=$v; [ "$v" = main ] && V=
  echo "== $v" >> gpurun_out/ab.log
  HADIS_LIB_VARIANT=$V timeout 300 python tools/graph_timing.py --steps 20 >> gpurun_out/ab.log 2>&1
  HADIS_LIB_VARIANT=$V timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
    --log-file gpurun_out/ab_launches.csv python tools/profile_run.py --runs 1 > /dev/null 2>&1
  python tools/launches.py gpurun_out/ab_launches.csv 2>/dev/null | head -14 >> gpurun_out/ab.log
done
