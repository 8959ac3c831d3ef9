# B3 iteration: stage timings (main + variants named in $VARIANTS), optional ncu capture
# (NCU=variant or main) and parity tests (PARITY=1)
mkdir -p gpurun_out
( python tools/b3_bench.py
  for v in $VARIANTS; do HADIS_LIB_VARIANT=$v python tools/b3_bench.py; done ) > gpurun_out/b3.log 2>&1
if [ -n "$NCU" ]; then
  V=$NCU; [ "$V" = main ] && V=
  HADIS_LIB_VARIANT=$V timeout 600 ncu --set full --clock-control none --import-source on -k regex:bucket_scatter_tma -c 1 -o gpurun_out/b3_new python tools/b3_bench.py --iters 1 > /dev/null 2>&1
fi
if [ "$PARITY" = 1 ]; then
  timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -x -q > gpurun_out/parity.log 2>&1; echo rc=$? >> gpurun_out/parity.log
fi
