# One GPU call: the GPU test suite, then graph timing + top kernels of the current build.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$? >> gpurun_out/gpu_tests.log
bash tools/variant_timing.sh ""
