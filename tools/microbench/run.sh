nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
mkdir -p gpurun_out
./tools/microbench/atomics 2>&1 | tee gpurun_out/microbench_atomics.txt
