mkdir -p gpurun_out
for d in 0 1 2 3; do
HADIS_DBG=$d timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:bucket_scatter -c 2 --csv python tools/profile_run.py --runs 2 2>/dev/null | grep -E "gpu__time|dram__" | tail -3 | sed "s/^/dbg$d /" >> gpurun_out/dbg.txt
done
