# compute-sanitizer over the device pipeline (c1 and c2 records -> table), the text path,
# the sharded merge and the planner tests.  Summary -> gpurun_out/sanitizer.txt
mkdir -p gpurun_out
out=gpurun_out/sanitizer.txt
: > $out
run() { echo "== $1" >> $out; shift; timeout 1200 "$@" >> $out 2>&1; echo "rc=$?" >> $out; }
CS="compute-sanitizer --print-limit 10"
run "memcheck c1" $CS --tool memcheck python tools/profile_run.py --config c1 --runs 1
run "racecheck c1" $CS --tool racecheck python tools/profile_run.py --config c1 --runs 1
run "synccheck c1" $CS --tool synccheck python tools/profile_run.py --config c1 --runs 1
run "memcheck c2" $CS --tool memcheck python tools/profile_run.py --config c2 --runs 1
run "racecheck c2 (TMA scatter, row walks)" $CS --tool racecheck python tools/profile_run.py --config c2 --runs 1
run "memcheck pytest (text, planner, sharded merge, cascade, router, prune)" $CS --tool memcheck \
    python -m pytest tests/test_gpu_text.py tests/test_gpu_parity.py -q -x \
    -k "text or planner_random or tune_weights or cascade or prune or fid_exact or sharded or graph"
grep -E "^==|ERROR SUMMARY|RACECHECK SUMMARY|passed|failed|rc=" $out > gpurun_out/sanitizer_summary.txt
