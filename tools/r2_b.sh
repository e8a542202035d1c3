cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 2>&1 | tail -25 > gpurun_out/r2b_gputests.log
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > gpurun_out/r2b_san_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/r2b_san_$tool.log
done
timeout 300 python tools/trace_exec.py --config c4b8 --partition 1 --claim 2 --out gpurun_out/r2b_trace_c4b8.json > gpurun_out/r2b_trace_c4b8.txt 2>&1
timeout 300 python tools/trace_exec.py --config c4 --partition 1 --claim 2 --out gpurun_out/r2b_trace_c4.json > gpurun_out/r2b_trace_c4.txt 2>&1
cat gpurun_out/r2b_gputests.log; tail -3 gpurun_out/r2b_san_*.log
