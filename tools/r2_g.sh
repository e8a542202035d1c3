cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "c1_fp32 or end_to_end or teacher or large_mixes or baseline_invariance_c2 or edge or bn256 or stage_split or steal or partition_rules or profile_batch or run_host or unfused" > gpurun_out/r2g_gputests.log 2>&1
echo "gpu tests rc=$?" >> gpurun_out/r2g_gputests.log
timeout 900 python tools/ab.py --libs abl/A.so,abl/P0.so,abl/P1.so --configs c2,c4,c4b8 --rounds 3 --runs 20 --knobs "c2=1,3;c4=1,2;c4b8=1,2" > gpurun_out/r2g_ab.txt 2>&1
timeout 600 compute-sanitizer --tool synccheck --print-limit 10 python tools/sanitize_run.py > gpurun_out/r2g_san_synccheck.log 2>&1; echo "rc=$?" >> gpurun_out/r2g_san_synccheck.log
timeout 300 python tools/trace_exec.py --config c4b8 --partition 1 --claim 2 --out gpurun_out/r2g_trace_c4b8.json > gpurun_out/r2g_trace_c4b8.txt 2>&1
tail -3 gpurun_out/r2g_gputests.log; cat gpurun_out/r2g_ab.txt; tail -2 gpurun_out/r2g_san_synccheck.log
