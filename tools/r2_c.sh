cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "end_to_end or teacher or large_mixes or baseline_invariance_c2 or edge or bn256" 2>&1 | tail -5 > gpurun_out/r2c_gputests.log
timeout 900 python tools/ab.py --libs abl/A.so,abl/B.so --configs c2,c3,c4,c4b8 --rounds 3 --runs 20 --knobs "c2=1,3;c3=1,0;c4=1,2;c4b8=1,2" > gpurun_out/r2c_ab.txt 2>&1
timeout 300 python tools/trace_exec.py --config c4b8 --partition 1 --claim 2 --out gpurun_out/r2c_trace_c4b8.json > gpurun_out/r2c_trace_c4b8.txt 2>&1
timeout 300 python tools/trace_exec.py --config c4 --partition 1 --claim 2 --out gpurun_out/r2c_trace_c4.json > gpurun_out/r2c_trace_c4.txt 2>&1
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_run.py > gpurun_out/r2c_san_synccheck.log 2>&1; echo "rc=$?" >> gpurun_out/r2c_san_synccheck.log
cat gpurun_out/r2c_gputests.log gpurun_out/r2c_ab.txt; tail -3 gpurun_out/r2c_san_synccheck.log
