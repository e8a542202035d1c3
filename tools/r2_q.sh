cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/r2q_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2q_tests.log
timeout 600 compute-sanitizer --tool synccheck --print-limit 10 python tools/sanitize_run.py > gpurun_out/r2q_san_synccheck.log 2>&1; echo "rc=$?" >> gpurun_out/r2q_san_synccheck.log
timeout 600 compute-sanitizer --tool memcheck --print-limit 10 python tools/sanitize_run.py > gpurun_out/r2q_san_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/r2q_san_memcheck.log
timeout 1200 python tools/ab.py --libs abl/A.so,abl/D1.so,abl/D3.so --configs c2,c4,c4b8 --rounds 3 --runs 20 --knobs "c2=1,3,2;c4=1,2,2;c4b8=1,2,2" > gpurun_out/r2q_ab.txt 2>&1
tail -2 gpurun_out/r2q_tests.log; cat gpurun_out/r2q_ab.txt; tail -2 gpurun_out/r2q_san_synccheck.log gpurun_out/r2q_san_memcheck.log
