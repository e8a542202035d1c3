cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python tools/ab.py --libs abl/A.so,abl/L1.so --configs c2,c4,c4b8 --rounds 3 --runs 20 --knobs "c2=1,3;c4=1,2;c4b8=1,2" > gpurun_out/r2h_ab.txt 2>&1
timeout 600 compute-sanitizer --tool synccheck --print-limit 10 python tools/sanitize_run.py > gpurun_out/r2h_san_synccheck.log 2>&1; echo "rc=$?" >> gpurun_out/r2h_san_synccheck.log
cat gpurun_out/r2h_ab.txt; tail -2 gpurun_out/r2h_san_synccheck.log
