cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
for v in D1 D2; do MT_LIB_PATH=abl/$v.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "(teacher_forced_every_op and (c2 or c4b8)) or baseline_invariance_c2 or unfused" > gpurun_out/r2p_tf_$v.log 2>&1; echo "$v rc=$? $(tail -1 gpurun_out/r2p_tf_$v.log)" >> gpurun_out/r2p_summary.txt; done
timeout 1200 python tools/ab.py --libs abl/A.so,abl/D1.so,abl/D2.so --configs c2,c4,c4b8 --rounds 3 --runs 20 --knobs "c2=1,3,2;c4=1,2,2;c4b8=1,2,2" > gpurun_out/r2p_ab.txt 2>&1
MT_LIB_PATH=abl/D2.so timeout 600 compute-sanitizer --tool synccheck --print-limit 10 python tools/sanitize_run.py > gpurun_out/r2p_san_synccheck.log 2>&1; echo "rc=$?" >> gpurun_out/r2p_san_synccheck.log
cat gpurun_out/r2p_summary.txt gpurun_out/r2p_ab.txt; tail -2 gpurun_out/r2p_san_synccheck.log
