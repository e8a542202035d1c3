cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
for v in B2 B3; do
  MT_LIB_PATH=abl/$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "teacher_forced_every_op and (c4 or c2)" > gpurun_out/r2f_tf_$v.log 2>&1
  echo "$v rc=$? $(tail -1 gpurun_out/r2f_tf_$v.log)" >> gpurun_out/r2f_summary.txt
done
timeout 1500 python tools/ab.py --libs abl/A.so,abl/B0.so,abl/B1.so,abl/B2.so,abl/B3.so --configs c2,c4,c4b8 --rounds 2 --runs 20 --knobs "c2=1,3;c4=1,2;c4b8=1,2" > gpurun_out/r2f_ab.txt 2>&1
cat gpurun_out/r2f_summary.txt gpurun_out/r2f_ab.txt
