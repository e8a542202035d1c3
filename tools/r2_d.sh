cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
ok=""
for v in A E1 E1RR E1RR0 E2 E2RR; do
  MT_LIB_PATH=abl/$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "teacher_forced_every_op and (c2 or c3 or c4b8)" > gpurun_out/r2d_tf_$v.log 2>&1
  rc=$?; echo "$v rc=$rc $(tail -1 gpurun_out/r2d_tf_$v.log)" >> gpurun_out/r2d_summary.txt
  if [ $rc = 0 ]; then ok="$ok,abl/$v.so"; fi
done
ok=${ok#,}
echo "passing: $ok" >> gpurun_out/r2d_summary.txt
timeout 1500 python tools/ab.py --libs $ok --configs c2,c3,c4,c4b8 --rounds 3 --runs 20 --knobs "c2=1,3;c3=1,0;c4=1,2;c4b8=1,2" > gpurun_out/r2d_ab.txt 2>&1
cat gpurun_out/r2d_summary.txt gpurun_out/r2d_ab.txt
