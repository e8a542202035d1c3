cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
for v in V4 V5; do
  MT_LIB_PATH=abl/$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "teacher_forced_every_op and (c2 or c3 or c4b8)" > gpurun_out/r2e_tf_$v.log 2>&1
  echo "$v rc=$? $(tail -1 gpurun_out/r2e_tf_$v.log)" >> gpurun_out/r2e_summary.txt
done
timeout 1500 python tools/ab.py --libs abl/A.so,abl/V1.so,abl/V2.so,abl/V3.so,abl/V4.so,abl/V5.so --configs c2,c4,c4b8 --rounds 2 --runs 20 --knobs "c2=1,3;c4=1,2;c4b8=1,2" > gpurun_out/r2e_ab.txt 2>&1
MT_LIB_PATH=abl/A.so timeout 300 python tools/trace_exec.py --config c4b8 --partition 1 --claim 2 --out gpurun_out/r2e_trace_A_c4b8.json > gpurun_out/r2e_trace_A_c4b8.txt 2>&1
MT_LIB_PATH=abl/V4.so timeout 300 python tools/trace_exec.py --config c4b8 --partition 1 --claim 2 --out gpurun_out/r2e_trace_V4_c4b8.json > gpurun_out/r2e_trace_V4_c4b8.txt 2>&1
cat gpurun_out/r2e_summary.txt gpurun_out/r2e_ab.txt
