cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
MT_LIB_PATH=abl/E5.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "teacher_forced_every_op or large_mixes or baseline_invariance_c2 or partition_rules or c1_fp32" > gpurun_out/r2r_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2r_tests.log
timeout 1200 python tools/ab.py --libs abl/A.so,abl/D3.so,abl/E5.so --configs c2,c4,c4b8 --rounds 3 --runs 20 --knobs "c2=1,3,2;c4=1,2,2;c4b8=1,2,2" > gpurun_out/r2r_ab.txt 2>&1
for kn in "1,0,2" "1,3,2" "0,2,2"; do echo "knobs $kn" >> gpurun_out/r2r_ab2.txt; timeout 600 python tools/ab.py --libs abl/D3.so,abl/E5.so --configs c4,c4b8 --rounds 1 --runs 20 --knobs "$kn" >> gpurun_out/r2r_ab2.txt 2>&1; done
tail -2 gpurun_out/r2r_tests.log; cat gpurun_out/r2r_ab.txt gpurun_out/r2r_ab2.txt
