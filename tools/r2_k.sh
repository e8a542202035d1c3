cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
MT_LIB_PATH=abl/R3.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "partition_rules or large_mixes or (teacher_forced_every_op and c4b8)" > gpurun_out/r2k_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2k_tests.log
timeout 900 python tools/ab.py --libs abl/A.so,abl/R3.so --configs c2,c4,c4b8 --rounds 2 --runs 20 --knobs "c2=1,3,2;c4=1,2,2;c4b8=1,2,2" > gpurun_out/r2k_ab_s2.txt 2>&1
timeout 900 python tools/ab.py --libs abl/A.so,abl/R3.so --configs c2,c4,c4b8 --rounds 2 --runs 20 --knobs "c2=1,3,3;c4=1,2,3;c4b8=1,2,3" > gpurun_out/r2k_ab_s3d.txt 2>&1
timeout 900 python tools/ab.py --libs abl/A.so,abl/R3.so --configs c2,c4,c4b8 --rounds 2 --runs 20 --knobs "c2=1,0,3;c4=1,0,3;c4b8=1,0,3" > gpurun_out/r2k_ab_s3.txt 2>&1
tail -2 gpurun_out/r2k_tests.log; cat gpurun_out/r2k_ab_s2.txt gpurun_out/r2k_ab_s3d.txt gpurun_out/r2k_ab_s3.txt
