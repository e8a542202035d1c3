cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "c1 or unfused or edge" > gpurun_out/r2m_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2m_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2m_smoke.log 2>&1
MT_LIB_PATH=abl/A.so timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2m_smoke_A.log 2>&1
for i in 1 2 3; do timeout 300 python tools/prof_exec.py --config c1 --runs 20 --knobs 0,0 2>&1 | grep "^run" | tail -10 >> gpurun_out/r2m_c1_new.txt; MT_LIB_PATH=abl/A.so timeout 300 python tools/prof_exec.py --config c1 --runs 20 --knobs 0,0 2>&1 | grep "^run" | tail -10 >> gpurun_out/r2m_c1_A.txt; done
tail -3 gpurun_out/r2m_tests.log; cat gpurun_out/r2m_smoke.log gpurun_out/r2m_smoke_A.log
