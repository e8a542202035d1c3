cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
for c in c4 c4b8 c2; do timeout 600 python tools/knob_scan.py --config $c --runs 9 > gpurun_out/r2n_knobs_$c.txt 2>&1; done
timeout 900 python -m pytest tests/test_bench_contract.py -m gpu -x -q > gpurun_out/r2n_contract.log 2>&1; echo "rc=$?" >> gpurun_out/r2n_contract.log
head -8 gpurun_out/r2n_knobs_c4.txt; head -8 gpurun_out/r2n_knobs_c4b8.txt; head -5 gpurun_out/r2n_knobs_c2.txt; tail -2 gpurun_out/r2n_contract.log
