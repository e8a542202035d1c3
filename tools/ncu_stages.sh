# per-stage ncu counters of the uniform 4-stage schedule (stage-split launches), one GPU
cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "stage_split" 2>&1 | tail -2
for spec in "c3 1,0" "c4b8 1,2"; do set -- $spec
  timeout 900 ncu --set full --clock-control none -k regex:executor -s 8 -c 4 -o gpurun_out/stg_$1 -f python tools/prof_exec.py --config $1 --schedule uniform4 --knobs $2 --stage-split --runs 3 > gpurun_out/stg_$1.log 2>&1
  tail -2 gpurun_out/stg_$1.log
done
