cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_bench_c2.csv python bench.py --steps 20 --warmup 5 --no-profile --no-cpu --no-baselines > gpurun_out/bench_under_ncu.txt 2>&1
for spec in "c2 1,3" "c3 1,0" "c4 0,0"; do set -- $spec
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:executor -s 5 -c 1 -o gpurun_out/full_$1 -f python tools/prof_exec.py --config $1 --knobs $2 --runs 8 > gpurun_out/ncu_$1.log 2>&1
done
ls -la gpurun_out/
