# round-2 final evidence on the shipped library: full GPU tests, bench line, reference arm, smoke,
# sanitizers, ncu launch list + executor captures (summarised on the box, reports removed)
cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
( time timeout 1500 python -m pytest tests -m gpu -x -q --durations=5 ) > gpurun_out/r2s_gputests.log 2>&1
( time timeout 900 python bench.py ) > gpurun_out/r2s_bench.json 2> gpurun_out/r2s_bench.err
( time timeout 600 python bench.py --impl reference --steps 3 --warmup 1 ) > gpurun_out/r2s_ref.json 2> gpurun_out/r2s_ref.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s_smoke.log 2>&1
for tool in memcheck racecheck synccheck; do timeout 900 compute-sanitizer --tool $tool --print-limit 10 python tools/sanitize_run.py > gpurun_out/r2s_san_$tool.log 2>&1; echo "rc=$?" >> gpurun_out/r2s_san_$tool.log; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/r2s_launches_bench.csv python bench.py --steps 10 --warmup 3 --no-profile --no-cpu --no-baselines --search-cand 8 > gpurun_out/r2s_bench_under_ncu.txt 2>&1
for spec in "c4 1,2" "c4b8 1,2" "c2 1,3" "c3 1,0"; do set -- $spec
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:executor -s 5 -c 1 -o gpurun_out/r2s_full_$1 -f python tools/prof_exec.py --config $1 --knobs $2 --runs 8 > gpurun_out/r2s_ncu_$1.log 2>&1
  ncu -i gpurun_out/r2s_full_$1.ncu-rep --page raw --csv > gpurun_out/r2s_full_$1.raw.csv 2>/dev/null
  ncu -i gpurun_out/r2s_full_$1.ncu-rep --page details --csv > gpurun_out/r2s_full_$1.details.csv 2>/dev/null
  ncu -i gpurun_out/r2s_full_$1.ncu-rep --page source --csv > gpurun_out/r2s_full_$1.source.csv 2>/dev/null
  rm -f gpurun_out/r2s_full_$1.ncu-rep
done
rm -f gpurun_out/*_raw.npy
du -sh gpurun_out; tail -4 gpurun_out/r2s_gputests.log; head -c 700 gpurun_out/r2s_bench.json; cat gpurun_out/r2s_smoke.log; tail -2 gpurun_out/r2s_san_*.log
