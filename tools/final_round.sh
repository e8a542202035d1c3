# round-end evidence refresh (one GPU): GPU tests, smoke, bench line, zoo/config table, ncu
cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/fin_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1
timeout 700 python bench.py > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err
timeout 1500 python tools/zoo_table.py --configs c2,c3,c4,c4b8,vgg_r18,r18_r34,r34_r50,r50_r101,vgg_r18_r50,r18_r34_r50,zoo5,alex_vgg_r18,r18_r34_r101,r18_r50_r101 --runs 20 --cands 128 --out gpurun_out/fin_zoo.json > gpurun_out/fin_zoo.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/fin_launches_c2.csv python bench.py --steps 20 --warmup 5 --no-profile --no-cpu --no-baselines > gpurun_out/fin_bench_ncu.txt 2>&1
for spec in "c2 1,3" "c3 1,0" "c4 1,2"; do set -- $spec
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:executor -s 5 -c 1 -o gpurun_out/fin_full_$1 -f python tools/prof_exec.py --config $1 --knobs $2 --runs 8 > gpurun_out/fin_ncu_$1.log 2>&1
done
cat gpurun_out/fin_gputests.log gpurun_out/fin_smoke.log; head -c 400 gpurun_out/fin_bench.json
