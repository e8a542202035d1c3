# round-2 evidence, part 2: f1 search study, f3 refresh, ncu captures, conv throughput, single tenants
cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python tools/search_study.py --out gpurun_out/r2j_search.json > gpurun_out/r2j_search.log 2>&1
for c in c3 c4; do timeout 300 python tools/issue_stall.py --config $c --runs 5 --out gpurun_out/r2j_issue_stall_$c.json > gpurun_out/r2j_issue_stall_$c.log 2>&1; done
timeout 600 python tools/prefilter_study.py --config c3 --n 1024 --keep 64 --out gpurun_out/r2j_prefilter_c3.json > gpurun_out/r2j_prefilter_c3.log 2>&1
timeout 600 python tools/prefilter_study.py --config c4 --n 512 --keep 64 --out gpurun_out/r2j_prefilter_c4.json > gpurun_out/r2j_prefilter_c4.log 2>&1
for spec in "256 256 56" "512 512 28" "128 128 112" "64 256 56"; do set -- $spec
  k=3; [ $1 = 64 ] && k=1; p=1; [ $k = 1 ] && p=0
  timeout 300 python tools/op_bench.py --cin $1 --cout $2 --k $k --p $p --hw $3 --batch 8 --runs 20 > gpurun_out/r2j_op_$1_$2_$3.log 2>&1
done
for c in r50 vgg mbv2 r18; do timeout 300 python tools/prof_exec.py --config $c --runs 12 --knobs 1,0 > gpurun_out/r2j_single_$c.log 2>&1; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/r2j_launches_bench.csv python bench.py --steps 10 --warmup 3 --no-profile --no-cpu --no-baselines --search-cand 8 > gpurun_out/r2j_bench_under_ncu.txt 2>&1
for spec in "c4 1,2" "c4b8 1,2" "c2 1,3" "c3 1,0"; do set -- $spec
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:executor -s 5 -c 1 -o gpurun_out/r2j_full_$1 -f python tools/prof_exec.py --config $1 --knobs $2 --runs 8 > gpurun_out/r2j_ncu_$1.log 2>&1
done
timeout 900 ncu --set full --clock-control none -k regex:executor -s 8 -c 4 -o gpurun_out/r2j_stages_c4b8 -f python tools/prof_exec.py --config c4b8 --knobs 1,2 --runs 3 --schedule uniform4 --stage-split > gpurun_out/r2j_ncu_stages.log 2>&1
# keep the box's gpurun_out small (<64 MiB): summaries of the ncu reports, not the reports
for f in gpurun_out/r2j_full_*.ncu-rep gpurun_out/r2j_stages_c4b8.ncu-rep; do
  [ -f "$f" ] || continue
  b=${f%.ncu-rep}
  ncu -i "$f" --page raw --csv > "$b.raw.csv" 2>/dev/null
  ncu -i "$f" --page details --csv > "$b.details.csv" 2>/dev/null
  ls -la "$f" >> gpurun_out/r2j_ncu_sizes.txt
  rm -f "$f"
done
rm -f gpurun_out/*_raw.npy
du -sh gpurun_out; ls -la gpurun_out/ | grep r2j | head -60; tail -5 gpurun_out/r2j_search.log
