cd $GRAFT_REPO_ROOT
for spec in "--cin 512 --cout 512 --k 3 --p 1 --hw 7" "--cin 960 --cout 160 --k 1 --p 0 --hw 7" "--cin 64 --cout 64 --k 3 --p 1 --hw 56" "--cin 256 --cout 256 --k 3 --p 1 --hw 14"; do
  echo "== $spec"; timeout 60 python tools/op_bench.py $spec --runs 10
done
timeout 120 ncu --set full --clock-control none --import-source on -k regex:"op_kernel$" -s 2 -c 1 -o gpurun_out/op_r18_20 python tools/op_bench.py --cin 512 --cout 512 --k 3 --p 1 --hw 7 --runs 3 > /dev/null 2>&1
timeout 120 ncu --set full --clock-control none --import-source on -k regex:"op_kernel$" -s 2 -c 1 -o gpurun_out/op_mb_47 python tools/op_bench.py --cin 960 --cout 160 --k 1 --p 0 --hw 7 --runs 3 > /dev/null 2>&1
ls gpurun_out
