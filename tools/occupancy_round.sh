# per-tenant occupancy traces under the calibrated knobs + throughput-regime conv op spans
cd $GRAFT_REPO_ROOT
timeout 200 python tools/trace_exec.py --config c2 --partition 1 --claim 3 --out gpurun_out/occ_c2.json > gpurun_out/occ_c2.txt 2>&1
timeout 200 python tools/trace_exec.py --config c3 --partition 1 --claim 0 --out gpurun_out/occ_c3.json > gpurun_out/occ_c3.txt 2>&1
timeout 200 python tools/trace_exec.py --config c4 --partition 1 --claim 2 --out gpurun_out/occ_c4.json > gpurun_out/occ_c4.txt 2>&1
for spec in "--cin 256 --cout 256 --k 3 --p 1 --hw 56 --batch 8" "--cin 512 --cout 512 --k 3 --p 1 --hw 28 --batch 8" "--cin 128 --cout 128 --k 3 --p 1 --hw 112 --batch 8" "--cin 64 --cout 256 --k 1 --p 0 --hw 56 --batch 8"; do
  echo "== $spec"; timeout 120 python tools/op_bench.py $spec --runs 10 2>&1 | tail -4
done > gpurun_out/opbench_b8.txt
grep -h "^tenant\|^total\|SM-busy" gpurun_out/occ_c*.txt
cat gpurun_out/opbench_b8.txt
