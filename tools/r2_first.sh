cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_smi.txt
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/r2a_gputests.log
timeout 600 python bench.py --config c4 --no-profile --steps 50 --warmup 5 > gpurun_out/r2a_bench_c4.json 2> gpurun_out/r2a_bench_c4.err
timeout 600 python bench.py --config c4b8 --no-profile --no-cpu --steps 30 --warmup 5 > gpurun_out/r2a_bench_c4b8.json 2> gpurun_out/r2a_bench_c4b8.err
cat gpurun_out/r2a_gputests.log; head -c 600 gpurun_out/r2a_bench_c4.json
