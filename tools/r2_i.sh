# round-2 evidence, part 1: full GPU test suite, default bench line, reference arm
cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
nproc > gpurun_out/r2i_host.txt; lscpu | grep -E "Model name|^CPU\(s\)|Thread" >> gpurun_out/r2i_host.txt
( time timeout 1500 python -m pytest tests -m gpu -x -q --durations=10 ) > gpurun_out/r2i_gputests.log 2>&1
( time timeout 900 python bench.py ) > gpurun_out/r2i_bench.json 2> gpurun_out/r2i_bench.err
( time timeout 600 python bench.py --impl reference --steps 3 --warmup 1 ) > gpurun_out/r2i_ref.json 2> gpurun_out/r2i_ref.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2i_smoke.log 2>&1
tail -15 gpurun_out/r2i_gputests.log; tail -3 gpurun_out/r2i_bench.err; head -c 1500 gpurun_out/r2i_bench.json; tail -3 gpurun_out/r2i_ref.err; cat gpurun_out/r2i_smoke.log
