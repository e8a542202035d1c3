cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
for c in r50 mbv2; do timeout 300 python tools/trace_exec.py --config $c --partition 1 --out gpurun_out/r2o_trace_$c.json > gpurun_out/r2o_trace_$c.txt 2>&1; done
rm -f gpurun_out/*_raw.npy
tail -3 gpurun_out/r2o_trace_r50.txt
