cd $GRAFT_REPO_ROOT
MT_BN_MIN=16 timeout 400 python -m pytest tests/test_gpu_parity.py -x -q -k "teacher_forced and (c2 or c3) or invariance_c2" 2>&1 | tail -2
for r in 1 2; do for v in 32 16; do
  echo "== bn_min $v round $r"
  MT_BN_MIN=$v timeout 300 python tools/partition_ab.py --configs c2,c3,c4 --runs 8 --modes 1:2:3,1:2:0,1:2:2 2>&1 | grep all_concurrent | cut -c 1-90
done; done
