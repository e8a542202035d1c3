cd $GRAFT_REPO_ROOT
for r in 1 2; do for v in 1.0 0.7 1.5 2.0; do
  echo "== scale $v round $r"
  MT_SM_AVAIL_SCALE=$v timeout 300 python tools/partition_ab.py --configs c2,c3,c4,c4b8 --runs 8 --modes 1:2:3,1:2:0,1:2:2 2>&1 | grep all_concurrent | cut -c 1-90
done; done
