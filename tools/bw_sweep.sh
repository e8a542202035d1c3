cd $GRAFT_REPO_ROOT
for r in 1 2; do for b in 160000 80000 50000; do
  echo "== bpus $b round $r"
  MT_TMA_BPUS=$b timeout 300 python tools/partition_ab.py --configs c2,c3,c4,c4b8 --runs 8 --modes 0:2:0,1:2:0,1:2:3,1:2:2 2>&1 | grep all_concurrent | cut -c 1-120
done; done
