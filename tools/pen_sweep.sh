cd $GRAFT_REPO_ROOT
for r in 1 2; do for p in 0 0.2 0.5 1.0; do
  echo "== pen $p round $r"
  MT_TILE_PEN=$p timeout 300 python tools/partition_ab.py --configs c2,c3,c4 --runs 8 --modes 1:2:3,1:2:0,1:2:2 2>&1 | grep all_concurrent | cut -c 1-100
done; done
