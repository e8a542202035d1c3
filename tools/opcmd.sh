cd $GRAFT_REPO_ROOT
for spec in "--cin 256 --cout 256 --k 3 --p 1 --hw 56 --batch 8" "--cin 512 --cout 512 --k 3 --p 1 --hw 28 --batch 8" "--cin 128 --cout 128 --k 3 --p 1 --hw 112 --batch 8" "--cin 64 --cout 256 --k 1 --p 0 --hw 56 --batch 8" "--cin 256 --cout 256 --k 3 --p 1 --hw 56 --batch 1"; do
  echo "== $spec"; timeout 120 python tools/op_bench.py $spec --runs 10 2>&1 | tail -4
done
