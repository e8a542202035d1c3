cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python tools/ab.py --libs abl/A.so,abl/C4.so --configs c2,c4,c4b8 --rounds 2 --runs 20 --knobs "c2=1,3,2;c4=1,2,2;c4b8=1,2,2" > gpurun_out/r2l_ab_s2.txt 2>&1
for kn in "1,2,4" "1,0,4" "0,2,4" "1,3,4" "0,0,4"; do
  echo "knobs $kn" >> gpurun_out/r2l_ab_s4.txt
  timeout 600 python tools/ab.py --libs abl/C4.so --configs c2,c4,c4b8 --rounds 1 --runs 20 --knobs "$kn" >> gpurun_out/r2l_ab_s4.txt 2>&1
done
cat gpurun_out/r2l_ab_s2.txt gpurun_out/r2l_ab_s4.txt
