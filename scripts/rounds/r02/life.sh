cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cp paper_2410_02367_b200/libsageattn_b200.so /tmp/orig.so
cp paper_2410_02367_b200/libsab_trace.so paper_2410_02367_b200/libsageattn_b200.so
for spec in "C4-128-1024-c 0" "C4-128-1024-c 300" "C4-128-1024-c 511" "C2 0 x 4" "C2 100 x 4" "C2 180 x 4" "C4-128-16384-nc 5000" "C4-64-1024-nc 200"; do
  set -- $spec
  out=gpurun_out/r02_life_$1_$2.npy
  if [ -n "$4" ]; then timeout 120 python scripts/trace_k2.py $1 $2 $out $4; else timeout 120 python scripts/trace_k2.py $1 $2 $out; fi > /dev/null 2>&1
  echo "== $spec"; python scripts/trace_life.py $out
done > gpurun_out/r02_life.txt 2>&1
cp /tmp/orig.so paper_2410_02367_b200/libsageattn_b200.so
cat gpurun_out/r02_life.txt
