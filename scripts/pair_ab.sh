cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
cp paper_2410_02367_b200/libsageattn_b200.so /tmp/lib_orig.so
for v in $VARIANTS; do
  cp paper_2410_02367_b200/$v.so paper_2410_02367_b200/libsageattn_b200.so
  echo "== $v" >> gpurun_out/${TAG}.log
  timeout 120 python scripts/pair_dbg.py >> gpurun_out/${TAG}.log 2>&1; echo rc=$? >> gpurun_out/${TAG}.log
done
cp /tmp/lib_orig.so paper_2410_02367_b200/libsageattn_b200.so
