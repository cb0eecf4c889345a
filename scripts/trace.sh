cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cp paper_2410_02367_b200/libsab_trace.so paper_2410_02367_b200/libsageattn_b200.so
for c in ${CTAS:-0 300}; do
  timeout 120 python scripts/trace_k2.py ${WORKLOAD:-C2} $c gpurun_out/${TAG:-t}_trace_${WORKLOAD:-C2}_$c.npy
done
