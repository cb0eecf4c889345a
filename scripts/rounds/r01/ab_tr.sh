# Parity of the current build, A/B of variant builds, then SAB_TRACE timelines.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${TAG:-x}
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
tail -2 gpurun_out/${TAG}_pytest.log
[ -n "$VARIANTS" ] && TAG=$TAG bash scripts/ab.sh
if [ -n "$TRACE" ]; then
cp paper_2410_02367_b200/libsab_trace.so paper_2410_02367_b200/libsageattn_b200.so
for w in $TRACE; do for c in ${CTAS:-0 700}; do
  timeout 120 python scripts/trace_k2.py $w $c gpurun_out/${TAG}_trace_${w}_$c.npy
done; done
fi
