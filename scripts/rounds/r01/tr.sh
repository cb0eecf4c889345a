# Parity of the current build, then a SAB_TRACE timeline of one CTA per workload.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${TAG:-t}
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
for w in ${WORKLOADS:-C2}; do
timeout 120 python bench.py --workload $w --steps 20 --warmup 5 --e2e-steps 2 --no-cpu-baseline > gpurun_out/${TAG}_bench_$w.json 2>/dev/null
done
cp paper_2410_02367_b200/libsab_trace.so paper_2410_02367_b200/libsageattn_b200.so
for w in ${WORKLOADS:-C2}; do for c in ${CTAS:-0 300}; do
  timeout 120 python scripts/trace_k2.py $w $c gpurun_out/${TAG}_trace_${w}_$c.npy
done; done
tail -2 gpurun_out/${TAG}_pytest.log
