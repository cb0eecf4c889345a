# A/B of k1_mean_and_q with K partials ordered after all Q chunks (SAB_K1_KLAST) on C2/C3, then the GPU suite.
mkdir -p gpurun_out/klast
for w in C2 C3; do
  for r in 1 0 1 0; do
    SAB_K1_KLAST=$r timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 3 \
      >> gpurun_out/klast/${w}_klast$r.jsonl 2>>gpurun_out/klast/err.log
  done
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/klast/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/klast/pytest_gpu.log
