# A/B of k1_k_fast's reversed unit/chunk walk on C2/C3, then the GPU suite.
mkdir -p gpurun_out/rev
for w in C2 C3; do
  for r in 1 0 1 0; do
    SAB_K1_REVERSE=$r timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 3 \
      >> gpurun_out/rev/${w}_rev$r.jsonl 2>>gpurun_out/rev/err.log
  done
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/rev/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/rev/pytest_gpu.log
