# A/B of programmatic dependent launch (K1a -> K1b -> K2) on C2/C3, then the GPU suite.
mkdir -p gpurun_out/pdl
for w in C2 C3; do
  for pdl in 1 0 1 0; do
    SAB_PDL=$pdl timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 3 \
      >> gpurun_out/pdl/${w}_pdl$pdl.jsonl 2>>gpurun_out/pdl/err.log
  done
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pdl/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pdl/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/pdl/smoke.log 2>&1
