cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu1_smi.txt 2>&1
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/gpu1_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/gpu1_smoke.log
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "prepass or int32" > gpurun_out/gpu1_pytest_a.log 2>&1; echo "rc=$?" >> gpurun_out/gpu1_pytest_a.log
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q > gpurun_out/gpu1_pytest_b.log 2>&1; echo "rc=$?" >> gpurun_out/gpu1_pytest_b.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/gpu1_bench.log 2>&1; echo "rc=$?" >> gpurun_out/gpu1_bench.log
tail -5 gpurun_out/gpu1_smoke.log gpurun_out/gpu1_pytest_a.log gpurun_out/gpu1_pytest_b.log gpurun_out/gpu1_bench.log
