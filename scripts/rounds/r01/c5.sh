cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "sampled_tiles_large" > gpurun_out/${TAG}_pytest_large.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest_large.log
timeout 600 python bench.py --workload C5 --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/${TAG}_bench_C5.json 2> gpurun_out/${TAG}_bench_C5.err; echo "rc=$?" >> gpurun_out/${TAG}_bench_C5.err
timeout 300 python bench.py --workload C5 --scaling strong --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1
tail -3 gpurun_out/${TAG}_pytest_large.log; tail -2 gpurun_out/${TAG}_bench_C5.err
