# mean_partial: __threadfence by the 16 partial writers only (v_fence) vs all 256 threads (v_base).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_rope.py -m gpu -q -x > gpurun_out/fence_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/fence_pytest.log; tail -2 gpurun_out/fence_pytest.log
for rep in 1 2; do VARIANTS="v_base v_fence" WORKLOADS="C2 C3 C4-128-16384-nc C4-128-1024-c C4-64-1024-nc" BENCH_ARGS="--no-dropin --no-secondary" TAG=fence bash scripts/ab.sh; done
