cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_variant_vb.py tests/test_gpu_persist.py -m gpu -q > gpurun_out/r02_vbfold2_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_vbfold2_pytest.log
tail -n 2 gpurun_out/r02_vbfold2_pytest.log
VARIANTS="v_mid v_new v_mid v_new" WORKLOADS="C2" TAG=r02_vbfold2 BENCH_ARGS="--variant VB --no-secondary --no-dropin" bash scripts/ab.sh 2>/dev/null
VARIANTS="v_mid v_new" WORKLOADS="C2 C3" TAG=r02_vtfold2 BENCH_ARGS="--variant VT --no-secondary --no-dropin" bash scripts/ab.sh 2>/dev/null
VARIANTS="v_mid v_new" WORKLOADS="C3" TAG=r02_vbfold2 BENCH_ARGS="--variant VB --no-secondary --no-dropin" bash scripts/ab.sh 2>/dev/null
