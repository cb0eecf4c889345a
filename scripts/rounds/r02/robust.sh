cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SAB_K2_PERSIST=1 timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02_robust_p1.log 2>&1; echo "persist=1 rc=$?" >> gpurun_out/r02_robust_p1.log
SAB_K2_PERSIST=0 timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02_robust_p0.log 2>&1; echo "persist=0 rc=$?" >> gpurun_out/r02_robust_p0.log
tail -3 gpurun_out/r02_robust_p1.log gpurun_out/r02_robust_p0.log
