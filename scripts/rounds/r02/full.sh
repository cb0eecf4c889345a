cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02_full_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_full_pytest.log
tail -8 gpurun_out/r02_full_pytest.log
