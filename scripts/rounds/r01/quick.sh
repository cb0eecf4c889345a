# Fast GPU sanity pass with tight timeouts (a hung kernel costs minutes, not the budget).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-q}
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; rc=$?; echo "smoke rc=$rc" >> gpurun_out/${TAG}_smoke.log
if [ $rc -ne 0 ]; then tail -5 gpurun_out/${TAG}_smoke.log; exit 1; fi
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 180 python bench.py --workload ${WORKLOAD:-C2} --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/${TAG}_bench.log
tail -2 gpurun_out/${TAG}_smoke.log; tail -3 gpurun_out/${TAG}_pytest.log; tail -2 gpurun_out/${TAG}_bench.log | cut -c1-400
