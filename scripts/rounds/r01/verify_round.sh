cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r01_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r01_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 300 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 300 python bench.py --variant VB --no-cpu-baseline > gpurun_out/bench_vb_c2.json 2> gpurun_out/bench_vb.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_vb.csv python bench.py --variant VB --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1
timeout 300 python bench.py --variant VT --no-cpu-baseline > gpurun_out/bench_vt_c2.json 2> gpurun_out/bench_vt.err
timeout 300 python bench.py --variant VB --workload C3 --no-cpu-baseline > gpurun_out/bench_vb_c3.json 2>> gpurun_out/bench_vb.err
