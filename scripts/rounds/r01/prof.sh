# Profiling pass (one GPU): tests, bench, ncu launch list, ncu --set full of K2 and K1.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
W=${WORKLOAD:-C2}
TAG=${TAG:-r01}
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 300 python bench.py --workload $W --steps 20 --warmup 5 ${BENCH_ARGS:---no-cpu-baseline} > gpurun_out/${TAG}_bench_${W}.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_bench_${W}.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/${TAG}_launches_${W}.csv python bench.py --workload $W --steps 3 --warmup 1 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1; echo "launches rc=$?"
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k2_attention -s 2 -c 1 -o gpurun_out/${TAG}_k2_${W} python bench.py --workload $W --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1; echo "k2 prof rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k1_ -s 3 -c 3 -o gpurun_out/${TAG}_k1_${W} python bench.py --workload $W --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1; echo "k1 prof rc=$?"
tail -3 gpurun_out/${TAG}_pytest.log; tail -2 gpurun_out/${TAG}_bench_${W}.log
