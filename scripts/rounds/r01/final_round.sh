# End-of-session evidence pass (one GPU): suite, smoke, bench lines, launch list, ncu of K2 and K1.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/fin
O=gpurun_out/fin
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout 400 python bench.py > $O/bench_C2.json 2> $O/bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2>> $O/bench.err
timeout 300 python bench.py --workload C3 --no-cpu-baseline > $O/bench_C3.json 2>> $O/bench.err
timeout 300 python bench.py --variant T --no-cpu-baseline > $O/bench_T_C2.json 2>> $O/bench.err
timeout 300 python bench.py --variant VB --no-cpu-baseline > $O/bench_VB_C2.json 2>> $O/bench.err
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file $O/launches_C2.csv python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1; echo "launches rc=$?"
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k2_attention -s 3 -c 1 -o $O/k2_C2 python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1; echo "k2 prof rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k1_ -s 6 -c 2 -o $O/k1_C2 python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1; echo "k1 prof rc=$?"
tail -n 2 $O/pytest_gpu.log
