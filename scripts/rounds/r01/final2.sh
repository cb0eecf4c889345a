cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/fin2; O=gpurun_out/fin2
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout 400 python bench.py > $O/bench_C2.json 2> $O/bench.err
timeout 400 python bench.py --workload C4-128-16384-nc --no-cpu-baseline --steps 10 --warmup 3 > $O/bench_C4-128-16384-nc.json 2>> $O/bench.err
