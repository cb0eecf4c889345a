cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for w in C4-128-16384-nc C2 C3 C4-128-1024-c; do
  echo "default $(timeout 300 python scripts/rounds/r02/e2e_probe.py $w 4 2>&1 | tail -1)" | tee -a gpurun_out/r02_e2e_final.txt
done
timeout 900 python -m pytest tests -q -x -m gpu -k "host or dropin or capi or dist or shard or vb or variant" > gpurun_out/r02_e2e_tests2.log 2>&1; echo rc=$? >> gpurun_out/r02_e2e_tests2.log
timeout 600 python bench.py > gpurun_out/r02_bench_default.json 2> gpurun_out/r02_bench_default.err; echo rc=$? >> gpurun_out/r02_bench_default.err
