# Final round-2 evidence pass on HEAD (one GPU): smoke, full GPU suite, headline bench line
# (with e2e_dropin and the CPU baseline), reference arm, per-config / variant lines, ncu launch
# list and ncu --set full of K2 and K1 at the headline.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=r02f
B="--no-cpu-baseline --no-dropin --no-secondary"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/${T}_smi.txt 2>&1
timeout 180 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${T}_smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/${T}_bench_default.json 2> gpurun_out/${T}_bench_default.err
timeout 400 python bench.py --impl reference > gpurun_out/${T}_bench_reference.json 2>&1
for w in C2 C3 C5 C4-64-16384-nc C4-128-1024-c; do
  timeout 400 python bench.py --workload $w $B > gpurun_out/${T}_bench_$w.json 2>&1
done
for v in T VB VT; do timeout 300 python bench.py --workload C2 --variant $v $B > gpurun_out/${T}_bench_${v}_C2.json 2>&1; done
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k1_|k2_" -c 40 --csv --log-file gpurun_out/${T}_launches_C4-128-16384-nc.csv python bench.py --steps 3 --warmup 1 --e2e-steps 1 $B > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k2_attention -s 2 -c 1 -o gpurun_out/${T}_k2_C4-128-16384-nc python bench.py --steps 2 --warmup 1 --e2e-steps 1 $B > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_ -s 2 -c 2 -o gpurun_out/${T}_k1_C4-128-16384-nc python bench.py --steps 2 --warmup 1 --e2e-steps 1 $B > /dev/null 2>&1
tail -3 gpurun_out/${T}_smoke.log; tail -3 gpurun_out/${T}_pytest_gpu.log
ls gpurun_out | grep ${T}_ | head -50
