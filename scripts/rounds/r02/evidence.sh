# Round-2 evidence pass (one GPU): headline bench line, reference arm, per-config lines,
# strong-scaling shard probes, ncu launch list and ncu --set full of K2 / K1 at the headline.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=r02
B="--no-cpu-baseline --no-dropin --no-secondary"
timeout 600 python bench.py > gpurun_out/${T}_bench_default.json 2> gpurun_out/${T}_bench_default.err
timeout 400 python bench.py --impl reference > gpurun_out/${T}_bench_reference.json 2>&1
for w in C2 C3 C5 C4-64-16384-nc C4-128-1024-c C4-64-1024-nc C4-128-32768-c; do
  timeout 400 python bench.py --workload $w $B > gpurun_out/${T}_bench_$w.json 2>&1
done
for sh in 8 4 2; do timeout 200 python bench.py --workload C2 --shard-of $sh $B > gpurun_out/${T}_bench_C2_shard$sh.json 2>&1; done
for v in T VB VT; do timeout 300 python bench.py --workload C2 --variant $v $B > gpurun_out/${T}_bench_${v}_C2.json 2>&1; done
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/${T}_launches_C4-128-16384-nc.csv python bench.py --steps 3 --warmup 1 --e2e-steps 1 $B > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k2_attention -s 2 -c 1 -o gpurun_out/${T}_k2_C4-128-16384-nc python bench.py --steps 2 --warmup 1 --e2e-steps 1 $B > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_ -s 2 -c 2 -o gpurun_out/${T}_k1_C4-128-16384-nc python bench.py --steps 2 --warmup 1 --e2e-steps 1 $B > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k2_attention -s 2 -c 1 -o gpurun_out/${T}_k2_C2_shard8 python bench.py --workload C2 --shard-of 8 --steps 2 --warmup 1 --e2e-steps 1 $B > /dev/null 2>&1
ls gpurun_out | grep ${T}_ | head -50
