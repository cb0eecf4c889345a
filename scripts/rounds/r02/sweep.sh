# Round-2 evidence: headline bench line + reference arm, the full C4 kernel-bench sweep
# (BASELINE metric: TOPS vs seq len, d 64/128, causal and not), C2/C3/C5, variants, shards,
# ncu of K2 at the headline.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=r02g
B="--no-cpu-baseline --no-dropin --no-secondary"
timeout 600 python bench.py > gpurun_out/${T}_bench_C4-128-16384-nc.json 2> gpurun_out/${T}_bench_default.err
timeout 400 python bench.py --impl reference > gpurun_out/${T}_bench_reference.json 2>&1
for d in 64 128; do for n in 1024 2048 4096 8192 16384 32768; do for c in c nc; do
  timeout 400 python bench.py --workload C4-$d-$n-$c --steps 10 --warmup 3 --e2e-steps 2 $B > gpurun_out/${T}_sweep_C4-$d-$n-$c.json 2>&1
done; done; done
for w in C2 C3 C5; do timeout 400 python bench.py --workload $w $B > gpurun_out/${T}_bench_$w.json 2>&1; done
for sh in 8 4 2; do timeout 200 python bench.py --workload C2 --shard-of $sh $B > gpurun_out/${T}_bench_C2_shard$sh.json 2>&1; done
for v in T VB VT; do timeout 300 python bench.py --workload C2 --variant $v $B > gpurun_out/${T}_bench_${v}_C2.json 2>&1; done
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k1_|k2_" -c 40 --csv --log-file gpurun_out/${T}_launches_C2.csv python bench.py --workload C2 --steps 3 --warmup 1 --e2e-steps 1 $B > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k2_attention -s 2 -c 1 -o gpurun_out/${T}_k2_C4-128-16384-nc python bench.py --steps 2 --warmup 1 --e2e-steps 1 $B > /dev/null 2>&1
ls gpurun_out | grep ${T}_ | wc -l
