# C4 kernel-bench sweep on HEAD (BASELINE metric: TOPS vs seq len, d 64/128, causal and not).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B="--no-cpu-baseline --no-dropin --no-secondary"
for d in 64 128; do for n in 1024 2048 4096 8192 16384 32768; do for c in c nc; do
  timeout 400 python bench.py --workload C4-$d-$n-$c --steps 10 --warmup 3 --e2e-steps 2 $B > gpurun_out/r02s_sweep_C4-$d-$n-$c.json 2>&1
done; done; done
ls gpurun_out | grep -c r02s_sweep
