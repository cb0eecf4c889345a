# BASELINE configs[3]: the kernel-bench sweep B=4, H=32, d in {64,128}, N in 1K..32K, causal and not.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for d in 64 128; do for n in 1024 2048 4096 8192 16384 32768; do for c in nc c; do
  w=C4-$d-$n-$c
  timeout 200 python bench.py --workload $w --steps 10 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/${TAG:-sw}_$w.json 2>/dev/null
done; done; done
