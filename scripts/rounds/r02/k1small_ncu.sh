# ncu --set full of both K1 kernels at the smallest C4 point (latency-bound K1).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B="--no-cpu-baseline --no-dropin --no-secondary --e2e-steps 1"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k1_mean_and_q|k1_k_fast" -s 4 -c 2 -o gpurun_out/r02f_k1_C4-128-1024-c python bench.py --workload C4-128-1024-c --steps 2 --warmup 3 $B > /dev/null 2>&1
ls -la gpurun_out | grep k1_C4
