cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k1_cluster -s 2 -c 1 -o gpurun_out/r02_k1cluster_C2 python bench.py --workload C2 --steps 2 --warmup 2 --e2e-steps 1 --no-cpu-baseline --no-secondary --no-dropin > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
