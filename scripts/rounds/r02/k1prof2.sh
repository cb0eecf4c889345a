cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_ -s 2 -c 2 -o gpurun_out/r02_k1_C4-128-1024-c python bench.py --workload C4-128-1024-c --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline --no-secondary --no-dropin > /dev/null 2>&1
ls gpurun_out/*.ncu-rep | tail -2
