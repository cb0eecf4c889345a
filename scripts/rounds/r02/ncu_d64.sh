cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B="--no-cpu-baseline --no-secondary --no-dropin"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k2_attention -s 2 -c 1 -o gpurun_out/r02_k2_C3 python bench.py --workload C3 --steps 2 --warmup 1 --e2e-steps 1 $B > gpurun_out/r02_ncu_c3.log 2>&1
echo rc=$? >> gpurun_out/r02_ncu_c3.log
