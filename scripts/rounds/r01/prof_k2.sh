# ncu --set full of K2 only (one GPU), plus the launch list.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
W=${WORKLOAD:-C2}
TAG=${TAG:-p}
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k2_attention -s 2 -c 1 -o gpurun_out/${TAG}_k2_${W} python bench.py --workload $W --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/${TAG}_ncu.log 2>&1; echo "k2 prof rc=$?"
