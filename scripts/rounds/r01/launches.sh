cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 20 --csv --log-file gpurun_out/${TAG:-l}_launches_${WORKLOAD:-C2}.csv python bench.py --workload ${WORKLOAD:-C2} --steps 3 --warmup 1 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1; echo "rc=$?"
