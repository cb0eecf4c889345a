# ncu launch lists (per-launch gpu__time_duration of this library's kernels only) for the
# headline, C2 and the smallest C4 point; dram bytes per launch for the C4 N=1K K1 kernels.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B="--no-cpu-baseline --no-dropin --no-secondary --e2e-steps 1"
for w in C4-128-16384-nc C2 C4-128-1024-c; do
  timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k1_|k2_" -c 40 --csv --log-file gpurun_out/r02f_launches_$w.csv python bench.py --workload $w --steps 3 --warmup 3 $B > /dev/null 2>&1
done
timeout 400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k1_" -c 8 --csv --log-file gpurun_out/r02f_k1_small.csv python bench.py --workload C4-128-1024-c --steps 3 --warmup 3 $B > /dev/null 2>&1
ls -la gpurun_out | grep r02f_
