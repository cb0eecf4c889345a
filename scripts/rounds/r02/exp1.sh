cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
# 1. trace of K2 on the headline point (two CTAs: first wave, mid-grid)
cp paper_2410_02367_b200/libsageattn_b200.so /tmp/lib_orig.so
cp paper_2410_02367_b200/libsab_trace.so paper_2410_02367_b200/libsageattn_b200.so
for c in 0 4000; do timeout 120 python scripts/trace_k2.py C4-128-16384-nc $c gpurun_out/r02_trace_c4_$c.npy; done
timeout 120 python scripts/trace_k2.py C4-128-8192-nc 2000 gpurun_out/r02_trace_c4n8k_2000.npy
cp /tmp/lib_orig.so paper_2410_02367_b200/libsageattn_b200.so
# 2. clock/power sensitivity of the exponential split
nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw,clocks_event_reasons.sw_power_cap --format=csv -lms 100 > gpurun_out/r02_exp1_smi.csv &
SMI=$!
VARIANTS="libsageattn_b200 v_poly0 v_poly4 libsageattn_b200" WORKLOADS="C4-128-16384-nc C4-64-16384-nc" TAG=r02_exp1 BENCH_ARGS="--no-secondary --no-dropin" bash scripts/ab.sh
kill $SMI
