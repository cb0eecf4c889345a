# Round evidence on one B200: smoke, GPU tests, bench lines for every config (default C2 with the
# CPU baseline, reference arm, 2-rank functional run), ncu launch list with DRAM bytes, ncu --set
# full of K2 and K1 on C2.  Outputs under gpurun_out/${TAG}_*.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T=${TAG:-r01}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > gpurun_out/${T}_smi.txt 2>&1
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${T}_smoke.log
timeout 500 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest_gpu.log
timeout 300 python bench.py > gpurun_out/${T}_bench_C2.json 2> gpurun_out/${T}_bench_C2.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${T}_bench_reference.json 2> gpurun_out/${T}_bench_reference.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/${T}_bench_C2_2rank_1gpu.json 2> gpurun_out/${T}_bench_2rank.err
for W in ${WORKLOADS:-C1 C3 C4-64-1024-nc C4-64-4096-c C4-64-16384-nc C4-64-32768-c C4-128-1024-c C4-128-4096-c C4-128-8192-nc C4-128-16384-nc C4-128-32768-c}; do
  timeout 200 python bench.py --workload $W --steps 10 --warmup 3 --e2e-steps 2 --no-cpu-baseline > gpurun_out/${T}_bench_${W}.json 2>/dev/null
done
timeout 600 python bench.py --workload C5 --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/${T}_bench_C5.json 2>/dev/null
for W in C2 C3 C4-128-16384-nc; do
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 12 --csv --log-file gpurun_out/${T}_launches_${W}.csv python bench.py --workload $W --steps 3 --warmup 1 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1
done
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k2_attention -s 2 -c 1 -o gpurun_out/${T}_k2_C2 python bench.py --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1; echo "k2 prof rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k1_ -s 2 -c 2 -o gpurun_out/${T}_k1_C2 python bench.py --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1; echo "k1 prof rc=$?"
tail -2 gpurun_out/${T}_smoke.log; tail -3 gpurun_out/${T}_pytest_gpu.log
