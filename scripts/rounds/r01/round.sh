# Full evidence pass on one B200: tests, bench (with CPU baseline), reference arm,
# 2-rank torchrun functional run, ncu launch list and full captures of K2 / K1.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-r01}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${T}_smi.txt 2>&1
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${T}_smoke.log
timeout 400 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest_gpu.log
timeout 300 python bench.py > gpurun_out/${T}_bench_default.json 2> gpurun_out/${T}_bench_default.err; echo "bench rc=$?" >> gpurun_out/${T}_bench_default.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${T}_bench_reference.json 2> gpurun_out/${T}_bench_reference.err; echo "ref rc=$?" >> gpurun_out/${T}_bench_reference.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/${T}_bench_2rank.json 2> gpurun_out/${T}_bench_2rank.err; echo "2rank rc=$?" >> gpurun_out/${T}_bench_2rank.err
for W in ${EXTRA_WORKLOADS:-C3 C4-128-16384-nc C4-64-16384-nc C4-128-4096-c}; do
  timeout 200 python bench.py --workload $W --steps 10 --warmup 3 --e2e-steps 2 --no-cpu-baseline > gpurun_out/${T}_bench_${W}.json 2>/dev/null
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/${T}_launches_C2.csv python bench.py --steps 3 --warmup 1 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1; echo "launches rc=$?"
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k2_attention -s 2 -c 1 -o gpurun_out/${T}_k2_C2 python bench.py --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1; echo "k2 prof rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k1_ -s 3 -c 3 -o gpurun_out/${T}_k1_C2 python bench.py --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1; echo "k1 prof rc=$?"
tail -2 gpurun_out/${T}_smoke.log; tail -3 gpurun_out/${T}_pytest_gpu.log
