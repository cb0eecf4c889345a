set -x
mkdir -p gpurun_out/ov
for g in off 4,28 8,24 2,30 16,16 4,8,20; do
  timeout 300 python bench.py --workload C2 --steps 20 --warmup 5 --groups $g --no-cpu-baseline --e2e-steps 3 > gpurun_out/ov/C2_$g.json 2>gpurun_out/ov/C2_$g.err
done
for g in off 8,52 4,56 15,45 30,30; do
  timeout 300 python bench.py --workload C3 --steps 10 --warmup 3 --groups $g --no-cpu-baseline --e2e-steps 3 > gpurun_out/ov/C3_$g.json 2>gpurun_out/ov/C3_$g.err
done
