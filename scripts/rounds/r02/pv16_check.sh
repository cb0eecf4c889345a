# Binary16 P~V accumulator arm: parity tests, then fp32 vs fp16 accumulator A/B.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pv16.py -x -q -s -m gpu > gpurun_out/r02_pv16_tests.log 2>&1; echo rc=$? >> gpurun_out/r02_pv16_tests.log
for rep in 1 2; do
  for acc in fp32 fp16; do
    for w in C4-128-16384-nc C2; do
      timeout 180 python bench.py --workload $w --pv-accum $acc --steps 20 --warmup 5 --e2e-steps 2 --no-cpu-baseline --no-secondary --no-dropin > /tmp/b.log 2>&1
      echo "$acc $w rc=$? $(python3 -c "
import json
l=[x for x in open('/tmp/b.log') if x.startswith('{')]
d=json.loads(l[0]) if l else None
print('NA' if d is None else '%.1f k2=%.1f k2ms=%.4f mhz=%s reasons=%s' % (d['value'], d['roofline']['achieved'], d['roofline']['ms_per_launch'], d['clocks']['sm_mhz'], d['clocks'].get('reasons')))
")" | tee -a gpurun_out/r02_pv16_ab.txt
    done
  done
done
