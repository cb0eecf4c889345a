# K1 as (mean partials) -> (Q chunks, own grid) -> (K chunks) (SAB_K1_SPLITQ=1) vs the default two launches.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SAB_K1_SPLITQ=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -q -x > gpurun_out/splitq_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/splitq_pytest.log; tail -2 gpurun_out/splitq_pytest.log
for rep in 1 2; do for m in 0 1; do
  for w in C2 C3 C4-128-16384-nc C4-128-1024-c C4-64-1024-nc C4-128-4096-nc; do
    SAB_K1_SPLITQ=$m timeout 180 python bench.py --workload $w --steps 20 --warmup 5 --e2e-steps 1 --no-cpu-baseline --no-dropin --no-secondary > /tmp/b.log 2>&1
    echo "splitq=$m $w rc=$? $(python3 -c "
import json
l=[x for x in open('/tmp/b.log') if x.startswith('{')]
d=json.loads(l[0]) if l else None
print('NA' if d is None else '%.1f ms=%.4f k2ms=%.4f k1ms=%.4f k1frac=%.3f mhz=%s' % (d['value'], d['ms_per_step'], d['roofline']['ms_per_launch'], d['roofline_k1']['ms_per_step'], d['roofline_k1']['frac'], d['clocks']['sm_mhz']))
")" | tee -a gpurun_out/splitq_ab.txt
  done
done; done
