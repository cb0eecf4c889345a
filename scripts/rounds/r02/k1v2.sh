cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_split.py tests/test_gpu_pdl.py -m gpu -q -x > gpurun_out/r02_k1v2b_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_k1v2b_pytest.log
tail -3 gpurun_out/r02_k1v2b_pytest.log
for leg in 0; do
for w in "C2 --shard-of 8" "C2" "C4-128-1024-c" "C4-64-1024-nc" "C3" "C4-128-16384-nc" "C4-128-4096-nc"; do
  SAB_K1_LEGACY=$leg timeout 200 python bench.py --workload $w --steps 20 --warmup 5 --e2e-steps 2 --no-cpu-baseline --no-secondary --no-dropin > /tmp/s.json 2>&1
  python3 -c "
import json
l=[x for x in open('/tmp/s.json') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('legacy=$leg $w', 'NA' if d is None else '%.1f ms=%.4f k2ms=%.4f k1ms=%.4f k1frac=%.3f mhz=%s' % (d['value'], d['ms_per_step'], d['roofline']['ms_per_launch'], d['roofline_k1']['ms_per_step'], d['roofline_k1']['frac'], d['clocks']['sm_mhz']))
" | tee -a gpurun_out/r02_k1v2b_ab.txt
done
done
