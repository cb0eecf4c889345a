cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SAB_K1_QPC=2 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -q -x > gpurun_out/r02_qpc_pytest.log 2>&1; echo "pytest qpc2 rc=$?" >> gpurun_out/r02_qpc_pytest.log
tail -n 2 gpurun_out/r02_qpc_pytest.log
for rep in 1 2; do
for q in 1 2; do
for w in "C4-128-1024-c" "C4-64-1024-nc" "C4-128-4096-nc" "C2" "C3" "C4-128-16384-nc"; do
  SAB_K1_QPC=$q timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --e2e-steps 2 --no-cpu-baseline --no-secondary --no-dropin > /tmp/s.json 2>&1
  python3 -c "
import json
l=[x for x in open('/tmp/s.json') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('qpc=$q $w', 'NA' if d is None else '%.1f ms=%.4f k2ms=%.4f k1ms=%.4f k1frac=%.3f' % (d['value'], d['ms_per_step'], d['roofline']['ms_per_launch'], d['roofline_k1']['ms_per_step'], d['roofline_k1']['frac']))
" | tee -a gpurun_out/r02_qpc_ab.txt
done
done
done
