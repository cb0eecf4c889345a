cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_split.py tests/test_gpu_configs.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/r02_split_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_split_pytest.log
tail -5 gpurun_out/r02_split_pytest.log
for sh in 8 4 2; do
  timeout 200 python bench.py --workload C2 --shard-of $sh --steps 20 --warmup 5 --e2e-steps 2 --no-cpu-baseline --no-secondary --no-dropin > gpurun_out/r02_c2_shard$sh.json 2>&1
  SAB_KV_SPLIT=0 timeout 200 python bench.py --workload C2 --shard-of $sh --steps 20 --warmup 5 --e2e-steps 2 --no-cpu-baseline --no-secondary --no-dropin > gpurun_out/r02_c2_shard${sh}_nosplit.json 2>&1
done
timeout 200 python bench.py --workload C2 --steps 20 --warmup 5 --e2e-steps 2 --no-cpu-baseline --no-secondary --no-dropin > gpurun_out/r02_c2_full.json 2>&1
for f in gpurun_out/r02_c2_*.json; do python3 -c "
import json,sys
l=[x for x in open('$f') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('$f', 'NA' if d is None else '%.1f ms=%.4f k2ms=%.4f k1ms=%.4f split=%s' % (d['value'], d['ms_per_step'], d['roofline']['ms_per_launch'], d['roofline_k1']['ms_per_step'], d['config'].get('kv_split')))
"; done
