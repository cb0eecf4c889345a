# k1_fused (one ticketed launch) vs the two-launch K1: GPU tests, then interleaved bench A/B.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_k1_fused.py tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -q -x > gpurun_out/k1f_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/k1f_pytest.log
tail -5 gpurun_out/k1f_pytest.log
for rep in 1 2; do
for mode in "SAB_K1_FUSED=1" "SAB_K1_FUSED=0" ${EXTRA_MODES}; do
  WL=("C4-128-16384-nc" "C2" "C2 --shard-of 8" "C4-128-1024-c" "C4-64-1024-nc" "C4-128-2048-c" "C3")
  for w in "${WL[@]}"; do
    env $mode timeout 180 python bench.py --workload $w --steps 20 --warmup 5 --e2e-steps 2 --no-cpu-baseline > /tmp/b.log 2>&1
    echo "$mode $w rc=$? $(python3 -c "
import json
l=[x for x in open('/tmp/b.log') if x.startswith('{')]
d=json.loads(l[0]) if l else None
print('NA' if d is None else '%.1f ms=%.4f k2ms=%.4f k1ms=%.4f k1frac=%.3f mhz=%s' % (d['value'], d['ms_per_step'], d['roofline']['ms_per_launch'], d['roofline_k1']['ms_per_step'], d['roofline_k1']['frac'], d['clocks']['sm_mhz']))
")" | tee -a gpurun_out/k1f_ab.txt
  done
done
done
