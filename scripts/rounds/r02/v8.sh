cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02_v8_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_v8_pytest.log
tail -n 3 gpurun_out/r02_v8_pytest.log
cp paper_2410_02367_b200/libsageattn_b200.so /tmp/orig.so
for rep in 1 2; do
for v in v_prev v_new; do
  cp paper_2410_02367_b200/$v.so paper_2410_02367_b200/libsageattn_b200.so
  for w in "C4-128-1024-nc" "C4-128-1024-c" "C4-64-1024-nc" "C4-128-4096-nc" "C2" "C3"; do
    timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --e2e-steps 2 --no-cpu-baseline --no-secondary --no-dropin > /tmp/s.json 2>&1
    python3 -c "
import json
l=[x for x in open('/tmp/s.json') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('$v $w', 'NA' if d is None else '%.1f ms=%.4f k2=%.1f k2ms=%.4f mhz=%s' % (d['value'], d['ms_per_step'], d['roofline']['achieved'], d['roofline']['ms_per_launch'], d['clocks']['sm_mhz']))
" | tee -a gpurun_out/r02_v8_ab.txt
  done
done
done
cp /tmp/orig.so paper_2410_02367_b200/libsageattn_b200.so
