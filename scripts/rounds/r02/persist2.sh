cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cp paper_2410_02367_b200/libsageattn_b200.so /tmp/orig.so
for rep in 1 2; do
for v in v_head v_new v_new0; do
  lib=$v; env=""; if [ $v = v_new0 ]; then lib=v_new; env="SAB_K2_PERSIST=0"; fi
  cp paper_2410_02367_b200/$lib.so paper_2410_02367_b200/libsageattn_b200.so
  for w in "C2" "C4-128-1024-c" "C3"; do
    env $env timeout 200 python bench.py --workload $w --steps 20 --warmup 5 --e2e-steps 2 --no-cpu-baseline --no-secondary --no-dropin > /tmp/s.json 2>&1
    python3 -c "
import json
l=[x for x in open('/tmp/s.json') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('$v $w', 'NA' if d is None else '%.1f k2=%.1f k2ms=%.4f mhz=%s' % (d['value'], d['roofline']['achieved'], d['roofline']['ms_per_launch'], d['clocks']['sm_mhz']))
" | tee -a gpurun_out/r02_persist2_ab.txt
  done
done
done
cp /tmp/orig.so paper_2410_02367_b200/libsageattn_b200.so
