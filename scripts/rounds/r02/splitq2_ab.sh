# Split-Q K1 with the mean-partials grid held to 3 or 4 CTAs/SM (v_pm3 / v_pm4) vs the default two launches (v_base).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cp paper_2410_02367_b200/libsageattn_b200.so /tmp/lib_orig.so
for rep in 1 2; do for v in v_base v_pm4 v_pm3; do
  cp paper_2410_02367_b200/$v.so paper_2410_02367_b200/libsageattn_b200.so
  m=1; [ $v = v_base ] && m=0
  for w in C2 C3 C4-128-16384-nc C4-128-1024-c C4-128-4096-nc; do
    SAB_K1_SPLITQ=$m timeout 180 python bench.py --workload $w --steps 20 --warmup 5 --e2e-steps 1 --no-cpu-baseline --no-dropin --no-secondary > /tmp/b.log 2>&1
    echo "$v splitq=$m $w rc=$? $(python3 -c "
import json
l=[x for x in open('/tmp/b.log') if x.startswith('{')]
d=json.loads(l[0]) if l else None
print('NA' if d is None else '%.1f ms=%.4f k2ms=%.4f k1ms=%.4f k1frac=%.3f mhz=%s' % (d['value'], d['ms_per_step'], d['roofline']['ms_per_launch'], d['roofline_k1']['ms_per_step'], d['roofline_k1']['frac'], d['clocks']['sm_mhz']))
")" | tee -a gpurun_out/splitq2_ab.txt
  done
done; done
cp /tmp/lib_orig.so paper_2410_02367_b200/libsageattn_b200.so
