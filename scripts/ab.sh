# A/B timing of alternative library builds: for each paper_2410_02367_b200/<name>.so in $VARIANTS,
# swap it in and run the bench for each workload in $WORKLOADS.  Tight timeouts.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-ab}
cp paper_2410_02367_b200/libsageattn_b200.so /tmp/lib_orig.so
for v in $VARIANTS; do
  cp paper_2410_02367_b200/$v.so paper_2410_02367_b200/libsageattn_b200.so
  for w in ${WORKLOADS:-C2}; do
    timeout 120 python bench.py $BENCH_ARGS --workload $w --steps 20 --warmup 5 --e2e-steps 2 --no-cpu-baseline > /tmp/b.log 2>&1
    echo "$v $w rc=$? $(python3 -c "
import json,sys
l=[x for x in open('/tmp/b.log') if x.startswith('{')]
d=json.loads(l[0]) if l else None
print('NA' if d is None else '%.1f k2=%.1f k2ms=%.4f k1ms=%.4f mhz=%s' % (d['value'], d['roofline']['achieved'], d['roofline']['ms_per_launch'], d['roofline_k1']['ms_per_step'], d['clocks']['sm_mhz']))
")" | tee -a gpurun_out/${TAG}_ab.txt
  done
done
cp /tmp/lib_orig.so paper_2410_02367_b200/libsageattn_b200.so
