# K1 partial-CTA size: nodes 32 vs 64 per CTA, 64- vs 80-register cap for the G >= 2 variants.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cp paper_2410_02367_b200/libsageattn_b200.so /tmp/lib_orig.so
SAB_K1_NODES=64 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "prepass_bit_exact or fixtures" > gpurun_out/nodes64_pytest.log 2>&1; echo "nodes=64 pytest rc=$?" | tee -a gpurun_out/nodes2_ab.txt
for rep in 1 2; do for v in v_base v_minb3; do for nd in 32 64; do
  cp paper_2410_02367_b200/$v.so paper_2410_02367_b200/libsageattn_b200.so
  for w in C4-128-1024-c C4-64-1024-nc C2 C3 C4-128-16384-nc; do
    SAB_K1_NODES=$nd timeout 180 python bench.py --workload $w --steps 20 --warmup 5 --e2e-steps 1 --no-cpu-baseline --no-dropin --no-secondary > /tmp/b.log 2>&1
    echo "$v nodes=$nd $w rc=$? $(python3 -c "
import json
l=[x for x in open('/tmp/b.log') if x.startswith('{')]
d=json.loads(l[0]) if l else None
print('NA' if d is None else '%.1f ms=%.4f k2ms=%.4f k1ms=%.4f k1frac=%.3f mhz=%s' % (d['value'], d['ms_per_step'], d['roofline']['ms_per_launch'], d['roofline_k1']['ms_per_step'], d['roofline_k1']['frac'], d['clocks']['sm_mhz']))
")" | tee -a gpurun_out/nodes2_ab.txt
  done
done; done; done
cp /tmp/lib_orig.so paper_2410_02367_b200/libsageattn_b200.so
