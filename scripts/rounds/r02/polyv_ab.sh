cd $GRAFT_REPO_ROOT
export VARIANTS="v_p0 v_p2 v_p4 v_p0 v_p2 v_p4" WORKLOADS="C2 C3"
TAG=r02_polyv_vb BENCH_ARGS="--variant VB --no-secondary --no-dropin" bash scripts/ab.sh
TAG=r02_polyv_vt BENCH_ARGS="--variant VT --no-secondary --no-dropin" bash scripts/ab.sh
cp paper_2410_02367_b200/v_p2.so paper_2410_02367_b200/libsageattn_b200.so
timeout 600 python -m pytest tests/test_gpu_variant_vb.py tests/test_gpu_variant_t.py -x -q -m gpu -k "not nothing" > gpurun_out/r02_polyv_tests.log 2>&1; echo rc=$? >> gpurun_out/r02_polyv_tests.log
