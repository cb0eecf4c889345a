cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
VARIANTS="v_base v_nb3 v_poly64_3 v_base v_nb3 v_poly64_3" WORKLOADS="C3 C4-64-4096-c C4-64-16384-nc C4-64-1024-nc" TAG=r02_d64 BENCH_ARGS="--no-secondary --no-dropin" bash scripts/ab.sh 2>/dev/null
