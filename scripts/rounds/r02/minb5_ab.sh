cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for rep in 1 2; do VARIANTS="v_base v_minb5" WORKLOADS="C2 C3 C4-128-16384-nc C4-128-1024-c C4-64-1024-nc" BENCH_ARGS="--no-dropin --no-secondary" TAG=minb5 bash scripts/ab.sh; done
