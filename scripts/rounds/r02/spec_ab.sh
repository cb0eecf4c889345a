cd $GRAFT_REPO_ROOT
export VARIANTS="v_base v_spec v_base v_spec" WORKLOADS="C3 C2 C4-64-16384-nc C4-128-16384-nc"
TAG=r02_spec BENCH_ARGS="--no-secondary --no-dropin" bash scripts/ab.sh
