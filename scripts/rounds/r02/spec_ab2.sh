cd $GRAFT_REPO_ROOT
export VARIANTS="v_base v_base1 v_spec1 v_base v_base1 v_spec1" WORKLOADS="C3 C2 C4-128-16384-nc"
TAG=r02_spec2 BENCH_ARGS="--no-secondary --no-dropin" bash scripts/ab.sh
