cd $GRAFT_REPO_ROOT
export VARIANTS="v_rot0 v_rot2 v_rot8 v_rot10 v_rot0 v_rot2 v_rot8 v_rot10" WORKLOADS="C3 C2"
TAG=r02_rot BENCH_ARGS="--no-secondary --no-dropin" bash scripts/ab.sh
