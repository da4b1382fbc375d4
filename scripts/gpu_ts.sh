cd ${GRAFT_REPO_ROOT:-.}
for M in "$@"; do
CVB_TC_DEBUG=$M timeout 300 python bench.py --profile-only --steps 1 --warmup 0 2> gpurun_out/ts_$M.log; echo rc $?
done
