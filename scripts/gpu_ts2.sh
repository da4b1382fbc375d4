cd ${GRAFT_REPO_ROOT:-.}
for M in "$@"; do
CVB_TC_DEBUG=$M CVB_TC_TS_FILE=gpurun_out/ts_$M.bin timeout 300 python bench.py --profile-only --steps 1 --warmup 0 --no-graph; echo rc $?
done
