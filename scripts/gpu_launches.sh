# usage: bash scripts/gpu_launches.sh TAG — ncu launch list (gpu__time_duration) of one C4 step
cd ${GRAFT_REPO_ROOT:-.}
TAG=${1:-r}
timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --profile-only --steps 1 --warmup 0 > gpurun_out/ncu_list_$TAG.log 2>&1
echo list rc $?
