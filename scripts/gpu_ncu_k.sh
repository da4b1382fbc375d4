# usage: bash scripts/gpu_ncu_k.sh TAG REGEX [SKIP] — full ncu capture of one launch of kernels matching REGEX
cd ${GRAFT_REPO_ROOT:-.}
TAG=${1:-r}; RE=${2:-gather}; SKIP=${3:-1}
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on \
  -k regex:"$RE" -s $SKIP -c 1 -o gpurun_out/prof_$TAG python bench.py --profile-only --steps 1 --warmup 0 > gpurun_out/ncu_$TAG.log 2>&1
echo ncu rc $?; tail -2 gpurun_out/ncu_$TAG.log
