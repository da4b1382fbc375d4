cd ${GRAFT_REPO_ROOT:-.}
TAG=$1; RE=$2
timeout 120 python scripts/tc_probe.py > gpurun_out/tc_probe_$TAG.log 2>&1; echo probe rc $?; tail -3 gpurun_out/tc_probe_$TAG.log
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on \
  -k regex:"$RE" -s 1 -c 1 -o gpurun_out/prof_$TAG python bench.py --profile-only --steps 1 --warmup 0 > gpurun_out/ncu_$TAG.log 2>&1
echo ncu rc $?; tail -2 gpurun_out/ncu_$TAG.log
