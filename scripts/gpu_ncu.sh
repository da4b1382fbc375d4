# usage: bash scripts/gpu_ncu.sh TAG  — launch list of one C4 step + full capture of the top kernels
cd ${GRAFT_REPO_ROOT:-.}
TAG=${1:-r}
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --profile-only --steps 1 --warmup 0 > gpurun_out/ncu_list_$TAG.log 2>&1
echo list rc $?
timeout 900 $NCU --set full --clock-control none --import-source on \
  -k regex:"partial_sample_kernel|partial_contract_tc_kernel" -s 2 -c 2 \
  -o gpurun_out/prof_$TAG python bench.py --profile-only --steps 1 --warmup 0 > gpurun_out/ncu_full_$TAG.log 2>&1
echo full rc $?
tail -3 gpurun_out/ncu_full_$TAG.log
ls -la gpurun_out/
