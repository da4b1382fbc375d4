# usage: bash scripts/gpu_ncu.sh TAG — full bench line, launch list of one C4 step, full capture of the top kernels
cd ${GRAFT_REPO_ROOT:-.}
TAG=${1:-r}
NCU=/usr/local/cuda/bin/ncu
timeout 900 python bench.py > gpurun_out/bench_full_$TAG.json 2> gpurun_out/bench_full_$TAG.err; echo bench rc $?
tail -c 600 gpurun_out/bench_full_$TAG.json
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --profile-only --steps 1 --warmup 0 > gpurun_out/ncu_list_$TAG.log 2>&1
echo list rc $?
# iteration 1 (warm) of each top kernel: skip the first launch (iteration 0)
timeout 900 $NCU --set full --clock-control none --import-source on \
  -k regex:"partial_contract_tcp_kernel|gather_kernel" -s 2 -c 2 \
  -o gpurun_out/prof_$TAG python bench.py --profile-only --steps 1 --warmup 0 > gpurun_out/ncu_full_$TAG.log 2>&1
echo full rc $?
tail -3 gpurun_out/ncu_full_$TAG.log
ls -la gpurun_out/
