# usage: bash scripts/gpu_profile_round.sh TAG — full bench line + ncu launch list + full captures
cd ${GRAFT_REPO_ROOT:-.}
TAG=${1:-r}
NCU=/usr/local/cuda/bin/ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python bench.py > gpurun_out/bench_full_$TAG.json 2> gpurun_out/bench_full_$TAG.err; echo bench rc $?
tail -c 400 gpurun_out/bench_full_$TAG.json
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --profile-only --steps 1 --warmup 0 > gpurun_out/ncu_list_$TAG.log 2>&1
echo list rc $?
# warm iteration (launch 2) of the contraction and the sampler; iteration 0 contraction; prep kernels
timeout 900 $NCU --set full --clock-control none --import-source on \
  -k regex:"partial_contract_tcp_kernel|gather_fast_kernel" -s 2 -c 2 \
  -o gpurun_out/prof_warm_$TAG python bench.py --profile-only --steps 1 --warmup 0 > gpurun_out/ncu_warm_$TAG.log 2>&1
echo warm rc $?
timeout 900 $NCU --set full --clock-control none --import-source on \
  -k regex:"partial_contract_tcp_kernel|split_f1_kernel|split_level_kernel|plan_kernel" -c 7 \
  -o gpurun_out/prof_cold_$TAG python bench.py --profile-only --steps 1 --warmup 0 > gpurun_out/ncu_cold_$TAG.log 2>&1
echo cold rc $?
ls -la gpurun_out/ | tail -5
