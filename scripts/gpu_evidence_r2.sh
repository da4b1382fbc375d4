# usage (GPU box): bash scripts/gpu_evidence_r2.sh TAG — round-2 (final build) evidence: launch list, full
# captures (C4 warm + cold, C1-C3 warm traffic, dense / on-demand / strict kernels), sanitizer
cd ${GRAFT_REPO_ROOT:-.}
TAG=${1:-e}
NCU=/usr/local/cuda/bin/ncu
mkdir -p gpurun_out
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --profile-only --steps 1 --warmup 0 > gpurun_out/ncu_list_$TAG.log 2>&1
echo list rc $?
timeout 900 $NCU --set full --clock-control none --import-source on \
  -k regex:"partial_contract_tcp_kernel|gather_fast_kernel" -s 2 -c 2 \
  -o gpurun_out/prof_warm_C4_$TAG python bench.py --profile-only --steps 1 --warmup 0 > gpurun_out/ncu_warm_C4_$TAG.log 2>&1
echo warm C4 rc $?
timeout 900 $NCU --set full --clock-control none --import-source on \
  -k regex:"pair_contract_kernel|split_f1_kernel|split_level_kernel|plan_kernel" -c 6 \
  -o gpurun_out/prof_cold_C4_$TAG python bench.py --profile-only --steps 1 --warmup 0 > gpurun_out/ncu_cold_C4_$TAG.log 2>&1
echo cold C4 rc $?
for C in C1 C2 C3; do
  timeout 900 $NCU --set full --clock-control none \
    -k regex:"partial_contract_tcp_kernel|gather_fast_kernel" -s 2 -c 2 \
    -o gpurun_out/prof_warm_${C}_$TAG python bench.py --config $C --profile-only --steps 1 --warmup 0 > gpurun_out/ncu_warm_${C}_$TAG.log 2>&1
  echo warm $C rc $?
done
timeout 900 $NCU --set full --clock-control none -k regex:"partial_contract_tcp_kernel" -c 1 \
  -o gpurun_out/prof_dense_C2_$TAG python scripts/prof_variants.py dense C2 > gpurun_out/ncu_dense_$TAG.log 2>&1
echo dense rc $?
timeout 900 $NCU --set full --clock-control none -k regex:"partial_contract_tcp_kernel|gather_fast_kernel" -s 4 -c 2 \
  -o gpurun_out/prof_ondemand_C4_$TAG python scripts/prof_variants.py ondemand C4 > gpurun_out/ncu_ondemand_$TAG.log 2>&1
echo ondemand rc $?
timeout 900 $NCU --set full --clock-control none -k regex:"lookup_on_demand_kernel" -c 1 \
  -o gpurun_out/prof_odffma_C4_$TAG python scripts/prof_variants.py ondemand_ffma C4 > gpurun_out/ncu_odffma_$TAG.log 2>&1
echo od_ffma rc $?
timeout 900 $NCU --set full --clock-control none -k regex:"partial_contract_kernel|gather_kernel" -s 2 -c 2 \
  -o gpurun_out/prof_strict_C4_$TAG python scripts/prof_variants.py partial C4 strict > gpurun_out/ncu_strict_$TAG.log 2>&1
echo strict rc $?
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 1200 $CS --tool $tool --error-exitcode 9 python scripts/sanitize_cases.py > gpurun_out/sanitize_${tool}_$TAG.log 2>&1
  echo "$tool rc $?"; grep -E "ERROR SUMMARY" gpurun_out/sanitize_${tool}_$TAG.log | head -2
done
ls gpurun_out/*.ncu-rep | tail -20
