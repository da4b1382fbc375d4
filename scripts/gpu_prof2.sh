# usage (GPU box): bash scripts/gpu_prof2.sh TAG — bench lines (C4 full, C1-C3, C5 sweep), launch list, ncu full of the top kernels
cd ${GRAFT_REPO_ROOT:-.}
TAG=${1:-p}
NCU=/usr/local/cuda/bin/ncu
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_full_$TAG.json 2> gpurun_out/bench_full_$TAG.err; echo bench rc $?
tail -c 400 gpurun_out/bench_full_$TAG.json
for C in C1 C2 C3; do
  timeout 600 python bench.py --config $C --no-cpu-baseline > gpurun_out/bench_${C}_$TAG.json 2> gpurun_out/bench_${C}_$TAG.err; echo $C rc $?
done
for B in 8 16 32 64; do
  timeout 900 python bench.py --config C5 --batch $B --steps 3 --warmup 3 > gpurun_out/bench_C5b${B}_$TAG.json 2> gpurun_out/bench_C5b${B}_$TAG.err; echo C5 $B rc $?
  cut -c1-400 gpurun_out/bench_C5b${B}_$TAG.json
done
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --profile-only --steps 1 --warmup 0 > gpurun_out/ncu_list_$TAG.log 2>&1
echo list rc $?
timeout 900 $NCU --set full --clock-control none --import-source on \
  -k regex:"partial_contract_tcp_kernel|gather_fast_kernel" -s 2 -c 4 \
  -o gpurun_out/prof_$TAG python bench.py --profile-only --steps 1 --warmup 0 > gpurun_out/ncu_full_$TAG.log 2>&1
echo full rc $?
tail -3 gpurun_out/ncu_full_$TAG.log
