# usage (GPU box): bash scripts/gpu_pair_prof.sh TAG — iteration-0 contraction: SM-pair kernel vs single-CTA kernel
cd ${GRAFT_REPO_ROOT:-.}
TAG=${1:-pp}
mkdir -p gpurun_out
for P in 1 0; do
  CVB_TC_PAIRS=$P timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-compare > gpurun_out/pp_$P.json 2>/dev/null
  python -c "
import json,statistics; d=json.loads(open('gpurun_out/pp_$P.json').read().strip().splitlines()[-1]); k=d['kernel_ms']
print('pairs=$P', d['value'], 'contract it0 %.3f warm %.4f gather %.4f' % (k['contract_ms'][0], statistics.mean(k['contract_ms'][1:]), statistics.mean(k['gather_ms'][1:])))"
done
timeout 600 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:"pair_contract_kernel" -c 1 \
  -o gpurun_out/prof_pair_$TAG python bench.py --profile-only --steps 1 --warmup 0 > gpurun_out/ncu_pair_$TAG.log 2>&1
echo ncu rc $?
