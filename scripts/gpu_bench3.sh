# three short C4 bench runs (value + per-kernel means)
cd ${GRAFT_REPO_ROOT:-.}
for i in 1 2 3; do
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-compare > gpurun_out/b3_$i.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/b3_$i.json')); k=d['kernel_ms']
print('ms/iter', d['value'], 'contract it0 %.3f warm %.3f gather %.3f' % (k['contract_ms'][0], sum(k['contract_ms'][1:])/11, sum(k['gather_ms'])/12))"
done
