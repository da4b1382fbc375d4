# contraction knockout study: bench per CVB_TC_DEBUG mask (results are wrong by design for mask != 0)
cd ${GRAFT_REPO_ROOT:-.}
TAG=${1:-k}; shift
for M in "$@"; do
CVB_TC_DEBUG=$M timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-compare > gpurun_out/knock_${TAG}_$M.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/knock_${TAG}_$M.json'))
c=d['kernel_ms']['contract_ms']; print('mask $M contract it0 %.3f warm %.3f' % (c[0], sum(c[1:])/len(c[1:])))"
done
