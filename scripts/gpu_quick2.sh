# quick A/B: gpu tests with the fast gather on, then bench with gather fast on/off
cd ${GRAFT_REPO_ROOT:-.}
TAG=${1:-q}
CVB_GATHER_FAST=1 timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo pytest rc $?; tail -3 gpurun_out/pytest_gpu_$TAG.log
for G in 1 0; do
CVB_GATHER_FAST=$G timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-compare > gpurun_out/bench_${TAG}_g$G.json 2> gpurun_out/bench_${TAG}_g$G.err; echo bench rc $?
python -c "
import json; d=json.load(open('gpurun_out/bench_${TAG}_g$G.json'))
print('G=$G ms/iter', d['value'])
print('contract', d['kernel_ms']['contract_ms']); print('gather', d['kernel_ms']['gather_ms'])"
done
