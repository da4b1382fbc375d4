# usage: bash scripts/gpu_round.sh TAG — probe, GPU tests, bench persistent vs non-persistent contraction
cd ${GRAFT_REPO_ROOT:-.}
TAG=${1:-q}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 180 python scripts/tc_probe.py > gpurun_out/tc_probe_$TAG.log 2>&1; echo probe rc $?; tail -6 gpurun_out/tc_probe_$TAG.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo pytest rc $?; tail -3 gpurun_out/pytest_gpu_$TAG.log
for P in 1 0; do
CVB_TC_PERSISTENT=$P timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-compare > gpurun_out/bench_${TAG}_p$P.json 2> gpurun_out/bench_${TAG}_p$P.err; echo bench p$P rc $?
python -c "
import json; d=json.load(open('gpurun_out/bench_${TAG}_p$P.json'))
print('ms/iter', d['value'], 'clocks', d['clocks'])
print('contract', d['kernel_ms']['contract_ms']); print('gather', d['kernel_ms']['gather_ms'])
print('roofline', d['roofline']['kernel'], d['roofline']['achieved'], d['roofline']['frac'])"
done
